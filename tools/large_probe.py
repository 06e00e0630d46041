"""Bisect the size at which the FP32 r=64 MTTKRP identity breaks."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2001_04321_b200 as P

for shape in ([600, 600, 600], [1000, 1000, 1000], [1300, 1300, 1300], [2000, 2000, 600], [2000, 2000, 2000]):
    rank = 64
    spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=0.0, seed=105)
    t, truth = P.generate(spec, dtype=np.float32)
    a = [np.asarray(x) for x in truth.factors]
    prov = P.GpuDenseProvider(t)
    grams = [x.T @ x for x in a]
    errs = []
    for mode in range(3):
        h = np.ones((rank, rank))
        for j, g in enumerate(grams):
            if j != mode:
                h *= g
        want = a[mode] @ h
        got = prov.mttkrp(a, mode)
        errs.append(float(np.linalg.norm(got - want) / np.linalg.norm(want)))
    print(shape, t.size / 2**31, ["%.2e" % e for e in errs], [prov.mttkrp_plan(rank, m) for m in range(3)], flush=True)
    prov.close()
    del t
