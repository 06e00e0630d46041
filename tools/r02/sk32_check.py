"""FP32 stream-K MTTKRP: per-mode parity (1e-5 relative, the FP32 bar) against
the oracle on the float values upcast, tree and direct plans (diagnostics)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

import paper_2001_04321_b200 as P  # noqa: E402
import pyoracle as O  # noqa: E402
from parity import rel_fro  # noqa: E402

for shape, rank in (([96, 80, 64], 32), ([64, 48, 40], 20), ([128, 100, 96], 64), ([500, 100, 64], 32),
                    ([40, 36, 34, 32], 24)):
    spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=0.01, seed=5)
    t, _ = P.generate(spec, dtype=np.float32)
    init = P.random_init(shape, rank, P.stream_seed(5, 1))
    prov = P.GpuDenseProvider(t)
    want = [O.mttkrp(t, init.factors, m) for m in range(len(shape))]
    for flags in (0, P.RUN_DIRECT):
        got = prov.mttkrp_all(init, flags=flags)
        errs = [rel_fro(g, w) for g, w in zip(got, want)]
        print(shape, rank, "tree" if flags == 0 else "direct", " ".join(f"{e:.1e}" for e in errs),
              "OK" if max(errs) <= 1e-5 else "FAIL", flush=True)
    print("   plans:", [prov.mttkrp_plan(rank, m) for m in range(len(shape))], flush=True)
    prov.close()
