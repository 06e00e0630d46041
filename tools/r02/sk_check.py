"""Stream-K DMMA MTTKRP: per-mode parity against the oracle on views that take
it (direct and tree plans), then per-pass timing at C2 / C3 (diagnostics)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

import paper_2001_04321_b200 as P  # noqa: E402
import pyoracle as O  # noqa: E402
from parity import rel_fro  # noqa: E402

for shape, rank in (([64, 48, 40], 20), ([40, 36, 34, 32], 16), ([120, 100, 80], 20), ([96, 80, 64], 32),
                    ([300, 300, 300], 20), ([100, 100, 100, 100], 16), ([70, 50, 48], 8), ([48, 40, 32], 24)):
    spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=0.01, seed=5)
    t, _ = P.generate(spec)
    init = P.random_init(shape, rank, P.stream_seed(5, 1))
    prov = P.GpuDenseProvider(t)
    want = [O.mttkrp(t, init.factors, m) for m in range(len(shape))]
    for flags in (0, P.RUN_DIRECT):
        got = prov.mttkrp_all(init, flags=flags)
        errs = [rel_fro(g, w) for g, w in zip(got, want)]
        print(shape, rank, "tree" if flags == 0 else "direct", " ".join(f"{e:.1e}" for e in errs),
              "OK" if max(errs) <= 1e-12 else "FAIL", flush=True)
    print("   plans:", [prov.mttkrp_plan(rank, m) for m in range(len(shape))], flush=True)
    prov.close()
