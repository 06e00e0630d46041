"""Timing probe for the e2e path (upload + her_run) -- diagnostics only."""
import sys
import time

import numpy as np

sys.path.insert(0, '.')
import paper_2001_04321_b200 as P  # noqa: E402

spec = P.SyntheticSpec(shape=[300, 300, 300], rank=20, noise_sigma=0.0, seed=102)
t, truth = P.generate(spec)
init = P.random_init([300, 300, 300], 20, P.stream_seed(102, 1))
ctx = P.Context(0)
t = np.asarray(t)
flags = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for rep in range(6):
    a = time.perf_counter()
    prov = P.GpuDenseProvider(t, ctx, full_shape=[300, 300, 300])
    b = time.perf_counter()
    m, tr = P.her_run(prov, init, P.AoConfig(max_outer_iters=200, flags=flags), P.HerParams(), ctx=ctx)
    c = time.perf_counter()
    prov.close()
    d = time.perf_counter()
    print(f"rep {rep}: upload {1e3 * (b - a):.1f} ms, her_run {1e3 * (c - b):.1f} ms (device {tr.records[-1].time_s * 1e3:.1f}),"
          f" close {1e3 * (d - c):.1f} ms", flush=True)
