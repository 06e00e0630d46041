"""Timing probe for the e2e path (upload + her_run) -- diagnostics only.
usage: python tools/e2e_probe.py [iters] [flags]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_2001_04321_b200 as P  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
spec = P.SyntheticSpec(shape=[300, 300, 300], rank=20, noise_sigma=0.0, seed=102)
tg, truth = P.generate(spec)
init = P.random_init([300, 300, 300], 20, P.stream_seed(102, 1))
ctx = P.Context(0)
buf = torch.empty(tg.shape, dtype=torch.float64, pin_memory=True)
t = buf.numpy()
np.copyto(t, tg)
for rep in range(6):
    a = time.perf_counter()
    prov = P.GpuDenseProvider(t, ctx, full_shape=[300, 300, 300])
    b = time.perf_counter()
    m, tr = P.her_run(prov, init, P.AoConfig(max_outer_iters=iters, flags=flags), P.HerParams(), ctx=ctx)
    c = time.perf_counter()
    prov.close()
    d = time.perf_counter()
    print(f"rep {rep}: upload {1e3 * (b - a):.2f} ms, her_run {1e3 * (c - b):.2f} ms (run clock {tr.records[-1].time_s * 1e3:.2f}),"
          f" close {1e3 * (d - c):.2f} ms; total {1e3 * (c - a):.2f} ms -> {iters / (c - a):.0f} iters/s", flush=True)
