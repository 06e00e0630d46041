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


def run(prov, k, tag):
    a = time.perf_counter()
    m, tr = P.her_run(prov, init, P.AoConfig(max_outer_iters=k), P.HerParams(), ctx=ctx)
    b = time.perf_counter()
    sw = sum(r.inner_sweeps for r in tr.records)
    print(f"{tag}: her_run {k} iters {1e3 * (b - a):.1f} ms, sweeps {sw}, final f {tr.records[-1].f:.3e}, "
          f"trace time {tr.records[-1].time_s * 1e3:.1f} ms", flush=True)


prov = P.GpuDenseProvider(t, ctx)
run(prov, 200, "A1")
run(prov, 200, "A2")
run(prov, 200, "A3")
prov.close()
prov = P.GpuDenseProvider(t, ctx)
run(prov, 200, "B1")
run(prov, 200, "B2")

# the bench's sequence: a Session first, then the C-ABI driver
prov.close()
prov = P.GpuDenseProvider(t, ctx, full_shape=[300, 300, 300])
sess = P.Session(prov, init, P.AoConfig(max_outer_iters=10**6), P.HerParams(), algo="her")
sess.step(10)
sess.sync()
sess.step(200)
sess.sync()
sess.set_kernel_timing(True)
sess.step(200)
sess.sync()
sess.set_kernel_timing(False)
sess.close()
a = time.perf_counter()
prov2 = P.GpuDenseProvider(t, ctx, full_shape=[300, 300, 300])
b = time.perf_counter()
print(f"C upload {1e3 * (b - a):.1f} ms")
run(prov2, 200, "C1")
run(prov2, 200, "C2")
