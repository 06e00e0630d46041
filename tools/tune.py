"""Per-mode MTTKRP kernel time of a BASELINE config through a solver session
(CUDA events around each launch), for plan tuning via NTF_FAST_* env vars."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2001_04321_b200 as P

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
shapes = {"c1": ([50, 50, 50], 10, np.float64), "c2": ([300, 300, 300], 20, np.float64),
          "c3": ([100, 100, 100, 100], 16, np.float64), "c4": ([500, 500, 500], 32, np.float32)}
shape, r, dt = shapes[cfg]
gen = np.random.default_rng(0)
t = gen.random(shape).astype(dt)
init = P.random_init(shape, r, 1)
prov = P.GpuDenseProvider(t)
s = P.Session(prov, init, P.AoConfig(max_outer_iters=10**6), P.HerParams())
s.step(2)
s.set_kernel_timing(True)
s.step(steps)
ms, cnt, _ = s.kernel_times()
per = [m / max(c, 1) for m, c in zip(ms, cnt)]
nbytes = P.mttkrp_bytes(shape, r, np.dtype(dt).itemsize)
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("NTF_FAST"))
print(cfg, env or "default", " ".join(f"{x*1e3:.1f}us" for x in per),
      " GB/s:", " ".join(f"{nbytes / (x / 1e3) / 1e9:.0f}" for x in per),
      " plans:", [prov.mttkrp_plan(r, m) for m in range(len(shape))][0])
s.set_kernel_timing(False)
tr = s.trace()
sw = [rec.inner_sweeps for rec in tr.records]
print(f"  inner sweeps/iteration: mean {np.mean(sw):.1f} max {max(sw)} over {len(sw)} iterations; "
      f"final f {tr.final_f():.3e}")
import ctypes as _C
from paper_2001_04321_b200 import _lib as _L
_buf = (_C.c_ulonglong * (8 + 384))()
if _L.lib().ntf_debug_nnls_prof(_buf, 1) == 0 and _buf[3]:
    loop, red, sw, calls, pc, npass, tri, _ = list(_buf)[:8]
    b = list(_buf)
    post, fin, fs = b[8:136], b[136:264], b[264:392]
    idx = [i for i in range(128) if post[i]]
    if idx:
        p0 = min(post[i] for i in idx)
        print("  pass-4 per warp (ns from first post): post / fin start / fin end")
        print("   " + " ".join(f"{post[i]-p0}/{fs[i]-p0}/{fin[i]-p0}" for i in idx[:24]))
    if os.environ.get("NTF_NNLS_OLD"):
        print(f"  nnls CTA0: {loop / calls:.0f} cyc/call, {sw / calls:.1f} sweeps/call, "
              f"{loop / max(sw, 1):.0f} cyc/sweep of which reduction {red / max(sw, 1):.0f}; "
              f"pass {pc / max(npass, 1):.0f} cyc (triangle {tri / max(npass, 1):.0f}), {npass / calls:.1f} passes/call")
    else:  # stream kernel: [0] loop, [1] prologue, [4] epilogue, [5] passes, [6] pass cycles (profile builds)
        print(f"  nnls (stream) CTA0 per call: prologue {red / calls:.0f} cyc, loop {loop / calls:.0f} cyc "
              f"({sw / calls:.1f} sweeps, {npass / calls:.1f} passes, {loop / max(sw, 1):.0f} cyc/sweep, "
              f"pass {tri / max(npass, 1):.0f} cyc), epilogue {pc / calls:.0f} cyc")
        ph = b[8 + 256 + 64: 8 + 256 + 72]
        ph2 = b[8 + 256 + 72: 8 + 256 + 75]
        print("  row loop/call: total %.0f cyc, gate waits %.0f cyc in %.1f waits" % (b[8 + 256 + 81] / calls, _buf[7] / calls, b[8 + 256 + 80] / calls))
        print("  G+C detail/call: to C issue %.0f | G loop %.0f | C stores (wait) %.0f" % tuple(x / calls for x in ph2))
        print("  phases/call: G+C loads %.0f | tables %.0f | cl.sync %.0f || writes %.0f | gram part %.0f | cl.sync %.0f | reduce %.0f | cl.sync+ %.0f"
              % tuple(x / calls for x in ph))
