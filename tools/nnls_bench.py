"""Time the AHALS kernel alone (ntf_solve_nnls, host buffers) at a BASELINE
shape: per-sweep cost from the difference of a 50-sweep and a 1-sweep call
(tol = 0 forces every sweep)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2001_04321_b200 as P

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 300
r = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g = np.random.default_rng(1)
A = [g.random((rows, r)) for _ in range(3)]
G = (A[1].T @ A[1]) * (A[2].T @ A[2])
C = A[0] @ G
w0 = g.random((rows, r))


def t(iters, reps=30):
    st = P.InnerStop(max_iters=iters, rel_change_tol=0.0)
    P.ahals_solve(G, C, w0, st)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        P.ahals_solve(G, C, w0, st)
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


t1, t50 = t(1), t(50)
print(f"nnls rows={rows} r={r} Q={os.environ.get('NTF_NNLS_Q', 'auto')}: 1 sweep {t1*1e6:.1f} us, 50 sweeps {t50*1e6:.1f} us,"
      f" per sweep {(t50 - t1) / 49 * 1e6:.2f} us = {(t50 - t1) / 49 * 1.965e9:.0f} cycles")

import ctypes as _C
from paper_2001_04321_b200 import _lib as _L
_buf = (_C.c_ulonglong * (8 + 384))()
_L.lib().ntf_debug_nnls_prof(_buf, 1)
t(50, reps=10)
if _L.lib().ntf_debug_nnls_prof(_buf, 1) == 0 and _buf[3]:
    loop, red, sw, calls, pc, npass, tri, _ = list(_buf)[:8]
    print(f"  CTA0: {loop / calls:.0f} cyc/call, {sw / calls:.1f} sweeps/call, {loop / max(sw, 1):.0f} cyc/sweep, "
          f"reduction {red / max(sw, 1):.0f}, pass {pc / max(npass, 1):.0f} (triangle {tri / max(npass, 1):.0f})")
