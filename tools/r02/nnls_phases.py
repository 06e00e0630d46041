"""Phase breakdown of the fused NNLS kernel in the production session
(CTA 0 cycle stamps, summed over calls; diagnostics): prologue (C / Gram
loads, Hadamard, tables), the sweep loop, and the epilogue phases.
usage: python tools/r02/nnls_phases.py c2|c3|c4 [iters]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2001_04321_b200 as P  # noqa: E402
from paper_2001_04321_b200 import _lib as L  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
t, truth, init = bench.make_instance(P, name)
prov = P.GpuDenseProvider(t)
sess = P.Session(prov, init, P.AoConfig(max_outer_iters=10 ** 6), P.HerParams(), algo="her")
sess.step(5)
sess.sync()
buf = (C.c_ulonglong * (8 + 384))()
L.lib().ntf_debug_nnls_prof(buf, 1)
# zero the phase counters too: read once, subtract afterwards
base = [0] * 8 + list(buf)[8:]  # g_nnls_prof was reset by the read
sess.step(iters)
sess.sync()
L.lib().ntf_debug_nnls_prof(buf, 1)
cur = list(buf)
d = [c - b for c, b in zip(cur, base)]
prof, skew = d[:8], d[8:]
calls = max(prof[3], 1)
ph = skew[2 * 128 + 64: 2 * 128 + 75]
names = ["prologue to tables", "tables", "cluster sync", "epi: write block", "epi: gram partials",
         "epi: cluster sync", "epi: cluster reduce", "epi: final sync+decision", "load C issue", "Hadamard",
         "store C"]
print(f"{name}: {calls} calls, {prof[2] / calls:.1f} sweeps/call, loop {prof[0] / calls:.0f} cyc/call "
      f"({prof[0] / max(prof[2], 1):.0f} cyc/sweep), outside loop {prof[1] / calls:.0f} + {prof[4] / calls:.0f}")
print(f"  row passes {prof[5]}, pass cycles/pass {prof[6] / max(prof[5], 1):.0f}, gate cycles/call {prof[7] / calls:.0f}")
for n, v in zip(names, ph):
    print(f"  {n:28s} {v / calls:8.0f} cyc/call")
sess.close()
