#!/usr/bin/env python
"""Top CUDA source lines by warp-stall samples (ncu source page in
cuda,sass mode, -lineinfo builds; diagnostics):
  python tools/ncu_lines_top.py REP FUNC_REGEX [N]"""
import csv
import io
import re
import subprocess
import sys

rep, fre = sys.argv[1], sys.argv[2]
top_n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = {}
fname, fn, hdr = "", "", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit() or not re.search(fre, fn):
        continue
    s = int(r[4]) if r[4].isdigit() else 0
    if not s:
        continue
    st = {}
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h and i < len(r) and r[i].isdigit() and int(r[i]):
            st[h[6:]] = int(r[i])
    e = agg.setdefault((fname, int(r[0]), r[1].strip()[:90]), [0, {}])
    e[0] += s
    for k, v in st.items():
        e[1][k] = e[1].get(k, 0) + v
tot = sum(v[0] for v in agg.values())
print(f"samples {tot}")
for (f, ln, src), (s, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top_n]:
    tops = " ".join(f"{k}:{v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
    print(f"{100 * s / max(tot, 1):5.1f}% {f}:{ln} {src:90s} {tops}")
