#!/usr/bin/env python
"""Top SASS instructions by warp-stall samples from an ncu report's source
page (diagnostics): python tools/ncu_source_top.py REP KERNEL_REGEX [N]
Prints per kernel the N hottest instructions with their dominant stall
reasons, plus a per-opcode summary and the shared-memory excess wavefronts."""
import collections
import csv
import io
import re
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top_n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = re.split(r'^"Kernel Name",', out, flags=re.M)
seen = 0
for blk in blocks[1:]:
    name, _, body = blk.partition("\n")
    if not re.search(kre, name):
        continue
    seen += 1
    rows = list(csv.reader(io.StringIO(body)))
    hdr = rows[0]
    recs = [dict(zip(hdr, r)) for r in rows[1:] if len(r) == len(hdr)]
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in recs)
    print(f"== {name.strip()[:140]}  samples {tot}")
    by_op = collections.Counter()
    shx = 0
    for r in recs:
        op = r["Source"].strip().split()[0] if r["Source"].strip() else "?"
        if op.startswith("@"):
            op = r["Source"].strip().split()[1]
        by_op[op.split(".")[0]] += int(r["Warp Stall Sampling (All Samples)"] or 0)
        shx += int(r.get("L1 Wavefronts Shared Excessive", "0") or 0)
    print("  by opcode:", ", ".join(f"{k} {100 * v / max(tot, 1):.1f}%" for k, v in by_op.most_common(12)))
    print(f"  shared excessive wavefronts: {shx}")
    hot = sorted(recs, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:top_n]
    for r in hot:
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        st = sorted(((int(r[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
        print(f"  {r['Address'][-5:]} {100 * s / max(tot, 1):5.1f}%  {r['Source'].strip()[:60]:60s} "
              + " ".join(f"{n}:{v}" for v, n in st if v))
if not seen:
    print("no kernel matched", kre)
