#!/usr/bin/env python
"""SASS instruction histogram of the hot kernels in libntf_b200.so
(cuobjdump -sass): proves which units the kernels use -- UTMALDG (TMA tensor
loads), UBLKCP (bulk copies), DMMA (FP64 MMA), DFMA / FFMA / FFMA2, LDS /
STS, SYNCS (mbarrier ops) -- per kernel instantiation.

  python tools/sass_hist.py [lib.so] > profiles/<round>/sass_hist.txt
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2001_04321_b200/libntf_b200.so"
KEYS = ["UTMALDG", "UBLKCP", "DMMA", "DFMA", "DMUL", "DADD", "FFMA", "FFMA2", "FMUL", "LDS", "LDSM", "STS",
        "LDG", "STG", "SYNCS", "BAR", "SHFL", "ATOMS", "RED", "ATOMG", "LDL", "STL", "UCGABAR_ARV", "MEMBAR"]
HOT = re.compile(r"mttkrp_fast|tree_mttkrp|nnls_stream|nnls_|objective|init_factors|norm_sq")


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            op = m.group(1)
            kernels[cur][op] += 1
            kernels[cur]["_total"] += 1
    demangled = {}
    names = list(kernels)
    try:
        dm = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
        demangled = dict(zip(names, dm))
    except OSError:
        pass
    print("kernel | " + " | ".join(KEYS) + " | total")
    for k, c in kernels.items():
        name = demangled.get(k, k).replace("(anonymous namespace)::", "")
        if not HOT.search(name):
            continue
        label = re.sub(r"\(.*", "", name).replace("void ", "")[:120]
        print(f"{label} | " + " | ".join(str(c.get(key, 0)) for key in KEYS) + f" | {c['_total']}")


if __name__ == "__main__":
    main()
