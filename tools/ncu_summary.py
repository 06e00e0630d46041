"""Summarise an ncu report: duration, DRAM bytes/throughput, pipe use, top
stall reasons and the hottest SASS lines (diagnostics)."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
def page(name, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))
raw = page("raw")
h, units, v = raw[0], raw[1], raw[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg"]
for k in want:
    if k in h:
        i = h.index(k)
        print(f"{k:70s} {v[i]} {units[i]}")
st = []
for k, x in zip(h, v):
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
        try: st.append((float(x), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError: pass
tot = sum(x for x, _ in st) or 1
print("stalls:", ", ".join(f"{k} {100*x/tot:.0f}%" for x, k in sorted(st, reverse=True)[:8]))
src = page("source", ("--print-source", "sass"))
hh = src[1]
ai, si, wi, ei = hh.index("Address"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
rows = []
for r in src[2:]:
    try: rows.append((int(r[wi] or 0), r[ai][-5:], r[si][:64], int(r[ei] or 0)))
    except ValueError: pass
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
for r in sorted(rows, reverse=True)[:n]:
    print(f"  {r[0]:6d} {r[1]} {r[2]:64s} x{r[3]}")
