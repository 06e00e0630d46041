"""Per-launch summary of an ncu report (every kernel in it): duration, DRAM
bytes, pipe utilisation, issue activity, shared-memory bank conflicts and the
top stall reasons. usage: ncu_raw_summary.py report.ncu-rep [raw.csv.gz]"""
import csv, gzip, io, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
if len(sys.argv) > 2:
    with gzip.open(sys.argv[2], "wt") as f:
        f.write(out)
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
idx = {k: i for i, k in enumerate(h)}
want = [("gpu__time_duration.sum", "dur"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("lts__t_bytes.sum", "l2_bytes"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
        ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma%"),
        ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", "fmaheavy%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
        ("smsp__inst_executed.sum", "inst"), ("sm__cycles_elapsed.avg", "cycles")]
for v in rows[2:]:
    if len(v) < len(h):
        continue
    print("==", v[idx["ID"]], v[idx["Kernel Name"]][:90])
    line = []
    for k, short in want:
        if k in idx:
            line.append(f"{short}={v[idx[k]]}{'' if short.endswith('%') else ' ' + units[idx[k]]}")
    print("   " + "; ".join(line))
    st = []
    for k, x in zip(h, v):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                st.append((float(x), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1
    print("   stalls: " + ", ".join(f"{k} {100 * x / tot:.0f}%" for x, k in sorted(st, reverse=True)[:7]))
