"""Per-kernel launch table from an ncu --csv launch list (diagnostics)."""
import collections, csv, io, sys

txt = open(sys.argv[1]).read().splitlines()
i = [k for k, l in enumerate(txt) if l.startswith('"ID"')][0]
rows = list(csv.DictReader(io.StringIO("\n".join(txt[i:]))))
per = collections.OrderedDict()
for r in rows:
    d = per.setdefault(r["ID"], {"name": r["Kernel Name"].split("(")[0][:58], "grid": r["Grid Size"]})
    v = float(r["Metric Value"].replace(",", ""))
    d[r["Metric Name"]] = v
agg = collections.OrderedDict()
for d in per.values():
    a = agg.setdefault(d["name"], [0, 0.0, 0.0])
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0) / 1e3
    a[2] += (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1e6
tot = sum(a[1] for a in agg.values())
for n, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:60s} {c:4d} {t / c:9.1f} us {100 * t / tot:5.1f}%  {b / c:9.2f} MB/launch")
