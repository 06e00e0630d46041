#!/bin/bash
# Kernel durations (ncu) of the standalone AHALS call for NNLS timing variants: apply
# tools/r02/nnls_experiments.patch, build one library per mask with
#   nvcc ... -DNTF_NNLS_X=<mask> -c kernels_nnls.cu  (+ link with the other objects) -> build/var/libntf_x<mask>.so
# then: bash tools/r02/nnls_variant_timing.sh 128 129 130 132 136 144 160 192 140 255
# (profiles/r02/nnls_variant_kernels_r02ar.txt). 1-sweep vs 50-sweep launches give the per-sweep cost.
O=gpurun_out/nnls_variants; mkdir -p $O
for X in "$@"; do
  NTF_B200_LIB=build/var/libntf_x$X.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l_$X.csv -k regex:nnls_stream python tools/nnls_bench.py 300 20 > /dev/null 2>&1
  python - $O/l_$X.csv $X <<'PY'
import csv,io,sys
txt=open(sys.argv[1]).read().splitlines()
i=[k for k,l in enumerate(txt) if l.startswith('"ID"')][0]
rows=list(csv.DictReader(io.StringIO("\n".join(txt[i:]))))
d=[float(r["Metric Value"].replace(",",""))/1e3 for r in rows]
# the bench launches: 1 warm + 30 one-sweep, then 1 warm + 30 fifty-sweep, then 1 + 10 fifty-sweep
one=sorted(d[1:31])[15]; fifty=sorted(d[32:62])[15]
print(f"X={sys.argv[2]}: 1 sweep {one:.1f} us, 50 sweeps {fifty:.1f} us, per sweep {(fifty-one)/49*1e3:.0f} ns = {(fifty-one)/49*1965:.0f} cycles (n={len(d)})")
PY
done | tee $O/nnls_variant_kernels.txt
