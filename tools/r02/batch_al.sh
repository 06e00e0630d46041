#!/bin/bash
# early hand-over NNLS: parity of the sweeps/traces + C2 bench at L = 3, 4; C3, C4
O=gpurun_out/r02al; mkdir -p $O
for L in 3 4; do
  NTF_NNLS_L=$L timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dimtree.py -m gpu -q > $O/pytest_L$L.log 2>&1; echo "L=$L pytest rc=$? $(tail -1 $O/pytest_L$L.log)"
  NTF_NNLS_L=$L timeout 300 python bench.py --no-cpu-baseline > $O/bench_c2_L$L.json 2> /dev/null
done
timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 100 > $O/bench_c3.json 2> /dev/null
timeout 300 python bench.py --config c4 --no-cpu-baseline --steps 50 > $O/bench_c4.json 2> /dev/null
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r02al/bench_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d["value"],1))
PY
