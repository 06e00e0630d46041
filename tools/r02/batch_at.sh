#!/bin/bash
# packed chain coefficient + window length 2/3/4 of the r = 20 plan: parity + C2 bench; C3/C4 for the other plans
O=gpurun_out/r02at; mkdir -p $O
for L in 2 3 4; do
  NTF_NNLS_L=$L timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vs_reference.py -m gpu -q 2>&1 | tail -1
  NTF_NNLS_L=$L timeout 300 python bench.py --no-cpu-baseline > $O/bench_c2_L$L.json 2> /dev/null
done
timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 100 > $O/bench_c3.json 2> /dev/null
timeout 300 python bench.py --config c4 --no-cpu-baseline --steps 50 > $O/bench_c4.json 2> /dev/null
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r02at/bench_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d["value"],1))
PY
