#!/bin/bash
O=gpurun_out/r02au; mkdir -p $O
for Q in 4 8; do
  NTF_NNLS_SQ=$Q timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "ahals_vs_oracle or her_trace_parity" 2>&1 | tail -1
  NTF_NNLS_SQ=$Q timeout 300 python bench.py --no-cpu-baseline > $O/bench_c2_Q$Q.json 2> /dev/null
done
timeout 300 python bench.py --config c4 --no-cpu-baseline --steps 50 > $O/bench_c4.json 2> /dev/null
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r02au/bench_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d["value"],1))
PY
