#!/bin/bash
# lanes per row of the r = 20 stream NNLS plan (NTF_NNLS_SQ) at C2
O=gpurun_out/r02as; mkdir -p $O
for Q in 4 2 1; do
  NTF_NNLS_SQ=$Q timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "ahals_vs_oracle or her_trace_parity" 2>&1 | tail -1
  NTF_NNLS_SQ=$Q timeout 300 python bench.py --no-cpu-baseline > $O/bench_c2_Q$Q.json 2> /dev/null
  python - $O/bench_c2_Q$Q.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d["value"],1))
PY
done
