#!/bin/bash
# NNLS window length sweep at r = 20 (NTF_NNLS_L): oracle parity of the sweeps + C2 bench
O=gpurun_out/r02ak; mkdir -p $O
for L in 4 3 5 6; do
  NTF_NNLS_L=$L timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "ahals_vs_oracle or her_trace_parity" > $O/pytest_L$L.log 2>&1; echo "L=$L pytest rc=$? $(tail -1 $O/pytest_L$L.log)"
  NTF_NNLS_L=$L timeout 300 python bench.py --no-cpu-baseline > $O/bench_c2_L$L.json 2> /dev/null
  python - $O/bench_c2_L$L.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d["value"],1))
PY
done
