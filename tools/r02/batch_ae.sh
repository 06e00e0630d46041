#!/bin/bash
# pipelined FP32 A=4 consumers: parity subset + C4 A/B
O=gpurun_out/r02ae; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_dimtree.py tests/test_sharded_gpu.py tests/test_large.py -m gpu -q -x > $O/pytest_subset.log 2>&1; echo "pytest rc=$?"
B="python bench.py --no-cpu-baseline"
timeout 300 $B --config c4 --steps 50 > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"
NTF_SK_F32A=8 timeout 300 $B --config c4 --steps 50 > $O/bench_c4_a8.json 2> /dev/null; echo "c4 a8 rc=$?"
NTF_SK_STAGES=4 timeout 300 $B --config c4 --steps 50 > $O/bench_c4_st4.json 2> /dev/null; echo "c4 st4 rc=$?"
for f in $O/bench_*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"],1), d["roofline"]["per_mode_ms"], round(d["roofline"]["frac"],3), d["roofline"].get("fma_frac"))
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
done
tail -3 $O/pytest_subset.log
