#!/bin/bash
O=gpurun_out/r02am; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_vs_reference.py tests/test_gpu_parity.py -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)"
grep -E "^FAILED|^ERROR" $O/pytest.log | head -20
timeout 300 python bench.py --no-cpu-baseline > $O/bench_c2.json 2> /dev/null
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r02am/bench_c2.json").read().strip().splitlines()[-1]); print("c2", round(d["value"],1), round(d["e2e"]["value"],1))
PY
