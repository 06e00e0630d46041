#!/bin/bash
O=gpurun_out/r02ap; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vs_reference.py -m gpu -q 2>&1 | tail -3
for c in c2 c3 c4; do timeout 300 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> /dev/null; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r02ap/bench_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d["value"],1))
PY
