#!/bin/bash
# U = 2W clip-free chain: parity (sweep counts, traces, determinism) + benches
O=gpurun_out/r02an; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_dimtree.py tests/test_gpu_vs_reference.py tests/test_solvers.py tests/test_acceptance_gpu.py -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)"
grep -E "^FAILED|^ERROR" $O/pytest.log | head
for c in c2 c3 c4; do timeout 300 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> /dev/null; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r02an/bench_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split('/')[-1], round(d["value"],1), "e2e", round(d["e2e"]["value"],1))
PY
