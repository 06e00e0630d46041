#!/bin/bash
# async upload + session without host syncs: full GPU suite, smoke, e2e probe, driver-style bench
O=gpurun_out/r02ai; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?"
python tools/e2e_probe.py 20 > $O/e2e_probe_20.txt 2>&1
python tools/e2e_probe.py 200 > $O/e2e_probe_200.txt 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c2_k20.json 2> $O/bench_c2_k20.err; echo "bench k20 rc=$?"
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench rc=$?"
tail -4 $O/pytest_gpu.log; tail -3 $O/e2e_probe_20.txt; tail -2 $O/e2e_probe_200.txt
python - <<'PY'
import json
for f in ("bench_c2_k20","bench_c2"):
    d=json.loads(open(f"gpurun_out/r02ai/{f}.json").read().strip().splitlines()[-1])
    print(f, round(d["value"],1), "e2e", round(d["e2e"]["value"],1), d["e2e"]["samples_s"])
PY
