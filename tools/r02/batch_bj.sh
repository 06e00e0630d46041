#!/bin/bash
# validation of the r02bj state: full GPU suite, smoke, driver-style bench lines, C3/C4/C5, launch list
O=gpurun_out/r02bj; mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_c2_k20.json 2> $O/bench_c2_k20.err; echo "bench k20 rc=$?"
timeout 300 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_ref_k20.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench rc=$?"
timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 100 > $O/bench_c3.json 2> /dev/null; echo "c3 rc=$?"
timeout 300 python bench.py --config c4 --no-cpu-baseline --steps 50 > $O/bench_c4.json 2> /dev/null; echo "c4 rc=$?"
timeout 400 python bench.py --config c5 --no-cpu-baseline --steps 10 > $O/bench_c5.json 2> /dev/null; echo "c5 rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/ncu_launch2.log 2>&1; echo "launch list rc=$?"
tail -4 $O/pytest_gpu.log
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r02bj/bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split('/')[-1], round(d["value"],2), "e2e", round(d["e2e"]["value"],2), d.get("roofline",{}).get("per_mode_ms"), d.get("roofline",{}).get("frac"), d.get("roofline",{}).get("fma_frac"))
    except Exception as e:
        print(f, "ERR", e)
PY
