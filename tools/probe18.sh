timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in c2 c4; do timeout 300 python bench.py --config $c --no-cpu-baseline 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['value'],1), d['roofline']['per_mode_ms'])"; done
