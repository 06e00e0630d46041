timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in c2 c3 c4; do python tools/tune.py $c 10 2>&1 | head -1; done
timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -1 | cut -c1-120
