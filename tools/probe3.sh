timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python tools/tune.py c2 10 2>&1 | tail -3
python tools/tune.py c3 10 2>&1 | tail -3
python tools/tune.py c4 10 2>&1 | tail -3
NTF_NNLS_OLD=1 python tools/tune.py c2 10 2>&1 | tail -1
timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400
