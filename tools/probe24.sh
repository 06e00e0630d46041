timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
export NTF_B200_LIB=$PWD/build/prof/libntf_b200_prof.so
for c in c2 c3 c4; do python tools/tune.py $c 10 2>&1 | grep -E "nnls \(|row loop"; done
unset NTF_B200_LIB
for c in c2 c3; do timeout 300 python bench.py --config $c --no-cpu-baseline 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:20], round(d['value'],1), d['roofline']['per_mode_ms'])"; done
