timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
export NTF_B200_LIB=$PWD/build/prof/libntf_b200_prof.so
for c in c2 c3 c4; do python tools/tune.py $c 10 2>&1 | grep "nnls (stream)"; done
unset NTF_B200_LIB
timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -1 | cut -c1-120
