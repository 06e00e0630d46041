export NTF_B200_LIB=$PWD/build/prof/libntf_b200_prof.so
python tools/nnls_bench.py 300 20
python tools/tune.py c2 10 2>&1 | tail -4
unset NTF_B200_LIB
python tools/nnls_bench.py 300 20
python tools/tune.py c2 10 2>&1 | tail -2
