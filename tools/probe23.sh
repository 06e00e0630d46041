export NTF_B200_LIB=$PWD/build/prof/libntf_b200_prof.so
for c in c2 c3; do python tools/tune.py $c 10 2>&1 | grep -E "nnls|row loop"; done
