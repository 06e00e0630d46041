export NTF_B200_LIB=$PWD/build/fprof/libntf_b200_fprof.so
NTF_FAST_PROF=1 python tools/prof_mttkrp.py c2 2 2>&1 | grep "fast-prof" | grep -v "units/CTA"
NTF_FAST_PROF=1 python tools/prof_mttkrp.py c3 1 2>&1 | grep "fast-prof" | grep -v "units/CTA"
unset NTF_B200_LIB
python tools/tune.py c2 10 2>&1 | head -1
NTF_FAST_SEPARATE_REDUCE=1 python tools/tune.py c2 10 2>&1 | head -1
