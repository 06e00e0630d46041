export NTF_B200_LIB=$PWD/build/fprof/libntf_b200_fprof.so
NTF_FAST_PROF=1 python tools/prof_mttkrp.py c2 2 2>&1 | grep -v "^\[fast-prof.*" | head; 
NTF_FAST_PROF=1 python tools/prof_mttkrp.py c2 2 2>&1 | grep "fast-prof"
NTF_FAST_PROF=1 python tools/prof_mttkrp.py c3 2 2>&1 | grep "fast-prof" | tail -8
