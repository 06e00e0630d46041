# fast-MTTKRP pipeline counters (profile build), C2 and C3 per-mode calls
mkdir -p gpurun_out/p28
export NTF_B200_LIB=$PWD/build/fprof/libntf_b200_fprof.so NTF_FAST_PROF=1
timeout 300 python tools/prof_mttkrp.py c2 2 > gpurun_out/p28/prof_c2.txt 2>&1
timeout 300 python tools/prof_mttkrp.py c3 2 > gpurun_out/p28/prof_c3.txt 2>&1
echo done
