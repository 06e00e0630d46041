timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
export NTF_B200_LIB=$PWD/build/fprof/libntf_b200_fprof.so
NTF_FAST_PROF=1 python tools/prof_mttkrp.py c2 1 2>&1 | grep "epilogue"
unset NTF_B200_LIB
timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['roofline']['per_mode_ms'], d['roofline']['frac'])"
