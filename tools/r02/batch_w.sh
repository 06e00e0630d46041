#!/bin/bash
O=gpurun_out/r02w; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_config_parity.py tests/test_dimtree.py tests/test_solvers.py tests/test_sharded_gpu.py -m gpu -q > $O/pytest_a.log 2>&1; echo "rc=$?" >> $O/pytest_a.log
timeout 300 python bench.py --no-cpu-baseline --steps 100 > $O/bench_c2.json 2> $O/bench_c2.err
NTF_NNLS_NO_PDL=1 timeout 300 python bench.py --no-cpu-baseline --steps 100 > $O/bench_c2_nopdl.json 2> /dev/null
timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 100 > $O/bench_c3.json 2> /dev/null
timeout 300 python bench.py --config c4 --no-cpu-baseline --steps 50 > $O/bench_c4.json 2> /dev/null
bash tools/r02/build_profile_lib.sh > $O/build_prof.log 2>&1
for c in c2 c4; do NTF_B200_LIB=/tmp/ntfprof/libntf_b200.so timeout 300 python tools/r02/nnls_phases.py $c 50 > $O/nnls_phases_$c.txt 2>&1; done
echo done
