#!/bin/bash
O=gpurun_out/r02q; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_dimtree.py tests/test_config_parity.py tests/test_sharded_gpu.py -m gpu -q -x > $O/pytest_a.log 2>&1; echo "rc=$?" >> $O/pytest_a.log
if ! grep -q "rc=0" $O/pytest_a.log; then echo "skip bench"; exit 0; fi
timeout 300 python bench.py --no-cpu-baseline --steps 100 > $O/bench_c2.json 2> $O/bench_c2.err
NTF_OVERLAP=0 timeout 300 python bench.py --no-cpu-baseline --steps 100 > $O/bench_c2_noov.json 2> $O/bench_c2_noov.err
timeout 300 python bench.py --config c4 --no-cpu-baseline --steps 50 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo done
