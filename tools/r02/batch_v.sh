#!/bin/bash
O=gpurun_out/r02v; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python tools/r02/c4_her_vs_ao.py 1000 > $O/c4_her_vs_ao.json 2> $O/c4_her_vs_ao.err
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"mttkrp_sk" -s 4 -c 2 -o $O/full_c4 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_c4.log 2>&1
echo done
