#!/bin/bash
O=gpurun_out/r02y; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --steps 100 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 100 > $O/bench_c3.json 2> /dev/null
timeout 300 python bench.py --config c4 --no-cpu-baseline --steps 50 > $O/bench_c4.json 2> /dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/ncu_launch2.log 2>&1
echo done
