#!/bin/bash
O=gpurun_out/r02l; mkdir -p $O
timeout 300 python tools/r02/sk_check.py > $O/sk_check.log 2>&1; echo "rc=$?" >> $O/sk_check.log
if grep -q FAIL $O/sk_check*.log; then echo "skip bench" >> $O/sk_check.log; exit 0; fi
timeout 300 python bench.py --no-cpu-baseline --steps 100 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 100 > $O/bench_c3.json 2> $O/bench_c3.err
NTF_SK_MW=8 timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 100 > $O/bench_c3_mw8.json 2> /dev/null
NTF_SK_NAW=2 timeout 300 python bench.py --no-cpu-baseline --steps 100 > $O/bench_c2_naw2.json 2> /dev/null
timeout 600 python -m pytest tests/test_host_api.py tests/test_tucker.py -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo done
