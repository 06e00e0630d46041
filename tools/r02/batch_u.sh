#!/bin/bash
O=gpurun_out/r02u; mkdir -p $O
timeout 300 python tools/r02/sk32_check.py > $O/sk32_check.log 2>&1; echo "rc=$?" >> $O/sk32_check.log
timeout 300 python tools/r02/sk_check.py > $O/sk_check.log 2>&1; echo "rc=$?" >> $O/sk_check.log
if grep -q FAIL $O/sk*_check.log; then echo "skip bench" >> $O/sk32_check.log; exit 0; fi
timeout 300 python bench.py --config c4 --no-cpu-baseline --steps 50 > $O/bench_c4.json 2> $O/bench_c4.err
NTF_SK_F32=0 timeout 300 python bench.py --config c4 --no-cpu-baseline --steps 50 > $O/bench_c4_old.json 2> /dev/null
timeout 900 python bench.py --config c5 --no-cpu-baseline --steps 5 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
echo done
