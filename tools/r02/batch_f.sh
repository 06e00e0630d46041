#!/bin/bash
O=gpurun_out/r02f; mkdir -p $O
timeout 300 python tools/r02/sk_check.py > $O/sk_check.log 2>&1; echo "rc=$?" >> $O/sk_check.log
if grep -q FAIL $O/sk_check.log || ! grep -q "rc=0" $O/sk_check.log; then echo "skip bench" >> $O/sk_check.log; exit 0; fi
timeout 300 python bench.py --no-cpu-baseline --steps 100 > $O/bench_c2_sk.json 2> $O/bench_c2_sk.err
NTF_SK=0 timeout 300 python bench.py --no-cpu-baseline --steps 100 > $O/bench_c2_old.json 2> $O/bench_c2_old.err
timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 100 > $O/bench_c3_sk.json 2> $O/bench_c3_sk.err
NTF_SK=0 timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 100 > $O/bench_c3_old.json 2> $O/bench_c3_old.err
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
echo done
