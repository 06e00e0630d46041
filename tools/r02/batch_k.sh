#!/bin/bash
O=gpurun_out/r02k; mkdir -p $O
timeout 300 python tools/r02/sk_check.py > $O/sk_check.log 2>&1; echo "rc=$?" >> $O/sk_check.log
if grep -q FAIL $O/sk_check*.log; then echo "skip bench" >> $O/sk_check.log; exit 0; fi
timeout 300 python bench.py --no-cpu-baseline --steps 100 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 100 > $O/bench_c3.json 2> $O/bench_c3.err
NTF_SK_MW=8 timeout 300 python bench.py --no-cpu-baseline --steps 100 > $O/bench_c2_mw8.json 2> /dev/null
timeout 600 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for c in c2 c3; do timeout 300 python tools/r02/nnls_phases.py $c 50 > $O/nnls_phases_$c.txt 2>&1; done
echo done
