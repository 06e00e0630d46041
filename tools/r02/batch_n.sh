#!/bin/bash
O=gpurun_out/r02n; mkdir -p $O
timeout 300 python tools/r02/sk_check.py > $O/sk_check.log 2>&1; echo "rc=$?" >> $O/sk_check.log
timeout 600 python -m pytest tests/test_solvers.py tests/test_host_api.py -m gpu -q -rf > $O/pytest_solvers.log 2>&1; echo "rc=$?" >> $O/pytest_solvers.log
if grep -q FAIL $O/sk_check*.log; then echo "skip bench" >> $O/sk_check.log; exit 0; fi
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 60 --warmup 5 > $O/c2_$tag.json 2>/dev/null; python -c "
import json; d=json.load(open('$O/c2_$tag.json')); print('$tag', round(d['value'],1), [round(x*1000,1) for x in d['roofline']['per_mode_ms']])" >> $O/sweep.txt; }
run default NTF_X=0
run st2 NTF_SK_STAGES=2
run st3 NTF_SK_STAGES=3
run mw8 NTF_SK_MW=8
run np4 NTF_SK_NP=4
timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 60 > $O/c3.json 2>/dev/null
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
echo done
