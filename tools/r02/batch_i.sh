#!/bin/bash
O=gpurun_out/r02i; mkdir -p $O
timeout 300 python tools/r02/sk_check.py > $O/sk_check.log 2>&1; echo "rc=$?" >> $O/sk_check.log
NTF_SK_DIRECTB=0 timeout 300 python tools/r02/sk_check.py > $O/sk_check_nodb.log 2>&1; echo "rc=$?" >> $O/sk_check_nodb.log
if grep -q FAIL $O/sk_check*.log; then echo "skip bench" >> $O/sk_check.log; exit 0; fi
timeout 300 python bench.py --no-cpu-baseline --steps 100 > $O/bench_c2.json 2> $O/bench_c2.err
NTF_SK_DIRECTB=0 timeout 300 python bench.py --no-cpu-baseline --steps 100 > $O/bench_c2_nodb.json 2> $O/bench_c2_nodb.err
for naw in 3 6; do NTF_SK_NAW=$naw timeout 300 python bench.py --no-cpu-baseline --steps 100 > $O/bench_c2_naw$naw.json 2> /dev/null; done
timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 100 > $O/bench_c3.json 2> $O/bench_c3.err
NTF_SK_NAW=6 timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 100 > $O/bench_c3_naw6.json 2> /dev/null
echo done
