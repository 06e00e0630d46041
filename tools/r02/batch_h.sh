#!/bin/bash
O=gpurun_out/r02h; mkdir -p $O
timeout 300 python tools/r02/sk_check.py > $O/sk_check.log 2>&1; echo "rc=$?" >> $O/sk_check.log
NTF_SK_MW=8 timeout 300 python tools/r02/sk_check.py > $O/sk_check_mw8.log 2>&1; echo "rc=$?" >> $O/sk_check_mw8.log
if grep -q FAIL $O/sk_check*.log; then echo "skip bench" >> $O/sk_check.log; exit 0; fi
for mw in 4 8; do
  NTF_SK_MW=$mw timeout 300 python bench.py --no-cpu-baseline --steps 100 > $O/bench_c2_mw$mw.json 2> $O/bench_c2_mw$mw.err
  NTF_SK_MW=$mw timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 100 > $O/bench_c3_mw$mw.json 2> $O/bench_c3_mw$mw.err
done
NTF_SK_MW=8 NTF_SK_NP=1 timeout 300 python bench.py --no-cpu-baseline --steps 100 > $O/bench_c2_mw8np1.json 2> $O/bench_c2_mw8np1.err
echo done
