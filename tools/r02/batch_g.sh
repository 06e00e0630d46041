#!/bin/bash
O=gpurun_out/r02g; mkdir -p $O
timeout 300 python tools/r02/sk_check.py > $O/sk_check.log 2>&1; echo "rc=$?" >> $O/sk_check.log
if grep -q FAIL $O/sk_check.log || ! grep -q "rc=0" $O/sk_check.log; then echo "skip bench" >> $O/sk_check.log; exit 0; fi
for np in 2 1; do
  NTF_SK_NP=$np timeout 300 python bench.py --no-cpu-baseline --steps 100 > $O/bench_c2_np$np.json 2> $O/bench_c2_np$np.err
  NTF_SK_NP=$np timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 100 > $O/bench_c3_np$np.json 2> $O/bench_c3_np$np.err
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"mttkrp_sk" -s 4 -c 2 -o $O/full_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_c2.log 2>&1
echo done
