#!/bin/bash
O=gpurun_out/r02ad; mkdir -p $O
./tools/chain_probe > $O/chain_probe.txt 2>&1; echo "probe rc=$?"
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mttkrp_sk" -s 4 -c 1 -f -o $O/full_c4_sk $B --config c4 > $O/ncu_c4_sk.log 2>&1; echo "c4 sk rc=$?"
NTF_SK_F32A=8 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mttkrp_sk" -s 4 -c 1 -f -o $O/full_c4_sk_a8 $B --config c4 > $O/ncu_c4_sk_a8.log 2>&1; echo "c4 sk a8 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"nnls_stream" -s 6 -c 1 -f -o $O/full_c2_nnls $B > $O/ncu_c2_nnls.log 2>&1; echo "c2 nnls rc=$?"
ls -la $O; cat $O/chain_probe.txt
