#!/bin/bash
# Full ncu captures (--set full) of one outer iteration's kernels at C2, C3, C4;
# the reports stay on the box (too large), per-launch summaries + raw CSVs come back.
O=gpurun_out/r02bd; mkdir -p $O
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
timeout 300 $B > $O/plain_c2.json 2> $O/plain_c2.err; echo "plain c2 rc=$?"
for c in c2:16:8 c3:20:10 c4:16:8; do
  IFS=: read cfg skip cnt <<< "$c"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mttkrp_sk|nnls_stream|tree2" -s $skip -c $cnt -f -o /tmp/full_$cfg $B --config $cfg > $O/ncu_$cfg.log 2>&1; echo "$cfg rc=$?"
  python tools/ncu_raw_summary.py /tmp/full_$cfg.ncu-rep $O/full_${cfg}_raw.csv.gz > $O/full_${cfg}_summary.txt 2>&1
done
# one compact report for the source page: the two C2 passes only
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mttkrp_sk" -s 4 -c 2 -f -o $O/full_c2_sk $B > $O/ncu_c2_sk.log 2>&1; echo "c2 sk rc=$?"
ls -la $O
