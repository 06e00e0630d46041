#!/bin/bash
# Round profile capture (run under gpurun from the repo root):
#   bench line, reference arm, launch list, full ncu capture of the top kernels.
set -u
R=${1:-r01}
O=gpurun_out
python bench.py > $O/bench_$R.json 2> $O/bench_$R.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_$R.json 2> $O/bench_ref_$R.err; echo "ref rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
$CMD > $O/plain_$R.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$R.csv $CMD > $O/ncu_launch_$R.log 2>&1
echo "launch list rc=$?"
$CMD > $O/plain2_$R.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"mttkrp_fast|nnls_stream|tree_mttkrp" -s 12 -c 6 \
      -f -o $O/prof_$R $CMD > $O/ncu_full_$R.log 2>&1
echo "full capture rc=$?"
for c in c3 c4; do python bench.py --config $c --no-cpu-baseline > $O/bench_${c}_$R.json 2> $O/bench_${c}_$R.err; echo "bench $c rc=$?"; done
