CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/p6_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"nnls_stream" -s 6 -c 1 -f -o gpurun_out/prof_nnls $CMD > gpurun_out/p6_ncu.log 2>&1; echo rc=$?
