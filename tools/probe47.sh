# launch lists at C3 and C4 (final round-1 code)
mkdir -p gpurun_out/p47
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p47/launches_c3.csv python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p47/ncu_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p47/launches_c4.csv python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p47/ncu_c4.log 2>&1
echo done
