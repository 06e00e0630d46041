mkdir -p gpurun_out/p20
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/p20/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p20/ncu_c3.log 2>&1
echo done
