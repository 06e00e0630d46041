# split tree: GPU tests, C2/C3 bench lines, C3 and C2 launch lists
mkdir -p gpurun_out/p22
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p22/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p22/pytest_gpu.log
for c in c2 c3; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/p22/bench_$c.json 2> gpurun_out/p22/bench_$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/p22/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p22/ncu_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/p22/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p22/ncu_c2.log 2>&1
echo done
