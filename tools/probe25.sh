# FP64 DMMA consumers: GPU tests, C2/C3 bench (DMMA vs DFMA), C2 launch list
mkdir -p gpurun_out/p25
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p25/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p25/pytest_gpu.log
for c in c2 c3; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/p25/bench_$c.json 2> gpurun_out/p25/bench_$c.err; done
NTF_FAST_MMA=0 timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/p25/bench_c2_dfma.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/p25/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p25/ncu_c2.log 2>&1
echo done
