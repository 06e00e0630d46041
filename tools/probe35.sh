# tree kernel on 8-CTA clusters (DSMEM chunk reduction): tests, C2/C3/C4 lines, launch list
mkdir -p gpurun_out/p35
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p35/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p35/pytest_gpu.log
for c in c2 c3 c4; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/p35/bench_$c.json 2> gpurun_out/p35/bench_$c.err; done
NTF_TREE_ATOMIC=1 timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/p35/bench_c2_atomic.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p35/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/p35/ncu_launch.log 2>&1
echo done
