# DMMA 80-row warps (4 x 2 consumer warps) at r = 20: tests, C2 bench, counters
mkdir -p gpurun_out/p29
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p29/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p29/pytest_gpu.log
timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/p29/bench_c2.json 2> gpurun_out/p29/bench_c2.err
NTF_FAST_CONS=12 timeout 300 python bench.py --config c3 --no-cpu-baseline > gpurun_out/p29/bench_c3_cons12.json 2>&1
echo done
