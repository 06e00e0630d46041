# tree kernel: W row pitch padded for DMMA B fragments: tests, C2/C3/C4
mkdir -p gpurun_out/p39
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p39/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p39/pytest_gpu.log
for c in c2 c3 c4; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/p39/bench_$c.json 2> gpurun_out/p39/bench_$c.err; done
echo done
