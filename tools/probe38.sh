# tree kernel: 128-thread tiles on up to 16-CTA clusters for wide views: tests, C2/C3/C4
mkdir -p gpurun_out/p38
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p38/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p38/pytest_gpu.log
for c in c2 c3 c4; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/p38/bench_$c.json 2> gpurun_out/p38/bench_$c.err; done
echo done
