# tree one-wave grid + DMMA: GPU tests, C2 bench, full ncu of both C2 passes
mkdir -p gpurun_out/p26
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p26/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p26/pytest_gpu.log
timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/p26/bench_c2.json 2> gpurun_out/p26/bench_c2.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mttkrp_fast -s 4 -c 2 -o gpurun_out/p26/fast_c2 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p26/ncu_fast.log 2>&1
echo done
