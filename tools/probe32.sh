# roofline over both passes (kernel timing of partial passes alone): tests, C2/C3 lines
mkdir -p gpurun_out/p32
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p32/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p32/pytest_gpu.log
timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/p32/bench_c2.json 2> gpurun_out/p32/bench_c2.err
timeout 300 python bench.py --config c3 --no-cpu-baseline > gpurun_out/p32/bench_c3.json 2> gpurun_out/p32/bench_c3.err
timeout 300 python bench.py --config c4 --no-cpu-baseline > gpurun_out/p32/bench_c4.json 2> gpurun_out/p32/bench_c4.err
echo done
