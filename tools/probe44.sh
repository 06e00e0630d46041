# FP32 partials for FP32 tensors: tests, C4 (and NTF_TREE_F64=1 control), C2
mkdir -p gpurun_out/p44
timeout 900 python -m pytest tests -m gpu -x -q -s -k "f32 or dimtree" > gpurun_out/p44/pytest_f32.log 2>&1; echo "rc=$?" >> gpurun_out/p44/pytest_f32.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p44/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p44/pytest_gpu.log
timeout 300 python bench.py --config c4 --no-cpu-baseline > gpurun_out/p44/bench_c4.json 2> gpurun_out/p44/bench_c4.err
NTF_TREE_F64=1 timeout 300 python bench.py --config c4 --no-cpu-baseline > gpurun_out/p44/bench_c4_f64.json 2>&1
timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/p44/bench_c2.json 2>&1
echo done
