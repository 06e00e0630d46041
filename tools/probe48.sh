# NNLS r = 24..32 on eight lanes per row with 9-warp CTAs (C4) vs four lanes
mkdir -p gpurun_out/p48
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p48/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p48/pytest_gpu.log
timeout 300 python bench.py --config c4 --no-cpu-baseline > gpurun_out/p48/bench_c4.json 2> gpurun_out/p48/bench_c4.err
NTF_NNLS_WIDE_CTA=0 timeout 300 python bench.py --config c4 --no-cpu-baseline > gpurun_out/p48/bench_c4_narrow.json 2>&1
echo done
