# NNLS at r = 20: 20-column 4-lane plan vs 24-column 8-lane plan
mkdir -p gpurun_out/p33
timeout 300 python tools/nnls_bench.py 300 20 > gpurun_out/p33/nnls.txt 2>&1
NTF_NNLS_R20_WIDE=1 timeout 300 python tools/nnls_bench.py 300 20 >> gpurun_out/p33/nnls.txt 2>&1
timeout 300 python bench.py --config c2 --no-cpu-baseline --steps 100 > gpurun_out/p33/bench_c2.json 2>&1
NTF_NNLS_R20_WIDE=1 timeout 300 python bench.py --config c2 --no-cpu-baseline --steps 100 > gpurun_out/p33/bench_c2_wide.json 2>&1
NTF_NNLS_R20_WIDE=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "ahals or her_trace" > gpurun_out/p33/pytest_wide.log 2>&1
echo done
