# dimension-tree split + fused tree reduction: GPU tests, then C2/C3 bench lines
mkdir -p gpurun_out/p21
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p21/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p21/pytest_gpu.log
for c in c2 c3 c4; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/p21/bench_$c.json 2> gpurun_out/p21/bench_$c.err; done
NTF_TREE_SPLIT=3 timeout 300 python bench.py --config c3 --no-cpu-baseline > gpurun_out/p21/bench_c3_split3.json 2>&1
echo done
