# tree path choice (clusters only for short chunks): tests incl. both paths, C2/C3 lines
mkdir -p gpurun_out/p36
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p36/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p36/pytest_gpu.log
NTF_TREE_ATOMIC=1 timeout 900 python -m pytest tests/test_dimtree.py -m gpu -x -q > gpurun_out/p36/pytest_atomic.log 2>&1; echo "rc=$?" >> gpurun_out/p36/pytest_atomic.log
for c in c2 c3; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/p36/bench_$c.json 2> gpurun_out/p36/bench_$c.err; done
echo done
