# NNLS 64 row lanes per CTA by default: GPU tests, C2/C3/C4 lines
mkdir -p gpurun_out/p46
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p46/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p46/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p46/smoke.log 2>&1
for c in c2 c3 c4; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/p46/bench_$c.json 2> gpurun_out/p46/bench_$c.err; done
echo done
