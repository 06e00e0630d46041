# programmatic dependent launch of the fused block update: tests, C2/C3 lines with and without
mkdir -p gpurun_out/p37
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p37/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p37/pytest_gpu.log
for c in c2 c3; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/p37/bench_$c.json 2> gpurun_out/p37/bench_$c.err
  NTF_PDL=0 timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/p37/bench_${c}_nopdl.json 2>&1
done
echo done
