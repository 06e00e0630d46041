#!/bin/bash
# Round-2 opening check: GPU tests, smoke, default bench line.
mkdir -p gpurun_out/r02a
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02a/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02a/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a/smoke.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02a/bench_c2.json 2> gpurun_out/r02a/bench_c2.err
echo done
