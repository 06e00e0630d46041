#!/bin/bash
# Round-1 closing check (r01h): GPU tests, smoke, default bench line, reference arm, C3/C4 lines, launch list.
mkdir -p gpurun_out/r01h
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r01h/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r01h/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01h/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r01h/bench_c2.json 2> gpurun_out/r01h/bench_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01h/bench_ref.json 2> gpurun_out/r01h/bench_ref.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/r01h/bench_c3.json 2>&1
timeout 600 python bench.py --config c4 --no-cpu-baseline > gpurun_out/r01h/bench_c4.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01h/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r01h/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mttkrp_fast -s 4 -c 2 -o gpurun_out/r01h/full_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01h/ncu_full.log 2>&1
echo done
