#!/bin/bash
# Round-1 re-measure (r01g): GPU tests, smoke, bench lines, reference arm, launch list.
mkdir -p gpurun_out/r01g
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r01g/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r01g/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r01g/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01g/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r01g/bench_c2.json 2> gpurun_out/r01g/bench_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01g/bench_ref.json 2> gpurun_out/r01g/bench_ref.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/r01g/bench_c3.json 2>&1
timeout 600 python bench.py --config c4 --no-cpu-baseline > gpurun_out/r01g/bench_c4.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01g/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r01g/ncu_launch.log 2>&1

timeout 600 ncu --set full --import-source on --clock-control none -k regex:mttkrp_fast -s 4 -c 2 -o gpurun_out/r01g/full_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01g/ncu_full.log 2>&1

timeout 900 python bench.py --config c5 --steps 10 --warmup 3 > gpurun_out/r01g/bench_c5.json 2> gpurun_out/r01g/bench_c5.err
echo done3
