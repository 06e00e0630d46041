timeout 900 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -E "C5|passed|failed|Error" | tail -5
timeout 1500 python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"; tail -c 2500 gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5.err
