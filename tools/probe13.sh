timeout 900 python -m pytest tests/test_large.py -x -q -s 2>&1 | tail -5
timeout 1200 python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"; tail -c 1500 gpurun_out/bench_c5.json
