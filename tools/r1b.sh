set -u
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpuinfo.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench_r01b.json 2> $O/bench_r01b.err; echo "bench rc=$?"
for c in c3 c4; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_${c}.json 2> $O/bench_${c}.err; echo "bench $c rc=$?"; done
