#!/bin/bash
# r02b: new parity tests (config fixtures, sharded path, one-rank NCCL), full GPU suite, smoke,
# compute-sanitizer on small production-path runs, bench lines.
O=gpurun_out/r02b; mkdir -p $O
timeout 900 python -m pytest tests/test_config_parity.py tests/test_sharded_gpu.py -m gpu -q -s -rA > $O/pytest_new.log 2>&1; echo "rc=$?" >> $O/pytest_new.log
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/r02/sanitize_case.py > $O/sanitizer_$tool.log 2>&1; echo "rc=$?" >> $O/sanitizer_$tool.log
done
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config c4 --no-cpu-baseline > $O/bench_c4_her.json 2> $O/bench_c4_her.err
timeout 600 python bench.py --config c4 --algo ao --no-cpu-baseline > $O/bench_c4_ao.json 2> $O/bench_c4_ao.err
echo done
