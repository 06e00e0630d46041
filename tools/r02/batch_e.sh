#!/bin/bash
# r02e: config parity with the measured bars, new GPU tests (drain, limits, determinism), full GPU suite, smoke.
O=gpurun_out/r02e; mkdir -p $O
NTF_PARITY_REPORT=$O timeout 900 python -m pytest tests/test_config_parity.py tests/test_sharded_gpu.py -m gpu -q -rA > $O/pytest_new.log 2>&1; echo "rc=$?" >> $O/pytest_new.log
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
echo done
