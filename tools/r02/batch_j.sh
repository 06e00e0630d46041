#!/bin/bash
O=gpurun_out/r02j; mkdir -p $O
timeout 600 python -m pytest tests/test_tucker.py -m gpu -q > $O/pytest_tucker.log 2>&1; echo "rc=$?" >> $O/pytest_tucker.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"mttkrp_sk" -s 4 -c 2 -o $O/full_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"mttkrp_sk" -s 8 -c 2 -o $O/full_c3 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_c3.log 2>&1
echo done
