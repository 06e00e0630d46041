#!/bin/bash
# r02c: config parity deviation profiles, NNLS phases, ncu full captures (source) of the C2/C3 hot kernels.
O=gpurun_out/r02c; mkdir -p $O
NTF_PARITY_REPORT=$O timeout 900 python -m pytest tests/test_config_parity.py -m gpu -q > $O/pytest_cfg.log 2>&1; echo "rc=$?" >> $O/pytest_cfg.log
for c in c2 c3 c4; do timeout 300 python tools/r02/nnls_phases.py $c 50 > $O/nnls_phases_$c.txt 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"mttkrp_fast|nnls_stream|tree_mttkrp" -s 12 -c 4 -o $O/full_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"mttkrp_fast" -s 8 -c 2 -o $O/full_c3 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_c3.log 2>&1
ls -la $O
echo done
