#!/bin/bash
O=gpurun_out/r02ao; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_vs_reference.py -m gpu -q 2>&1 | tail -12
timeout 600 python tools/r02/paths_probe.py > $O/paths_probe.json 2> $O/paths_probe.err; echo "probe rc=$?"; cat $O/paths_probe.json; tail -3 $O/paths_probe.err
