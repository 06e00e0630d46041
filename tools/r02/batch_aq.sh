#!/bin/bash
# NNLS timing experiments: variants of the stream kernel with parts compiled out (-DNTF_NNLS_X=mask;
# wrong results, timing only): bits 0-6 per-column work, 128 ignore the stop rule, 256 reducer polls
# without nanosleep, 512 the rows' gate polls without nanosleep. Host-timed 50-sweep calls (300 x 20).
O=gpurun_out/r02aq; mkdir -p $O
for X in "$@"; do
  echo "X=$X $(NTF_B200_LIB=build/var/libntf_x$X.so timeout 120 python tools/nnls_bench.py 300 20 2>&1 | head -1)"
done | tee -a $O/nnls_variants.txt
