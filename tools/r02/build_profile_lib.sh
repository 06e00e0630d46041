#!/bin/bash
# Builds a diagnostics copy of libntf_b200.so with the NNLS cycle stamps
# compiled in (-DNTF_NNLS_PROFILE=1) under /tmp/ntfprof; use it with
# NTF_B200_LIB=/tmp/ntfprof/libntf_b200.so (tools/r02/nnls_phases.py).
set -e
rm -rf /tmp/ntfprof && mkdir -p /tmp/ntfprof/src
cp -r paper_2001_04321_b200/csrc /tmp/ntfprof/src/csrc
mkdir -p /tmp/ntfprof/include && cp include/*.h /tmp/ntfprof/include/
cd /tmp/ntfprof/src/csrc
sed -i 's|\.\./\.\./include/ntf_b200.h|../../include/ntf_b200.h|' Makefile
make -j16 OUT=/tmp/ntfprof/libntf_b200.so BUILD=/tmp/ntfprof/build NVEXTRA="-DNTF_NNLS_PROFILE=1 -I/tmp/ntfprof/include" > /tmp/ntfprof/build.log 2>&1
ls -la /tmp/ntfprof/libntf_b200.so
