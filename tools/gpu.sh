#!/bin/bash
# usage: tools/gpu.sh NAME 'command'  — runs on the B200 box from the repo root,
# log in gpurun_out/NAME.log (background-friendly).
cd /root/repo || exit 1
name=$1; shift
timeout 2700 /usr/local/graft/bin/gpurun --timeout ${GPU_TIMEOUT:-900} -- "$@" > gpurun_out/$name.log 2>&1
