#!/bin/bash
O=gpurun_out/r02m; mkdir -p $O
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 60 --warmup 5 > $O/c2_$tag.json 2>/dev/null; python -c "
import json; d=json.load(open('$O/c2_$tag.json')); print('$tag', round(d['value'],1), [round(x*1000,1) for x in d['roofline']['per_mode_ms']])" >> $O/sweep.txt; }
run st2naw4 NTF_SK_STAGES=2 NTF_SK_NAW=4
run st4naw2 NTF_SK_STAGES=4 NTF_SK_NAW=2
run st3naw2 NTF_SK_NAW=2 NTF_SK_STAGES=3
run st2naw2 NTF_SK_STAGES=2 NTF_SK_NAW=2
run st4naw4mw8 NTF_SK_STAGES=4 NTF_SK_NAW=4 NTF_SK_MW=8
run st2naw4mw8 NTF_SK_STAGES=2 NTF_SK_NAW=4 NTF_SK_MW=8
run np1st4 NTF_SK_NP=1 NTF_SK_STAGES=4 NTF_SK_NAW=4
run old NTF_SK=0
echo done
