#!/bin/bash
O=gpurun_out/r02z; mkdir -p $O
run() { cfg=$1; tag=$2; shift; shift; env "$@" timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 30 --warmup 5 > $O/${cfg}_$tag.json 2>/dev/null; python -c "
import json; d=json.load(open('$O/${cfg}_$tag.json')); r=d['roofline']; print('$cfg $tag', round(d['value'],1), round(r['fma_tflops'],1), [round(x*1000,1) for x in r['per_mode_ms']])" >> $O/sweep.txt; }
run c4 base NTF_X=0
run c4 mw8 NTF_SK_MW=8
run c4 np4 NTF_SK_NP=4
run c4 st4 NTF_SK_STAGES=4
run c4 naw2 NTF_SK_NAW=2
run c5 base NTF_X=0
run c5 mw8 NTF_SK_MW=8
echo done
