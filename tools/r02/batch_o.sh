#!/bin/bash
O=gpurun_out/r02o; mkdir -p $O
run() { cfg=$1; tag=$2; shift; shift; env "$@" timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 60 --warmup 5 > $O/${cfg}_$tag.json 2>/dev/null; python -c "
import json; d=json.load(open('$O/${cfg}_$tag.json')); print('$cfg $tag', round(d['value'],1), round(d['roofline']['frac'],3), [round(x*1000,1) for x in d['roofline']['per_mode_ms']])" >> $O/sweep.txt; }
run c3 np2 NTF_SK_NP=2
run c3 np4 NTF_SK_NP=4
run c3 np4mw8 NTF_SK_NP=4 NTF_SK_MW=8
run c2 np4 NTF_SK_NP=4
run c2 np4st8 NTF_SK_NP=4 NTF_SK_STAGES=8
run c2 np4mw8 NTF_SK_NP=4 NTF_SK_MW=8
run c2 np2st2 NTF_SK_NP=2 NTF_SK_STAGES=2
echo done
