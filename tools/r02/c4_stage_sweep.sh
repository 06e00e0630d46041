#!/bin/bash
for cfg in "" "NTF_SK_F32A=8 NTF_SK_MW=8 NTF_SK_NP=1" "NTF_SK_NP=1" "NTF_SK_NP=3" "NTF_SK_F32A=8 NTF_SK_MW=8 NTF_SK_NP=1 NTF_SK_STAGES=2"; do
  env $cfg timeout 300 python bench.py --config c4 --no-cpu-baseline --steps 30 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', round(d['value'],1), d['roofline']['per_mode_ms'][:2], d['roofline'].get('fma_frac'))"
done
