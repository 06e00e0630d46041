# consumer-warp sweep for C4 (FP32, r = 32) and C3 (DMMA, r = 16)
mkdir -p gpurun_out/p31
run() { name=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 100 --warmup 5 ${CFG} 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), [round(x*1e3,1) for x in d['roofline']['per_mode_ms']])" >> gpurun_out/p31/sweep.txt 2>&1; }
for CFG in "--config c4" "--config c3"; do
  echo "== $CFG" >> gpurun_out/p31/sweep.txt
  run base X=1
  run cons6 NTF_FAST_CONS=6
  run cons8 NTF_FAST_CONS=8
  run np1 NTF_FAST_NP=1
  run np1cons8 NTF_FAST_NP=1 NTF_FAST_CONS=8
  run np1cons12 NTF_FAST_NP=1 NTF_FAST_CONS=12
done
echo done
