# NNLS stream kernel: row lanes per CTA (cluster size) sweep at C2/C3
mkdir -p gpurun_out/p45
run() { name=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 100 --warmup 5 ${CFG} 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), d['final_f'], d['restarts'])" >> gpurun_out/p45/sweep.txt 2>&1; }
for CFG in "--config c2" "--config c3"; do
  echo "== $CFG" >> gpurun_out/p45/sweep.txt
  run base X=1
  run rl64 NTF_NNLS_ROW_LANES=64
  run rl128 NTF_NNLS_ROW_LANES=128
  run rl80 NTF_NNLS_ROW_LANES=80
done
echo done
