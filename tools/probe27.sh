# COL box pitch (conflict-free DMMA loads) + producer/consumer sweeps at C2/C3
mkdir -p gpurun_out/p27
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p27/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p27/pytest_gpu.log
run() { name=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 100 --warmup 5 ${CFG} 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), [round(x*1e3,1) for x in d['roofline']['per_mode_ms']])" >> gpurun_out/p27/sweep.txt 2>&1; }
for CFG in "--config c2" "--config c3"; do
  echo "== $CFG" >> gpurun_out/p27/sweep.txt
  run base X=1
  run np4 NTF_FAST_NP=4
  run np1 NTF_FAST_NP=1
  run cons4 NTF_FAST_CONS=4
  run cons12 NTF_FAST_CONS=12
  run st4 NTF_FAST_STAGES=4
done
echo done
