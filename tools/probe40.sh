# dimension-tree split h = 1 (tall COL partial) vs h = N-1 (tall ROW partial) at C2/C4
mkdir -p gpurun_out/p40
run() { name=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 100 --warmup 5 ${CFG} 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), [round(x*1e3,1) for x in d['roofline']['per_mode_ms']])" >> gpurun_out/p40/sweep.txt 2>&1; }
for CFG in "--config c2" "--config c4"; do
  echo "== $CFG" >> gpurun_out/p40/sweep.txt
  run base X=1
  run split1 NTF_TREE_SPLIT=1
done
echo done
