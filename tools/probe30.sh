# C5 (2000^3 r=64 FP32) FFMA blocking: 8x8 (G=8) vs 8x16 (G=4) tiles
mkdir -p gpurun_out/p30
timeout 600 python bench.py --config c5 --steps 10 --warmup 3 > gpurun_out/p30/bench_c5.json 2> gpurun_out/p30/bench_c5.err
NTF_FAST_ALT=4 timeout 600 python bench.py --config c5 --steps 10 --warmup 3 > gpurun_out/p30/bench_c5_alt4.json 2> gpurun_out/p30/bench_c5_alt4.err
echo done
