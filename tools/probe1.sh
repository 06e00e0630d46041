./tools/fp64_latency; ./tools/chain_probe
python tools/nnls_bench.py 300 20; NTF_NNLS_Q=1 python tools/nnls_bench.py 300 20
python tools/nnls_bench.py 100 16; python tools/nnls_bench.py 500 32; python tools/nnls_bench.py 2000 64
python tools/tune.py c2 10 2>&1 | tail -3
