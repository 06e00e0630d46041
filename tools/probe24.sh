# full ncu captures: tree kernel and NNLS kernel (C2), Y_R COL pass (C3)
mkdir -p gpurun_out/p24
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tree_mttkrp -s 4 -c 1 -o gpurun_out/p24/tree_c2 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p24/ncu_tree.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:nnls_stream -s 6 -c 1 -o gpurun_out/p24/nnls_c2 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p24/ncu_nnls.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mttkrp_fast -s 2 -c 2 -o gpurun_out/p24/fast_c3 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p24/ncu_fast.log 2>&1
echo done
