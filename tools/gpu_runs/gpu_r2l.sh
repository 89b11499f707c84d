# ncu --set full of k_walk_batch on C2 and C4 (source lines)
mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none -k regex:k_walk_batch -c 1 --launch-skip 3"
timeout 600 $NCU -o gpurun_out/r2l_c2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r2l_ncu_c2.log 2>&1; echo ncu_c2=$?
timeout 600 $NCU -o gpurun_out/r2l_c4 -f python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r2l_ncu_c4.log 2>&1; echo ncu_c4=$?
