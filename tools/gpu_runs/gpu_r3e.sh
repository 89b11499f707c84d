mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none -k regex:k_walk_batch -c 1 --launch-skip 3"
timeout 600 $NCU -o gpurun_out/r3e_c2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r3e_ncu_c2.log 2>&1; echo ncu_c2=$?
