mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none -k regex:k_walk_batch -c 1 --launch-skip 3"
timeout 900 $NCU -o gpurun_out/r2v_c3 -f python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r2v_ncu_c3.log 2>&1; echo ncu_c3=$?
timeout 900 $NCU -o gpurun_out/r2v_c5 -f python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r2v_ncu_c5.log 2>&1; echo ncu_c5=$?
