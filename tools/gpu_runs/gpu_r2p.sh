# ncu source-line profiles of the 3-key (n < 28) and 5-key (n >= 28) batched walks
mkdir -p gpurun_out
L=$PWD/paper_2407_20205_b200/lib/ab
NCU="ncu --set full --import-source on --clock-control none -k regex:k_walk_batch -c 1 --launch-skip 3"
TRITPERM_LIB=$L/lib_small3.so timeout 600 $NCU -o gpurun_out/r2p_c2s3 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r2p_ncu_c2.log 2>&1; echo ncu_c2=$?
TRITPERM_LIB=$L/lib_big5.so timeout 600 $NCU -o gpurun_out/r2p_c4b5 -f python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r2p_ncu_c4.log 2>&1; echo ncu_c4=$?
TRITPERM_LIB=$L/lib_big5.so timeout 600 $NCU -o gpurun_out/r2p_c3b5 -f python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r2p_ncu_c3.log 2>&1; echo ncu_c3=$?
