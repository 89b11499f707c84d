mkdir -p gpurun_out
L=$PWD/paper_2407_20205_b200/lib/ab
NCU="ncu --set full --import-source on --clock-control none -k regex:k_walk_batch -c 1 --launch-skip 3"
timeout 600 $NCU -o gpurun_out/r3n_carry -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r3n_1.log 2>&1; echo ncu1=$?
TRITPERM_LIB=$L/lib_head.so timeout 600 $NCU -o gpurun_out/r3n_head -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r3n_2.log 2>&1; echo ncu2=$?
