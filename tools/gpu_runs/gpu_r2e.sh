mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none -k regex:k_walk_bucket -c 1 --launch-skip 2"
timeout 600 $NCU -o gpurun_out/r2e_c2_main -f python bench.py --workload c2 --steps 1 --warmup 2 --no-cpu-baseline --c5-steps 0 > gpurun_out/r2e_ncu1.log 2>&1; echo n1=$?
timeout 600 $NCU -o gpurun_out/r2e_c5_main -f python bench.py --workload c5 --c5-log2-steps 40 --steps 1 --warmup 2 --no-cpu-baseline --c5-steps 0 > gpurun_out/r2e_ncu2.log 2>&1; echo n2=$?
TRITPERM_LIB=$PWD/paper_2407_20205_b200/lib/ab/lib_r1.so timeout 600 $NCU -o gpurun_out/r2e_c5_r1 -f python bench.py --workload c5 --c5-log2-steps 40 --steps 1 --warmup 2 --no-cpu-baseline --c5-steps 0 > gpurun_out/r2e_ncu3.log 2>&1; echo n3=$?
tools/ab_run.sh r2e "c3 c4 c5" main keys4 keys5 > gpurun_out/r2e_ab.txt 2>&1
