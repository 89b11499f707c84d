mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/r2x_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r2x_pytest.log
bash tools/gpu_ab.sh r2x -
NCU="ncu --set full --import-source on --clock-control none -k regex:k_walk_batch -c 1 --launch-skip 3"
timeout 900 $NCU -o gpurun_out/r2x_c3 -f python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r2x_ncu_c3.log 2>&1; echo ncu_c3=$?
