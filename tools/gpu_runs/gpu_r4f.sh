mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x -k "not c5_config_full" > gpurun_out/r4f_pytest.log 2>&1; echo pytest=$? $(tail -1 gpurun_out/r4f_pytest.log)
tools/ab_run.sh r4f "c2 c3 c4 c5" main > gpurun_out/r4f_ab.txt 2>&1
cat gpurun_out/r4f_ab.txt
NCU="ncu --set full --import-source on --clock-control none -k regex:k_walk_batch -c 1 --launch-skip 3"
timeout 600 $NCU -o gpurun_out/r4f_c2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r4f_ncu_c2.log 2>&1; echo ncu_c2=$?
