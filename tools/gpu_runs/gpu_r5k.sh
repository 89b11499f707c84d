mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r5k_pytest.log 2>&1; echo pytest=$? $(tail -1 gpurun_out/r5k_pytest.log)
tools/ab_run.sh r5k "c2 c4 c5" main > gpurun_out/r5k_ab.txt 2>&1; cat gpurun_out/r5k_ab.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5k_launches_c4.csv python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r5k_ncu.log 2>&1; echo ncu=$?
