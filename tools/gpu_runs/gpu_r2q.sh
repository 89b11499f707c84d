mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/r2q_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r2q_pytest.log
TRITPERM_BATCH=0 timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "bucketed or c2_batch or c3 or async or n64 or three or montecarlo" > gpurun_out/r2q_pytest_old.log 2>&1; echo pytest_old=$?
tail -1 gpurun_out/r2q_pytest_old.log
bash tools/gpu_ab.sh r2q - TRITPERM_BATCH=0
