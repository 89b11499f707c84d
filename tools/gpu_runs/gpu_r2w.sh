mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/r2w_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r2w_pytest.log
bash tools/gpu_ab.sh r2w -
