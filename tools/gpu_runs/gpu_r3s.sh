mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "c4 or c5 or n64 or wide or distributed or range" > gpurun_out/r3s_pytest.log 2>&1; echo pytest=$? $(tail -1 gpurun_out/r3s_pytest.log)
TRITPERM_STICKY=2 timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "c4 or c5 or n64 or wide or distributed or range or bucketed" > gpurun_out/r3s_pytest2.log 2>&1; echo pytest_sticky2=$? $(tail -1 gpurun_out/r3s_pytest2.log)
bash tools/gpu_ab.sh r3s -
