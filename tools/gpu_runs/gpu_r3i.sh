mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/r3i_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r3i_pytest.log
L=$PWD/paper_2407_20205_b200/lib/ab
TRITPERM_LIB=$L/lib_nb8.so timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "bucketed or c2_batch or c3 or n64 or three or montecarlo" > gpurun_out/r3i_pytest_nb8.log 2>&1; echo pytest_nb8=$?
bash tools/gpu_ab.sh r3i - TRITPERM_LIB=$L/lib_nb8.so TRITPERM_LIB=$L/lib_head.so
