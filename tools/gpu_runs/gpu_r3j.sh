mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/r3j_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/r3j_pytest.log
L=$PWD/paper_2407_20205_b200/lib/ab
bash tools/gpu_ab.sh r3j - TRITPERM_LIB=$L/lib_head.so
