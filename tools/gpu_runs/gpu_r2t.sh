mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/r2t_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r2t_pytest.log
L=$PWD/paper_2407_20205_b200/lib/ab
bash tools/gpu_ab.sh r2t - TRITPERM_LIB=$L/lib_notab.so TRITPERM_LIB=$L/lib_notriple.so TRITPERM_LIB=$L/lib_noflat.so
