mkdir -p gpurun_out
L=paper_2407_20205_b200/lib/ab
TRITPERM_LIB=$PWD/$L/lib_paired.so timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "bucketed or c2_batch or c3 or async or smoke or n64 or three or montecarlo" > gpurun_out/r2n_pytest_paired.log 2>&1; echo pytest_paired=$?
tail -2 gpurun_out/r2n_pytest_paired.log
bash tools/gpu_ab.sh r2n - "TRITPERM_LIB=$PWD/$L/lib_paired.so"
