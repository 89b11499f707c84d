mkdir -p gpurun_out
L=$PWD/paper_2407_20205_b200/lib/ab
for v in small3 big5; do
TRITPERM_LIB=$L/lib_$v.so timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "bucketed or c2_batch or c3 or async or smoke or n64 or three or montecarlo" > gpurun_out/r2o_pytest_$v.log 2>&1; echo pytest_$v=$?
tail -1 gpurun_out/r2o_pytest_$v.log
done
bash tools/gpu_ab.sh r2o - "TRITPERM_LIB=$L/lib_small3.so" "TRITPERM_LIB=$L/lib_big5.so"
