mkdir -p gpurun_out
L=$PWD/paper_2407_20205_b200/lib/ab
for v in pf u2; do
TRITPERM_LIB=$L/lib_$v.so timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "bucketed or c2_batch or c3 or n64 or three or montecarlo" > gpurun_out/r3a_pytest_$v.log 2>&1; echo pytest_$v=$?
done
bash tools/gpu_ab.sh r3a - TRITPERM_LIB=$L/lib_pf.so TRITPERM_LIB=$L/lib_u2.so
