mkdir -p gpurun_out
L=$PWD/paper_2407_20205_b200/lib/ab
for v in nonvol emaj emajnv; do
TRITPERM_LIB=$L/lib_$v.so timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "bucketed or c2_batch or c3 or n64" > gpurun_out/r3o_pytest_$v.log 2>&1; echo pytest_$v=$? $(tail -1 gpurun_out/r3o_pytest_$v.log)
done
bash tools/gpu_ab.sh r3o - TRITPERM_LIB=$L/lib_nonvol.so TRITPERM_LIB=$L/lib_emaj.so TRITPERM_LIB=$L/lib_emajnv.so
