mkdir -p gpurun_out
L=$PWD/paper_2407_20205_b200/lib/ab
TRITPERM_LIB=$L/lib_f14k2.so timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "bucketed or c2_batch or async or smoke or filter" > gpurun_out/r2i_pytest_f14k2.log 2>&1; echo pytest=$?
tools/ab_run.sh r2i "c2" main f14k2 k3f14 > gpurun_out/r2i_ab.txt 2>&1
tools/ab_run.sh r2i1 "c1" main r1 > gpurun_out/r2i_ab1.txt 2>&1
