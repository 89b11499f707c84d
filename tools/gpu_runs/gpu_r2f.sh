mkdir -p gpurun_out
L=$PWD/paper_2407_20205_b200/lib/ab
TRITPERM_LIB=$L/lib_combo.so timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "bucket or c3 or coverage or dense or filter or n64 or c4_c5 or pi50 or variant" > gpurun_out/r2f_pytest_combo.log 2>&1; echo pytest_combo=$?
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "checked" > gpurun_out/r2f_pytest_checked.log 2>&1; echo checked=$?
tools/ab_run.sh r2f "c2" main k3f14 > gpurun_out/r2f_ab_c2.txt 2>&1
tools/ab_run.sh r2f345 "c3 c4 c5" main keys4 r1 > gpurun_out/r2f_ab_c345.txt 2>&1
