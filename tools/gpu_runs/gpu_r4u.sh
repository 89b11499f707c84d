mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > gpurun_out/r4u_pytest.log 2>&1; echo pytest_main=$? $(tail -1 gpurun_out/r4u_pytest.log)
TRITPERM_LIB=$PWD/paper_2407_20205_b200/lib/ab/lib_nbw8.so timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -k "not bounds_checked" > gpurun_out/r4u_pytest8.log 2>&1; echo pytest_nbw8=$? $(tail -1 gpurun_out/r4u_pytest8.log)
tools/ab_run.sh r4u "c2 c3 c4 c5" main nbw8 > gpurun_out/r4u_ab.txt 2>&1
cat gpurun_out/r4u_ab.txt
