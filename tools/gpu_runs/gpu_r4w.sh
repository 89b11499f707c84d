mkdir -p gpurun_out
TRITPERM_LIB=$PWD/paper_2407_20205_b200/lib/ab/lib_c2nb8.so timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "c2 or bucketed or filter_list or options or smoke or large" > gpurun_out/r4w_pytest.log 2>&1; echo pytest_c2nb8=$? $(tail -1 gpurun_out/r4w_pytest.log)
tools/ab_run.sh r4w "c2" main c2nb8 > gpurun_out/r4w_ab.txt 2>&1
cat gpurun_out/r4w_ab.txt
