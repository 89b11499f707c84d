mkdir -p gpurun_out
TRITPERM_LIB=$PWD/paper_2407_20205_b200/lib/ab/lib_six10.so timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "bucketed or c2 or c3 or c4 or wide or large or range or n64" > gpurun_out/r4h_pytest.log 2>&1; echo pytest_six=$? $(tail -1 gpurun_out/r4h_pytest.log)
tools/ab_run.sh r4h "c2 c3 c4 c5" main six10 > gpurun_out/r4h_ab.txt 2>&1
cat gpurun_out/r4h_ab.txt
