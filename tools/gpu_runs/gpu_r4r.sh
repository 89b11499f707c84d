mkdir -p gpurun_out
TRITPERM_LIB=$PWD/paper_2407_20205_b200/lib/ab/lib_nb8.so timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "c3 or n30 or filter_list or large or bucketed or options" > gpurun_out/r4r_pytest.log 2>&1; echo pytest_nb8=$? $(tail -1 gpurun_out/r4r_pytest.log)
tools/ab_run.sh r4r "c3" main nb8 > gpurun_out/r4r_ab.txt 2>&1
cat gpurun_out/r4r_ab.txt
TRITPERM_LIB=$PWD/paper_2407_20205_b200/lib/ab/lib_nb8.so timeout 300 python tools/c3_families.py > gpurun_out/r4r_fam.txt 2>&1; cat gpurun_out/r4r_fam.txt | cut -c1-110
