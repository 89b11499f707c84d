mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > gpurun_out/r4t_pytest.log 2>&1; echo pytest_main=$? $(tail -1 gpurun_out/r4t_pytest.log)
TRITPERM_LIB=$PWD/paper_2407_20205_b200/lib/ab/lib_nb8all.so timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -k "not bounds_checked" > gpurun_out/r4t_pytest8.log 2>&1; echo pytest_nb8all=$? $(tail -1 gpurun_out/r4t_pytest8.log)
tools/ab_run.sh r4t "c2 c3 c4 c5" main nb8n nb8all > gpurun_out/r4t_ab.txt 2>&1
cat gpurun_out/r4t_ab.txt
TRITPERM_LIB=$PWD/paper_2407_20205_b200/lib/ab/lib_nb8all.so timeout 300 python tools/c3_families.py > gpurun_out/r4t_fam.txt 2>&1; cat gpurun_out/r4t_fam.txt | cut -c1-110
