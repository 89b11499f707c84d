mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/r3k_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/r3k_pytest.log
L=$PWD/paper_2407_20205_b200/lib/ab
bash tools/gpu_ab.sh r3k - TRITPERM_LIB=$L/lib_head.so
python tools/c3_families.py > gpurun_out/r3k_fam.txt 2>&1; cat gpurun_out/r3k_fam.txt
