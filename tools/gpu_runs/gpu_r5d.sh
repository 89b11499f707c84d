mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > gpurun_out/r5d_pytest.log 2>&1; echo pytest=$? $(tail -1 gpurun_out/r5d_pytest.log)
timeout 300 python tools/c3_families.py > gpurun_out/r5d_fam.txt 2>&1; echo fam=$?; cat gpurun_out/r5d_fam.txt
tools/ab_run.sh r5d "c2 c3 c4 c5" main > gpurun_out/r5d_ab.txt 2>&1
cat gpurun_out/r5d_ab.txt
