mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r4i_pytest.log 2>&1; echo pytest=$? $(tail -1 gpurun_out/r4i_pytest.log)
tools/ab_run.sh r4i "c2 c3 c4 c5" main > gpurun_out/r4i_ab.txt 2>&1
cat gpurun_out/r4i_ab.txt
