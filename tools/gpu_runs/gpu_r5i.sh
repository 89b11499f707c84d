mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r5i_pytest.log 2>&1; echo pytest=$? $(tail -1 gpurun_out/r5i_pytest.log)
timeout 2400 python tools/table4.py --scale 1.0 > gpurun_out/r5i_table4.jsonl 2>&1; echo table4=$?
tail -1 gpurun_out/r5i_table4.jsonl
