mkdir -p gpurun_out
timeout 2400 python tools/table4.py --scale 1.0 > gpurun_out/r4l_table4.jsonl 2>&1; echo rc=$?
tail -1 gpurun_out/r4l_table4.jsonl
