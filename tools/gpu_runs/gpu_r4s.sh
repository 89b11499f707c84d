mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r4s_pytest.log 2>&1; echo pytest=$? $(tail -1 gpurun_out/r4s_pytest.log)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4s_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/r4s_bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/r4s_bench.log | cut -c1-400
tools/ab_run.sh r4s "c3 c4 c5" main > gpurun_out/r4s_ab.txt 2>&1; cat gpurun_out/r4s_ab.txt
