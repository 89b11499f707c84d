# Re-entry check of HEAD on the B200: full GPU suite, smoke, default bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r2j_pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2j_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/r2j_bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/r2j_bench.log
