mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider --durations=8 > gpurun_out/r4a_pytest.log 2>&1; echo pytest=$?
tail -14 gpurun_out/r4a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4a_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/r4a_bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/r4a_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/r4a_ref.log 2>&1; echo ref=$?
tail -1 gpurun_out/r4a_ref.log
