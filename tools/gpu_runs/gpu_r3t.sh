mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r3t_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r3t_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3t_smoke.log 2>&1; echo smoke=$?
