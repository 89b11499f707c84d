mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -k "filter_list_lengths" > gpurun_out/r4m_pytest.log 2>&1; echo pytest=$? $(tail -1 gpurun_out/r4m_pytest.log)
tail -30 gpurun_out/r4m_pytest.log
