mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "bucketed or c2_batch or c3 or n64 or three or montecarlo or checked" > gpurun_out/r3m_pytest.log 2>&1; echo pytest=$?
tail -1 gpurun_out/r3m_pytest.log
L=$PWD/paper_2407_20205_b200/lib/ab
bash tools/gpu_ab.sh r3m - TRITPERM_LIB=$L/lib_head.so
