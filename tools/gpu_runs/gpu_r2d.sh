mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "c3_all or integration or nccl or c5_config" > gpurun_out/r2d_pytest.log 2>&1; echo pytest=$?
tools/ab_run.sh r2d "c2" main k3f14 > gpurun_out/r2d_ab_c2.txt 2>&1
tools/ab_run.sh r2d45 "c4 c5" main r1 > gpurun_out/r2d_ab_c45.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_case.py > gpurun_out/r2d_memcheck.log 2>&1; echo memcheck=$?
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python tools/sanitize_case.py > gpurun_out/r2d_racecheck.log 2>&1; echo racecheck=$?
