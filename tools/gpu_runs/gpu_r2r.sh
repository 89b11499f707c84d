# re-entry verification of HEAD on a fresh box: smoke, GPU suite, bench lines, reference arm, launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2r_smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r2r_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r2r_pytest.log
timeout 600 python bench.py > gpurun_out/r2r_bench_c2.log 2>&1; echo bench=$?
for wl in c1 c3 c4 c5; do timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --c5-steps 0 > gpurun_out/r2r_bench_$wl.log 2>&1; echo bench_$wl=$?; done
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2r_bench_ref.log 2>&1; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2r_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r2r_ncu_launch.log 2>&1; echo ncu_launch=$?
nproc; lscpu | grep "Model name"
