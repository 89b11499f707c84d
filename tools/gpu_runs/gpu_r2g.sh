# round-2 full pass on the default build: tests, smoke, bench lines, C5/Pi50 full runs, ncu
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r2g_pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/r2g_bench_c2.log 2>&1; echo bench=$?
for wl in c1 c3 c4 c5; do timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --c5-steps 0 > gpurun_out/r2g_bench_$wl.log 2>&1; echo bench_$wl=$?; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2g_bench_ref.log 2>&1; echo ref=$?
timeout 900 python tools/c5_full.py --skip-packed --out gpurun_out/r2g_c5_full.json > gpurun_out/r2g_c5.log 2>&1; echo c5=$?
timeout 900 python tools/pi50.py > gpurun_out/r2g_pi50.jsonl 2>&1; echo pi50=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2g_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r2g_ncu_launch.log 2>&1; echo ncu_launch=$?
NCU="ncu --set full --import-source on --clock-control none -k regex:k_walk_bucket -c 1 --launch-skip 3"
timeout 600 $NCU -o gpurun_out/r2g_c2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r2g_ncu_c2.log 2>&1; echo ncu_c2=$?
timeout 600 $NCU -o gpurun_out/r2g_c4 -f python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r2g_ncu_c4.log 2>&1; echo ncu_c4=$?
timeout 600 $NCU -o gpurun_out/r2g_c3 -f python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r2g_ncu_c3.log 2>&1; echo ncu_c3=$?
