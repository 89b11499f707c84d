# round-2 final-build measurement pass (min3 filter, six-entry loop, balanced verify, forced rows, batches of 8 for n > 32)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r4v_pytest.log 2>&1; echo pytest=$? $(tail -1 gpurun_out/r4v_pytest.log)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4v_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/r4v_bench_c2.log 2>&1; echo bench=$?
for wl in c1 c3 c4 c5; do timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --c5-steps 0 > gpurun_out/r4v_bench_$wl.log 2>&1; echo bench_$wl=$?; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r4v_bench_ref.log 2>&1; echo ref=$?
timeout 900 python tools/c5_full.py --skip-packed --out gpurun_out/r4v_c5_full.json > gpurun_out/r4v_c5.log 2>&1; echo c5=$?
timeout 900 python tools/pi50.py > gpurun_out/r4v_pi50.jsonl 2>&1; echo pi50=$?
timeout 300 python tools/c3_families.py > gpurun_out/r4v_fam.txt 2>&1; echo fam=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4v_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r4v_ncu_launch.log 2>&1; echo ncu_launch=$?
NCU="ncu --set full --import-source on --clock-control none -k regex:k_walk_batch -c 1 --launch-skip 3"
timeout 600 $NCU -o gpurun_out/r4v_c2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r4v_ncu_c2.log 2>&1; echo ncu_c2=$?
timeout 600 $NCU -o gpurun_out/r4v_c4 -f python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r4v_ncu_c4.log 2>&1; echo ncu_c4=$?
timeout 900 $NCU -o gpurun_out/r4v_c3 -f python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r4v_ncu_c3.log 2>&1; echo ncu_c3=$?
