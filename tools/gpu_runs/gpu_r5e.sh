# C3 after the segments: bench line, families, ncu summary; plus the default bench line and smoke on the final build
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5e_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/r5e_bench_c2.log 2>&1; echo bench=$?
for wl in c3 c4 c5; do timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --c5-steps 0 > gpurun_out/r5e_bench_$wl.log 2>&1; echo bench_$wl=$?; done
timeout 300 python tools/c3_families.py > gpurun_out/r5e_fam.txt 2>&1; echo fam=$?
NCU="ncu --set full --import-source on --clock-control none -k regex:k_walk_batch -c 1 --launch-skip 3"
timeout 900 $NCU -o gpurun_out/r5e_c3 -f python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline --c5-steps 0 > gpurun_out/r5e_ncu_c3.log 2>&1; echo ncu_c3=$?
