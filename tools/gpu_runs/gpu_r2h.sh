mkdir -p gpurun_out
: > gpurun_out/r2h_items.txt
for mi in 4 16 64; do for wl in c4 c5 c3; do
  st=10; [ $wl = c3 ] && st=3; [ $wl = c5 ] && st=3
  TRITPERM_BUCKET_MIN_ITEMS=$mi python bench.py --workload $wl --steps $st --warmup 2 --no-cpu-baseline --c5-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('min_items', $mi, '$wl', d['ms_per_step'])" >> gpurun_out/r2h_items.txt
done; done
tools/ab_run.sh r2h "c2 c3 c4" main vote1 > gpurun_out/r2h_ab.txt 2>&1
python bench.py --workload c1 --no-cpu-baseline --c5-steps 0 > gpurun_out/r2h_c1.log 2>&1
