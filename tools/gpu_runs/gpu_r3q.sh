mkdir -p gpurun_out
: > gpurun_out/r3q.txt
for rep in 1 2; do for mi in 2 3 4 6 8 12; do for wl in c4; do
  TRITPERM_BUCKET_MIN_ITEMS=$mi timeout 600 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline --c5-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('min_items', $mi, '$wl', d['ms_per_step'])" >> gpurun_out/r3q.txt
done; done; done
cat gpurun_out/r3q.txt
