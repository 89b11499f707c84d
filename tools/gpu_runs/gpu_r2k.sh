# batched walk: GPU suite + A/B against k_walk_bucket (TRITPERM_BATCH=0)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/r2k_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r2k_pytest.log
: > gpurun_out/r2k_ab.txt
for rep in 1 2; do for b in 1 0; do for wl in c2 c3 c4 c5; do
  st=10; [ $wl = c3 ] && st=3; [ $wl = c5 ] && st=3
  TRITPERM_BATCH=$b timeout 600 python bench.py --workload $wl --steps $st --warmup 2 --no-cpu-baseline --c5-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('batch', $b, '$wl', 'ms %.3f' % d['ms_per_step'], 'walk %.3f' % r['walk_ms_avg'], 'frac %.3f' % r['frac'])" >> gpurun_out/r2k_ab.txt
done; done; done
cat gpurun_out/r2k_ab.txt
