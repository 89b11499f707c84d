# usage: tools/gpu_ab.sh TAG "ENV1" "ENV2" ...   (each ENV a space-separated list of VAR=value, "-" for none)
# -> gpurun_out/ab_TAG.txt: C2-C5 walk times per environment, two repetitions
TAG=$1; shift
mkdir -p gpurun_out
OUT=gpurun_out/ab_$TAG.txt; : > $OUT
for rep in 1 2; do for envs in "$@"; do for wl in c2 c3 c4 c5; do
  st=10; [ $wl = c3 ] && st=3; [ $wl = c5 ] && st=3
  E=""; [ "$envs" != "-" ] && E="$envs"
  env $E timeout 600 python bench.py --workload $wl --steps $st --warmup 2 --no-cpu-baseline --c5-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('%-40s' % '$envs', '$wl', 'ms %.3f' % d['ms_per_step'], 'walk %.3f' % r['walk_ms_avg'], 'frac %.3f' % r['frac'])" >> $OUT
done; done; done
cat $OUT
