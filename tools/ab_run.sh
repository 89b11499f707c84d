#!/bin/bash
# On the GPU box: bench lines of library variants (tools/ab_build.sh) for the
# bucketed workloads.  tools/ab_run.sh TAG "c2 c4 c5" variant1 variant2 ...
# -> gpurun_out/ab_TAG.jsonl (one line per variant x workload, with "variant")
REPO=$(cd "$(dirname "$0")/.." && pwd)
TAG=$1; WLS=$2; shift 2
OUT=$REPO/gpurun_out/ab_$TAG.jsonl
mkdir -p "$REPO/gpurun_out"; : > "$OUT"
for rep in 1 2; do
for v in "$@"; do
  for wl in $WLS; do
    if [ "$v" = "main" ]; then LIB=""; else LIB=$REPO/paper_2407_20205_b200/lib/ab/lib_$v.so; fi
    steps=10; [ "$wl" = "c3" ] && steps=3; [ "$wl" = "c5" ] && steps=3
    line=$(TRITPERM_LIB=$LIB timeout 600 python "$REPO/bench.py" --workload $wl --steps $steps --warmup 2 \
           --no-cpu-baseline --c5-steps 0 2>"$REPO/gpurun_out/ab_${TAG}_${v}_${wl}.err" | tail -1)
    echo "{\"variant\": \"$v\", \"rep\": $rep, \"line\": ${line:-null}}" >> "$OUT"
  done
done
done
python - "$OUT" <<'PY'
import json, sys
for ln in open(sys.argv[1]):
    d = json.loads(ln)
    l = d["line"] or {}
    r = l.get("roofline") or {}
    print(d["variant"], d["rep"], l.get("config", {}).get("n"), "ms/step %.3f" % l.get("ms_per_step", -1),
          "walk %.3f" % (r.get("walk_ms_avg") or -1), "frac %.3f" % (r.get("frac") or -1))
PY
