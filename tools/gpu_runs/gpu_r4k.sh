mkdir -p gpurun_out
timeout 900 python tools/table4.py --scale 0.01 > gpurun_out/r4k_table4_scale001.jsonl 2>&1; echo rc=$?
python - <<'PY'
import json
for ln in open('gpurun_out/r4k_table4_scale001.jsonl'):
    try: d=json.loads(ln)
    except Exception: print(ln.rstrip()); continue
    if 'n' in d: print(d['n'], d['trials'], d['zero_fraction'], d['z_vs_paper'], d['seconds'], '%.3e'%d['terms_per_s'], d['kernel'])
    else: print(d)
PY
