mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "montecarlo or table4 or tower or 3x3 or cli or census or smoke" > gpurun_out/r5h_pytest.log 2>&1; echo pytest=$? $(tail -1 gpurun_out/r5h_pytest.log)
timeout 600 python tools/table4.py --scale 0.01 --nmax 16 > gpurun_out/r5h_table4.jsonl 2>&1
python - <<'PY'
import json
for ln in open('gpurun_out/r5h_table4.jsonl'):
    d=json.loads(ln)
    if 'n' in d: print(d['n'], d['trials'], d['zero_count'], d['z_vs_paper'], d['seconds'], '%.3e'%d['terms_per_s'])
PY
