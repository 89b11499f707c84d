mkdir -p gpurun_out
for v in main t4 main t4; do
  if [ "$v" = "main" ]; then LIB=""; else LIB=$PWD/paper_2407_20205_b200/lib/ab/lib_$v.so; fi
  echo "== $v"
  TRITPERM_LIB=$LIB timeout 600 python tools/table4.py --nmin 21 --nmax 23 2>&1 | python -c "
import sys,json
for ln in sys.stdin:
    d=json.loads(ln)
    if 'n' in d: print(d['n'], d['seconds'], '%.3e'%d['terms_per_s'])"
done
