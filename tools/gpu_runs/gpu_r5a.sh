mkdir -p gpurun_out
tools/ab_run.sh r5a "c3" seg48 seg36 seg30 seg24 > gpurun_out/r5a_ab.txt 2>&1
cat gpurun_out/r5a_ab.txt
for v in seg36 seg24; do TRITPERM_LIB=$PWD/paper_2407_20205_b200/lib/ab/lib_$v.so timeout 300 python tools/c3_families.py 2>&1 | cut -c1-100; done
