mkdir -p gpurun_out
tools/ab_run.sh r4z "c3" main seg66 seg48 > gpurun_out/r4z_ab.txt 2>&1
cat gpurun_out/r4z_ab.txt
for v in seg66 seg48; do TRITPERM_LIB=$PWD/paper_2407_20205_b200/lib/ab/lib_$v.so timeout 300 python tools/c3_families.py 2>&1 | cut -c1-100; done
