mkdir -p gpurun_out
tools/ab_run.sh r5g "c3" main nb17 > gpurun_out/r5g_ab.txt 2>&1
cat gpurun_out/r5g_ab.txt
TRITPERM_LIB=$PWD/paper_2407_20205_b200/lib/ab/lib_nb17.so timeout 300 python tools/c3_families.py 2>&1 | cut -c1-100
