mkdir -p gpurun_out
# the N-rank bench path under torchrun with NCCL (one rank: gpurun has one GPU)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r4j_torchrun1.log 2>&1; echo torchrun1=$? 
tail -1 gpurun_out/r4j_torchrun1.log | cut -c1-300
TRITPERM_BENCH_DIST=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r4j_dist1.log 2>&1; echo dist1=$?
tail -1 gpurun_out/r4j_dist1.log | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print(d['n_gpus'], d['ms_per_step'], d['c5_strong'])"
timeout 600 python bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/r4j_ref2.log 2>&1; echo ref2=$?; tail -2 gpurun_out/r4j_ref2.log | cut -c1-200
