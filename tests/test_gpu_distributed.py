"""The multi-process path with the real device compute: two ranks on the one
GPU a gpurun box has, each running its split_steps part through the CUDA
library (parallel.distributed_counts' default counts), the 16-byte counters
meeting in one all_reduce(SUM) over gloo (NCCL refuses two ranks on one
device).  The ranks' kernels are independent -- nothing on the device waits
on the other rank -- so this is the north_star's partition + single
reduction (src/permanent.py:232-255) executed end to end, not a stand-in
for GPUs that are not there.  tests/test_parallel_gloo.py covers the same
partition on CPU with the oracle as the per-rank compute."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from conftest import REPO, centred, dec, load_golden

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, REPO)
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["TRITPERM_DEVICE"] = "0"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2407_20205_b200 import _kernels, parallel
        from paper_2407_20205_b200.permanent import MatrixF3

        torch.cuda.set_device(0)
        g = load_golden("anchors.json")
        out = {}
        # C4: the seed-0 36x36 matrix's full 2^36 traversal, half per rank
        # (each half is large enough for the bucketed walk)
        w = g["c4_full"]
        m = MatrixF3(centred(dec(w["a"], 36)))
        _kernels.walk_tested(0)
        out["c4"] = parallel.distributed_counts(m, 1, 1 << 36, device="cpu")
        out["c4_class"] = parallel.perm_mod3_distributed(m, device="cpu")
        out["c4_tested"] = _kernels.walk_tested(0)
        out["c4_range"] = parallel.rank_range(36, rank, world, 1, 1 << 36)
        # C5's 2^36-step window of the 50x50 matrix
        w5 = g["c5_window36"]
        m5 = MatrixF3(centred(dec(w5["a"], 50)))
        out["c5w"] = parallel.distributed_counts(m5, w5["lo"], w5["hi"], device="cpu")
        # a 20x20 anchor on an unaligned sub-range (generic walk heads/tails)
        c1 = g["c1"][0]
        m1 = MatrixF3(centred(dec(c1["a"], 20)))
        out["c1_sub"] = parallel.distributed_counts(m1, 12345, 678901, device="cpu")
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results(gpu):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def test_two_ranks_c4_full_traversal(results):
    w = load_golden("anchors.json")["c4_full"]
    for r in (0, 1):
        p, q = results[r]["c4"]
        assert p - q == w["partial"]
        assert results[r]["c4_class"] % 3 == w["class"]
        assert results[r]["c4_tested"] > 0  # each rank's half went through the bucketed walk
    (a0, a1), (b0, b1) = results[0]["c4_range"], results[1]["c4_range"]
    assert a0 == 1 and a1 == b0 and b1 == 1 << 36


def test_two_ranks_c5_window_and_unaligned_range(results, oracle):
    g = load_golden("anchors.json")
    w5 = g["c5_window36"]
    c1 = g["c1"][0]
    a = dec(c1["a"], 20)
    mags, sgns = oracle.planes_from_classes(a)
    for r in (0, 1):
        p, q = results[r]["c5w"]
        assert p - q == w5["partial"]
        p, q = results[r]["c1_sub"]
        assert p - q == oracle.chunk_sum(mags, sgns, 20, 12345, 678901)
