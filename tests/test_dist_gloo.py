"""World-size-2 gloo tests (CPU) of the output-channel-sharded path's host logic:
shard ranges, per-rank packs == rows of the full pack (bitwise), rank-major all-gather
layout -> [B, N], uid broadcast and max-over-ranks timing.  The per-shard compute uses
the oracle (this is a CPU test of the orchestration; the GPU data path is covered by
tests/test_gpu_parity.py and bench.py under torchrun)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B, N, K, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        import synth
        from paper_2511_10645_b200 import dist as pd
        p = synth.make_problem(N, K, B, seed=7)
        r0, r1 = pd.shard_rows(N, world, rank)
        shard = O.oracle_pack(p["W"][r0:r1], p["s"], p["theta"], p["pairs"])
        full = O.oracle_pack(p["W"], p["s"], p["theta"], p["pairs"])
        same_pack = (np.array_equal(shard["codes"], full["codes"][r0:r1])
                     and np.array_equal(shard["scales"].view(np.uint16), full["scales"][r0:r1].view(np.uint16))
                     and np.array_equal(shard["zeros"], full["zeros"][r0:r1]))
        y_local = torch.from_numpy(O.oracle_linear(p["x"], shard, p["s"], p["theta"], p["pairs"]))
        gathered = [torch.empty_like(y_local) for _ in range(world)]
        dist.all_gather(gathered, y_local)
        y = pd.rank_major_to_rows(torch.stack(gathered)).numpy()
        y_full = O.oracle_linear(p["x"], full, p["s"], p["theta"], p["pairs"])
        uid = pd.broadcast_bytes(b"uid-%d" % 42 if rank == 0 else None)
        tmax = pd.max_over_ranks(1.0 + rank)
        q.put((rank, same_pack, float(np.max(np.abs(y - y_full)) / np.max(np.abs(y_full))), uid, tmax))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B", [1, 3])
def test_sharded_linear_world2_gloo(B):
    world, N, K = 2, 256, 256
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, N, K, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, same_pack, err, uid, tmax in res:
        assert same_pack, f"rank {rank}: shard pack != rows of the full pack"
        assert err <= 1e-12, f"rank {rank}: gathered y differs from the full product ({err})"
        assert uid == b"uid-42"
        assert tmax == 2.0


def test_shard_rows_partition():
    from paper_2511_10645_b200 import dist as pd
    for N, world in [(28672, 8), (8192, 4), (1024, 2), (4096, 1)]:
        cover = []
        for r in range(world):
            a, b = pd.shard_rows(N, world, r)
            cover += list(range(a, b))
        assert cover == list(range(N))
    with pytest.raises(ValueError):
        pd.shard_rows(1000, 3, 0)
