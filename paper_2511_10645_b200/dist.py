"""Host-side plumbing of the output-channel-sharded linear.

torch.distributed is used only as the process-group plumbing (the NCCL unique-id
broadcast, barriers, max-over-ranks timing); the data path is paro_linear_allgather
(GEMV kernel + ncclAllGather on the caller's stream) inside libparo.so.
"""
from __future__ import annotations


def shard_rows(N: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [r0, r1) of the output channels owned by `rank` (contiguous, equal shards)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if N % world:
        raise ValueError(f"N={N} not divisible by world={world}")
    n = N // world
    return rank * n, (rank + 1) * n


def broadcast_bytes(payload: bytes | None, src: int = 0, group=None) -> bytes:
    """Broadcast a small byte string (the NCCL unique id) from `src` over a torch
    process group (gloo or nccl)."""
    import torch.distributed as dist
    obj = [payload]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


def make_comm(rank: int, world: int, group=None) -> int:
    """Create this rank's NCCL communicator for paro_linear_allgather."""
    import paper_2511_10645_b200 as paro
    uid = paro.paro_comm_unique_id() if rank == 0 else None
    uid = broadcast_bytes(uid, 0, group)
    return paro.paro_comm_init(uid, rank, world)


def rank_major_to_rows(gathered):
    """[world, B, Ns] (what an all-gather of per-rank [B, Ns] outputs produces) ->
    [B, world * Ns]; the same permutation paro_linear_allgather applies on the GPU for
    B > 1 (for B = 1 the rank-major buffer already is [N])."""
    world, B, Ns = gathered.shape
    return gathered.permute(1, 0, 2).reshape(B, world * Ns)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (bench timing rule: time = max over ranks)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def make_p2p(rank: int, world: int, N_full: int, out_dtype=None, device=None, group=None):
    """Exchange buffers for paro_linear_allgather_p2p: every rank allocates one (zeroed), shares
    its CUDA IPC handle over the process group and opens the peers'.  Returns (local_buf,
    peer_ptrs, opened) -- close `opened` with paro_ipc_close_handle when done."""
    import torch.distributed as dist

    import paper_2511_10645_b200 as paro
    buf = paro.p2p_buffer(N_full, world, out_dtype, device=device)
    handles = [None] * world
    dist.all_gather_object(handles, paro.paro_ipc_get_handle(buf), group=group)
    ptrs, opened = [], []
    for q in range(world):
        if q == rank:
            ptrs.append(buf.data_ptr())
        else:
            p = paro.paro_ipc_open_handle(handles[q])
            ptrs.append(p)
            opened.append(p)
    return buf, ptrs, opened
