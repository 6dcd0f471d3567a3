"""Host-side logic of scenario sharding: which scenarios a
rank owns and how the NCCL unique id reaches every rank.  torch.distributed is
plumbing only (rank bootstrap); the per-iteration exchange is an NCCL
all-gather inside the library's CUDA graph."""

from __future__ import annotations


def shard_range(q_total: int, rank: int, world: int):
    """Balanced contiguous split of scenarios 0..q_total-1: the first
    q_total % world ranks get one extra scenario."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if q_total < world:
        raise ValueError(f"q_total={q_total} < world={world}: every rank needs a scenario")
    base, rem = divmod(q_total, world)
    j0 = rank * base + min(rank, rem)
    return j0, j0 + base + (1 if rank < rem else 0)


def broadcast_bytes(payload: bytes | None, src: int = 0, group=None) -> bytes:
    """Broadcast a small byte string from `src` over the default torch process
    group (gloo or nccl)."""
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"
    n = torch.zeros(1, dtype=torch.int64, device=dev)
    if dist.get_rank(group) == src:
        n[0] = len(payload)
    dist.broadcast(n, src, group=group)
    buf = torch.zeros(int(n.item()), dtype=torch.uint8, device=dev)
    if dist.get_rank(group) == src:
        buf.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(buf, src, group=group)
    return bytes(buf.cpu().numpy().tobytes())


def horizon_range(n: int, rank: int, world: int):
    """Balanced contiguous split of the steps 0..n-1 into horizon blocks (rank 0
    holds k = 0, the consensus cell)."""
    return shard_range(n, rank, world)


def make_dist(q_total: int, group=None, unique_id_fn=None, horizon: int = None):
    """admm_dist for this rank + NCCL id from rank 0 (unique_id_fn defaults to the
    library's admm_nccl_unique_id).  horizon=None: scenario sharding (rank r owns
    a balanced range of the q_total scenarios); horizon=n: horizon blocks (rank r
    owns a balanced range of the n steps of every scenario)."""
    import torch.distributed as dist

    from . import _lib

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if unique_id_fn is None:
        unique_id_fn = _lib.admm_nccl_unique_id
    uid = unique_id_fn() if rank == 0 else None
    uid = broadcast_bytes(uid, 0, group)
    return dist_for(rank, world, q_total, uid, horizon)


def dist_for(rank: int, world: int, q_total: int, nccl_id: bytes, horizon: int = None):
    """admm_dist of one rank (no process group needed: world = 1 runs the collective
    path on one GPU)."""
    from . import _lib

    d = _lib.admm_dist()
    d.rank, d.world = rank, world
    if horizon is None:
        d.j_begin, d.j_end = shard_range(q_total, rank, world)
        d.mode = _lib.ADMM_SHARD_SCENARIOS
    else:
        d.j_begin, d.j_end = 0, q_total
        d.k_begin, d.k_end = horizon_range(horizon, rank, world)
        d.mode = _lib.ADMM_SHARD_HORIZON
    for t in range(128):
        d.nccl_id[t] = nccl_id[t]
    return d
