"""The N>1 path on CPU (gloo, world size 2, 127.0.0.1): the sharding host logic
of the product (shard_range / horizon_range, NCCL-id broadcast, admm_dist) and
the collective algebra of both partitions of SURVEY.md §8(e):
  * scenario shards -- the oracle on each rank's scenarios with its (6c) sum and
    residual maxima all-reduced over gloo equals the unsharded oracle;
  * horizon blocks -- the oracle on each rank's steps [k_begin, k_end) of every
    scenario, with the row sums over k of (6b)/(6d) and the initial 1'z
    all-reduced and the k = 1 consensus cell on rank 0 only, equals the
    unsharded oracle (the exchange the library's horizon mode performs).
No GPU."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q_total, n, iters, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_1903_10041_b200.dist import broadcast_bytes, shard_range

        # --- NCCL-id broadcast path of make_dist (fake id: no GPU here)
        payload = bytes(range(128)) if rank == 0 else None
        got = broadcast_bytes(payload, 0)
        assert got == bytes(range(128))
        # --- sharded oracle
        j0, j1 = shard_range(q_total, rank, world)
        P = synth.phev_problem(n, j1 - j0, j0=j0)

        def reduce(buf, op):
            t = torch.from_numpy(buf)
            dist.all_reduce(t, op=dist.ReduceOp.SUM if op == 0 else dist.ReduceOp.MAX)

        prm = oracle.default_params(r_bar=1e-6 * P["c"][1])
        o = oracle.Oracle(P, prm, q_total=q_total, reduce=reduce)
        info, hist = o.run(iters)
        out_q.put((rank, j0, j1, o.state(), info, hist))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("q_total", [6, 7])
def test_sharded_oracle_equals_unsharded(q_total):
    import oracle
    import synth

    n, iters, world = 300, 120, 2
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q_total, n, iters, out_q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [out_q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    P = synth.phev_problem(n, q_total)
    o = oracle.Oracle(P, oracle.default_params(r_bar=1e-6 * P["c"][1]))
    info, hist = o.run(iters)
    S = o.state()
    sx = 1e5
    for rank, j0, j1, Sr, ir, hr in res:
        # identical rho schedule and decisions on every rank
        assert np.array_equal(hr[:, 3:7], hist[:, 3:7])
        assert np.array_equal(hr[:, 14:16], hist[:, 14:16])
        # the shard's iterates equal the unsharded ones up to the summation order over j
        assert np.abs(Sr["x"] - S["x"][:, j0:j1]).max() / sx <= 1e-11
        assert np.abs(Sr["x1"] - S["x1"]).max() / sx <= 1e-11
        assert np.abs(Sr["nu"] - S["nu"][:, j0:j1]).max() / sx <= 1e-11
        assert abs(ir["objective"] - info["objective"]) <= 1e-11 * abs(info["objective"])


def _hz_worker(rank, world, port, n, q, iters, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_1903_10041_b200.dist import horizon_range

        k0, k1 = horizon_range(n, rank, world)
        P = synth.horizon_problem(n) if q == 1 else synth.phev_problem(n, q)
        Pl = dict(P)
        for k in ("a2", "a1", "a0", "b2", "b1", "b0"):
            Pl[k] = np.ascontiguousarray(P[k][:, :, k0:k1])
        for k in ("lo", "hi", "y"):
            Pl[k] = np.ascontiguousarray(P[k][:, k0:k1])
        Pl["n"] = k1 - k0

        def reduce(buf, op):
            t = torch.from_numpy(buf)
            dist.all_reduce(t, op=dist.ReduceOp.SUM if op == 0 else dist.ReduceOp.MAX)

        cf = np.where(np.isfinite(P["c"]), P["c"], 0).max()
        prm = oracle.default_params(r_bar=1e-6 * cf)
        o = oracle.Oracle(Pl, prm, reduce=reduce, horizon=(n, k0))
        info, hist = o.run(iters)
        out_q.put((rank, k0, k1, o.state(), info, hist))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,q", [(3001, 1), (700, 3)])
def test_horizon_blocks_oracle_equals_unsharded(n, q):
    import oracle
    import synth

    iters, world = 120, 2
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_hz_worker, args=(r, world, port, n, q, iters, out_q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [out_q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    P = synth.horizon_problem(n) if q == 1 else synth.phev_problem(n, q)
    cf = np.where(np.isfinite(P["c"]), P["c"], 0).max()
    o = oracle.Oracle(P, oracle.default_params(r_bar=1e-6 * cf))
    info, hist = o.run(iters)
    S = o.state()
    sx = max(np.abs(P["lo"]).max(), np.abs(P["hi"]).max())
    g = (P["b2"] * S["x"] + P["b1"]) * S["x"] + P["b0"]
    sh = max(np.abs(P["c"][np.isfinite(P["c"])]).max(), n * np.abs(g).max())
    for rank, k0, k1, Sr, ir, hr in res:
        assert np.array_equal(hr[:, 3:7], hist[:, 3:7])  # identical rho schedule
        assert np.array_equal(hr[:, 14:16], hist[:, 14:16])
        assert np.abs(Sr["x"] - S["x"][:, :, k0:k1]).max() / sx <= 1e-11
        assert np.abs(Sr["x1"] - S["x1"]).max() / sx <= 1e-11
        assert np.abs(Sr["h"] - S["h"]).max() / sh <= 1e-11
        assert np.abs(Sr["p"] - S["p"]).max() / sh <= 1e-11
        assert np.abs(Sr["s"] - S["s"][:, k0:k1]).max() / np.abs(P["y"]).max() <= 1e-11
        if k0 == 0:
            assert np.abs(Sr["nu"] - S["nu"]).max() / sx <= 1e-11
        assert abs(ir["objective"] - info["objective"]) <= 1e-11 * abs(info["objective"])
        # residual columns agree up to the summation order of the row sums
        assert np.allclose(hr[:, 7:14], hist[:, 7:14], rtol=1e-9, atol=1e-9 * sh)


def test_make_dist_fields():
    """admm_dist as the product builds it for each rank (single process: world 1)."""
    from paper_1903_10041_b200 import _lib
    from paper_1903_10041_b200.dist import shard_range

    d = _lib.admm_dist()
    j0, j1 = shard_range(100001, 3, 8)
    d.rank, d.world, d.j_begin, d.j_end = 3, 8, j0, j1
    assert (d.j_end - d.j_begin) in (12500, 12501)
    assert _lib.admm_dist.nccl_id.size == 128
    from paper_1903_10041_b200.dist import dist_for

    uid = bytes(range(128))
    h = dist_for(1, 4, 3, uid, horizon=1000003)
    assert h.mode == _lib.ADMM_SHARD_HORIZON and (h.j_begin, h.j_end) == (0, 3)
    assert (h.k_begin, h.k_end) == (250001, 500002)
    s = dist_for(2, 4, 10, uid)
    assert s.mode == _lib.ADMM_SHARD_SCENARIOS and (s.j_begin, s.j_end) == (6, 8)
    assert bytes(s.nccl_id) == uid
