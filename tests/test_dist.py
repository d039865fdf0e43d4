"""Multi-process (gloo, world size 2, CPU) tests of the hidden-dim sharding host logic:
shard partition + one all-reduce of partial outputs reproduces the unsharded oracle (north_star (5)),
and the NCCL-unique-id broadcast path used by sffn.Comm."""
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


def _worker(rank, world, port, q, mode="contiguous"):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_2603_23198_b200.sharding import broadcast_id, shard_perm, shard_range
        cfg = synth.CONFIGS["tiny"]
        n0, Nl = shard_range(cfg.N, world, rank, cfg.T)
        units = shard_perm(cfg.N, world, cfg.T, mode)[n0:n0 + Nl]  # this rank's hidden units (weight rows)
        X = synth.gen_x(cfg)
        Wg, Wu, Wd = (synth.gen_w(cfg, w)[units] for w in "gud")
        # each rank: pack its shard (local indices) and compute its partial Eq.3 sum
        words, counts, ov, A = oracle.pack_from_inputs(X, Wg, cfg.T, cfg.C)
        Yr = oracle.ffn_twell(X, words, Wu, Wd, Nl, cfg.T, cfg.C, A=A)
        t = torch.from_numpy(Yr)
        dist.all_reduce(t)  # the one collective of the sharded forward
        idb = broadcast_id(bytes(range(128)) if rank == 0 else None, rank, world)
        q.put((rank, t.numpy(), int(counts.sum()), idb, (n0, Nl), units))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("mode", ["contiguous", "round_robin"])
def test_hidden_sharding_gloo_world2(mode):
    """World-2 gloo run of the sharded computation: each rank packs its shard (contiguous rows, or TwELL tiles dealt
    round-robin) with local indices, computes its partial Eq.3 sum, one all-reduce; the sum equals the
    unsharded Eq.1 oracle and the ranks' units are an exact permutation of all hidden units."""
    import oracle
    import synth
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q, mode)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    cfg = synth.CONFIGS["tiny"]
    X = synth.gen_x(cfg)
    Wg, Wu, Wd = (synth.gen_w(cfg, w) for w in "gud")
    Y = oracle.ffn_dense(X, Wg, Wu, Wd)
    _, _, _, A = oracle.pack_from_inputs(X, Wg, cfg.T, cfg.C)
    for rank, Ysum, nnz, idb, (n0, Nl), units in res:
        assert np.max(np.abs(Ysum - Y)) <= 1e-12 * np.max(np.abs(Y))
        assert idb == bytes(range(128))
        assert n0 == rank * cfg.N // world and Nl == cfg.N // world
        tiles = np.unique(units // cfg.T)
        assert len(units) == len(tiles) * cfg.T  # whole TwELL tiles per rank
        if mode == "round_robin":
            assert (tiles % world == rank).all()
    assert np.array_equal(np.sort(np.concatenate([r[5] for r in res])), np.arange(cfg.N))  # exact permutation
    # shards partition the non-zeros of the unsharded gate
    assert sum(r[2] for r in res) == int((A > 0).sum())


def test_shard_range_errors():
    from paper_2603_23198_b200.sharding import shard_range
    assert shard_range(14336, 8, 7, 256) == (7 * 1792, 1792)
    with pytest.raises(ValueError):
        shard_range(14336, 3, 0, 256)
    with pytest.raises(ValueError):
        shard_range(1024, 2, 2, 256)
