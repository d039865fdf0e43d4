"""Host-side logic of hidden-dim sharding (north_star (5)): which hidden units a rank owns, and the
broadcast of the NCCL unique id.  No compute here."""
from __future__ import annotations


def shard_range(N: int, world: int, rank: int, T: int) -> tuple[int, int]:
    """Contiguous block of hidden units [n0, n0 + Nl) owned by `rank`; every shard a multiple of the
    TwELL tile T so each rank packs whole tiles with local indices."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if N % (world * T):
        raise ValueError(f"N={N} must be a multiple of world*T={world * T}")
    Nl = N // world
    return rank * Nl, Nl


def shard_perm(N: int, world: int, T: int, mode: str = "contiguous"):
    """Hidden-unit order of the G shards: rank r owns units perm[r N/G : (r+1) N/G] (its weight rows, in this order;
    its TwELL indices are local positions in that slice).  "contiguous": the identity.  "round_robin": TwELL tiles of
    T units dealt to ranks in turn (tile t -> rank t mod G, SURVEY §8e load balance: hot and dead neurons cluster
    in contiguous blocks less), each rank keeping its tiles in ascending order.  Any such order is a consistent
    permutation of hidden units, so sum_r Y_r is unchanged (Eq.1 is a sum over n).  Applied once, at load time."""
    import numpy as np
    shard_range(N, world, 0, T)  # validates N % (world * T)
    if mode == "contiguous":
        return np.arange(N, dtype=np.int64)
    if mode != "round_robin":
        raise ValueError(f"unknown shard mode {mode!r}")
    tiles = np.arange(N // T).reshape(-1, world).T  # [world, tiles per rank]: rank r gets tiles r, r+G, ...
    return (tiles[:, :, None] * T + np.arange(T)[None, None, :]).reshape(-1).astype(np.int64)


def broadcast_id(id_bytes: bytes | None, rank: int, world: int, group=None) -> bytes:
    """Rank 0's 128-byte id to every rank through torch.distributed (any backend)."""
    if world == 1:
        assert id_bytes is not None
        return id_bytes
    import torch.distributed as dist
    obj = [list(id_bytes) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    out = bytes(obj[0])
    if len(out) != 128:
        raise ValueError("unique id must be 128 bytes")
    return out
