"""Helpers shared by the GPU tests: numpy bf16 bits <-> torch CUDA tensors, comparisons."""
import numpy as np
import torch


def to_dev(a: np.ndarray) -> torch.Tensor:
    """numpy uint16 bf16 bits -> torch.bfloat16 CUDA tensor (bit-exact)."""
    assert a.dtype == np.uint16
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).cuda()


def words_np(tw: torch.Tensor) -> np.ndarray:
    return tw.cpu().numpy().view(np.uint32)


def bf16_np(t: torch.Tensor) -> np.ndarray:
    """torch bf16 -> numpy float64 (exact)."""
    return t.float().cpu().numpy().astype(np.float64)


def rel_fro(a: np.ndarray, b: np.ndarray) -> float:
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a))


def twell_invariants(words: np.ndarray, N: int, T: int, C: int):
    """Structural checks on every (row, tile) of a packed TwELL: count <= T, stored indices inside the
    tile and strictly ascending, stored values > 0."""
    W = T // C
    M = words.shape[0]
    blk = words.reshape(M, N // T, W)
    cnt = blk[:, :, 0].astype(np.int64)
    assert (cnt <= T).all()
    z = np.minimum(cnt, W - 1)
    slots = blk[:, :, 1:]
    idx = (slots & 0xFFFF).astype(np.int64)
    val = (slots >> 16).astype(np.uint16)
    valid = np.arange(1, W)[None, None, :] <= z[:, :, None]
    t0 = (np.arange(N // T) * T)[None, :, None]
    assert ((idx >= t0) & (idx < t0 + T) | ~valid).all(), "index outside its tile"
    asc = np.diff(idx, axis=2) > 0
    assert (asc | ~valid[:, :, 1:]).all(), "indices not strictly ascending"
    pos = (val & 0x8000) == 0
    nonzero = (val & 0x7FFF) != 0
    assert ((pos & nonzero) | ~valid).all(), "stored value not > 0"
