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


def row_rel(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Per-row relative error ||a_m - b_m|| / ||b_m||; a row whose reference is exactly 0 must be exactly 0
    (else inf)."""
    d = np.linalg.norm(a - b, axis=1)
    n = np.linalg.norm(b, axis=1)
    return np.where(n > 0, d / np.where(n > 0, n, 1.0), np.where(d > 0, np.inf, 0.0))


# bf16 unit roundoff (8 significant bits): every bf16 rounding is within a relative U_BF16 of its argument
U_BF16 = 2.0 ** -8
# per-row bar against Eq.1 with the EXACT gate: a row with a single active unit sees three bf16 roundings of its one
# term (the stored gate h_v, reading A10; h = h_v * u on the union path, R9; the bf16 output) -> 3u + 3u^2
ROW_TOL_EQ1 = 3 * U_BF16 + 3 * U_BF16 ** 2


def assert_y(y: np.ndarray, ref: np.ndarray, tol: float = 1e-2, rows=None, row_tol: float | None = None):
    """The Y bar: relative Frobenius error over the compared rows below `tol` (north_star: 1e-2 bf16 / 1e-5 fp32)
    AND the worst row's relative error below `row_tol` (default `tol`; the per-row bar catches a dropped term in a
    single row, which the global norm would dilute).  Against Eq.3 with the stored gate a row's terms see at most two
    bf16 roundings (h and the output: 2u + u^2 = 7.8e-3 < 1e-2); against Eq.1 (exact gate) pass
    row_tol=ROW_TOL_EQ1.  Logs the worst row and the per-row max-abs error."""
    row_tol = tol if row_tol is None else row_tol
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert y.shape == ref.shape, (y.shape, ref.shape)
    fro = rel_fro(y, ref)
    if y.ndim == 1 or y.shape[0] == 0:
        assert fro < tol, f"rel_fro {fro:.3e} >= {tol}"
        return fro
    rr = row_rel(y, ref)
    w = int(np.argmax(rr))
    mabs = float(np.abs(y - ref).max()) if y.size else 0.0
    name = f"row {rows[w]}" if rows is not None else f"row {w}"
    print(f"[Y] rows={y.shape[0]} rel_fro={fro:.3e} worst {name} rel={rr[w]:.3e} max_abs={mabs:.3e}")
    assert fro < tol, f"rel_fro {fro:.3e} >= {tol}"
    assert rr[w] < row_tol, f"{name}: row-relative error {rr[w]:.3e} >= {row_tol:.3e} (rel_fro {fro:.3e})"
    return fro


def twell_invariants(words: np.ndarray, N: int, T: int, C: int, chunk: int = 8192):
    """Structural checks on every (row, tile) of a packed TwELL: count <= T, stored indices inside the
    tile and strictly ascending, stored values > 0.  Row chunks bound the host memory."""
    M = words.shape[0]
    if M > chunk:
        for r0 in range(0, M, chunk):
            twell_invariants(words[r0:r0 + chunk], N, T, C, chunk)
        return
    W = T // C
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
