"""CPU oracle for the sparse gated-FFN forward — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2603_23198_b200``) never imports it and shares no code with it.

Thin numpy/ctypes wrapper over ``oracle.c`` (plain fp64 C loops, each function citing
the PAPER.md passage it follows).  See oracle.c's header for the pins.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(src):
        # -O2 without -ffast-math: fp64 sums keep the literal k-ascending order.
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fno-fast-math", "-ffp-contract=off", "-shared",
                               "-fPIC", "-o", _LIB, src, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        vp, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        lib.oracle_bf16_to_double.argtypes = [ctypes.c_uint16]
        lib.oracle_bf16_to_double.restype = ctypes.c_double
        lib.oracle_f32_to_bf16_rne.argtypes = [ctypes.c_float]
        lib.oracle_f32_to_bf16_rne.restype = ctypes.c_uint16
        lib.oracle_gate_preact.argtypes = [vp, vp, i64, i64, i64, vp]
        lib.oracle_gate_preact_f32.argtypes = [vp, vp, i64, i64, i64, vp]
        lib.oracle_pack.argtypes = [vp, i64, i64, ci, ci, vp, vp]
        lib.oracle_pack.restype = i64
        lib.oracle_unpack.argtypes = [vp, i64, i64, ci, ci, vp]
        lib.oracle_ffn_dense.argtypes = [vp, vp, vp, vp, i64, i64, i64, vp, vp]
        lib.oracle_ffn_twell.argtypes = [vp, vp, vp, vp, i64, i64, i64, ci, ci, ci, vp, vp]
        lib.oracle_ffn_nongated_dense.argtypes = [vp, vp, vp, i64, i64, i64, vp]
        lib.oracle_down_twell.argtypes = [vp, vp, i64, i64, i64, ci, ci, ci, vp, vp]
        lib.oracle_pack_soa.argtypes = [vp, i64, i64, ci, ci, vp, vp, vp]
        lib.oracle_twell_to_ell.argtypes = [vp, i64, i64, ci, ci, i64, vp, vp, vp, vp]
        lib.oracle_hybrid_sddmm.argtypes = [vp, vp, i64, i64, i64, i64, vp, vp, vp, vp, i64, vp, vp, ci, vp, vp]
        lib.oracle_hybrid_spmm.argtypes = [vp, vp, vp, vp, i64, i64, i64, vp, vp, vp, i64, i64, vp]
        lib.oracle_pack_soa.restype = i64
        lib.oracle_ffn_dense_f32.argtypes = [vp, vp, vp, vp, i64, i64, i64, vp]
        lib.oracle_ffn_soa_f32.argtypes = [vp, vp, vp, vp, vp, vp, i64, i64, i64, ci, ci, vp]
        _lib = lib
    return _lib


def _u16(a):
    a = np.ascontiguousarray(a)
    assert a.dtype == np.uint16, a.dtype
    return a


def bf16_rne(f: np.ndarray) -> np.ndarray:
    lib = _load()
    f = np.asarray(f, dtype=np.float32).ravel()
    return np.array([lib.oracle_f32_to_bf16_rne(float(v)) for v in f], dtype=np.uint16)


def gate_preact(X, Wg) -> np.ndarray:
    """A = X W_g^T in fp64 (Eq.1), X [M,K] and W_g [N,K] as bf16 bits."""
    X, Wg = _u16(X), _u16(Wg)
    M, K = X.shape
    N = Wg.shape[0]
    A = np.empty((M, N), dtype=np.float64)
    _load().oracle_gate_preact(X.ctypes.data, Wg.ctypes.data, M, K, N, A.ctypes.data)
    return A


def gate_preact_matmul(X, Wg, rows_per_call: int = 4096) -> np.ndarray:
    """The same A = X W_g^T with the product taken by ONE library primitive (numpy's fp64 matmul) instead of the
    k-ascending C loop — the allowed "library primitive as a step" for row samples too large for the loop (the
    loop streams all of W_g once per row).  On dyadic-grid inputs every product and partial sum is exactly
    representable (< 2^20 units of 2^-11), so the result equals gate_preact bit for bit whatever
    the BLAS summation order; tests/test_oracle_pins.py pins that equality.  Off the grid it differs from
    gate_preact by fp64 rounding only."""
    X, Wg = _u16(X), _u16(Wg)
    Wt = ((Wg.astype(np.uint32) << 16).view(np.float32).astype(np.float64)).T
    M = X.shape[0]
    A = np.empty((M, Wg.shape[0]), dtype=np.float64)
    for r0 in range(0, M, rows_per_call):
        x = (X[r0:r0 + rows_per_call].astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        np.matmul(x, Wt, out=A[r0:r0 + rows_per_call])
    return A


def pack(S, T: int, C: int):
    """Alg.1 lines 7-17 packed as P:869 on fp32 S [M,N] -> (words uint32 [M,N/C], counts [M,N/T], n_overflow).
    Slots beyond each block's count are zero-initialised here (unspecified in the format)."""
    S = np.ascontiguousarray(S, dtype=np.float32)
    M, N = S.shape
    assert N % T == 0 and T % C == 0 and T // C >= 2
    words = np.zeros((M, N // C), dtype=np.uint32)
    counts = np.zeros((M, N // T), dtype=np.uint32)
    ov = _load().oracle_pack(S.ctypes.data, M, N, T, C, words.ctypes.data, counts.ctypes.data)
    return words, counts, int(ov)


def unpack(words, N: int, T: int, C: int) -> np.ndarray:
    words = np.ascontiguousarray(words, dtype=np.uint32)
    M = words.shape[0]
    H = np.empty((M, N), dtype=np.float32)
    _load().oracle_unpack(words.ctypes.data, M, N, T, C, H.ctypes.data)
    return H


def ffn_dense(X, Wg, Wu, Wd, want_h: bool = False):
    """Eq.1 with ReLU gate, fp64.  Returns Y [M,K] (and h [M,N])."""
    X, Wg, Wu, Wd = map(_u16, (X, Wg, Wu, Wd))
    M, K = X.shape
    N = Wg.shape[0]
    Y = np.empty((M, K), dtype=np.float64)
    H = np.empty((M, N), dtype=np.float64) if want_h else None
    _load().oracle_ffn_dense(X.ctypes.data, Wg.ctypes.data, Wu.ctypes.data, Wd.ctypes.data, M, K, N,
                             Y.ctypes.data, H.ctypes.data if want_h else None)
    return (Y, H) if want_h else Y


def ffn_twell(X, words, Wu, Wd, N: int, T: int, C: int, A=None) -> np.ndarray:
    """Eq.3 over a packed TwELL; gate = stored bf16 value, or exact A if given."""
    X, Wu, Wd = map(_u16, (X, Wu, Wd))
    words = np.ascontiguousarray(words, dtype=np.uint32)
    M, K = X.shape
    Y = np.empty((M, K), dtype=np.float64)
    mode = 0
    Ap = None
    if A is not None:
        A = np.ascontiguousarray(A, dtype=np.float64)
        mode, Ap = 1, A.ctypes.data
    _load().oracle_ffn_twell(X.ctypes.data, words.ctypes.data, Wu.ctypes.data, Wd.ctypes.data, M, K, N, T, C,
                             mode, Ap, Y.ctypes.data)
    return Y


def pack_from_inputs(X, Wg, T: int, C: int, matmul: bool = False):
    """The oracle's TwELL for relu(X W_g^T): fp64 pre-activation -> fp32 (exact on grid inputs) -> Alg.1.
    matmul=True takes the pre-activation from gate_preact_matmul (bit-identical on grid inputs)."""
    A = gate_preact_matmul(X, Wg) if matmul else gate_preact(X, Wg)
    words, counts, ov = pack(A.astype(np.float32), T, C)
    return words, counts, ov, A


def valid_prefix_equal(w_a: np.ndarray, w_b: np.ndarray, T: int, C: int) -> np.ndarray:
    """Per (row, tile) block: counts equal and the stored prefix min(count, cap) equal.
    Returns a bool array [M, N/T]."""
    W = T // C
    M = w_a.shape[0]
    a = w_a.reshape(M, -1, W)
    b = w_b.reshape(M, -1, W)
    cnt_eq = a[:, :, 0] == b[:, :, 0]
    cap = W - 1
    z = np.minimum(a[:, :, 0], cap)
    slot = np.arange(1, W)[None, None, :]
    valid = slot <= z[:, :, None]
    slots_eq = np.all((a[:, :, 1:] == b[:, :, 1:]) | ~valid, axis=2)
    return cnt_eq & slots_eq


# ---------------------------------------------------------------- fp32 mode (reading R19)
def _f32(a):
    a = np.ascontiguousarray(a)
    assert a.dtype == np.float32, a.dtype
    return a


def gate_preact_f32(X, Wg) -> np.ndarray:
    X, Wg = _f32(X), _f32(Wg)
    M, K = X.shape
    N = Wg.shape[0]
    A = np.empty((M, N), dtype=np.float64)
    _load().oracle_gate_preact_f32(X.ctypes.data, Wg.ctypes.data, M, K, N, A.ctypes.data)
    return A


def pack_soa(S, T: int, C: int):
    """Alg.1 SoA outputs (h_v, h_I, h_nz) with capacity T/C; slots past the count are zero here."""
    S = np.ascontiguousarray(S, dtype=np.float32)
    M, N = S.shape
    hv = np.zeros((M, N // C), dtype=np.float32)
    hi = np.zeros((M, N // C), dtype=np.uint16)
    hnz = np.zeros((M, N // T), dtype=np.uint32)
    ov = _load().oracle_pack_soa(S.ctypes.data, M, N, T, C, hv.ctypes.data, hi.ctypes.data, hnz.ctypes.data)
    return hv, hi, hnz, int(ov)


def ffn_dense_f32(X, Wg, Wu, Wd) -> np.ndarray:
    X, Wg, Wu, Wd = map(_f32, (X, Wg, Wu, Wd))
    M, K = X.shape
    N = Wg.shape[0]
    Y = np.empty((M, K), dtype=np.float64)
    _load().oracle_ffn_dense_f32(X.ctypes.data, Wg.ctypes.data, Wu.ctypes.data, Wd.ctypes.data, M, K, N, Y.ctypes.data)
    return Y


def ffn_soa_f32(X, hv, hi, hnz, Wu, Wd, N: int, T: int, C: int) -> np.ndarray:
    X, Wu, Wd = map(_f32, (X, Wu, Wd))
    hv = np.ascontiguousarray(hv, dtype=np.float32)
    hi = np.ascontiguousarray(hi, dtype=np.uint16)
    hnz = np.ascontiguousarray(hnz, dtype=np.uint32)
    M, K = X.shape
    Y = np.empty((M, K), dtype=np.float64)
    _load().oracle_ffn_soa_f32(X.ctypes.data, hv.ctypes.data, hi.ctypes.data, hnz.ctypes.data, Wu.ctypes.data,
                               Wd.ctypes.data, M, K, N, T, C, Y.ctypes.data)
    return Y


def soa_prefix_equal(a, b, T: int, C: int) -> np.ndarray:
    """(hv, hi, hnz) triples: counts equal and the stored prefix (capacity T/C) equal, per (row, tile)."""
    hva, hia, nza = a
    hvb, hib, nzb = b
    M = nza.shape[0]
    W = T // C
    cnt_eq = nza == nzb
    z = np.minimum(nza, W)
    valid = np.arange(W)[None, None, :] < z[:, :, None]
    va, vb = hva.reshape(M, -1, W), hvb.reshape(M, -1, W)
    ia, ib = hia.reshape(M, -1, W), hib.reshape(M, -1, W)
    eq = ((va.view(np.uint32) == vb.view(np.uint32)) & (ia == ib)) | ~valid
    return cnt_eq & np.all(eq, axis=2)


# ---------------------------------------------------------------- non-gated variant (App.C, NEXT-2)
def ffn_nongated_dense(X, Wu, Wd) -> np.ndarray:
    """y = relu(x W_u) W_d, fp64."""
    X, Wu, Wd = map(_u16, (X, Wu, Wd))
    M, K = X.shape
    N = Wu.shape[0]
    Y = np.empty((M, K), dtype=np.float64)
    _load().oracle_ffn_nongated_dense(X.ctypes.data, Wu.ctypes.data, Wd.ctypes.data, M, K, N, Y.ctypes.data)
    return Y


def down_twell(words, Wd, K: int, N: int, T: int, C: int, A=None) -> np.ndarray:
    """sum over stored entries of h_v * W_d[n, :] (Listing 3 semantics); exact A instead of h_v if given."""
    Wd = _u16(Wd)
    words = np.ascontiguousarray(words, dtype=np.uint32)
    M = words.shape[0]
    Y = np.empty((M, K), dtype=np.float64)
    mode, Ap = 0, None
    if A is not None:
        A = np.ascontiguousarray(A, dtype=np.float64)
        mode, Ap = 1, A.ctypes.data
    _load().oracle_down_twell(words.ctypes.data, Wd.ctypes.data, M, K, N, T, C, mode, Ap, Y.ctypes.data)
    return Y


# ---------------------------------------------------------------- training entry: TwELL -> hybrid (NEXT-4)
def twell_to_ell(words, N: int, T: int, C: int, ell_w: int):
    """(ell_val uint16 [M, ell_w] (0 past nnz), ell_col int16 [M, ell_w] (-1 past nnz), row_nnz, (l0, l1))."""
    words = np.ascontiguousarray(words, dtype=np.uint32)
    M = words.shape[0]
    val = np.zeros((M, ell_w), dtype=np.uint16)
    col = np.full((M, ell_w), -1, dtype=np.int16)
    nnz = np.zeros(M, dtype=np.int32)
    l = np.zeros(2, dtype=np.float64)
    _load().oracle_twell_to_ell(words.ctypes.data, M, N, T, C, ell_w, val.ctypes.data, col.ctypes.data,
                                nnz.ctypes.data, l.ctypes.data)
    return val, col, nnz, (float(l[0]), float(l[1]))


# ---------------------------------------------------------------- training forward on the hybrid format (NEXT-4)
def hybrid_sddmm(A, B, ell_col, row_nnz, row_loc, P_ell, dense_map, P_dense, gate: bool):
    """Listing 5 + Alg.3 dense tail (oracle_hybrid_sddmm): (out_ell fp64 [M, ell_w], out_dense fp64 [n_dense, N]);
    entries outside the pattern are 0."""
    A, B = _u16(A), _u16(B)
    M, K = A.shape
    N = B.shape[0]
    ell_col = np.ascontiguousarray(ell_col, dtype=np.int16)
    ell_w = ell_col.shape[1]
    row_nnz = np.ascontiguousarray(row_nnz, dtype=np.int32)
    row_loc = np.ascontiguousarray(row_loc, dtype=np.int32)
    P_ell = _u16(P_ell) if P_ell is not None else np.zeros((M, ell_w), dtype=np.uint16)
    dense_map = np.ascontiguousarray(dense_map, dtype=np.int32)
    nd = dense_map.shape[0]
    P_dense = _u16(P_dense) if nd else np.zeros((1, N), dtype=np.uint16)
    out_ell = np.zeros((M, ell_w), dtype=np.float64)
    out_dense = np.zeros((max(nd, 1), N), dtype=np.float64)
    _load().oracle_hybrid_sddmm(A.ctypes.data, B.ctypes.data, M, K, N, ell_w, ell_col.ctypes.data, row_nnz.ctypes.data,
                                row_loc.ctypes.data, P_ell.ctypes.data, nd, dense_map.ctypes.data, P_dense.ctypes.data,
                                1 if gate else 0, out_ell.ctypes.data, out_dense.ctypes.data)
    return out_ell, out_dense[:nd]


def hybrid_spmm(ell_val, ell_col, row_nnz, row_loc, dense_map, D, W) -> np.ndarray:
    """Listing 6 + Alg.3 (oracle_hybrid_spmm): Y fp64 [M, K]; values ell_val / D given in fp64."""
    W = _u16(W)
    N, K = W.shape
    ell_val = np.ascontiguousarray(ell_val, dtype=np.float64)
    M, ell_w = ell_val.shape
    ell_col = np.ascontiguousarray(ell_col, dtype=np.int16)
    row_nnz = np.ascontiguousarray(row_nnz, dtype=np.int32)
    row_loc = np.ascontiguousarray(row_loc, dtype=np.int32)
    dense_map = np.ascontiguousarray(dense_map, dtype=np.int32)
    nd = dense_map.shape[0]
    D = np.ascontiguousarray(D, dtype=np.float64) if nd else np.zeros((1, N), dtype=np.float64)
    Y = np.empty((M, K), dtype=np.float64)
    _load().oracle_hybrid_spmm(ell_val.ctypes.data, ell_col.ctypes.data, row_nnz.ctypes.data, row_loc.ctypes.data, M,
                               ell_w, nd, dense_map.ctypes.data, D.ctypes.data, W.ctypes.data, N, K, Y.ctypes.data)
    return Y


def hybrid_from_dense(H, ell_w: int, dense_cap: int):
    """Reference hybrid partition of a dense matrix: rows with <= ell_w non-zeros -> ELL (ascending columns),
    wider rows -> dense tail in row order (row_loc = slot), beyond dense_cap -> dropped (-2).  Plain numpy; used to
    build SpMM / SDDMM test inputs, not a GPU-kernel model."""
    H = np.asarray(H)
    M, N = H.shape
    col = np.full((M, ell_w), -1, dtype=np.int16)
    nnz = np.zeros(M, dtype=np.int32)
    loc = np.full(M, -1, dtype=np.int32)
    dmap = []
    for m in range(M):
        idx = np.flatnonzero(H[m])
        nnz[m] = len(idx)
        if len(idx) <= ell_w:
            col[m, :len(idx)] = idx.astype(np.int64).astype(np.uint16).view(np.int16)
        elif len(dmap) < dense_cap:
            loc[m] = len(dmap)
            dmap.append(m)
        else:
            loc[m] = -2
    return col, nnz, loc, np.array(dmap, dtype=np.int32)
