"""Thin ctypes binding over libsffn.so (include/sffn.h) — argument marshalling only.

Every step of the path runs in the library's sm_100a kernels; this module only turns torch tensors into
device pointers + sizes and the current CUDA stream into a ``cudaStream_t``.  There is no CPU fallback:
if the shared library is missing or the device is not a B200 the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SFFN_LIB") or os.path.join(_HERE, "libsffn.so")

OK, ERR_INVALID_ARG, ERR_SHAPE, ERR_TILE_OVERFLOW, ERR_CUDA, ERR_NCCL, ERR_UNSUPPORTED = range(7)
ALGO_AUTO, ALGO_GATHER, ALGO_UNION = 0, 1, 2
_ALGOS = {"auto": ALGO_AUTO, "gather": ALGO_GATHER, "union": ALGO_UNION}


def _algo(a) -> int:
    return _ALGOS[a] if isinstance(a, str) else int(a)

_lib = None

# name -> (restype, argtypes); mirrors include/sffn.h
_vp, _i64, _int, _sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
_SIGS = {
    "sffn_status_string": (ctypes.c_char_p, [_int]),
    "sffn_version": (ctypes.c_char_p, []),
    "sffn_twell_words": (_i64, [_i64, _i64, _int, _int]),
    "sffn_up_down_workspace_bytes": (_sz, [_i64, _i64, _i64, _int, _int, _int]),
    "sffn_forward_workspace_bytes": (_sz, [_i64, _i64, _i64, _int, _int, _int]),
    "sffn_pack": (_int, [_vp, _vp, _i64, _i64, _i64, _int, _int, _vp, _vp, _vp]),
    "sffn_unpack": (_int, [_vp, _i64, _i64, _int, _int, _i64, _i64, _vp, _vp]),
    "sffn_up_down": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _int, _vp, _vp, _sz, _int, _vp]),
    "sffn_forward": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _int, _vp, _vp, _sz, _vp, _int, _vp]),
    "sffn_dense_forward": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "sffn_transpose_bf16": (_int, [_vp, _i64, _i64, _vp, _vp]),
    "sffn_gate_gemm_f32": (_int, [_vp, _vp, _i64, _i64, _i64, _vp, _vp]),
    "sffn_overflow_check": (_int, [_vp, _vp, ctypes.POINTER(ctypes.c_uint32)]),
    "sffn_comm_unique_id": (_int, [_vp]),
    "sffn_comm_init": (_int, [ctypes.POINTER(_vp), _int, _int, _vp, _int]),
    "sffn_comm_destroy": (_int, [_vp]),
    "sffn_comm_size": (_int, [_vp]),
    "sffn_sharded_forward": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _int, _vp, _vp, _sz, _vp,
                                    _int, _int, _vp]),
    "sffn_allreduce_bf16": (_int, [_vp, _vp, _i64, _vp]),
    "sffn_f32_twell_bytes": (_sz, [_i64, _i64, _int, _int]),
    "sffn_union_stats": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp]),
    "sffn_hybrid_workspace_bytes": (_sz, [_i64, _i64, _i64, _int, _int, _int, _i64]),
    "sffn_forward_hybrid": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _int, _vp, _vp, _sz, _i64, _vp, _vp,
                                   _int, _vp]),
    "sffn_twell_to_hybrid": (_int, [_vp, _i64, _i64, _int, _int, _int, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp,
                                    _vp]),
    "sffn_down": (_int, [_vp, _vp, _i64, _i64, _i64, _int, _int, _vp, _vp, _sz, _int, _vp]),
    "sffn_forward_nongated": (_int, [_vp, _vp, _vp, _i64, _i64, _i64, _int, _int, _vp, _vp, _sz, _vp, _int, _vp]),
    "sffn_forward_host_stage_bytes": (_sz, [_i64, _i64]),
    "sffn_forward_host_chunks": (_i64, [_i64, _i64, _vp, _i64]),
    "sffn_comm_symmetric_init": (_int, [_vp, _i64, _i64]),
    "sffn_comm_symmetric_info": (_int, [_vp, _vp, _vp, _vp]),
    "sffn_allreduce_sym_bf16": (_int, [_vp, _vp, _vp, _i64, _i64, _vp]),
    "sffn_reduce_scatter_sym_bf16": (_int, [_vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp]),
    "sffn_sharded_forward_sym": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _int, _vp, _vp, _sz, _vp,
                                        _int, _vp]),
    "sffn_sharded_forward_fused": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _int, _vp, _vp, _sz, _vp,
                                          _vp]),
    "sffn__forward_fused": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _int, _vp, _vp, _sz, _vp, _vp, _int,
                                   _int, _int, _vp]),
    "sffn_hybrid_mm_workspace_bytes": (_sz, [_i64, _i64, _i64]),
    "sffn_hybrid_sddmm": (_int, [_vp, _vp, _i64, _i64, _i64, _int, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _int, _vp,
                                 _vp, _vp, _sz, _vp]),
    "sffn_hybrid_spmm": (_int, [_vp, _vp, _vp, _vp, _i64, _int, _i64, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _sz,
                                _vp]),
    "sffn_forward_train": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _int, _vp, _int, _vp, _vp, _vp, _vp, _vp,
                                  _i64, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp, _vp]),
    "sffn_launch_count": (_i64, []),
    "sffn_union_block_rows": (_int, []),
    "sffn_forward_host": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _int, _vp, _vp, _sz, _vp, _sz, _vp, _int,
                                 _i64, _vp]),
    "sffn_pack_f32": (_int, [_vp, _vp, _i64, _i64, _i64, _int, _int, _vp, _vp, _vp, _vp, _vp]),
    "sffn_up_down_f32": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _int, _vp, _vp]),
    "sffn_forward_f32": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _int, _vp, _vp, _sz, _vp, _vp]),
}


class SffnError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {status_string(status)} ({status})")


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `make` (or __graft_entry__.build()); "
                              "there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            if not hasattr(L, name) and os.environ.get("SFFN_LIB"):
                continue  # an older build under A/B (SFFN_LIB): bind what it exports
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def status_string(s: int) -> str:
    return lib().sffn_status_string(s).decode()


def version() -> str:
    return lib().sffn_version().decode()


def _chk(status: int, what: str):
    if status != OK:
        raise SffnError(status, what)


def _p(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("sffn: tensors must be CUDA tensors (device memory)")
    if not t.is_contiguous():
        raise ValueError("sffn: tensors must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _bf16(t: torch.Tensor, name: str):
    if t.dtype != torch.bfloat16:
        raise TypeError(f"sffn: {name} must be bfloat16, got {t.dtype}")
    return _p(t)


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def twell_words(M: int, N: int, T: int, C: int) -> int:
    return int(lib().sffn_twell_words(M, N, T, C))


def workspace_bytes(M: int, K: int, N: int, T: int, C: int, algo="auto") -> int:
    """Bytes of workspace sffn_forward needs (TwELL + up/down workspace)."""
    return int(lib().sffn_forward_workspace_bytes(M, K, N, T, C, _algo(algo)))


def up_down_workspace_bytes(M: int, K: int, N: int, T: int, C: int, algo="auto") -> int:
    return int(lib().sffn_up_down_workspace_bytes(M, K, N, T, C, _algo(algo)))


def _ws(nbytes: int, device, ws=None):
    if ws is not None:
        return ws
    return torch.empty(max(nbytes, 16), dtype=torch.uint8, device=device)


def pack(x: torch.Tensor, wg: torch.Tensor, T: int = 256, C: int = 8, out: torch.Tensor | None = None,
         overflow: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """TwELL of relu(x wg^T) (Alg.1).  Returns int32 [M, N/C] holding the packed uint32 words."""
    M, K = x.shape
    N = wg.shape[0]
    if out is None:
        out = torch.empty((M, N // C), dtype=torch.int32, device=x.device)
    _chk(lib().sffn_pack(_bf16(x, "x"), _bf16(wg, "wg"), M, K, N, T, C, _p(out), _p(overflow), _stream(stream)),
         "sffn_pack")
    return out


def unpack(tw: torch.Tensor, N: int, T: int = 256, C: int = 8, out: torch.Tensor | None = None,
           col_offset: int = 0, stream=None) -> torch.Tensor:
    M = tw.shape[0]
    if out is None:
        out = torch.empty((M, N), dtype=torch.bfloat16, device=tw.device)
    _chk(lib().sffn_unpack(_p(tw), M, N, T, C, col_offset, out.shape[1], _bf16(out, "out"), _stream(stream)),
         "sffn_unpack")
    return out


def up_down(x, tw, wu, wd, T: int = 256, C: int = 8, out=None, workspace=None, algo="auto",
            stream=None) -> torch.Tensor:
    M, K = x.shape
    N = wu.shape[0]
    a = _algo(algo)
    if out is None:
        out = torch.empty((M, K), dtype=torch.bfloat16, device=x.device)
    workspace = _ws(up_down_workspace_bytes(M, K, N, T, C, a), x.device, workspace)
    _chk(lib().sffn_up_down(_bf16(x, "x"), _p(tw), _bf16(wu, "wu"), _bf16(wd, "wd"), M, K, N, T, C,
                            _bf16(out, "out"), _p(workspace), workspace.numel() * workspace.element_size(), a,
                            _stream(stream)), "sffn_up_down")
    return out


def twell_view(workspace: torch.Tensor, M: int, N: int, C: int) -> torch.Tensor:
    """The packed TwELL (int32 [M, N/C]) that sffn_forward leaves at the start of its workspace."""
    return workspace[: M * (N // C) * 4].view(torch.int32).view(M, N // C)


def forward(x, wg, wu, wd, T: int = 256, C: int = 8, out=None, workspace=None, overflow=None, algo="auto",
            stream=None) -> torch.Tensor:
    """Sparse FFN forward (pack + fused up/down).  workspace: uint8 device buffer >= workspace_bytes."""
    M, K = x.shape
    N = wg.shape[0]
    a = _algo(algo)
    if out is None:
        out = torch.empty((M, K), dtype=torch.bfloat16, device=x.device)
    workspace = _ws(workspace_bytes(M, K, N, T, C, a), x.device, workspace)
    _chk(lib().sffn_forward(_bf16(x, "x"), _bf16(wg, "wg"), _bf16(wu, "wu"), _bf16(wd, "wd"), M, K, N, T, C,
                            _bf16(out, "out"), _p(workspace), workspace.numel() * workspace.element_size(),
                            _p(overflow), a, _stream(stream)), "sffn_forward")
    return out


def launch_count() -> int:
    """Kernels launched (or captured) by the library so far in this process."""
    return int(lib().sffn_launch_count())


def forward_host_chunks(M: int, chunk_rows: int = 4096) -> list:
    """The row-chunk schedule of forward_host (host-side planner of the C library)."""
    n = int(lib().sffn_forward_host_chunks(M, chunk_rows, None, 0))
    buf = (ctypes.c_int64 * max(1, n))()
    lib().sffn_forward_host_chunks(M, chunk_rows, ctypes.cast(buf, ctypes.c_void_p), n)
    return [int(buf[i]) for i in range(n)]


def forward_host(x_host, wg, wu, wd, T: int = 256, C: int = 8, out=None, workspace=None, stage=None,
                 overflow=None, algo="auto", chunk_rows: int = 4096, stream=None, stage_slots: int = 2,
                 synchronize: bool = True) -> torch.Tensor:
    """Sparse forward with X / Y in (pinned) host memory; copies overlap compute (sffn_forward_host).
    stage_slots: X / Y staging slots on the device (>= 2; more lets copies run further ahead).
    The device-to-host copies into `out` are stream-ordered: with synchronize=True (default) the stream is
    synchronized before returning, so `out` can be read at once; with synchronize=False the caller must
    synchronize the stream before reading `out` (reading a host tensor does not wait for CUDA work)."""
    M, K = x_host.shape
    N = wg.shape[0]
    if x_host.is_cuda or x_host.dtype != torch.bfloat16 or not x_host.is_contiguous():
        raise ValueError("x_host must be a contiguous bf16 CPU tensor (pinned for overlap)")
    if out is None:
        out = torch.empty((M, K), dtype=torch.bfloat16, pin_memory=True)
    a = _algo(algo)
    rows = min(chunk_rows, ((M + 127) // 128) * 128)
    wsz = workspace_bytes(min(rows, M), K, N, T, C, a)
    # two workspaces: consecutive chunks compute on two streams (sffn_forward_host)
    workspace = _ws((wsz + 1023) // 1024 * 1024 + wsz, wg.device, workspace)
    stage = _ws(int(lib().sffn_forward_host_stage_bytes(K, rows)) * max(2, stage_slots) // 2, wg.device, stage)
    _chk(lib().sffn_forward_host(ctypes.c_void_p(x_host.data_ptr()), _bf16(wg, "wg"), _bf16(wu, "wu"),
                                 _bf16(wd, "wd"), M, K, N, T, C, ctypes.c_void_p(out.data_ptr()), _p(workspace),
                                 workspace.numel() * workspace.element_size(), _p(stage),
                                 stage.numel() * stage.element_size(), _p(overflow), a, chunk_rows,
                                 _stream(stream)), "sffn_forward_host")
    if synchronize:
        (torch.cuda.current_stream() if stream is None else stream).synchronize()
    return out


def forward_hybrid(x, wg, wu, wd, T: int = 256, C: int = 8, backup_rows: int | None = None, out=None,
                   workspace=None, backup_count=None, overflow=None, algo="auto", stream=None):
    """Overflow-exact sparse forward: rows with an overflowed TwELL tile are recomputed densely (NEXT-1)."""
    M, K = x.shape
    N = wg.shape[0]
    a = _algo(algo)
    R = max(128, M // 8) if backup_rows is None else backup_rows
    if out is None:
        out = torch.empty((M, K), dtype=torch.bfloat16, device=x.device)
    workspace = _ws(int(lib().sffn_hybrid_workspace_bytes(M, K, N, T, C, a, R)), x.device, workspace)
    _chk(lib().sffn_forward_hybrid(_bf16(x, "x"), _bf16(wg, "wg"), _bf16(wu, "wu"), _bf16(wd, "wd"), M, K, N, T, C,
                                   _bf16(out, "out"), _p(workspace), workspace.numel() * workspace.element_size(), R,
                                   _p(backup_count), _p(overflow), a, _stream(stream)), "sffn_forward_hybrid")
    return out


def twell_to_hybrid(tw, N: int, T: int = 256, C: int = 8, ell_w: int = 128, dense_cap: int | None = None,
                    stream=None) -> dict:
    """TwELL -> hybrid (ELL + dense tail + row locations) with L0/L1 statistics (NEXT-4, Listing 4)."""
    M = tw.shape[0]
    dev = tw.device
    D = max(1, M // 8) if dense_cap is None else dense_cap
    out = {"ell_val": torch.empty((M, ell_w), dtype=torch.bfloat16, device=dev),
           "ell_col": torch.empty((M, ell_w), dtype=torch.int16, device=dev),
           "row_nnz": torch.empty(M, dtype=torch.int32, device=dev),
           "row_loc": torch.empty(M, dtype=torch.int32, device=dev),
           "dense_rows": torch.empty((max(D, 1), N), dtype=torch.bfloat16, device=dev),
           "dense_map": torch.empty(max(D, 1), dtype=torch.int32, device=dev),
           "dense_count": torch.zeros(1, dtype=torch.int32, device=dev),
           "l0l1": torch.zeros(2, dtype=torch.float64, device=dev)}
    _chk(lib().sffn_twell_to_hybrid(_p(tw), M, N, T, C, ell_w, _p(out["ell_val"]), _p(out["ell_col"]),
                                    _p(out["row_nnz"]), _p(out["row_loc"]), D, _p(out["dense_rows"]),
                                    _p(out["dense_map"]), _p(out["dense_count"]), _p(out["l0l1"]), _stream(stream)),
         "sffn_twell_to_hybrid")
    return out


def forward_train(x, wg, wu, wd, T: int = 256, C: int = 8, ell_w: int = 128, dense_cap: int | None = None, out=None,
                  workspace=None, overflow=None, stream=None):
    """Training forward through the union path: (Y, hyb_g, hyb_h) — hyb_g the hybrid form of h_g (as twell_to_hybrid),
    hyb_h the same pattern holding h = h_g (.) x W_u (what hybrid_sddmm computes), both dicts."""
    M, K = x.shape
    N = wg.shape[0]
    dev = x.device
    D = max(1, M // 8) if dense_cap is None else dense_cap
    if out is None:
        out = torch.empty((M, K), dtype=torch.bfloat16, device=dev)
    g = {"ell_val": torch.empty((M, ell_w), dtype=torch.bfloat16, device=dev),
         "ell_col": torch.empty((M, ell_w), dtype=torch.int16, device=dev),
         "row_nnz": torch.empty(M, dtype=torch.int32, device=dev),
         "row_loc": torch.empty(M, dtype=torch.int32, device=dev),
         "dense_rows": torch.empty((max(D, 1), N), dtype=torch.bfloat16, device=dev),
         "dense_map": torch.empty(max(D, 1), dtype=torch.int32, device=dev),
         "dense_count": torch.zeros(1, dtype=torch.int32, device=dev),
         "l0l1": torch.zeros(2, dtype=torch.float64, device=dev)}
    h = dict(g)
    h["ell_val"] = torch.zeros_like(g["ell_val"])
    h["dense_rows"] = torch.zeros_like(g["dense_rows"])
    workspace = _ws(workspace_bytes(M, K, N, T, C, "union"), dev, workspace)
    _chk(lib().sffn_forward_train(_bf16(x, "x"), _bf16(wg, "wg"), _bf16(wu, "wu"), _bf16(wd, "wd"), M, K, N, T, C,
                                  _bf16(out, "out"), ell_w, _p(g["ell_val"]), _p(h["ell_val"]), _p(g["ell_col"]),
                                  _p(g["row_nnz"]), _p(g["row_loc"]), D, _p(g["dense_rows"]), _p(h["dense_rows"]),
                                  _p(g["dense_map"]), _p(g["dense_count"]), _p(g["l0l1"]), _p(workspace),
                                  workspace.numel() * workspace.element_size(), _p(overflow), _stream(stream)),
         "sffn_forward_train")
    return out, g, h


def hybrid_sddmm(a, b, hyb: dict, gate: bool = True, workspace=None, stream=None) -> dict:
    """Training forward, dense -> hybrid (Listing 5 + Alg.3): h = g (.) a b^T on the pattern of `hyb` (a dict from
    twell_to_hybrid), g = the pattern values (gate=True) or its 0/1 mask.  Returns a hybrid dict with the same
    pattern arrays and new "ell_val" / "dense_rows"."""
    M, K = a.shape
    N = b.shape[0]
    ell_w = hyb["ell_col"].shape[1]
    D = hyb["dense_map"].shape[0]
    out = dict(hyb)
    out["ell_val"] = torch.zeros_like(hyb["ell_val"])
    out["dense_rows"] = torch.zeros_like(hyb["dense_rows"])
    workspace = _ws(int(lib().sffn_hybrid_mm_workspace_bytes(D, K, N)), a.device, workspace)
    _chk(lib().sffn_hybrid_sddmm(_bf16(a, "a"), _bf16(b, "b"), M, K, N, ell_w, _p(hyb["ell_col"]), _p(hyb["row_nnz"]),
                                 _p(hyb["row_loc"]), _p(hyb["ell_val"]), D, _p(hyb["dense_map"]),
                                 _p(hyb["dense_count"]), _p(hyb["dense_rows"]), 1 if gate else 0, _p(out["ell_val"]),
                                 _p(out["dense_rows"]), _p(workspace), workspace.numel() * workspace.element_size(),
                                 _stream(stream)), "sffn_hybrid_sddmm")
    return out


def hybrid_spmm(hyb: dict, w, out=None, workspace=None, stream=None) -> torch.Tensor:
    """Training forward, hybrid -> dense (Listing 6 + Alg.3): Y = h W for the hybrid h and W [N, K] (hidden-major)."""
    M, ell_w = hyb["ell_col"].shape
    N, K = w.shape
    D = hyb["dense_map"].shape[0]
    if out is None:
        out = torch.empty((M, K), dtype=torch.bfloat16, device=w.device)
    workspace = _ws(int(lib().sffn_hybrid_mm_workspace_bytes(D, K, N)), w.device, workspace)
    _chk(lib().sffn_hybrid_spmm(_p(hyb["ell_val"]), _p(hyb["ell_col"]), _p(hyb["row_nnz"]), _p(hyb["row_loc"]), M,
                                ell_w, D, _p(hyb["dense_map"]), _p(hyb["dense_count"]), _p(hyb["dense_rows"]),
                                _bf16(w, "w"), N, K, _bf16(out, "out"), _p(workspace),
                                workspace.numel() * workspace.element_size(), _stream(stream)), "sffn_hybrid_spmm")
    return out


def down(tw, wd, K: int, T: int = 256, C: int = 8, out=None, workspace=None, algo="auto", stream=None):
    """Non-gated down projection from a TwELL of h = relu(x W_u) (App.C)."""
    M = tw.shape[0]
    N = wd.shape[0]
    a = _algo(algo)
    if out is None:
        out = torch.empty((M, K), dtype=torch.bfloat16, device=wd.device)
    workspace = _ws(up_down_workspace_bytes(M, K, N, T, C, a), wd.device, workspace)
    _chk(lib().sffn_down(_p(tw), _bf16(wd, "wd"), M, K, N, T, C, _bf16(out, "out"), _p(workspace),
                         workspace.numel() * workspace.element_size(), a, _stream(stream)), "sffn_down")
    return out


def forward_nongated(x, wu, wd, T: int = 256, C: int = 8, out=None, workspace=None, overflow=None, algo="auto",
                     stream=None):
    """Non-gated sparse FFN y = relu(x W_u) W_d (App.C)."""
    M, K = x.shape
    N = wu.shape[0]
    a = _algo(algo)
    if out is None:
        out = torch.empty((M, K), dtype=torch.bfloat16, device=x.device)
    workspace = _ws(workspace_bytes(M, K, N, T, C, a), x.device, workspace)
    _chk(lib().sffn_forward_nongated(_bf16(x, "x"), _bf16(wu, "wu"), _bf16(wd, "wd"), M, K, N, T, C,
                                     _bf16(out, "out"), _p(workspace), workspace.numel() * workspace.element_size(),
                                     _p(overflow), a, _stream(stream)), "sffn_forward_nongated")
    return out


def dense_forward(x, wg, wu, wdT, h=None, out=None, stream=None) -> torch.Tensor:
    """The library's dense tcgen05 FFN (speedup denominator).  wdT = W_d^T, [K, N]."""
    M, K = x.shape
    N = wg.shape[0]
    if h is None:
        h = torch.empty((M, N), dtype=torch.bfloat16, device=x.device)
    if out is None:
        out = torch.empty((M, K), dtype=torch.bfloat16, device=x.device)
    _chk(lib().sffn_dense_forward(_bf16(x, "x"), _bf16(wg, "wg"), _bf16(wu, "wu"), _bf16(wdT, "wdT"), M, K, N,
                                  _bf16(h, "h"), _bf16(out, "out"), _stream(stream)), "sffn_dense_forward")
    return out


def transpose(a: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    R, Cc = a.shape
    if out is None:
        out = torch.empty((Cc, R), dtype=torch.bfloat16, device=a.device)
    _chk(lib().sffn_transpose_bf16(_bf16(a, "a"), R, Cc, _bf16(out, "out"), _stream(stream)), "sffn_transpose_bf16")
    return out


def gate_gemm_f32(x, wg, out=None, stream=None) -> torch.Tensor:
    M, K = x.shape
    N = wg.shape[0]
    if out is None:
        out = torch.empty((M, N), dtype=torch.float32, device=x.device)
    _chk(lib().sffn_gate_gemm_f32(_bf16(x, "x"), _bf16(wg, "wg"), M, K, N, _p(out), _stream(stream)),
         "sffn_gate_gemm_f32")
    return out


def union_stats(up_down_workspace: torch.Tensor, M: int, K: int, N: int, stream=None) -> dict:
    """Union sizes left in an sffn_up_down(algo="union") workspace (synchronizes the stream)."""
    a, b, t = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _chk(lib().sffn_union_stats(_p(up_down_workspace), M, K, N, ctypes.byref(a), ctypes.byref(b), ctypes.byref(t),
                                _stream(stream)), "sffn_union_stats")
    return {"padded_sum": a.value, "union_sum": b.value, "up_tiles": t.value,
            "block_rows": int(lib().sffn_union_block_rows())}


def overflow_check(overflow: torch.Tensor, stream=None) -> int:
    """Synchronizes the stream and returns the device overflow count (0 = OK)."""
    h = ctypes.c_uint32(0)
    s = lib().sffn_overflow_check(_p(overflow), _stream(stream), ctypes.byref(h))
    if s not in (OK, ERR_TILE_OVERFLOW):
        _chk(s, "sffn_overflow_check")
    return int(h.value)


def _f32(t: torch.Tensor, name: str):
    if t.dtype != torch.float32:
        raise TypeError(f"sffn: {name} must be float32, got {t.dtype}")
    return _p(t)


def pack_f32(x, wg, T: int = 256, C: int = 8, overflow=None, stream=None):
    """fp32 mode: SoA TwELL (h_v float32 [M, N/C], h_I int16-stored uint16 [M, N/C], h_nz int32 [M, N/T])."""
    M, K = x.shape
    N = wg.shape[0]
    hv = torch.empty((M, N // C), dtype=torch.float32, device=x.device)
    hi = torch.empty((M, N // C), dtype=torch.int16, device=x.device)
    hnz = torch.empty((M, N // T), dtype=torch.int32, device=x.device)
    _chk(lib().sffn_pack_f32(_f32(x, "x"), _f32(wg, "wg"), M, K, N, T, C, _p(hv), _p(hi), _p(hnz), _p(overflow),
                             _stream(stream)), "sffn_pack_f32")
    return hv, hi, hnz


def up_down_f32(x, hv, hi, hnz, wu, wd, T: int = 256, C: int = 8, out=None, stream=None):
    M, K = x.shape
    N = wu.shape[0]
    if out is None:
        out = torch.empty((M, K), dtype=torch.float32, device=x.device)
    _chk(lib().sffn_up_down_f32(_f32(x, "x"), _p(hv), _p(hi), _p(hnz), _f32(wu, "wu"), _f32(wd, "wd"), M, K, N, T, C,
                                _f32(out, "out"), _stream(stream)), "sffn_up_down_f32")
    return out


def forward_f32(x, wg, wu, wd, T: int = 256, C: int = 8, out=None, workspace=None, overflow=None, stream=None):
    M, K = x.shape
    N = wg.shape[0]
    if out is None:
        out = torch.empty((M, K), dtype=torch.float32, device=x.device)
    nb = int(lib().sffn_f32_twell_bytes(M, N, T, C))
    workspace = _ws(nb, x.device, workspace)
    _chk(lib().sffn_forward_f32(_f32(x, "x"), _f32(wg, "wg"), _f32(wu, "wu"), _f32(wd, "wd"), M, K, N, T, C,
                                _f32(out, "out"), _p(workspace), workspace.numel() * workspace.element_size(),
                                _p(overflow), _stream(stream)), "sffn_forward_f32")
    return out


class Comm:
    """The library's own NCCL communicator for hidden-dim sharding; torch.distributed only broadcasts the id."""

    def __init__(self, rank: int, world: int, device: int, group=None):
        from .sharding import broadcast_id
        raw_id = None
        if rank == 0:
            buf = (ctypes.c_uint8 * 128)()
            _chk(lib().sffn_comm_unique_id(ctypes.cast(buf, ctypes.c_void_p)), "sffn_comm_unique_id")
            raw_id = bytes(buf)
        raw_id = broadcast_id(raw_id, rank, world, group)
        raw = (ctypes.c_uint8 * 128)(*raw_id)
        h = ctypes.c_void_p()
        _chk(lib().sffn_comm_init(ctypes.byref(h), world, rank, ctypes.cast(raw, ctypes.c_void_p), device),
             "sffn_comm_init")
        self.h, self.rank, self.world = h, rank, world

    def sharded_forward(self, x, wg_s, wu_s, wd_s, T=256, C=8, out=None, workspace=None, overflow=None,
                        algo="auto", n_chunks=1, stream=None):
        M, K = x.shape
        N_local = wg_s.shape[0]
        a = _algo(algo)
        if out is None:
            out = torch.empty((M, K), dtype=torch.bfloat16, device=x.device)
        workspace = _ws(workspace_bytes(M, K, N_local, T, C, a), x.device, workspace)
        _chk(lib().sffn_sharded_forward(self.h, _bf16(x, "x"), _bf16(wg_s, "wg"), _bf16(wu_s, "wu"),
                                        _bf16(wd_s, "wd"), M, K, N_local, T, C, _bf16(out, "out"), _p(workspace),
                                        workspace.numel() * workspace.element_size(), _p(overflow), a, n_chunks,
                                        _stream(stream)), "sffn_sharded_forward")
        return out

    # ------------------------------------------------------------ NEXT-3: symmetric-memory all-reduce
    def symmetric_init(self, max_rows: int, K: int) -> bool:
        """Collective: registers a max_rows x K bf16 symmetric window + NCCL device communicator.  False when
        the platform cannot (SFFN_ERR_UNSUPPORTED); other errors raise."""
        st = int(lib().sffn_comm_symmetric_init(self.h, max_rows, K))
        if st == 6:
            return False
        _chk(st, "sffn_comm_symmetric_init")
        return True

    def symmetric_info(self) -> dict:
        mm, rows, k = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()
        st = int(lib().sffn_comm_symmetric_info(self.h, ctypes.byref(mm), ctypes.byref(rows), ctypes.byref(k)))
        return {"ready": st == 0, "multimem": bool(mm.value), "max_rows": rows.value, "K": k.value}

    def allreduce_sym(self, src, out=None, stream=None):
        rows, K = src.shape
        if out is None:
            out = torch.empty_like(src)
        _chk(lib().sffn_allreduce_sym_bf16(self.h, _bf16(src, "src"), _bf16(out, "out"), rows, K, _stream(stream)),
             "sffn_allreduce_sym_bf16")
        return out

    def reduce_scatter_sym(self, src, stream=None):
        """This rank's row slice of the sum over ranks of `src` [rows, K] (NEXT-3 reduce-scatter variant)."""
        rows, K = src.shape
        r0, nr = ctypes.c_int64(), ctypes.c_int64()
        n = rows * (self.rank + 1) // self.world - rows * self.rank // self.world
        out = torch.empty((n, K), dtype=torch.bfloat16, device=src.device)
        _chk(lib().sffn_reduce_scatter_sym_bf16(self.h, _bf16(src, "src"), rows, K, _p(out) if n else None,
                                                ctypes.byref(r0), ctypes.byref(nr), _stream(stream)),
             "sffn_reduce_scatter_sym_bf16")
        return out, r0.value

    def sharded_forward_sym(self, x, wg_s, wu_s, wd_s, T=256, C=8, out=None, workspace=None, overflow=None,
                            algo="auto", stream=None):
        M, K = x.shape
        N_local = wg_s.shape[0]
        a = _algo(algo)
        if out is None:
            out = torch.empty((M, K), dtype=torch.bfloat16, device=x.device)
        workspace = _ws(workspace_bytes(M, K, N_local, T, C, a), x.device, workspace)
        _chk(lib().sffn_sharded_forward_sym(self.h, _bf16(x, "x"), _bf16(wg_s, "wg"), _bf16(wu_s, "wu"),
                                            _bf16(wd_s, "wd"), M, K, N_local, T, C, _bf16(out, "out"), _p(workspace),
                                            workspace.numel() * workspace.element_size(), _p(overflow), a,
                                            _stream(stream)), "sffn_sharded_forward_sym")
        return out

    def sharded_forward_fused(self, x, wg_s, wu_s, wd_s, T=256, C=8, out=None, workspace=None, overflow=None,
                              stream=None):
        """Union forward with the all-reduce fused into the DOWN GEMM (2048-row windows reduced as they finish);
        needs symmetric_init(max_rows >= M, K)."""
        M, K = x.shape
        N_local = wg_s.shape[0]
        if out is None:
            out = torch.empty((M, K), dtype=torch.bfloat16, device=x.device)
        workspace = _ws(workspace_bytes(M, K, N_local, T, C, ALGO_UNION), x.device, workspace)
        _chk(lib().sffn_sharded_forward_fused(self.h, _bf16(x, "x"), _bf16(wg_s, "wg"), _bf16(wu_s, "wu"),
                                              _bf16(wd_s, "wd"), M, K, N_local, T, C, _bf16(out, "out"),
                                              _p(workspace), workspace.numel() * workspace.element_size(),
                                              _p(overflow), _stream(stream)), "sffn_sharded_forward_fused")
        return out

    def allreduce(self, buf, stream=None):
        _chk(lib().sffn_allreduce_bf16(self.h, _bf16(buf, "buf"), buf.numel(), _stream(stream)),
             "sffn_allreduce_bf16")
        return buf

    def close(self):
        if self.h:
            lib().sffn_comm_destroy(self.h)
            self.h = None
