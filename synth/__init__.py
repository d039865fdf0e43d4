"""Seeded synthetic FFN inputs (X, W_g, W_u, W_d) — input generation only.

Shared by the CPU oracle tests and the CUDA path.  Holds none of the method's
arithmetic (no GEMM, threshold or TwELL packing); see synth.c for the recipe and
DESIGN.md §"Input recipe" for how it maps to the paper's workload statistics.

Arrays are returned as numpy ``uint16`` bf16 bit patterns (``dtype="bf16"``) or
``float32`` (``dtype="f32"``), row-major ``[rows, K]``; weights are hidden-major
``[N, K]`` for all three matrices.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libsynth.so")


class _Cfg(ctypes.Structure):
    _fields_ = [
        ("M", ctypes.c_int64), ("K", ctypes.c_int64), ("N", ctypes.c_int64),
        ("seed", ctypes.c_uint64),
        ("sparsity", ctypes.c_double), ("dead_frac", ctypes.c_double),
        ("tok_sigma", ctypes.c_double), ("pmax_ratio", ctypes.c_double),
        ("pos_alpha", ctypes.c_double),
        ("seq_len", ctypes.c_int64), ("Kb", ctypes.c_int64),
        ("share_q", ctypes.c_int32), ("x_exp", ctypes.c_int32), ("w_exp", ctypes.c_int32),
    ]


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "synth.c")
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", _LIB, src, "-lm"])
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.POINTER(_Cfg)
        lib.synth_token_targets.argtypes = [P, ctypes.c_void_p]
        lib.synth_x.argtypes = [P, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                ctypes.c_void_p, ctypes.c_void_p]
        lib.synth_w.argtypes = [P, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
        lib.synth_neuron.argtypes = [P, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        lib.synth_pattern.argtypes = [P, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                      ctypes.c_void_p]
        _lib = lib
    return _lib


@dataclasses.dataclass(frozen=True)
class Config:
    """One workload from BASELINE.json:configs."""
    name: str
    M: int
    K: int
    N: int
    sparsity: float
    T: int = 256
    C: int = 8
    dead_frac: float = 0.30
    tok_sigma: float = 1.0
    pmax_ratio: float = 3.5
    pos_alpha: float = 0.25
    seq_len: int = 2048
    Kb: int = 64
    share_q: int = 1
    x_exp: int = 3
    w_exp: int = 8
    seed: int = 0

    def replace(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)

    def _c(self) -> _Cfg:
        return _Cfg(self.M, self.K, self.N, self.seed, self.sparsity, self.dead_frac, self.tok_sigma,
                    self.pmax_ratio, self.pos_alpha, self.seq_len, self.Kb, self.share_q, self.x_exp,
                    self.w_exp)


CONFIGS = {
    # BASELINE.json configs[0]: tiny, CPU oracle in seconds; "tile 32" = T=32 columns
    "tiny": Config("tiny", M=128, K=64, N=256, sparsity=0.90, T=32, C=2, dead_frac=0.10,
                   pmax_ratio=1.5, Kb=8),
    # configs[1]: 1B-scale, heavy-tailed per-token nnz
    "1B": Config("1B", M=16384, K=2048, N=8192, sparsity=0.99),
    # configs[2]: 7B-scale headline
    "7B": Config("7B", M=32768, K=4096, N=14336, sparsity=0.99),
    # robustness: the paper's ">10x mean" tail with C=4
    "7B-tail": Config("7B-tail", M=32768, K=4096, N=14336, sparsity=0.99, C=4, pmax_ratio=10.0),
    # configs[3]: sparsity sweep
    "7B-s90": Config("7B-s90", M=32768, K=4096, N=14336, sparsity=0.90, C=2, pmax_ratio=3.0, dead_frac=0.10),
    "7B-s95": Config("7B-s95", M=32768, K=4096, N=14336, sparsity=0.95, C=2, pmax_ratio=6.0, dead_frac=0.20),
    "7B-s99": Config("7B-s99", M=32768, K=4096, N=14336, sparsity=0.99),
    "7B-s995": Config("7B-s995", M=32768, K=4096, N=14336, sparsity=0.995, pmax_ratio=7.0),
    "7B-s999": Config("7B-s999", M=32768, K=4096, N=14336, sparsity=0.999, pmax_ratio=10.0),
    # configs[4]: 70B-scale, hidden-dim sharded
    "70B": Config("70B", M=65536, K=8192, N=28672, sparsity=0.99),
}


def token_targets(cfg: Config) -> np.ndarray:
    lib = _load()
    c = cfg._c()
    p = np.empty(cfg.M, dtype=np.float64)
    lib.synth_token_targets(ctypes.byref(c), p.ctypes.data)
    return p


def gen_x(cfg: Config, row0: int = 0, nrows: int | None = None, dtype: str = "bf16",
          p: np.ndarray | None = None, return_bias: bool = False):
    lib = _load()
    nrows = cfg.M - row0 if nrows is None else nrows
    if p is None:
        p = token_targets(cfg)
    out = np.empty((nrows, cfg.K), dtype=np.float32 if dtype == "f32" else np.uint16)
    cb = np.empty(nrows, dtype=np.int32)
    c = cfg._c()
    lib.synth_x(ctypes.byref(c), p.ctypes.data, row0, nrows, int(dtype == "f32"), out.ctypes.data,
                cb.ctypes.data)
    return (out, cb) if return_bias else out


def gen_x_rows(cfg: Config, rows, dtype: str = "bf16", p: np.ndarray | None = None) -> np.ndarray:
    """X at an arbitrary set of row indices (each row is generated independently)."""
    if p is None:
        p = token_targets(cfg)
    rows = np.asarray(rows, dtype=np.int64)
    out = np.empty((len(rows), cfg.K), dtype=np.float32 if dtype == "f32" else np.uint16)
    for i, r in enumerate(rows):
        out[i] = gen_x(cfg, int(r), 1, dtype, p)[0]
    return out


def gen_w(cfg: Config, which: str, row0: int = 0, nrows: int | None = None, dtype: str = "bf16") -> np.ndarray:
    lib = _load()
    w = {"g": 0, "u": 1, "d": 2}[which]
    nrows = cfg.N - row0 if nrows is None else nrows
    out = np.empty((nrows, cfg.K), dtype=np.float32 if dtype == "f32" else np.uint16)
    c = cfg._c()
    lib.synth_w(ctypes.byref(c), w, row0, nrows, int(dtype == "f32"), out.ctypes.data)
    return out


def gen_pattern(cfg: Config, row0: int = 0, nrows: int | None = None, pop_sigma: float = 1.0,
                p: np.ndarray | None = None) -> np.ndarray:
    """"Direct TwELL" mode: a dense bf16 [nrows, N] activation matrix with the generator's per-token
    densities and a LogNormal(., pop_sigma) per-neuron popularity, values q * 2^-4 (q = 1..15), no gate GEMM.
    Pack it with the oracle (oracle.pack) to feed the fused up/down alone."""
    lib = _load()
    nrows = cfg.M - row0 if nrows is None else nrows
    if p is None:
        p = token_targets(cfg)
    out = np.empty((nrows, cfg.N), dtype=np.uint16)
    c = cfg._c()
    lib.synth_pattern(ctypes.byref(c), p.ctypes.data, row0, nrows, pop_sigma, out.ctypes.data)
    return out


def neuron_params(cfg: Config):
    """(beta_n * 64, dead_n) per neuron: the bias coefficient of the lognormal popularity model and the dead flag."""
    lib = _load()
    c = cfg._c()
    b = np.empty(cfg.N, dtype=np.int32)
    d = np.empty(cfg.N, dtype=np.int32)
    bi, di = ctypes.c_int32(), ctypes.c_int32()
    for n in range(cfg.N):
        lib.synth_neuron(ctypes.byref(c), n, ctypes.byref(bi), ctypes.byref(di))
        b[n], d[n] = bi.value, di.value
    return b, d


def q_bits(q: int, e: int) -> np.uint16:
    """bf16 bits of the grid value q * 2^-e (|q| < 16: exact)."""
    assert abs(q) < 16
    return np.uint16(np.array([q * 2.0 ** -e], dtype=np.float32).view(np.uint32)[0] >> 16)


def bf16_to_f32(a: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns (uint16) to float32."""
    return (a.astype(np.uint32) << 16).view(np.float32)


def worst_case_units(cfg: Config) -> int:
    """Bound on |sum_k q_x q_w| for any subset of k: must stay below 2^20."""
    return cfg.Kb * 14 * 7 + (cfg.K - cfg.Kb) * 14 * 7
