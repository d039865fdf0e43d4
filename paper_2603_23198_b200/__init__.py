"""B200-native (sm_100a) sparse gated-FFN forward with the TwELL format (arxiv 2603.23198).

The compute path is the C-ABI library ``libsffn.so`` (include/sffn.h); ``sffn`` is its thin binding.
"""
from . import sffn  # noqa: F401
from .sffn import (Comm, SffnError, dense_forward, down, forward, forward_hybrid, forward_nongated, forward_f32, forward_host, forward_host_chunks, forward_train, gate_gemm_f32, hybrid_sddmm, hybrid_spmm, launch_count,  # noqa: F401
                   overflow_check, pack, pack_f32, transpose, twell_to_hybrid, twell_view, twell_words, union_stats, unpack,
                   up_down, up_down_f32, up_down_workspace_bytes, workspace_bytes)
