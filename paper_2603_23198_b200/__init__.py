"""B200-native (sm_100a) sparse gated-FFN forward with the TwELL format (arxiv 2603.23198).

The compute path is the C-ABI library ``libsffn.so`` (include/sffn.h); ``sffn`` is its thin binding.
"""
from . import sffn  # noqa: F401
from .sffn import (Comm, SffnError, dense_forward, forward, gate_gemm_f32, overflow_check, pack,  # noqa: F401
                   twell_view, up_down_workspace_bytes, pack_f32, up_down_f32, forward_f32,
                   transpose, twell_words, unpack, up_down, workspace_bytes)
