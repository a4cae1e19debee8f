"""B200-native SRT hot path (arXiv 2601.09083): per-prompt tree caches in HBM,
batched insert / draft / lossless verify as hand-written sm_100a CUDA kernels
behind the C ABI of include/srt.h.  See DESIGN.md.

This package never imports the test oracle (``oracle/``) and has no CPU
fallback: without libsrt.so or a CUDA device every call raises.
"""
from ._lib import SrtError, load as load_library  # noqa: F401
from .srt import (DraftOut, SrtCache, VerifyOut, config, log_det_range, noise_table,  # noqa: F401
                  row_noise, stream_read)

__all__ = ["SrtCache", "DraftOut", "VerifyOut", "config", "noise_table", "log_det_range",
           "row_noise", "stream_read", "SrtError",
           "load_library"]
