"""LOPC hot path (arxiv 2603.26968) on B200: quantize -> local-order repair ->
chunked lossless coding, and the matching decoder, as hand-written sm_100a
CUDA kernels behind the C-ABI in include/lopc.h."""
from .lopc import (LopcError, compress, compress_bound, decompress, last_stats, load, repair,  # noqa: F401
                   set_timing, stream_info)
