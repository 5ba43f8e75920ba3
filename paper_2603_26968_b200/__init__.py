"""LOPC hot path (arxiv 2603.26968) on B200: quantize -> local-order repair ->
chunked lossless coding, and the matching decoder, as hand-written sm_100a
CUDA kernels behind the C-ABI in include/lopc.h."""
from .lopc import (Comm, LopcError, check, critical_points, comm_unique_id, compress, compress_bound, compress_slab,  # noqa: F401
                   compress_noa, compress_slabs_local, decompress, decompress_slab, last_stats, load, repair, set_repair_engine, set_timing,
                   slab_bound, slab_info, slab_partition, stream_info, value_range, write_header)
from .lopc import noa_eps, set_decoder, set_index64  # noqa: F401
