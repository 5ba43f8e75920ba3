"""Host-side logic of the multi-GPU slab mode, torch.distributed
only: range bounds, payload offsets, and assembling the single-GPU stream from
the per-rank outputs of lopc_compress_slab.  No LOPC arithmetic happens here;
the kernels run behind lopc_compress_slab on every rank."""
from __future__ import annotations

import struct

HDR = 64


def payload_offsets(n_chunks: int, payload_sizes: list[int]) -> tuple[list[int], int]:
    """Exclusive scan of the per-rank payload sizes after the header and the
    8-byte-per-chunk size table: (offset of each rank's payload slice, total
    stream bytes).  lopc_compress_slab computes the same from its allgather."""
    off = HDR + 8 * n_chunks
    offs = []
    for p in payload_sizes:
        offs.append(off)
        off += p
    return offs, off


def split_local(local: bytes, n_chunks_local: int) -> tuple[bytes, bytes]:
    """A rank's out_local = table slice (8 bytes per owned chunk) ‖ payload slice."""
    return local[: 8 * n_chunks_local], local[8 * n_chunks_local:]


def assemble_stream(header: bytes, locals_: list[bytes], chunks_per_rank: list[int]) -> bytes:
    """header ‖ table slices in rank order ‖ payload slices in rank order."""
    tables, pays = zip(*(split_local(b, c) for b, c in zip(locals_, chunks_per_rank)))
    total = HDR + sum(len(t) for t in tables) + sum(len(p) for p in pays)
    if struct.unpack_from("<Q", header, 56)[0] != total:
        raise ValueError("header total does not match the slices")
    return header + b"".join(tables) + b"".join(pays)


def gather_stream(local: bytes, header: bytes, n_chunks_local: int, group=None) -> bytes | None:
    """Collect every rank's out_local on rank 0 (torch.distributed objects)
    and assemble the stream there; other ranks get None."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    objs = [None] * world
    dist.all_gather_object(objs, (local, n_chunks_local), group=group)
    if dist.get_rank(group) != 0:
        return None
    return assemble_stream(header, [o[0] for o in objs], [o[1] for o in objs])
