"""Host logic of the multi-GPU slab mode, on CPU: the range
partition and halo geometry exported by liblopc.so (host-only functions), the
halo exchange pattern over a real 2-process gloo group, and the distributed
stream assembly (per-rank table/payload slices + allgathered offsets) against
the oracle's single-stream bytes."""
import os
import socket

import numpy as np
import pytest
import torch

from synth.fields import eps_noa, random_field

lopc = pytest.importorskip("paper_2603_26968_b200")


def _have_lib():
    try:
        lopc.load(require_gpu=False)
        return True
    except ImportError:
        return False


pytestmark = pytest.mark.skipif(not _have_lib(), reason="liblopc.so not built")


def star_offsets(ndims):
    """Kuhn/Freudenthal star offsets, written out (G1)."""
    es = [(0, 1), (1, 0), (1, 1)] if ndims == 2 else [(0, 0, 1), (0, 1, 0), (0, 1, 1), (1, 0, 0), (1, 0, 1),
                                                      (1, 1, 0), (1, 1, 1)]
    return es + [tuple(-v for v in e) for e in es]


def neighbours_outside(shape, e0, e1):
    """Brute force: linear indices outside [e0, e1) that are star neighbours
    of an owned point."""
    idx = np.arange(int(np.prod(shape))).reshape(shape)
    out = set()
    own = np.zeros(idx.size, bool)
    own[e0:e1] = True
    coords = np.argwhere(own.reshape(shape))
    for off in star_offsets(len(shape)):
        q = coords + np.array(off)
        ok = np.all((q >= 0) & (q < np.array(shape)), axis=1)
        lin = np.ravel_multi_index(q[ok].T, shape)
        out.update(int(v) for v in lin if not own[v])
    return out


@pytest.mark.parametrize("shape,dt,world", [((20, 30, 40), torch.float32, 3), ((9, 50, 70), torch.float64, 2),
                                            ((300, 500), torch.float32, 4), ((64, 64), torch.float64, 2),
                                            ((100, 500, 500), torch.float32, 8)])
def test_partition_and_geometry(shape, dt, world):
    k = 4 if dt == torch.float32 else 8
    W = 16384 // k
    n = int(np.prod(shape))
    b = lopc.slab_partition(shape, dt, world)
    assert b[0] == 0 and b[-1] == n and all(b[i] < b[i + 1] for i in range(world))
    assert all(v % W == 0 for v in b[1:-1])
    infos = [lopc.slab_info(shape, dt, b[r], b[r + 1], r > 0, r + 1 < world) for r in range(world)]
    for r, inf in enumerate(infos):
        # the neighbours' send counts match our ghost counts
        if r > 0:
            assert infos[r - 1]["send_hi"] == inf["ghosts_lo"]
        if r + 1 < world:
            assert infos[r + 1]["send_lo"] == inf["ghosts_hi"]
        assert inf["box_begin"] <= b[r] - inf["ghosts_lo"]
        assert b[r + 1] + inf["ghosts_hi"] <= inf["box_begin"] + inf["box_points"]
        assert inf["chunks"] == -(-(b[r + 1] - b[r]) // W)
        if n <= 200000:
            # every star neighbour of an owned point is a ghost, and comes
            # from the adjacent rank
            outside = neighbours_outside(shape, b[r], b[r + 1])
            lo = set(range(b[r] - inf["ghosts_lo"], b[r]))
            hi = set(range(b[r + 1], b[r + 1] + inf["ghosts_hi"]))
            assert outside <= lo | hi
            if r > 0:
                assert lo <= set(range(b[r - 1], b[r]))
            if r + 1 < world:
                assert hi <= set(range(b[r + 1], b[r + 2]))


def test_bad_ranges_rejected():
    shape, dt = (20, 30, 40), torch.float32
    with pytest.raises(lopc.LopcError):
        lopc.slab_info(shape, dt, 100, 8192, True, True)  # not chunk aligned
    with pytest.raises(lopc.LopcError):
        lopc.slab_info((20, 100, 100), dt, 4096, 8192, True, True)  # middle range shorter than H = 10101
    with pytest.raises(lopc.LopcError):
        lopc.slab_partition((4, 8, 1000), dt, 16)  # ranges would be shorter than H


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shape, dtname, seed, q):
    try:
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from paper_2603_26968_b200 import dist as ldist

        dt = torch.float32 if dtname == "f32" else torch.float64
        x = random_field(shape, dtname, "smooth", seed)
        eps = eps_noa(x, 1e-2)
        b = lopc.slab_partition(shape, dt, world)
        e0, e1 = b[rank], b[rank + 1]
        inf = lopc.slab_info(shape, dt, e0, e1, rank > 0, rank + 1 < world)
        flat = torch.from_numpy(np.ascontiguousarray(x).reshape(-1).copy())
        # halo exchange pattern of lopc_compress_slab, over gloo
        reqs = []
        recv_lo = torch.empty(inf["ghosts_lo"], dtype=flat.dtype)
        recv_hi = torch.empty(inf["ghosts_hi"], dtype=flat.dtype)
        if inf["send_lo"]:
            reqs.append(dist.isend(flat[e0:e0 + inf["send_lo"]].clone(), rank - 1))
        if inf["send_hi"]:
            reqs.append(dist.isend(flat[e1 - inf["send_hi"]:e1].clone(), rank + 1))
        if inf["ghosts_lo"]:
            reqs.append(dist.irecv(recv_lo, rank - 1))
        if inf["ghosts_hi"]:
            reqs.append(dist.irecv(recv_hi, rank + 1))
        for r in reqs:
            r.wait()
        ok_halo = bool(torch.equal(recv_lo, flat[e0 - inf["ghosts_lo"]:e0]) and
                       torch.equal(recv_hi, flat[e1:e1 + inf["ghosts_hi"]]))
        # distributed assembly: this rank's chunks (oracle chunk encoder on the
        # global least fixpoint), table slice ‖ payload slice, offsets by allgather
        s = oracle.subbins(x, eps)
        W = 16384 // x.itemsize
        c0, c1 = e0 // W, -(-e1 // W)
        table, pay = b"", b""
        for c in range(c0, c1):
            bb, uu = oracle.encode_chunk(x, eps, s, c)
            table += np.array([len(bb), len(uu)], np.uint32).tobytes()
            pay += bb + uu
        sizes = [None] * world
        dist.all_gather_object(sizes, len(pay))
        offs, total = ldist.payload_offsets(-(-x.size // W), sizes)
        header = lopc.write_header(x.shape, dt, eps, total)
        st = ldist.gather_stream(table + pay, header, c1 - c0)
        ok_stream = True
        if rank == 0:
            ok_stream = st == oracle.compress(x, eps)
        q.put((rank, ok_halo, ok_stream, offs[rank]))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e), False, -1))


@pytest.mark.parametrize("shape,dtname", [((24, 40, 50), "f32"), ((400, 120), "f64")])
def test_gloo_world2_halo_and_assembly(shape, dtname):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, shape, dtname, 7, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(60)
    for rank, ok_halo, ok_stream, _ in res:
        assert ok_halo is True, res
        assert ok_stream is True, res
