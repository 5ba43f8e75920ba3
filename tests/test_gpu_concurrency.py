"""SURVEY §8(b) concurrency contract: "calls on different streams or
workspaces are independent".  Two host threads call the C-ABI at the same
time, each on its own CUDA stream and workspace (device I/O and the pipelined
host-I/O decompress, which uses the library's side streams), on different
fields; every result must equal the oracle's, and each thread's
lopc_last_stats must describe its own call."""
import ctypes as C
import threading

import numpy as np
import pytest

from synth.fields import CONFIGS, eps_noa

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: -m gpu tests must run on a B200")
    import paper_2603_26968_b200 as lopc

    lopc.load()
    return lopc


def test_two_threads_two_streams(ref, gpu):
    import torch

    from paper_2603_26968_b200 import lopc as B

    L = B.load()
    fields = [CONFIGS["cfg2"].generate((24, 120, 100)), CONFIGS["cfg4"].generate((300, 512))]
    cases = []
    for x in fields:
        eps = eps_noa(x, 1e-3)
        cases.append((x, eps, ref.compress(x, eps)))
    results = [[] for _ in cases]
    errors = []
    barrier = threading.Barrier(len(cases))

    def worker(i):
        try:
            x, eps, st_ref = cases[i]
            s = torch.cuda.Stream()
            xt = torch.from_numpy(x).cuda()
            dims = B._dims(x.shape)
            wsb = max(L.lopc_compress_workspace_bytes(x.ndim, dims, B._dtype_code(xt.dtype), 0),
                      L.lopc_decompress_workspace_bytes(len(st_ref) + 64, x.nbytes, 1))
            ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
            cap = B.compress_bound(x.shape, xt.dtype)
            out = torch.empty(cap, dtype=torch.uint8, device="cuda")
            yh = torch.empty(x.shape, dtype=xt.dtype).pin_memory()
            barrier.wait()
            for _ in range(6):
                n = C.c_size_t(cap)
                rc = L.lopc_compress_ex(C.c_void_p(xt.data_ptr()), x.ndim, dims, B._dtype_code(xt.dtype), float(eps),
                                        C.c_void_p(out.data_ptr()), C.byref(n), C.c_void_p(ws.data_ptr()), wsb,
                                        C.c_void_p(s.cuda_stream))
                st = B.Stats()
                L.lopc_last_stats(C.byref(st))
                s.synchronize()
                sb = out[: n.value].cpu().numpy().tobytes()
                sh = torch.from_numpy(np.frombuffer(sb, np.uint8).copy()).pin_memory()
                rc2 = L.lopc_decompress_ex(C.c_void_p(sh.data_ptr()), sh.numel(), C.c_void_p(yh.data_ptr()), x.nbytes,
                                           C.c_void_p(ws.data_ptr()), wsb, C.c_void_p(s.cuda_stream))
                results[i].append((rc, rc2, int(st.n_elems), int(st.total_bytes), sb, yh.numpy().tobytes()))
        except Exception as e:  # reported by the main thread
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(i,)) for i in range(len(cases))]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    assert not errors, errors
    for (x, eps, st_ref), res in zip(cases, results):
        y_ref = ref.decompress(st_ref).tobytes()
        assert len(res) == 6
        for rc, rc2, n_el, tot, sb, yb in res:
            assert rc == 0 and rc2 == 0
            assert n_el == x.size and tot == len(st_ref)  # this thread's own stats
            assert sb == st_ref
            assert yb == y_ref
