"""Host logic of the z-slab path (SURVEY 8(b) slab rule, 8(e) bootstrap), on
the CPU: the slab rule exported by the C ABI, and a world_size-2 gloo
process group doing what bench.py / a user does before creating a
multi-rank grid (NCCL unique id from rank 0 broadcast to every rank, each
rank taking its slab of the whole-grid model, timings reduced as the max
over ranks)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pkg():
    from paper_1902_09699_b200 import build as b
    b.build()
    import paper_1902_09699_b200 as p
    return p


@pytest.mark.parametrize("nz", [1, 2, 7, 8, 64, 129, 256, 512])
@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_slab_rule_tiles_the_grid(pkg, nz, G):
    from paper_1902_09699_b200.dist import slab
    if G > nz:
        return
    z = 0
    sizes = []
    for r in range(G):
        z0, n = slab(nz, G, r)
        assert z0 == z                       # contiguous, in rank order
        sizes.append(n)
        z += n
    assert z == nz
    q, m = divmod(nz, G)
    assert sizes == [q + 1] * m + [q] * (G - m)   # the first nz mod G ranks hold one more


def test_slab_rule_rejects_bad_arguments(pkg):
    import ctypes as C
    L = pkg.lib()
    a, b = C.c_int64(), C.c_int64()
    assert L.sip_slab(0, 1, 0, C.byref(a), C.byref(b)) == -1
    assert L.sip_slab(8, 0, 0, C.byref(a), C.byref(b)) == -1
    assert L.sip_slab(8, 2, 2, C.byref(a), C.byref(b)) == -1
    assert L.sip_slab(8, 2, 0, None, C.byref(b)) == -1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1902_09699_b200.dist import comm_desc, local_slab_of, max_over_ranks
        cd = comm_desc()
        m = np.arange(9 * 4 * 8, dtype=np.float64).reshape(9, 4, 8)
        part = local_slab_of(m, cd["nranks"], cd["rank"])
        t = max_over_ranks(1.0 + rank)
        q.put((rank, cd["nranks"], bytes(cd["uid"]), part, t))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_bootstrap(pkg):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda o: o[0])
    (_, w0, uid0, part0, t0), (_, w1, uid1, part1, t1) = out
    assert w0 == w1 == 2
    assert uid0 == uid1 and any(uid0)                 # one NCCL id, from rank 0
    m = np.arange(9 * 4 * 8, dtype=np.float64).reshape(9, 4, 8)
    np.testing.assert_array_equal(np.concatenate([part0, part1]), m)   # slabs tile the grid
    assert part0.shape[0] == 5 and part1.shape[0] == 4
    assert t0 == t1 == 2.0                            # max over ranks
