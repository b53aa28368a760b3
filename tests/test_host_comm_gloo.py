"""World-size-2 CPU test of the host transport behind Context(host_comm=...)
(sdr_ctx_create_hostcomm, include/sdr_b200.h): torch_host_comm over gloo,
called through the same C-callable trampolines (_host_comm_struct) the
library invokes for its allreduce / allgather / halo exchange.

Checks the semantics the distributed solver relies on:
- allreduce_sum leaves bitwise-identical sums on every rank (rank-ordered);
- allgather_i64 returns the per-rank blocks in rank order;
- exchange swaps unequal halo lengths with a peer, including an empty side;
- a failing collective becomes a nonzero status (the library's SDR_ENCCL)."""
import ctypes as C
import os

import numpy as np

from tests.test_dist_gloo import _free_port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    import paper_2311_14206_b200 as sk

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fns = sk.torch_host_comm()
        st, *_keep = sk._host_comm_struct(fns)
        rng = np.random.default_rng(100 + rank)
        # values whose float sum depends on the order: rank-ordered summation must agree bitwise
        a = rng.standard_normal(37) * 10.0 ** rng.integers(-8, 8, 37)
        mine = a.copy()
        buf = a.copy()
        rc_ar = st.allreduce_sum(buf.ctypes.data_as(C.POINTER(C.c_double)), buf.size, None)

        g_in = np.array([rank, 10 * rank + 1, -rank], dtype=np.int64)
        g_out = np.zeros(3 * world, dtype=np.int64)
        rc_ag = st.allgather_i64(g_in.ctypes.data_as(C.POINTER(C.c_int64)), 3, g_out.ctypes.data_as(C.POINTER(C.c_int64)), None)

        peer = 1 - rank
        nsend = 5 if rank == 0 else 0  # one-sided halo: rank 0 sends 5, rank 1 sends nothing
        send = np.arange(nsend, dtype=np.float64) + 100.0 * (rank + 1)
        nrecv = 0 if rank == 0 else 5
        recv = np.full(max(nrecv, 1), -1.0)
        rc_ex1 = st.exchange(peer, send.ctypes.data_as(C.POINTER(C.c_double)) if nsend else None, nsend,
                             recv.ctypes.data_as(C.POINTER(C.c_double)) if nrecv else None, nrecv, None)
        recv1 = recv[:nrecv].copy()
        # symmetric exchange of unequal lengths (3 from rank 0, 4 from rank 1)
        ns = 3 if rank == 0 else 4
        nr = 4 if rank == 0 else 3
        send2 = rank * 1000.0 + np.arange(ns, dtype=np.float64)
        recv2 = np.zeros(nr)
        rc_ex2 = st.exchange(peer, send2.ctypes.data_as(C.POINTER(C.c_double)), ns,
                             recv2.ctypes.data_as(C.POINTER(C.c_double)), nr, None)

        def boom(_a):
            raise RuntimeError("transport down")

        st_bad, *_keep2 = sk._host_comm_struct(dict(fns, allreduce_sum=boom))
        z = np.zeros(2)
        rc_bad = st_bad.allreduce_sum(z.ctypes.data_as(C.POINTER(C.c_double)), 2, None)
        q.put((rank, mine, buf, g_out, recv1, recv2, (rc_ar, rc_ag, rc_ex1, rc_ex2, rc_bad)))
    finally:
        dist.destroy_process_group()


def test_torch_host_comm_world2_semantics():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, a0, s0, g0, r10, r20, rc0), (_, a1, s1, g1, r11, r21, rc1) = res
    assert rc0[:4] == (0, 0, 0, 0) and rc1[:4] == (0, 0, 0, 0)
    assert rc0[4] != 0 and rc1[4] != 0
    # rank-ordered sum, identical bits on both ranks
    assert s0.tobytes() == s1.tobytes()
    assert s0.tobytes() == (a0 + a1).tobytes()
    assert g0.tolist() == g1.tolist() == [0, 1, 0, 1, 11, -1]
    assert r10.size == 0 and r11.tolist() == [100.0, 101.0, 102.0, 103.0, 104.0]
    assert r20.tolist() == [1000.0, 1001.0, 1002.0, 1003.0]
    assert r21.tolist() == [0.0, 1.0, 2.0]
