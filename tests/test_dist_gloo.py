"""World-size-2 CPU test of the 1-D row-partitioned (z-slab) Arnoldi path
 with torch.distributed/gloo standing in for NCCL.

Each rank builds its slab with the product's generator (global column
indices), derives its halo plan with the product's sdr_partition_halo,
exchanges halo planes with send/recv, runs the local SpMV in the extended
layout the device kernels use, forms its partial window dots / norms / sketch
rows at GLOBAL row indices (SRDCT and sparse sign), sums them with ONE
allreduce per phase, and forms the MGS coefficients exactly as K1/K2 do
(inverse compact-WY from window dots + Gram entries). The resulting H and SV
must equal the single-process oracle's truncated Arnoldi to 1e-12."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, sketch_kind, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import paper_2311_14206_b200 as sk

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, beta, t, m, s = 8, (100.0, 50.0, 25.0), 2, 6, 40
        N, n2 = n ** 3, n * n
        rb, re = sk.partition_rows(N, world, n2)
        r0, r1 = int(rb[rank]), int(re[rank])
        off, col, val = sk.gen_convdiff3d(n, *beta, z_begin=r0 // n2, z_end=r1 // n2)
        mn, mx = int(col.min()), int(col.max())
        ranges = torch.tensor([r0, r1, mn, mx], dtype=torch.int64)
        allr = [torch.zeros(4, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allr, ranges)
        allr = torch.stack(allr).numpy()
        plan = sk.partition_halo(rank, allr[:, 0], allr[:, 1], allr[:, 2], allr[:, 3])
        ext_begin = min(mn, r0)
        ext_len = max(mx + 1, r1) - ext_begin
        nloc = r1 - r0
        gidx = np.arange(r0, r1)
        if sketch_kind == "srdct":
            rows, signs = sk.srdct_indices(N, s, 0x5EED)
            k = rows[:, None].astype(np.float64)
            alpha = np.where(rows == 0, np.sqrt(1.0 / N), np.sqrt(2.0 / N))[:, None]
            Sloc = np.sqrt(N / s) * alpha * np.cos(np.pi * k * (2 * gidx[None, :] + 1) / (2 * N)) * signs[gidx][None, :]
        else:
            srows, ssigns = sk.sparse_sign_entries(s, 0x5EED, 8, r0, nloc)
            Sloc = np.zeros((s, nloc))
            for l in range(8):
                np.add.at(Sloc, (srows[:, l], np.arange(nloc)), ssigns[:, l] / np.sqrt(8))

        def halo(v_own):
            ext = np.zeros(ext_len)
            ext[r0 - ext_begin:r1 - ext_begin] = v_own
            reqs = []
            for p in range(world):
                if plan["send_cnt"][p]:
                    lo = int(plan["send_lo"][p]) - r0
                    reqs.append(dist.isend(torch.from_numpy(v_own[lo:lo + int(plan["send_cnt"][p])].copy()), p))
            for p in range(world):
                if plan["recv_cnt"][p]:
                    buf = torch.zeros(int(plan["recv_cnt"][p]), dtype=torch.float64)
                    dist.recv(buf, p)
                    lo = int(plan["recv_lo"][p]) - ext_begin
                    ext[lo:lo + len(buf)] = buf.numpy()
            for r in reqs:
                r.wait()
            return ext

        def spmv(v_own):
            ext = halo(v_own)
            y = np.empty(nloc)
            for i in range(nloc):
                a, b = off[i], off[i + 1]
                y[i] = np.dot(val[a:b], ext[col[a:b] - ext_begin])
            return y

        def allreduce(a):
            tt = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
            dist.all_reduce(tt)
            return tt.numpy()

        b = sk.gaussian_vector(N, 1)[r0:r1]
        W = [b.copy()]  # unnormalised basis, v_i = c_i w_i
        red = allreduce(np.concatenate([[b @ b], Sloc @ b]))
        beta0 = np.sqrt(red[0])
        c = [1.0 / beta0]
        gram = {}
        H = np.zeros((m + 1, m))
        SV = np.zeros((s, m + 1))
        SV[:, 0] = red[1:] / beta0
        for j in range(m):
            y = spmv(W[j])
            nwin = min(t, j + 1)
            partial = [y @ y] + [y @ W[j - d] for d in range(nwin)]
            tot = allreduce(np.array(partial))  # one small allreduce (window dots)
            cj = c[j]
            h = np.zeros(nwin)
            for d in range(nwin - 1, -1, -1):
                i = j - d
                acc = cj * c[i] * tot[1 + d]
                for d2 in range(nwin - 1, d, -1):
                    l = j - d2
                    acc -= h[d2] * (c[l] * c[i] * gram[(i, l)])
                h[d] = acc
            w = cj * y
            for d in range(nwin - 1, -1, -1):
                w = w - h[d] * c[j - d] * W[j - d]
            ngram = min(t - 1, j + 1)
            partial = [w @ w] + [w @ W[j + 1 - g] for g in range(1, ngram + 1)] + list(Sloc @ w)
            tot = allreduce(np.array(partial))  # one allreduce: norm, Gram, sketch rows
            hn = np.sqrt(tot[0])
            for g in range(1, ngram + 1):
                gram[(j + 1, j + 1 - g)] = tot[g]
            for d in range(nwin):
                H[j - d, j] = h[d]
            H[j + 1, j] = hn
            W.append(w)
            c.append(1.0 / hn)
            SV[:, j + 1] = tot[1 + ngram:] / hn
        q.put((rank, H, SV, plan["recv_cnt"].tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sketch_kind", ["srdct", "sparse_sign"])
def test_zslab_arnoldi_world2_matches_oracle(O, sketch_kind):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, sketch_kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    results.sort()
    (_, H0, SV0, recv0), (_, H1, SV1, recv1) = results
    assert np.array_equal(H0, H1) and np.array_equal(SV0, SV1)  # replicated host state is identical
    assert recv0 == [0, 64] and recv1 == [64, 0]  # one 8x8 plane each way
    n = 8
    N = n ** 3
    A = O.gen_convdiff3d(n, 100.0, 50.0, 25.0)
    S = (O.SketchOperator.subsampled_dct(N, 40, 0x5EED) if sketch_kind == "srdct"
         else O.SketchOperator.sparse_sign(N, 40, 0x5EED, 8))
    st = O.run_arnoldi(A, O.gaussian_vector(N, 1), S, 2, 6)
    assert np.linalg.norm(H0 - st.H) <= 1e-12 * np.linalg.norm(st.H)
    assert np.linalg.norm(SV0 - st.SV) <= 1e-12 * np.linalg.norm(st.SV)
