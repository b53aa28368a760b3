"""B200-native GMRES-SDR (sketched GMRES with truncated Arnoldi, deflated
restarting and Krylov-subspace recycling) — Python mirror of the reference
``skrylov`` C++ interface over the C-ABI in ``include/sdr_b200.h``.

Names, argument meaning and error behaviour follow the reference:

=============================  =========================================
reference (proj/include/...)   here
=============================  =========================================
SparseMatrix / OperatorRef     :class:`SparseMatrix` (device SELL-32)
SketchOperator                 :class:`SketchOperator`
SolverConfig                   :class:`SolverConfig`
RecycleSpace                   :class:`RecycleSpace` (U in HBM)
solve(A, b, cfg, space, ...)   :func:`solve`
solve_sequence(seq, cfg, ...)  :func:`solve_sequence`
IncrementalQR                  :class:`IncrementalQR` (host)
harmonic_pairs                 :func:`harmonic_pairs`
gaussian_vector, gen_convdiff  :func:`gaussian_vector`, :func:`gen_convdiff`
=============================  =========================================

``std::invalid_argument`` surfaces as ``ValueError``, ``std::domain_error``
as ``ArithmeticError``, ``std::logic_error``/``std::runtime_error`` as
``RuntimeError``. Every compute call runs the sm_100a kernels in
``_lib/libsdr_b200.so``; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import sdr_config, sdr_baseline_config, sdr_callbacks, ITER_CB, RES_CB

__all__ = [
    "Context", "default_context", "SparseMatrix", "SketchOperator", "SolverConfig", "RecycleSpace", "SolveReport",
    "SolveResult", "SequenceResult", "ProblemInstance", "solve", "solve_sequence",
    "BaselineConfig", "BaselineResult", "baseline_gmres", "read_matrix_market", "write_matrix_market",
    "matrix_market_string", "save_recycle_space", "load_recycle_space", "read_space_file", "space_file_bytes", "IncrementalQR", "harmonic_pairs",
    "gaussian_vector", "gen_convdiff", "gen_convdiff2d", "gen_convdiff3d", "gen_neumann", "neumann_sequence",
    "convdiff_sequence", "sparse_sign_entries", "partition_halo",
    "partition_rows", "SdrError", "CudaError", "torch_host_comm", "DeviceVector",
]

_lib = _capi.load()

STATUS = {0: "converged", 1: "max_restarts", 2: "breakdown", 3: "diverged"}
VARIANT = {"reuse": 0, "exact": 1, "inexact": 2}
PROVENANCE = {0: "empty", 1: "fresh", 2: "reused", 3: "exact-resketch", 4: "inexact-carryover"}
PROVENANCE_ID = {v: k for k, v in PROVENANCE.items()}
PHASES = ("setup", "cycle_init", "step_wait", "host_step", "check", "drain", "basis_cond", "recycle", "qr_append", "ls_solve",
          "recycle_harmonic", "harmonic_svd", "harmonic_schur", "harmonic_rest")


class SdrError(RuntimeError):
    pass


class CudaError(SdrError):
    pass


def _check(rc):
    if rc == 0:
        return
    msg = _lib.sdr_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise ArithmeticError(msg)
    if rc in (5, 6, 7):
        raise CudaError(msg)
    raise SdrError(msg)


def _is_torch_cuda(a):
    return type(a).__module__.startswith("torch") and getattr(a, "is_cuda", False)


def _ptr(a, dtype=np.float64):
    """(keepalive, pointer, length) for a numpy array or a CUDA torch tensor."""
    if a is None:
        return None, None, 0
    if _is_torch_cuda(a):
        import torch
        t = a.contiguous()
        if t.dtype != torch.float64:
            raise ValueError("device vectors must be float64")
        return t, C.c_void_p(t.data_ptr()), t.numel()
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr, arr.ctypes.data_as(C.c_void_p), arr.size


_nccl_preloaded = False


def _preload_nccl():
    """Load the NCCL that PyTorch links (the nvidia-nccl wheel) before the
    library dlopens "libnccl.so.2" by soname, so both share one NCCL. Without
    it a process that creates a distributed context before importing torch
    would bind the system libnccl, and torch's later import fails against it
    (undefined symbol ncclDevCommCreate: the system NCCL is older)."""
    global _nccl_preloaded
    if _nccl_preloaded:
        return
    _nccl_preloaded = True
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        for d in (spec.submodule_search_locations if spec else []):
            path = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(path):
                C.CDLL(path, mode=os.RTLD_NOW | os.RTLD_GLOBAL)
                return
    except (ImportError, OSError, ValueError):
        pass


class Context:
    """One GPU, one CUDA stream, optional NCCL rank (sdr_ctx)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 host_comm: dict | None = None):
        """host_comm: {"allreduce_sum": f(np.ndarray) in place, "allgather_i64": f(np.ndarray) -> np.ndarray
        (world x count), "exchange": f(peer, send np.ndarray, recv np.ndarray)} — the host-staged
        transport (sdr_ctx_create_hostcomm), e.g. :func:`torch_host_comm`."""
        h = C.c_void_p()
        if host_comm is not None:
            self._hc = _host_comm_struct(host_comm)
            _check(_lib.sdr_ctx_create_hostcomm(device, rank, world, C.byref(self._hc[0]), C.byref(h)))
        elif world > 1 or nccl_id is not None:  # world = 1 with an id: one-rank NCCL, distributed code path
            _preload_nccl()
            buf = C.create_string_buffer(bytes(nccl_id), 128)
            _check(_lib.sdr_ctx_create_dist(device, rank, world, buf, C.byref(h)))
        else:
            _check(_lib.sdr_ctx_create(device, C.byref(h)))
        self._h = h
        self.device, self.rank, self.world = device, rank, world

    @staticmethod
    def nccl_unique_id() -> bytes:
        _preload_nccl()
        buf = C.create_string_buffer(128)
        _check(_lib.sdr_nccl_unique_id(buf))
        return buf.raw

    @property
    def num_sms(self):
        n = C.c_int()
        _check(_lib.sdr_ctx_info(self._h, None, None, None, C.byref(n)))
        return n.value

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        _check(_lib.sdr_ctx_stream(self._h, C.byref(s)))
        return s.value or 0

    def synchronize(self):
        _check(_lib.sdr_ctx_synchronize(self._h))

    def set_timing(self, on: bool):
        _check(_lib.sdr_ctx_set_timing(self._h, int(on)))

    def timing_reset(self):
        _check(_lib.sdr_ctx_timing_reset(self._h))

    def timing(self, kernel: str):
        n = C.c_int64()
        ms = C.c_double()
        _check(_lib.sdr_ctx_timing_get(self._h, kernel.encode(), C.byref(n), C.byref(ms)))
        return n.value, ms.value

    @property
    def launches(self) -> int:
        n = C.c_int64()
        _check(_lib.sdr_ctx_launch_count(self._h, C.byref(n)))
        return n.value

    def close(self):
        if getattr(self, "_h", None):
            _lib.sdr_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _host_comm_struct(fns):
    """ctypes callbacks over Python collectives; exceptions become a nonzero
    status (the library raises SDR_ENCCL with a message)."""
    def allreduce(buf, n, user):
        try:
            fns["allreduce_sum"](np.ctypeslib.as_array(buf, shape=(n,)))
            return 0
        except Exception:  # noqa: BLE001
            return 1

    def allgather(inp, count, out, user):
        try:
            got = fns["allgather_i64"](np.ctypeslib.as_array(inp, shape=(count,)).copy())
            flat = np.ascontiguousarray(got, dtype=np.int64).ravel()
            np.ctypeslib.as_array(out, shape=(flat.size,))[:] = flat
            return 0
        except Exception:  # noqa: BLE001
            return 1

    def exchange(peer, send, nsend, recv, nrecv, user):
        try:
            s_arr = np.ctypeslib.as_array(send, shape=(nsend,)).copy() if nsend else np.empty(0)
            r_arr = np.ctypeslib.as_array(recv, shape=(nrecv,)) if nrecv else np.empty(0)
            fns["exchange"](peer, s_arr, r_arr)
            return 0
        except Exception:  # noqa: BLE001
            return 1

    cbs = (_capi.HC_ALLREDUCE(allreduce), _capi.HC_ALLGATHER(allgather), _capi.HC_EXCHANGE(exchange))
    return (_capi.sdr_host_comm(cbs[0], cbs[1], cbs[2], None),) + cbs


def torch_host_comm(group=None):
    """Host collectives over an initialised torch.distributed process group
    (gloo) for Context(host_comm=...). The allreduce gathers every rank's
    values and sums them in rank order, so all ranks hold bitwise-identical
    sums (they must form identical MGS coefficients and restart decisions)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)

    def allreduce_sum(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p
        a[:] = acc.numpy()

    def allgather_i64(a):
        t = torch.from_numpy(a)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
        return torch.stack(parts).numpy()

    def exchange(peer, send, recv):
        reqs = []
        if send.size:
            reqs.append(dist.isend(torch.from_numpy(send), peer, group=group))
        rt = torch.from_numpy(recv) if recv.size else None
        if rt is not None:
            reqs.append(dist.irecv(rt, peer, group=group))
        for r in reqs:
            r.wait()

    return {"allreduce_sum": allreduce_sum, "allgather_i64": allgather_i64, "exchange": exchange}


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("LOCAL_RANK", "0")) if os.environ.get("SDR_DEVICE") is None
                               else int(os.environ["SDR_DEVICE"]))
    return _default_ctx


# --------------------------------------------------------------------- operator

class DeviceVector:
    """A borrowed float64 device vector handed to an operator callback
    (SparseMatrix.from_callable); exposes __cuda_array_interface__, so
    ``torch.as_tensor(v, device="cuda")`` views it without a copy."""

    def __init__(self, ptr, n, readonly):
        self.ptr, self.n, self.readonly = ptr or 0, n, readonly

    @property
    def __cuda_array_interface__(self):
        return {"shape": (self.n,), "typestr": "<f8", "data": (self.ptr, self.readonly), "version": 3,
                "strides": None}

    def tensor(self):
        import torch
        return torch.as_tensor(self, device="cuda")


class SparseMatrix:
    """CSR operator resident on the device (sparse.hpp:27-150 + OperatorRef).

    ``SparseMatrix(rows, cols, offsets, columns, values)`` validates exactly as
    the reference constructor and raises ``ValueError`` with its message.
    """

    def __init__(self, rows, cols, offsets, columns, values, ctx: Context | None = None, *, row_begin=None,
                 local_rows=None, _handle=None):
        self.ctx = ctx or default_context()
        if _handle is not None:
            self._h = _handle
        else:
            o, po, _ = _ptr(np.asarray(offsets, dtype=np.int64), np.int64)
            c_, pc, _ = _ptr(np.asarray(columns, dtype=np.int64), np.int64)
            v, pv, _ = _ptr(np.asarray(values, dtype=np.float64))
            h = C.c_void_p()
            if row_begin is None:
                _check(_lib.sdr_csr_create(self.ctx._h, rows, cols, po, pc, pv, C.byref(h)))
            else:
                _check(_lib.sdr_csr_create_local(self.ctx._h, rows, cols, row_begin, local_rows, po, pc, pv,
                                                 C.byref(h)))
            self._h = h
        vals = [C.c_int64() for _ in range(7)]
        _check(_lib.sdr_csr_info(self._h, *[C.byref(x) for x in vals]))
        (self.rows, self.cols, self.nnz, self.row_begin, self.local_rows, self.halo_lo,
         self.halo_hi) = (x.value for x in vals)
        fmt, dg, st, nb = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int64()
        _check(_lib.sdr_csr_storage(self._h, C.byref(fmt), C.byref(dg), C.byref(st), C.byref(nb)))
        # device storage: "sell" or "dia", diagonals per slice, stored entries, bytes per SpMV
        self.storage = dict(format=("sell", "dia", "zsell", "callable")[fmt.value], diagonals=dg.value, stored=st.value,
                            bytes=nb.value)

    @classmethod
    def from_callable(cls, rows, cols, apply, ctx=None):
        """OperatorRef(rows, cols, Apply) (operator_ref.hpp:22-25): apply(x, y, stream) computes
        y = A x for :class:`DeviceVector` x (cols) and y (rows), enqueued on the CUDA stream
        handle `stream` (e.g. ``torch.cuda.ExternalStream(stream)``) or finished before it
        returns. Non-owning like the reference: keep what apply uses alive."""
        ctx = ctx or default_context()

        def tramp(x, y, stream, user):
            try:
                apply(DeviceVector(x, cols, True), DeviceVector(y, rows, False), stream or 0)
                return 0
            except Exception:  # noqa: BLE001 — reported as SDR_ERUNTIME by the library
                import traceback
                traceback.print_exc()
                return 1

        fn = _capi.APPLY_FN(tramp)
        h = C.c_void_p()
        _check(_lib.sdr_operator_create_callback(ctx._h, rows, cols, fn, None, C.byref(h)))
        obj = cls(0, 0, None, None, None, ctx, _handle=h)
        obj._apply_fn = fn
        return obj

    @classmethod
    def from_complex(cls, rows, cols, offsets, columns, values, ctx=None):
        """Complex fp64 CSR (values complex128): the operator on interleaved
        (re, im) vectors of length 2·rows, stored as ZSELL (BASELINE C4)."""
        ctx = ctx or default_context()
        o = np.ascontiguousarray(offsets, dtype=np.int64)
        c_ = np.ascontiguousarray(columns, dtype=np.int64)
        v = np.ascontiguousarray(values, dtype=np.complex128).view(np.float64)
        h = C.c_void_p()
        _check(_lib.sdr_csr_create_complex(ctx._h, rows, cols, o.ctypes.data_as(C.c_void_p),
                                           c_.ctypes.data_as(C.c_void_p), v.ctypes.data_as(C.c_void_p), C.byref(h)))
        A = cls(0, 0, None, None, None, ctx=ctx, _handle=h)
        A.complex_rows = rows
        return A

    def apply_complex(self, z):
        """y = A z for a complex operator (from_complex) on a complex128 vector."""
        x = np.ascontiguousarray(z, dtype=np.complex128).view(np.float64)
        return self.apply(x).view(np.complex128)

    @classmethod
    def from_matrix_market(cls, path, ctx=None):
        """read_matrix_market_file (matrix_market.hpp:161-165) straight to the device."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(_lib.sdr_csr_read_matrix_market(ctx._h, os.fsencode(path), C.byref(h)))
        return cls(0, 0, None, None, None, ctx=ctx, _handle=h)

    @classmethod
    def from_triplets(cls, rows, cols, r, c, v, ctx=None):
        """Duplicates summed, exact zeros dropped (sparse.hpp:40-73)."""
        r = np.asarray(r, dtype=np.int64)
        c = np.asarray(c, dtype=np.int64)
        v = np.asarray(v, dtype=np.float64)
        bad = (r < 0) | (r >= rows) | (c < 0) | (c >= cols)
        if bad.any():
            i = int(np.argmax(bad))
            raise ValueError(f"SparseMatrix::from_triplets: entry ({r[i]}, {c[i]}) outside {rows}x{cols}")
        order = np.lexsort((c, r))
        r, c, v = r[order], c[order], v[order]
        key = r * max(cols, 1) + c
        uniq, start = np.unique(key, return_index=True)
        sums = np.add.reduceat(v, start) if len(v) else v
        keep = sums != 0.0
        rr, cc, vv = r[start][keep], c[start][keep], sums[keep]
        offsets = np.zeros(rows + 1, dtype=np.int64)
        np.add.at(offsets, rr + 1, 1)
        return cls(rows, cols, np.cumsum(offsets), cc, vv, ctx)

    @classmethod
    def from_dense(cls, A, ctx=None):
        A = np.asarray(A, dtype=np.float64)
        r, c = np.nonzero(A)
        return cls.from_triplets(A.shape[0], A.shape[1], r, c, A[r, c], ctx)

    @classmethod
    def from_scipy(cls, M, ctx=None):
        M = M.tocsr()
        M.sort_indices()
        return cls(M.shape[0], M.shape[1], M.indptr.astype(np.int64), M.indices.astype(np.int64),
                   M.data.astype(np.float64), ctx)

    @classmethod
    def convdiff3d_device(cls, n, bx, by, bz, z_begin=0, z_end=None, ctx=None, ny=None, nz=None):
        """7-point −Δ + β·∇ on an n×ny×nz grid built directly in HBM (no host
        CSR; C5 scale). ny, nz default to n; each rank passes its z-slab."""
        ctx = ctx or default_context()
        ny = n if ny is None else ny
        nz = n if nz is None else nz
        h = C.c_void_p()
        _check(_lib.sdr_csr_create_convdiff3d(ctx._h, n, ny, nz, bx, by, bz, z_begin, nz if z_end is None else z_end,
                                              C.byref(h)))
        return cls(0, 0, None, None, None, ctx, _handle=h)

    def apply(self, x):
        """y = A x (OperatorRef::apply); numpy in -> numpy out, CUDA tensor -> CUDA tensor."""
        keep, px, n = _ptr(x)
        if _is_torch_cuda(x):
            import torch
            y = torch.empty(self.local_rows, dtype=torch.float64, device=x.device)
            py = C.c_void_p(y.data_ptr())
        else:
            y = np.empty(self.local_rows)
            py = y.ctypes.data_as(C.c_void_p)
        _check(_lib.sdr_spmv(self.ctx._h, self._h, px, n, py))
        return y

    __matmul__ = apply

    def apply_batch(self, X):
        """Y = A X for an n x nb block (numpy, column-major copy taken), one
        pass over A per 8 columns (the exact-refresh product)."""
        X = np.asfortranarray(X, dtype=np.float64)
        if X.ndim != 2 or X.shape[0] != self.cols:
            raise ValueError(f"apply_batch: expected {self.cols} x nb block, got {X.shape}")
        Y = np.empty((self.local_rows, X.shape[1]), order="F")
        _check(_lib.sdr_spmm(self.ctx._h, self._h, X.shape[1], X.ctypes.data_as(C.c_void_p), X.shape[0],
                             Y.ctypes.data_as(C.c_void_p), Y.shape[0]))
        return Y

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.sdr_csr_destroy(self._h)
            self._h = None


# ----------------------------------------------------------------------- sketch

class SketchOperator:
    """Randomized embedding S (sketch.hpp:93-193): subsampled DCT, identity,
    or the new sparse-sign map."""

    def __init__(self, handle, ctx):
        self._h = handle
        self.ctx = ctx
        kind = C.c_int()
        n = C.c_int64()
        s = C.c_int64()
        seed = C.c_uint64()
        zeta = C.c_int64()
        _check(_lib.sdr_sketch_info(handle, C.byref(kind), C.byref(n), C.byref(s), C.byref(seed), C.byref(zeta)))
        self.kind = {0: "subsampled_dct", 1: "identity", 2: "sparse_sign"}[kind.value]
        self.input_dim, self.sketch_dim, self.seed, self.zeta = n.value, s.value, seed.value, zeta.value

    @classmethod
    def subsampled_dct(cls, n, s, seed, ctx=None):
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(_lib.sdr_sketch_create_srdct(ctx._h, n, s, seed, C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def identity(cls, n, ctx=None):
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(_lib.sdr_sketch_create_identity(ctx._h, n, C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def sparse_sign(cls, n, s, seed, zeta=8, ctx=None):
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(_lib.sdr_sketch_create_sparse_sign(ctx._h, n, s, seed, zeta, C.byref(h)))
        return cls(h, ctx)

    def rows(self):
        out = np.empty(self.sketch_dim, dtype=np.int64)
        _check(_lib.sdr_sketch_rows(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def signs(self):
        out = np.empty(self.input_dim)
        _check(_lib.sdr_sketch_signs(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def apply(self, x):
        keep, px, n = _ptr(x)
        out = np.empty(self.sketch_dim)
        _check(_lib.sdr_sketch_apply(self.ctx._h, self._h, px, n, out.ctypes.data_as(C.c_void_p)))
        return out

    def dense(self):
        n = self.input_dim
        D = np.empty((self.sketch_dim, n))
        e = np.zeros(n)
        for j in range(n):
            e[j] = 1.0
            D[:, j] = self.apply(e)
            e[j] = 0.0
        return D

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.sdr_sketch_destroy(self._h)
            self._h = None


# ----------------------------------------------------------------- host pieces

def gaussian_vector(n, seed):
    """rng.hpp:87-96, bit-identical (std::mt19937_64 + Box–Muller)."""
    out = np.empty(n)
    _check(_lib.sdr_gaussian_vector(n, seed, out.ctypes.data_as(C.c_void_p)))
    return out


def uniform_stream(seed, n):
    """Rng(seed).uniform() draws (rng.hpp:32), bit-identical."""
    out = np.empty(n)
    _check(_lib.sdr_uniform_stream(n, seed, out.ctypes.data_as(C.c_void_p)))
    return out


def srdct_indices(n, s, seed, with_signs=True):
    """(rows, signs) of SketchOperator::subsampled_dct(n, s, seed), host-side (sketch.hpp:105-122)."""
    rows = np.empty(s, dtype=np.int64)
    signs = np.empty(n) if with_signs else None
    _check(_lib.sdr_srdct_indices(n, s, seed, rows.ctypes.data_as(C.c_void_p),
                                  signs.ctypes.data_as(C.c_void_p) if with_signs else None))
    return rows, signs


def sparse_sign_entries(s, seed, zeta, j0, count):
    rows = np.empty(count * zeta, dtype=np.int64)
    signs = np.empty(count * zeta)
    _check(_lib.sdr_sparse_sign_entries(s, seed, zeta, j0, count, rows.ctypes.data_as(C.c_void_p),
                                        signs.ctypes.data_as(C.c_void_p)))
    return rows.reshape(count, zeta), signs.reshape(count, zeta)


def _gen_csr(fn, *args):
    nnz = C.c_int64()
    _check(fn(*args, C.byref(nnz), None, None, None))
    return nnz.value


def gen_convdiff2d(n, bx, by, shift=0.0, diag_rel=None):
    """(offsets, columns, values) of −Δu + β·∇u on an n×n grid; equals
    −gen_convdiff(n, −β) for bx == by (problems.hpp:70-88)."""
    keep, pd, _ = _ptr(diag_rel)
    nnz = _gen_csr(_lib.sdr_gen_convdiff2d, n, bx, by, shift, pd)
    off = np.empty(n * n + 1, dtype=np.int64)
    col = np.empty(nnz, dtype=np.int64)
    val = np.empty(nnz)
    _check(_lib.sdr_gen_convdiff2d(n, bx, by, shift, pd, None, off.ctypes.data_as(C.c_void_p),
                                   col.ctypes.data_as(C.c_void_p), val.ctypes.data_as(C.c_void_p)))
    return off, col, val


def gen_convdiff(n, alpha):
    """Reference gen_convdiff(n, alpha) (problems.hpp:70-88) = −convdiff2d(n, −alpha, −alpha)."""
    off, col, val = gen_convdiff2d(n, -alpha, -alpha)
    return off, col, -val


def gen_neumann(grid_side, shift):
    """(offsets, columns, values) of gen_neumann (problems.hpp:38-61)."""
    nnz = _gen_csr(_lib.sdr_gen_neumann, grid_side, shift)
    n = grid_side * grid_side
    off = np.empty(n + 1, dtype=np.int64)
    col = np.empty(nnz, dtype=np.int64)
    val = np.empty(nnz)
    _check(_lib.sdr_gen_neumann(grid_side, shift, None, off.ctypes.data_as(C.c_void_p), col.ctypes.data_as(C.c_void_p),
                                val.ctypes.data_as(C.c_void_p)))
    return off, col, val


def neumann_sequence(grid_side, shift, count, seed, tol, ctx=None):
    """problems.hpp:92-107: one operator, rhs i = gaussian_vector(n, seed + i),
    target_tol = tol; solve with solve_sequence(..., shared_matrix=True)."""
    off, col, val = gen_neumann(grid_side, shift)
    n = grid_side * grid_side
    A = SparseMatrix(n, n, off, col, val, ctx=ctx)
    return [ProblemInstance(A, gaussian_vector(n, seed + i), target_tol=tol) for i in range(count)]


def convdiff_sequence(n, alphas, tol, ctx=None):
    """problems.hpp:109-123: one gen_convdiff(n, alpha) system per alpha, all-ones rhs."""
    out = []
    for a in alphas:
        off, col, val = gen_convdiff(n, a)
        out.append(ProblemInstance(SparseMatrix(n * n, n * n, off, col, val, ctx=ctx), np.ones(n * n), target_tol=tol))
    return out


def gen_convdiff3d(n, bx, by, bz, z_begin=0, z_end=None):
    z_end = n if z_end is None else z_end
    nnz = _gen_csr(_lib.sdr_gen_convdiff3d, n, bx, by, bz, z_begin, z_end)
    off = np.empty((z_end - z_begin) * n * n + 1, dtype=np.int64)
    col = np.empty(nnz, dtype=np.int64)
    val = np.empty(nnz)
    _check(_lib.sdr_gen_convdiff3d(n, bx, by, bz, z_begin, z_end, None, off.ctypes.data_as(C.c_void_p),
                                   col.ctypes.data_as(C.c_void_p), val.ctypes.data_as(C.c_void_p)))
    return off, col, val


def partition_rows(rows, world, granule=1):
    rb = np.empty(world, dtype=np.int64)
    re = np.empty(world, dtype=np.int64)
    _check(_lib.sdr_partition_rows(rows, world, granule, rb.ctypes.data_as(C.c_void_p), re.ctypes.data_as(C.c_void_p)))
    return rb, re


def partition_halo(rank, row_begin, row_end, min_col, max_col):
    world = len(row_begin)
    arrs = [np.ascontiguousarray(a, dtype=np.int64) for a in (row_begin, row_end, min_col, max_col)]
    outs = [np.zeros(world, dtype=np.int64) for _ in range(4)]
    _check(_lib.sdr_partition_halo(world, rank, *[a.ctypes.data_as(C.c_void_p) for a in arrs],
                                   *[o.ctypes.data_as(C.c_void_p) for o in outs]))
    return dict(recv_lo=outs[0], recv_cnt=outs[1], send_lo=outs[2], send_cnt=outs[3])


class IncrementalQR:
    """incremental_qr.hpp:26-162 (host, BLAS-2 through OpenBLAS)."""

    def __init__(self, rows, capacity, rank_tol=1e-12):
        h = C.c_void_p()
        _check(_lib.sdr_qr_create(rows, capacity, rank_tol, C.byref(h)))
        self._h = h
        self.rows = rows

    @property
    def cols(self):
        n = C.c_int64()
        _check(_lib.sdr_qr_cols(self._h, C.byref(n)))
        return n.value

    def append(self, col):
        keep, p, n = _ptr(col)
        c = C.c_int64()
        rd = C.c_int()
        _check(_lib.sdr_qr_append(self._h, p, n, C.byref(c), C.byref(rd)))
        return c.value, bool(rd.value)

    def exclude(self, column):
        _check(_lib.sdr_qr_exclude(self._h, column))

    def solve(self, rhs):
        keep, p, n = _ptr(rhs)
        y = np.empty(self.cols)
        res = C.c_double()
        _check(_lib.sdr_qr_solve(self._h, p, n, y.ctypes.data_as(C.c_void_p), C.byref(res)))
        return y, res.value

    def factors(self):
        p = self.cols
        Q = np.empty(self.rows * p)
        R = np.empty(p * p)
        _check(_lib.sdr_qr_factors(self._h, Q.ctypes.data_as(C.c_void_p), R.ctypes.data_as(C.c_void_p)))
        return Q.reshape(p, self.rows).T, R.reshape(p, p).T

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.sdr_qr_destroy(self._h)
            self._h = None


def harmonic_pairs(SAW, SW, k, rank_tol=1e-12, via_qr=False):
    """truncated_svd + fill_pencil + harmonic_pairs (recycle.hpp:98-218).
    via_qr: through the solver's per-cycle QR of SAW (see sdr_harmonic_qr)."""
    SAW = np.asfortranarray(SAW, dtype=np.float64)
    SW = np.asfortranarray(SW, dtype=np.float64)
    s, p = SAW.shape
    rank, keff = C.c_int64(), C.c_int64()
    pe, rl = C.c_int(), C.c_int()
    kk = max(k, 0) + 2
    coeffs = np.zeros(p * kk)
    mre, mim = np.zeros(kk), np.zeros(kk)
    _check(_lib.sdr_harmonic_qr(SAW.ctypes.data_as(C.c_void_p), SW.ctypes.data_as(C.c_void_p), s, p, k, rank_tol,
                             int(via_qr), C.byref(rank), C.byref(keff), C.byref(pe), C.byref(rl),
                             coeffs.ctypes.data_as(C.c_void_p), mre.ctypes.data_as(C.c_void_p),
                             mim.ctypes.data_as(C.c_void_p)))
    ke = keff.value
    return dict(rank=rank.value, k_effective=ke, k_requested=k, pair_extended=bool(pe.value),
                rank_limited=bool(rl.value), coeffs=coeffs[: p * ke].reshape(ke, p).T.copy(),
                mu=mre[:ke] + 1j * mim[:ke])


# ----------------------------------------------------------------------- solver

@dataclass
class SolverConfig:
    """solver.hpp:48-79 (same defaults)."""
    m: int = 100
    t: int = 2
    k: int = 20
    s: int = 0
    tol: float = 1e-6
    safety_init: float = 1.4
    max_restarts: int = 10
    variant: str = "reuse"
    sketch_seed: int = 0x5EED
    rank_tol: float = 1e-12
    breakdown_tol: float = 1e-14

    def c(self):
        return sdr_config(self.m, self.t, self.k, self.s, self.tol, self.safety_init, self.max_restarts,
                          VARIANT[self.variant], self.sketch_seed, self.rank_tol, self.breakdown_tol)

    def validate(self):
        c = self.c()
        _check(_lib.sdr_config_validate(C.byref(c)))


class RecycleSpace:
    """recycle.hpp:31-72: U (n x k) in HBM, SU / SAU (s x k) on the host."""

    def __init__(self, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        _check(_lib.sdr_recycle_create(self.ctx._h, C.byref(h)))
        self._h = h

    def _info(self):
        rows, s, dim = C.c_int64(), C.c_int64(), C.c_int64()
        prov = C.c_int()
        _check(_lib.sdr_recycle_info(self._h, C.byref(rows), C.byref(s), C.byref(dim), C.byref(prov)))
        return rows.value, s.value, dim.value, prov.value

    def dim(self):
        return self._info()[2]

    def empty(self):
        return self.dim() == 0

    @property
    def provenance(self):
        return PROVENANCE[self._info()[3]]

    def get(self):
        rows, s, dim, _ = self._info()
        U = np.empty(rows * dim)
        SU = np.empty(s * dim)
        SAU = np.empty(s * dim)
        _check(_lib.sdr_recycle_get(self.ctx._h, self._h, U.ctypes.data_as(C.c_void_p), SU.ctypes.data_as(C.c_void_p),
                                    SAU.ctypes.data_as(C.c_void_p)))
        return U.reshape(dim, rows).T, SU.reshape(dim, s).T, SAU.reshape(dim, s).T

    @property
    def U(self):
        return self.get()[0]

    @property
    def SU(self):
        return self.get()[1]

    @property
    def SAU(self):
        return self.get()[2]

    def set(self, U, SU, SAU, provenance="fresh"):
        U, SU, SAU = (np.asfortranarray(a, dtype=np.float64) for a in (U, SU, SAU))
        _check(_lib.sdr_recycle_set(self.ctx._h, self._h, U.shape[0], SU.shape[0], U.shape[1],
                                    U.ctypes.data_as(C.c_void_p), SU.ctypes.data_as(C.c_void_p),
                                    SAU.ctypes.data_as(C.c_void_p), PROVENANCE_ID[provenance]))

    def drop_columns(self, cols):
        a = np.ascontiguousarray(cols, dtype=np.int64)
        _check(_lib.sdr_recycle_drop_columns(self._h, a.ctypes.data_as(C.c_void_p), len(a)))

    def refresh(self, A: SparseMatrix, S: SketchOperator, mode="exact"):
        """refresh_for_new_matrix (recycle.hpp:297-318); returns the counters spent."""
        cnt = np.zeros(3, dtype=np.int64)
        _check(_lib.sdr_recycle_refresh(self.ctx._h, self._h, A._h, S._h, 0 if mode == "exact" else 1,
                                        cnt.ctypes.data_as(C.c_void_p)))
        return dict(matvecs=int(cnt[0]), inner_products=int(cnt[1]), sketch_applies=int(cnt[2]))

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.sdr_recycle_destroy(self._h)
            self._h = None


@dataclass
class SolveReport:
    """report.hpp:50-63."""
    status: str = "max_restarts"
    iterations: int = 0
    cycles: int = 0
    rhs_norm: float = 0.0
    final_relative_residual: float = float("nan")
    counters: dict = field(default_factory=dict)
    sketched_residuals: list = field(default_factory=list)
    true_residuals: list = field(default_factory=list)
    cycle_stats: list = field(default_factory=list)
    notes: list = field(default_factory=list)
    error: str = ""
    seconds: float = 0.0
    device_ms: float = 0.0
    host_wait_ms: float = 0.0
    phases: dict = field(default_factory=dict)


def _report(h) -> SolveReport:
    st, cy = C.c_int(), C.c_int32()
    it = C.c_int64()
    rhs, frr, sec = C.c_double(), C.c_double(), C.c_double()
    _check(_lib.sdr_report_summary(h, C.byref(st), C.byref(it), C.byref(cy), C.byref(rhs), C.byref(frr),
                                   C.byref(sec)))
    mv, ip, sk = C.c_int64(), C.c_int64(), C.c_int64()
    _check(_lib.sdr_report_counters(h, C.byref(mv), C.byref(ip), C.byref(sk)))
    samples = []
    for w in (0, 1):
        n = C.c_int64()
        _check(_lib.sdr_report_samples(h, w, C.byref(n), None, None))
        its = np.empty(n.value, dtype=np.int64)
        vals = np.empty(n.value)
        _check(_lib.sdr_report_samples(h, w, C.byref(n), its.ctypes.data_as(C.c_void_p),
                                       vals.ctypes.data_as(C.c_void_p)))
        samples.append(list(zip(its.tolist(), vals.tolist())))
    n = C.c_int64()
    _check(_lib.sdr_report_cycles(h, C.byref(n), None))
    buf = np.empty(8 * max(n.value, 1))
    _check(_lib.sdr_report_cycles(h, C.byref(n), buf.ctypes.data_as(C.c_void_p)))
    cs = [dict(steps=int(buf[8 * i]), entry_residual=buf[8 * i + 1], sketched_entry=buf[8 * i + 2],
               exit_sres=buf[8 * i + 3], exit_residual=buf[8 * i + 4], safety_after=buf[8 * i + 5],
               basis_cond=buf[8 * i + 6], deflation_rank=int(buf[8 * i + 7])) for i in range(n.value)]
    nn = C.c_int64()
    _check(_lib.sdr_report_notes(h, C.byref(nn)))
    notes = [_lib.sdr_report_note(h, i).decode() for i in range(nn.value)]
    phases = {}
    for name in PHASES:
        v = C.c_double()
        _check(_lib.sdr_report_phase(h, name.encode(), C.byref(v)))
        phases[name] = v.value
    dev, wait, tot = C.c_double(), C.c_double(), C.c_double()
    _check(_lib.sdr_report_timing(h, C.byref(dev), C.byref(wait), C.byref(tot)))
    rep = SolveReport(STATUS[st.value], it.value, cy.value, rhs.value, frr.value,
                      dict(matvecs=mv.value, inner_products=ip.value, sketch_applies=sk.value), samples[0],
                      samples[1], cs, notes, (_lib.sdr_report_error(h) or b"").decode(), sec.value, dev.value,
                      wait.value, phases)
    _lib.sdr_report_destroy(h)
    return rep


@dataclass
class SolveResult:
    x: object
    report: SolveReport
    space: RecycleSpace


def _make_callbacks(callbacks):
    if not callbacks:
        return None, None
    on_it = callbacks.get("on_iteration")
    on_res = callbacks.get("on_residual_check")

    def it_cb(ev, user):
        e = ev.contents
        y = np.ctypeslib.as_array(e.y, shape=(e.y_len,)).copy() if e.y_len else np.empty(0)
        on_it(dict(cycle=e.cycle, step=e.step, iteration=e.iteration, sres=e.sres,
                   new_basis_sketch_norm=e.new_basis_sketch_norm, y=y, space_dim=e.space_dim))

    def res_cb(ev, user):
        e = ev.contents
        on_res(dict(cycle=e.cycle, iteration=e.iteration, sres=e.sres, true_residual=e.true_residual))

    fi = ITER_CB(it_cb) if on_it else ITER_CB()
    fr = RES_CB(res_cb) if on_res else RES_CB()
    cb = sdr_callbacks(fi, fr, None)
    return cb, (fi, fr)


def solve(A: SparseMatrix, b, cfg: SolverConfig, space: RecycleSpace | None = None,
          sketch: SketchOperator | None = None, x0=None, callbacks: dict | None = None, out=None) -> SolveResult:
    """solver.hpp:269-365. b / x0: numpy (host) or float64 CUDA tensors (device).
    out: optional destination for x (numpy, e.g. a view of pinned memory, or a
    CUDA tensor) of the rhs length."""
    ctx = A.ctx
    space = space if space is not None else RecycleSpace(ctx)
    kb, pb, nb = _ptr(b)
    if nb != A.local_rows:
        raise ValueError(f"solve: rhs length {nb} does not match operator size {A.local_rows}")
    kx0, px0, nx0 = _ptr(x0)
    if x0 is not None and nx0 != nb:
        raise ValueError(f"solve: x0 length {nx0} does not match rhs length {nb}")
    if out is not None:
        kx, px, nx = _ptr(out)
        if kx is not out:
            raise ValueError("solve: out must be a contiguous float64 array or CUDA tensor")
        if nx != nb:
            raise ValueError(f"solve: out length {nx} does not match rhs length {nb}")
        x = out
    elif _is_torch_cuda(b):
        import torch
        x = torch.empty(nb, dtype=torch.float64, device=b.device)
        px = C.c_void_p(x.data_ptr())
    else:
        x = np.empty(nb)
        px = x.ctypes.data_as(C.c_void_p)
    c = cfg.c()
    cb, keep = _make_callbacks(callbacks)
    rep = C.c_void_p()
    _check(_lib.sdr_solve(ctx._h, A._h, pb, px0, C.byref(c), space._h, sketch._h if sketch else None,
                          C.byref(cb) if cb is not None else None, px, C.byref(rep)))
    return SolveResult(x, _report(rep), space)


# ------------------------------------------------------------------- files
# matrix_market.hpp:83-181 and the SKRYRCY1 recycle-space dump (recycle.hpp:337-390)

def _host_csr(h):
    try:
        r, c, nz = C.c_int64(), C.c_int64(), C.c_int64()
        _check(_lib.sdr_host_csr_info(h, C.byref(r), C.byref(c), C.byref(nz)))
        po, pc, pv = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)(), C.POINTER(C.c_double)()
        _check(_lib.sdr_host_csr_arrays(h, C.byref(po), C.byref(pc), C.byref(pv)))
        off = np.ctypeslib.as_array(po, (r.value + 1,)).copy()
        col = np.ctypeslib.as_array(pc, (nz.value,)).copy() if nz.value else np.zeros(0, np.int64)
        val = np.ctypeslib.as_array(pv, (nz.value,)).copy() if nz.value else np.zeros(0)
        return r.value, c.value, off, col, val
    finally:
        _lib.sdr_host_csr_destroy(h)


def read_matrix_market(path=None, text=None):
    """Parses a Matrix Market file (or string) into CSR arrays
    (rows, cols, offsets, columns, values); errors raise SdrError with the
    reference's message, including the line number."""
    h = C.c_void_p()
    if text is not None:
        t = text.encode() if isinstance(text, str) else bytes(text)
        _check(_lib.sdr_mm_read_string(t, len(t), C.byref(h)))
    else:
        _check(_lib.sdr_mm_read_file(os.fsencode(path), C.byref(h)))
    return _host_csr(h)


def _csr_args(offsets, columns, values):
    o = np.ascontiguousarray(offsets, dtype=np.int64)
    c_ = np.ascontiguousarray(columns, dtype=np.int64)
    v = np.ascontiguousarray(values, dtype=np.float64)
    return (o, c_, v), (o.ctypes.data_as(C.c_void_p), c_.ctypes.data_as(C.c_void_p), v.ctypes.data_as(C.c_void_p))


def write_matrix_market(path, rows, cols, offsets, columns, values):
    keep, ptrs = _csr_args(offsets, columns, values)
    _check(_lib.sdr_mm_write_file(os.fsencode(path), rows, cols, *ptrs))


def matrix_market_string(rows, cols, offsets, columns, values) -> str:
    keep, ptrs = _csr_args(offsets, columns, values)
    n = C.c_int64()
    _check(_lib.sdr_mm_write_string(rows, cols, *ptrs, None, C.byref(n)))
    buf = C.create_string_buffer(n.value)
    _check(_lib.sdr_mm_write_string(rows, cols, *ptrs, buf, C.byref(n)))
    return buf.value.decode()


def read_space_file(path=None, data=None) -> dict:
    """SKRYRCY1 dump -> {n, s, k, provenance, U (n x k), SU, SAU (s x k)}."""
    h = C.c_void_p()
    if data is not None:
        _check(_lib.sdr_space_file_read_bytes(bytes(data), len(data), C.byref(h)))
    else:
        _check(_lib.sdr_space_file_read(os.fsencode(path), C.byref(h)))
    try:
        n, s_, k, prov = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int()
        _check(_lib.sdr_space_file_info(h, C.byref(n), C.byref(s_), C.byref(k), C.byref(prov)))
        pu, psu, psau = (C.POINTER(C.c_double)() for _ in range(3))
        _check(_lib.sdr_space_file_arrays(h, C.byref(pu), C.byref(psu), C.byref(psau)))

        def mat(p, r, c):
            if r * c == 0:
                return np.zeros((r, c), order="F")
            return np.ctypeslib.as_array(p, (r * c,)).copy().reshape((r, c), order="F")
        return dict(n=n.value, s=s_.value, k=k.value, provenance=PROVENANCE[prov.value],
                    U=mat(pu, n.value, k.value), SU=mat(psu, s_.value, k.value), SAU=mat(psau, s_.value, k.value))
    finally:
        _lib.sdr_space_file_destroy(h)


def _space_args(U, SU, SAU):
    U = np.asfortranarray(U, dtype=np.float64)
    SU = np.asfortranarray(SU, dtype=np.float64)
    SAU = np.asfortranarray(SAU, dtype=np.float64)
    return (U, SU, SAU), (U.ctypes.data_as(C.c_void_p), SU.ctypes.data_as(C.c_void_p), SAU.ctypes.data_as(C.c_void_p))


def space_file_bytes(U, SU, SAU, provenance="fresh") -> bytes:
    keep, ptrs = _space_args(U, SU, SAU)
    n, k = keep[0].shape
    s_ = keep[1].shape[0]
    ln = C.c_int64()
    _check(_lib.sdr_space_file_write_bytes(n, s_, k, PROVENANCE_ID[provenance], *ptrs, None, C.byref(ln)))
    buf = C.create_string_buffer(ln.value)
    _check(_lib.sdr_space_file_write_bytes(n, s_, k, PROVENANCE_ID[provenance], *ptrs, buf, C.byref(ln)))
    return buf.raw[:ln.value]


def save_recycle_space(path, space):
    """save_recycle_space_file (recycle.hpp:380-384) of a device space."""
    _check(_lib.sdr_recycle_save_file(space.ctx._h, space._h, os.fsencode(path)))


def load_recycle_space(path, ctx=None):
    """load_recycle_space_file (recycle.hpp:386-390) into a new device space."""
    sp = RecycleSpace(ctx)
    _check(_lib.sdr_recycle_load_file(sp.ctx._h, sp._h, os.fsencode(path)))
    return sp


@dataclass
class BaselineConfig:
    """baseline.hpp:24-39 (same defaults)."""
    m: int = 100
    tol: float = 1e-6
    max_restarts: int = 10
    breakdown_tol: float = 1e-14

    def c(self):
        return sdr_baseline_config(self.m, self.tol, self.max_restarts, self.breakdown_tol)


@dataclass
class BaselineResult:
    """baseline.hpp:41-44."""
    x: object
    report: SolveReport


def baseline_gmres(A: SparseMatrix, b, cfg: BaselineConfig | None = None, x0=None) -> BaselineResult:
    """Classical restarted GMRES on the device (baseline.hpp:51-216): the
    reference's comparison point. b / x0: numpy or float64 CUDA tensors."""
    cfg = cfg or BaselineConfig()
    ctx = A.ctx
    kb, pb, nb = _ptr(b)
    if nb != A.local_rows:
        raise ValueError(f"baseline_gmres: rhs length {nb} does not match operator size {A.local_rows}")
    kx0, px0, nx0 = _ptr(x0)
    if x0 is not None and nx0 != nb:
        raise ValueError(f"baseline_gmres: x0 length {nx0} does not match rhs length {nb}")
    if _is_torch_cuda(b):
        import torch
        x = torch.empty(nb, dtype=torch.float64, device=b.device)
        px = C.c_void_p(x.data_ptr())
    else:
        x = np.empty(nb)
        px = x.ctypes.data_as(C.c_void_p)
    c = cfg.c()
    rep = C.c_void_p()
    _check(_lib.sdr_baseline_gmres(ctx._h, A._h, pb, px0, C.byref(c), px, C.byref(rep)))
    return BaselineResult(x, _report(rep))


@dataclass
class ProblemInstance:
    """problems.hpp:17-22."""
    matrix: SparseMatrix
    rhs: object
    x0: object = None
    target_tol: float = 0.0


@dataclass
class SequenceResult:
    reports: list
    solutions: list
    space: RecycleSpace


def solve_sequence(problems, cfg: SolverConfig, sketch: SketchOperator | None = None,
                   initial_space: RecycleSpace | None = None, shared_matrix: bool = False,
                   outs=None) -> SequenceResult:
    """solver.hpp:385-459 (matrix change detected by object identity).
    outs: optional per-system solution buffers (numpy arrays or CUDA float64
    tensors of the system's length, written in place); default new numpy arrays."""
    n = len(problems)
    if n == 0:
        cfg.validate()
        return SequenceResult([], [], initial_space or RecycleSpace())
    ctx = problems[0].matrix.ctx if problems[0].matrix is not None else default_context()
    space = initial_space if initial_space is not None else RecycleSpace(ctx)
    keep = []
    mats = (C.c_void_p * n)(*[p.matrix._h if p.matrix is not None else None for p in problems])
    rhs = (C.c_void_p * n)()
    x0s = (C.c_void_p * n)()
    xs = []
    xo = (C.c_void_p * n)()
    for i, p in enumerate(problems):
        kb, pb, nb = _ptr(p.rhs)
        keep.append(kb)
        rhs[i] = pb
        if p.x0 is not None:
            k0, p0, _ = _ptr(p.x0)
            keep.append(k0)
            x0s[i] = p0
        if outs is not None:
            if len(outs) != n:
                raise ValueError("solve_sequence: outs needs one buffer per problem")
            ko, po, no = _ptr(outs[i])
            if no != nb or ko is not outs[i]:  # a copy would be written instead of the caller's buffer
                raise ValueError("solve_sequence: outs[%d] must be a contiguous float64 buffer of length %d" % (i, nb))
            xs.append(outs[i])
            xo[i] = po
        else:
            x = np.zeros(nb)
            xs.append(x)
            xo[i] = x.ctypes.data_as(C.c_void_p)
    tols = np.array([p.target_tol for p in problems], dtype=np.float64)
    reps = (C.c_void_p * n)()
    c = cfg.c()
    _check(_lib.sdr_solve_sequence(ctx._h, n, mats, rhs, x0s, tols.ctypes.data_as(C.c_void_p), int(shared_matrix),
                                   C.byref(c), sketch._h if sketch else None, space._h, xo, reps))
    reports = [_report(reps[i]) for i in range(n)]
    sols = [xs[i] if not reports[i].error else np.empty(0) for i in range(n)]
    return SequenceResult(reports, sols, space)
