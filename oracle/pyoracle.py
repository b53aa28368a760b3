"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes bindings over oracle/_build/liboracle.so, the single-threaded CPU
restatement of the reference `skrylov` library (see skrylov_oracle.hpp for
the file:line map). Imported only by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / --impl reference leg; the product package never
imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

STATUS = {0: "converged", 1: "max_restarts", 2: "breakdown", 3: "diverged"}
VARIANT = {"reuse": 0, "exact": 1, "inexact": 2}
PROVENANCE = {0: "empty", 1: "fresh", 2: "reused", 3: "exact-resketch", 4: "inexact-carryover"}


class OracleError(RuntimeError):
    pass


class orc_config(C.Structure):
    _fields_ = [
        ("m", C.c_int64), ("t", C.c_int64), ("k", C.c_int64), ("s", C.c_int64),
        ("tol", C.c_double), ("safety_init", C.c_double),
        ("max_restarts", C.c_int32), ("variant", C.c_int32),
        ("sketch_seed", C.c_uint64),
        ("rank_tol", C.c_double), ("breakdown_tol", C.c_double),
    ]


ORC_APPLY = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p)


def build():
    subprocess.check_call(["make", "-s", "-C", _HERE])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        vp, i64, u64, f64, i32 = C.c_void_p, C.c_int64, C.c_uint64, C.c_double, C.c_int32
        P = C.POINTER
        sig = {
            "orc_last_error": (C.c_char_p, []),
            "orc_mt_stream": (None, [u64, i64, P(u64)]),
            "orc_gaussian_vector": (None, [i64, u64, P(f64)]),
            "orc_gaussian_stream": (None, [u64, i64, P(f64)]),
            "orc_uniform_stream": (None, [u64, i64, P(f64)]),
            "orc_uniform_below_stream": (C.c_int, [u64, u64, i64, P(u64)]),
            "orc_sign_stream": (None, [u64, i64, P(f64)]),
            "orc_sample_without_replacement": (C.c_int, [i64, i64, u64, P(i64)]),
            "orc_csr_create": (vp, [i64, i64, P(i64), P(i64), P(f64)]),
            "orc_csr_from_triplets": (vp, [i64, i64, i64, P(i64), P(i64), P(f64)]),
            "orc_gen_convdiff": (vp, [i64, f64]),
            "orc_gen_neumann": (vp, [i64, f64]),
            "orc_gen_convdiff2d": (vp, [i64, f64, f64, f64, P(f64)]),
            "orc_gen_convdiff3d": (vp, [i64, f64, f64, f64]),
            "orc_csr_rows": (i64, [vp]), "orc_csr_cols": (i64, [vp]), "orc_csr_nnz": (i64, [vp]),
            "orc_csr_export": (None, [vp, P(i64), P(i64), P(f64)]),
            "orc_csr_apply": (C.c_int, [vp, P(f64), i64, P(f64)]),
            "orc_csr_free": (None, [vp]),
            "orc_sketch_srdct": (vp, [i64, i64, u64, C.c_int]),
            "orc_sketch_identity": (vp, [i64]),
            "orc_sketch_sparse_sign": (vp, [i64, i64, u64, i64]),
            "orc_sketch_apply": (C.c_int, [vp, P(f64), i64, P(f64)]),
            "orc_sketch_dim": (i64, [vp]), "orc_sketch_input_dim": (i64, [vp]),
            "orc_sketch_rows": (None, [vp, P(i64)]),
            "orc_sketch_signs": (None, [vp, P(f64)]),
            "orc_sketch_sparse_entries": (None, [vp, i64, i64, P(i64), P(f64)]),
            "orc_sketch_free": (None, [vp]),
            "orc_krylov_run": (vp, [vp, P(f64), i64, vp, i64, i64, i64, f64]),
            "orc_krylov_info": (None, [vp, P(i64), P(i32), P(f64), P(i64)]),
            "orc_krylov_get": (None, [vp, C.c_int, P(f64)]),
            "orc_krylov_free": (None, [vp]),
            "orc_step_sample": (i64, [vp, P(f64), i64, vp, i64, i64, P(f64), P(f64)]),
            "orc_zcsr_create": (vp, [i64, P(i64), P(i64), P(f64)]), "orc_zcsr_free": (None, [vp]),
            "orc_zcsr_apply": (None, [vp, P(f64), P(f64)]),
            "orc_zspace_create": (vp, []), "orc_zspace_free": (None, [vp]), "orc_zspace_dim": (i64, [vp]),
            "orc_zspace_get": (None, [vp, P(f64), P(f64), P(f64)]),
            "orc_zspace_set": (None, [vp, i64, i64, i64, P(f64), P(f64), P(f64)]),
            "orc_zsolve": (vp, [vp, P(f64), P(orc_config), vp, vp, P(f64)]),
            "orc_zrefresh": (C.c_int, [vp, vp, vp, P(i64)]),
            "orc_solve_callable": (vp, [i64, i64, ORC_APPLY, vp, P(f64), i64, P(orc_config), vp, vp, P(f64)]),
            "orc_harmonic": (C.c_int, [P(f64), P(f64), i64, i64, i64, f64, P(i64), P(i64), P(i32),
                                       P(f64), P(f64), P(f64), P(f64)]),
            "orc_space_create": (vp, []), "orc_space_free": (None, [vp]),
            "orc_space_dim": (i64, [vp]), "orc_space_rows": (i64, [vp]), "orc_space_srows": (i64, [vp]),
            "orc_space_provenance": (C.c_int, [vp]),
            "orc_space_get": (None, [vp, P(f64), P(f64), P(f64)]),
            "orc_space_set": (None, [vp, i64, i64, i64, P(f64), P(f64), P(f64), C.c_int]),
            "orc_solve": (vp, [vp, P(f64), i64, P(orc_config), vp, vp, P(f64), P(f64)]),
            "orc_baseline_gmres": (vp, [vp, P(f64), i64, i64, f64, i32, f64, P(f64), P(f64)]),
            "orc_solve_sequence": (C.c_int, [i32, P(vp), P(P(f64)), P(P(f64)), P(f64), i32, P(orc_config),
                                             vp, vp, P(P(f64)), P(vp)]),
            "orc_report_status": (C.c_int, [vp]), "orc_report_iterations": (i64, [vp]),
            "orc_report_cycles": (i32, [vp]), "orc_report_rhs_norm": (f64, [vp]),
            "orc_report_final_rel": (f64, [vp]), "orc_report_seconds": (f64, [vp]),
            "orc_report_counters": (None, [vp, P(i64)]),
            "orc_report_n_samples": (i64, [vp, C.c_int]),
            "orc_report_samples": (None, [vp, C.c_int, P(i64), P(f64)]),
            "orc_report_n_cycle_stats": (i64, [vp]),
            "orc_report_cycle_stats": (None, [vp, i64, P(f64)]),
            "orc_report_n_notes": (i64, [vp]), "orc_report_note": (C.c_char_p, [vp, i64]),
            "orc_report_error": (C.c_char_p, [vp]), "orc_report_free": (None, [vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _err():
    return lib().orc_last_error().decode()


def _raise(rc):
    if rc == 1:
        raise ValueError(_err())
    if rc == 2:
        raise ArithmeticError(_err())
    if rc == 3:
        raise OracleError("logic: " + _err())
    if rc:
        raise OracleError(_err())


def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(C.POINTER(C.c_double))


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(C.POINTER(C.c_int64))


# ------------------------------------------------------------------- rng

def mt_stream(seed, n):
    out = np.empty(n, dtype=np.uint64)
    lib().orc_mt_stream(seed, n, out.ctypes.data_as(C.POINTER(C.c_uint64)))
    return out


def gaussian_vector(n, seed):
    out = np.empty(n)
    lib().orc_gaussian_vector(n, seed, _f64(out)[1])
    return out


def uniform_stream(seed, n):
    out = np.empty(n)
    lib().orc_uniform_stream(seed, n, _f64(out)[1])
    return out


def uniform_below_stream(seed, bound, n):
    out = np.empty(n, dtype=np.uint64)
    _raise(lib().orc_uniform_below_stream(seed, bound, n, out.ctypes.data_as(C.POINTER(C.c_uint64))))
    return out


def sign_stream(seed, n):
    out = np.empty(n)
    lib().orc_sign_stream(seed, n, _f64(out)[1])
    return out


def sample_without_replacement(n, k, seed):
    out = np.empty(max(k, 0), dtype=np.int64)
    _raise(lib().orc_sample_without_replacement(n, k, seed, _i64(out)[1]))
    return out


# --------------------------------------------------------------- matrices

class SparseMatrix:
    """Oracle CSR (sparse.hpp:27-150)."""

    def __init__(self, handle):
        if not handle:
            raise ValueError(_err())
        self._h = handle

    @classmethod
    def from_csr(cls, rows, cols, offsets, columns, values):
        o, po = _i64(offsets)
        c, pc = _i64(columns)
        v, pv = _f64(values)
        return cls(lib().orc_csr_create(rows, cols, po, pc, pv))

    @classmethod
    def from_triplets(cls, rows, cols, r, c, v):
        r, pr = _i64(r)
        c, pc = _i64(c)
        v, pv = _f64(v)
        return cls(lib().orc_csr_from_triplets(rows, cols, len(r), pr, pc, pv))

    @classmethod
    def from_dense(cls, A):
        A = np.asarray(A, dtype=np.float64)
        r, c = np.nonzero(A)
        return cls.from_triplets(A.shape[0], A.shape[1], r, c, A[r, c])

    @property
    def rows(self):
        return lib().orc_csr_rows(self._h)

    @property
    def cols(self):
        return lib().orc_csr_cols(self._h)

    @property
    def nnz(self):
        return lib().orc_csr_nnz(self._h)

    def csr(self):
        off = np.empty(self.rows + 1, dtype=np.int64)
        col = np.empty(self.nnz, dtype=np.int64)
        val = np.empty(self.nnz)
        lib().orc_csr_export(self._h, _i64(off)[1], _i64(col)[1], _f64(val)[1])
        return off, col, val

    def dense(self):
        off, col, val = self.csr()
        D = np.zeros((self.rows, self.cols))
        for r in range(self.rows):
            D[r, col[off[r]:off[r + 1]]] = val[off[r]:off[r + 1]]
        return D

    def apply(self, x):
        x, px = _f64(x)
        y = np.empty(self.rows)
        _raise(lib().orc_csr_apply(self._h, px, len(x), _f64(y)[1]))
        return y

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_csr_free(self._h)
            self._h = None


def gen_convdiff(n, alpha):
    return SparseMatrix(lib().orc_gen_convdiff(n, alpha))


def gen_neumann(g, shift):
    return SparseMatrix(lib().orc_gen_neumann(g, shift))


def gen_convdiff2d(n, bx, by, shift=0.0, diag_rel=None):
    if diag_rel is None:
        return SparseMatrix(lib().orc_gen_convdiff2d(n, bx, by, shift, None))
    d, pd = _f64(diag_rel)
    return SparseMatrix(lib().orc_gen_convdiff2d(n, bx, by, shift, pd))


def gen_convdiff3d(n, bx, by, bz):
    return SparseMatrix(lib().orc_gen_convdiff3d(n, bx, by, bz))


# ----------------------------------------------------------------- sketch

class SketchOperator:
    """Oracle sketch (sketch.hpp:93-193 plus the new sparse-sign map)."""

    def __init__(self, handle):
        if not handle:
            raise ValueError(_err())
        self._h = handle

    @classmethod
    def subsampled_dct(cls, n, s, seed, backend="automatic"):
        b = {"automatic": 0, "fft": 1, "direct": 2}[backend]
        return cls(lib().orc_sketch_srdct(n, s, seed, b))

    @classmethod
    def identity(cls, n):
        return cls(lib().orc_sketch_identity(n))

    @classmethod
    def sparse_sign(cls, n, s, seed, zeta=8):
        return cls(lib().orc_sketch_sparse_sign(n, s, seed, zeta))

    @property
    def sketch_dim(self):
        return lib().orc_sketch_dim(self._h)

    @property
    def input_dim(self):
        return lib().orc_sketch_input_dim(self._h)

    def rows(self):
        out = np.empty(self.sketch_dim, dtype=np.int64)
        lib().orc_sketch_rows(self._h, _i64(out)[1])
        return out

    def signs(self):
        out = np.empty(self.input_dim)
        lib().orc_sketch_signs(self._h, _f64(out)[1])
        return out

    def sparse_entries(self, j0, count, zeta):
        rows = np.empty(count * zeta, dtype=np.int64)
        signs = np.empty(count * zeta)
        lib().orc_sketch_sparse_entries(self._h, j0, count, _i64(rows)[1], _f64(signs)[1])
        return rows.reshape(count, zeta), signs.reshape(count, zeta)

    def apply(self, x):
        x, px = _f64(x)
        out = np.empty(self.sketch_dim)
        _raise(lib().orc_sketch_apply(self._h, px, len(x), _f64(out)[1]))
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
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_sketch_free(self._h)
            self._h = None


# ---------------------------------------------------------------- arnoldi

@dataclass
class KrylovState:
    V: np.ndarray
    H: np.ndarray
    SV: np.ndarray
    SAV: np.ndarray
    j: int
    breakdown: bool
    r0_norm: float
    counters: tuple


def run_arnoldi(A: SparseMatrix, r0, S: SketchOperator, t, m, steps=None, breakdown_tol=1e-14):
    r0, pr = _f64(r0)
    n = len(r0)
    steps = m if steps is None else steps
    h = lib().orc_krylov_run(A._h, pr, n, S._h, t, m, steps, breakdown_tol)
    if not h:
        msg = _err()
        if "zero initial residual" in msg:
            raise ArithmeticError(msg)
        raise ValueError(msg)
    try:
        j = C.c_int64()
        br = C.c_int32()
        r0n = C.c_double()
        cnt = (C.c_int64 * 3)()
        lib().orc_krylov_info(h, C.byref(j), C.byref(br), C.byref(r0n), cnt)
        s = S.sketch_dim
        shapes = [(n, m + 1), (m + 1, m), (s, m + 1), (s, m)]
        mats = []
        for w, shp in enumerate(shapes):
            a = np.empty(shp[0] * shp[1])
            lib().orc_krylov_get(h, w, _f64(a)[1])
            mats.append(a.reshape(shp[1], shp[0]).T.copy())
        return KrylovState(*mats, j=j.value, breakdown=bool(br.value), r0_norm=r0n.value,
                           counters=tuple(cnt))
    finally:
        lib().orc_krylov_free(h)


def step_sample(A: SparseMatrix, r0, S: SketchOperator, t, steps):
    """init_krylov + `steps` solve_cycle steps (arnoldi_step, QR append, LS
    solve); returns (steps, init seconds, step seconds) — bench.py's CPU
    baseline sample."""
    r0, pr = _f64(r0)
    a, b = C.c_double(), C.c_double()
    done = lib().orc_step_sample(A._h, pr, len(r0), S._h, t, steps, C.byref(a), C.byref(b))
    if done < 0:
        raise ValueError(_err())
    return done, a.value, b.value


def harmonic(SAW, SW, k, rank_tol=1e-12):
    SAW = np.asfortranarray(SAW, dtype=np.float64)
    SW = np.asfortranarray(SW, dtype=np.float64)
    s, p = SAW.shape
    rank = C.c_int64()
    keff = C.c_int64()
    flags = (C.c_int32 * 2)()
    coeffs = np.zeros((k + 2) * p)
    mu_re = np.zeros(k + 2)
    mu_im = np.zeros(k + 2)
    sigma = np.zeros(p)
    P = C.POINTER(C.c_double)
    _raise(lib().orc_harmonic(SAW.ctypes.data_as(P), SW.ctypes.data_as(P), s, p, k, rank_tol,
                              C.byref(rank), C.byref(keff), flags, _f64(coeffs)[1], _f64(mu_re)[1],
                              _f64(mu_im)[1], _f64(sigma)[1]))
    ke = keff.value
    return dict(rank=rank.value, k_effective=ke, pair_extended=bool(flags[0]), rank_limited=bool(flags[1]),
                coeffs=coeffs[: p * ke].reshape(ke, p).T.copy(),
                mu=mu_re[:ke] + 1j * mu_im[:ke], sigma=sigma[: rank.value])


# ------------------------------------------------------------------ solve

@dataclass
class SolverConfig:
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
        return orc_config(self.m, self.t, self.k, self.s, self.tol, self.safety_init, self.max_restarts,
                          VARIANT[self.variant], self.sketch_seed, self.rank_tol, self.breakdown_tol)


@dataclass
class SolveReport:
    status: str
    iterations: int
    cycles: int
    rhs_norm: float
    final_relative_residual: float
    counters: dict
    sketched_residuals: list
    true_residuals: list
    cycle_stats: list
    notes: list
    error: str
    seconds: float


def _report(h) -> SolveReport:
    L = lib()
    cnt = (C.c_int64 * 3)()
    L.orc_report_counters(h, cnt)
    samples = []
    for w in (0, 1):
        n = L.orc_report_n_samples(h, w)
        it = np.empty(n, dtype=np.int64)
        val = np.empty(n)
        if n:
            L.orc_report_samples(h, w, _i64(it)[1], _f64(val)[1])
        samples.append(list(zip(it.tolist(), val.tolist())))
    cs = []
    buf = np.empty(8)
    for i in range(L.orc_report_n_cycle_stats(h)):
        L.orc_report_cycle_stats(h, i, _f64(buf)[1])
        cs.append(dict(steps=int(buf[0]), entry_residual=buf[1], sketched_entry=buf[2], exit_sres=buf[3],
                       exit_residual=buf[4], safety_after=buf[5], basis_cond=buf[6], deflation_rank=int(buf[7])))
    notes = [L.orc_report_note(h, i).decode() for i in range(L.orc_report_n_notes(h))]
    r = SolveReport(STATUS[L.orc_report_status(h)], L.orc_report_iterations(h), L.orc_report_cycles(h),
                    L.orc_report_rhs_norm(h), L.orc_report_final_rel(h),
                    dict(matvecs=cnt[0], inner_products=cnt[1], sketch_applies=cnt[2]),
                    samples[0], samples[1], cs, notes, L.orc_report_error(h).decode(), L.orc_report_seconds(h))
    L.orc_report_free(h)
    return r


class RecycleSpace:
    def __init__(self):
        self._h = lib().orc_space_create()

    @property
    def dim(self):
        return lib().orc_space_dim(self._h)

    @property
    def provenance(self):
        return PROVENANCE[lib().orc_space_provenance(self._h)]

    def get(self):
        n, s, k = lib().orc_space_rows(self._h), lib().orc_space_srows(self._h), self.dim
        U, SU, SAU = np.empty(n * k), np.empty(s * k), np.empty(s * k)
        lib().orc_space_get(self._h, _f64(U)[1], _f64(SU)[1], _f64(SAU)[1])
        return U.reshape(k, n).T, SU.reshape(k, s).T, SAU.reshape(k, s).T

    def set(self, U, SU, SAU, provenance=1):
        U, SU, SAU = (np.asfortranarray(a, dtype=np.float64) for a in (U, SU, SAU))
        P = C.POINTER(C.c_double)
        lib().orc_space_set(self._h, U.shape[0], SU.shape[0], U.shape[1], U.ctypes.data_as(P),
                            SU.ctypes.data_as(P), SAU.ctypes.data_as(P), provenance)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_space_free(self._h)
            self._h = None


def solve(A: SparseMatrix, b, cfg: SolverConfig, space: RecycleSpace | None = None,
          sketch: SketchOperator | None = None, x0=None):
    b, pb = _f64(b)
    x = np.empty(len(b))
    px0 = None
    if x0 is not None:
        x0, px0 = _f64(x0)
    c = cfg.c()
    h = lib().orc_solve(A._h, pb, len(b), C.byref(c), space._h if space else None,
                        sketch._h if sketch else None, px0, _f64(x)[1])
    if not h:
        raise ValueError(_err())
    return x, _report(h)


def solve_callable(rows, cols, apply, b, cfg: SolverConfig, space: RecycleSpace | None = None,
                   sketch: SketchOperator | None = None):
    """solve() on OperatorRef(rows, cols, Apply): apply(x, y) fills the numpy y."""
    def tramp(x, y, user):
        try:
            apply(np.ctypeslib.as_array(x, shape=(cols,)), np.ctypeslib.as_array(y, shape=(rows,)))
            return 0
        except Exception:  # noqa: BLE001
            return 1
    fn = ORC_APPLY(tramp)
    b, pb = _f64(b)
    x = np.empty(len(b))
    c = cfg.c()
    h = lib().orc_solve_callable(rows, cols, fn, None, pb, len(b), C.byref(c), space._h if space else None,
                                 sketch._h if sketch else None, _f64(x)[1])
    if not h:
        raise ValueError(_err())
    return x, _report(h)


class ZSparseMatrix:
    """Complex CSR for the complex GMRES-SDR oracle (skrylov_oracle_complex.hpp)."""

    def __init__(self, n, offsets, columns, values):
        self.n = n
        off, po = _i64(np.asarray(offsets))
        col, pc = _i64(np.asarray(columns))
        v = np.ascontiguousarray(np.asarray(values, dtype=np.complex128)).view(np.float64)
        self._keep = (off, col, v)
        self._h = lib().orc_zcsr_create(n, po, pc, v.ctypes.data_as(C.POINTER(C.c_double)))

    def apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.complex128)
        y = np.empty(self.n, dtype=np.complex128)
        lib().orc_zcsr_apply(self._h, x.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)),
                             y.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)))
        return y

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_zcsr_free(self._h)
            self._h = None


class ZRecycleSpace:
    def __init__(self):
        self._h = lib().orc_zspace_create()

    @property
    def dim(self):
        return lib().orc_zspace_dim(self._h)

    def get(self, n, s):
        k = self.dim
        U = np.empty((k, n), dtype=np.complex128)
        SU = np.empty((k, s), dtype=np.complex128)
        SAU = np.empty((k, s), dtype=np.complex128)
        dp = lambda a: a.view(np.float64).ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
        lib().orc_zspace_set  # noqa: B018
        lib().orc_zspace_get(self._h, dp(U), dp(SU), dp(SAU))
        return U.T, SU.T, SAU.T

    def set(self, U, SU, SAU):
        U, SU, SAU = (np.ascontiguousarray(np.asarray(a, dtype=np.complex128).T) for a in (U, SU, SAU))
        dp = lambda a: a.view(np.float64).ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
        lib().orc_zspace_set(self._h, U.shape[1], SU.shape[1], U.shape[0], dp(U), dp(SU), dp(SAU))

    def refresh(self, A: ZSparseMatrix, S: SketchOperator):
        cnt = np.zeros(3, dtype=np.int64)
        _raise(lib().orc_zrefresh(self._h, A._h, S._h, _i64(cnt)[1]))
        return dict(matvecs=int(cnt[0]), inner_products=int(cnt[1]), sketch_applies=int(cnt[2]))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_zspace_free(self._h)
            self._h = None


def zsolve(A: ZSparseMatrix, b, cfg: SolverConfig, sketch: SketchOperator, space: ZRecycleSpace | None = None):
    """Complex GMRES-SDR (skrylov_oracle_complex.hpp); b complex. Returns (x, report)."""
    b = np.ascontiguousarray(b, dtype=np.complex128)
    x = np.empty_like(b)
    c = cfg.c()
    dp = lambda a: a.view(np.float64).ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    h = lib().orc_zsolve(A._h, dp(b), C.byref(c), space._h if space else None, sketch._h, dp(x))
    if not h:
        raise ValueError(_err())
    return x, _report(h)


def baseline_gmres(A: SparseMatrix, b, m=100, tol=1e-6, max_restarts=10, breakdown_tol=1e-14, x0=None):
    """Classical restarted GMRES (baseline.hpp:51-216)."""
    b, pb = _f64(b)
    x = np.empty(len(b))
    px0 = None
    if x0 is not None:
        x0, px0 = _f64(x0)
    h = lib().orc_baseline_gmres(A._h, pb, len(b), m, tol, max_restarts, breakdown_tol, px0, _f64(x)[1])
    if not h:
        raise ValueError(_err())
    return x, _report(h)


def solve_sequence(mats, rhss, cfg: SolverConfig, tols=None, x0s=None, shared_matrix=False,
                   sketch: SketchOperator | None = None, space: RecycleSpace | None = None):
    n = len(mats)
    P = C.POINTER(C.c_double)
    keep = []
    mat_arr = (C.c_void_p * n)(*[m._h if m is not None else None for m in mats])
    rhs_arr = (P * n)()
    x0_arr = (P * n)()
    xs = []
    x_arr = (P * n)()
    for i in range(n):
        b, pb = _f64(rhss[i])
        keep.append(b)
        rhs_arr[i] = pb
        if x0s is not None and x0s[i] is not None:
            x0, px0 = _f64(x0s[i])
            keep.append(x0)
            x0_arr[i] = px0
        x = np.zeros(len(b))
        xs.append(x)
        x_arr[i] = _f64(x)[1]
    tol_arr, ptol = _f64(np.zeros(n) if tols is None else tols)
    reps = (C.c_void_p * n)()
    c = cfg.c()
    _raise(lib().orc_solve_sequence(n, mat_arr, rhs_arr, x0_arr, ptol, int(shared_matrix), C.byref(c),
                                    sketch._h if sketch else None, space._h if space else None, x_arr, reps))
    return xs, [_report(reps[i]) for i in range(n)]
