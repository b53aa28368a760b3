"""BASELINE C4 on the device against complex GMRES-SDR.

The device solves C4 as real GMRES-SDR on the realified system (ZSELL
complex storage, interleaved (re, im) vectors). The oracle
runs complex GMRES-SDR (oracle/skrylov_oracle_complex.hpp: conjugated inner
products, complex least squares, complex-Schur harmonic pencil) on the full
32^3 x 64 lattice — tests/golden/c4_complex_oracle.json. The realified
method must be no worse: same status per system, iterations at most the
complex solver's + 2 %, for the single system and the 10-system sequence
(m0 += 0.01, recycle space carried, exact refresh)."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c4_complex_oracle.json")


def no_worse(got, ref):
    return got <= ref + max(1, 0.02 * ref)


def test_c4_full_lattice_and_sequence_no_worse_than_complex_gmres_sdr(sk, O):
    from tools.c4_problem import c4_complex_csr
    g = json.load(open(GOLD))
    c = g["config"]
    dims = tuple(c["dims"])
    N = int(np.prod(dims))
    gz = sk.gaussian_vector(2 * N, 4)  # (re, im) pairs = the interleaved rhs
    cfg = sk.SolverConfig(m=c["m"], k=c["k"], t=c["t"], s=c["s"], tol=c["tol"], max_restarts=c["max_restarts"],
                          variant="exact")
    S = sk.SketchOperator.subsampled_dct(2 * N, c["s"], cfg.sketch_seed)
    probs = []
    for i in range(len(g["sequence"])):
        off, col, val = c4_complex_csr(dims, m0=-0.8 + 0.01 * i, seed=2, uniform=sk.uniform_stream)
        A = sk.SparseMatrix.from_complex(N, N, off, col, val)
        assert A.storage["format"] == "zsell"
        probs.append(sk.ProblemInstance(A, gz, target_tol=c["tol"]))
    single = sk.solve(probs[0].matrix, gz, cfg, sketch=S)
    ref = g["single"]
    assert single.report.status == ref["status"] == "converged"
    assert no_worse(single.report.iterations, ref["iterations"]), (single.report.iterations, ref["iterations"])
    assert single.report.final_relative_residual < c["tol"]
    seq = sk.solve_sequence(probs, cfg, sketch=S)
    for i, (r, o) in enumerate(zip(seq.reports, g["sequence"])):
        assert r.status == o["status"], i
        assert no_worse(r.iterations, o["iterations"]), (i, r.iterations, o["iterations"])
