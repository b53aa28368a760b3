"""Campaign artifacts in the reference schema, the
cases of proj/tests/test_campaign.cpp run through the device solvers."""
import csv
import json
import os

import pytest

pytestmark = pytest.mark.gpu


def small_config(sk):
    return sk.SolverConfig(m=20, t=2, k=4, s=100, tol=1e-8, max_restarts=10)


def neumann_sequence(sk, O, grid, shift, count, seed, tol):
    """problems.hpp neumann_sequence: one operator, rhs gaussian_vector(n, seed + i)."""
    M = O.gen_neumann(grid, shift)
    off, col, val = M.csr()
    A = sk.SparseMatrix(M.rows, M.cols, off, col, val)
    return [sk.ProblemInstance(A, sk.gaussian_vector(M.rows, seed + i), target_tol=tol) for i in range(count)]


def read_csv(path):
    with open(path) as fh:
        return list(csv.reader(fh))


def test_campaign_writes_complete_artifact_set(sk, O, tmp_path):
    from paper_2311_14206_b200 import campaign as cp
    d = str(tmp_path / "sdr")
    spec = cp.CampaignSpec(name="grid-family", sequence=neumann_sequence(sk, O, 12, 0.1, 2, 42, 1e-8),
                           solver="gmres-sdr", config=small_config(sk), shared_matrix=True, problem_seed=42,
                           out_dir=d)
    out = cp.run_campaign(spec)
    assert len(out.reports) == 2 and all(r.status == "converged" for r in out.reports)
    assert len(out.files) == 5 and all(os.path.exists(f) for f in out.files)
    with open(os.path.join(d, "manifest.json")) as fh:
        man = json.load(fh)
    assert man["solver"] == "gmres-sdr" and man["problem_count"] == 2
    assert man["statuses"] == ["converged", "converged"]
    assert man["config"]["m"] == 20 and man["config"]["k"] == 4
    assert man["recycle"]["final_dim"] >= 4 and man["versions"]["skrylov"]
    assert "metrics.csv" in man["files"]
    conv = read_csv(os.path.join(d, "convergence_gmres-sdr_p0.csv"))
    assert conv[0] == ["iteration", "sketched_residual", "true_residual"]
    assert len(conv) == out.reports[0].iterations + 1
    assert all(conv[r][0] == str(r) for r in range(1, len(conv)))
    assert conv[-1][2] != ""  # the converging step was verified
    met = read_csv(os.path.join(d, "metrics.csv"))
    assert len(met) == 3 and len(met[0]) == 10 and met[1][1] == "gmres-sdr" and met[2][2] == "converged"


def test_solver_names_and_sgmres_drops_deflation(sk, O, tmp_path):
    from paper_2311_14206_b200 import campaign as cp
    assert cp.known_solver("gmres-sdr") and cp.known_solver("sgmres") and cp.known_solver("gmres")
    assert not cp.known_solver("cg")
    d = str(tmp_path / "sg")
    spec = cp.CampaignSpec(name="sketch-only", sequence=neumann_sequence(sk, O, 12, 0.1, 1, 21, 1e-8),
                           solver="sgmres", config=small_config(sk), out_dir=d)
    out = cp.run_campaign(spec)
    assert out.reports[0].status == "converged" and out.space.dim() == 0
    with open(os.path.join(d, "manifest.json")) as fh:
        assert json.load(fh)["config"]["k"] == 0
    spec.solver = "minres"
    with pytest.raises(ValueError):
        cp.run_campaign(spec)
    spec.solver, spec.out_dir = "sgmres", ""
    with pytest.raises(ValueError):
        cp.run_campaign(spec)


def test_baseline_emits_same_artifact_shapes(sk, O, tmp_path):
    from paper_2311_14206_b200 import campaign as cp
    d = str(tmp_path / "base")
    spec = cp.CampaignSpec(name="baseline", sequence=neumann_sequence(sk, O, 12, 0.1, 2, 42, 1e-8), solver="gmres",
                           config=small_config(sk), out_dir=d)
    out = cp.run_campaign(spec)
    assert len(out.reports) == 2 and all(r.status == "converged" for r in out.reports)
    assert os.path.exists(os.path.join(d, "convergence_gmres_p0.csv"))
    assert os.path.exists(os.path.join(d, "convergence_gmres_p1.csv"))
    with open(os.path.join(d, "manifest.json")) as fh:
        man = json.load(fh)
    assert man["solver"] == "gmres" and "recycle" not in man
    assert out.reports[1].iterations >= out.reports[0].iterations - 5


def test_recycle_space_survives_save_and_load(sk, O, tmp_path):
    from paper_2311_14206_b200 import campaign as cp
    space_file = str(tmp_path / "space.bin")
    first = cp.CampaignSpec(name="cold", sequence=neumann_sequence(sk, O, 12, 0.1, 2, 42, 1e-8), solver="gmres-sdr",
                            config=small_config(sk), shared_matrix=True, out_dir=str(tmp_path / "d1"),
                            save_space_path=space_file)
    cold = cp.run_campaign(first)
    assert os.path.exists(space_file)
    second = cp.CampaignSpec(name="warm", sequence=neumann_sequence(sk, O, 12, 0.1, 1, 77, 1e-8), solver="gmres-sdr",
                             config=small_config(sk), out_dir=str(tmp_path / "d2"), load_space_path=space_file)
    warm = cp.run_campaign(second)
    assert warm.reports[0].status == "converged"
    assert warm.reports[0].iterations < cold.reports[0].iterations
    with open(os.path.join(str(tmp_path / "d2"), "manifest.json")) as fh:
        assert json.load(fh)["recycle"]["loaded"] == space_file


def test_distortion_trace_pairs_estimates_with_verified(sk, O, tmp_path):
    from paper_2311_14206_b200 import campaign as cp
    M = O.gen_neumann(10, 0.5)
    off, col, val = M.csr()
    A = sk.SparseMatrix(M.rows, M.cols, off, col, val)
    d = str(tmp_path / "trace")
    spec = cp.TraceSpec(name="trace", problem=sk.ProblemInstance(A, sk.gaussian_vector(M.rows, 3)),
                        config=sk.SolverConfig(m=15, t=2, k=0, s=80, tol=1e-6, max_restarts=10), out_dir=d)
    files = cp.run_distortion_trace(spec)
    assert len(files) == 2 and all(os.path.exists(f) for f in files)
    rows = read_csv(os.path.join(d, "distortion_trace.csv"))
    assert rows[0] == ["iteration", "inverse_basis_sketch_norm", "sketched_residual", "true_residual", "ratio"]
    with open(os.path.join(d, "manifest.json")) as fh:
        man = json.load(fh)
    assert man["statuses"][0] == "converged"
    assert len(rows) == man["problems"][0]["iterations"] + 1
    verified = 0
    for r in range(1, len(rows)):
        assert rows[r][0] == str(r) and float(rows[r][1]) > 0.0 and float(rows[r][2]) >= 0.0
        if rows[r][3] != "":
            verified += 1
            assert 0.5 < float(rows[r][4]) < 2.0
    assert verified >= 1
