"""Campaign artifacts in the reference's schema (
proj/tools/campaign.cpp:76-311): per-problem ``convergence_<solver>_p<i>.csv``,
``metrics.csv``, ``metrics.txt`` and ``manifest.json`` for a problem sequence
solved on the device, plus the one-problem ``distortion_trace.csv``. Same
column sets, number formatting (``%.17g``), status strings, keep-going on a
failed system, and manifest keys (sorted, as nlohmann::json objects are), so
GPU runs line up with the CPU oracle's files side by side.

Solvers: ``gmres-sdr`` (sketching + deflation + recycling), ``sgmres``
(deflation size forced to 0) and ``gmres`` (the classical restarted baseline,
run on the device by :func:`baseline_gmres`)."""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field

from . import (BaselineConfig, ProblemInstance, RecycleSpace, SolverConfig, SolveReport, _check, _lib,
               baseline_gmres, load_recycle_space, save_recycle_space, solve, solve_sequence)

REFERENCE_API_VERSION = "0.1.0"  # version.hpp:9 of the interface mirrored here


def engine_version() -> str:
    v = [C.c_int() for _ in range(3)]
    _check(_lib.sdr_version(*[C.byref(x) for x in v]))
    return "%d.%d.%d" % tuple(x.value for x in v)


def known_solver(name: str) -> bool:  # campaign.cpp:185-187
    return name in ("gmres-sdr", "sgmres", "gmres")


def resolve_out_dir(flag_value: str, fallback: str) -> str:  # campaign.cpp:189-193
    if flag_value:
        return flag_value
    env = os.environ.get("SKRYLOV_OUT_DIR", "")
    return env if env else fallback


def num(v: float) -> str:
    """Shortest round-trip decimal ("%.17g", campaign.cpp:27-31)."""
    return "%.17g" % v


def _json_number(v):
    return v if v == v and v not in (float("inf"), float("-inf")) else None


def _status(rep: SolveReport) -> str:
    return "error" if rep.error else rep.status


@dataclass
class CampaignSpec:  # campaign.hpp:16-25
    name: str
    sequence: list  # ProblemInstance
    solver: str = "gmres-sdr"
    config: SolverConfig = field(default_factory=SolverConfig)
    shared_matrix: bool = False
    problem_seed: int = 0  # recorded only
    out_dir: str = ""
    load_space_path: str = ""
    save_space_path: str = ""


@dataclass
class CampaignOutcome:
    reports: list
    solutions: list
    space: RecycleSpace | None
    files: list


def config_json(cfg: SolverConfig) -> dict:
    return {"m": cfg.m, "t": cfg.t, "k": cfg.k, "s": cfg.s, "tol": cfg.tol, "safety_init": cfg.safety_init,
            "max_restarts": cfg.max_restarts, "variant": cfg.variant, "sketch_seed": cfg.sketch_seed,
            "rank_tol": cfg.rank_tol, "breakdown_tol": cfg.breakdown_tol}


def report_json(index: int, rep: SolveReport) -> dict:
    return {"index": index, "status": _status(rep), "iterations": rep.iterations, "cycles": rep.cycles,
            "matvecs": rep.counters.get("matvecs", 0), "inner_products": rep.counters.get("inner_products", 0),
            "sketch_applies": rep.counters.get("sketch_applies", 0),
            "final_relative_residual": _json_number(rep.final_relative_residual), "seconds": rep.seconds,
            "notes": list(rep.notes), "error": rep.error or None}


def write_convergence_csv(d: str, solver: str, index: int, rep: SolveReport) -> str:
    name = f"convergence_{solver}_p{index}.csv"
    verified = {int(i): v for i, v in rep.true_residuals}
    with open(os.path.join(d, name), "w") as fh:
        fh.write("iteration,sketched_residual,true_residual\n")
        for i, v in rep.sketched_residuals:
            fh.write(f"{int(i)},{num(v)},")
            if int(i) in verified:
                fh.write(num(verified[int(i)]))
            fh.write("\n")
    return name


def write_metrics_csv(d: str, solver: str, reports: list) -> str:
    with open(os.path.join(d, "metrics.csv"), "w") as fh:
        fh.write("problem,solver,status,iterations,cycles,matvecs,inner_products,sketch_applies,"
                 "final_relative_residual,seconds\n")
        for i, r in enumerate(reports):
            c = r.counters
            fh.write(f"{i},{solver},{_status(r)},{r.iterations},{r.cycles},{c.get('matvecs', 0)},"
                     f"{c.get('inner_products', 0)},{c.get('sketch_applies', 0)},"
                     f"{num(r.final_relative_residual)},{num(r.seconds)}\n")
    return "metrics.csv"


def write_metrics_txt(d: str, spec: CampaignSpec, reports: list) -> str:
    tot = {"matvecs": 0, "inner_products": 0, "sketch_applies": 0}
    with open(os.path.join(d, "metrics.txt"), "w") as fh:
        fh.write(f"campaign: {spec.name}\nsolver: {spec.solver}\nproblems: {len(reports)}\n\n")
        fh.write("%-8s %-13s %6s %6s %8s %12s %8s %12s %9s\n" % (
            "problem", "status", "iters", "cycles", "matvecs", "inner_prods", "sketches", "rel_resid", "seconds"))
        for i, r in enumerate(reports):
            for k in tot:
                tot[k] += r.counters.get(k, 0)
            fh.write("%-8d %-13s %6d %6d %8d %12d %8d %12.3e %9.3f\n" % (
                i, _status(r), r.iterations, r.cycles, r.counters.get("matvecs", 0),
                r.counters.get("inner_products", 0), r.counters.get("sketch_applies", 0),
                r.final_relative_residual, r.seconds))
        fh.write("%-8s %-13s %6s %6s %8d %12d %8d\n" % ("total", "", "", "", tot["matvecs"], tot["inner_products"],
                                                         tot["sketch_applies"]))
        for i, r in enumerate(reports):
            for note in r.notes:
                fh.write(f"note (problem {i}): {note}\n")
    return "metrics.txt"


def _versions() -> dict:
    return {"skrylov": REFERENCE_API_VERSION, "engine": f"paper_2311_14206_b200 {engine_version()} (sm_100a)"}


def _write_manifest(d: str, manifest: dict) -> str:
    with open(os.path.join(d, "manifest.json"), "w") as fh:
        fh.write(json.dumps(manifest, indent=2, sort_keys=True) + "\n")
    return "manifest.json"


def _run_baseline_sequence(problems: list, cfg: SolverConfig):  # campaign.cpp:146-181
    reports, sols = [], []
    for i, p in enumerate(problems):
        local = BaselineConfig(m=cfg.m, tol=p.target_tol if p.target_tol > 0.0 else cfg.tol,
                               max_restarts=cfg.max_restarts, breakdown_tol=cfg.breakdown_tol)
        try:
            if p.matrix is None:
                raise ValueError(f"baseline sequence: problem {i} has no matrix")
            res = baseline_gmres(p.matrix, p.rhs, local, x0=p.x0)
            reports.append(res.report)
            sols.append(res.x)
        except Exception as e:  # keep going, as the reference does
            rep = SolveReport(error=str(e))
            rep.notes.append(f"system {i} aborted: {e}")
            reports.append(rep)
            sols.append(None)
    return reports, sols


def run_campaign(spec: CampaignSpec) -> CampaignOutcome:  # campaign.cpp:195-280
    if not known_solver(spec.solver):
        raise ValueError(f"unknown solver '{spec.solver}' (expected gmres-sdr, sgmres or gmres)")
    if not spec.out_dir:
        raise ValueError("campaign needs an output directory")
    cfg = SolverConfig(**{k: getattr(spec.config, k) for k in config_json(spec.config)})
    if spec.solver == "sgmres":
        cfg.k = 0
    cfg.validate()
    os.makedirs(spec.out_dir, exist_ok=True)
    space = None
    if spec.solver == "gmres":
        reports, sols = _run_baseline_sequence(spec.sequence, cfg)
    else:
        initial = load_recycle_space(spec.load_space_path) if spec.load_space_path else None
        res = solve_sequence(spec.sequence, cfg, initial_space=initial, shared_matrix=spec.shared_matrix)
        reports, sols, space = res.reports, res.solutions, res.space
        if spec.save_space_path:
            save_recycle_space(spec.save_space_path, space)
    files = [write_convergence_csv(spec.out_dir, spec.solver, i, r) for i, r in enumerate(reports)]
    files.append(write_metrics_csv(spec.out_dir, spec.solver, reports))
    files.append(write_metrics_txt(spec.out_dir, spec, reports))
    manifest = {"campaign": spec.name, "solver": spec.solver, "problem_seed": spec.problem_seed,
                "problem_count": len(reports), "config": config_json(cfg), "versions": _versions(),
                "statuses": [_status(r) for r in reports],
                "problems": [report_json(i, r) for i, r in enumerate(reports)]}
    if spec.solver != "gmres":
        manifest["recycle"] = {"loaded": spec.load_space_path or None, "saved": spec.save_space_path or None,
                               "final_dim": space.dim(), "final_provenance": space.provenance}
    manifest["files"] = list(files) + ["manifest.json"]
    files.append(_write_manifest(spec.out_dir, manifest))
    return CampaignOutcome(reports, sols, space, [os.path.join(spec.out_dir, f) for f in files])


@dataclass
class TraceSpec:  # campaign.hpp:52-57
    name: str
    problem: ProblemInstance
    config: SolverConfig = field(default_factory=SolverConfig)
    out_dir: str = ""


def run_distortion_trace(spec: TraceSpec) -> list:  # campaign.cpp:282-339
    if spec.problem.matrix is None:
        raise ValueError("distortion trace needs a matrix")
    if not spec.out_dir:
        raise ValueError("distortion trace needs an output directory")
    cfg = SolverConfig(**{k: getattr(spec.config, k) for k in config_json(spec.config)})
    if spec.problem.target_tol > 0.0:
        cfg.tol = spec.problem.target_tol
    cfg.validate()
    os.makedirs(spec.out_dir, exist_ok=True)
    rows = []

    def on_it(ev):
        nb = ev["new_basis_sketch_norm"]
        rows.append({"iteration": ev["iteration"], "inv": 1.0 / nb if nb > 0.0 else 0.0, "sres": ev["sres"],
                     "true": None})

    def on_res(ev):
        if rows and rows[-1]["iteration"] == ev["iteration"]:
            rows[-1]["true"] = ev["true_residual"]

    res = solve(spec.problem.matrix, spec.problem.rhs, cfg, x0=spec.problem.x0,
                callbacks={"on_iteration": on_it, "on_residual_check": on_res})
    with open(os.path.join(spec.out_dir, "distortion_trace.csv"), "w") as fh:
        fh.write("iteration,inverse_basis_sketch_norm,sketched_residual,true_residual,ratio\n")
        for r in rows:
            fh.write(f"{r['iteration']},{num(r['inv'])},{num(r['sres'])},")
            if r["true"] is not None:
                fh.write(f"{num(r['true'])},")
                if r["sres"] > 0.0:
                    fh.write(num(r["true"] / r["sres"]))
            else:
                fh.write(",")
            fh.write("\n")
    manifest = {"campaign": spec.name, "solver": "gmres-sdr", "config": config_json(cfg), "versions": _versions(),
                "statuses": [_status(res.report)], "problems": [report_json(0, res.report)],
                "files": ["distortion_trace.csv", "manifest.json"]}
    _write_manifest(spec.out_dir, manifest)
    return [os.path.join(spec.out_dir, "distortion_trace.csv"), os.path.join(spec.out_dir, "manifest.json")]
