"""The benchmark harness around the hot path, mirroring
/root/reference/proj/include/slab/bench.hpp and the JSON schema of report.hpp: the HPCG-mandated
symmetry test on LCG vectors, repeated timed solves on identical inputs, per-level timing shares
(the methodology behind the paper's "MG 80-90 %, RBGS > 50 %" statements) and a report whose JSON
has the reference's keys, so outputs are diffable against `slab bench --format json`.

Everything here is host-side composition of the operator API; all arithmetic runs in the CUDA
library through the C ABI.
"""
from __future__ import annotations

import json
import math
import time
from dataclasses import asdict, dataclass, field
from typing import Callable, List, Optional

from . import _capi as slab

STENCIL_DIAGONAL_VALUE = 26.0  # problem.hpp:45


@dataclass
class BenchConfig:  # report.hpp:46-61
    dims: tuple = (16, 16, 16)
    levels: int = 4
    sweeps: int = 1
    max_iters: int = 500
    rtol: float = 1e-6
    fixed_iterations: Optional[int] = None
    runs: int = 10
    seed: int = 1
    use_preconditioner: bool = True
    threads: int = 0  # kept for schema compatibility; parallelism is the GPU's
    skip_symmetry: bool = False


@dataclass
class SymmetryReport:  # report.hpp:63-75
    skipped: bool = False
    matrix_pass: bool = False
    matrix_diff: float = 0.0
    precond_pass: bool = False
    precond_diff: float = 0.0
    tolerance: float = 0.0

    def all_pass(self) -> bool:
        return self.skipped or (self.matrix_pass and self.precond_pass)


@dataclass
class LevelTimings:  # report.hpp:77-86
    level: int = 0
    n: int = 0
    smoother_seconds: float = 0.0
    transfer_seconds: float = 0.0
    mg_seconds: float = 0.0
    nnz_visited: int = 0


@dataclass
class RunRecord:  # report.hpp:88-98
    run: int = 0
    solve_seconds: float = 0.0
    iterations: int = 0
    final_residual: float = 0.0
    converged: bool = False
    residual_history: List[float] = field(default_factory=list)
    levels: List[LevelTimings] = field(default_factory=list)


@dataclass
class LevelShares:  # report.hpp:100-106
    level: int = 0
    smoother_share: float = 0.0
    transfer_share: float = 0.0


@dataclass
class Aggregate:  # report.hpp:108-115
    mean_solve_seconds: float = 0.0
    mg_share: float = 0.0
    levels: List[LevelShares] = field(default_factory=list)


@dataclass
class Report:  # report.hpp:117-125
    config: BenchConfig = field(default_factory=BenchConfig)
    generation_seconds: float = 0.0
    symmetry: SymmetryReport = field(default_factory=SymmetryReport)
    runs: List[RunRecord] = field(default_factory=list)
    aggregate: Aggregate = field(default_factory=Aggregate)


# ---------------------------------------------------------------- bench.hpp:53-105


def symmetry_tolerance(x: slab.DenseVector, y: slab.DenseVector) -> float:
    """1e-8 * |x| * |y| * 26 * sqrt(n)  (bench.hpp:53-57)"""
    nx = math.sqrt(slab.dot(x, x))
    ny = math.sqrt(slab.dot(y, y))
    return 1e-8 * nx * ny * STENCIL_DIAGONAL_VALUE * math.sqrt(float(x.size()))


def bilinear_asymmetry(apply: Callable[[slab.DenseVector, slab.DenseVector], None], x: slab.DenseVector,
                       y: slab.DenseVector) -> float:
    """|x'(Op y) - y'(Op x)| for out <- Op(in)  (bench.hpp:63-70)"""
    tmp = slab.DenseVector(x.ctx, x.size())
    apply(tmp, y)
    lhs = slab.dot(x, tmp)
    apply(tmp, x)
    rhs = slab.dot(y, tmp)
    return abs(lhs - rhs)


def symmetry_test(hierarchy: slab.ProblemLevel, seed: int,
                  smoother_cfg: slab.SmootherConfig = slab.SmootherConfig()) -> SymmetryReport:
    """bench.hpp:80-105: two LCG vectors from one generator; operator and V-cycle (from a zero
    guess) must act symmetrically on them within the scaled tolerance. Never throws on failure."""
    ctx = hierarchy.ctx
    n = hierarchy.n()
    x, state = ctx.random_vector(n, seed)
    y, _ = ctx.random_vector(n, state)  # the same generator keeps drawing (rng.hpp:59-65)
    out = SymmetryReport()
    out.tolerance = symmetry_tolerance(x, y)
    A = hierarchy.A

    def apply_matrix(result, vec):
        slab.mxv(result, A, vec)

    out.matrix_diff = bilinear_asymmetry(apply_matrix, x, y)
    out.matrix_pass = out.matrix_diff <= out.tolerance

    def apply_precond(result, vec):
        slab.set_all(result, 0.0)
        slab.mg_vcycle(hierarchy, result, vec, smoother_cfg)

    out.precond_diff = bilinear_asymmetry(apply_precond, x, y)
    out.precond_pass = out.precond_diff <= out.tolerance
    return out


# ---------------------------------------------------------------- bench.hpp:107-206


def snapshot_levels(finest: slab.ProblemLevel) -> List[LevelTimings]:
    out, level, index = [], finest, 0
    while level is not None:
        s = level.stats
        out.append(LevelTimings(index, level.n(), s.smoother_ns * 1e-9, s.transfer_ns * 1e-9, s.mg_ns * 1e-9,
                                s.nnz_visited))
        level, index = level.coarser, index + 1
    return out


def aggregate_runs(runs: List[RunRecord], levels: int) -> Aggregate:
    agg = Aggregate()
    if not runs:
        return agg
    total_solve = sum(r.solve_seconds for r in runs)
    agg.mean_solve_seconds = total_solve / len(runs)
    denom = total_solve if total_solve > 0.0 else 1.0
    total_mg = 0.0
    for level in range(levels):
        smoother = sum(r.levels[level].smoother_seconds for r in runs)
        transfer = sum(r.levels[level].transfer_seconds for r in runs)
        total_mg += sum(r.levels[level].mg_seconds for r in runs)
        agg.levels.append(LevelShares(level, smoother / denom, transfer / denom))
    agg.mg_share = total_mg / denom
    return agg


def run_benchmark(ctx: slab.Context, cfg: BenchConfig, profile_levels: bool = True) -> Report:
    """bench.hpp:156-206. With profile_levels the solves run with the LevelStats timers on
    (launch by launch, CUDA events around the reference's sections); without it they replay the
    CUDA graph and only nnz_visited / solve time are reported."""
    if cfg.runs < 1:
        raise slab.InvalidArgument("BenchConfig: runs must be at least 1")
    if cfg.levels < 1:
        raise slab.InvalidArgument("BenchConfig: levels must be at least 1")
    report = Report(config=cfg)
    t0 = time.perf_counter()
    hierarchy = ctx.build_hierarchy(cfg.dims, cfg.levels)
    ctx.sync()
    report.generation_seconds = time.perf_counter() - t0

    smoother_cfg = slab.SmootherConfig(cfg.sweeps)
    if cfg.skip_symmetry:
        report.symmetry.skipped = True
    else:
        report.symmetry = symmetry_test(hierarchy, cfg.seed, smoother_cfg)
        if not report.symmetry.all_pass():
            return report

    b = ctx.build_rhs(cfg.dims)
    x0 = ctx.DenseVector(hierarchy.n(), 0.0)
    x = ctx.DenseVector(hierarchy.n())
    solver_cfg = slab.CGConfig(cfg.max_iters, cfg.rtol, cfg.use_preconditioner, cfg.fixed_iterations)
    ctx.set_profiling(profile_levels)
    try:
        for run in range(cfg.runs):
            hierarchy.reset_stats()
            result = slab.cg_solve(hierarchy, b, x0, solver_cfg, smoother_cfg, out=x)
            record = RunRecord(run=run, solve_seconds=result.solve_ms * 1e-3, iterations=result.iterations,
                               final_residual=result.residual_history[-1], converged=result.converged,
                               residual_history=list(result.residual_history), levels=snapshot_levels(hierarchy))
            report.runs.append(record)
    finally:
        ctx.set_profiling(False)
    report.aggregate = aggregate_runs(report.runs, hierarchy.depth())
    return report


# ---------------------------------------------------------------- report.hpp:128-262 (JSON keys)


def report_to_json(report: Report) -> str:
    c = report.config
    doc = {
        "config": {"nx": c.dims[0], "ny": c.dims[1], "nz": c.dims[2], "levels": c.levels, "sweeps": c.sweeps,
                   "max_iters": c.max_iters, "rtol": c.rtol, "runs": c.runs, "seed": c.seed,
                   "preconditioner": c.use_preconditioner, "threads": c.threads, "skip_symmetry": c.skip_symmetry,
                   "fixed_iterations": c.fixed_iterations},
        "generation_seconds": report.generation_seconds,
        "symmetry": asdict(report.symmetry),
        "runs": [asdict(r) for r in report.runs],
        "aggregate": asdict(report.aggregate),
    }
    return json.dumps(doc, indent=2)


def report_from_json(text: str) -> Report:
    doc = json.loads(text)
    c = doc["config"]
    cfg = BenchConfig((c["nx"], c["ny"], c["nz"]), c["levels"], c["sweeps"], c["max_iters"], c["rtol"],
                      c["fixed_iterations"], c["runs"], c["seed"], c["preconditioner"], c["threads"], c["skip_symmetry"])
    runs = [RunRecord(r["run"], r["solve_seconds"], r["iterations"], r["final_residual"], r["converged"],
                      list(r["residual_history"]), [LevelTimings(**l) for l in r["levels"]]) for r in doc["runs"]]
    agg = Aggregate(doc["aggregate"]["mean_solve_seconds"], doc["aggregate"]["mg_share"],
                    [LevelShares(**l) for l in doc["aggregate"]["levels"]])
    return Report(cfg, doc["generation_seconds"], SymmetryReport(**doc["symmetry"]), runs, agg)


# ---------------------------------------------------------------- report.hpp:270-360 (CSV projection)


@dataclass
class CsvRow:  # report.hpp:273-280; level is None for per-run summary rows
    run: int = 0
    level: Optional[int] = None
    kernel: str = ""
    value: float = 0.0


def report_to_rows(report: Report) -> List[CsvRow]:
    rows: List[CsvRow] = []
    for run in report.runs:
        for lt in run.levels:
            rows.append(CsvRow(run.run, lt.level, "smoother_seconds", lt.smoother_seconds))
            rows.append(CsvRow(run.run, lt.level, "transfer_seconds", lt.transfer_seconds))
            rows.append(CsvRow(run.run, lt.level, "mg_seconds", lt.mg_seconds))
            rows.append(CsvRow(run.run, lt.level, "nnz_visited", float(lt.nnz_visited)))
        rows.append(CsvRow(run.run, None, "solve_seconds", run.solve_seconds))
        rows.append(CsvRow(run.run, None, "iterations", float(run.iterations)))
        rows.append(CsvRow(run.run, None, "final_residual", run.final_residual))
        rows.append(CsvRow(run.run, None, "converged", 1.0 if run.converged else 0.0))
    return rows


def _double_to_string(v: float) -> str:
    """text.hpp:28-33 — std::to_chars: the shortest decimal form that parses back identically."""
    if v == int(v) and abs(v) < 1e15:
        return str(int(v)) if v != 0 or math.copysign(1.0, v) > 0 else "-0"
    text = repr(float(v))
    if "e" in text:  # to_chars prints 1e-05 as 1e-05 too; both forms round-trip
        mant, exp = text.split("e")
        sign = "-" if exp.startswith("-") else "+"
        digits = exp.lstrip("+-").rjust(2, "0")
        return f"{mant}e{sign}{digits}"
    return text


def rows_to_csv(rows: List[CsvRow]) -> str:
    out = ["run,level,kernel,value"]
    for row in rows:
        level = "" if row.level is None else str(row.level)
        out.append(f"{row.run},{level},{row.kernel},{_double_to_string(row.value)}")
    return "\n".join(out) + "\n"


def csv_to_rows(text: str) -> List[CsvRow]:
    lines = text.split("\n")
    if not lines or lines[0] != "run,level,kernel,value":
        raise slab.InvalidArgument("csv_to_rows: missing or unexpected header")
    rows = []
    for line in lines[1:]:
        if not line:
            continue
        fields = line.split(",")
        if len(fields) != 4:
            raise slab.InvalidArgument(f"csv_to_rows: expected 4 fields, got line '{line}'")
        try:
            rows.append(CsvRow(int(fields[0]), None if fields[1] == "" else int(fields[1]), fields[2], float(fields[3])))
        except ValueError as exc:
            raise slab.InvalidArgument(f"csv_to_rows: cannot parse '{line}'") from exc
    return rows


def report_to_csv(report: Report) -> str:
    return rows_to_csv(report_to_rows(report))
