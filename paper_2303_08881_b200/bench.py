"""One-call pipeline with the reference's timing boundaries (bench.py:72-140 of
the reference): setup_s = partition + classify + orderings + extraction +
factorisation; solve_s is measured inside fgmres."""

from __future__ import annotations

import csv
import io
import json
import time
from dataclasses import dataclass, field

import torch

from .factor import FillRule
from .krylov import KrylovConfig, SolveReport, fgmres
from .ordering import classify_and_order, partition, row_block_owner
from .precond import PRECONDITIONER_NAMES, make_preconditioner
from .problems import ProblemSpec, default_rhs

__all__ = ["RunConfig", "run", "sweep", "to_json", "to_csv", "solve_prepared", "COLUMNS", "REPORT_SCHEMA"]

COLUMNS = ("problem", "n", "p", "precond", "fill", "its", "converged", "setup_s", "solve_s", "final_relres", "error")


@dataclass(frozen=True)
class RunConfig:
    """bench.py:72-105."""

    problem: ProblemSpec
    domains: int = 1
    partition: str = "grid"
    precond: str = "bj"
    fill: FillRule = field(default_factory=lambda: FillRule("ilu0"))
    restart: int = 50
    rtol: float = 1e-8
    max_iters: int = 20000
    inner_iters: int = 3
    history: bool = False
    seed: int = 0

    def __post_init__(self):
        if self.domains < 1:
            raise ValueError("domains must be at least 1")
        if self.partition not in ("grid", "rows"):
            raise ValueError(f"unknown partition shape {self.partition!r}")
        if self.precond not in PRECONDITIONER_NAMES:
            raise ValueError(f"unknown preconditioner {self.precond!r}")
        if self.inner_iters < 1:
            raise ValueError("inner_iters must be at least 1")


def solve_prepared(cfg: RunConfig, a, hint, b):
    """Timed part of `run` for an already built matrix / right-hand side."""
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if cfg.partition == "rows":
        owner = row_block_owner(a.n_rows, cfg.domains)
    else:
        owner = partition(a, cfg.domains, grid_hint=hint)
    layout = classify_and_order(a, owner, cfg.domains)
    m = make_preconditioner(cfg.precond, a, layout, cfg.fill, inner_iters=cfg.inner_iters)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    kcfg = KrylovConfig(restart=cfg.restart, rtol=cfg.rtol, max_iters=cfg.max_iters)
    x, report = fgmres(a, b, m=m.apply if m is not None else None, cfg=kcfg)
    report.setup_seconds = setup_s
    record = {
        "problem": cfg.problem.label(), "n": a.n_rows, "p": cfg.domains, "precond": cfg.precond,
        "fill": str(cfg.fill), "its": report.iterations, "converged": report.converged, "setup_s": setup_s,
        "solve_s": report.solve_seconds, "final_relres": report.final_relres, "error": None,
    }
    if cfg.history:
        record["history"] = [float(v) for v in report.residual_history]
    return record, report, x, m


def run(cfg: RunConfig) -> tuple[dict, SolveReport]:
    """bench.py:108-140."""
    a, hint = cfg.problem.build()
    b = default_rhs(a)
    record, report, _, _ = solve_prepared(cfg, a, hint, b)
    return record, report


# ---------------------------------------------------------------------------
# sweep + serialisation (bench.py:36-69, 143-195 of the reference): plain host code

_RUN_FIELDS = {
    "problem": {"type": "string"}, "n": {"type": ["integer", "null"]}, "p": {"type": "integer", "minimum": 1},
    "precond": {"enum": list(PRECONDITIONER_NAMES)}, "fill": {"type": "string"},
    "its": {"type": ["integer", "null"]}, "converged": {"type": ["boolean", "null"]},
    "setup_s": {"type": ["number", "null"]}, "solve_s": {"type": ["number", "null"]},
    "final_relres": {"type": ["number", "null"]}, "error": {"type": ["string", "null"]},
    "history": {"type": "array", "items": {"type": "number"}},
}
REPORT_SCHEMA = json.dumps({
    "$schema": "https://json-schema.org/draft/2020-12/schema", "title": "benchmark report", "type": "object",
    "required": ["runs"],
    "properties": {"runs": {"type": "array", "items": {
        "type": "object", "required": list(COLUMNS), "properties": _RUN_FIELDS, "additionalProperties": True}}},
}, indent=2) + "\n"


def sweep(cfgs) -> list[dict]:
    """Run every configuration in order; a failing run becomes an error row and the sweep goes on."""
    if not cfgs:
        raise ValueError("sweep needs at least one configuration")
    rows = []
    for cfg in cfgs:
        try:
            rows.append(run(cfg)[0])
        except Exception as exc:
            row = dict.fromkeys(COLUMNS)
            row.update(problem=cfg.problem.label() if cfg.problem is not None else "", p=cfg.domains,
                       precond=cfg.precond, fill=str(cfg.fill), error=f"{type(exc).__name__}: {exc}")
            rows.append(row)
    return rows


def to_json(records) -> str:
    return json.dumps({"runs": records}, indent=2) + "\n"


def to_csv(records) -> str:
    """Fixed columns; booleans as true/false, floats with repr, missing values empty."""
    def cell(v):
        if v is None:
            return ""
        if isinstance(v, bool):
            return "true" if v else "false"
        return repr(v) if isinstance(v, float) else str(v)

    out = io.StringIO()
    w = csv.writer(out, lineterminator="\n")
    w.writerow(COLUMNS)
    w.writerows([cell(rec.get(col)) for col in COLUMNS] for rec in records)
    return out.getvalue()
