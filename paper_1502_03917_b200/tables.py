"""Iteration tables on the GPU.

The reference's table runner (cli.py:35-186: ExperimentSpec, run_table,
the markdown / csv / json renderers) sweeps every (smoother, alpha, level)
cell with the reference solve protocol (Multigrid.solve: zero right-hand
side, seeded random start, stop when the L-norm of the iterate drops by
`tolerance`; multigrid.py:161-204).  Here the same sweep runs every solve on
the device; `gs_mode` picks the NE-GS execution mode (the default,
"wavefront", keeps the reference's sweep order, so the counts are the
reference's).  The defaults are the reference's: levels 5..8 (Poisson) /
4..7 (Stokes), alphas 1, 1e-6, 1e-12, W-cycle, tolerance 1e-6, seed 1234.
Vanka (Stokes) is outside the device scope and is reported as an error
cell, as the reference does for any failing cell.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field

from .multigrid import CycleConfig, Multigrid, assemble_hierarchy
from .smoothers import SmootherKind, check_applicability

DEFAULT_SMOOTHERS = {
    "poisson": ("normal", "lsgs", "slsgs", "cgs"),
    "stokes": ("normal", "lsgs", "slsgs", "vanka"),
}
DEFAULT_LEVELS = {"poisson": (5, 8), "stokes": (4, 7)}
DEFAULT_ALPHAS = (1.0, 1e-6, 1e-12)


@dataclass
class ExperimentSpec:
    """One table run (cli.py:35-75)."""

    problem: str
    smoothers: tuple = ()
    levels: tuple = ()
    alphas: tuple = DEFAULT_ALPHAS
    cycle: str = "w"
    nu: tuple | None = None          # None: 2+2, symmetrized sweep 1+1
    tau: float | None = None
    tolerance: float = 1e-6
    seed: int = 1234
    max_iterations: int = 200
    coarsest_level: int = 1
    fmt: str = "markdown"
    gs_mode: str = "wavefront"

    def __post_init__(self):
        if self.problem not in ("poisson", "stokes"):
            raise ValueError(f"unknown problem '{self.problem}'")
        if not self.smoothers:
            self.smoothers = DEFAULT_SMOOTHERS[self.problem]
        if not self.levels:
            self.levels = DEFAULT_LEVELS[self.problem]
        if not (self.coarsest_level < self.levels[0] <= self.levels[1]):
            raise ValueError("level range must be increasing and above the "
                             "coarsest level")
        if not self.alphas:
            raise ValueError("need at least one regularization parameter")
        if self.fmt not in ("markdown", "csv", "json"):
            raise ValueError(f"unknown format '{self.fmt}'")

    def smoother_nu(self, name):
        if self.nu is not None:
            return self.nu
        return (1, 1) if name == "slsgs" else (2, 2)


@dataclass
class TableCell:
    smoother: str
    alpha: float
    level: int
    iterations: int | None    # None: failed or diverged
    converged: bool
    error: str | None = None

    @property
    def text(self):
        return str(self.iterations) if self.converged else "div"


@dataclass
class TableResult:
    spec: ExperimentSpec
    cells: list = field(default_factory=list)

    def cell(self, smoother, alpha, level):
        for c in self.cells:
            if (c.smoother, c.alpha, c.level) == (smoother, alpha, level):
                return c
        raise KeyError((smoother, alpha, level))


def run_table(spec: ExperimentSpec):
    """Every (alpha, smoother, level) cell, in the reference's loop order
    (cli.py:104-139); a failing cell is recorded and the sweep continues."""
    result = TableResult(spec=spec)
    k_lo, k_hi = spec.levels
    for alpha in spec.alphas:
        systems, transfers = assemble_hierarchy(
            spec.problem, spec.coarsest_level, k_hi, alpha)
        for name in spec.smoothers:
            nu_pre, nu_post = spec.smoother_nu(name)
            for k in range(k_lo, k_hi + 1):
                n_levels = k - spec.coarsest_level + 1
                try:
                    kind = SmootherKind(name, spec.tau)
                    check_applicability(kind, spec.problem)
                    config = CycleConfig(
                        smoother=kind, cycle=spec.cycle, nu_pre=nu_pre,
                        nu_post=nu_post, coarsest_level=spec.coarsest_level,
                        max_iterations=spec.max_iterations,
                        tolerance=spec.tolerance, rng_seed=spec.seed,
                        gs_mode=spec.gs_mode)
                    solver = Multigrid(systems[:n_levels],
                                       transfers[:n_levels - 1], config)
                    report = solver.solve()
                    result.cells.append(TableCell(
                        smoother=name, alpha=alpha, level=k,
                        iterations=report.iterations,
                        converged=report.converged and not report.diverged))
                except Exception as exc:  # keep sibling cells running
                    result.cells.append(TableCell(
                        smoother=name, alpha=alpha, level=k,
                        iterations=None, converged=False, error=str(exc)))
    return result


def render_markdown(result: TableResult):
    spec = result.spec
    lines = [f"# {spec.problem} control: iterations per (smoother, alpha), "
             f"{spec.cycle.upper()}-cycle, tol {spec.tolerance:g}, "
             f"seed {spec.seed}"]
    cols = [(s, a) for s in spec.smoothers for a in spec.alphas]
    lines.append("| level | " + " | ".join(f"{s} a={a:g}" for s, a in cols) + " |")
    lines.append("|" + "---|" * (len(cols) + 1))
    for k in range(spec.levels[0], spec.levels[1] + 1):
        lines.append("".join([f"| {k} "] + [f"| {result.cell(s, a, k).text} "
                                            for s, a in cols]) + "|")
    return "\n".join(lines) + "\n"


def render_csv(result: TableResult):
    lines = ["problem,smoother,alpha,level,iterations,converged"]
    for c in result.cells:
        iters = "" if c.iterations is None else c.iterations
        lines.append(f"{result.spec.problem},{c.smoother},{c.alpha:g},"
                     f"{c.level},{iters},{str(c.converged).lower()}")
    return "\r\n".join(lines) + "\r\n"


def render_json(result: TableResult):
    return json.dumps({
        "problem": result.spec.problem, "cycle": result.spec.cycle,
        "seed": result.spec.seed,
        "cells": [{"smoother": c.smoother, "alpha": c.alpha, "level": c.level,
                   "iterations": c.iterations, "converged": c.converged}
                  for c in result.cells],
    }, indent=2) + "\n"


RENDERERS = {"markdown": render_markdown, "csv": render_csv,
             "json": render_json}


def render_table(result: TableResult):
    return RENDERERS[result.spec.fmt](result)
