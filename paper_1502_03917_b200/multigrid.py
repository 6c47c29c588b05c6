"""V/W-cycle driver, exact coarse solve and solve loops (multigrid.py:1-225).

The cycle runs on the device: ``Multigrid`` hands its levels, transfers and
coarse factorization to a native hierarchy (csrc/ocmg_capi.cu) whose C++
recursion issues every kernel of a cycle into one CUDA stream, and
``solve_to_tolerance`` replays a captured CUDA graph per cycle.  Python only
orchestrates; no per-level work happens here.
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np
import scipy.linalg

from . import _lib
from ._vec import as_device, back_inplace, device_scalar, zeros
from .assembly import (_Handle, build_poisson_system, build_stokes_system,
                       pressure_mean_projection)
from .smoothers import SmootherKind, SmootherState
from .transfer import system_transfer

MAX_COARSE_DIM = 5000          # multigrid.py:25
DIVERGENCE_FACTOR = 1e6        # multigrid.py:26


@dataclass(frozen=True)
class CycleConfig:
    """Multigrid cycle parameters (multigrid.py:29-52) plus the NE-GS
    execution mode of the device smoother."""

    smoother: SmootherKind
    cycle: str = "w"
    nu_pre: int = 2
    nu_post: int = 2
    coarsest_level: int = 1
    max_iterations: int = 200
    tolerance: float = 1e-6
    rng_seed: int = 1234
    gs_mode: str = "wavefront"

    def __post_init__(self):
        if self.cycle not in ("v", "w"):
            raise ValueError("cycle must be 'v' or 'w'")
        if self.nu_pre + self.nu_post < 1:
            raise ValueError("need at least one smoothing step per cycle")
        if self.tolerance <= 0:
            raise ValueError("tolerance must be positive")
        if self.gs_mode not in _lib.GS_MODES:
            raise ValueError(f"gs_mode must be one of {tuple(_lib.GS_MODES)}")


@dataclass
class SolveReport:
    """multigrid.py:55-64."""

    iterations: int
    norm_history: list
    converged: bool
    wall_time: float
    seed: int | None = None
    diverged: bool = False


class CoarseSolver:
    """Exact coarsest-level solve (multigrid.py:67-102): the pivoted LU is
    factorized once on the host (LAPACK getrf, as the reference) and the
    substitution runs on the device.  Stokes pins the first p and mu dof,
    projects the RHS and re-centres the solution."""

    def __init__(self, system):
        if system.n > MAX_COARSE_DIM:
            raise ValueError(
                f"coarsest system has dimension {system.n} > "
                f"{MAX_COARSE_DIM}; raise coarsest_level")
        self.system = system
        dense = system.to_scipy().toarray()
        p_off = mu_off = n_p = 0
        if system.problem == "stokes":
            p_off = system.layout.offset("pressure")
            mu_off = system.layout.offset("adjoint_pressure")
            n_p = system.layout.counts[1]
            for i in (p_off, mu_off):
                dense[i, :] = 0.0
                dense[:, i] = 0.0
                dense[i, i] = 1.0
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            lu, piv = scipy.linalg.lu_factor(dense)
        if np.any(np.diag(lu) == 0.0):
            raise _lib.SingularMatrixError("exactly singular pivot in LU "
                                           "factorization")
        lu_cm = np.ascontiguousarray(lu.T)     # column-major element order
        piv = np.ascontiguousarray(piv, dtype=np.int64)
        h = _lib.new_handle()
        _lib.call("ocmg_coarse_create",
                  _lib.STOKES if system.problem == "stokes" else _lib.POISSON,
                  system.n, _lib.hptr(lu_cm), _lib.hptr(piv), p_off, mu_off,
                  n_p, ctypes.byref(h))
        self._h = _Handle(h, "ocmg_coarse_destroy")

    @property
    def handle(self):
        return self._h.ptr

    def solve(self, rhs):
        import torch
        bd, was_np = as_device(rhs, self.system.n)
        x = torch.empty_like(bd)
        _lib.call("ocmg_coarse_solve", self.handle, _lib.dptr(bd),
                  _lib.dptr(x), _lib.stream_ptr())
        return x.cpu().numpy() if was_np else x


class _NativeHierarchy:
    def __init__(self, systems, transfers, coarse, config):
        n_levels = len(systems) - 1
        lv = (ctypes.c_void_p * n_levels)(*[s.handle for s in systems[1:]])
        tr = (ctypes.c_void_p * n_levels)(*[t.handle for t in transfers])
        kind = config.smoother
        cfg = _lib.CycleConfigC(
            1 if config.cycle == "w" else 0, config.nu_pre, config.nu_post,
            _lib.SMOOTHER_IDS[kind.name], _lib.GS_MODES[config.gs_mode],
            float(kind.resolved_tau(systems[-1].problem) or 0.0))
        h = _lib.new_handle()
        _lib.call("ocmg_hierarchy_create", n_levels, lv, tr, coarse.handle,
                  ctypes.byref(cfg), ctypes.byref(h))
        self._keep = (systems, transfers, coarse)
        self._h = _Handle(h, "ocmg_hierarchy_destroy")

    @property
    def handle(self):
        return self._h.ptr


class Multigrid:
    """Multigrid over systems[0] (coarsest) .. systems[-1] (finest)
    (multigrid.py:105-159)."""

    def __init__(self, systems, transfers, config: CycleConfig):
        if len(transfers) != len(systems) - 1:
            raise ValueError("need one transfer pair per consecutive "
                             "level pair")
        if systems[0].level != config.coarsest_level:
            raise ValueError("coarsest assembled level does not match the "
                             "configured coarsest_level")
        self.systems = systems
        self.transfers = transfers
        self.config = config
        self.coarse = CoarseSolver(systems[0])
        self.states = [None] + [SmootherState(s, config.smoother,
                                              gs_mode=config.gs_mode)
                                for s in systems[1:]]
        self._native = {}

    @property
    def finest(self):
        return self.systems[-1]

    def native(self, level_index=None):
        """Native hierarchy topped at ``level_index`` (default: finest)."""
        li = len(self.systems) - 1 if level_index is None else level_index
        if li not in self._native:
            self._native[li] = _NativeHierarchy(
                self.systems[:li + 1], self.transfers[:li], self.coarse,
                self.config)
        return self._native[li]

    def cycle(self, level_index, x, rhs):
        """One cycle at hierarchy index ``level_index`` (multigrid.py:
        130-159); mutates and returns x."""
        if level_index == 0:
            return self.coarse.solve(rhs)
        n = self.systems[level_index].n
        xd, xnp = as_device(x, n)
        fd, _ = as_device(rhs, n)
        _lib.call("ocmg_cycle", self.native(level_index).handle,
                  _lib.dptr(xd), _lib.dptr(fd), _lib.stream_ptr())
        back_inplace(xd, x, xnp)
        return x

    def solve(self, x0=None):
        """Reference protocol (multigrid.py:161-204): zero RHS, seeded random
        start, stop when the L-norm of the iterate drops by ``tolerance``."""
        system = self.finest
        seed = self.config.rng_seed
        t0 = time.perf_counter()
        if x0 is None:
            xh = np.random.default_rng(seed).uniform(-1.0, 1.0, system.n)
        else:
            xh = np.array(x0, dtype=np.float64)
        x, _ = as_device(xh, system.n)
        pressure_mean_projection(system, x)
        rhs = zeros(system.n)
        norm0 = system.norm(x)
        history = [norm0]
        if norm0 == 0.0:
            return SolveReport(0, history, True, time.perf_counter() - t0,
                               seed)
        converged = diverged = False
        it = 0
        for _ in range(self.config.max_iterations):
            self.cycle(len(self.systems) - 1, x, rhs)
            pressure_mean_projection(system, x)
            it += 1
            nrm = system.norm(x)
            history.append(nrm)
            if nrm <= self.config.tolerance * norm0:
                converged = True
                break
            if nrm > DIVERGENCE_FACTOR * norm0 or not np.isfinite(nrm):
                diverged = True
                break
        return SolveReport(it, history, converged, time.perf_counter() - t0,
                           seed, diverged)

    def run(self, f=None, tol_kind="rel_residual", **kw):
        """One entry point for the two stopping rules:
        tol_kind="l_norm_iterate" is the reference's own protocol
        (``solve``: zero right-hand side, seeded start, L-norm of the iterate
        against ``config.tolerance``) and returns its SolveReport;
        "rel_residual" is the BASELINE protocol (``solve_to_tolerance``:
        ||f - A x|| / ||f|| against ``tol``) and returns (x, history)."""
        if tol_kind == "l_norm_iterate":
            if f is not None:
                raise ValueError("the l_norm_iterate protocol has a zero right-hand side")
            return self.solve(**kw)
        if tol_kind == "rel_residual":
            if f is None:
                raise ValueError("the rel_residual protocol needs a right-hand side")
            return self.solve_to_tolerance(f, **kw)
        raise ValueError("tol_kind must be 'l_norm_iterate' or 'rel_residual'")

    def solve_to_tolerance(self, f, tol=1e-8, max_cycles=300, x=None,
                           use_graph=True):
        """BASELINE.json protocol: x0 = 0 (or ``x``), repeat
        {cycle; mean projection; rel = ||f-Ax||_2/||f||_2} until rel <= tol.
        Runs entirely on the device (one graph replay + one scalar read per
        cycle).  Returns (x, rel_history).  Like ``solve`` it stops once
        rel exceeds DIVERGENCE_FACTOR times the entering relative residual
        (multigrid.py:26,198-200); ``self.last_diverged`` records it."""
        system = self.finest
        fd, _ = as_device(f, system.n)
        fresh = x is None
        if fresh:
            # a persistent start buffer keeps the captured cycle graph valid
            # across calls (the graph is keyed on the x and f pointers)
            if getattr(self, "_x0", None) is None:
                self._x0 = zeros(system.n)
            x = self._x0
            x.zero_()
        xd, xnp = as_device(x, system.n)
        hist = np.zeros(max_cycles)
        done, div = ctypes.c_int(), ctypes.c_int()
        _lib.call("ocmg_solve_ex", self.native().handle, _lib.dptr(xd),
                  _lib.dptr(fd), float(tol), int(max_cycles),
                  1 if use_graph else 0, float(DIVERGENCE_FACTOR),
                  _lib.hptr(hist), ctypes.byref(done), ctypes.byref(div),
                  _lib.stream_ptr())
        self.last_diverged = bool(div.value)
        back_inplace(xd, x, xnp)
        if fresh:
            x = x.clone()
        return x, hist[:done.value].tolist()


def assemble_hierarchy(problem, k_min, k_max, alpha):
    """Systems coarse to fine and their transfer pairs (multigrid.py:
    207-217)."""
    builders = {"poisson": build_poisson_system,
                "stokes": build_stokes_system}
    if problem not in builders:
        raise ValueError(f"unknown problem '{problem}'")
    if not 0 <= k_min < k_max:
        raise ValueError(f"need 0 <= k_min < k_max, got ({k_min}, {k_max})")
    systems = [builders[problem](k, alpha) for k in range(k_min, k_max + 1)]
    transfers = [system_transfer(c, f)
                 for c, f in zip(systems[:-1], systems[1:])]
    return systems, transfers


def build_solver(problem, k_max, alpha, config: CycleConfig):
    """multigrid.py:220-225."""
    systems, transfers = assemble_hierarchy(problem, config.coarsest_level,
                                            k_max, alpha)
    return Multigrid(systems, transfers, config)


def baseline_rhs(system, seed, add_sine=False):
    """BASELINE.json inputs: y_D / v_D ~ U[-1,1] from
    default_rng(seed) in the reference layout (plus sin(pi x) sin(pi y) for
    config 3); f = (M y_D, 0), formed on the device as the state rows of
    A [y_D, 0] (the adjoint rows are zeroed)."""
    import torch
    rng = np.random.default_rng(seed)
    if system.problem == "poisson":
        nv = system.layout.counts[0]
        yd = rng.uniform(-1.0, 1.0, nv)
        if add_sine:
            x, y = system.mesh.vertex_xy()
            yd = yd + np.sin(np.pi * x) * np.sin(np.pi * y)
        sl = system.layout.slice_of("state")
    else:
        sl = system.layout.slice_of("velocity")
        yd = rng.uniform(-1.0, 1.0, sl.stop - sl.start)
    xd = zeros(system.n)
    xd[sl] = torch.from_numpy(yd).to("cuda")
    f = torch.empty_like(xd)
    _lib.call("ocmg_residual", system.handle, _lib.dptr(xd), None,
              _lib.dptr(f), _lib.stream_ptr())
    f.neg_()
    mask = torch.zeros_like(f)
    mask[sl] = 1.0
    f.mul_(mask)
    return f
