"""Normal-equation smoothers on the device (smoothers.py:1-285).

Same names and semantics as the reference: a ``SmootherState`` binds a kind
to one level; ``sweep(x, r)`` mutates the iterate and the maintained
residual in place and accumulates the touched-entry count in ``op_count``.
All five kinds run on the device: the normal-equation family (``normal`` =
NE-Jacobi, ``lsgs`` = NE-GS, ``slsgs``), the collective pair smoother
(``cgs``, Poisson) and the Vanka patch smoother (``vanka``, Stokes; SURVEY.md
§8(f) ranks 1 and 4).

NE-GS runs in one of three modes (``gs_mode``):
  * ``"wavefront"`` -- reference sweep order; on structured Poisson levels
    the fused pipelined kernel, elsewhere the level schedule;
  * ``"reference"`` -- reference order and reference arithmetic
    (level-scheduled, bit-identical to kernels.lsgs_sweep);
  * ``"multicolour"`` -- distance-2 multicolour order (a different
    smoother with its own convergence factor).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _lib
from ._vec import as_device, back_inplace, zeros

SMOOTHER_NAMES = ("normal", "lsgs", "slsgs", "cgs", "vanka")
DEVICE_SMOOTHERS = ("normal", "lsgs", "slsgs", "cgs", "vanka")
GS_MODES = tuple(_lib.GS_MODES)

# damping defaults of the experiment protocol (smoothers.py:25-29)
DEFAULT_TAU = {
    ("normal", "poisson"): 0.4,
    ("normal", "stokes"): 0.35,
    ("vanka", "stokes"): 0.4,
}


@dataclass(frozen=True)
class SmootherKind:
    """Smoother selector plus damping (smoothers.py:32-49)."""

    name: str
    tau: float | None = None

    def __post_init__(self):
        if self.name not in SMOOTHER_NAMES:
            raise ValueError(f"unknown smoother '{self.name}'; choose from "
                             f"{SMOOTHER_NAMES}")
        if self.tau is not None and not 0.0 < self.tau < 2.0:
            raise ValueError("damping parameter must lie in (0, 2)")

    def resolved_tau(self, problem):
        if self.tau is not None:
            return self.tau
        return DEFAULT_TAU.get((self.name, problem))


def check_applicability(kind, problem):
    """smoothers.py:52-60, plus the device scope."""
    if kind.name == "cgs" and problem != "poisson":
        raise ValueError("the collective pair smoother only applies to the "
                         "scalar control problem")
    if kind.name == "vanka" and problem != "stokes":
        raise ValueError("the patch smoother only applies to the velocity "
                         "tracking problem")
    if kind.name not in DEVICE_SMOOTHERS:
        raise NotImplementedError(
            f"smoother '{kind.name}' is outside the B200 hot path "
            "(normal / lsgs / slsgs / cgs / vanka only)")
    if kind.name in ("normal", "vanka") and kind.resolved_tau(problem) is None:
        raise ValueError(f"smoother '{kind.name}' needs a damping parameter")


class SmootherState:
    """Per-level smoother binding (smoothers.py:179-244).  The device level
    already holds what the reference precomputes here (row_scaled, n_diag,
    column mirror, dependency schedule)."""

    def __init__(self, system, kind: SmootherKind, gs_mode="wavefront"):
        check_applicability(kind, system.problem)
        if gs_mode not in GS_MODES:
            raise ValueError(f"gs_mode must be one of {GS_MODES}")
        self.system = system
        self.kind = kind
        self.gs_mode = gs_mode
        self.tau = kind.resolved_tau(system.problem)
        self.op_count = 0
        self._update = None
        self.patches = None
        if kind.name == "vanka":
            # smoothers.py:219-223: patches once per system, shared by the
            # states bound to it
            from . import vanka
            if getattr(system, "_vanka", None) is None:
                system._vanka = vanka.build_vanka_patches(system)
                vanka.attach(system, system._vanka)
            self.patches = system._vanka

    def _scratch(self):
        if self._update is None:
            self._update = zeros(self.system.n)
        return self._update

    def sweep(self, x, r, post=False):
        """One smoothing step of the bound kind (smoothers.py:226-244);
        ``post`` only matters for the patch smoother."""
        name = self.kind.name
        if name == "vanka":
            return vanka_sweep(self, x, r,
                               order="backward" if post else "forward")
        if name == "cgs":
            return cgs_sweep(self, x, r)
        if name == "normal":
            return normal_equation_sweep(self, x, r)
        if name == "lsgs":
            return lsgs_sweep(self, x, r)
        return slsgs_sweep(self, x, r)


def make_smoother(system, kind, tau=None, gs_mode="wavefront"):
    """smoothers.py:247-253."""
    if isinstance(kind, str):
        kind = SmootherKind(name=kind, tau=tau)
    elif tau is not None:
        kind = SmootherKind(name=kind.name, tau=tau)
    return SmootherState(system, kind, gs_mode=gs_mode)


def _pair(state, x, r):
    n = state.system.n
    xd, xnp = as_device(x, n)
    rd, rnp = as_device(r, n)
    return xd, xnp, rd, rnp


def normal_equation_sweep(state, x, r):
    """Damped Richardson step on the weighted normal equations
    (smoothers.py:256-267 -> kernels.py:17-39)."""
    xd, xnp, rd, rnp = _pair(state, x, r)
    ops = ctypes.c_int64()
    _lib.call("ocmg_ne_jacobi_sweep", state.system.handle, float(state.tau),
              _lib.dptr(xd), _lib.dptr(rd), _lib.dptr(state._scratch()),
              _lib.stream_ptr(), ctypes.byref(ops))
    state.op_count += ops.value
    back_inplace(xd, x, xnp)
    back_inplace(rd, r, rnp)
    return x, r


def lsgs_sweep(state, x, r, order="forward"):
    """Least-squares Gauss-Seidel sweep (smoothers.py:270-278 ->
    kernels.py:43-66)."""
    if order not in ("forward", "backward"):
        raise ValueError("order must be 'forward' or 'backward'")
    xd, xnp, rd, rnp = _pair(state, x, r)
    ops = ctypes.c_int64()
    _lib.call("ocmg_ne_gs_sweep", state.system.handle,
              _lib.GS_MODES[state.gs_mode], 1 if order == "forward" else 0,
              _lib.dptr(xd), _lib.dptr(rd), _lib.stream_ptr(),
              ctypes.byref(ops))
    state.op_count += ops.value
    back_inplace(xd, x, xnp)
    back_inplace(rd, r, rnp)
    return x, r


def lsgs_sweep_into(state, x, r_in, r_out, order="forward"):
    """The NE-GS sweep with the residual out of place (device tensors only):
    r_out receives the new residual, r_in may be overwritten.  The cycle
    driver's form for multicolour levels (no copy-back); B200 addition."""
    if order not in ("forward", "backward"):
        raise ValueError("order must be 'forward' or 'backward'")
    n = state.system.n
    for t in (x, r_in, r_out):
        if not (hasattr(t, "is_cuda") and t.is_cuda and t.numel() == n):
            raise ValueError(f"expected CUDA tensors of length {n}")
    ops = ctypes.c_int64()
    _lib.call("ocmg_ne_gs_sweep_into", state.system.handle,
              _lib.GS_MODES[state.gs_mode], 1 if order == "forward" else 0,
              _lib.dptr(x), _lib.dptr(r_in), _lib.dptr(r_out),
              _lib.stream_ptr(), ctypes.byref(ops))
    state.op_count += ops.value
    return x, r_out


def cgs_sweep(state, x, r):
    """Collective Gauss-Seidel over state/adjoint pairs (smoothers.py:288-295
    -> kernels.py:70-96).  gs_mode "reference"/"wavefront": the reference's
    vertex order, bit-identical; "multicolour": 3-colour order."""
    if state.system.problem != "poisson":
        raise ValueError("collective sweep needs a scalar control system")
    xd, xnp, rd, rnp = _pair(state, x, r)
    ops = ctypes.c_int64()
    _lib.call("ocmg_cgs_sweep", state.system.handle, _lib.GS_MODES[state.gs_mode],
              _lib.dptr(xd), _lib.dptr(rd), _lib.dptr(state._scratch()),
              _lib.stream_ptr(), ctypes.byref(ops))
    state.op_count += ops.value
    back_inplace(xd, x, xnp)
    back_inplace(rd, r, rnp)
    return x, r


def vanka_sweep(state, x, r, tau=None, order="forward"):
    """Multiplicative patch sweep with damping (smoothers.py:298-309 ->
    kernels.py:99-131), bit-identical to the reference."""
    if order not in ("forward", "backward"):
        raise ValueError("order must be 'forward' or 'backward'")
    if state.patches is None:
        raise ValueError("the state is not bound to the patch smoother")
    t = state.tau if tau is None else tau
    xd, xnp, rd, rnp = _pair(state, x, r)
    ops = ctypes.c_int64()
    _lib.call("ocmg_vanka_sweep", state.system.handle, float(t),
              1 if order == "forward" else 0, _lib.dptr(xd), _lib.dptr(rd),
              _lib.stream_ptr(), ctypes.byref(ops))
    state.op_count += ops.value
    back_inplace(xd, x, xnp)
    back_inplace(rd, r, rnp)
    return x, r


def slsgs_sweep(state, x, r):
    """Forward then backward NE-GS (smoothers.py:281-285)."""
    lsgs_sweep(state, x, r, order="forward")
    lsgs_sweep(state, x, r, order="backward")
    return x, r
