"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (north_star): bit-exact where the arithmetic is the reference's
(residual, NE-Jacobi, reference-mode NE-GS, transfers); wavefront-mode
NE-GS iterates within 1e-12 relative with identical cycle counts; the
multicolour mode is compared with the oracle run in the same colour order.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1502_03917_b200 as P  # noqa: E402
from paper_1502_03917_b200 import _lib  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.cpu().numpy()


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


SYSTEMS = {}


def systems(prob, k, alpha):
    key = (prob, k, alpha)
    if key not in SYSTEMS:
        if prob == "poisson":
            SYSTEMS[key] = (O.poisson_system(k, alpha),
                            P.build_poisson_system(k, alpha))
        else:
            SYSTEMS[key] = (O.stokes_system(k, alpha),
                            P.build_stokes_system(k, alpha))
    return SYSTEMS[key]


def inputs(osys, seed):
    rng = np.random.default_rng(seed)
    x0 = rng.uniform(-1, 1, osys.n)
    f = rng.uniform(-1, 1, osys.n)
    osys.mean_project(x0)
    return x0, f, osys.residual(x0, f)


CASES = [("poisson", 2, 1e-6), ("poisson", 3, 1e-6), ("poisson", 5, 1e-4),
         ("poisson", 6, 1.0), ("stokes", 2, 1e-4), ("stokes", 4, 1e-6)]


@pytest.mark.parametrize("prob,k,alpha", CASES)
def test_residual_bitwise(prob, k, alpha):
    osys, dsys = systems(prob, k, alpha)
    x0, f, r0 = inputs(osys, 1)
    assert np.array_equal(host(dsys.residual(dev(x0), dev(f))), r0)
    assert np.array_equal(host(dsys.residual(dev(x0))),
                          osys.residual(x0))


@pytest.mark.parametrize("prob,k,alpha", CASES)
def test_ne_jacobi_bitwise(prob, k, alpha):
    osys, dsys = systems(prob, k, alpha)
    x0, f, r0 = inputs(osys, 2)
    st = P.make_smoother(dsys, "normal")
    xd, rd = dev(x0), dev(r0)
    for _ in range(3):
        st.sweep(xd, rd)
    xo, ro = x0.copy(), r0.copy()
    ost = O.OracleSmoother(osys, "normal")
    for _ in range(3):
        ost.sweep(xo, ro)
    assert np.array_equal(host(xd), xo)
    assert np.array_equal(host(rd), ro)
    # (both count 2 nnz per sweep of the exactly assembled operator; the
    # reference's own Stokes matrix also stores the quadrature's ~1e-17 entries)
    assert st.op_count == ost.op_count


@pytest.mark.parametrize("prob,k,alpha", CASES)
@pytest.mark.parametrize("order", ["forward", "backward"])
def test_ne_gs_reference_mode_bitwise(prob, k, alpha, order):
    osys, dsys = systems(prob, k, alpha)
    x0, f, r0 = inputs(osys, 3)
    st = P.make_smoother(dsys, "lsgs", gs_mode="reference")
    xd, rd = dev(x0), dev(r0)
    P.lsgs_sweep(st, xd, rd, order=order)
    P.lsgs_sweep(st, xd, rd, order=order)
    xo, ro = x0.copy(), r0.copy()
    ost = O.OracleSmoother(osys, "lsgs")
    for _ in range(2):
        ost.lsgs(xo, ro, forward=(order == "forward"))
    assert np.array_equal(host(xd), xo)
    assert np.array_equal(host(rd), ro)


@pytest.mark.parametrize("mode", ["reference", "wavefront"])
def test_ne_gs_exact_small_level_unaligned_views(mode):
    """Small levels run the one-CTA sweep (16-byte cp.async staging); views at
    an odd double offset take the launch-per-level (reference) or banded
    (wavefront) path.  Reference mode bitwise, wavefront mode 1e-12."""
    osys, dsys = systems("poisson", 5, 1e-4)
    x0, f, r0 = inputs(osys, 5)
    st = P.make_smoother(dsys, "lsgs", gs_mode=mode)
    res = []
    for off in (0, 1):
        xb = torch.zeros(osys.n + 1, dtype=torch.float64, device="cuda")
        rb = torch.zeros_like(xb)
        xd, rd = xb[off:off + osys.n], rb[off:off + osys.n]
        xd.copy_(dev(x0))
        rd.copy_(dev(r0))
        P.lsgs_sweep(st, xd, rd, order="forward")
        P.lsgs_sweep(st, xd, rd, order="backward")
        res.append((host(xd), host(rd)))
    xo, ro = x0.copy(), r0.copy()
    ost = O.OracleSmoother(osys, "lsgs")
    ost.lsgs(xo, ro, forward=True)
    ost.lsgs(xo, ro, forward=False)
    for off, (xh, rh) in enumerate(res):
        if mode == "wavefront":  # FMA arithmetic: 1e-12
            assert rel(xh, xo) < 1e-12
            assert rel(rh, ro) < 1e-11
        else:
            assert np.array_equal(xh, xo)
            assert np.array_equal(rh, ro)


@pytest.mark.parametrize("k", [7, 8])
@pytest.mark.parametrize("order", ["forward", "backward"])
@pytest.mark.parametrize("mode", ["reference", "wavefront"])
def test_ne_gs_exact_mid_levels_bitwise(k, order, mode):
    """L7-L8 run the one-CTA anti-diagonal ring sweep in both exact modes:
    bit-identical to the reference loop in reference mode, 1e-12 in the
    wavefront mode's FMA arithmetic."""
    osys, dsys = systems("poisson", k, 1e-6)
    x0, f, r0 = inputs(osys, 6)
    st = P.make_smoother(dsys, "lsgs", gs_mode=mode)
    xd, rd = dev(x0), dev(r0)
    for _ in range(2):
        P.lsgs_sweep(st, xd, rd, order=order)
    xo, ro = x0.copy(), r0.copy()
    ost = O.OracleSmoother(osys, "lsgs")
    for _ in range(2):
        ost.lsgs(xo, ro, forward=(order == "forward"))
    if mode == "reference":
        assert np.array_equal(host(xd), xo)
        assert np.array_equal(host(rd), ro)
    else:  # FMA arithmetic: the 1e-12 bar
        assert rel(host(xd), xo) < 1e-12
        assert rel(host(rd), ro) < 1e-11


@pytest.mark.parametrize("prob,k,alpha", CASES)
def test_ne_gs_wavefront_mode(prob, k, alpha):
    """Reference order, delta-form arithmetic: 1e-12 (north_star bar)."""
    osys, dsys = systems(prob, k, alpha)
    x0, f, r0 = inputs(osys, 4)
    st = P.make_smoother(dsys, "slsgs", gs_mode="wavefront")
    xd, rd = dev(x0), dev(r0)
    for _ in range(2):
        st.sweep(xd, rd)
    xo, ro = x0.copy(), r0.copy()
    ost = O.OracleSmoother(osys, "slsgs")
    for _ in range(2):
        ost.sweep(xo, ro)
    assert rel(host(xd), xo) < 1e-12
    # residual coherence: maintained r equals f - A x
    assert rel(host(rd), osys.residual(host(xd), f)) < 1e-11
    assert rel(host(rd), ro) < 1e-11


@pytest.mark.parametrize("k,alpha", [(5, 1e-4), (6, 1e-6)])
def test_stokes_wavefront_level_launches(k, alpha):
    """Generic levels above the one-CTA size (a launch per dependency level,
    a warp per row): 1e-12 against the reference loop, both directions."""
    osys, dsys = systems("stokes", k, alpha)
    x0, f, r0 = inputs(osys, 7)
    st = P.make_smoother(dsys, "slsgs", gs_mode="wavefront")
    xd, rd = dev(x0), dev(r0)
    for _ in range(2):
        st.sweep(xd, rd)
    xo, ro = x0.copy(), r0.copy()
    ost = O.OracleSmoother(osys, "slsgs")
    for _ in range(2):
        ost.sweep(xo, ro)
    assert rel(host(xd), xo) < 1e-12
    assert rel(host(rd), ro) < 1e-11


@pytest.mark.parametrize("k", [7, 8, 10, 12])
@pytest.mark.parametrize("order", ["forward", "backward"])
def test_wavefront_vs_reference_mode_many_bands(k, order):
    """The fused wavefront kernel against the bitwise reference-order path at
    levels with many bands (L12: 129 bands of 32 rows)."""
    dsys = P.build_poisson_system(k, 1e-6)
    g = torch.Generator(device="cuda").manual_seed(k)
    x0 = torch.rand(dsys.n, dtype=torch.float64, device="cuda",
                    generator=g) - 0.5
    f = torch.rand(dsys.n, dtype=torch.float64, device="cuda", generator=g)
    r0 = dsys.residual(x0, f)
    out = {}
    for mode in ("wavefront", "reference"):
        st = P.make_smoother(dsys, "lsgs", gs_mode=mode)
        x, r = x0.clone(), r0.clone()
        for _ in range(2):
            P.lsgs_sweep(st, x, r, order=order)
        out[mode] = (x, r)
    xw, rw = out["wavefront"]
    xr, rr = out["reference"]
    ex = float((xw - xr).abs().max() / xr.abs().max())
    er = float((rw - rr).abs().max() / rr.abs().max())
    assert ex < 1e-12, ex
    assert er < 1e-10, er


def _colour_perm(osys, dsys):
    """Unknown order of the multicolour sweep."""
    if osys.problem == "poisson":
        # vertex colours (ix + 2 iy) mod 7 in turn; each vertex's state then
        # adjoint unknown
        n1 = 2 ** osys.k + 1
        iy, ix = np.divmod(np.arange(n1 * n1), n1)
        col = (ix + 2 * iy) % 7
        N = n1 * n1
        verts = np.concatenate([np.flatnonzero(col == c) for c in range(7)])
        return np.stack([verts, verts + N], axis=1).reshape(-1)
    # generic levels: greedy distance-2 colouring in index order
    A = osys.A
    colour = -np.ones(osys.n, dtype=np.int64)
    for i in range(osys.n):
        nb = A.indices[A.indptr[i]:A.indptr[i + 1]]
        used = set()
        for j in nb:
            used.update(colour[A.indices[A.indptr[j]:A.indptr[j + 1]]])
        c = 0
        while c in used:
            c += 1
        colour[i] = c
    return np.argsort(colour, kind="stable")


@pytest.mark.parametrize("prob,k,alpha", [("poisson", 4, 1e-6),
                                          ("poisson", 6, 1.0),
                                          ("stokes", 3, 1e-4)])
def test_ne_gs_multicolour_matches_permuted_oracle(prob, k, alpha):
    osys, dsys = systems(prob, k, alpha)
    x0, f, r0 = inputs(osys, 5)
    st = P.make_smoother(dsys, "lsgs", gs_mode="multicolour")
    xd, rd = dev(x0), dev(r0)
    st.sweep(xd, rd)
    perm = _colour_perm(osys, dsys)
    Ap = O.ocmg_oracle._canon(osys.A[perm][:, perm])
    psys = O.OracleSystem(osys.problem, osys.k, osys.alpha, Ap, osys.L[perm],
                          osys.fields, osys.mass)
    xo, ro = x0[perm].copy(), r0[perm].copy()
    O.OracleSmoother(psys, "lsgs").lsgs(xo, ro, True)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size)
    assert rel(host(xd), xo[inv]) < 1e-13
    assert rel(host(rd), ro[inv]) < 1e-10


@pytest.mark.parametrize("k", [3, 4, 6, 8, 10, 12])
@pytest.mark.parametrize("forward", [True, False])
def test_multicolour_one_launch_matches_colour_passes(k, forward):
    """The pipelined one-launch multicolour sweep (strip tiles with halo,
    all 14 colours in flight) is bit-identical to 14 in-place colour passes."""
    import ctypes
    dsys = P.build_poisson_system(k, 1e-6)
    g = torch.Generator(device="cuda").manual_seed(11 + k)
    x = torch.rand(dsys.n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    r = torch.rand(dsys.n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    x2, r2 = x.clone(), r.clone()
    st = P.make_smoother(dsys, "lsgs", gs_mode="multicolour")
    for _ in range(2):
        if forward:
            st.sweep(x, r)
        else:
            P.smoothers.lsgs_sweep(st, x, r, order="backward")
        fn = _lib.load().ocmg__debug_mc_passes
        fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                       ctypes.c_void_p, ctypes.c_void_p]
        _lib.check(fn(dsys.handle, int(forward), _lib.dptr(x2), _lib.dptr(r2),
                      _lib.stream_ptr()))
    torch.cuda.synchronize()
    assert torch.equal(x, x2)
    assert torch.equal(r, r2)


def test_rolling_window_multicolour_kernel_is_bit_identical():
    """The experimental rolling-window one-launch kernel (ocmg_p1_mc2.cuh,
    opt-in with OCMG_MC_SWEEP=roll, read once per process) against the
    colour passes and, through the strip entry point, against itself on the
    whole level: child processes, since the switch is per process."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, OCMG_MC_SWEEP="roll")
    for k in (7, 10):
        out = subprocess.run([sys.executable, os.path.join(root, "scripts", "mc_check.py"), str(k)],
                             env=env, capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        lines = [ln for ln in out.stdout.splitlines() if ln.startswith("k=")]
        assert len(lines) == 2 and all("equal=True" in ln for ln in lines), out.stdout
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                          os.path.join(root, "tests", "test_gpu_parity.py"), "-k",
                          "test_strip_sweeps_match_single_gpu and 10"],
                         env=env, capture_output=True, text=True, timeout=900, cwd=root)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]


@pytest.mark.parametrize("k", [4, 8, 10])
@pytest.mark.parametrize("mode", ["multicolour", "wavefront"])
def test_sweep_into_matches_in_place(k, mode):
    dsys = P.build_poisson_system(k, 1e-4)
    g = torch.Generator(device="cuda").manual_seed(3 + k)
    x = torch.rand(dsys.n, dtype=torch.float64, device="cuda", generator=g)
    r = torch.rand(dsys.n, dtype=torch.float64, device="cuda", generator=g)
    x2, ra, rb = x.clone(), r.clone(), torch.empty_like(r)
    st = P.make_smoother(dsys, "lsgs", gs_mode=mode)
    st.sweep(x, r)
    P.smoothers.lsgs_sweep_into(st, x2, ra, rb)
    torch.cuda.synchronize()
    assert torch.equal(x, x2)
    assert torch.equal(r, rb)


@pytest.mark.parametrize("k,ws", [(8, 2), (10, 3), (10, 4), (12, 8)])
def test_strip_sweeps_match_single_gpu(k, ws):
    """Strip decomposition: every rank's strip sweep on its
    slab (ghosts exchanged by loopback copies, ranks run one after another)
    reproduces the single-GPU multicolour sweep bit for bit, 2 sweeps fwd+bwd."""
    from paper_1502_03917_b200.strips import (LoopbackExchange, StripPartition,
                                              strip_sweep)
    dsys = P.build_poisson_system(k, 1e-6)
    n1 = 2 ** k + 1
    g = torch.Generator(device="cuda").manual_seed(17 + k)
    x = torch.rand(dsys.n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    r = torch.rand(dsys.n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    parts = [StripPartition(n1, ws, p) for p in range(ws)]
    xs = [p.scatter(x) for p in parts]
    rs = [p.scatter(r) for p in parts]
    outs = [torch.empty_like(t) for t in rs]
    lb = LoopbackExchange(parts)
    st = P.make_smoother(dsys, "lsgs", gs_mode="multicolour")
    for fwd in (True, False):
        P.smoothers.lsgs_sweep(st, x, r, order="forward" if fwd else "backward")
        lb.exchange(rs)
        for p, xo, ri, ro in zip(parts, xs, rs, outs):
            strip_sweep(dsys, p, xo, ri, ro, forward=fwd)
        rs, outs = outs, rs
    torch.cuda.synchronize()
    xg = torch.cat([p.own(xo) for p, xo in zip(parts, xs)], dim=1).reshape(-1)
    rg = torch.cat([p.own(ri) for p, ri in zip(parts, rs)], dim=1).reshape(-1)
    assert torch.equal(xg, x)
    assert torch.equal(rg, r)


@pytest.mark.parametrize("cycle,smoother,k,coarsest", [
    ("w", "lsgs", 8, 3), ("v", "slsgs", 7, 3), ("w", "lsgs", 5, 3),
    ("w", "lsgs", 8, 1), ("v", "lsgs", 6, 1), ("w", "slsgs", 5, 1),
    ("v", "lsgs", 7, 2), ("w", "lsgs", 6, 2)])
def test_fused_coarse_block_is_bit_identical(cycle, smoother, k, coarsest):
    """The one-launch coarse end of the cycle (ocmg_subcycle.cuh) reproduces
    the per-level cycle bit for bit, down to the reference's default
    coarsest level L1 (the generic CSR level L2 inside the block)."""
    import ctypes
    cfg = P.CycleConfig(smoother=P.SmootherKind(smoother), cycle=cycle,
                        coarsest_level=coarsest, gs_mode="multicolour")
    mg = P.build_solver("poisson", k, 1e-6, cfg)
    f = P.baseline_rhs(mg.finest, 0, add_sine=True)
    fn = _lib.load().ocmg__debug_hierarchy_fuse
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    set_collapse(mg, 0)  # the fused block, not the collapsed map
    xs, hs = [], []
    for on in (1, 0):
        _lib.check(fn(mg.native().handle, on))
        x, hist = mg.solve_to_tolerance(f, tol=0.0, max_cycles=3)
        xs.append(host(x) if hasattr(x, "cpu") else x)
        hs.append(hist)
    assert np.array_equal(xs[0], xs[1])
    assert hs[0] == hs[1]


def set_collapse(mg, max_n):
    """Collapse the coarse end of mg's finest hierarchy for levels of at
    most max_n unknowns (0 off, -1 the library default); returns the
    collapsed hierarchy index (0: none)."""
    import ctypes
    fn = _lib.load().ocmg__debug_hierarchy_collapse
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int)]
    out = ctypes.c_int()
    _lib.check(fn(mg.native().handle, max_n, ctypes.byref(out)))
    return out.value


@pytest.mark.parametrize("prob,k,cycle,smoother,mode,co", [
    ("poisson", 8, "w", "lsgs", "wavefront", 1),
    ("poisson", 8, "w", "lsgs", "multicolour", 1),
    ("poisson", 7, "v", "slsgs", "wavefront", 2),
    ("poisson", 7, "w", "normal", "multicolour", 1),
    ("poisson", 7, "w", "cgs", "multicolour", 3),
    ("stokes", 4, "w", "lsgs", "wavefront", 1),
    ("stokes", 4, "v", "normal", "multicolour", 1)])
def test_collapsed_coarse_end_matches_per_level_cycle(prob, k, cycle, smoother, mode, co):
    """The coarse end of the cycle as one dense map (setup_collapse: the
    coarse correction of the deepest levels built column by column from the
    device's own sub-cycle on unit vectors) gives the per-level cycle's
    iterates to 1e-12 of max|x| and the same residual history to 1e-9."""
    kind = (P.SmootherKind("normal", tau=0.35 if prob == "stokes" else 0.4)
            if smoother == "normal" else P.SmootherKind(smoother))
    cfg = P.CycleConfig(smoother=kind, cycle=cycle, coarsest_level=co, gs_mode=mode)
    mg = P.build_solver(prob, k, 1e-4, cfg)
    f = P.baseline_rhs(mg.finest, 0, add_sine=False)
    xs, hs, cols = [], [], []
    for max_n in (0, -1):
        cols.append(set_collapse(mg, max_n))
        x, hist = mg.solve_to_tolerance(f, tol=0.0, max_cycles=4)
        xs.append(host(x))
        hs.append(np.array(hist))
    assert cols[0] == 0 and cols[1] >= 1, cols
    assert np.abs(xs[1] - xs[0]).max() <= 1e-12 * np.abs(xs[0]).max()
    assert np.allclose(hs[1], hs[0], rtol=1e-9, atol=0)


def test_reference_mode_never_collapses():
    cfg = P.CycleConfig(smoother=P.SmootherKind("lsgs"), cycle="w", coarsest_level=1,
                        gs_mode="reference")
    mg = P.build_solver("poisson", 7, 1e-4, cfg)
    assert set_collapse(mg, -1) == 0


@pytest.mark.parametrize("k,ws,cycle,smoother,co", [(8, 2, "v", "lsgs", 3),
                                                     (9, 4, "w", "lsgs", 3),
                                                     (9, 3, "v", "slsgs", 3),
                                                     (9, 2, "w", "lsgs", 1),
                                                     (9, 3, "v", "normal", 3),
                                                     (10, 4, "w", "normal", 1)])
def test_strip_multigrid_matches_single_gpu(k, ws, cycle, smoother, co):
    """The strip-partitioned cycle, every rank run in this
    process with loopback exchanges, reproduces the single-GPU cycle bit for
    bit -- multicolour NE-GS (15 ghost rows per sweep) and NE-Jacobi (r and
    p ghost rows, one each), down to the reference's coarsest level L1; the
    stopping norms agree to rounding."""
    from paper_1502_03917_b200.strips import LoopbackComm, StripMultigrid
    kind = (P.SmootherKind("normal", tau=0.4) if smoother == "normal"
            else P.SmootherKind(smoother))
    cfg = P.CycleConfig(smoother=kind, cycle=cycle, coarsest_level=co,
                        gs_mode="multicolour")
    mg = P.build_solver("poisson", k, 1e-6, cfg)
    f = P.baseline_rhs(mg.finest, 0, add_sine=True)
    x1, h1 = mg.solve_to_tolerance(f, tol=0.0, max_cycles=3)
    sm = StripMultigrid(mg, ws, list(range(ws)), LoopbackComm())
    sm.load(f)
    h2 = sm.solve(tol=0.0, max_cycles=3)
    torch.cuda.synchronize()
    assert torch.equal(sm.gather_x(), x1)
    assert np.allclose(h1, h2, rtol=1e-12, atol=0)


def test_strip_partition_knobs():
    """n_gpus / collapse_threshold: the loopback partition over 3
    ranks with every level below L9 kept whole is still the single-GPU cycle
    bit for bit; tol_kind selects the stopping rule."""
    from paper_1502_03917_b200.strips import partition
    cfg = P.CycleConfig(smoother=P.SmootherKind("lsgs"), cycle="v", coarsest_level=3,
                        gs_mode="multicolour")
    mg = P.build_solver("poisson", 9, 1e-6, cfg)
    f = P.baseline_rhs(mg.finest, 0, add_sine=True)
    x1, h1 = mg.run(f, tol_kind="rel_residual", tol=0.0, max_cycles=2)
    sm = partition(mg, n_gpus=3, collapse_threshold=mg.finest.n)
    assert sm.first == len(mg.systems) - 1
    sm.load(f)
    sm.solve(tol=0.0, max_cycles=2)
    torch.cuda.synchronize()
    assert torch.equal(sm.gather_x(), x1)
    with pytest.raises(ValueError):
        mg.run(f, tol_kind="energy")
    with pytest.raises(ValueError):
        partition(mg, n_gpus=3, collapse_threshold=10 * mg.finest.n)


@pytest.mark.parametrize("prob,kc", [("poisson", 1), ("poisson", 4),
                                     ("stokes", 1), ("stokes", 3)])
def test_transfers_bitwise(prob, kc):
    alpha = 1e-4
    oc, dc = systems(prob, kc, alpha)
    of, df = systems(prob, kc + 1, alpha)
    otr = O.system_transfer(oc, of)
    dtr = P.system_transfer(dc, df)
    rng = np.random.default_rng(6)
    rf = rng.uniform(-1, 1, of.n)
    c = rng.uniform(-1, 1, oc.n)
    xf = rng.uniform(-1, 1, of.n)
    assert np.array_equal(host(dtr.restriction.matvec(dev(rf))),
                          O.ocmg_oracle.csr_matvec(otr.R, rf))
    xd = dev(xf)
    dtr.prolong_add(dev(c), xd)
    assert np.array_equal(host(xd), xf + O.ocmg_oracle.csr_matvec(otr.P, c))


@pytest.mark.parametrize("prob,alpha", [("poisson", 1e-6), ("stokes", 1e-4)])
def test_coarse_solve(prob, alpha, golden):
    osys, dsys = systems(prob, 1, alpha)
    d = golden(f"coarse_{prob}.npz")
    cs = P.CoarseSolver(dsys)
    x = host(cs.solve(dev(d["rhs"])))
    assert rel(x, d["x"]) < 1e-12
    assert rel(x, O.OracleCoarse(osys).solve(d["rhs"])) < 1e-12


BASELINE = [
    # tag, problem, k, alpha, smoother, cycle, coarsest, seed, sine, mode
    ("c1_lsgs", "poisson", 6, 1e-6, "lsgs", "v", 1, 0, False, "wavefront"),
    ("c1_lsgs", "poisson", 6, 1e-6, "lsgs", "v", 1, 0, False, "reference"),
    ("c1_normal", "poisson", 6, 1e-6, "normal", "v", 1, 0, False, "wavefront"),
    ("c1_slsgs", "poisson", 6, 1e-6, "slsgs", "v", 1, 0, False, "wavefront"),
    ("c4_lsgs", "stokes", 5, 1e-4, "lsgs", "v", 1, 1, False, "wavefront"),
    ("c4_normal", "stokes", 5, 1e-4, "normal", "v", 1, 1, False, "wavefront"),
    ("p5w_sine", "poisson", 5, 1e-6, "lsgs", "w", 1, 0, True, "wavefront"),
    ("p6_a1e-4_c2", "poisson", 6, 1e-4, "lsgs", "v", 2, 0, False,
     "wavefront"),
    # CGS collective smoother, reference vertex order
    ("c1_cgs", "poisson", 6, 1e-6, "cgs", "v", 1, 0, False, "reference"),
    ("p6_a1e-4_c2_cgs", "poisson", 6, 1e-4, "cgs", "v", 2, 0, False,
     "reference"),
    ("p5w_sine_cgs", "poisson", 5, 1e-6, "cgs", "w", 1, 0, True, "reference"),
]


@pytest.mark.parametrize("case", BASELINE,
                         ids=[f"{c[0]}-{c[-1]}" for c in BASELINE])
def test_baseline_protocol_vs_reference_golden(case, golden):
    """Full solves against fixtures made by the reference itself: same
    cycle count, every kept iterate and the final iterate within 1e-12."""
    tag, prob, k, alpha, sm, cyc, co, seed, sine, mode = case
    d = golden(f"baseline_{tag}.npz")
    nu = 1 if sm == "slsgs" else 2
    cfg = P.CycleConfig(smoother=P.SmootherKind(sm), cycle=cyc, nu_pre=nu,
                        nu_post=nu, coarsest_level=co, gs_mode=mode)
    mg = P.build_solver(prob, k, alpha, cfg)
    f = P.baseline_rhs(mg.finest, seed, add_sine=sine)
    assert rel(host(f), d["f"]) <= 1e-15
    x = torch.zeros_like(f)
    its = []
    for c in range(len(d["iterates"])):
        mg.cycle(len(mg.systems) - 1, x, f)
        P.pressure_mean_projection(mg.finest, x)
        its.append(host(x).copy())
    for a, b in zip(its, d["iterates"]):
        assert rel(a, b) < 1e-12
    x, hist = mg.solve_to_tolerance(f, tol=1e-8, max_cycles=300)
    assert len(hist) == len(d["hist"])
    assert rel(host(x), d["x_final"]) < 1e-12
    assert rel(np.array(hist), d["hist"]) < 1e-6


@pytest.mark.parametrize("k", [2, 4, 6])
def test_cgs_sweep_bitwise(k, golden):
    """CGS sweep (kernels.py:70-96) in the reference's vertex order: the
    anti-diagonal levels (k >= 3) or the sequential CSR kernel (k <= 2) are
    bit-identical to the oracle; at k = 4 also to the reference's fixture."""
    osys, dsys = systems("poisson", k, 1e-6)
    if k == 4:
        d = golden("sweep_poisson_k4_cgs.npz")
        x0, r0 = d["x0"], d["r0"]
    else:
        x0, _, r0 = inputs(osys, 9)
    xo, ro = x0.copy(), r0.copy()
    ost = O.OracleSmoother(osys, "cgs")
    st = P.make_smoother(dsys, "cgs", gs_mode="reference")
    xd, rd = dev(x0), dev(r0)
    for _ in range(2):
        ost.sweep(xo, ro)
        st.sweep(xd, rd)
    assert np.array_equal(host(xd), xo)
    assert np.array_equal(host(rd), ro)
    assert st.op_count == ost.op_count
    if k == 4:
        x1, r1 = d["x0"].copy(), d["r0"].copy()
        P.make_smoother(dsys, "cgs", gs_mode="reference").sweep(
            dev_x := dev(x1), dev_r := dev(r1))
        assert np.array_equal(host(dev_x), d["cgs_x"])
        assert np.array_equal(host(dev_r), d["cgs_r"])


def test_cgs_multicolour_matches_permuted_oracle():
    """3-colour CGS = the reference algorithm run in colour order."""
    k = 5
    osys, dsys = systems("poisson", k, 1e-6)
    x0, _, r0 = inputs(osys, 4)
    n1 = 2 ** k + 1
    iy, ix = np.divmod(np.arange(n1 * n1), n1)
    vperm = np.concatenate([np.flatnonzero((ix + iy) % 3 == c) for c in range(3)])
    perm = np.concatenate([vperm, vperm + n1 * n1])
    Ap = O.ocmg_oracle._canon(osys.A[perm][:, perm])
    psys = O.OracleSystem(osys.problem, osys.k, osys.alpha, Ap, osys.L[perm],
                          osys.fields, osys.mass)
    xo, ro = x0[perm].copy(), r0[perm].copy()
    O.OracleSmoother(psys, "cgs").sweep(xo, ro)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size)
    st = P.make_smoother(dsys, "cgs", gs_mode="multicolour")
    xd, rd = dev(x0), dev(r0)
    st.sweep(xd, rd)
    assert rel(host(xd), xo[inv]) < 1e-13
    assert rel(host(rd), ro[inv]) < 1e-11


@pytest.mark.parametrize("k", [10, 12])
def test_cgs_one_launch_matches_six_launch(k):
    """The pipelined one-launch 3-colour CGS sweep is bit-identical to the
    six-launch (solve + gather per colour) form."""
    import ctypes
    dsys = P.build_poisson_system(k, 1e-6)
    g = torch.Generator(device="cuda").manual_seed(21 + k)
    x = torch.rand(dsys.n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    r = torch.rand(dsys.n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    x2, r2 = x.clone(), r.clone()
    st = P.make_smoother(dsys, "cgs", gs_mode="multicolour")
    fn = _lib.load().ocmg__debug_cgs_six_launch
    fn.argtypes = [ctypes.c_int]
    for _ in range(2):
        st.sweep(x, r)
    _lib.check(fn(1))
    try:
        for _ in range(2):
            st.sweep(x2, r2)
    finally:
        _lib.check(fn(0))
    torch.cuda.synchronize()
    assert torch.equal(x, x2)
    assert torch.equal(r, r2)


def test_cgs_multicolour_solve_converges():
    cfg = P.CycleConfig(smoother=P.SmootherKind("cgs"), cycle="v",
                        gs_mode="multicolour")
    mg = P.build_solver("poisson", 7, 1e-6, cfg)
    f = P.baseline_rhs(mg.finest, 0)
    _, hist = mg.solve_to_tolerance(f, tol=1e-8, max_cycles=100)
    assert hist[-1] <= 1e-8 and len(hist) <= 30


@pytest.mark.parametrize("prob", ["poisson", "stokes"])
def test_table_runner_matches_reference(prob):
    """The iteration table (cli.run_table) on the GPU
    reproduces the reference's own table cell by cell (reference protocol,
    W-cycle, tol 1e-6, seed 1234; tests/golden/table_small.json)."""
    import json
    import os

    from paper_1502_03917_b200 import tables as T
    want = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                       "table_small.json")))[prob]
    smoothers = tuple(dict.fromkeys(c[0] for c in want))
    levels = (min(c[2] for c in want), max(c[2] for c in want))
    spec = T.ExperimentSpec(problem=prob, smoothers=smoothers, levels=levels,
                            alphas=(1.0, 1e-6))
    res = T.run_table(spec)
    got = [(c.smoother, c.alpha, c.level, c.iterations, c.converged)
           for c in res.cells]
    assert got == [tuple(c) for c in want]
    assert "| level |" in T.render_table(res)


def test_multicolour_solve_converges():
    """Multicolour mode is a different smoother: report its own cycle count
    (config-1 shape) and check it converges like NE-GS."""
    cfg = P.CycleConfig(smoother=P.SmootherKind("lsgs"), cycle="v",
                        gs_mode="multicolour")
    mg = P.build_solver("poisson", 6, 1e-6, cfg)
    f = P.baseline_rhs(mg.finest, 0)
    _, hist = mg.solve_to_tolerance(f, tol=1e-8, max_cycles=100)
    assert hist[-1] <= 1e-8 and len(hist) <= 40


def test_reference_protocol_solve(golden):
    d = golden("refproto_p4_lsgs.npz")
    cfg = P.CycleConfig(smoother=P.SmootherKind("lsgs"), cycle="w")
    mg = P.build_solver("poisson", 4, 1.0, cfg)
    rep = mg.solve()
    assert rep.iterations == int(d["iterations"]) and rep.converged
    assert rel(np.array(rep.norm_history), d["hist"]) < 1e-12


def test_numpy_arrays_drop_in():
    """Reference-style numpy callers work unchanged (copied through)."""
    osys, dsys = systems("poisson", 4, 1e-6)
    x0, f, r0 = inputs(osys, 7)
    st = P.make_smoother(dsys, "lsgs", gs_mode="reference")
    x, r = x0.copy(), r0.copy()
    st.sweep(x, r)
    xo, ro = x0.copy(), r0.copy()
    O.OracleSmoother(osys, "lsgs").sweep(xo, ro)
    assert np.array_equal(x, xo) and np.array_equal(r, ro)
    assert np.array_equal(dsys.residual(x0, f), r0)


def test_errors_map_to_reference_exceptions():
    osys, dsys = systems("poisson", 4, 1e-6)
    st = P.make_smoother(dsys, "lsgs")
    with pytest.raises(ValueError):
        P.lsgs_sweep(st, dev(np.zeros(osys.n)), dev(np.zeros(osys.n)),
                     order="sideways")
    with pytest.raises(ValueError):
        dsys.residual(dev(np.zeros(osys.n + 1)))
    with pytest.raises(ValueError):
        P.build_poisson_system(4, -1.0)


@pytest.mark.parametrize("mode", ["wavefront", "multicolour", "reference"])
def test_fixed_point_full_size(mode):
    """Size-independent property at a large level: r = 0 is a fixed point of
    every sweep, and after a sweep from a random state the maintained
    residual stays coherent with f - A x."""
    k = 10 if mode == "reference" else 12
    dsys = P.build_poisson_system(k, 1e-6)
    n = dsys.n
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    r = torch.zeros_like(x)
    st = P.make_smoother(dsys, "lsgs", gs_mode=mode)
    x0 = x.clone()
    st.sweep(x, r)
    assert torch.equal(x, x0) and int(torch.count_nonzero(r)) == 0
    f = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    r = dsys.residual(x, f)
    st.sweep(x, r)
    r2 = dsys.residual(x, f)
    err = float((r - r2).abs().max() / r2.abs().max())
    assert err < 1e-9, err


def test_solve_divergence_stop():
    """The on-device loop stops like Multigrid.solve once the relative
    residual exceeds DIVERGENCE_FACTOR times its entering value
    (multigrid.py:26,198-200): with the factor forced tiny, one cycle
    already counts as divergence."""
    import ctypes
    cfg = P.CycleConfig(smoother=P.SmootherKind("lsgs"), cycle="v")
    mg = P.build_solver("poisson", 5, 1e-6, cfg)
    f = P.baseline_rhs(mg.finest, 0)
    x = torch.zeros_like(f)
    hist = np.zeros(10)
    done, div = ctypes.c_int(), ctypes.c_int()
    _lib.call("ocmg_solve_ex", mg.native().handle, _lib.dptr(x), _lib.dptr(f),
              1e-8, 10, 1, 1e-30, _lib.hptr(hist), ctypes.byref(done),
              ctypes.byref(div), _lib.stream_ptr())
    assert div.value == 1 and done.value == 1
    # the default factor (1e6) never fires on a converging solve
    _, h = mg.solve_to_tolerance(f, tol=1e-8, max_cycles=60)
    assert not mg.last_diverged and h[-1] <= 1e-8
