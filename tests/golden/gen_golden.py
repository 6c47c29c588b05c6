"""Generate golden fixtures by running the reference package ``ocmg`` itself.

Run in the build container only (``/root/reference`` does not exist on the
GPU box): ``python tests/golden/gen_golden.py``.  Writes small ``.npz``
fixtures next to this script; they pin the CPU oracle (``oracle/``) and,
through it, the CUDA path.  The reference is imported read-only: bytecode
writing is disabled and numba's cache is redirected to /tmp so nothing is
written under /root/reference.

Protocols:
  * BASELINE protocol: f = (M y_D, 0), y_D ~ U[-1,1] from default_rng(seed)
    (Poisson seed 0, Stokes seed 1), x0 = 0, cycle + pressure mean
    projection, stop at ||f - A x||_2 <= 1e-8 ||f||_2.
  * reference protocol: Multigrid.solve() (rhs 0, random x0, L-norm 1e-6).
"""
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/ocmg_numba_cache")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402
import ocmg  # noqa: E402
from ocmg import mesh as ocmg_mesh  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def csr_dict(prefix, m):
    return {f"{prefix}_indptr": np.asarray(m.row_offsets),
            f"{prefix}_indices": np.asarray(m.col_indices),
            f"{prefix}_data": np.asarray(m.values),
            f"{prefix}_shape": np.array(m.shape)}


def operators(problem, k, alpha):
    kc = k - 1
    systems, transfers = ocmg.assemble_hierarchy(problem, kc, k, alpha)
    fine = systems[-1]
    st = ocmg.make_smoother(fine, "lsgs")
    d = {}
    d.update(csr_dict("A", fine.matrix))
    d.update(csr_dict("P", transfers[0].prolongation))
    d.update(csr_dict("R", transfers[0].restriction))
    d["L"] = np.asarray(fine.norm_diag)
    d["n_diag"] = np.asarray(st.n_diag)
    d["row_scaled"] = np.asarray(st.row_scaled)
    np.savez_compressed(os.path.join(OUT, f"ops_{problem}_k{k}.npz"), **d)


def sweeps(problem, k, alpha, seed):
    s = ocmg.assemble_hierarchy(problem, k - 1, k, alpha)[0][-1]
    rng = np.random.default_rng(seed)
    x0 = rng.uniform(-1.0, 1.0, s.n)
    f = rng.uniform(-1.0, 1.0, s.n)
    ocmg.pressure_mean_projection(s, x0)
    r0 = s.residual(x0, f)
    d = {"x0": x0, "f": f, "r0": r0}
    for name in ("normal", "lsgs", "slsgs"):
        st = ocmg.make_smoother(s, name)
        x, r = x0.copy(), r0.copy()
        st.sweep(x, r)
        d[f"{name}_x"], d[f"{name}_r"] = x, r
        d[f"{name}_ops"] = np.array(st.op_count)
    st = ocmg.make_smoother(s, "lsgs")
    x, r = x0.copy(), r0.copy()
    ocmg.lsgs_sweep(st, x, r, order="backward")
    d["lsgs_bwd_x"], d["lsgs_bwd_r"] = x, r
    # two chained forward sweeps (the nu=2 pre-smoothing of one visit)
    x, r = x0.copy(), r0.copy()
    st.sweep(x, r)
    st.sweep(x, r)
    d["lsgs2_x"], d["lsgs2_r"] = x, r
    np.savez_compressed(os.path.join(OUT, f"sweep_{problem}_k{k}.npz"), **d)


def baseline(problem, k, alpha, smoother, cycle, coarsest, seed, tag,
             add_sine=False, keep=3):
    cfg = ocmg.CycleConfig(smoother=ocmg.SmootherKind(smoother), cycle=cycle,
                           nu_pre=2 if smoother != "slsgs" else 1,
                           nu_post=2 if smoother != "slsgs" else 1,
                           coarsest_level=coarsest)
    mg = ocmg.build_solver(problem, k, alpha, cfg)
    fine = mg.finest
    rng = np.random.default_rng(seed)
    if problem == "poisson":
        lv = fine.mesh
        yd = rng.uniform(-1.0, 1.0, lv.n_vertices)
        if add_sine:
            vx, vy = lv.vertices[:, 0], lv.vertices[:, 1]
            yd = yd + np.sin(np.pi * vx) * np.sin(np.pi * vy)
        sl = fine.layout.slice_of("state")
    else:
        sl = fine.layout.slice_of("velocity")
        yd = rng.uniform(-1.0, 1.0, sl.stop - sl.start)
    a = fine.matrix.to_scipy()
    f = np.zeros(fine.n)
    f[sl] = a[sl, sl] @ yd
    x = np.zeros(fine.n)
    nf = np.linalg.norm(f)
    hist, its = [], []
    for c in range(300):
        x = mg.cycle(len(mg.systems) - 1, x, f)
        ocmg.pressure_mean_projection(fine, x)
        rel = np.linalg.norm(fine.residual(x, f)) / nf
        hist.append(rel)
        if c < keep:
            its.append(x.copy())
        if rel <= 1e-8:
            break
    np.savez_compressed(os.path.join(OUT, f"baseline_{tag}.npz"),
                        f=f, hist=np.array(hist), x_final=x,
                        iterates=np.array(its))
    print(tag, len(hist), hist[:3], hist[-1])


def cgs_sweep_fixture(k, alpha, seed):
    """CGS collective smoother (kernels.py:70-96, smoothers.py:288-295): one
    sweep from the same seeded state as sweeps()."""
    s = ocmg.assemble_hierarchy("poisson", k - 1, k, alpha)[0][-1]
    rng = np.random.default_rng(seed)
    x0 = rng.uniform(-1.0, 1.0, s.n)
    f = rng.uniform(-1.0, 1.0, s.n)
    r0 = s.residual(x0, f)
    st = ocmg.make_smoother(s, "cgs")
    x, r = x0.copy(), r0.copy()
    st.sweep(x, r)
    d = {"x0": x0, "f": f, "r0": r0, "cgs_x": x, "cgs_r": r,
         "cgs_ops": np.array(st.op_count)}
    x2, r2 = x.copy(), r.copy()
    st.sweep(x2, r2)
    d["cgs2_x"], d["cgs2_r"] = x2, r2
    np.savez_compressed(os.path.join(OUT, f"sweep_poisson_k{k}_cgs.npz"), **d)


def vanka_fixture(k, alpha, seed):
    """Vanka patch smoother (kernels.py:99-131, smoothers.py:87-176,
    297-...): the patches of a Stokes level and forward / backward sweeps
    from the same seeded state as sweeps()."""
    s = ocmg.assemble_hierarchy("stokes", k - 1, k, alpha)[0][-1]
    rng = np.random.default_rng(seed)
    x0 = rng.uniform(-1.0, 1.0, s.n)
    f = rng.uniform(-1.0, 1.0, s.n)
    ocmg.pressure_mean_projection(s, x0)
    r0 = s.residual(x0, f)
    st = ocmg.make_smoother(s, "vanka")
    pt = st.patches
    d = {"x0": x0, "f": f, "r0": r0, "offsets": pt.offsets, "dofs": pt.dofs,
         "sizes": pt.sizes, "inverses": pt.inverses, "vertex_ids": pt.vertex_ids}
    x, r = x0.copy(), r0.copy()
    st.sweep(x, r)
    d["fwd_x"], d["fwd_r"] = x.copy(), r.copy()
    st.sweep(x, r, post=True)
    d["fwdbwd_x"], d["fwdbwd_r"] = x.copy(), r.copy()
    # the reference's operator (its P2 quadrature leaves ~1e-17 entries
    # where the exact assembly has zeros): the sweep's own input
    d.update(csr_dict("A", s.matrix))
    np.savez_compressed(os.path.join(OUT, f"sweep_stokes_k{k}_vanka.npz"), **d)


def reference_protocol(problem, k, alpha, smoother, tag):
    cfg = ocmg.CycleConfig(smoother=ocmg.SmootherKind(smoother))
    mg = ocmg.build_solver(problem, k, alpha, cfg)
    rep = mg.solve()
    np.savez_compressed(os.path.join(OUT, f"refproto_{tag}.npz"),
                        hist=np.array(rep.norm_history),
                        iterations=np.array(rep.iterations))
    print(tag, rep.iterations)


def coarse(problem, alpha):
    s = ocmg.assemble_hierarchy(problem, 1, 2, alpha)[0][0]
    cs = ocmg.CoarseSolver(s)
    rhs = np.random.default_rng(7).uniform(-1.0, 1.0, s.n)
    np.savez_compressed(os.path.join(OUT, f"coarse_{problem}.npz"),
                        rhs=rhs, x=cs.solve(rhs))


def table_fixture():
    """cli.run_table on a small sweep."""
    from ocmg import cli
    out = {}
    for prob, levels, smoothers in (("poisson", (3, 5), ("normal", "lsgs", "slsgs", "cgs")),
                                    ("stokes", (2, 3), ("normal", "lsgs", "slsgs"))):
        spec = cli.ExperimentSpec(problem=prob, smoothers=smoothers,
                                  levels=levels, alphas=(1.0, 1e-6))
        res = cli.run_table(spec)
        out[prob] = [(c.smoother, c.alpha, c.level, c.iterations, c.converged)
                     for c in res.cells]
        print(cli.render_markdown(res))
    import json
    with open(os.path.join(OUT, "table_small.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__" and sys.argv[1:] == ["table"]:
    ocmg_mesh.MAX_LEVEL = 12
    table_fixture()
    sys.exit(0)

if __name__ == "__main__" and sys.argv[1:2] == ["vanka"]:
    # the Vanka patch smoother (added in round 1)
    ocmg_mesh.MAX_LEVEL = 12
    vanka_fixture(3, 1e-4, 12)
    if sys.argv[2:] != ["sweep"]:
        baseline("stokes", 4, 1e-4, "vanka", "v", 1, 1, "s4_vanka")
        baseline("stokes", 5, 1e-4, "vanka", "v", 1, 1, "c4_vanka", keep=1)
    sys.exit(0)

if __name__ == "__main__" and sys.argv[1:] == ["cgs"]:
    # the CGS smoother (added in round 1)
    ocmg_mesh.MAX_LEVEL = 12
    cgs_sweep_fixture(4, 1e-6, 11)
    baseline("poisson", 6, 1e-6, "cgs", "v", 1, 0, "c1_cgs")
    baseline("poisson", 6, 1e-4, "cgs", "v", 2, 0, "p6_a1e-4_c2_cgs", keep=1)
    baseline("poisson", 5, 1e-6, "cgs", "w", 1, 0, "p5w_sine_cgs", add_sine=True,
             keep=1)
    sys.exit(0)

if __name__ == "__main__":
    ocmg_mesh.MAX_LEVEL = 12
    operators("poisson", 3, 1e-6)
    operators("stokes", 2, 1e-4)
    sweeps("poisson", 4, 1e-6, 11)
    sweeps("stokes", 3, 1e-4, 12)
    coarse("poisson", 1e-6)
    coarse("stokes", 1e-4)
    # BASELINE config 1 / config 4 (NE-GS) + the other smoothers
    baseline("poisson", 6, 1e-6, "lsgs", "v", 1, 0, "c1_lsgs")
    baseline("poisson", 6, 1e-6, "normal", "v", 1, 0, "c1_normal", keep=1)
    baseline("poisson", 6, 1e-6, "slsgs", "v", 1, 0, "c1_slsgs", keep=1)
    baseline("stokes", 5, 1e-4, "lsgs", "v", 1, 1, "c4_lsgs")
    baseline("stokes", 5, 1e-4, "normal", "v", 1, 1, "c4_normal", keep=1)
    # small W-cycle with the config-3 input shape (U[-1,1] + sin sin)
    baseline("poisson", 5, 1e-6, "lsgs", "w", 1, 0, "p5w_sine",
             add_sine=True)
    # config-2 shape at a small level (coarsest L2)
    baseline("poisson", 6, 1e-4, "lsgs", "v", 2, 0, "p6_a1e-4_c2")
    reference_protocol("poisson", 4, 1.0, "lsgs", "p4_lsgs")
    reference_protocol("stokes", 3, 1e-6, "normal", "s3_normal")
