"""Full-size parity pins: run the reference package ``ocmg`` itself on the
BASELINE configs 2 (Poisson L10), 3 (Poisson L12) and 5 (Stokes L10) and
record, per cycle, enough of the iterate to check the device at 1e-12.

Run in the build container only (``/root/reference`` is not on the GPU box;
the L12 run needs ~46 GB of host RAM and ~15 min, each Stokes L10 solve
~45 GB and 10-15 min):

    python tests/golden/gen_fullsize.py c2      # config 2, 6 solves, ~10 min
    python tests/golden/gen_fullsize.py c3      # config 3
    python tests/golden/gen_fullsize.py c5 1e-2 # config 5, one alpha per run

Each run writes ``tests/golden/full_<tag>.npz`` with

* ``hist``     per-cycle ||f - A x||_2 / ||f||_2 (after the mean projection),
* ``idx``      sorted sample indices (seeded, fixed per size; they include the
               first and last unknown of every field),
* ``xs``       x[idx] after every cycle, shape (cycles, len(idx)),
* ``lnorm``    per-cycle BlockSystem.norm(x) = sqrt(sum L_i x_i^2)
               (``assembly.py:265-267``), a checksum over the whole iterate,
* ``sum``, ``absmax`` per-cycle sum(x) and max|x|.

Protocol, the same as ``gen_golden.baseline``:
f = (A[state,state] y_D, 0), y_D ~ U[-1,1] from default_rng(seed) (Poisson
seed 0, + sin(pi x) sin(pi y) for config 3; Stokes seed 1, velocity block),
x0 = 0, ``Multigrid.cycle`` (``multigrid.py:130-159``) then
``pressure_mean_projection`` (``assembly.py:381-388``), stop at 1e-8.
The reference is imported read-only (no bytecode, numba cache in /tmp).
"""
import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/ocmg_numba_cache")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sample_indices(counts, n_per_field, seed=20260):
    """Seeded sample of unknown indices: n_per_field per field plus each
    field's first and last unknown.  ``counts`` are the field sizes in the
    reference layout order."""
    rng = np.random.default_rng(seed)
    out, off = [], 0
    for c in counts:
        out.append(off + rng.choice(c, size=min(c, n_per_field), replace=False))
        out.append(np.array([off, off + c - 1]))
        off += c
    return np.unique(np.concatenate(out)).astype(np.int64)


def run(problem, k, alpha, smoother, cycle, coarsest, seed, tag,
        add_sine=False, n_per_field=512, max_cycles=300):
    import ocmg
    from ocmg import mesh as ocmg_mesh
    ocmg_mesh.MAX_LEVEL = 12
    t0 = time.time()
    nu = 1 if smoother == "slsgs" else 2
    cfg = ocmg.CycleConfig(smoother=ocmg.SmootherKind(smoother), cycle=cycle,
                           nu_pre=nu, nu_post=nu, coarsest_level=coarsest)
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
    del a
    setup = time.time() - t0
    idx = sample_indices(fine.layout.counts, n_per_field)
    x = np.zeros(fine.n)
    nf = np.linalg.norm(f)
    hist, xs, ln, sm, am = [], [], [], [], []
    t1 = time.time()
    for c in range(max_cycles):
        x = mg.cycle(len(mg.systems) - 1, x, f)
        ocmg.pressure_mean_projection(fine, x)
        rel = np.linalg.norm(fine.residual(x, f)) / nf
        hist.append(rel)
        xs.append(x[idx].copy())
        ln.append(fine.norm(x))
        sm.append(float(np.sum(x)))
        am.append(float(np.abs(x).max()))
        print(f"{tag} cycle {c + 1}: {rel:.9e}  ({time.time() - t1:.0f} s)",
              flush=True)
        if rel <= 1e-8:
            break
    np.savez_compressed(
        os.path.join(OUT, f"full_{tag}.npz"), hist=np.array(hist), idx=idx,
        xs=np.array(xs), lnorm=np.array(ln), sum=np.array(sm),
        absmax=np.array(am), norm_f=np.array(nf), n=np.array(fine.n),
        counts=np.array(fine.layout.counts),
        setup_s=np.array(setup), solve_s=np.array(time.time() - t1))
    print(tag, "cycles", len(hist), "final", hist[-1], "setup", setup,
          "solve", time.time() - t1, flush=True)


if __name__ == "__main__":
    what = sys.argv[1]
    if what == "c2":
        for alpha, at in ((1.0, "1"), (1e-4, "1e-4"), (1e-8, "1e-8")):
            for sm, st in (("lsgs", "lsgs"), ("normal", "normal")):
                run("poisson", 10, alpha, sm, "v", 2, 0, f"c2_a{at}_{st}")
    elif what == "c3":
        run("poisson", 12, 1e-6, "lsgs", "w", 1, 0, "c3_lsgs", add_sine=True,
            n_per_field=1024)
    elif what == "c5":
        at = sys.argv[2]
        run("stokes", 10, float(at), "lsgs", "v", 1, 1, f"c5_a{at}_lsgs",
            n_per_field=256)
    elif what == "small":
        # quick self-check of this script against the committed L6 fixture
        run("poisson", 6, 1e-6, "lsgs", "v", 1, 0, "selfcheck_c1")
    else:
        raise SystemExit(f"unknown target {what}")
