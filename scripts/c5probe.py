import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1502_03917_b200 as P
for tag, alpha in (("c5_a1e-2_lsgs", 1e-2), ("c5_a1e-6_lsgs", 1e-6)):
    d = np.load(f"tests/golden/full_{tag}.npz")
    cfg = P.CycleConfig(smoother=P.SmootherKind("lsgs"), cycle="v", coarsest_level=1, gs_mode="wavefront")
    mg = P.build_solver("stokes", 10, alpha, cfg)
    f = P.baseline_rhs(mg.finest, 1)
    idx = torch.from_numpy(d["idx"]).cuda()
    x = torch.zeros_like(f)
    for c in range(len(d["hist"])):
        x, h = mg.solve_to_tolerance(f, tol=1e-8, max_cycles=1, x=x)
        xs = x[idx].cpu().numpy(); ref = d["xs"][c]
        err = np.abs(xs - ref).max() / np.abs(ref).max()
        ln = mg.finest.norm(x)
        print(tag, c, f"x {err:.2e} lnorm {abs(ln - d['lnorm'][c]) / d['lnorm'][c]:.2e} hist {h[0]:.6e} ref {d['hist'][c]:.6e}", flush=True)
    del mg
