"""Locate wavefront-vs-reference mismatches (debug aid)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1502_03917_b200 as P

for k in [int(a) for a in sys.argv[1:]] or [4, 5, 6, 7]:
    s = P.build_poisson_system(k, 1e-6)
    n1 = 2 ** k + 1
    N = n1 * n1
    g = torch.Generator(device="cuda").manual_seed(k)
    x0 = torch.rand(s.n, dtype=torch.float64, device="cuda", generator=g) - .5
    f = torch.rand(s.n, dtype=torch.float64, device="cuda", generator=g)
    r0 = s.residual(x0, f)
    res = {}
    for mode in ("wavefront", "reference"):
        st = P.make_smoother(s, "lsgs", gs_mode=mode)
        x, r = x0.clone(), r0.clone()
        P.lsgs_sweep(st, x, r, order="forward")
        res[mode] = (x.cpu().numpy(), r.cpu().numpy())
    for name, a, b in (("x", res["wavefront"][0], res["reference"][0]),
                       ("r", res["wavefront"][1], res["reference"][1])):
        d = np.abs(a - b) / np.abs(b).max()
        bad = np.flatnonzero(d > 1e-12)
        print(f"k={k} {name}: max rel {d.max():.3e}, bad {bad.size}")
        if bad.size:
            fld, v = np.divmod(bad[:12], N)
            iy, ix = np.divmod(v, n1)
            print("   first bad (field, ix, iy):", list(zip(fld, ix, iy)))
            fl, vv = np.divmod(bad, N)
            iyy, ixx = np.divmod(vv, n1)
            for ff in (0, 1):
                m = fl == ff
                if m.any():
                    print(f"   field {ff}: ix in [{ixx[m].min()},{ixx[m].max()}]"
                          f" iy in [{iyy[m].min()},{iyy[m].max()}] count {m.sum()}")
