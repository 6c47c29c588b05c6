"""Exact-order sweeps of the small structured levels: the dense-map path
(wavefront mode, k <= 5) against the reference-mode sweep, and timings
(dev tool).  python scripts/dense_check.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1502_03917_b200 as P  # noqa: E402

for k in (3, 4, 5, 6):
    s = P.build_poisson_system(k, 1e-6)
    g = torch.Generator(device="cuda").manual_seed(k)
    x0 = torch.rand(s.n, dtype=torch.float64, device="cuda", generator=g) - .5
    r0 = torch.rand(s.n, dtype=torch.float64, device="cuda", generator=g) - .5
    out = {}
    for mode in ("reference", "wavefront"):
        st = P.make_smoother(s, "slsgs", gs_mode=mode)
        x, r = x0.clone(), r0.clone()
        for _ in range(3):
            st.sweep(x, r)
        out[mode] = (x, r)
        reps = 50
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            st.sweep(x, r)
        e1.record()
        e1.synchronize()
        print(f"k={k} {mode:9s} {e0.elapsed_time(e1) / reps / 2 * 1e3:7.1f} us per sweep")
    xr, rr = out["reference"]
    xw, rw = out["wavefront"]
    ex = float((xw - xr).abs().max() / xr.abs().max())
    er = float((rw - rr).abs().max() / rr.abs().max())
    print(f"k={k} wavefront vs reference: x {ex:.2e}  r {er:.2e}")
