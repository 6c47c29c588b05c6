"""Exact-order (wavefront) sweep: time per level and agreement with the
bitwise reference-order path.  python scripts/wf_time.py [k ...]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1502_03917_b200 as P  # noqa: E402

levels = [int(a) for a in sys.argv[1:]] or [9, 10, 11, 12]
for k in levels:
    s = P.build_poisson_system(k, 1e-6)
    g = torch.Generator(device="cuda").manual_seed(k)
    x0 = torch.rand(s.n, dtype=torch.float64, device="cuda", generator=g) - 0.5
    r0 = s.residual(x0, torch.rand(s.n, dtype=torch.float64, device="cuda", generator=g))
    res = {}
    for mode in ("wavefront", "reference"):
        st = P.make_smoother(s, "lsgs", gs_mode=mode)
        for order in ("forward", "backward"):
            x, r = x0.clone(), r0.clone()
            P.lsgs_sweep(st, x, r, order=order)
            P.lsgs_sweep(st, x, r, order=order)
            res[mode, order] = (x, r)
    for order in ("forward", "backward"):
        xw, rw = res["wavefront", order]
        xr, rr = res["reference", order]
        ex = float((xw - xr).abs().max() / xr.abs().max())
        er = float((rw - rr).abs().max() / rr.abs().max())
        print(f"k={k} {order}: x rel {ex:.2e}  r rel {er:.2e}", flush=True)
    st = P.make_smoother(s, "lsgs", gs_mode="wavefront")
    x, r = x0.clone(), r0.clone()
    for _ in range(3):
        st.sweep(x, r)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n):
        st.sweep(x, r)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"k={k} n={s.n}: wavefront sweep {ms:.3f} ms = {s.n / ms / 1e6:.2f} G DOF/s,"
          f" {32 * s.n / ms / 1e6 / 6549.8 * 100:.1f}% of HBM", flush=True)
