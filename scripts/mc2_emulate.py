"""CPU emulation of k_p1_mc_roll's schedule (dev tool): the own masks, the
window inheritance, ring slots, phase duties and tile decomposition, line by
line as in ocmg_p1_mc2.cuh, against a plain colour-by-colour sweep.  The
arithmetic is a stand-in (position-dependent coefficients, zero for absent
neighbours); what is checked is the order and the data movement.

python scripts/mc2_emulate.py [n1] [W] [nseg_total] [forward]
"""
import sys

import numpy as np

NC, H, GL, STRIDE, AHEAD, RETIRE, RING, NWARP = 7, 14, 8, 234, 7, 21, 33, 21
OFF = [(-1, -1), (0, -1), (-1, 0), (0, 0), (1, 0), (0, 1), (1, 1)]


def coef(x, y, n1, f):
    rng = np.random.default_rng(1000 * f + 7 * min(x, 3) + 11 * min(y, 3)
                                + 13 * min(n1 - 1 - x, 3) + 17 * min(n1 - 1 - y, 3))
    w = rng.uniform(0.1, 1, 14)
    a = rng.uniform(0.1, 1, 14)
    for d, (dx, dy) in enumerate(OFF):
        if not (0 <= x + dx < n1 and 0 <= y + dy < n1):
            w[d] = w[7 + d] = a[d] = a[7 + d] = 0.0
    return w, a, 1.0 / (1.0 + w.sum())


def node_update(v, c):
    w, a, inv = c
    p = (sum(w[d] * v[d][0] for d in range(7)) + sum(w[7 + d] * v[d][1] for d in range(7))) * inv
    for d in range(7):
        v[d] = (v[d][0] - a[d] * p, v[d][1] - a[7 + d] * p)
    return p


def reference(n1, x, r, fwd):
    x, r = x.copy(), r.copy()
    for b in range(7):
        c = b if fwd else 6 - b
        for iy in range(n1):
            for ix in range(n1):
                if (ix + 2 * iy) % 7 != c:
                    continue
                v = []
                for dx, dy in OFF:
                    xx, yy = ix + dx, iy + dy
                    v.append((r[0, yy, xx], r[1, yy, xx]) if 0 <= xx < n1 and 0 <= yy < n1 else (0.0, 0.0))
                fs = (0, 1) if fwd else (1, 0)
                for f in fs:
                    p = node_update(v, coef(ix, iy, n1, f))
                    x[f, iy, ix] += p
                for d, (dx, dy) in enumerate(OFF):
                    xx, yy = ix + dx, iy + dy
                    if 0 <= xx < n1 and 0 <= yy < n1:
                        r[:, yy, xx] = v[d]
    return x, r


def cta(n1, W, nstrips, base, rem, bid, rin, rout, x, fwd, y_begin, y_end):
    strip, seg = bid % nstrips, bid // nstrips
    nseg = base + (1 if strip < rem else 0)
    if seg >= nseg:
        return
    rows = y_end - y_begin
    seg_h = (rows + nseg - 1) // nseg
    X0, X1 = strip * n1 // nstrips, (strip + 1) * n1 // nstrips
    Y0 = y_begin + seg * seg_h
    Y1 = min(y_end, Y0 + seg_h)
    if Y0 >= Y1:
        return
    xl, xr = max(0, X0 - H), min(n1, X1 + H)
    Ylo, Yhi = max(0, Y0 - H), min(n1, Y1 + H)
    rmax = min(Yhi, n1 - 1)
    ring = np.full((RING, STRIDE, 2), np.nan)
    dring = np.full((RING, W, 2), np.nan)

    def load_row(ry):
        row = Ylo + ry
        for lc in range(STRIDE):
            gx = xl - GL + lc
            ok = xl <= gx < xr and 0 <= row <= rmax
            ring[(ry + 1) % RING, lc] = rin[:, row, gx] if ok else 0.0

    for ry in range(-1, AHEAD):
        load_row(ry)
    st = [dict(k=0, ry=w, v=[(np.nan, np.nan)] * 7) for w in range(NWARP)]
    lanes = [[dict(v=[(np.nan, np.nan)] * 7) for _ in range(32)] for _ in range(NWARP)]
    S_end = (Y1 - 1 - Ylo) + RETIRE + 1
    for S in range(S_end):
        stores = []   # (kind, slot, col, value): applied at the barrier (checks independence)
        touched = set()

        def put(kind, slot, col, val):
            key = (kind, slot, col)
            assert key not in touched, ("two writers in one step", key, S)
            touched.add(key)
            stores.append((kind, slot, col, val))

        reads = set()

        def get(slot, col):
            reads.add((0, slot, col))
            return tuple(ring[slot, col])

        for w in range(NWARP):
            ph = (S + 3 - w % 3) % 3
            W_ = st[w]
            if ph == 0:
                if S < w:
                    continue
                k, ry = W_["k"], W_["ry"]
                y = Ylo + ry
                rowact = y < Yhi
                introw = 3 <= y <= n1 - 4
                for lane in range(32):
                    L = lanes[w][lane]
                    xs0 = xl - (xl + 2 * y) % 7 + 7 * lane
                    if k == 0:
                        cl = max(xl, 3) if introw else xl
                        cr = min(xr, n1 - 3) if introw else xr
                        if fwd:
                            qlo = cl - xs0
                            qhi = min(cr - 1 - xs0, xs0 - X0 + 13, (X1 + 12 - xs0 + 300) // 3 - 100)
                        else:
                            qlo = xs0 + 6 - (cr - 1)
                            qhi = min(xs0 + 6 - cl, X1 + 6 - xs0, (xs0 + 19 - X0 + 300) // 3 - 100)
                        qhi = min(qhi, (y - Y0 + 13 + 300) // 2 - 150, (Y1 + 12 - y + 300) // 2 - 150)
                        qlo, qhi = max(qlo, 0), min(qhi, 6)
                        L["mask2"] = (((2 << qhi) - (1 << qlo)) << 1) if (rowact and qhi >= qlo) else 0
                    if not rowact:
                        continue
                    m2 = L["mask2"]
                    own, prev, nxt = (m2 >> (k + 1)) & 1, (m2 >> k) & 1, (m2 >> (k + 2)) & 1
                    xc = xs0 + (k if fwd else 6 - k)
                    col = xc - xl + GL
                    sl = ry % RING
                    sB, sC, sU = sl, (sl + 1) % RING, (sl + 2) % RING
                    v = L["v"]
                    addr = [(sB, col - 1), (sB, col), (sC, col - 1), (sC, col), (sC, col + 1),
                            (sU, col), (sU, col + 1)]
                    if introw:
                        if fwd:
                            v[0], v[2], v[3], v[5] = v[1], v[3], v[4], v[6]
                            new, rest = (1, 4, 6), (0, 2, 3, 5)
                        else:
                            v[6], v[4], v[3], v[1] = v[5], v[3], v[2], v[0]
                            new, rest = (0, 2, 5), (1, 3, 4, 6)
                        if own:
                            for d in new:
                                v[d] = get(*addr[d])
                            if not prev:
                                for d in rest:
                                    v[d] = get(*addr[d])
                            # colour check + exact domain class
                            assert (xc + 2 * y) % 7 == (k if fwd else 6 - k)
                            assert 3 <= xc <= n1 - 4
                    else:
                        if own:
                            for d in range(7):
                                v[d] = get(*addr[d])
                    if own:
                        f0, f1 = (0, 1) if fwd else (1, 0)
                        pa = node_update(v, coef(xc, y, n1, f0))
                        pb = node_update(v, coef(xc, y, n1, f1))
                        if introw:
                            if fwd:
                                out, outrest = (0, 2, 5), (1, 3, 4, 6)
                            else:
                                out, outrest = (1, 4, 6), (0, 2, 3, 5)
                            for d in out:
                                put(0, addr[d][0], addr[d][1], v[d])
                            if not nxt:
                                for d in outrest:
                                    put(0, addr[d][0], addr[d][1], v[d])
                        else:
                            for d in range(7):
                                put(0, addr[d][0], addr[d][1], v[d])
                        if Y0 <= y < Y1 and X0 <= xc < X1:
                            put(1, sC, xc - X0, (pa, pb) if fwd else (pb, pa))
                W_["k"] += 1
                if W_["k"] == NC:
                    W_["k"] = 0
                    W_["ry"] += NWARP
            elif ph == 1 and w < 3:
                R = Ylo + S - RETIRE
                if Y0 <= R < Y1:
                    sl = (S - RETIRE + 1) % RING
                    for gt in range(X1 - X0):
                        rv = ring[sl, X0 - xl + GL + gt]
                        dv = dring[sl, gt]
                        assert not np.isnan(dv).any(), ("delta missing", R, X0 + gt)
                        rout[:, R, X0 + gt] = rv
                        x[:, R, X0 + gt] += dv
                        dring[sl, gt] = np.nan
            elif ph == 2 and w < 3:
                if Ylo + S + AHEAD <= Yhi:
                    # loads land before their first use; emulate as immediate
                    # but check the slot's previous row has retired
                    pass
                for lane in range(2 * NC):
                    side, q = divmod(lane, NC)
                    rq = S - 3 * q
                    yb = Ylo + rq
                    bside = (xl == 0) if side == 0 else (xr == n1)
                    colour = q if fwd else NC - 1 - q
                    mg = 2 * (NC - 1 - q) + 1
                    c0 = 0 if side == 0 else n1 - 3
                    ob = (colour - 2 * yb - c0) % 7
                    xb = c0 + ob
                    if (bside and rq >= 0 and ob < 3 and 3 <= yb <= n1 - 4
                            and max(Ylo, Y0 - mg) <= yb < min(Yhi, Y1 + mg)
                            and max(xl, X0 - mg) <= xb < min(xr, X1 + mg)):
                        col = xb - xl + GL
                        sl = rq % RING
                        sB, sC, sU = sl, (sl + 1) % RING, (sl + 2) % RING
                        addr = [(sB, col - 1), (sB, col), (sC, col - 1), (sC, col), (sC, col + 1),
                                (sU, col), (sU, col + 1)]
                        u = [get(*a) for a in addr]
                        f0, f1 = (0, 1) if fwd else (1, 0)
                        pa = node_update(u, coef(xb, yb, n1, f0))
                        pb = node_update(u, coef(xb, yb, n1, f1))
                        for d in range(7):
                            put(0, addr[d][0], addr[d][1], u[d])
                        if Y0 <= yb < Y1 and X0 <= xb < X1:
                            put(1, sC, xb - X0, (pa, pb) if fwd else (pb, pa))
        # a step's stores touch nothing another vertex of the step read
        for kind, slot, col, val in stores:
            if kind == 0:
                ring[slot, col] = val
            else:
                dring[slot, col] = val
        if Ylo + S + AHEAD <= Yhi:
            load_row(S + AHEAD)


def main():
    n1 = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    W = int(sys.argv[2]) if len(sys.argv) > 2 else 171
    total = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    fwd = (int(sys.argv[4]) if len(sys.argv) > 4 else 1) != 0
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, (2, n1, n1))
    r = rng.uniform(-1, 1, (2, n1, n1))
    xr_, rr_ = reference(n1, x, r, fwd)
    nstrips = (n1 + W - 1) // W
    total = max(total, nstrips)
    base, rem = total // nstrips, total % nstrips
    grid = nstrips * (base + (1 if rem else 0))
    rout = np.full_like(r, np.nan)
    x2 = x.copy()
    for bid in range(grid):
        cta(n1, W, nstrips, base, rem, bid, r, rout, x2, fwd, 0, n1)
    print("n1", n1, "W", W, "grid", grid, "fwd", fwd,
          "max|dr|", np.nanmax(np.abs(rout - rr_)), "nan", int(np.isnan(rout).sum()),
          "max|dx|", np.abs(x2 - xr_).max())


main()
