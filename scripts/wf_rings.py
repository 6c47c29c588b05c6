"""Check wavefront ring contents (p1, u, p2) of one forward sweep (debug)."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_1502_03917_b200 as P
from paper_1502_03917_b200 import _lib

lib = _lib.load()
fn = lib.ocmg__debug_wf_ring
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
               ctypes.POINTER(ctypes.c_int64)]

def ring(s, which):
    cnt = ctypes.c_int64()
    _lib.check(fn(s.handle, which, None, ctypes.byref(cnt)))
    t = torch.empty(cnt.value, dtype=torch.float64, device="cuda")
    _lib.check(fn(s.handle, which, _lib.dptr(t), ctypes.byref(cnt)))
    return t.cpu().numpy()

k = int(sys.argv[1]) if len(sys.argv) > 1 else 6
s = P.build_poisson_system(k, 1e-6)
n1 = 2 ** k + 1; N = n1 * n1; REAL = 29; nb = (n1 + REAL - 1) // REAL; RW = 512
g = torch.Generator(device="cuda").manual_seed(k)
x0 = torch.rand(s.n, dtype=torch.float64, device="cuda", generator=g) - .5
f = torch.rand(s.n, dtype=torch.float64, device="cuda", generator=g)
r0 = s.residual(x0, f)
ref = P.make_smoother(s, "lsgs", gs_mode="reference")
xr, rr = x0.clone(), r0.clone(); ref.sweep(xr, rr)
wf = P.make_smoother(s, "lsgs", gs_mode="wavefront")
xw, rw = x0.clone(), r0.clone(); wf.sweep(xw, rw)
torch.cuda.synchronize()
p_ref = (xr - x0).cpu().numpy()
p1 = p_ref[:N].reshape(n1, n1); p2 = p_ref[N:].reshape(n1, n1)
xu = x0.clone(); xu[:N] += torch.from_numpy(p_ref[:N]).cuda()
u_ref = s.residual(xu, f).cpu().numpy()     # residual after the state chain
R1, R2, RU = ring(s, 0), ring(s, 1), ring(s, 2)
R1 = R1.reshape(nb, 32, RW); R2 = R2.reshape(nb, 32, RW)
RU = RU.reshape(nb, 2, 32, RW)
for name, R, ref_arr in (("p1", R1, [p1]), ("p2", R2, [p2]),
                         ("u", RU, [u_ref[:N].reshape(n1, n1), u_ref[N:].reshape(n1, n1)])):
    worst = []
    for b in range(nb):
        for i in range(REAL):
            iy = REAL * b + i
            if iy >= n1: continue
            for fld, arr in enumerate(ref_arr):
                got = R[b, fld, i] if name == "u" else R[b, i]
                cols = np.arange(max(0, n1 - 448), n1)
                d = np.abs(got[cols & (RW - 1)] - arr[iy, cols]) / (np.abs(arr).max())
                bad = np.flatnonzero(d > 1e-12)
                if bad.size:
                    worst.append((b, i, fld, cols[bad[:6]].tolist(), float(d.max())))
    print(name, "bad rows:", len(worst))
    for w in worst[:8]:
        print("   band %d row %d field %d cols %s max %.2e" % w)
