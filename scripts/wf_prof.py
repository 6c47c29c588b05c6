"""Per-warp stage timing of one wavefront sweep (needs the -DOCMG_WF_PROFILE build)."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_1502_03917_b200 as P
from paper_1502_03917_b200 import _lib

k = int(sys.argv[1]) if len(sys.argv) > 1 else 12
s = P.build_poisson_system(k, 1e-6)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand(s.n, dtype=torch.float64, device="cuda", generator=g) - .5
r = s.residual(x, torch.rand(s.n, dtype=torch.float64, device="cuda", generator=g))
st = P.make_smoother(s, "lsgs", gs_mode="wavefront")
for _ in range(3):
    st.sweep(x, r)
torch.cuda.synchronize()
lib = _lib.load()
fn = lib.ocmg__debug_wf_prof
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]
dims = (ctypes.c_int64 * 4)()
_lib.check(fn(s.handle, None, dims))
nb, niter, nw, cnt = dims
buf = np.zeros(cnt, dtype=np.uint64)
_lib.check(fn(s.handle, buf.ctypes.data_as(ctypes.c_void_p), dims))
t = buf.reshape(nb, niter, nw, 2).astype(np.int64)
t0 = t[t > 0].min()
t = t - t0
names = ["chain1", "chain2", "scout"] + [f"{s}{i}" for s in ("G1_", "u_", "G2_", "r_") for i in range(4)]
print(f"k={k} nb={nb} niter={niter} total {(t.max())/1e3:.1f} us")
for b in (0, nb // 2, nb - 1):
    dur = t[b, :, :, 1] - t[b, :, :, 0]
    it_len = np.diff(t[b, :, 0, 0])
    print(f"band {b}: start {t[b,0,0,0]/1e3:.1f} us end {t[b,-1,:,1].max()/1e3:.1f} us;"
          f" iteration period median {np.median(it_len)/1e3:.2f} us")
    for w in range(nw):
        d = dur[:, w]
        d = d[d > 0]
        if d.size:
            print(f"   {names[w]:7s} median {np.median(d)/1e3:7.2f} us  max {d.max()/1e3:7.2f} us")
# band-to-band start offset
starts = t[:, 0, 0, 0]
print("band start offsets (us):", np.round(np.diff(starts)[:8] / 1e3, 2), "...")
