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
t = buf.reshape(nb, niter, nw, 3).astype(np.int64)
t0 = t[..., 0][t[..., 0] > 0].min()
t[..., 0] -= t0
t[:, :, 0, 1] -= t0
t[:, :, 8, 1] = np.where(t[:, :, 8, 1] > 0, t[:, :, 8, 1] - t0, 0)
names = ["chain1", "chain2", "G1", "u", "G2", "r", "loader", "writer", "scout"]
print(f"k={k} nb={nb} niter={niter} total {(t.max())/1e3:.1f} us")
for b in (0, nb // 2, nb - 1):
    dur = t[b, :, :, 2] / 1.965   # SM cycles -> ns at 1965 MHz
    mid = t[b, :, :, 1] / 1.965
    it_len = np.diff(t[b, :, 0, 0])
    print(f"band {b}: start {t[b,0,0,0]/1e3:.1f} us end {t[b,-1,:,0].max()/1e3:.1f} us;"
          f" iteration period median {np.median(it_len)/1e3:.2f} us")
    for w in range(nw):
        d = dur[:, w]
        d = d[d > 0]
        if d.size:
            print(f"   {names[w]:7s} median {np.median(d)/1e3:7.2f} us  max {d.max()/1e3:7.2f} us"
                  f"  (issue part median {np.median(mid[:, w])/1e3:.2f} us)")
# band-to-band start offset
starts = t[:, 0, 0, 0]
print("band start offsets (us):", np.round(np.diff(starts)[:8] / 1e3, 2), "...")
np.save(f"gpurun_out/wfprof_k{k}.npy", t)
# hand-off latency: band b's iteration c+1 may start once band b-1 finished
# c + DOWN (its iteration c + DOWN + 1 has started): the gap between the two
DOWN = 9
gaps = []
for b in range(1, nb):
    s_b = t[b, :, 0, 0]
    s_p = t[b - 1, :, 0, 0]
    c = np.arange(5, niter - DOWN - 2)
    gaps.append(s_b[c + 1] - s_p[c + DOWN + 1])
gaps = np.concatenate(gaps)
print("start(b, c+1) - start(b-1, c+DOWN+1) us: median %.2f p10 %.2f p90 %.2f" %
      (np.median(gaps) / 1e3, np.percentile(gaps, 10) / 1e3, np.percentile(gaps, 90) / 1e3))
per = np.diff(t[:, :, 0, 0], axis=1)
print("iteration period us: median %.2f p90 %.2f" % (np.median(per) / 1e3, np.percentile(per, 90) / 1e3))
# flag hand-off: band b's scout saw band b-1's counter (need = c + DOWN + 1
# iterations done) at scout[c][1]; band b-1 issued that release at
# chain1[c + DOWN][1] (warp 0's mid slot holds the release time in ns)
lat = []
for b in range(1, nb):
    for c in range(20, niter - DOWN - 2):
        seen = t[b, c, 8, 1]
        rel = t[b - 1, c + DOWN, 0, 1]
        if seen > 0 and rel > 0:
            lat.append(int(seen) - int(rel))
lat = np.array(lat)
if lat.size:
    print("release -> seen by the band below (ns): median %d p10 %d p90 %d; "
          "negative = seen before the release time was stamped" %
          (np.median(lat), np.percentile(lat, 10), np.percentile(lat, 90)))
