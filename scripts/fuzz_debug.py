"""Narrow an adaptive fuzz failure to single points (development aid)."""
import sys, os
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
os.environ["STKDE_ENGINE"] = "2"
import numpy as np, torch
import oracle
import paper_1705_09366_b200 as S
from test_gpu_fuzz import draw_case, draw_bandwidths
k = int(sys.argv[1])
g, kernel, pts, cut = draw_case(k)
bw = draw_bandwidths(k, g, len(pts))
dev = torch.device("cuda", 0)
def gpu_run(p_, b_):
    with S.Plan(max_n=len(p_), kernel=kernel, device=0, **g) as p:
        out = p.compute_adaptive(torch.from_numpy(p_).to(dev), torch.from_numpy(b_).to(dev)).cpu().numpy()
        p.check()
        return out.astype(np.float64)
ref = oracle.stkde_pb_adaptive(pts, bw, kernel=kernel, **g)
out = gpu_run(pts, bw)
d = out - ref.vol
vmax = ref.vol.max()
bad = np.argwhere(np.abs(d) > 1e-5 * vmax + ref.slack)
print("case", k, g, "n", len(pts), "vmax", vmax, "bad", len(bad), "max |d|/vmax", np.abs(d).max() / vmax)
X, Y, T = bad[np.argmax(np.abs(d[tuple(bad.T)]))]
print("worst voxel", X, Y, T, out[X, Y, T], ref.vol[X, Y, T])
# points whose cylinder holds this voxel
xc = g["x0"] + (X + 0.5) * g["sres"]; yc = g["y0"] + (Y + 0.5) * g["sres"]; tc = g["t0"] + (T + 0.5) * g["tres"]
P = pts.astype(np.float64); B = bw.astype(np.float64)
inside = ((P[:, 0] - xc) ** 2 + (P[:, 1] - yc) ** 2 < B[:, 0] ** 2) & (np.abs(P[:, 2] - tc) <= B[:, 1])
idx = np.flatnonzero(inside)
print("contributing points", len(idx), "distinct", len(np.unique(pts[idx], axis=0)))
Wmax = (1 / (B[:, 0] ** 2 * B[:, 1])).max()
for i in idx[:12]:
    p1, b1 = pts[i:i + 1], bw[i:i + 1]
    r1 = oracle.stkde_pb_adaptive(p1, b1, kernel=kernel, **g).vol
    o1 = gpu_run(p1, b1)
    # the same point inside the whole set's weight scale: pair it with the heaviest-weight point
    j = int(np.argmax(1 / (B[:, 0] ** 2 * B[:, 1])))
    p2 = np.ascontiguousarray(np.stack([pts[i], pts[j]])); b2 = np.ascontiguousarray(np.stack([bw[i], bw[j]]))
    r2 = oracle.stkde_pb_adaptive(p2, b2, kernel=kernel, **g).vol
    o2 = gpu_run(p2, b2)
    print(i, pts[i], bw[i], "W/Wmax %.4f" % (1 / (B[i, 0] ** 2 * B[i, 1]) / Wmax),
          "alone: gpu %.9e ref %.9e rel %.2e" % (o1[X, Y, T], r1[X, Y, T], (o1[X, Y, T] - r1[X, Y, T]) / max(r1[X, Y, T], 1e-300)),
          "| with heaviest: max|d|/max %.2e" % (np.abs(o2 - r2).max() / r2.max()))
