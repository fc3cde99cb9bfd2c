"""Grids of more than 2^31 voxels (int64 voxel indexing end to end) against the FP64 oracle.

A 2048 x 2048 x Gt grid (8.7 GB of float32) with a few hundred points, some placed next to the
far corner so that their voxels' linear indices (X Gy + Y) Gt + T exceed 2^31: the tile kernel's
epilogue (TMA tensor store for a 4-aligned G_t, warp-coalesced stores for an unaligned one; the
short-window FP32 engine's staged stores) must address them exactly.  Checked on the device at
voxels the oracle evaluates one by one (Alg. 1, `oracle.stkde_vb_voxels`): around every point,
the far corner, and random voxels."""
import numpy as np
import pytest

from parity import assert_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("eng", [2, 3], ids=["tc", "ws"])
@pytest.mark.parametrize("Gt", [520, 523], ids=["aligned", "unaligned"])
def test_grid_beyond_int32_voxels(oracle_mod, Gt, eng, monkeypatch):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    monkeypatch.setenv("STKDE_ENGINE", str(eng))
    import paper_1705_09366_b200 as S
    Gx = Gy = 2048
    assert Gx * Gy * Gt > 2 ** 31
    g = dict(x0=0.0, y0=0.0, t0=0.0, sres=1.0, tres=1.0, Gx=Gx, Gy=Gy, Gt=Gt, hs=6.0, ht=5.0)
    rng = np.random.default_rng(7)
    pts = np.concatenate([
        rng.uniform([0, 0, 0], [Gx, Gy, Gt], size=(200, 3)),
        rng.uniform([Gx - 12, Gy - 12, Gt - 10], [Gx, Gy, Gt], size=(60, 3)),   # near the far corner
    ]).astype(np.float32)
    dev = torch.device("cuda", 0)
    t = torch.from_numpy(pts).to(dev)
    with S.Plan(max_n=len(pts), device=0, **g) as p:
        assert p.info()["engine"] == eng
        out = p.compute(t)
        torch.cuda.synchronize()
        p.check()
    # voxels to check: a 7 x 7 x 5 block around each point, the far corner block, random voxels
    vox = []
    for x, y, tt in pts[::3]:
        X, Y, T = int(x), int(y), int(tt)
        for dx in range(-3, 4):
            for dy in range(-3, 4):
                for dt in range(-2, 3):
                    a, b, c = X + dx, Y + dy, T + dt
                    if 0 <= a < Gx and 0 <= b < Gy and 0 <= c < Gt:
                        vox.append((a * Gy + b) * Gt + c)
    for a in range(Gx - 4, Gx):
        for b in range(Gy - 4, Gy):
            for c in range(Gt - 4, Gt):
                vox.append((a * Gy + b) * Gt + c)
    vox += list(rng.integers(0, Gx * Gy * Gt, size=2000))
    vox = np.unique(np.array(vox, dtype=np.int64))
    assert vox.max() > 2 ** 31
    gpu = out.view(-1)[torch.from_numpy(vox).to(dev)].cpu().numpy()
    ref, slack, amb = oracle_mod.stkde_vb_voxels(pts, vox, **g)
    assert ref.max() > 0 and (ref[vox > 2 ** 31] > 0).any()      # the far-corner voxels are covered
    assert_parity(gpu, ref, slack, amb, what="Gt=%d beyond 2^31 voxels" % Gt)
    del out
    torch.cuda.empty_cache()
