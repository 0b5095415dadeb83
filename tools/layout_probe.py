"""Physical layout of a species after k pushes (continuous voxel order vs
in-place): distinct voxels per 8-record lane run, the fraction of records
whose voxel differs from their run's first, and monotonicity."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_13133_b200 as pic  # noqa: E402
from bench import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "thermal"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
for vo in (1, 0):
    cfg = CONFIGS[name]
    g = pic.make_grid(cfg["n"], cfg["h"], dt=cfg["dt"])
    ctx = pic.Context(g)
    ctx._set_voxel_order(bool(vo))
    sids = []
    for nm, q, m, ppc, uth, drift in cfg["species"]:
        sid = ctx.add_species(nm, q, m, ppc * g.interior)
        ctx.load_synthetic(sid, ppc, uth, drift, seed=7)
        sids.append(sid)
    for _ in range(steps):
        ctx.step()
    pos, mom, lidx = ctx._download_physical(0)
    v = pos[:, 3].view(np.int32)
    n = v.size // 256 * 256
    runs = v[:n].reshape(-1, 8)
    distinct = np.array([len(set(r)) for r in runs[:200000]])
    out = (runs != runs[:, :1]).mean()
    print(f"vo={vo} steps={steps}: distinct/run {distinct.mean():.3f}, outliers {out:.4f}, "
          f"nondecreasing {np.mean(v[1:] >= v[:-1]):.4f}, first ids {v[:12].tolist()}")
    ctx.close()


def key_cover(v, nslots):
    """Fraction of records outside the first nslots distinct keys (memory
    order: first, first different, last different) of their 8-record run,
    and the fraction of 256-record slices with at least one."""
    n = v.size // 256 * 256
    runs = v[:n].reshape(-1, 8)
    first = runs[:, :1]
    d = runs != first
    idx_first_diff = np.where(d.any(1), d.argmax(1), 0)
    c1 = np.where(d.any(1), runs[np.arange(len(runs)), idx_first_diff], -1)
    idx_last_diff = np.where(d.any(1), 7 - d[:, ::-1].argmax(1), 0)
    c2 = np.where(d.any(1), runs[np.arange(len(runs)), idx_last_diff], -1)
    keys = [first[:, 0], c1, c2][:nslots]
    inside = np.zeros_like(runs, dtype=bool)
    for k in keys:
        inside |= runs == k[:, None]
    outside = ~inside
    per_slice = outside.reshape(-1, 32 * 8).any(1)
    return outside.mean(), per_slice.mean()


if __name__ == "__main__" and len(sys.argv) > 3:
    cfg = CONFIGS[name]
    g = pic.make_grid(cfg["n"], cfg["h"], dt=cfg["dt"])
    ctx = pic.Context(g)
    sids = []
    for nm, q, m, ppc, uth, drift in cfg["species"]:
        sid = ctx.add_species(nm, q, m, ppc * g.interior)
        ctx.load_synthetic(sid, ppc, uth, drift, seed=7)
        sids.append(sid)
    for _ in range(steps):
        ctx.step()
    for s in sids:
        pos, mom, lidx = ctx._download_physical(s)
        v = pos[:, 3].view(np.int32)
        print(f"species {s}: outside 1 key {key_cover(v, 1)}, 2 keys {key_cover(v, 2)}, 3 keys {key_cover(v, 3)}")
