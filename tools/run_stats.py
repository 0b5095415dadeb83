"""Run statistics of the push's lane runs (8 consecutive particles of a
voxel-sorted store) as the store ages: distinct voxels per run, and the
fraction of particles outside the two seeded slots (advance_p_lean's seeding
rule), per deck and staleness.  Diagnostic for DESIGN.md §5."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_13133_b200 as pic  # noqa: E402
from bench import CONFIGS  # noqa: E402


def seed_slots(run):
    first = run[0]
    other = [k for k in run if k != first]
    if not other:
        return first, -1
    c1, c2 = other[0], other[-1]
    n1, n2 = run.count(c1), run.count(c2)
    return first, (c2 if n2 > n1 else c1)


for name in sys.argv[1].split(",") if len(sys.argv) > 1 else ["two_stream", "thermal"]:
    cfg = CONFIGS[name]
    g = pic.make_grid(64, cfg["h"], dt=cfg["dt"])
    ctx = pic.Context(g)
    sids = []
    for sname, q, m, ppc, uth, drift in cfg["species"]:
        sid = ctx.add_species(sname, q, m, ppc * g.interior)
        ctx.load_synthetic(sid, ppc, uth, drift, seed=7)
        sids.append(sid)
    for step in range(20):
        if step in (0, 1, 5, 10, 19):
            for sid in sids[:1]:
                _, ids = ctx.download_species(sid)
                runs = ids[: (ids.size // 8) * 8].reshape(-1, 8)
                nd = np.array([len(set(r.tolist())) for r in runs[:200000]])
                out = 0
                for r in runs[:50000]:
                    a, b = seed_slots(r.tolist())
                    out += sum(1 for k in r.tolist() if k != a and k != b)
                print(f"{name} stale {step}: distinct voxels per run mean {nd.mean():.2f} "
                      f"hist {np.bincount(nd, minlength=6)[1:6] / nd.size}, outliers {out / (50000 * 8):.3f}",
                      flush=True)
        ctx.step()
    ctx.close()
