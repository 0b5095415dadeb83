"""Run lengths of the sort permutation (consecutive source indices) after k
steps of a bench deck on 64^3 (how contiguous the deferred gather is)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_13133_b200 as pic  # noqa: E402
from bench import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "two_stream"
cfg = CONFIGS[name]
g = pic.make_grid(64, cfg["h"], dt=cfg["dt"])
ctx = pic.Context(g)
sids = []
for sname, q, m, ppc, uth, drift in cfg["species"]:
    sid = ctx.add_species(sname, q, m, ppc * g.interior)
    ctx.load_synthetic(sid, ppc, uth, drift, seed=7)
    sids.append(sid)
for k in range(21):
    if k in (1, 10, 20):
        _, ids = ctx.download_species(sids[0])
        perm = np.argsort(ids, kind="stable")
        d = np.diff(perm.astype(np.int64))
        starts = np.concatenate([[0], np.nonzero(d != 1)[0] + 1])
        lens = np.diff(np.concatenate([starts, [perm.size]]))
        print(f"{name} stale {k}: runs {starts.size} of {perm.size}, mean run {lens.mean():.2f}, "
              f"median {np.median(lens):.0f}, in-runs-of-1 {np.mean(lens == 1) * 100:.1f}%", flush=True)
    ctx.step()
