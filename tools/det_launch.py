"""Two deterministic steps of a bench config (for an ncu launch list)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_13133_b200 as pic  # noqa: E402
from bench import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "two_stream"]
g = pic.make_grid(cfg["n"], cfg["h"], dt=cfg["dt"])
ctx = pic.Context(g)
for sname, q, m, ppc, uth, drift in cfg["species"]:
    sid = ctx.add_species(sname, q, m, ppc * g.interior)
    ctx.load_synthetic(sid, ppc, uth, drift, seed=1234)
for _ in range(2):
    ctx.step(deterministic=True)
ctx.synchronize()
