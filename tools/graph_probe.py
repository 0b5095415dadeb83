"""Per-step device time of the graphed step on a bench deck (sort cadence
of the bench), with the graph capture / replay counts: finds steps that
fall off the graph path.  python tools/graph_probe.py CONFIG STEPS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_13133_b200 as pic  # noqa: E402
from bench import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "thermal"
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 60
cfg = CONFIGS[name]
g = pic.make_grid(cfg["n"], cfg["h"], dt=cfg["dt"])
ctx = pic.Context(g)
sids = []
for nm, q, m, ppc, uth, drift in cfg["species"]:
    sid = ctx.add_species(nm, q, m, ppc * g.interior)
    ctx.load_synthetic(sid, ppc, uth, drift, seed=7)
    sids.append(sid)
for s in sids:
    ctx.sort_particles(s)
out = []
for k in range(1, nsteps + 1):
    st0 = ctx._graph_stats()
    ctx.event(0)
    ctx.step()
    ctx.event(1)
    ms = ctx.elapsed_ms(0, 1)
    st1 = ctx._graph_stats()
    kind = "R" if st1[1] > st0[1] else ("C" if st1[0] > st0[0] else "P")
    out.append(f"{k}:{ms:.3f}{kind}")
    if k % cfg["sort_interval"] == 0:
        for s in sids:
            ctx.sort_particles(s)
print(name, " ".join(out))
print("graph stats (captures, replays, plain):", ctx._graph_stats())
