"""Per-species push kernel times (device events) inside the step sequence
of the bench workload, over `steps` steps with the blocked sort every
sort_interval — to compare the in-loop duration of one push launch with
ncu's isolated replay of the same launch.

    python tools/kernel_probe.py [config] [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_13133_b200 as pic  # noqa: E402
from bench import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "two_stream"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 24
cfg = CONFIGS[name]
g = pic.make_grid(cfg["n"], cfg["h"], dt=cfg["dt"])
ctx = pic.Context(g)
sids = []
for sname, q, m, ppc, uth, drift in cfg["species"]:
    sid = ctx.add_species(sname, q, m, ppc * g.interior)
    ctx.load_synthetic(sid, ppc, uth, drift, seed=1234)
    sids.append(sid)
for s in sids:
    ctx.sort_particles(s)
ctx.synchronize()
for st in range(1, steps + 1):
    ctx.clear_accumulator()
    ctx.clear_currents()
    ctx.load_interpolators()
    ctx.event(0)
    for i, s in enumerate(sids):
        ctx.advance_p(s)
        ctx.event(i + 1)
    ctx.ghost_fold_currents()
    ctx.advance_b(0.5)
    ctx.ghost_sync_fields()
    ctx.unload_advance_e()
    ctx.ghost_sync_fields()
    ctx.advance_b(0.5)
    ctx.ghost_sync_fields()
    ctx.synchronize()
    t = [ctx.elapsed_ms(i, i + 1) for i in range(len(sids))]
    print(f"step {st:3d} stale {(st - 1) % cfg['sort_interval']:2d} push ms " + " ".join(f"{x:7.3f}" for x in t),
          flush=True)
    if st % cfg["sort_interval"] == 0:
        for s in sids:
            ctx.sort_particles(s)
ctx.synchronize()
