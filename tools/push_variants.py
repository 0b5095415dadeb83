"""Times the advance_p strategies on a bench workload (device events).

Each (staleness, variant) cell starts from a fresh synthetic load (voxel
sorted), advances `stale` steps with the default variant, then times 3 steps
with the variant under test, so every variant sees the same particle order."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_13133_b200 as pic  # noqa: E402
from bench import CONFIGS  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "two_stream"
variants = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 3, 10, 11, 12]
stales = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0, 10]
# "resort": sort the stores after the stale steps (run with PIC_SORT_DEFER=0),
# so the timed steps see a fresh order at a later physical time
resort = len(sys.argv) > 4 and sys.argv[4] == "resort"
cfg = CONFIGS[cfg_name]
g = pic.make_grid(cfg["n"], cfg["h"], dt=cfg["dt"])
ctx = pic.Context(g)
sids = []
for name, q, m, ppc, uth, drift in cfg["species"]:
    sids.append(ctx.add_species(name, q, m, ppc * g.interior))
res = {}
for stale in stales:
    for var in variants:
        for sid, (name, q, m, ppc, uth, drift) in zip(sids, cfg["species"]):
            ctx.load_synthetic(sid, ppc, uth, drift, seed=7)
        npart = sum(ctx.species_count(s) for s in sids)
        ctx._set_push_variant(2)
        for _ in range(stale):
            ctx.step()
        if resort:
            for sid in sids:
                ctx.sort_particles(sid)
        ctx._set_push_variant(var)
        ctx.phase_timing(True)
        ctx.phase_timings(reset=True)
        k = 3
        for _ in range(k):
            ctx.step()
        ph = ctx.phase_timings(reset=True)
        ctx.phase_timing(False)
        rate = npart * k / (ph["push"] / 1e3)
        res[f"stale{stale}_v{var}"] = rate
        print(f"stale={stale:2d} variant={var:2d} push={ph['push'] / k:8.3f} ms/step  rate={rate:.3e}", flush=True)
ctx.synchronize()
print(json.dumps(res))
