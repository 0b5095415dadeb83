"""Per-step push-phase rate of a bench deck (fresh synthetic load, sort
cadence of the bench), for the continuous-voxel-order A/B and ncu launch
lists: python tools/order_probe.py CONFIG STEPS [voxel_order 0|1]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_13133_b200 as pic  # noqa: E402
from bench import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "weak"
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
vo = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cfg = CONFIGS[name]
g = pic.make_grid(cfg["n"], cfg["h"], dt=cfg["dt"])
ctx = pic.Context(g)
ctx._set_voxel_order(bool(vo))
sids = []
for nm, q, m, ppc, uth, drift in cfg["species"]:
    sid = ctx.add_species(nm, q, m, ppc * g.interior)
    ctx.load_synthetic(sid, ppc, uth, drift, seed=7)
    sids.append(sid)
npart = sum(ctx.species_count(s) for s in sids)
ctx.phase_timing(True)
out = []
for k in range(nsteps):
    ctx.phase_timings(reset=True)
    ctx.step()
    ph = ctx.phase_timings(reset=True)
    if (k + 1) % cfg["sort_interval"] == 0:
        for s in sids:
            ctx.sort_particles(s)
    out.append(f"{k + 1}:{npart / (ph['push'] / 1e3) / 1e10:.2f}")
ctx.synchronize()
print(name, f"voxel_order={vo}", "push rate (1e10/s) per step:", " ".join(out))
