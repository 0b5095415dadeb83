"""Whole-step rate of the deterministic mode (PIC_DETERMINISTIC: staged
deposits replayed in particle order, bit-exact J) vs the fast mode on a
bench config, with the phase split."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_13133_b200 as pic  # noqa: E402
from bench import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "two_stream"
cfg = CONFIGS[name]
g = pic.make_grid(cfg["n"], cfg["h"], dt=cfg["dt"])
ctx = pic.Context(g)
sids = []
for sname, q, m, ppc, uth, drift in cfg["species"]:
    sid = ctx.add_species(sname, q, m, ppc * g.interior)
    ctx.load_synthetic(sid, ppc, uth, drift, seed=1234)
    sids.append(sid)
npart = sum(ctx.species_count(s) for s in sids)
for det in (False, True):
    for _ in range(2):
        ctx.step(deterministic=det)
    ctx.phase_timing(True)
    ctx.phase_timings(reset=True)
    k = 5
    ctx.synchronize()
    ctx.event(0)
    for _ in range(k):
        ctx.step(deterministic=det)
    ctx.event(1)
    ctx.synchronize()
    ms = ctx.elapsed_ms(0, 1) / k
    ph = ctx.phase_timings(reset=True)
    ctx.phase_timing(False)
    print(f"{name} deterministic={det}: {ms:.2f} ms/step, {npart / ms * 1e3:.3e} pushes/s, phases "
          + ", ".join(f"{a} {b / k:.2f}" for a, b in ph.items()), flush=True)
