"""Times sort_particles on a bench deck (device events), per variant, after
`stale` steps, for every species of the deck."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_13133_b200 as pic  # noqa: E402
from bench import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "two_stream"]
stale = int(sys.argv[2]) if len(sys.argv) > 2 else 10
variants = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0, 1]
g = pic.make_grid(cfg["n"], cfg["h"], dt=cfg["dt"])
ctx = pic.Context(g)
sids = []
for name, q, m, ppc, uth, drift in cfg["species"]:
    sid = ctx.add_species(name, q, m, ppc * g.interior)
    ctx.load_synthetic(sid, ppc, uth, drift, seed=7)
    sids.append(sid)
for rep in range(2):
    for _ in range(stale):
        ctx.step()
    ctx.synchronize()
    for var in variants:
        ctx._set_sort_variant(var)
        for s in sids:
            t0 = time.perf_counter()
            ctx.event(0)
            ctx.sort_particles(s)
            ctx.event(1)
            ms = ctx.elapsed_ms(0, 1)
            print(f"rep {rep} stale {stale} variant {var} species {s}: {ms:.2f} ms device, "
                  f"{(time.perf_counter() - t0) * 1e3:.1f} ms host", flush=True)
