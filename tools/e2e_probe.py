"""pic_step_host throughput vs pipeline chunk size (two-stream deck)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_13133_b200 as pic  # noqa: E402
from bench import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "two_stream"]
chunks = [int(c) for c in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1 << 23, 1 << 24, 1 << 25, 1 << 26]
g = pic.make_grid(cfg["n"], cfg["h"], dt=cfg["dt"])
ctx = pic.Context(g)
sids = []
for name, q, m, ppc, uth, drift in cfg["species"]:
    sid = ctx.add_species(name, q, m, ppc * g.interior)
    ctx.load_synthetic(sid, ppc, uth, drift, seed=7)
    sids.append(sid)
host = []
for s in sids:
    p, ids = ctx.download_species(s)
    pic.host_register(p)
    pic.host_register(ids)
    host.append((p, ids))
npart = sum(h[1].size for h in host)
for ch in chunks:
    ctx._set_host_chunk(ch)
    ctx.step_host([h[0] for h in host], [h[1] for h in host])
    t0 = time.perf_counter()
    k = 2
    for _ in range(k):
        ctx.step_host([h[0] for h in host], [h[1] for h in host])
    dt = (time.perf_counter() - t0) / k
    print(f"chunk {ch}: {dt * 1e3:.1f} ms/step  {npart / dt:.3e} pushes/s  {npart * 32 / dt / 1e9:.1f} GB/s each way",
          flush=True)
