import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_2102_13133_b200.simstate import Deck, SimState
cfg = bench.CONFIGS["thermal"]
text = bench.deck_text(cfg).replace("steps = 0", "steps = 20") + "diag_interval = 10\n"
sim = SimState.initialize(Deck(text))
ctx = sim.context
def segs(sid):
    n = ctx.species_count(sid)
    pos = torch.empty((n, 4), dtype=torch.float32, device="cuda"); mom = torch.empty_like(pos)
    torch.cuda.synchronize(); ctx.download_records(sid, pos, mom); torch.cuda.synchronize()
    k = pos[:, 3].contiguous().view(torch.int32)
    ch = (k[1:] != k[:-1]).float().mean().item()
    return ch * 32
for st in range(8):
    print("step", st, "segments per warp (logical order) e/i:", round(segs(0), 2), round(segs(1), 2), "ordered", ctx._species_ordered(0))
    sim.step()
