"""Times SimState's diagnostics pieces on the thermal C1 deck (tools only)."""
import time
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2102_13133_b200.simstate import Deck, SimState

cfg = bench.CONFIGS["thermal"]
text = bench.deck_text(cfg).replace("steps = 0", "steps = 20") + "diag_interval = 10\n"
sim = SimState.initialize(Deck(text))
for _ in range(4):
    sim.step()
ctx = sim.context
ctx.synchronize()
for name, fn in [("step", sim.step), ("refresh_charge", sim.refresh_charge_diagnostics),
                 ("emit_row", sim.emit_diagnostics)]:
    fn(); ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        fn()
    ctx.synchronize()
    print(name, "%.3f ms" % ((time.perf_counter() - t0) / 5 * 1e3))
