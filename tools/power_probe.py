"""Is the push power-bound?  Times every step's push phase (device events)
of the bench workload over two sort cycles run back to back, then over two
cycles with an idle gap before each step, with NVML board power, SM clock
and clock-event reasons sampled during each step.

    python tools/power_probe.py [config] [gap_s]
"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_13133_b200 as pic  # noqa: E402
from bench import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "two_stream"
gap = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
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
npart = sum(ctx.species_count(s) for s in sids)

import pynvml as n  # noqa: E402

n.nvmlInit()
h = n.nvmlDeviceGetHandleByIndex(0)
limit_w = n.nvmlDeviceGetEnforcedPowerLimit(h) / 1e3
rows = []
stop = threading.Event()


def poll():
    while not stop.wait(0.002):
        bits = n.nvmlDeviceGetCurrentClocksEventReasons(h)
        rows.append((time.perf_counter(), n.nvmlDeviceGetPowerUsage(h) / 1e3,
                     n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM), n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_MEM),
                     bits))


th = threading.Thread(target=poll, daemon=True)
th.start()
step = [0]
print(f"{name}: {npart} particles, enforced power limit {limit_w:.0f} W", flush=True)


def run(label, nsteps, idle):
    out = []
    for _ in range(nsteps):
        if idle:
            ctx.synchronize()
            time.sleep(idle)
        ctx.phase_timing(True)
        ctx.phase_timings(reset=True)
        t0 = time.perf_counter()
        ctx.step()
        step[0] += 1
        ctx.synchronize()
        t1 = time.perf_counter()
        ph = ctx.phase_timings(reset=True)
        ctx.phase_timing(False)
        sel = [r for r in rows if t0 <= r[0] <= t1]
        pw = max((r[1] for r in sel), default=float("nan"))
        sm = sorted(r[2] for r in sel)[len(sel) // 2] if sel else float("nan")
        mem = sorted(r[3] for r in sel)[len(sel) // 2] if sel else float("nan")
        cap = sum(1 for r in sel if r[4] & 0x4)
        out.append(ph["push"])
        print(f"{label} step {step[0]:3d} stale {(step[0] - 1) % cfg['sort_interval']:2d} push {ph['push']:7.3f} ms "
              f"({npart / (ph['push'] / 1e3):.3e}/s)  power max {pw:6.0f} W  sm {sm:5.0f}  mem {mem:5.0f}  "
              f"power_cap {cap}/{len(sel)}", flush=True)
        if step[0] % cfg["sort_interval"] == 0:
            for s in sids:
                ctx.sort_particles(s)
    return out


a = run("busy", 2 * cfg["sort_interval"], 0)
b = run("idle", 2 * cfg["sort_interval"], gap)
stop.set()
print(f"mean push ms: busy {sum(a) / len(a):.3f}  idle-gapped {sum(b) / len(b):.3f}")
