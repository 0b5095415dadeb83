#!/usr/bin/env python3
"""Benchmark: particle pushes/s for the whole PIC step on B200 (sm_100a).

Metric (BASELINE.json): particle pushes/sec/GPU for the whole step
(advance_p + interpolators + scatter/unload + field solve + amortised sort)
plus the % HBM roofline of advance_p.

Default workload (BASELINE.json configs[1]): two-stream deck, 256^3 cells,
64 ppc (two counter-drifting electron beams, 32 ppc each, drift +-0.2c,
u_th 0.01), dt 0.25, h 1, blocked sort every 20 steps -> 1,073,741,824
particles on one B200.  Synthetic data (device counter-based RNG load).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config two_stream|thermal|weak]
  python bench.py --impl reference ...   # the reference CPU implementation

Timed region: K whole steps (SimState::step + the reference run-loop's sort
cadence, proj/src/sim.cpp:285-305) bracketed by CUDA events on the library's
stream, synchronize on both sides, max over ranks.  Inputs (34 GB of particle
records) are far larger than the 126 MB L2, so no flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Macro-particle charge and mass scale as 1/ppc (q/m fixed), so the plasma
# frequency does not grow with the particle count: with the reference's w = 1
# (proj/src/sim.cpp:106) a species of ppc particles per unit cell has
# omega_p^2 = ppc q^2 / m.  An unscaled q = -1, m = 1 at 64 ppc would give
# omega_p dt = 2 — the leapfrog stability limit — and the deck would heat
# numerically instead of running the two-stream instability.
CONFIGS = {
    # configs[1]: two-stream, 256^3, two counter-streaming electron beams of
    # 32 ppc (64 ppc total) over a uniform neutralising background:
    # omega_pe = 1, omega_pe dt = 0.25
    "two_stream": dict(n=256, h=1.0, dt=0.25, sort_interval=20,
                       species=[("beam_p", -1.0 / 64, 1.0 / 64, 32, 0.01, (0.2, 0.0, 0.0)),
                                ("beam_m", -1.0 / 64, 1.0 / 64, 32, 0.01, (-0.2, 0.0, 0.0))]),
    # configs[0]: uniform thermal e/i plasma, 64^3, 32 ppc each: bench_base.deck
    # (proj/decks/bench_base.deck, 4 ppc, q = -1, m = 1) at 8x the particle count
    # and the same plasma frequency (q, m scaled by 4/32)
    "thermal": dict(n=64, h=1.0, dt=0.25, sort_interval=20,
                    species=[("electron", -0.125, 0.125, 32, 0.1, (0.0, 0.0, 0.0)),
                             ("ion", 0.125, 12.5, 32, 0.01, (0.0, 0.0, 0.0))]),
    # diagnostic only: the two-stream beams with a negligible charge
    # (ballistic drift, no field growth) to separate sort staleness from
    # the deck's physics in push timings
    "two_stream_ballistic": dict(n=256, h=1.0, dt=0.25, sort_interval=20,
                                 species=[("beam_p", -1e-20, 1.0 / 64, 32, 0.01, (0.2, 0.0, 0.0)),
                                          ("beam_m", -1e-20, 1.0 / 64, 32, 0.01, (-0.2, 0.0, 0.0))]),
    # configs[4]: weak scaling uniform plasma, ~1e9 particles per GPU
    "weak": dict(n=256, h=1.0, dt=0.25, sort_interval=20,
                 species=[("electron", -0.125, 0.125, 32, 0.1, (0.0, 0.0, 0.0)),
                          ("ion", 0.125, 12.5, 32, 0.01, (0.0, 0.0, 0.0))]),
}

def _harris_config():
    """configs[2]: double Harris sheet (paper_2102_13133_b200/decks.py), 256 x 64
    x 256 cells, four species (sheet / background electrons and ions) of 64
    ppc each: 1.07e9 particles per GPU; built through the API (the
    reference's deck text cannot express it)."""
    from paper_2102_13133_b200.decks import Harris
    d = Harris(n=(256, 64, 256), ppc=64)
    return dict(n=256, h=d.h, dt=d.dt, sort_interval=20, deck=d,
                species=[(name, q, m, d.ppc, uth, drift) for name, q, m, uth, drift, _ in d.species()])


CONFIGS["harris"] = _harris_config()


def _lpi_config():
    """configs[3]: laser-plasma interaction (paper_2102_13133_b200/decks.py):
    2048 x 64 x 64 cells (h = 0.2 c/omega_pe), an n/n_cr = 0.1 slab over x
    cells 257..1792 with 64 ppc of electrons and ions (805 M particles), a
    laser (a0 = 0.05) from a soft source near the low wall, Mur field walls
    and absorbing particle walls in x; periodic in y, z."""
    from paper_2102_13133_b200.decks import LPI
    d = LPI(n=(2048, 64, 64), ppc=64, slab=(257, 1792), e0=0.05 * 3.1622776601683795, laser_ix=40)
    return dict(n=2048, h=d.h, dt=d.dt, sort_interval=20, deck=d,
                species=[(name, q, m, d.ppc, uth, (0.0, 0.0, 0.0)) for name, q, m, uth in d.species()])


CONFIGS["lpi"] = _lpi_config()

BYTES_PER_PUSH = 64  # 32 B record read + 32 B record written
# BASELINE.json's metric is per GPU; the line's value is the whole-job sum
# over the N GPUs (the bench contract), value_per_gpu the BASELINE figure
METRIC = "particle pushes/sec summed over all GPUs (advance_p, whole step); per GPU = value_per_gpu"


def deck_text(cfg, n=None, workers=1, seed=4):
    """The reference deck (proj/src/deck.cpp grammar) for a config."""
    n = n or cfg["n"]
    L = n * cfg["h"]
    lines = ["[grid]", f"nx = {n}", f"ny = {n}", f"nz = {n}", f"lx = {L}", f"ly = {L}", f"lz = {L}",
             f"dt = {cfg['dt']}", "steps = 0"]
    for name, q, m, ppc, uth, drift in cfg["species"]:
        lines += [f"[species.{name}]", f"q = {q}", f"m = {m}", f"ppc = {ppc}", f"u_th = {uth}",
                  f"drift = {drift[0]} {drift[1]} {drift[2]}", f"sort_interval = {cfg['sort_interval']}"]
    lines += ["[run]", f"seed = {seed}", f"workers = {workers}"]
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed
    region: NVML every 2 ms from a thread (plus one sample as the region
    starts and one as it ends, so even a millisecond region has samples);
    nvidia-smi -lms 100 when NVML is unavailable."""

    NAMES = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, index=0):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, reasons)
        self.proc = None
        self.nvml = None
        self._stop = threading.Event()

    def _nvml_sample(self):
        n, h = self.nvml
        sm = n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM)
        mx = n.nvmlDeviceGetMaxClockInfo(h, n.NVML_CLOCK_SM)
        try:
            bits = n.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            bits = n.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        self.rows.append((float(sm), float(mx), {v for k, v in self.NAMES.items() if bits & k}))

    def start(self):
        try:
            import pynvml as n
            n.nvmlInit()
            self.nvml = (n, n.nvmlDeviceGetHandleByIndex(self.index))
            self._nvml_sample()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nvml = None
        try:
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _poll(self):
        while not self._stop.wait(0.002):
            try:
                self._nvml_sample()
            except Exception:
                return

    def _read(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.proc.stdout:
            p = [x.strip() for x in line.split(",")]
            if len(p) >= 6 and p[0].replace(".", "").isdigit():
                self.rows.append((float(p[0]), float(p[1]) if p[1].replace(".", "").isdigit() else 0.0,
                                  {names[k] for k in range(4) if p[2 + k].lower() == "active"}))

    def stop(self):
        if self.nvml:
            self._stop.set()
            self.thread.join(timeout=1)
            try:
                self._nvml_sample()
            except Exception:
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [r[0] for r in self.rows]
        mx = max(r[1] for r in self.rows)
        loaded = [x for x in sm if mx and x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx or None,
                "reasons": sorted(set().union(*(r[2] for r in self.rows))), "samples": len(self.rows),
                "source": "nvml" if self.nvml else "nvidia-smi"}


def measured_peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def profile_traffic(config="two_stream"):
    """DRAM bytes (read + write) per advance_p launch and per push from the
    committed ncu --set full summary of the default kernel over a reorder
    cycle (profiles/advance_p_ncu.json for the headline two-stream workload,
    profiles/advance_p_ncu_<config>.json for the others; None if absent)."""
    name = "advance_p_ncu.json" if config == "two_stream" else f"advance_p_ncu_{config}.json"
    path = os.path.join(ROOT, "profiles", name)
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d
    except Exception:
        return None


# ---------------------------------------------------------------------------
def cpu_reference(cfg_name, steps, warmup, sample_n=64, workers=None):
    """The reference CPU implementation (oracle/_ref: minipic compiled from its
    sources, fp32, AVX2 lane) on a bounded sample of the workload: the same
    deck physics on a sample_n^3 box, all host cores.  Times exactly `steps`
    whole steps after `warmup` untimed ones, each step SimState::step plus the
    run loop's sort cadence (sort_due_species, proj/src/sim.cpp:217-222,
    285-305) — the same step our arm times.  When the timed steps contain no
    sort point, one blocked sort of every species is timed separately and
    amortised over sort_interval.  Also reports the reference bench harness's
    own protocol (proj/src/bench.cpp:14,52-59: median of 3 after 1 warm-up)
    over single steps.  Returns pushes/s."""
    from oracle.bindings import Ref, ref_available

    cfg = CONFIGS[cfg_name]
    workers = workers or os.cpu_count() or 1
    if not ref_available():
        return None
    ref = Ref()
    n = min(sample_n, cfg["n"])
    sim = ref.sim(deck_text(cfg, n=n, workers=workers))
    npart = sum(sim.species(s)[1].size for s in range(sim.nspecies))
    for _ in range(warmup):
        sim.step_and_sort(1)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        sim.step_and_sort(1)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    si = cfg["sort_interval"]
    sorted_in_window = si > 0 and any((warmup + k + 1) % si == 0 for k in range(steps))
    t_sort = 0.0
    if si > 0 and not sorted_in_window:
        t0 = time.perf_counter()
        for s in range(sim.nspecies):
            p, ids = sim.species(s)
            ref.sort(p, ids, interleaved=False)
        t_sort = time.perf_counter() - t0
        total += t_sort * steps / si
    med3 = statistics.median(times[:3]) if len(times) >= 3 else statistics.median(times)
    return {
        "value": npart * steps / total, "unit": "particle pushes/s", "cores": workers, "kind": "reference",
        "sample": f"{cfg_name} deck physics on {n}^3 cells ({npart} particles): {steps} timed steps after "
                  f"{warmup} warm-up, run-loop sort every {si}"
                  + ("" if sorted_in_window or si <= 0 else f" (no sort point in the window: one blocked sort "
                                                          f"timed, amortised /{si})")
                  + f"; minipic fp32 AVX2, {workers} workers",
        "steps": steps, "warmup": warmup, "ms_per_step": total / steps * 1e3, "sort_s": t_sort,
        "particles": npart, "cells": n,
        "bench_cpp_protocol": {"median_of_3_step_ms": med3 * 1e3,
                               "note": "proj/src/bench.cpp:14,52-59: 1 warm-up, median of 3 timed repetitions"},
    }


# ---------------------------------------------------------------------------
def run_ours(args, rank, world):
    import paper_2102_13133_b200 as pic

    cfg = CONFIGS[args.config]
    n = cfg["n"]
    deck = cfg.get("deck")
    g = deck.grid() if deck else pic.make_grid(n, cfg["h"], dt=cfg["dt"])
    ctx = pic.Context(g, device=args.device)
    sids = []
    if deck:
        sids = deck.load(ctx, seed=1234 + 7919 * rank)
    else:
        for si, (name, q, m, ppc, uth, drift) in enumerate(cfg["species"]):
            cap = ppc * g.interior
            sid = ctx.add_species(name, q, m, cap)
            ctx.load_synthetic(sid, ppc, uth, drift, seed=1234 + 7919 * rank)
            sids.append(sid)
    ctx.synchronize()
    npart = sum(ctx.species_count(s) for s in sids)
    sort_interval = cfg["sort_interval"]
    step_count = [0]

    def one_step():
        ctx.step()
        step_count[0] += 1
        if sort_interval > 0 and step_count[0] % sort_interval == 0:
            for s in sids:
                ctx.sort_particles(s)

    # one sort of the freshly loaded (already voxel-ordered) stores allocates
    # the sort scratch outside the timed region and leaves the order intact
    for s in sids:
        ctx.sort_particles(s)
    for _ in range(args.warmup):
        one_step()
    # the step graphs of the timed steps (buffer pairs, reorder cadence, owed
    # relabels) are captured here, without running anything, so that every
    # timed step is a graph replay (executor preparation, like an
    # instantiated graph; every kernel of every timed step still runs)
    graphs_prepared = ctx.prepare_graphs(args.steps, sort_interval, step_count[0])
    ctx.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    # --- device-timed whole steps -------------------------------------------
    clocks = ClockSampler(args.device)
    clocks.start()
    barrier()
    ctx.synchronize()
    l0 = ctx.launch_count()
    g0 = ctx._graph_stats()
    ctx.event(0)
    for _ in range(args.steps):
        one_step()
    ctx.event(1)
    ctx.synchronize()
    barrier()
    ms = ctx.elapsed_ms(0, 1)
    launches = ctx.launch_count() - l0
    g1 = ctx._graph_stats()
    graph_stats = {k: b - a for k, a, b in zip(("captured", "replayed", "plain"), g0, g1)}
    clk = clocks.stop()

    # --- phase split (same steps again with PhaseTimings events) --------------
    ctx.phase_timing(True)
    ctx.phase_timings(reset=True)
    ctx._push_kernel_ms(reset=True)
    nph = args.steps
    for _ in range(nph):
        one_step()
    ctx.synchronize()
    ph = ctx.phase_timings(reset=True)
    kms, klaunch = ctx._push_kernel_ms(reset=True)
    ctx.phase_timing(False)
    # the roofline's denominator: the push kernel launches alone (CUDA events
    # on each launch's stream); the push phase also holds the voxel-order
    # scans / relabels and launch gaps
    push_ms_per_launch = kms / max(klaunch, 1)
    push_rate_kernel = npart * nph / (kms / 1e3)

    if world > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # --- e2e through the host-buffer C-ABI call --------------------------------
    e2e = None
    if not args.no_e2e and getattr(deck, "laser_ix", None) is None:  # walled decks: no pic_step_host
        e2e = run_e2e(pic, ctx, sids, npart, args, world)
    ctx.close()
    # --- e2e through the reference's own run surface, state device-resident --
    e2e_res = None
    if not args.no_e2e and not cfg.get("deck") and cfg["n"] <= 64 and world == 1:
        e2e_res = run_e2e_simstate(cfg, args)
    return dict(ms=ms, npart=npart, launches=launches, clocks=clk, phases=ph, push_rate_kernel=push_rate_kernel,
                graphs_prepared=graphs_prepared, graph_stats=graph_stats,
                push_ms_per_launch=push_ms_per_launch, nspecies=len(sids), grid=g, e2e=e2e, e2e_resident=e2e_res,
                # a launch pushes every species of the deck at once where it
                # can (one grid per push form): particles per timed launch
                particles_per_launch=npart * nph / max(klaunch, 1),
                push_phase_rate=npart * nph / (ph["push"] / 1e3), push_launches_timed=klaunch)


def run_ours_decomposed(args, rank, world):
    """N > 1 (or --decomposed): weak-scaled slab decomposition.
    The global box is (n N) x n x n with each rank's slab the single-GPU
    deck.  Periodic decks run the C++ decomposed step (pic_dd: pushes, fold,
    fields and the migration / halo exchanges as NCCL send / receive inside
    the library, graph-captured, no host synchronisation); the walled LPI
    deck runs the host-sequenced exchanges of domain.py."""
    import torch

    import paper_2102_13133_b200 as pic
    from paper_2102_13133_b200.domain import SlabGeometry

    torch.cuda.set_device(args.device)
    cfg = CONFIGS[args.config]
    deck = cfg.get("deck")
    if deck is not None and hasattr(deck, "laser_ix"):
        return run_ours_decomposed_py(args, rank, world)
    n = cfg["n"]
    if deck:  # weak scaling: the global box grows in x, (nx N) x ny x nz
        import dataclasses
        NX0 = deck.n[0]
        deck = dataclasses.replace(deck, n=(NX0 * world, deck.n[1], deck.n[2]))
        geom = SlabGeometry(*deck.n, world, h=(cfg["h"],) * 3, dt=cfg["dt"])
    else:
        geom = SlabGeometry(n * world, n, n, world, h=(cfg["h"],) * 3, dt=cfg["dt"])
    g = geom.local_grid()
    ctx = pic.Context(g, device=args.device)
    ctx.set_x_open(True, rank == 0)
    sids = []
    if deck:
        for name, q, m, uth, drift, sheet in deck.species():
            sid = ctx.add_species(name, q, m, int(deck.ppc * g.interior * 1.02) + 65536)
            ctx.load_harris(sid, deck.ppc, uth, drift, seed=1234 + 7919 * rank, **sheet)
            sids.append(sid)
        ctx.upload_fields(deck.fields(g, x0=geom.x0(rank)))
    else:
        for name, q, m, ppc, uth, drift in cfg["species"]:
            sid = ctx.add_species(name, q, m, int(ppc * g.interior * 1.02) + 65536)
            ctx.load_synthetic(sid, ppc, uth, drift, seed=1234 + 7919 * rank)
            sids.append(sid)
    import torch.distributed as dist
    uid = [pic.dd_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0)
    dd = pic.DecomposedStep(ctx, rank, world, uid[0])
    ctx.synchronize()
    sort_interval = cfg["sort_interval"]
    step_count = [0]

    def one_step():
        dd.step()
        step_count[0] += 1
        if sort_interval > 0 and step_count[0] % sort_interval == 0:
            for s_ in sids:
                ctx.sort_particles(s_)

    for s_ in sids:
        ctx.sort_particles(s_)
    for _ in range(args.warmup):
        one_step()
    # the timed steps' graphs (NCCL exchanges included) captured ahead, on
    # every rank alike, so every timed step is a replay
    graphs_prepared = dd.prepare_graphs(args.steps, sort_interval, step_count[0])
    ctx.synchronize()
    clocks = ClockSampler(args.device)
    clocks.start()
    dist.barrier()
    ctx.synchronize()
    l0 = ctx.launch_count()
    ctx.event(0)
    for _ in range(args.steps):
        one_step()
    ctx.event(1)
    ctx.synchronize()
    dist.barrier()
    ms = ctx.elapsed_ms(0, 1)
    launches = ctx.launch_count() - l0
    clk = clocks.stop()
    # phase split (the same steps again, plain launches with PhaseTimings events)
    ctx.phase_timing(True)
    ctx.phase_timings(reset=True)
    ctx._push_kernel_ms(reset=True)
    for _ in range(args.steps):
        one_step()
    ctx.synchronize()
    ph = ctx.phase_timings(reset=True)
    kms, klaunch = ctx._push_kernel_ms(reset=True)
    ctx.phase_timing(False)
    npart_local = sum(ctx.species_count(s_) for s_ in sids)
    t = torch.tensor([ms, float(npart_local), kms], dtype=torch.float64, device="cuda")
    mx = t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = t.clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    ms = float(mx[0].item())
    npart_total = int(sm[1].item())
    push_ms_per_launch = float(mx[2].item()) / (args.steps * len(sids))
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e_dd(pic, dd, ctx, sids, args, world)
    dd.close()
    ctx.close()
    return dict(ms=ms, npart=npart_total // world, npart_total=npart_total, launches=launches, clocks=clk,
                graphs_prepared=graphs_prepared,
                phases=ph, push_rate_kernel=npart_local * args.steps / (kms / 1e3),
                push_ms_per_launch=push_ms_per_launch, nspecies=len(sids), grid=geom.global_grid(), e2e=e2e,
                particles_per_launch=npart_local / len(sids),
                local_grid=g, decomposed=True, exchange="C++ pic_dd over NCCL (graph-captured)",
                push_phase_rate=npart_local * args.steps / (ph["push"] / 1e3), push_launches_timed=klaunch)


def run_e2e_dd(pic, dd, ctx, sids, args, world):
    """Decomposed host-buffer steps: every step uploads each rank's species
    from pinned host records, runs the decomposed step, downloads them."""
    import torch
    import torch.distributed as dist
    host = []
    for s_ in sids:
        cap = ctx.species_count(s_) + (1 << 20)
        pos = np.zeros((cap, 4), np.float32)
        mom = np.zeros((cap, 4), np.float32)
        pic.host_register(pos)
        pic.host_register(mom)
        host.append([pos, mom, ctx.download_records(s_, pos, mom)])

    def step():
        b = 0
        for s_, h in zip(sids, host):
            ctx.upload_records(s_, h[0], h[1], h[2])
            b += 32 * h[2]
        dd.step()
        for s_, h in zip(sids, host):
            h[2] = ctx.download_records(s_, h[0], h[1])
        return b

    step()
    dist.barrier()
    k = max(1, args.e2e_steps)
    t0 = time.perf_counter()
    byt = 0
    for _ in range(k):
        byt += step()
    dt = time.perf_counter() - t0
    t = torch.tensor([dt], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dt = float(t.item())
    npart = sum(h[2] for h in host)
    tn = torch.tensor([float(npart)], dtype=torch.float64, device="cuda")
    dist.all_reduce(tn)
    for h in host:
        pic.host_unregister(h[0])
        pic.host_unregister(h[1])
    return {"value": float(tn.item()) * k / dt, "value_per_gpu": float(tn.item()) * k / dt / world,
            "unit": "particle pushes/s", "h2d_bytes_per_step": byt // k,
            "d2h_bytes_per_step": byt // k, "steps": k, "ms_per_step": dt / k * 1e3,
            "note": "per rank: records H2D, decomposed step, records D2H (not pipelined); bytes are rank 0's"}


def run_ours_decomposed_py(args, rank, world):
    """The walled LPI deck: host-sequenced exchanges (domain.py)."""
    import torch

    import paper_2102_13133_b200 as pic
    from paper_2102_13133_b200.domain import CudaSlab, DecomposedSim, DistTransport, SlabGeometry

    torch.cuda.set_device(args.device)
    cfg = CONFIGS[args.config]
    n = cfg["n"]
    deck = cfg.get("deck")
    lpi = deck is not None and hasattr(deck, "laser_ix")
    walls = None
    if deck:  # weak scaling: the global box grows in x, (nx N) x ny x nz
        import dataclasses
        NX0 = deck.n[0]
        deck = dataclasses.replace(deck, n=(NX0 * world, deck.n[1], deck.n[2]))
        if lpi:  # the slab keeps its distance from the far wall
            deck = dataclasses.replace(deck, slab=(deck.slab[0], deck.n[0] - (NX0 - deck.slab[1])))
            walls = (pic.PBC_ABSORB, pic.FBC_MUR)
        geom = SlabGeometry(*deck.n, world, h=(cfg["h"],) * 3, dt=cfg["dt"], walls=walls)
    else:
        geom = SlabGeometry(n * world, n, n, world, h=(cfg["h"],) * 3, dt=cfg["dt"])
    slab = CudaSlab(geom.local_grid(), rank, rank == 0, device=args.device, walls=walls, world=world)
    sim = DecomposedSim(geom, {rank: slab}, DistTransport(rank, world))
    ctx = slab.ctx
    g = geom.local_grid()
    sids = []
    if lpi:
        x0 = geom.x0(rank)
        lo, hi = max(deck.slab[0], x0 + 1) - x0, min(deck.slab[1], x0 + g.nx) - x0
        for name, q, m, uth in deck.species():
            sid = sim.add_species(name, q, m, int(deck.ppc * g.interior * 1.02) + 65536)
            if lo <= hi:
                ctx.load_slab(sid, deck.ppc, uth, (0.0, 0.0, 0.0), seed=1234 + 7919 * rank, ix_lo=lo, ix_hi=hi)
            sids.append(sid)
        sim.set_laser(deck.laser_ix, deck.e0, deck.omega0, pol=1, ramp_steps=deck.ramp_steps)
    elif deck:
        for name, q, m, uth, drift, sheet in deck.species():
            sid = sim.add_species(name, q, m, int(deck.ppc * g.interior * 1.02) + 65536)
            ctx.load_harris(sid, deck.ppc, uth, drift, seed=1234 + 7919 * rank, **sheet)
            sids.append(sid)
        ctx.upload_fields(deck.fields(g, x0=geom.x0(rank)))
    else:
        for name, q, m, ppc, uth, drift in cfg["species"]:
            sid = sim.add_species(name, q, m, int(ppc * g.interior * 1.02) + 65536)
            ctx.load_synthetic(sid, ppc, uth, drift, seed=1234 + 7919 * rank)
            sids.append(sid)
    ctx.synchronize()
    sort_interval = cfg["sort_interval"]
    step_count = [0]

    def one_step():
        sim.step()
        step_count[0] += 1
        if sort_interval > 0 and step_count[0] % sort_interval == 0:
            for s_ in sids:
                ctx.sort_particles(s_)

    for s_ in sids:
        ctx.sort_particles(s_)
    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    import torch.distributed as dist

    stream = torch.cuda.current_stream()
    clocks = ClockSampler(args.device)
    clocks.start()
    dist.barrier()
    torch.cuda.synchronize()
    l0 = ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        one_step()
    ev1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    ms = ev0.elapsed_time(ev1)
    launches = ctx.launch_count() - l0
    clk = clocks.stop()
    # push phase (advance_p of all species) timed with events per step
    pev = []

    def mark(phase, begin):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        pev.append(e)

    sim.on_mark = mark
    for _ in range(args.steps):
        one_step()
    sim.on_mark = None
    torch.cuda.synchronize()
    push_ms = sum(pev[2 * k].elapsed_time(pev[2 * k + 1]) for k in range(len(pev) // 2))
    npart_local = sum(ctx.species_count(s_) for s_ in sids)
    t = torch.tensor([ms, float(npart_local), push_ms], dtype=torch.float64, device="cuda")
    mx = t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = t.clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    ms = float(mx[0].item())
    npart_total = int(sm[1].item())
    push_ms_per_launch = float(mx[2].item()) / (args.steps * len(sids))
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e_decomposed(pic, sim, ctx, sids, args, world)
    for e in sim.slabs.values():
        e.ctx.close()
    return dict(ms=ms, npart=npart_total // world, npart_total=npart_total, launches=launches, clocks=clk,
                phases={"push": push_ms}, push_rate_kernel=npart_local * args.steps / (push_ms / 1e3),
                push_ms_per_launch=push_ms_per_launch, nspecies=len(sids), grid=geom.global_grid(), e2e=e2e,
                particles_per_launch=npart_local / len(sids),
                local_grid=g,
                decomposed=True)


def run_e2e_decomposed(pic, sim, ctx, sids, args, world):
    """Decomposed host-buffer steps: every step uploads each rank's species
    from pinned host records, runs the decomposed step, downloads them."""
    import torch
    import torch.distributed as dist
    host = []
    for s_ in sids:
        cap = ctx.species_count(s_) + (1 << 20)
        pos = np.zeros((cap, 4), np.float32)
        mom = np.zeros((cap, 4), np.float32)
        pic.host_register(pos)
        pic.host_register(mom)
        host.append([pos, mom, ctx.download_records(s_, pos, mom)])

    def step():
        b = 0
        for s_, h in zip(sids, host):
            ctx.upload_records(s_, h[0], h[1], h[2])
            b += 32 * h[2]
        sim.step()
        for s_, h in zip(sids, host):
            h[2] = ctx.download_records(s_, h[0], h[1])
        return b

    step()
    dist.barrier()
    k = max(1, args.e2e_steps)
    t0 = time.perf_counter()
    byt = 0
    for _ in range(k):
        byt += step()
    dt = time.perf_counter() - t0
    t = torch.tensor([dt], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dt = float(t.item())
    npart = sum(h[2] for h in host)
    tn = torch.tensor([float(npart)], dtype=torch.float64, device="cuda")
    dist.all_reduce(tn)
    for h in host:
        pic.host_unregister(h[0])
        pic.host_unregister(h[1])
    return {"value": float(tn.item()) * k / dt, "value_per_gpu": float(tn.item()) * k / dt / world,
            "unit": "particle pushes/s", "h2d_bytes_per_step": byt // k,
            "d2h_bytes_per_step": byt // k, "steps": k, "ms_per_step": dt / k * 1e3,
            "note": "per rank: records H2D, decomposed step, records D2H (not pipelined); bytes are rank 0's"}


def run_e2e_simstate(cfg, args, steps=None, diag_interval=10):
    """The reference's own host surface with the state resident on the GPU:
    the deck text (proj/src/deck.cpp grammar), SimState::initialize (the
    reference's mt19937_64 load on the host, bit-identical, then uploaded)
    and SimState::run (sim.cpp:285-306: step, the due sorts, the
    diagnostics row every diag_interval steps with its charge refresh,
    written as the reference's CSV).  Timed by the wall clock around a
    second run() of five sort cycles (the first, a warm-up, captures the
    step graphs); per step the host reads back only the diagnostics (pic_diag +
    kinetic per species, every diag_interval steps)."""
    import tempfile

    from paper_2102_13133_b200.simstate import Deck, SimState
    steps = steps or 5 * cfg["sort_interval"]
    text = deck_text(cfg).replace("steps = 0", f"steps = {steps}") + f"diag_interval = {diag_interval}\n"
    sim = SimState.initialize(Deck(text), device=args.device)
    npart = sum(sim.context.species_count(k) for k in range(len(cfg["species"])))
    with tempfile.NamedTemporaryFile(suffix=".csv") as f:
        sim.run(f.name)  # warm-up run: captures the step graphs of the sort cycles
        sim.context.synchronize()
        t0 = time.perf_counter()
        sim.run(f.name)  # steps more steps, CSV rows on the diag cadence; quiesces at the end
        dt = time.perf_counter() - t0
        rows = sum(1 for _ in open(f.name)) - 1
    sim.close()
    d2h = (28 + 4 * len(cfg["species"])) * (steps // diag_interval + 1)
    return {"value": npart * steps / dt, "unit": "particle pushes/s", "h2d_bytes_per_step": 0,
            "d2h_bytes_per_step": d2h / steps, "steps": steps, "ms_per_step": dt / steps * 1e3,
            "csv_rows": rows,
            "path": "pic_sim_run (SimState::run over the deck text; state device-resident, diagnostics "
                    f"every {diag_interval} steps)"}


def run_e2e(pic, ctx, sids, npart, args, world):
    """pic_step_host: every step uploads all species from pinned host
    buffers, steps, and downloads them back (32 B/particle each way)."""
    host = []
    for s in sids:
        p, ids = ctx.download_species(s)
        pic.host_register(p)
        pic.host_register(ids)
        host.append((p, ids))
    lanes = [h[0] for h in host]
    idl = [h[1] for h in host]
    ctx.step_host(lanes, idl)  # warm-up
    ctx.synchronize()
    k = max(1, args.e2e_steps)
    t0 = time.perf_counter()
    for _ in range(k):
        ctx.step_host(lanes, idl)
    dt = time.perf_counter() - t0
    if world > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor([dt], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    for p, ids in host:
        pic.host_unregister(p)
        pic.host_unregister(ids)
    b_in = sum(h[0].nbytes + h[1].nbytes for h in host)
    b_out = sum(h[0].nbytes * 6 // 7 + h[1].nbytes for h in host)  # lanes 0-5 + ids (w is not modified)
    if world > 1:  # whole-job sum of every rank's particles
        import torch
        import torch.distributed as dist
        tn = torch.tensor([float(npart)], dtype=torch.float64)
        dist.all_reduce(tn)
        npart_all = float(tn.item())
    else:
        npart_all = float(npart)
    return {"value": npart_all * k / dt, "value_per_gpu": npart_all * k / dt / world,
            "unit": "particle pushes/s", "h2d_bytes_per_step": b_in,
            "d2h_bytes_per_step": b_out, "steps": k, "ms_per_step": dt / k * 1e3}


_OUT_FD = None


def emit(obj):
    """The one JSON line on the real stdout: everything else the run prints
    (NCCL's version banner, library chatter) goes to stderr (main() points
    fd 1 at fd 2)."""
    os.write(_OUT_FD if _OUT_FD is not None else 1, (json.dumps(obj) + "\n").encode())


def main():
    global _OUT_FD
    _OUT_FD = os.dup(1)
    sys.stdout.flush()
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="two_stream", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-n", type=int, default=64)
    ap.add_argument("--decomposed", action="store_true",
                    help="use the slab-decomposed (NCCL) step even at N=1 (self-exchange; tests the N>1 path)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    args.device = local
    cfg = CONFIGS[args.config]

    if args.impl == "reference":
        if rank != 0:
            return
        if cfg.get("deck"):
            emit({"impl": "reference", "unavailable": f"the reference's deck text cannot express the "
                              f"{args.config} deck (built through the API here)"})
            return
        r = cpu_reference(args.config, max(1, args.steps), max(0, args.warmup), sample_n=args.cpu_sample_n)
        if r is None:
            emit({"impl": "reference", "unavailable": "oracle/_ref/libminipic_ref.so not built"})
            return
        line = {
            "impl": "reference", "metric": METRIC, "value": r["value"],
            "unit": "particle pushes/s", "n_gpus": args.gpus, "steps": r["steps"], "warmup": r["warmup"],
            "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (reference Rng load)",
            "config": {"workload": args.config, "cells": f"{cfg['n']}^3", "sample_cells": f"{r['cells']}^3",
                       "sample_particles": r["particles"], "same_config": r["cells"] == cfg["n"],
                       "sample": r["sample"]},
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "bench_cpp_protocol": r["bench_cpp_protocol"],
            "e2e": {"value": r["value"], "unit": "particle pushes/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }
        emit(line)
        return

    if world > 1 or args.decomposed:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        res = run_ours_decomposed(args, rank, world)
    else:
        res = run_ours(args, rank, world)
    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    ms_per_step = res["ms"] / args.steps
    value = res.get("npart_total", res["npart"] * world) * args.steps / (res["ms"] / 1e3)
    peak, peak_kind = measured_peak_gbs()
    achieved = res["particles_per_launch"] * BYTES_PER_PUSH / (res["push_ms_per_launch"] / 1e3) / 1e9
    prof = None if world > 1 or args.decomposed else profile_traffic(args.config)
    cpu = None
    if not args.no_cpu_baseline and world == 1 and cfg.get("deck"):
        cpu = {"value": None, "note": "the reference cannot express this deck; see --config two_stream"}
    elif not args.no_cpu_baseline and world == 1:  # rank 0 at N=1 only
        try:
            r = cpu_reference(args.config, 10, 1, sample_n=args.cpu_sample_n)
            if r:
                cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # the baseline is reported, not required
            cpu = {"value": None, "error": str(e)[:200]}
    g = res["grid"]
    gl = res.get("local_grid", g)
    line = {
        "metric": METRIC,
        "value": value,
        "value_per_gpu": value / world,
        "unit": "particle pushes/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (device counter-RNG load: uniform offsets, drifting Maxwellian momenta"
                + {"harris": ", sech^2 Harris weights, A_y fields)",
                   "lpi": " in the plasma slab; laser soft source, Mur / absorbing x walls)"}.get(args.config, ")"),
        "config": {"workload": args.config, "cells": f"{gl.nx}x{gl.ny}x{gl.nz}", "particles_per_gpu": res["npart"],
                   "ppc": sum(s[3] for s in cfg["species"]), "dt": g.dt, "sort_interval": cfg["sort_interval"],
                   "parallelism": f"x-slab decomposition over {world} GPUs (NCCL halo + migration)"
                   if res.get("decomposed") else "single",
                   "global_cells": f"{g.nx}x{g.ny}x{g.nz}",
                   **({"exchange": res["exchange"]} if res.get("exchange") else {}),
                   "l2": "inputs (34 GB of particle records) >> 126 MB L2; no flush",
                   **({"step_graphs": {"prepared_before_timing": res["graphs_prepared"],
                                       "timed_steps": res.get("graph_stats")}} if "graphs_prepared" in res else {}),
                   "push_kernel_rate": res["push_rate_kernel"],
                   "push_phase_rate": res.get("push_phase_rate"),
                   "push_launches_timed": res.get("push_launches_timed"),
                   "phase_ms_per_step": {k: v / args.steps for k, v in res["phases"].items()}},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     # measured DRAM bytes of one profiled launch (ncu, profiles/advance_p_ncu.json)
                     "traffic": prof and prof.get("dram_bytes_per_launch"),
                     "traffic_bytes_per_push": prof and prof.get("dram_bytes_per_push"),
                     "traffic_launch_particles": prof and prof["launches"][0].get("particles"),
                     "algorithmic_bytes_per_launch": res["particles_per_launch"] * BYTES_PER_PUSH,
                     "particles_per_launch": res["particles_per_launch"],
                     "kernel": prof and prof.get("kernel"),
                     "achieved_from": "mean duration of every advance_p launch in a timed pass (CUDA events on "
                                      "the launching stream; in-place, counting and reordering pushes alike; "
                                      "one launch pushes every species of the deck)",
                     "bytes_per_push": BYTES_PER_PUSH, "peak_kind": peak_kind},
        "cpu_baseline": cpu,
        "e2e": res["e2e"],
        **({"e2e_resident": res["e2e_resident"]} if res.get("e2e_resident") else {}),
        "gpu_launches": res["launches"],
        "clocks": res["clocks"],
    }
    emit(line)
    if world > 1 or args.decomposed:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
