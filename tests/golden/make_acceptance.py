"""Generates tests/golden/acceptance_ref.json: the reference's own values for
the physics acceptance criteria that the fast (atomic) GPU path is checked
against in tests/test_gpu_acceptance.py.

TEST INFRASTRUCTURE.  Runs the unmodified reference (oracle/_ref, minipic
fp32 built from /root/reference by oracle/Makefile) in this container; the
GPU box has no /root/reference, so the values travel as this fixture.

Cases (reference test each restates, /root/reference/proj/tests/...):
  gauss       acceptance.cpp:87-134   Gauss residual constancy, 200 steps
  divb        acceptance.cpp:137-204  div B after 1000 field-only steps
  yee         acceptance.cpp:207-285  vacuum Yee dispersion of one mode
  plasma      acceptance.cpp:288-336  field energy line at 2 omega_p
  energy      test_sim.cpp:371-412    total energy bounded (3 % in fp32)
  thermal     SURVEY §8d C1 (bench.py thermal deck at 64^3): deterministic
              state hashes after 5 and 21 steps (sort at 20) and the total
              energy history of 200 steps
  two_stream  configs[1] at 64^3: field energy history (growth rate)
The random fields of divb are drawn here with numpy (the reference test's
std::mt19937_64 draw is not reproduced: the property, not the draw, is the
criterion) and stored, so the GPU run starts from the identical state.

    python tests/golden/make_acceptance.py
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.bindings import Orc, Ref  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "acceptance_ref.json")
WORKERS = os.cpu_count() or 1

GAUSS_DECK = """[grid]
nx = 16
ny = 16
nz = 16
lx = 16
ly = 16
lz = 16
dt = 0.1
steps = 200

[species.electron]
q = -1
m = 1
ppc = 8
u_th = 0.05
sort_interval = 20

[species.positron]
q = 1
m = 1
ppc = 8
u_th = 0.05
sort_interval = 20

[run]
seed = 11
diag_interval = 10
"""

DIVB_DECK = """[grid]
nx = 16
ny = 16
nz = 16
lx = 16
ly = 16
lz = 16
steps = 0

[species.none]
q = 0
m = 1
ppc = 0

[run]
seed = 1
"""

YEE_DECK = """[grid]
nx = 64
ny = 4
nz = 4
lx = 64
ly = 4
lz = 4
dt = 0.5
steps = 0

[species.none]
q = 0
m = 1
ppc = 0

[run]
seed = 1
"""


def plasma_deck():
    h = 4.0 ** (1.0 / 3.0)
    return (f"[grid]\nnx = 32\nny = 32\nnz = 32\nlx = {32 * h!r}\nly = {32 * h!r}\nlz = {32 * h!r}\n"
            "dt = 0.1\nsteps = 0\n[species.electron]\nq = -1\nm = 1\nppc = 4\nu_th = 0\n"
            "sort_interval = 25\nperturb_ux = 0.01\nperturb_kmode = 1\n[run]\nseed = 9\n")


ENERGY_DECK = """[grid]
nx = 16
ny = 16
nz = 16
lx = 16
ly = 16
lz = 16
dt = 0.1
steps = 500

[species.electron]
q = -1
m = 1
ppc = 1
u_th = 0
sort_interval = 25
perturb_ux = 0.01
perturb_kmode = 1

[run]
seed = 3
diag_interval = 500
"""


def bench_deck(name, n=64, deterministic=False, workers=1):
    from bench import CONFIGS, deck_text
    text = deck_text(CONFIGS[name], n=n, workers=workers)
    return text + ("deterministic = true\n" if deterministic else "")


# ---- criterion metrics (shared with the GPU test) ------------------------------
def divb_fields(nx=16, seed=7):
    """B = discrete curl of a random periodic vector potential (the
    construction of acceptance.cpp:159-186) on an nx^3 grid, h = 1; numpy
    draw, ghost planes synced by the oracle."""
    n = nx
    p = n + 2
    rng = np.random.default_rng(seed)
    a = [rng.uniform(-1, 1, (n, n, n)) for _ in range(3)]  # [z, y, x]
    ax, ay, az = a
    f = np.zeros((16, p * p * p), np.float32)

    def sh(x, axis):  # value at +1 along axis (periodic)
        return np.roll(x, -1, axis=axis)
    bx = (sh(az, 1) - az) - (sh(ay, 0) - ay)
    by = (sh(ax, 0) - ax) - (sh(az, 2) - az)
    bz = (sh(ay, 2) - ay) - (sh(ax, 1) - ax)
    for lane, b in ((4, bx), (5, by), (6, bz)):
        g = np.zeros((p, p, p), np.float32)
        g[1:-1, 1:-1, 1:-1] = b.astype(np.float32)
        f[lane] = g.reshape(-1)
    return f


def yee_fields(nx=64, ny=4, nz=4, mode=3):
    kx = 2 * math.pi * mode / nx
    f = np.zeros((16, (nx + 2) * (ny + 2) * (nz + 2)), np.float32)
    ix = np.arange(nx + 2)
    line = np.sin(kx * ix).astype(np.float32)
    f[2] = np.tile(line, (ny + 2) * (nz + 2))
    return f


def yee_projection(f, nx=64, ny=4, nz=4, mode=3):
    kx = 2 * math.pi * mode / nx
    ez = f[2].reshape(nz + 2, ny + 2, nx + 2)[1:-1, 1:-1, 1:-1].astype(np.float64)
    prof = np.sin(kx * np.arange(1, nx + 1))
    return float((ez * prof[None, None, :]).sum())


def yee_omega(series, dt=0.5, nx=64, mode=3):
    s = np.asarray(series, np.float64)
    num = float(((s[2:] + s[:-2]) * s[1:-1]).sum())
    den = float((2 * s[1:-1] * s[1:-1]).sum())
    c = max(-1.0, min(1.0, num / den))
    omega = math.acos(c) / dt
    kx = 2 * math.pi * mode / nx
    lhs = (math.sin(omega * dt / 2) / dt) ** 2
    rhs = math.sin(kx / 2) ** 2
    return omega, abs(lhs - rhs) / rhs


def energy_line(e_energy, dt=0.1):
    """Hann-windowed direct Fourier scan for the field-energy line
    (acceptance.cpp:311-330)."""
    e = np.asarray(e_energy, np.float64)
    n = e.size
    mean = e.mean()
    t = (np.arange(n) + 1) * dt
    win = 0.5 - 0.5 * np.cos(2 * math.pi * np.arange(n) / (n - 1))
    x = (e - mean) * win
    best_w, best = 0.0, -1.0
    for k in range(2001):
        w = 1.0 + 0.001 * k
        mag = abs(np.sum(x * np.exp(-1j * w * t)))
        if mag > best:
            best, best_w = mag, w
    return best_w


def growth_rate(e_energy, dt, lo_frac=1e-3, hi_frac=0.1):
    """Exponential growth rate of the field energy (2 gamma) by a log-linear
    fit over the window where it rises from hi_frac-decades above its start
    to hi_frac of its peak."""
    e = np.asarray(e_energy, np.float64)
    t = np.arange(e.size) * dt
    peak = int(np.argmax(e))
    top = e[peak]
    start = e[: max(2, peak // 4)].min()
    sel = np.where((e >= max(start * 30.0, top * lo_frac)) & (e <= top * hi_frac) & (np.arange(e.size) < peak))[0]
    if sel.size < 4:
        return float("nan"), 0, 0
    sl, _ = np.polyfit(t[sel], np.log(e[sel]), 1)
    return float(sl), int(sel[0]), int(sel[-1])


def two_stream_theory(v_drift_u=0.2, omega_p2_beam=0.5):
    """Maximum growth rate of the field energy (2 gamma_max) for two equal
    cold counter-streaming beams: gamma_max = omega_b / 2 with the beams'
    longitudinal (gamma^3) mass."""
    g = math.sqrt(1.0 + v_drift_u ** 2)
    wb = math.sqrt(omega_p2_beam / g ** 3)
    return 2 * (wb / 2)


def state_hash(species, fields):
    h = hashlib.sha256()
    for p, ids in species:
        h.update(np.ascontiguousarray(p, np.float32).tobytes())
        h.update(np.ascontiguousarray(ids, np.int32).tobytes())
    h.update(np.ascontiguousarray(fields, np.float32).tobytes())
    return h.hexdigest()


# ---- reference runs -------------------------------------------------------------
def run_gauss(ref):
    s = ref.sim(GAUSS_DECK)
    series = [s.diagnostics(False)["max_div_e_err"]]
    for k in range(1, 201):
        s.step_and_sort(1)
        if k % 10 == 0:
            series.append(s.diagnostics(True)["max_div_e_err"])
    worst = max(abs(series[i + 1] - series[i]) for i in range(len(series) - 1))
    return {"series": series, "worst_change": worst, "tol": 1e-5}


def run_divb(ref, orc):
    from oracle.bindings import Grid
    f = divb_fields()
    g = Grid(16, 16, 16, 1.0, 1.0, 1.0, 0.0)
    s = ref.sim(DIVB_DECK)
    g = s.grid
    orc.ghost_sync(g, f)
    maxb = float(np.abs(f[4:7]).max())
    s.set_fields(f)
    s.step(1000)
    d = s.diagnostics(True)
    return {"max_div_b": d["max_div_b_err"], "maxb": maxb, "tol_rel": 1e-6,
            "note": "the fp32 reference misses this threshold itself (proj/README.md:47-52)"}


def run_yee(ref, orc):
    s = ref.sim(YEE_DECK)
    f = yee_fields()
    orc.ghost_sync(s.grid, f)
    s.set_fields(f)
    series = [yee_projection(f)]
    for _ in range(200):
        s.step(1)
        series.append(yee_projection(s.fields()))
    omega, rel = yee_omega(series)
    return {"omega": omega, "rel": rel, "tol": 1e-3, "series": series}


def run_plasma(ref):
    s = ref.sim(plasma_deck())
    e = []
    for _ in range(2000):
        s.step_and_sort(1)
        e.append(s.diagnostics(False)["e_energy"])
    w = energy_line(e)
    return {"best_w": w, "rel": abs(w - 2.0) / 2.0, "tol": 0.03, "e_energy": e}


def run_energy(ref):
    s = ref.sim(ENERGY_DECK)
    tot = [s.diagnostics(False)["total_energy"]]
    for _ in range(500):
        s.step_and_sort(1)
        tot.append(s.diagnostics(False)["total_energy"])
    e0 = tot[50]
    worst = max(abs(tot[k + 1] - e0) for k in range(50, 500) if k % 25 == 0)
    return {"total": tot, "e0": e0, "worst": worst, "worst_rel": worst / e0, "tol_rel": 0.03}


def run_thermal(ref):
    s = ref.sim(bench_deck("thermal", deterministic=True, workers=WORKERS))
    out = {}
    for k in range(1, 22):
        s.step_and_sort(1)
        if k in (5, 21):
            sp = [s.species(i) for i in range(s.nspecies)]
            out[f"hash_{k}"] = state_hash(sp, s.fields())
    s2 = ref.sim(bench_deck("thermal", deterministic=True, workers=WORKERS))
    tot = [s2.diagnostics(False)["total_energy"]]
    for k in range(1, 201):
        s2.step_and_sort(1)
        if k % 10 == 0:
            tot.append(s2.diagnostics(False)["total_energy"])
    out["total_every_10"] = tot
    out["drift_rel"] = (tot[-1] - tot[0]) / tot[0]
    return out


def run_two_stream(ref):
    s = ref.sim(bench_deck("two_stream", deterministic=True, workers=WORKERS))
    e = [s.diagnostics(False)["e_energy"]]
    for k in range(1, 161):
        s.step_and_sort(1)
        e.append(s.diagnostics(False)["e_energy"])
    rate, i0, i1 = growth_rate(e, 0.25)
    return {"e_energy": e, "rate": rate, "window": [i0, i1], "theory_rate": two_stream_theory()}


def main():
    ref, orc = Ref(), Orc()
    out = {"generator": "tests/golden/make_acceptance.py", "reference": "oracle/_ref (minipic fp32)",
           "workers": WORKERS}
    which = sys.argv[1:] or ["gauss", "divb", "yee", "plasma", "energy", "thermal", "two_stream"]
    if os.path.exists(OUT):
        with open(OUT) as fh:
            out.update(json.load(fh))
    for name in which:
        fn = {"gauss": lambda: run_gauss(ref), "divb": lambda: run_divb(ref, orc), "yee": lambda: run_yee(ref, orc),
              "plasma": lambda: run_plasma(ref), "energy": lambda: run_energy(ref),
              "thermal": lambda: run_thermal(ref), "two_stream": lambda: run_two_stream(ref)}[name]
        out[name] = fn()
        brief = {k: v for k, v in out[name].items() if not isinstance(v, list)}
        print(name, brief, flush=True)
    with open(OUT, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
