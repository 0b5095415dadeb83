"""The reference's physics acceptance criteria on the FAST (benchmarked) GPU
path — hardware float atomics, continuous voxel order — each held to the
reference's own threshold AND to the reference's own value on the same deck
(tests/golden/acceptance_ref.json, made by tests/golden/make_acceptance.py
from the unmodified reference, oracle/_ref).

  gauss      acceptance.cpp:87-134   Gauss residual constancy over 200 steps
  divb       acceptance.cpp:137-204  div B after 1000 field-only steps
  yee        acceptance.cpp:207-285  vacuum Yee dispersion
  plasma     acceptance.cpp:288-336  field energy line at 2 omega_p
  continuity acceptance.cpp:563-661  node d(rho)/dt + div J = 0, 1000 moves
  energy     test_sim.cpp:371-412    total energy bounded over 500 steps
  thermal    SURVEY §8d C1 (64^3, 32 ppc e/i): deterministic state bitwise
             after 5 and 21 steps; 200 fast steps' energy drift
  two_stream configs[1] at 64^3: field-energy growth rate vs the reference
             and cold-beam theory

Field-only criteria (divb, yee) run the deterministic stencils: the values
are bit-identical to the reference's.  Particle criteria differ from the
reference only by the atomics' summation order; scalars that are physical
(energy line, energies, growth rate) are compared with the reference's
within the stated relative tolerances.
"""
import json
import os

import numpy as np
import pytest

from tests.golden import make_acceptance as A

pytestmark = pytest.mark.gpu

REF = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "acceptance_ref.json")))


@pytest.fixture(scope="module")
def pic():
    import paper_2102_13133_b200 as pic
    pic.lib()
    return pic


@pytest.fixture(scope="module")
def orc():
    from oracle.bindings import Orc
    return Orc()


def sim_of(text):
    from paper_2102_13133_b200.simstate import Deck, SimState
    return SimState(Deck(text))


def test_gauss_residual_constancy(pic):
    r = REF["gauss"]
    with sim_of(A.GAUSS_DECK) as s:
        ctx = s.context
        series = [ctx.diagnostics()["max_div_e_err"]]
        for k in range(1, 201):
            s.step()
            if k % 10 == 0:
                s.refresh_charge_diagnostics()
                series.append(ctx.diagnostics()["max_div_e_err"])
    worst = max(abs(series[i + 1] - series[i]) for i in range(len(series) - 1))
    assert worst <= r["tol"], (worst, r["worst_change"])
    # the residual itself (div E - rho at the worst node) tracks the reference's
    np.testing.assert_allclose(series, r["series"], rtol=1e-5)


def test_div_b_preservation(pic, orc):
    r = REF["divb"]
    with sim_of(A.DIVB_DECK) as s:
        ctx = s.context
        f = A.divb_fields()
        orc.ghost_sync(_og(ctx.grid), f)
        ctx.upload_fields(f)
        for _ in range(1000):
            s.step()
        s.refresh_charge_diagnostics()
        got = ctx.diagnostics()["max_div_b_err"]
    # deterministic stencils: the reference's own value, bit for bit (the
    # fp32 reference misses the 1e-6 max|B| criterion itself, README:47-52)
    assert np.float32(got) == np.float32(r["max_div_b"]), (got, r["max_div_b"])
    assert got <= 1e-5 * r["maxb"]


def _og(g):
    from oracle.bindings import Grid
    return Grid(g.nx, g.ny, g.nz, g.hx, g.hy, g.hz, g.dt)


def test_yee_dispersion(pic, orc):
    r = REF["yee"]
    with sim_of(A.YEE_DECK) as s:
        ctx = s.context
        f = A.yee_fields()
        orc.ghost_sync(_og(ctx.grid), f)
        ctx.upload_fields(f)
        series = [A.yee_projection(f)]
        for _ in range(200):
            s.step()
            series.append(A.yee_projection(ctx.download_fields()))
    omega, rel = A.yee_omega(series)
    assert rel <= r["tol"]
    assert series == r["series"]  # bit-identical fields give identical projections
    assert omega == r["omega"]


def test_plasma_oscillation_line(pic):
    r = REF["plasma"]
    with sim_of(A.plasma_deck()) as s:
        ctx = s.context
        e = []
        for _ in range(2000):
            s.step()
            e.append(ctx.field_energy()[0])
    w = A.energy_line(e)
    assert abs(w - 2.0) / 2.0 <= r["tol"], w
    assert abs(w - r["best_w"]) <= 1e-3 * r["best_w"] + 1e-3, (w, r["best_w"])  # one scan bin
    # the oscillation's energy history itself (a smooth 2 omega_p line): within
    # a percent of the reference's over the run (roundoff grows chaotically)
    ref = np.asarray(r["e_energy"])
    assert np.abs(np.asarray(e) - ref).max() <= 0.02 * ref.max()


def test_total_energy_bounded(pic):
    r = REF["energy"]
    with sim_of(A.ENERGY_DECK) as s:
        ctx = s.context
        tot = [ctx.diagnostics()["total_energy"]]
        for _ in range(500):
            s.step()
            tot.append(ctx.diagnostics()["total_energy"])
    e0 = tot[50]
    worst = max(abs(tot[k + 1] - e0) for k in range(50, 500) if k % 25 == 0)
    assert worst <= r["tol_rel"] * e0
    # drift within the reference's (north_star): at most 10 % above it, or
    # 1e-4 of the energy when both are at the roundoff floor
    assert worst <= 1.1 * r["worst"] + 1e-4 * e0, (worst / e0, r["worst_rel"])
    np.testing.assert_allclose(tot, r["total"], rtol=1e-3)


def test_deposition_continuity(pic, orc):
    """1000 random single-particle moves (speeds up to 0.98 c, any direction,
    random charge) on a 4^3 periodic grid, dt 0.4, zero fields: the node
    charge change and the divergence of the unloaded current cancel to 1e-5
    (acceptance.cpp:563-661); the oracle's residual (the reference's exact
    summation order) is computed for the same moves."""
    g = pic.make_grid((4, 4, 4), 1.0, dt=0.4)
    o = _og(g)
    rng = np.random.default_rng(515)
    nodes = 64
    worst = worst_orc = 0.0

    def trilinear(ix, iy, iz, x, y, z, qw):
        out = np.zeros(nodes)
        f = qw / 8.0
        for sx in (0, 1):
            for sy in (0, 1):
                for sz in (0, 1):
                    cx = ix % 4 + 1 if sx else ix
                    cy = iy % 4 + 1 if sy else iy
                    cz = iz % 4 + 1 if sz else iz
                    out[(cz - 1) * 16 + (cy - 1) * 4 + (cx - 1)] += (f * ((1 + x) if sx else (1 - x))
                                                                    * ((1 + y) if sy else (1 - y))
                                                                    * ((1 + z) if sz else (1 - z)))
        return out

    def residual(f16, q, p0, p1, v0, v1):
        c0, c1 = o.coords(int(v0)), o.coords(int(v1))
        rb = trilinear(*c0, *[float(t) for t in p0[:3]], q)
        ra = trilinear(*c1, *[float(t) for t in p1[:3]], q)
        jx = f16[8].reshape(6, 6, 6).astype(np.float64)
        jy = f16[9].reshape(6, 6, 6).astype(np.float64)
        jz = f16[10].reshape(6, 6, 6).astype(np.float64)
        w = 0.0
        lo = lambda i: 4 if i == 1 else i - 1  # noqa: E731
        for kz in range(1, 5):
            for ky in range(1, 5):
                for kx in range(1, 5):
                    divj = ((jx[kz, ky, kx] - jx[kz, ky, lo(kx)]) + (jy[kz, ky, kx] - jy[kz, lo(ky), kx])
                            + (jz[kz, ky, kx] - jz[lo(kz), ky, kx]))
                    node = (kz - 1) * 16 + (ky - 1) * 4 + (kx - 1)
                    w = max(w, abs((ra[node] - rb[node]) / 0.4 + divj))
        return w

    zero_f = np.zeros((16, g.padded), np.float32)
    interp = orc.load_interpolators(o, zero_f)
    with pic.Context(g) as ctx:
        for trial in range(1000):
            q = float(rng.uniform(-1, 1))
            v = rng.uniform(-0.9, 0.9, 3)
            vv = min(0.98, float(np.sqrt((v * v).sum())))
            gm = 1.0 / np.sqrt(1 - vv * vv)
            p = np.zeros((7, 1), np.float32)
            p[0:3, 0] = rng.uniform(-1, 1, 3)
            p[3:6, 0] = v * gm
            p[6, 0] = 1.0
            ids = np.array([g.voxel(*(int(t) for t in 1 + rng.integers(0, 4, 3)))], np.int32)
            sid = ctx.add_species(f"p{trial}", q, 1.0, 1)  # one species per move (its own charge)
            ctx.upload_species(sid, p, ids)
            ctx.upload_fields(zero_f)
            ctx.load_interpolators()
            ctx.clear_accumulator()
            ctx.advance_p(sid)
            ctx.ghost_fold_currents()
            ctx.clear_currents()
            ctx.unload_currents()
            gp, gids = ctx.download_species(sid)
            f16 = ctx.download_fields()
            worst = max(worst, residual(f16, q, p[:, 0], gp[:, 0], ids[0], gids[0]))
            # the oracle on the same move
            op, oids = p.copy(), ids.copy()
            acc = np.zeros((g.padded, 12), np.float32)
            orc.advance_particles(o, q, 1.0, op, oids, interp, acc, False)
            orc.ghost_fold(o, acc)
            of = np.zeros((16, g.padded), np.float32)
            orc.unload(o, acc, of)
            worst_orc = max(worst_orc, residual(of, q, p[:, 0], op[:, 0], ids[0], oids[0]))
    assert worst <= 1e-5, (worst, worst_orc)
    assert worst_orc <= 1e-5


def _hash_sim(s):
    ctx = s.context
    sp = [ctx.download_species(i) for i in range(len(ctx.species_names))]
    return A.state_hash(sp, ctx.download_fields())


def test_thermal_c1_deterministic_bitwise(pic):
    """SURVEY §8d C1 (the thermal deck of bench.py at 64^3, 32 ppc each of
    electrons and ions, 16.8 M particles) in deterministic mode: the whole
    state — every particle record and every field lane — is bit-identical to
    the reference after 5 steps and after 21 (sort at 20)."""
    r = REF["thermal"]
    with sim_of(A.bench_deck("thermal", deterministic=True)) as s:
        for k in range(1, 22):
            s.step()
            if k in (5, 21):
                assert _hash_sim(s) == r[f"hash_{k}"], f"state differs from the reference after {k} steps"


def test_thermal_c1_fast_energy_drift(pic):
    """C1 over 200 fast steps (sorts every 20): the total energy history
    stays within 1e-3 of the reference's and its drift within the
    reference's drift x 1.1 (+ 1e-4 of the energy at the roundoff floor)."""
    r = REF["thermal"]
    with sim_of(A.bench_deck("thermal")) as s:
        ctx = s.context
        tot = [ctx.diagnostics()["total_energy"]]
        for k in range(1, 201):
            s.step()
            if k % 10 == 0:
                tot.append(ctx.diagnostics()["total_energy"])
    drift = (tot[-1] - tot[0]) / tot[0]
    np.testing.assert_allclose(tot, r["total_every_10"], rtol=1e-3)
    assert abs(drift) <= 1.1 * abs(r["drift_rel"]) + 1e-4, (drift, r["drift_rel"])


def test_two_stream_growth_rate(pic):
    """configs[1] (two counter-streaming electron beams, 32 ppc each, u = 0.2)
    at 64^3: the field energy's exponential growth rate within 5 % of the
    reference's on the same deck and within 30 % of cold-beam theory
    (2 gamma_max = omega_b with the beams' gamma^3 mass; the grid's finite
    k resolution near the fastest mode lowers the measured rate)."""
    r = REF["two_stream"]
    with sim_of(A.bench_deck("two_stream")) as s:
        ctx = s.context
        e = [ctx.field_energy()[0]]
        for _ in range(160):
            s.step()
            e.append(ctx.field_energy()[0])
    rate, i0, i1 = A.growth_rate(e, 0.25)
    assert abs(rate - r["rate"]) <= 0.05 * r["rate"], (rate, r["rate"], (i0, i1), r["window"])
    assert abs(rate - r["theory_rate"]) <= 0.30 * r["theory_rate"], (rate, r["theory_rate"])
