"""Device diagnostics against the oracle restatement of
refresh_charge_diagnostics / current_diagnostics (proj/src/sim.cpp:230-266).

Bar: compute_div_errors and max_abs_lane bit-exact given the same inputs;
rho (float atomics, order not fixed) within RHO_RTOL x max|rho|; energies
(fp64 device sums vs the reference's fp32 strided partial sums) within
ENERGY_RTOL relative.
"""
import numpy as np
import pytest

from tests.helpers import assert_bitwise, assert_close, rand_fields, rand_particles

pytestmark = pytest.mark.gpu

RHO_RTOL = 1e-5
ENERGY_RTOL = 1e-5


@pytest.fixture(scope="module")
def pic():
    import paper_2102_13133_b200 as pic
    pic.lib()
    return pic


@pytest.fixture(scope="module")
def orc():
    from oracle.bindings import Orc
    return Orc()


def og(g):
    from oracle.bindings import Grid
    return Grid(g.nx, g.ny, g.nz, g.hx, g.hy, g.hz, g.dt)


CASES = [((6, 5, 4), (1.0, 1.0, 1.0), 3000, True), ((9, 7, 5), (1.0, 0.9, 1.2), 20000, False),
         ((2, 2, 2), (1.0, 1.0, 1.0), 50, True), ((16, 16, 16), (1.0, 1.0, 1.0), 131072, True)]


@pytest.mark.parametrize("dims,h,n,sort", CASES)
def test_rho_and_div_errors(pic, orc, dims, h, n, sort):
    g = pic.make_grid(dims, h, cfl_frac=0.8)
    o = og(g)
    rng = np.random.default_rng(3)
    f = rand_fields(g, rng, scale=0.4, sync=lambda gg, ff: orc.ghost_sync(o, ff))
    sp = [(-1.0, *rand_particles(g, rng, n, sort=sort)), (1.0, *rand_particles(g, rng, n // 3 + 1, sort=sort))]
    with pic.Context(g) as ctx:
        for si, (q, p, ids) in enumerate(sp):
            sid = ctx.add_species(f"s{si}", q, 1.0 if q < 0 else 100.0, ids.size)
            ctx.upload_species(sid, p, ids)
        ctx.upload_fields(f)
        ctx.refresh_charge_diagnostics()
        gf = ctx.download_fields()
        gmax_e = ctx.max_abs_lane(pic.F["div_e_err"])
        gmax_b = ctx.max_abs_lane(pic.F["div_b_err"])
    want = f.copy()
    want[pic.F["rhof"]] = 0
    for q, p, ids in sp:
        orc.deposit_rho(o, q, p, ids, want)
    orc.compute_div_errors(o, want)
    rho = pic.F["rhof"]
    assert_close(gf[rho], want[rho], RHO_RTOL, what="rhof")
    # div B: the stencil alone, bit-exact
    assert_bitwise(gf[pic.F["div_b_err"]], want[pic.F["div_b_err"]], "div_b_err")
    # div E - rho with the device's own rho: bit-exact stencil
    chk = gf.copy()
    orc.compute_div_errors(o, chk)
    assert_bitwise(gf[pic.F["div_e_err"]], chk[pic.F["div_e_err"]], "div_e_err stencil")
    assert_close(gf[pic.F["div_e_err"]], want[pic.F["div_e_err"]], 1e-5, what="div_e_err")
    # max_abs_lane: exact for the device's own lanes
    assert gmax_e == orc.max_abs_lane(o, gf, pic.F["div_e_err"])
    assert gmax_b == orc.max_abs_lane(o, gf, pic.F["div_b_err"])
    assert gmax_b == orc.max_abs_lane(o, want, pic.F["div_b_err"])


@pytest.mark.parametrize("dims,h,n,sort", CASES)
def test_energies(pic, orc, dims, h, n, sort):
    g = pic.make_grid(dims, h, cfl_frac=0.8)
    o = og(g)
    rng = np.random.default_rng(11)
    f = rand_fields(g, rng, scale=0.4, sync=lambda gg, ff: orc.ghost_sync(o, ff))
    q, m = -1.0, 1.0
    p, ids = rand_particles(g, rng, n, u_scale=0.7, sort=sort)
    with pic.Context(g) as ctx:
        sid = ctx.add_species("e", q, m, n)
        ctx.upload_species(sid, p, ids)
        ctx.upload_fields(f)
        ge, gb = ctx.field_energy()
        ctx.load_interpolators()
        gk = ctx.kinetic_energy(sid, centered=True)
        gk0 = ctx.kinetic_energy(sid, centered=False)
        d = ctx.diagnostics()
    we, wb = orc.field_energy(o, f)
    i18 = orc.load_interpolators(o, f)
    wk = orc.kinetic_energy_centered(o, q, m, p, ids, i18)
    g64 = np.sqrt(1.0 + (p[3].astype(np.float64) ** 2 + p[4] ** 2 + p[5] ** 2))
    wk0 = float(np.sum(p[6].astype(np.float64) * m * (g64 - 1.0)))
    for got, want, what in ((ge, we, "e_energy"), (gb, wb, "b_energy"), (gk, wk, "kinetic centred"),
                            (gk0, wk0, "kinetic")):
        assert abs(got - want) <= ENERGY_RTOL * abs(want), f"{what}: {got} vs {want}"
    assert d["e_energy"] == ge and d["b_energy"] == gb
    assert d["kinetic"][0] == gk
    assert d["particle_count"] == n
    assert abs(d["total_energy"] - (we + wb + wk)) <= ENERGY_RTOL * abs(we + wb + wk)


def test_diagnostics_track_a_run(pic, orc):
    """Energy history of a short e/i run: device diagnostics vs the oracle's
    functions on the oracle's own (deterministic-mode identical) state."""
    g = pic.make_grid((10, 8, 6), 1.0, dt=0.25)
    o = og(g)
    species = [(-1.0, 1.0, 6, 0.2, (0.05, 0.0, 0.0)), (1.0, 100.0, 4, 0.02, (0.0, 0.0, 0.0))]
    state = []
    for si, (q, m, ppc, uth, drift) in enumerate(species):
        p, ids = orc.load_species(o, 4, si, ppc, uth, drift)
        state.append((q, m, p, ids))
    f = np.zeros((16, g.padded), np.float32)
    with pic.Context(g) as ctx:
        for si, (q, m, p, ids) in enumerate(state):
            sid = ctx.add_species(f"s{si}", q, m, ids.size)
            ctx.upload_species(sid, p, ids)
        for step in range(4):
            ctx.step(deterministic=True)
            orc.step(o, state, f)
            ctx.refresh_charge_diagnostics()
            d = ctx.diagnostics()
            want = f.copy()
            want[pic.F["rhof"]] = 0
            for q, m, p, ids in state:
                orc.deposit_rho(o, q, p, ids, want)
            orc.compute_div_errors(o, want)
            we, wb = orc.field_energy(o, want)
            i18 = orc.load_interpolators(o, want)
            wk = [orc.kinetic_energy_centered(o, q, m, p, ids, i18) for q, m, p, ids in state]
            assert abs(d["e_energy"] - we) <= ENERGY_RTOL * abs(we) + 1e-30
            assert abs(d["b_energy"] - wb) <= ENERGY_RTOL * abs(wb) + 1e-30
            for a, b in zip(d["kinetic"], wk):
                assert abs(a - b) <= ENERGY_RTOL * abs(b)
            assert d["particle_count"] == sum(ids.size for _, _, _, ids in state)
            mb = orc.max_abs_lane(o, want, pic.F["div_b_err"])
            assert d["max_div_b_err"] == mb
            me = orc.max_abs_lane(o, want, pic.F["div_e_err"])
            assert abs(d["max_div_e_err"] - me) <= 1e-5 * max(me, 1e-6)
