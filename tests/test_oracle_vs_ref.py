"""Pins the plain-C oracle (oracle/pic_oracle.c) to the unmodified reference
(oracle/_ref: minipic compiled from /root/reference/proj sources, fp32):
bit-identical on every hot-path function, on the reference's own SimState
runs, and on the known-answer cases of the reference's test suite."""
import numpy as np
import pytest

from oracle.bindings import Grid, Orc, Ref, make_grid, ref_available
from tests.helpers import assert_bitwise, rand_particles

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference here)")


@pytest.fixture(scope="module")
def orc():
    return Orc()


@pytest.fixture(scope="module")
def ref():
    return Ref()


def rand_fields(g, rng, scale=0.5):
    f = np.zeros((16, g.padded), np.float32)
    for lane in (0, 1, 2, 4, 5, 6, 8, 9, 10):
        f[lane] = (rng.standard_normal(g.padded) * scale).astype(np.float32)
    return f


GRIDS = [((5, 4, 3), (1.0, 1.0, 1.0), 0.9), ((7, 6, 5), (0.7, 1.3, 0.9), 0.5), ((2, 2, 2), (1.0, 2.0, 0.5), 0.95)]


@pytest.mark.parametrize("dims,h,cfl", GRIDS)
def test_field_functions_bitwise(orc, ref, dims, h, cfl):
    g = make_grid(dims, h, cfl_frac=cfl)
    rng = np.random.default_rng(5)
    f = rand_fields(g, rng)
    a, b = f.copy(), f.copy()
    orc.ghost_sync(g, a)
    ref.ghost_sync(g, b)
    assert_bitwise(a, b, "ghost_sync")
    assert_bitwise(orc.load_interpolators(g, a), ref.load_interpolators(g, b), "load_interpolators")
    orc.advance_b(g, a, 0.5)
    ref.advance_b(g, b, 0.5)
    assert_bitwise(a, b, "advance_b")
    orc.advance_e(g, a)
    ref.advance_e(g, b)
    assert_bitwise(a, b, "advance_e")
    orc.clear_currents(g, a)
    ref.clear_currents(g, b)
    assert_bitwise(a, b, "clear_currents")


@pytest.mark.parametrize("dims", [(5, 4, 3), (2, 3, 2)])
def test_fold_unload_bitwise(orc, ref, dims):
    g = make_grid(dims, (1.0, 0.8, 1.2), cfl_frac=0.7)
    rng = np.random.default_rng(6)
    acc = rng.standard_normal((g.padded, 12)).astype(np.float32)
    a, b = acc.copy(), acc.copy()
    orc.ghost_fold(g, a)
    ref.ghost_fold(g, b)
    assert_bitwise(a, b, "ghost_fold")
    f = rand_fields(g, rng)
    fa, fb = f.copy(), f.copy()
    orc.unload(g, a, fa)
    ref.unload(g, b, fb)
    assert_bitwise(fa, fb, "unload")


@pytest.mark.parametrize("n,u", [(4000, 0.5), (2000, 3.0), (1, 0.1)])
@pytest.mark.parametrize("sort", [True, False])
def test_advance_particles_bitwise(orc, ref, n, u, sort):
    g = make_grid((6, 5, 4), 1.0, cfl_frac=0.9)
    rng = np.random.default_rng(7)
    f = rand_fields(g, rng, 0.4)
    orc.ghost_sync(g, f)
    interp = orc.load_interpolators(g, f)
    p, ids = rand_particles(g, rng, n, u_scale=u, sort=sort)
    pa, ia = p.copy(), ids.copy()
    acc_a = np.zeros((g.padded, 12), np.float32)
    orc.advance_particles(g, -1.0, 1.0, pa, ia, interp, acc_a)
    sb = ref.scatter(g, backend=2, workers=1)  # sequential backend
    pb, ib = p.copy(), ids.copy()
    ref.advance_particles(g, -1.0, 1.0, pb, ib, interp, sb)
    assert_bitwise(ia, ib, "ids")
    assert_bitwise(pa, pb, "lanes")
    assert_bitwise(acc_a, sb.reduce(), "accumulator")
    # the reference's deterministic (staged + replay) mode gives the same sums
    sd = ref.scatter(g, backend=0, workers=1)
    pc, ic = p.copy(), ids.copy()
    ref.advance_particles(g, -1.0, 1.0, pc, ic, interp, sd, deterministic=True)
    assert_bitwise(acc_a, sd.reduce(), "accumulator (reference deterministic)")


@pytest.mark.parametrize("interleaved", [False, True])
def test_sort_bitwise(orc, ref, interleaved):
    g = make_grid((7, 5, 4))
    rng = np.random.default_rng(8)
    p, ids = rand_particles(g, rng, 5000, sort=False)
    ids[:700] = ids[3]
    a, ia = p.copy(), ids.copy()
    b, ib = p.copy(), ids.copy()
    orc.sort(a, ia, interleaved)
    ref.sort(b, ib, interleaved)
    assert_bitwise(ia, ib, "ids")
    assert_bitwise(a, b, "lanes")


DECK = """[grid]
nx = 6
ny = 5
nz = 4
lx = 6
ly = 5
lz = 4
dt = 0.25
steps = 8
[species.electron]
q = -1
m = 1
ppc = 5
u_th = 0.3
drift = 0.05 0 0
perturb_ux = 0.02
perturb_kmode = 2
sort_interval = 3
[species.ion]
q = 1
m = 25
ppc = 3
u_th = 0.05
sort_interval = 4
sort_order = interleaved
[run]
seed = 17
"""


def test_simstate_steps_bitwise(orc, ref):
    """SimState::initialize + 8 steps of step() and the run-loop sort cadence,
    against the oracle's restatement (load, step, sort)."""
    sim = ref.sim(DECK)
    g = sim.grid
    species = [(-1.0, 1.0, 5, 0.3, (0.05, 0.0, 0.0), 0.02, 2, 3, False),
               (1.0, 25.0, 3, 0.05, (0.0, 0.0, 0.0), 0.0, 1, 4, True)]
    state = []
    for si, (q, m, ppc, uth, drift, pert, kmode, sint, inter) in enumerate(species):
        p, ids = orc.load_species(g, 17, si, ppc, uth, drift, pert, kmode)
        rp, rids = sim.species(si)
        assert_bitwise(p, rp, f"initial load species {si}")
        assert_bitwise(ids, rids, f"initial ids species {si}")
        state.append([q, m, p, ids, sint, inter])
    f = sim.fields()  # includes the initial charge diagnostics
    for step in range(1, 9):
        orc.step(g, [(s[0], s[1], s[2], s[3]) for s in state], f)
        for s in state:
            if step % s[4] == 0:
                orc.sort(s[2], s[3], s[5])
        sim.step_and_sort(1)
        assert_bitwise(f, sim.fields(), f"fields after step {step}")
        for si, s in enumerate(state):
            rp, rids = sim.species(si)
            assert_bitwise(s[3], rids, f"ids species {si} step {step}")
            assert_bitwise(s[2], rp, f"lanes species {si} step {step}")


def test_diagnostics_bitwise(orc, ref):
    g = make_grid((5, 4, 6), (1.0, 0.9, 1.1), cfl_frac=0.6)
    rng = np.random.default_rng(9)
    f = rand_fields(g, rng)
    orc.ghost_sync(g, f)
    p, ids = rand_particles(g, rng, 3000, u_scale=0.4)
    fa, fb = f.copy(), f.copy()
    orc.deposit_rho(g, -1.0, p, ids, fa)
    ref.deposit_rho(g, -1.0, p, ids, fb)
    assert_bitwise(fa, fb, "deposit_rho")
    orc.compute_div_errors(g, fa)
    ref.compute_div_errors(g, fb)
    assert_bitwise(fa, fb, "compute_div_errors")
    assert_bitwise(orc.field_energy(g, fa), ref.field_energy(g, fb), "field_energy")
    i18 = orc.load_interpolators(g, fa)
    assert np.float32(orc.kinetic_energy_centered(g, -1.0, 1.0, p, ids, i18)).view(np.uint32) == \
        np.float32(ref.kinetic_energy_centered(g, -1.0, 1.0, p, ids, i18)).view(np.uint32)
    for lane in (3, 7):
        assert orc.max_abs_lane(g, fa, lane) == ref.max_abs_lane(g, fb, lane)


def test_cfl_violation_is_run_abort_in_both(orc, ref):
    from oracle.bindings import RunAbort
    g = make_grid((4, 4, 4), 1.0, cfl_frac=0.5)
    interp = np.zeros((18, g.padded), np.float32)
    p = np.zeros((7, 1), np.float32)
    p[3, 0] = np.nan
    p[6, 0] = 1
    ids = np.array([g.voxel(2, 2, 2)], np.int32)
    with pytest.raises(RunAbort):
        orc.advance_particles(g, 1.0, 1.0, p.copy(), ids.copy(), interp, np.zeros((g.padded, 12), np.float32))
    with pytest.raises(RunAbort):
        ref.advance_particles(g, 1.0, 1.0, p.copy(), ids.copy(), interp, ref.scatter(g))
