"""Non-periodic x boundaries, laser and emitter (csrc/boundary.cu; SURVEY §8f
item 4).  NOT IN REFERENCE — minipic is periodic only — so the checks are
self-consistency properties, exact where the geometry allows:

* reflect: a ballistic particle that crosses a reflecting wall ends as the
  exact mirror image (cell, x offset, u_x) of the same particle in the
  periodic run of the CPU restatement — bit for bit, fast and deterministic
  paths;
* absorb: the particles that wrapped in the periodic run are exactly the
  ones removed, per side; the survivors are bit-identical;
* charge conservation: with reflecting walls and real charges, Gauss's law
  residual div E - rho stays fixed at every node off the wall planes (the
  mirror fold of the current beyond the wall is charge-conserving);
* PEC reflects a pulse with its energy and a sign flip of E_y; Mur absorbs
  it; the laser source radiates ~e0 and its front moves at c;
* the emitter injects per_cell particles per boundary cell per step,
  inside the boundary layer, moving inward.
"""
import numpy as np
import pytest

from paper_2102_13133_b200 import F, FBC_MUR, FBC_PEC, PBC_ABSORB, PBC_REFLECT

pytestmark = pytest.mark.gpu


def _og(g):
    from oracle.bindings import Grid
    return Grid(g.nx, g.ny, g.nz, g.hx, g.hy, g.hz, g.dt)


def _ballistic_state(g, n, seed, ux_scale=0.25):
    """Particles with unique weight tags and x-dominated momenta; charge so
    small that the fields they raise cannot change u (|kick| << ulp(u))."""
    rng = np.random.default_rng(seed)
    ix = rng.integers(1, g.nx + 1, n)
    iy = rng.integers(1, g.ny + 1, n)
    iz = rng.integers(1, g.nz + 1, n)
    ids = (ix + (g.nx + 2) * (iy + (g.ny + 2) * iz)).astype(np.int32)
    p = np.zeros((7, n), np.float32)
    p[0:3] = rng.uniform(-1, 1, (3, n)).astype(np.float32)
    p[3] = (ux_scale * rng.standard_normal(n)).astype(np.float32)
    p[4:6] = (0.02 * rng.standard_normal((2, n))).astype(np.float32)
    p[6] = (1.0 + np.arange(n) * 2.0 ** -23).astype(np.float32)
    return p, ids


Q, M = -1e-20, 1.0 / 64  # |q dt / 2m| = 8e-20: inside the call-free push's range


def _periodic_reference(g, p, ids, steps):
    """CPU restatement, periodic box; returns final (p, ids) and the net x
    wrap count of every particle (+1 through the high face, -1 low)."""
    from oracle.bindings import Orc
    orc = Orc()
    og = _og(g)
    state = [(Q, M, p.copy(), ids.copy())]
    f = np.zeros((16, g.padded), np.float32)
    wraps = np.zeros(ids.size, np.int64)
    for _ in range(steps):
        ix0 = state[0][3] % (g.nx + 2)
        orc.step(og, state, f)
        ix1 = state[0][3] % (g.nx + 2)
        wraps += ((ix0 == g.nx) & (ix1 == 1)).astype(np.int64) - ((ix0 == 1) & (ix1 == g.nx)).astype(np.int64)
    return state[0][2], state[0][3], wraps


def _by_tag(p, ids):
    o = np.argsort(p[6].view(np.uint32), kind="stable")
    return p[:, o], ids[o]


@pytest.mark.parametrize("deterministic", [False, True])
def test_reflect_is_mirror_of_periodic(deterministic):
    import paper_2102_13133_b200 as pic
    g = pic.make_grid((7, 3, 4), 1.0, dt=0.25)
    p, ids = _ballistic_state(g, 3000, seed=1)
    steps = 16
    want_p, want_ids, wraps = _periodic_reference(g, p, ids, steps)
    assert (np.abs(wraps) <= 1).all() and (wraps != 0).sum() > 50
    with pic.Context(g) as ctx:
        ctx.set_x_boundary(0, PBC_REFLECT, FBC_PEC)
        ctx.set_x_boundary(1, PBC_REFLECT, FBC_PEC)
        sid = ctx.add_species("e", Q, M, ids.size)
        ctx.upload_species(sid, p, ids)
        for _ in range(steps):
            ctx.step(deterministic=deterministic)
        gp, gids = ctx.download_species(sid)
    assert gids.size == ids.size
    gp, gids = _by_tag(gp, gids)
    pitch = g.nx + 2
    ix_w = want_ids % pitch
    rest = want_ids - ix_w
    exp_ix = np.where(wraps == 1, g.nx + 1 - ix_w, np.where(wraps == -1, g.nx + 1 - ix_w, ix_w))
    exp_ids = (rest + exp_ix).astype(np.int32)
    exp_p = want_p.copy()
    m = wraps != 0
    exp_p[0, m] = -want_p[0, m]
    exp_p[3, m] = -want_p[3, m]
    assert (gids == exp_ids).all()
    assert (gp.view(np.uint32) == exp_p.view(np.uint32)).all()


def test_absorb_removes_exactly_the_leavers():
    import paper_2102_13133_b200 as pic
    g = pic.make_grid((7, 3, 4), 1.0, dt=0.25)
    p, ids = _ballistic_state(g, 3000, seed=2)
    steps = 16
    want_p, want_ids, wraps = _periodic_reference(g, p, ids, steps)
    with pic.Context(g) as ctx:
        ctx.set_x_boundary(0, PBC_ABSORB, FBC_MUR)
        ctx.set_x_boundary(1, PBC_ABSORB, FBC_MUR)
        sid = ctx.add_species("e", Q, M, ids.size)
        ctx.upload_species(sid, p, ids)
        for _ in range(steps):
            ctx.step()
        lo, hi = ctx.absorbed_counts()
        gp, gids = ctx.download_species(sid)
    keep = wraps == 0
    assert (lo, hi) == (int((wraps == -1).sum()), int((wraps == 1).sum()))
    assert gids.size == keep.sum()
    gp, gids = _by_tag(gp, gids)
    assert (gids == want_ids[keep]).all()
    assert (gp.view(np.uint32) == want_p[:, keep].view(np.uint32)).all()


def test_reflect_conserves_charge():
    """Thermal e/i plasma between reflecting conductor walls: div E - rho is
    constant in time at every node off the two wall planes."""
    import paper_2102_13133_b200 as pic
    g = pic.make_grid((12, 6, 5), 1.0, dt=0.25)
    with pic.Context(g) as ctx:
        ctx.set_x_boundary(0, PBC_REFLECT, FBC_PEC)
        ctx.set_x_boundary(1, PBC_REFLECT, FBC_PEC)
        e = ctx.add_species("e", -1.0 / 16, 1.0 / 16, 16 * g.interior)
        i = ctx.add_species("i", 1.0 / 16, 25.0 / 16, 16 * g.interior)
        ctx.load_synthetic(e, 16, 0.3, seed=3)
        ctx.load_synthetic(i, 16, 0.05, seed=4)

        def residual():
            ctx.refresh_charge_diagnostics()
            r = ctx.download_fields()[F["div_e_err"]].reshape(g.nz + 2, g.ny + 2, g.nx + 2)
            return r[1:-1, 1:-1, 2:g.nx + 1].astype(np.float64)  # nodes 2..nx

        r0 = residual()
        for _ in range(60):
            ctx.step()
        r1 = residual()
        n = ctx.species_count(e) + ctx.species_count(i)
    assert n == 32 * g.interior
    assert np.abs(r0).max() > 0
    assert np.abs(r1 - r0).max() <= 1e-4 * np.abs(r0).max(), np.abs(r1 - r0).max() / np.abs(r0).max()


def _pulse(g, x0, sigma, amp=1e-2):
    """+x travelling E_y / B_z Gaussian pulse (c = 1: cB_z = E_y), uniform in y, z."""
    f = np.zeros((16, g.padded), np.float32)
    ey = f[F["ey"]].reshape(g.nz + 2, g.ny + 2, g.nx + 2)
    bz = f[F["cbz"]].reshape(g.nz + 2, g.ny + 2, g.nx + 2)
    xe = (np.arange(g.nx + 2) - 1) * g.hx          # E_y node planes
    xb = (np.arange(g.nx + 2) - 0.5) * g.hx        # B_z cell centres
    ey[:] = (amp * np.exp(-((xe - x0) / sigma) ** 2))[None, None, :]
    bz[:] = (amp * np.exp(-((xb - x0) / sigma) ** 2))[None, None, :]
    ey[:, :, 0] = 0
    bz[:, :, 0] = 0
    return f


def _energy(ctx):
    e, b = ctx.field_energy()
    return e + b


@pytest.mark.parametrize("fbc", [FBC_PEC, FBC_MUR])
def test_pulse_at_conductor_and_absorber(fbc):
    import paper_2102_13133_b200 as pic
    g = pic.make_grid((160, 2, 2), 1.0, dt=0.5)
    with pic.Context(g) as ctx:
        ctx.set_x_boundary(0, PBC_ABSORB, fbc)
        ctx.set_x_boundary(1, PBC_ABSORB, fbc)
        ctx.upload_fields(_pulse(g, 100.0, 6.0))
        e0 = _energy(ctx)
        for _ in range(200):  # front reaches x = 160 at t ~ 60 - 80; back at ~ 100
            ctx.step()
        e1 = _energy(ctx)
        ey = ctx.download_fields()[F["ey"]].reshape(g.nz + 2, g.ny + 2, g.nx + 2)[1, 1, 1:-1]
    if fbc == FBC_PEC:
        assert abs(e1 - e0) <= 0.02 * e0, (e0, e1)
        # reflected pulse moving -x, inverted: centre near 160 - (100 - 60) = 120
        k = int(np.argmax(np.abs(ey)))
        assert 105 <= k <= 135 and ey[k] < 0, (k, ey[k])
    else:
        assert e1 <= 0.02 * e0, (e0, e1)


def test_laser_amplitude_and_front():
    import paper_2102_13133_b200 as pic
    g = pic.make_grid((240, 2, 2), 1.0, dt=0.5)
    e0, omega, ix = 1e-2, 0.6, 40
    with pic.Context(g) as ctx:
        ctx.set_x_boundary(0, PBC_ABSORB, FBC_MUR)
        ctx.set_x_boundary(1, PBC_ABSORB, FBC_MUR)
        ctx.set_laser(ix, e0, omega, pol=1, ramp_steps=20)
        for _ in range(200):  # t = 100: front at x ~ 39 + 100 = 139
            ctx.step()
        ey = ctx.download_fields()[F["ey"]].reshape(g.nz + 2, g.ny + 2, g.nx + 2)[1, 1, 1:-1]
    x = np.arange(g.nx) * g.hx
    behind = (x > 60) & (x < 120)
    ahead = x > 150
    amp = np.abs(ey[behind]).max()
    assert abs(amp - e0) <= 0.1 * e0, amp
    assert np.abs(ey[ahead]).max() <= 0.02 * e0


def test_emitter_injects_inward():
    import paper_2102_13133_b200 as pic
    g = pic.make_grid((16, 4, 3), 1.0, dt=0.25)
    with pic.Context(g) as ctx:
        ctx.set_x_boundary(0, PBC_ABSORB, FBC_MUR)
        ctx.set_x_boundary(1, PBC_ABSORB, FBC_MUR)
        sid = ctx.add_species("e", -1.0 / 64, 1.0 / 64, 100000)
        ctx.set_emitter(sid, 0, 5, 0.05, (0.1, 0.0, 0.0), seed=9)
        ctx.step()
        p1, ids1 = ctx.download_species(sid)
        ctx.step()
        n2 = ctx.species_count(sid)
    assert ids1.size == 5 * g.ny * g.nz
    assert n2 == 2 * ids1.size
    assert (ids1 % (g.nx + 2) == 1).all()
    assert (p1[3] > 0).all()
    assert (np.abs(p1[0:3]) <= 1).all()


def test_walls_usage_errors():
    import paper_2102_13133_b200 as pic
    g = pic.make_grid((6, 3, 3), 1.0, dt=0.25)
    with pic.Context(g) as ctx:
        with pytest.raises(pic.UsageError):
            ctx.set_x_boundary(0, PBC_REFLECT, 0)  # particles walled, fields periodic
        ctx.set_x_boundary(0, PBC_REFLECT, FBC_PEC)
        ctx.add_species("e", -1.0, 1.0, 10)
        with pytest.raises(pic.UsageError):
            ctx.step()  # only one side walled
        ctx.set_x_boundary(1, PBC_ABSORB, FBC_MUR)
        ctx.step()
        with pytest.raises(pic.UsageError):
            ctx.set_x_open(False)  # walls need the x faces open


# --------------------------------------------------------------------- decomposed
def _decomposed(world, NX, NY, NZ, walls, dt, h=1.0):
    from paper_2102_13133_b200.domain import CudaSlab, DecomposedSim, LocalTransport, SlabGeometry
    geom = SlabGeometry(NX, NY, NZ, world=world, h=(h,) * 3, dt=dt, walls=walls)
    slabs = {r: CudaSlab(geom.local_grid(), r, r == 0, walls=walls, world=world) for r in range(world)}
    return geom, slabs, DecomposedSim(geom, slabs, LocalTransport())


@pytest.mark.parametrize("world", [2, 4])
def test_decomposed_laser_between_mur_walls_matches_single_domain(world):
    """No particles: the decomposed field solve with the global Mur walls and
    the laser on one slab equals the single-domain run bit for bit."""
    import paper_2102_13133_b200 as pic
    NX, NY, NZ, dt = 96, 3, 2, 0.5
    g = pic.make_grid((NX, NY, NZ), 1.0, dt=dt)
    with pic.Context(g) as ctx:
        ctx.set_x_boundary(0, PBC_ABSORB, FBC_MUR)
        ctx.set_x_boundary(1, PBC_ABSORB, FBC_MUR)
        ctx.set_laser(30, 1e-2, 0.6, pol=2, ramp_steps=10, waist=1.5, y0=1.5, z0=1.0)
        for _ in range(150):
            ctx.step()
        want = ctx.download_fields()
    geom, slabs, sim = _decomposed(world, NX, NY, NZ, (PBC_ABSORB, FBC_MUR), dt)
    sim.set_laser(30, 1e-2, 0.6, pol=2, ramp_steps=10, waist=1.5, y0=1.5, z0=1.0)
    for _ in range(150):
        sim.step()
    got = geom.join_fields([slabs[r].ctx.download_fields() for r in range(world)])
    for e in slabs.values():
        e.ctx.close()
    for name in ("ex", "ey", "ez", "cbx", "cby", "cbz"):
        a = got[F[name]].reshape(NZ + 2, NY + 2, NX + 2)[1:-1, 1:-1, 1:-1]
        b = want[F[name]].reshape(NZ + 2, NY + 2, NX + 2)[1:-1, 1:-1, 1:-1]
        assert (a.view(np.uint32) == b.view(np.uint32)).all(), name
    assert np.abs(want[F["ez"]]).max() > 1e-3


@pytest.mark.parametrize("pbc", [PBC_REFLECT, PBC_ABSORB])
def test_decomposed_walls_particles(pbc):
    """Ballistic particles across 3 slabs with global walls: reflection is the
    exact mirror of the periodic run, absorption removes exactly the leavers."""
    g_nx, ny, nz = 9, 3, 4
    import paper_2102_13133_b200 as pic
    g = pic.make_grid((g_nx, ny, nz), 1.0, dt=0.25)
    p, ids = _ballistic_state(g, 3000, seed=5)
    steps = 16
    want_p, want_ids, wraps = _periodic_reference(g, p, ids, steps)
    geom, slabs, sim = _decomposed(3, g_nx, ny, nz, (pbc, FBC_PEC if pbc == PBC_REFLECT else FBC_MUR), 0.25)
    sid = sim.add_species("e", Q, M, ids.size)
    for r, part in enumerate(geom.split(p, ids)):
        slabs[r].ctx.upload_species(sid, *part)
    for _ in range(steps):
        sim.step()
    parts = [slabs[r].ctx.download_species(sid) for r in range(3)]
    gp = np.concatenate([q for q, _ in parts], axis=1)
    gids = np.concatenate([geom.to_global_ids(r, parts[r][1]) for r in range(3)])
    for e in slabs.values():
        e.ctx.close()
    gp, gids = _by_tag(gp, gids)
    if pbc == PBC_ABSORB:
        keep = wraps == 0
        assert sim.absorbed == [int((wraps == -1).sum()), int((wraps == 1).sum())]
        assert (gids == want_ids[keep]).all()
        assert (gp.view(np.uint32) == want_p[:, keep].view(np.uint32)).all()
    else:
        pitch = g.nx + 2
        ix_w = want_ids % pitch
        exp_ids = np.where(wraps != 0, want_ids - ix_w + (g.nx + 1 - ix_w), want_ids).astype(np.int32)
        exp_p = want_p.copy()
        m = wraps != 0
        exp_p[0, m] = -want_p[0, m]
        exp_p[3, m] = -want_p[3, m]
        assert (gids == exp_ids).all()
        assert (gp.view(np.uint32) == exp_p.view(np.uint32)).all()


# ------------------------------------------------------------------ y / z walls
def _ballistic_axis(g, n, seed, axis):
    """Ballistic particles moving mostly along `axis` (see _ballistic_state)."""
    p, ids = _ballistic_state(g, n, seed)
    p[[3, 3 + axis]] = p[[3 + axis, 3]]
    return p, ids


def _periodic_reference_axis(g, p, ids, steps, axis):
    from oracle.bindings import Orc
    orc = Orc()
    og = _og(g)
    state = [(Q, M, p.copy(), ids.copy())]
    f = np.zeros((16, g.padded), np.float32)
    n = (g.nx, g.ny, g.nz)[axis]
    pitch = (1, g.nx + 2, (g.nx + 2) * (g.ny + 2))[axis]
    size = (g.nx + 2, g.ny + 2, g.nz + 2)[axis]
    coord = lambda i: (i // pitch) % size  # noqa: E731
    wraps = np.zeros(ids.size, np.int64)
    for _ in range(steps):
        c0 = coord(state[0][3])
        orc.step(og, state, f)
        c1 = coord(state[0][3])
        wraps += ((c0 == n) & (c1 == 1)).astype(np.int64) - ((c0 == 1) & (c1 == n)).astype(np.int64)
    return state[0][2], state[0][3], wraps


@pytest.mark.parametrize("axis", [1, 2])
@pytest.mark.parametrize("pbc", [PBC_REFLECT, PBC_ABSORB])
def test_yz_walls_exact(axis, pbc):
    """Walls on the y or z faces: reflection is the bit-exact mirror of the
    periodic run along that axis, absorption removes exactly the leavers."""
    import paper_2102_13133_b200 as pic
    g = pic.make_grid((4, 6, 5) if axis == 1 else (4, 3, 6), 1.0, dt=0.25)
    p, ids = _ballistic_axis(g, 3000, seed=7 + axis, axis=axis)
    steps = 16
    want_p, want_ids, wraps = _periodic_reference_axis(g, p, ids, steps, axis)
    assert (np.abs(wraps) <= 1).all() and (wraps != 0).sum() > 50
    with pic.Context(g) as ctx:
        fbc = FBC_PEC if pbc == PBC_REFLECT else FBC_MUR
        ctx.set_boundary(2 * axis, pbc, fbc)
        ctx.set_boundary(2 * axis + 1, pbc, fbc)
        sid = ctx.add_species("e", Q, M, ids.size)
        ctx.upload_species(sid, p, ids)
        for _ in range(steps):
            ctx.step()
        if pbc == PBC_ABSORB:
            lo, hi = ctx.absorbed_counts()
        gp, gids = ctx.download_species(sid)
    gp, gids = _by_tag(gp, gids)
    if pbc == PBC_ABSORB:
        keep = wraps == 0
        assert (lo, hi) == (int((wraps == -1).sum()), int((wraps == 1).sum()))
        assert (gids == want_ids[keep]).all()
        assert (gp.view(np.uint32) == want_p[:, keep].view(np.uint32)).all()
        return
    n = (g.nx, g.ny, g.nz)[axis]
    pitch = (1, g.nx + 2, (g.nx + 2) * (g.ny + 2))[axis]
    c = (want_ids // pitch) % (n + 2)
    exp_ids = np.where(wraps != 0, want_ids + (n + 1 - 2 * c) * pitch, want_ids).astype(np.int32)
    exp_p = want_p.copy()
    m = wraps != 0
    exp_p[axis, m] = -want_p[axis, m]
    exp_p[3 + axis, m] = -want_p[3 + axis, m]
    assert (gids == exp_ids).all()
    assert (gp.view(np.uint32) == exp_p.view(np.uint32)).all()


def test_closed_box_conserves_charge_and_particles():
    """Reflecting conductor walls on all six faces around a thermal e/i
    plasma: no particle is lost and div E - rho stays fixed at every node off
    the wall planes."""
    import paper_2102_13133_b200 as pic
    g = pic.make_grid((10, 8, 7), 1.0, dt=0.25)
    with pic.Context(g) as ctx:
        for face in range(6):
            ctx.set_boundary(face, PBC_REFLECT, FBC_PEC)
        e = ctx.add_species("e", -1.0 / 16, 1.0 / 16, 16 * g.interior)
        i = ctx.add_species("i", 1.0 / 16, 25.0 / 16, 16 * g.interior)
        ctx.load_synthetic(e, 16, 0.3, seed=3)
        ctx.load_synthetic(i, 16, 0.05, seed=4)

        def residual():
            ctx.refresh_charge_diagnostics()
            r = ctx.download_fields()[F["div_e_err"]].reshape(g.nz + 2, g.ny + 2, g.nx + 2)
            return r[2:g.nz + 1, 2:g.ny + 1, 2:g.nx + 1].astype(np.float64)  # off the wall planes

        r0 = residual()
        for _ in range(60):
            ctx.step()
        r1 = residual()
        n = ctx.species_count(e) + ctx.species_count(i)
    assert n == 32 * g.interior
    assert np.abs(r1 - r0).max() <= 1e-4 * np.abs(r0).max(), np.abs(r1 - r0).max() / np.abs(r0).max()


@pytest.mark.parametrize("fbc", [FBC_PEC, FBC_MUR])
def test_pulse_along_y(fbc):
    """An E_z / B_x pulse travelling +y: PEC y walls reflect it with its
    energy, Mur y walls let it out."""
    import paper_2102_13133_b200 as pic
    g = pic.make_grid((2, 160, 2), 1.0, dt=0.5)
    f = np.zeros((16, g.padded), np.float32)
    ez = f[F["ez"]].reshape(g.nz + 2, g.ny + 2, g.nx + 2)
    bx = f[F["cbx"]].reshape(g.nz + 2, g.ny + 2, g.nx + 2)
    ye = (np.arange(g.ny + 2) - 1) * g.hy          # E_z on y node planes
    yb = (np.arange(g.ny + 2) - 0.5) * g.hy        # B_x at y cell centres
    ez[:] = (1e-2 * np.exp(-((ye - 100.0) / 6.0) ** 2))[None, :, None]
    bx[:] = (1e-2 * np.exp(-((yb - 100.0) / 6.0) ** 2))[None, :, None]  # +y: E x B = E_z z x B_x x = +y
    ez[:, 0, :] = 0
    bx[:, 0, :] = 0
    with pic.Context(g) as ctx:
        ctx.set_boundary(2, PBC_ABSORB, fbc)
        ctx.set_boundary(3, PBC_ABSORB, fbc)
        ctx.upload_fields(f)
        e0 = sum(ctx.field_energy())
        for _ in range(200):
            ctx.step()
        e1 = sum(ctx.field_energy())
        ezf = ctx.download_fields()[F["ez"]].reshape(g.nz + 2, g.ny + 2, g.nx + 2)[1, 1:-1, 1]
    if fbc == FBC_PEC:
        assert abs(e1 - e0) <= 0.02 * e0, (e0, e1)
        k = int(np.argmax(np.abs(ezf)))
        assert 105 <= k <= 135 and ezf[k] < 0, (k, ezf[k])
    else:
        assert e1 <= 0.02 * e0, (e0, e1)
