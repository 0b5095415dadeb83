"""Harris deck construction (paper_2102_13133_b200/decks.py), CPU side: the
field array is the discrete curl of A_y (div B = 0 to round-off in the
reference's div_b stencil, fields.cpp:253-274), B_x follows the double-sheet
tanh profile, the ghosts are periodic images, and the species parameters
satisfy the Harris equilibrium relations."""
import math

import numpy as np

from paper_2102_13133_b200 import F, make_grid
from paper_2102_13133_b200.decks import Harris


def _lane(f, g, name):
    return f[F[name]].reshape(g.nz + 2, g.ny + 2, g.nx + 2)


def test_harris_fields_divergence_free_and_profile():
    d = Harris(n=(32, 2, 48), psi0=0.1)
    g = make_grid(d.n, d.h, dt=d.dt)
    f = d.fields(g)
    bx, by, bz = (_lane(f, g, n).astype(np.float64) for n in ("cbx", "cby", "cbz"))
    div = ((bx[1:-1, 1:-1, 2:] - bx[1:-1, 1:-1, 1:-1]) / g.hx + (by[1:-1, 2:, 1:-1] - by[1:-1, 1:-1, 1:-1]) / g.hy
           + (bz[2:, 1:-1, 1:-1] - bz[1:-1, 1:-1, 1:-1]) / g.hz)
    assert np.abs(div).max() < 1e-6 * d.b0
    # unperturbed profile: B_x(z) = B0 (tanh1 - tanh2 - 1) at the x-face centres z = (iz - 1/2) hz
    d0 = Harris(n=(32, 2, 48), psi0=0.0)
    b = _lane(d0.fields(g), g, "cbx")
    z = (np.arange(1, g.nz + 1) - 0.5) * g.hz
    L = d0.half_width
    want = d0.b0 * (np.tanh((z - d0.z1) / L) - np.tanh((z - d0.z2) / L) - 1.0)
    assert np.allclose(b[1:-1, 1, 3], want, atol=2e-2 * d0.b0)  # centred difference of A_y, h / L = 0.4
    assert np.abs(_lane(d0.fields(g), g, "cbz")).max() == 0.0
    # periodic ghosts
    for name in ("cbx", "cbz"):
        a = _lane(f, g, name)
        assert (a[0] == a[g.nz]).all() and (a[g.nz + 1] == a[1]).all()
        assert (a[:, :, 0] == a[:, :, g.nx]).all() and (a[:, :, g.nx + 1] == a[:, :, 1]).all()
    for name in ("ex", "ey", "ez"):
        assert not _lane(f, g, name).any()


def test_harris_equilibrium_relations():
    d = Harris()
    n0 = 1.0
    assert math.isclose(d.b0 ** 2 / 2, n0 * (d.te + d.ti), rel_tol=1e-12)
    sp = {s[0]: s for s in d.species()}
    # current of the sheet: J_y = n0 (V_i - V_e) = B0 / L (Ampere at the sheet centre)
    vi, ve = sp["sheet_i"][4][1], sp["sheet_e"][4][1]
    assert math.isclose(n0 * (vi - ve), d.b0 / d.half_width, rel_tol=1e-12)
    # omega_pe = 1 at unit weight: ppc (q^2 / m) / h^3 = 1 for the electrons
    q, m = sp["sheet_e"][1], sp["sheet_e"][2]
    assert math.isclose(d.ppc * q * q / m / d.h ** 3, 1.0, rel_tol=1e-12)
    assert math.isclose(sp["sheet_i"][2] / sp["sheet_i"][1], d.mi_me * m / -q, rel_tol=1e-12)


def test_harris_slab_fields_match_global():
    """Each x-slab's field array (decomposed runs) equals the global box's
    field array split into slabs, ghosts included."""
    from paper_2102_13133_b200.domain import SlabGeometry
    d = Harris(n=(24, 2, 16))
    geom = SlabGeometry(*d.n, world=3, h=(d.h,) * 3, dt=d.dt)
    whole = d.fields(geom.global_grid())
    parts = geom.split_fields(whole)
    for r in range(3):
        mine = d.fields(geom.local_grid(), x0=geom.x0(r))
        for name in ("cbx", "cbz"):
            assert (mine[F[name]] == parts[r][F[name]]).all(), (r, name)
