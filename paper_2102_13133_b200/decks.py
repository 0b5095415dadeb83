"""Physics decks built through the API (BASELINE configs[2]: double Harris
sheet).  The reference's deck text only expresses uniform drifting
Maxwellians (proj/src/deck.cpp:149-395, proj/src/sim.cpp:74-134), so — as
SURVEY §8d (C3) notes — a Harris sheet is built by the caller: particles with
pic_species_load_harris (device loader, sech^2 weights, drift reversed on
the second sheet) and the magnetic field from a vector potential A_y on the
Yee grid (so div B = 0 to round-off), uploaded as a field array.  Periodic
in every direction, so the CPU restatement of the reference runs the same
state (tests/test_gpu_decks.py checks the GPU step against it bit for bit in
deterministic mode).

Units: c = 1, e = 1, m_e = 1, peak sheet density n0 = 1 (omega_pe = 1 at
w = 1).  A species of ppc particles per cell carries q = +-h^3/ppc and
m = m_s h^3/ppc per particle, so a weight-w particle stands for w n0.
Equilibrium: B0^2 / 2 = n0 (Te + Ti); drifts V_s = 2 T_s / (q_s B0 L).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

from . import F


@dataclasses.dataclass(frozen=True)
class Harris:
    """Double Harris sheet in an (nx, ny, nz) periodic box, sheets normal to z."""

    n: tuple = (64, 2, 64)
    h: float = 1.0          # cell size in d_e
    dt: float = 0.25        # omega_pe dt
    ppc: int = 16           # particles per cell per species
    mi_me: float = 25.0
    ti_te: float = 5.0
    b0: float = 0.5         # omega_ce / omega_pe
    half_width: float = 2.5  # L, in d_e
    background: float = 0.2  # n_b / n0
    psi0: float = 0.1       # X-point perturbation, fraction of B0 L

    @property
    def lz(self) -> float:
        return self.n[2] * self.h

    @property
    def lx(self) -> float:
        return self.n[0] * self.h

    @property
    def z1(self) -> float:
        return 0.25 * self.lz

    @property
    def z2(self) -> float:
        return 0.75 * self.lz

    @property
    def te(self) -> float:
        return 0.5 * self.b0 ** 2 / (1.0 + self.ti_te)

    @property
    def ti(self) -> float:
        return self.te * self.ti_te

    def species(self):
        """(name, q, m, u_th, drift, sheet kwargs) in load order: sheet e/i,
        background e/i."""
        v = self.h ** 3 / self.ppc
        uth_e, uth_i = math.sqrt(self.te), math.sqrt(self.ti / self.mi_me)
        vd_i = 2.0 * self.ti / (self.b0 * self.half_width)   # +y on sheet 1
        vd_e = -2.0 * self.te / (self.b0 * self.half_width)  # electrons opposite
        sheet = dict(z1=self.z1, z2=self.z2, half_width=self.half_width, background=0.0, amplitude=1.0,
                     flip_drift=True)
        bg = dict(z1=self.z1, z2=self.z2, half_width=self.half_width, background=self.background,
                  amplitude=0.0, flip_drift=False)
        return [("sheet_e", -v, v, uth_e, (0.0, vd_e, 0.0), sheet),
                ("sheet_i", v, self.mi_me * v, uth_i, (0.0, vd_i, 0.0), sheet),
                ("bg_e", -v, v, uth_e, (0.0, 0.0, 0.0), bg),
                ("bg_i", v, self.mi_me * v, uth_i, (0.0, 0.0, 0.0), bg)]

    def vector_potential(self, x, z):
        """A_y(x, z): B_x = -dA_y/dz = B0 (tanh1 - tanh2 - 1) plus the
        X-point perturbation psi0 B0 L cos(2 pi x / Lx) cos(2 pi (z - z1) / Lz)."""
        L, b0 = self.half_width, self.b0
        a = -b0 * (L * np.log(np.cosh((z - self.z1) / L)) - L * np.log(np.cosh((z - self.z2) / L)) - z)
        return a + self.psi0 * b0 * L * np.cos(2 * np.pi * x / self.lx) * np.cos(2 * np.pi * (z - self.z1) / self.lz)

    def fields(self, g, x0: int = 0) -> np.ndarray:
        """Field array (16 lanes x padded voxels): cbx, cbz from the discrete
        curl of A_y on y-edges (x_i, z_k) = ((ix-1) hx, (iz-1) hz) of voxel
        (ix, iy, iz) — B_x on x-faces, B_z on z-faces — so the discrete
        div B vanishes; periodic ghosts filled; E = 0.  x0: the grid is the
        x-slab starting at global cell x0 of this deck's box (decomposed
        runs); its x ghosts then hold the neighbouring slabs' values."""
        nx, ny, nz = g.nx, g.ny, g.nz
        NX = self.n[0]
        ix = np.arange(nx + 2)
        iz = np.arange(nz + 2)
        gx = (x0 + ix - 1) % NX  # global node index (periodic)
        X, Z = np.meshgrid(gx * g.hx, (iz - 1) * g.hz, indexing="ij")  # (nx+2, nz+2) edge nodes
        A = self.vector_potential(X.astype(np.float64), Z.astype(np.float64))
        # one more node column in x for the last B_z differences
        Xe, Ze = np.meshgrid(np.array([((x0 + nx + 1) % NX) * g.hx]), (iz - 1) * g.hz, indexing="ij")
        Ae = self.vector_potential(Xe.astype(np.float64), Ze.astype(np.float64))
        bx = np.zeros_like(A)
        bz = np.zeros_like(A)
        bx[:, :-1] = -(A[:, 1:] - A[:, :-1]) / g.hz
        A1 = np.concatenate([A[1:, :], Ae], axis=0)
        bz[:, :] = (A1 - A) / g.hx
        # z ghosts periodic: interior 1..n, ghost 0 = n, ghost n+1 = 1 (the
        # x ghosts are already the periodic / neighbour values)
        for b in (bx, bz):
            b[:, 0], b[:, nz + 1] = b[:, nz], b[:, 1]
        f = np.zeros((16, (nx + 2) * (ny + 2) * (nz + 2)), np.float32)
        # voxel index ix + (nx+2) (iy + (ny+2) iz): broadcast over iy
        shape = (nz + 2, ny + 2, nx + 2)
        f[F["cbx"]] = np.broadcast_to(bx.T[:, None, :], shape).reshape(-1).astype(np.float32)
        f[F["cbz"]] = np.broadcast_to(bz.T[:, None, :], shape).reshape(-1).astype(np.float32)
        return f

    def grid(self):
        from . import make_grid
        return make_grid(self.n, self.h, dt=self.dt)

    def load(self, ctx, seed: int = 11):
        """Creates and loads the four species on a context of this deck's grid,
        uploads the fields; returns the species ids."""
        g = ctx.grid
        sids = []
        for name, q, m, uth, drift, sheet in self.species():
            sid = ctx.add_species(name, q, m, self.ppc * g.interior)
            ctx.load_harris(sid, self.ppc, uth, drift, seed, **sheet)
            sids.append(sid)
        ctx.upload_fields(self.fields(g))
        return sids


@dataclasses.dataclass(frozen=True)
class LPI:
    """Laser-plasma interaction deck (BASELINE configs[3]): a laser launched
    from a soft source near the low x wall into a plasma slab, absorbing
    (Mur) field walls and absorbing particle walls on both x faces, periodic
    in y and z.  Units: c = 1, omega_pe = 1 at unit weight (per-particle
    q = -h^3/ppc, m = h^3/ppc), so n / n_cr = 1 / omega0^2.  Not expressible
    in the reference, which is periodic only."""

    n: tuple = (400, 2, 2)
    h: float = 0.2
    dt: float = 0.1
    ppc: int = 8
    omega0: float = 3.1622776601683795  # n / n_cr = 0.1
    e0: float = 1e-3                     # laser field amplitude (a0 = e0 / omega0)
    laser_ix: int = 20
    ramp_steps: float = 40.0
    slab: tuple = (150, 250)             # cells [ix_lo, ix_hi] holding plasma
    mi_me: float = 100.0
    u_th: float = 0.01

    def grid(self):
        from . import make_grid
        return make_grid(self.n, self.h, dt=self.dt)

    def species(self):
        v = self.h ** 3 / self.ppc
        return [("electron", -v, v, self.u_th), ("ion", v, self.mi_me * v, self.u_th / math.sqrt(self.mi_me))]

    def load(self, ctx, seed: int = 5):
        from . import FBC_MUR, PBC_ABSORB
        g = ctx.grid
        nslab = (self.slab[1] - self.slab[0] + 1) * g.ny * g.nz
        sids = []
        for name, q, m, uth in self.species():
            sid = ctx.add_species(name, q, m, self.ppc * nslab + 65536)
            ctx.load_slab(sid, self.ppc, uth, (0.0, 0.0, 0.0), seed, ix_lo=self.slab[0], ix_hi=self.slab[1])
            sids.append(sid)
        for side in (0, 1):
            ctx.set_x_boundary(side, PBC_ABSORB, FBC_MUR)
        ctx.set_laser(self.laser_ix, self.e0, self.omega0, pol=1, ramp_steps=self.ramp_steps)
        return sids
