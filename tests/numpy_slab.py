"""A numpy/oracle engine for paper_2102_13133_b200.domain.DecomposedSim — test
infrastructure only.

It mirrors the x-open semantics of the CUDA slab (csrc/domain.cu and the
x-open branches of push.cu / fields.cpp restatements) on the CPU so the
decomposed step's host sequencing (exchanges, migration bookkeeping,
transport matching) can be exercised with world_size > 1 over gloo in the
CPU suite, and compared against the oracle's single-domain run of the
global box.  Local physics comes from the oracle (oracle/pic_oracle.c):

* advance_p: the oracle push (periodic in x), then particles that wrapped
  through an x face get their ghost voxel id back and are listed as
  emigrants (with >= 3 cells per slab a wrap is unambiguous);
* fold: the oracle fold — the x ghost planes were already sent and zeroed;
* ghost sync: the oracle sync — its x part is overwritten by the exchange;
* unload: the oracle scatter with the x-high edges of the last plane fed
  from the x ghost plane 0 (the low neighbour's folded plane), which is what
  the gather form does with an open x face.
"""
from __future__ import annotations

import numpy as np
import torch

from oracle.bindings import Grid as OGrid
from oracle.bindings import Orc


class NumpySlab:
    def __init__(self, grid, rank: int, low_wraps: bool, walls=None, world: int = 1):
        self.g = OGrid(grid.nx, grid.ny, grid.nz, grid.hx, grid.hy, grid.hz, grid.dt)
        self.grid = grid
        self.rank = rank
        self.orc = Orc()
        self.V = grid.padded
        self.f = np.zeros((16, self.V), np.float32)
        self.acc = np.zeros((self.V, 12), np.float32)
        self.interp = np.zeros((18, self.V), np.float32)
        self.sp = []  # [q, m, p7, ids, mig_low, mig_high]
        self.pnx, self.pny, self.pnz = grid.nx + 2, grid.ny + 2, grid.nz + 2
        # global x walls (absorbing particles, PEC fields only) on the outer slabs
        if walls is not None:
            assert tuple(walls) == (1, 1), "numpy engine: absorbing particle walls with PEC fields only"
        self.wall = [walls is not None and rank == 0, walls is not None and rank == world - 1]

    # --- geometry helpers ---------------------------------------------------------
    def _ix(self, ids):
        return ids % self.pnx

    def _plane(self, ix):
        iy, iz = np.meshgrid(np.arange(self.pny), np.arange(self.pnz), indexing="xy")
        return (ix + self.pnx * (iy + self.pny * iz)).ravel()  # iy fastest

    # --- buffers --------------------------------------------------------------------
    def buffer(self, nbytes):
        return torch.empty(max(int(nbytes), 0), dtype=torch.uint8)

    def count_buffer(self, values):
        return torch.tensor(values, dtype=torch.int64)

    def read_counts(self, t):
        return [int(x) for x in t.tolist()]

    def add_species(self, name, q, m, capacity):
        self.sp.append([q, m, np.zeros((7, 0), np.float32), np.zeros(0, np.int32), [], []])
        return len(self.sp) - 1

    def upload(self, sid, p7, ids):
        self.sp[sid][2] = np.ascontiguousarray(p7, np.float32).copy()
        self.sp[sid][3] = np.ascontiguousarray(ids, np.int32).copy()

    # --- step pieces ----------------------------------------------------------------
    def prologue(self):
        self.acc[:] = 0
        self.orc.clear_currents(self.g, self.f)
        self.interp[:] = self.orc.load_interpolators(self.g, self.f)

    def advance_p(self, sid, flags):
        q, m, p7, ids = self.sp[sid][:4]
        old = self._ix(ids).copy()
        self.orc.advance_particles(self.g, q, m, p7, ids, self.interp, self.acc, bool(flags & 1))
        new = self._ix(ids)
        nx = self.grid.nx
        low = np.nonzero((old == 1) & (new == nx))[0]
        high = np.nonzero((old == nx) & (new == 1))[0]
        ids[low] -= nx  # ix = nx -> 0
        ids[high] += nx  # ix = 1 -> nx + 1
        self.sp[sid][4] = list(low)
        self.sp[sid][5] = list(high)

    def fold_yz(self):
        self.orc.ghost_fold(self.g, self.acc)

    def advance_b(self, frac):
        self.orc.advance_b(self.g, self.f, frac)

    def sync_yz(self):
        # the oracle sync is fully periodic; an open x face keeps its x ghost
        # planes (neighbour halo or wall), whose own y / z ghosts are then
        # synced like the CUDA kernel's y / z faces over the padded x range
        keep = {ix: self.f[:, self._plane(ix)].copy() for ix in (0, self.grid.nx + 1)}
        self.orc.ghost_sync(self.g, self.f)
        ny, nz = self.grid.ny, self.grid.nz
        for ix, vals in keep.items():
            self.f[:, self._plane(ix)] = vals
            f = self.f.reshape(16, self.pnz, self.pny, self.pnx)
            f[:, :, 0, ix] = f[:, :, ny, ix]
            f[:, :, ny + 1, ix] = f[:, :, 1, ix]
            f[:, 0, :, ix] = f[:, nz, :, ix]
            f[:, nz + 1, :, ix] = f[:, 1, :, ix]

    def wall_stage(self, stage, frac=0.0):
        """pic_wall_stage for absorbing particle / PEC field walls: FOLD drops
        the accumulator's ghost plane beyond a wall, AFTER_E zeroes the
        tangential E on the wall plane (and E_x outside)."""
        nx = self.grid.nx
        for side in (0, 1):
            if not self.wall[side]:
                continue
            ghost = 0 if side == 0 else nx + 1
            if stage == 0:  # STAGE_FOLD
                self.acc[self._plane(ghost)] = 0
            elif stage == 3:  # STAGE_AFTER_E
                wall_plane = self._plane(1 if side == 0 else nx + 1)
                self.f[1, wall_plane] = 0
                self.f[2, wall_plane] = 0
                self.f[0, self._plane(ghost)] = 0

    def unload_advance_e(self):
        a = self.acc.copy()
        hi, gh = self._plane(self.grid.nx), self._plane(0)
        for lane in (6, 7, 9, 11):
            a[hi, lane] = self.acc[gh, lane]
        self.orc.unload(self.g, a, self.f)
        self.orc.advance_e(self.g, self.f)

    # --- halos ----------------------------------------------------------------------
    def halo_bytes(self, kind):
        return self.pny * self.pnz * (12, 6, 1)[kind] * 4

    def _view(self, kind, ix):
        pl = self._plane(ix)
        if kind == 0:
            return pl, None
        lanes = [0, 1, 2, 4, 5, 6] if kind == 1 else [11]
        return pl, lanes

    def halo_pack(self, kind, ix, buf, zero_after=False):
        pl, lanes = self._view(kind, ix)
        out = buf.numpy().view(np.float32)
        if kind == 0:
            out[:] = self.acc[pl].ravel()
            if zero_after:
                self.acc[pl] = 0
        else:
            out[:] = self.f[np.ix_(lanes, pl)].ravel()
            if zero_after:
                self.f[np.ix_(lanes, pl)] = 0

    def halo_unpack(self, kind, ix, buf, accumulate=False):
        pl, lanes = self._view(kind, ix)
        src = buf.numpy().view(np.float32)
        if kind == 0:
            s = src.reshape(-1, 12)
            self.acc[pl] = self.acc[pl] + s if accumulate else s
        else:
            s = src.reshape(len(lanes), -1)
            cur = self.f[np.ix_(lanes, pl)]
            self.f[np.ix_(lanes, pl)] = cur + s if accumulate else s

    # --- migration --------------------------------------------------------------------
    def migrate_counts(self, sid):
        return len(self.sp[sid][4]), len(self.sp[sid][5])

    def _records(self, p7, ids, idx, translate_ix):
        n = len(idx)
        rec = np.zeros((n, 8), np.float32)
        if n == 0:
            return rec
        i = np.asarray(idx)
        lid = ids[i] - self._ix(ids[i]) + translate_ix
        rec[:, 0:3] = p7[0:3, i].T
        rec[:, 3] = lid.astype(np.int32).view(np.float32)
        rec[:, 4:8] = p7[3:7, i].T
        return rec

    def migrate_pack(self, sid, low, high):
        q, m, p7, ids, ml, mh = self.sp[sid]
        nx = self.grid.nx
        low.numpy().view(np.float32)[:] = self._records(p7, ids, sorted(ml), nx).ravel()
        high.numpy().view(np.float32)[:] = self._records(p7, ids, sorted(mh), 1).ravel()
        # compaction: holes below n' filled from the tail in index order
        allm = sorted(ml + mh)
        n = ids.size
        nn = n - len(allm)
        holes = [i for i in allm if i < nn]
        em = set(allm)
        fillers = [i for i in range(nn, n) if i not in em]
        assert len(holes) == len(fillers)
        for h, fl in zip(holes, fillers):
            p7[:, h] = p7[:, fl]
            ids[h] = ids[fl]
        self.sp[sid][2] = np.ascontiguousarray(p7[:, :nn])
        self.sp[sid][3] = np.ascontiguousarray(ids[:nn])
        self.sp[sid][4] = []
        self.sp[sid][5] = []

    def migrate_append(self, sid, buf, count):
        rec = buf.numpy().view(np.float32).reshape(count, 8)
        p7 = np.zeros((7, count), np.float32)
        p7[0:3] = rec[:, 0:3].T
        p7[3:7] = rec[:, 4:8].T
        ids = rec[:, 3].copy().view(np.int32)
        self.sp[sid][2] = np.concatenate([self.sp[sid][2], p7], axis=1)
        self.sp[sid][3] = np.concatenate([self.sp[sid][3], ids])

    # --- diagnostics (energies only; rho halo exercised through the planes) ------------
    def clear_rho(self):
        self.f[11] = 0

    def deposit_rho(self, sid):
        q, m, p7, ids = self.sp[sid][:4]
        # deposit with the x-high wrap replaced by the ghost plane: shift the
        # last plane's particles' +x weights into ghost nx+1 (the oracle
        # wraps them to plane 1): deposit into a widened copy
        nx = self.grid.nx
        tmp = np.zeros_like(self.f)
        self.orc.deposit_rho(self.g, q, p7, ids, tmp)
        # weights the oracle wrapped onto plane 1 from plane-nx particles
        hi = self._ix(ids) == nx
        wrapped = np.zeros_like(self.f)
        if hi.any():
            self.orc.deposit_rho(self.g, q, np.ascontiguousarray(p7[:, hi]), np.ascontiguousarray(ids[hi]), wrapped)
        one, gh = self._plane(1), self._plane(nx + 1)
        moved = wrapped[11, one].copy()
        tmp[11, one] -= moved
        tmp[11, gh] += moved
        self.f[11] += tmp[11]

    def compute_div_errors(self):
        self.orc.compute_div_errors(self.g, self.f)

    def local_diag(self):
        e, b = self.orc.field_energy(self.g, self.f)
        i18 = self.orc.load_interpolators(self.g, self.f)
        kin = [self.orc.kinetic_energy_centered(self.g, q, m, p7, ids, i18) for q, m, p7, ids, _, _ in self.sp]
        return dict(e=float(e), b=float(b), kinetic=kin,
                    max_div_e=self.orc.max_abs_lane(self.g, self.f, 3), max_div_b=self.orc.max_abs_lane(self.g, self.f, 7),
                    count=sum(s[3].size for s in self.sp))

    def synchronize(self):
        pass
