"""Slab domain decomposition of the PIC step across GPUs.

The reference (minipic) runs one periodic box in one process.  Here a
global periodic box of NX x NY x NZ cells is cut into ``world`` equal slabs
along x, one per rank (one process per GPU, ``torch.distributed`` over NCCL;
or several slabs inside one process for testing).  Each slab is an ordinary
context whose x faces are *open* (``pic_set_x_open``): the three places where
the single-domain step wraps x become neighbour exchanges —

* particle migration after advance_p      (replaces particles.cpp:348-350)
* accumulator halo-add before unload       (replaces grid.cpp:78-86)
* E/B halo copy after each field update    (replaces fields.cpp:35-44)

plus one more plane copy the gather-form unload needs (the low neighbour's
folded accumulator plane in the x ghost).  Each exchange is a single
neighbour send/recv per face; packing and unpacking are sm_100a kernels in
``csrc/domain.cu``, the transport is ``torch.distributed.batch_isend_irecv``
on the stream the library runs on, so copies order with the kernels.

Per-step order (the reference's SimState::step, proj/src/sim.cpp:143-183):
  clear; interpolators; advance_p (all species, deck order); migrate;
  accumulator x halo-add; y/z fold; unload ghost copy; B(1/2); sync;
  unload + E; sync; B(1/2); sync          (sync = y/z ghost sync + x halo)

The engine protocol (``CudaSlab`` below) is what the sequencing talks to, so
the same ``DecomposedSim`` drives the CUDA library in production and a
numpy engine in the CPU (gloo) tests.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from . import (HALO_ACCUMULATOR, HALO_FIELDS, HALO_RHO, PIC_DETERMINISTIC, PIC_EXACT_GYRATION, STAGE_AFTER_B,
               STAGE_AFTER_E, STAGE_BEFORE_E, STAGE_EMIT, STAGE_FOLD, F, Context, UsageError, make_grid)

DOWN, UP = 0, 1  # message travels to the low (DOWN) or high (UP) neighbour


@dataclasses.dataclass(frozen=True)
class SlabGeometry:
    """Equal slabs of a global box along x: periodic, or with walls = (particle
    bc, field bc) on the two global x faces (pic_set_x_boundary; the outer
    slabs own them, no exchange crosses them)."""

    NX: int
    NY: int
    NZ: int
    world: int
    h: tuple = (1.0, 1.0, 1.0)
    dt: float | None = None
    walls: tuple | None = None

    def crosses_wall(self, rank: int, d: int) -> bool:
        """A message from `rank` in direction d would cross a global wall."""
        return self.walls is not None and ((rank == 0 and d == DOWN) or (rank == self.world - 1 and d == UP))

    def __post_init__(self):
        if self.world < 1 or self.NX % self.world:
            raise UsageError(f"slab decomposition: NX={self.NX} not divisible by world={self.world}")
        if self.NX // self.world < 3:
            raise UsageError("slab decomposition: each slab needs >= 3 cells in x")

    @property
    def nx(self) -> int:
        return self.NX // self.world

    def global_grid(self):
        return make_grid((self.NX, self.NY, self.NZ), self.h, dt=self.dt)

    def local_grid(self):
        g = self.global_grid()  # dt from the global box (identical cells)
        return make_grid((self.nx, self.NY, self.NZ), self.h, dt=g.dt)

    def x0(self, rank: int) -> int:
        return rank * self.nx

    def low(self, rank: int) -> int:
        return (rank - 1) % self.world

    def high(self, rank: int) -> int:
        return (rank + 1) % self.world

    # --- host-side helpers (uploads / parity checks) ------------------------
    def split(self, p7: np.ndarray, ids: np.ndarray):
        """Global-box particles (field-major lanes + global voxel ids) ->
        per-rank lists (p7, local ids), keeping the input order per rank."""
        pnx, pny = self.NX + 2, self.NY + 2
        ix = ids % pnx
        rest = ids // pnx
        iy, iz = rest % pny, rest // pny
        out = []
        lpnx = self.nx + 2
        for r in range(self.world):
            m = (ix > self.x0(r)) & (ix <= self.x0(r) + self.nx)
            lix = ix[m] - self.x0(r)
            lid = (lix + lpnx * (iy[m] + pny * iz[m])).astype(np.int32)
            out.append((np.ascontiguousarray(p7[:, m]), lid))
        return out

    def to_global_ids(self, rank: int, lid: np.ndarray) -> np.ndarray:
        lpnx, pny, pnx = self.nx + 2, self.NY + 2, self.NX + 2
        ix = lid % lpnx
        rest = lid // lpnx
        iy, iz = rest % pny, rest // pny
        return (ix + self.x0(rank) + pnx * (iy + pny * iz)).astype(np.int32)

    def split_fields(self, f16: np.ndarray):
        """Global (16, V) fields -> per-rank (16, V_local) incl. ghosts."""
        G = f16.reshape(16, self.NZ + 2, self.NY + 2, self.NX + 2)
        return [np.ascontiguousarray(G[:, :, :, self.x0(r):self.x0(r) + self.nx + 2]).reshape(16, -1)
                for r in range(self.world)]

    def join_fields(self, parts):
        """Per-rank fields -> global interior-consistent (16, V) array."""
        out = np.zeros((16, self.NZ + 2, self.NY + 2, self.NX + 2), np.float32)
        for r, f in enumerate(parts):
            L = f.reshape(16, self.NZ + 2, self.NY + 2, self.nx + 2)
            out[:, :, :, self.x0(r) + 1:self.x0(r) + self.nx + 1] = L[:, :, :, 1:self.nx + 1]
        return out.reshape(16, -1)


# ---------------------------------------------------------------------------
# transports
class LocalTransport:
    """All slabs in this process (tests, one-GPU runs): copies."""

    def exchange(self, msgs):
        """msgs: list of (src_rank, dst_rank, direction, send_buf, recv_buf)
        with both ends local."""
        for _, _, _, snd, rcv in msgs:
            if snd is not None and rcv is not None and rcv.numel():
                rcv.copy_(snd)

    def allreduce(self, values, op="sum"):
        return values


class DistTransport:
    """One slab per process, torch.distributed point-to-point (NCCL on GPU
    buffers, gloo on CPU buffers)."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group = rank, world, group

    def exchange(self, msgs):
        import torch.distributed as dist
        ops = []
        local = []
        # the messages between one pair of ranks are matched in issue order:
        # both sides issue them sorted by (peer, direction)
        sends = sorted(((d, k, s) for (src, d, k, s, _) in msgs if src == self.rank), key=lambda x: (x[0], x[1]))
        recvs = sorted(((s_, k, r) for (s_, dst, k, _, r) in msgs if dst == self.rank), key=lambda x: (x[0], x[1]))
        for dst, k, buf in sends:
            if dst == self.rank:
                local.append((k, buf))
            elif buf.numel():
                ops.append(dist.P2POp(dist.isend, buf, dst, self.group))
        for src, k, buf in recvs:
            if src == self.rank:
                for kk, sb in local:
                    if kk == k and buf.numel():
                        buf.copy_(sb)
            elif buf.numel():
                ops.append(dist.P2POp(dist.irecv, buf, src, self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def allreduce(self, values, op="sum"):
        import torch
        import torch.distributed as dist
        t = torch.tensor(values, dtype=torch.float64)
        if dist.get_backend(self.group) == "nccl":
            t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX, group=self.group)
        return t.cpu().tolist()


class HostStagedTransport:
    """DistTransport over a CPU backend (gloo) for device buffers: every
    message is staged through host memory (tests of the CUDA engine across
    processes where NCCL cannot run, e.g. several ranks on one GPU)."""

    def __init__(self, rank: int, world: int, group=None):
        self.inner = DistTransport(rank, world, group)

    def exchange(self, msgs):
        staged, back = [], []
        for src, dst, k, snd, rcv in msgs:
            hs = snd.cpu() if snd is not None else None
            hr = None
            if rcv is not None:
                hr = rcv.new_empty(rcv.shape, device="cpu")
                back.append((hr, rcv))
            staged.append((src, dst, k, hs, hr))
        self.inner.exchange(staged)
        for hr, rcv in back:
            if rcv.numel():
                rcv.copy_(hr)

    def allreduce(self, values, op="sum"):
        return self.inner.allreduce(values, op)


# ---------------------------------------------------------------------------
_SLAB_STREAMS = {}


def slab_stream(device: int = 0):
    """The one CUDA stream the decomposed step runs on per device: the
    library's kernels (pic_set_stream), torch's buffer copies and NCCL's
    send/recv (ordered after work on the current stream) all see it, and it
    is made torch's current stream."""
    import torch
    s = _SLAB_STREAMS.get(device)
    if s is None:
        s = torch.cuda.Stream(torch.device("cuda", device))
        _SLAB_STREAMS[device] = s
    torch.cuda.set_stream(s)
    return s


class CudaSlab:
    """Engine adapter: one x-open sm_100a context (the product path)."""

    def __init__(self, grid, rank: int, low_wraps: bool, device: int = 0, walls=None, world: int = 1):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", device)
        self.ctx = Context(grid, device)
        self.ctx.set_x_open(True, low_wraps and walls is None)
        if walls is not None:  # the outer slabs own the global walls
            if rank == 0:
                self.ctx.set_x_boundary(0, *walls)
            if rank == world - 1:
                self.ctx.set_x_boundary(1, *walls)
        self.stream = slab_stream(device)
        self.ctx.set_stream(self.stream.cuda_stream)
        self.grid = grid
        self.rank = rank
        self.species = []

    def buffer(self, nbytes: int):
        return self.torch.empty(max(int(nbytes), 0), dtype=self.torch.uint8, device=self.device)

    def count_buffer(self, values):
        return self.torch.tensor(values, dtype=self.torch.int64, device=self.device)

    def add_species(self, name, q, m, capacity):
        sid = self.ctx.add_species(name, q, m, capacity)
        self.species.append(sid)
        return sid

    # step pieces
    def prologue(self):
        self.ctx.clear_accumulator()
        self.ctx.clear_currents()
        self.ctx.load_interpolators()

    def advance_p(self, sid, flags):
        self.ctx.advance_p(sid, exact_gyration=bool(flags & PIC_EXACT_GYRATION),
                           deterministic=bool(flags & PIC_DETERMINISTIC))

    def fold_yz(self):
        self.ctx.ghost_fold_currents()  # x-open: the y and z passes only

    def advance_b(self, frac):
        self.ctx.advance_b(frac)

    def sync_yz(self):
        self.ctx.ghost_sync_fields()  # x-open: the y and z faces only

    def unload_advance_e(self):
        self.ctx.unload_advance_e()

    def halo_bytes(self, kind):
        return self.ctx.halo_plane_bytes(kind)

    def halo_pack(self, kind, ix, buf, zero_after=False):
        self.ctx.halo_pack(kind, ix, buf.data_ptr(), zero_after)

    def halo_unpack(self, kind, ix, buf, accumulate=False):
        self.ctx.halo_unpack(kind, ix, buf.data_ptr(), accumulate)

    def migrate_counts(self, sid):
        return self.ctx.migrate_counts(sid)

    def migrate_pack(self, sid, low, high):
        self.ctx.migrate_pack(sid, low.data_ptr(), high.data_ptr())

    def migrate_append(self, sid, buf, count):
        self.ctx.migrate_append(sid, buf.data_ptr(), count)

    def read_counts(self, t):
        return [int(x) for x in t.tolist()]

    def wall_stage(self, stage, frac=0.0):
        self.ctx.wall_stage(stage, frac)

    # diagnostics pieces
    def clear_rho(self):
        self.ctx.clear_rho()

    def deposit_rho(self, sid):
        self.ctx.deposit_rho(sid)

    def compute_div_errors(self):
        self.ctx.compute_div_errors()

    def local_diag(self):
        e, b = self.ctx.field_energy()
        self.ctx.load_interpolators()
        kin = [self.ctx.kinetic_energy(s, centered=True) for s in self.species]
        return dict(e=e, b=b, kinetic=kin, max_div_e=self.ctx.max_abs_lane(F["div_e_err"]),
                    max_div_b=self.ctx.max_abs_lane(F["div_b_err"]),
                    count=sum(self.ctx.species_count(s) for s in self.species))

    def synchronize(self):
        self.ctx.synchronize()


class DecomposedSim:
    """Sequences the decomposed step over the local slabs of this process.

    slabs: {rank: engine} for the ranks this process owns (all of them with a
    LocalTransport, one with a DistTransport)."""

    def __init__(self, geom: SlabGeometry, slabs: dict, transport):
        self.geom = geom
        self.slabs = dict(sorted(slabs.items()))
        self.transport = transport
        self.nspecies = 0
        self._bufs = {}
        self.on_mark = None  # optional callable(phase, begin) for timing
        self.absorbed = [0, 0]  # particles this process's slabs lost through the low / high wall

    def add_species(self, name, q, m, capacity_per_slab):
        sids = {r: e.add_species(name, q, m, capacity_per_slab) for r, e in self.slabs.items()}
        assert len(set(sids.values())) == 1
        self.nspecies += 1
        return next(iter(sids.values()))

    def _buf(self, rank, key, nbytes):
        k = (rank, key)
        b = self._bufs.get(k)
        if b is None or b.numel() < nbytes:
            b = self.slabs[rank].buffer(max(nbytes, 16))
            self._bufs[k] = b
        return b[:nbytes]

    def _plane_exchange(self, kind, send_ix, recv_ix, zero_after, accumulate, tag):
        """Every slab sends plane send_ix[d] in direction d (DOWN = to the low
        neighbour, UP = to the high one) and unpacks what arrives from the
        opposite side into plane recv_ix[d]."""
        g = self.geom
        msgs = []
        for r, e in self.slabs.items():
            nb = e.halo_bytes(kind)
            for d in (DOWN, UP):
                if send_ix[d] is None or g.crosses_wall(r, d):
                    continue
                sb = self._buf(r, (tag, "s", d), nb)
                e.halo_pack(kind, send_ix[d], sb, zero_after)
                dst = g.low(r) if d == DOWN else g.high(r)
                msgs.append((r, dst, d, sb, None))
        # receivers
        full = []
        for r, e in self.slabs.items():
            nb = e.halo_bytes(kind)
            for d in (DOWN, UP):
                src = g.high(r) if d == DOWN else g.low(r)  # a DOWN message comes from the high side
                if send_ix[d] is None or g.crosses_wall(src, d):
                    continue
                rb = self._buf(r, (tag, "r", d), nb)
                full.append((src, r, d, rb))
        self._run(msgs, full)
        for r, e in self.slabs.items():
            for d in (DOWN, UP):
                src = g.high(r) if d == DOWN else g.low(r)
                if send_ix[d] is None or g.crosses_wall(src, d):
                    continue
                e.halo_unpack(kind, recv_ix[d], self._buf(r, (tag, "r", d), e.halo_bytes(kind)), accumulate)

    def _run(self, sends, recvs):
        """Pairs sends (src, dst, d, buf, None) with recvs (src, dst, d, buf)
        and hands the transport one message list."""
        by_key = {(s, t, d): b for s, t, d, b, _ in sends}
        msgs = []
        for s, t, d, rb in recvs:
            msgs.append((s, t, d, by_key.get((s, t, d)), rb))
        for s, t, d, sb, _ in sends:
            if not any(m[0] == s and m[1] == t and m[2] == d for m in msgs):
                msgs.append((s, t, d, sb, None))
        self.transport.exchange(msgs)

    # --- the three exchanges ----------------------------------------------------
    def migrate(self, sids=None):
        """Particle migration after the pushes, every species in one round:
        one count exchange (one host read-back) and one payload exchange
        for all species, then the appends in species order."""
        g = self.geom
        sids = list(range(self.nspecies)) if sids is None else list(sids)
        if not sids:
            return
        counts = {r: [e.migrate_counts(sid) for sid in sids] for r, e in self.slabs.items()}
        # 1) counts: one message per direction holding every species' count
        sends, recvs = [], []
        for r, e in self.slabs.items():
            for d in (DOWN, UP):
                dst = g.low(r) if d == DOWN else g.high(r)
                if g.crosses_wall(r, d):  # particles leaving through an absorbing wall
                    self.absorbed[d] += sum(c[d] for c in counts[r])
                else:
                    sends.append((r, dst, d, e.count_buffer([c[d] for c in counts[r]]), None))
                src = g.high(r) if d == DOWN else g.low(r)
                if not g.crosses_wall(src, d):
                    recvs.append((src, r, d, e.count_buffer([0] * len(sids))))
        self._run(sends, recvs)
        incoming = {(r, d, k): 0 for r in self.slabs for d in (DOWN, UP) for k in range(len(sids))}
        for src, r, d, buf in recvs:
            for k, c in enumerate(self.slabs[r].read_counts(buf)):
                incoming[(r, d, k)] = c
        # 2) payloads (32 B records), packed while the stores compact
        sends, recvs = [], []
        for k, sid in enumerate(sids):
            for r, e in self.slabs.items():
                lo = self._buf(r, ("mig", sid, "s", DOWN), 32 * counts[r][k][DOWN])
                hi = self._buf(r, ("mig", sid, "s", UP), 32 * counts[r][k][UP])
                e.migrate_pack(sid, lo, hi)  # a wall side's buffer is packed and dropped
                if not g.crosses_wall(r, DOWN):
                    sends.append((r, g.low(r), (DOWN, k), lo, None))
                if not g.crosses_wall(r, UP):
                    sends.append((r, g.high(r), (UP, k), hi, None))
                for d in (DOWN, UP):
                    src = g.high(r) if d == DOWN else g.low(r)
                    if not g.crosses_wall(src, d):
                        recvs.append((src, r, (d, k), self._buf(r, ("mig", sid, "r", d), 32 * incoming[(r, d, k)])))
        self._run(sends, recvs)
        # 3) append: from the low neighbour (UP messages) first, then the high
        for k, sid in enumerate(sids):
            for r, e in self.slabs.items():
                for d in (UP, DOWN):
                    n = incoming[(r, d, k)]
                    if n:
                        e.migrate_append(sid, self._buf(r, ("mig", sid, "r", d), 32 * n), n)

    def fold_accumulator(self):
        """x halo-add: ghost plane 0 -> low neighbour's plane nx, ghost nx+1 ->
        high neighbour's plane 1 (ghosts zeroed), then the local y/z fold,
        then the folded plane nx -> high neighbour's ghost 0 for the unload."""
        nx = self.geom.nx
        self._plane_exchange(HALO_ACCUMULATOR, (0, nx + 1), (nx, 1), True, True, "accfold")
        for e in self.slabs.values():
            self._wall(e, STAGE_FOLD)
            e.fold_yz()
        self._plane_exchange(HALO_ACCUMULATOR, (None, nx), (None, 0), False, False, "accghost")

    def sync_fields(self):
        nx = self.geom.nx
        for e in self.slabs.values():
            e.sync_yz()
        self._plane_exchange(HALO_FIELDS, (1, nx), (nx + 1, 0), False, False, "fields")

    # --- SimState::step ---------------------------------------------------------
    def _wall(self, e, stage, frac=0.0):
        if self.geom.walls is not None:
            e.wall_stage(stage, frac)

    def step(self, deterministic=False, exact_gyration=False):
        flags = (PIC_DETERMINISTIC if deterministic else 0) | (PIC_EXACT_GYRATION if exact_gyration else 0)
        mark = self.on_mark or (lambda phase, begin: None)
        for e in self.slabs.values():
            e.prologue()
            mark("push", True)
            for sid in range(self.nspecies):
                e.advance_p(sid, flags)
            mark("push", False)
        # the field half of the step needs only the accumulator, the
        # migration only the particle stores: the fields go first so the
        # migration's count read-back (a host sync) comes after all of the
        # step's device work has been queued
        self.fold_accumulator()
        for e in self.slabs.values():
            e.advance_b(0.5)
            self._wall(e, STAGE_AFTER_B, 0.5)
        self.sync_fields()
        for e in self.slabs.values():
            self._wall(e, STAGE_BEFORE_E)
            e.unload_advance_e()
            self._wall(e, STAGE_AFTER_E)
        self.sync_fields()
        for e in self.slabs.values():
            e.advance_b(0.5)
            self._wall(e, STAGE_AFTER_B, 0.5)
        self.sync_fields()
        self.migrate()
        for e in self.slabs.values():
            self._wall(e, STAGE_EMIT)

    def set_laser(self, ix_global: int, e0: float, omega: float, **kw):
        """The laser plane (global node index) on the slab that owns it."""
        r, ix = divmod(ix_global - 1, self.geom.nx)
        if r in self.slabs:
            self.slabs[r].ctx.set_laser(ix + 1, e0, omega, **kw)

    # --- diagnostics (SimState::refresh_charge_diagnostics + current_diagnostics)
    def diagnostics(self):
        nx = self.geom.nx
        for e in self.slabs.values():
            e.clear_rho()
            for sid in range(self.nspecies):
                e.deposit_rho(sid)
        self._plane_exchange(HALO_RHO, (None, nx + 1), (None, 1), True, True, "rho")
        for e in self.slabs.values():
            e.compute_div_errors()
        loc = [e.local_diag() for e in self.slabs.values()]
        sums = [sum(d["e"] for d in loc), sum(d["b"] for d in loc), sum(d["count"] for d in loc)] + \
            [sum(d["kinetic"][k] for d in loc) for k in range(self.nspecies)]
        mx = [max(d["max_div_e"] for d in loc), max(d["max_div_b"] for d in loc)]
        sums = self.transport.allreduce(sums, "sum")
        mx = self.transport.allreduce(mx, "max")
        kin = sums[3:]
        return {"e_energy": sums[0], "b_energy": sums[1], "kinetic": kin,
                "total_energy": sums[0] + sums[1] + sum(kin), "max_div_e_err": mx[0], "max_div_b_err": mx[1],
                "particle_count": int(round(sums[2]))}

    def synchronize(self):
        for e in self.slabs.values():
            e.synchronize()
