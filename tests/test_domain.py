"""Slab domain decomposition against the single-domain oracle run
of the global periodic box.

Bar (SURVEY §8e "Oracle"): the first step's particle state is bit-exact as a
set (fields identical before it, only deposit summation order differs);
after that particles and fields agree within fp32 tolerance (the current
fold order at slab faces is not the reference's).  Particles are matched by
a unique weight tag (w is never modified by the step).

CPU tests drive the host sequencing with the numpy/oracle slab engine
(tests/numpy_slab.py): in-process (LocalTransport) and over gloo with
world_size 2.  GPU tests drive the sm_100a slabs through the same
DecomposedSim in one process.
"""
import os
import tempfile

import numpy as np
import pytest

from paper_2102_13133_b200.domain import DecomposedSim, DistTransport, LocalTransport, SlabGeometry

SPECIES = [(-1.0 / 8, 1.0 / 8, 5, 0.25, (0.08, 0.0, 0.0)), (1.0 / 8, 100.0 / 8, 3, 0.02, (0.0, 0.0, 0.0))]
DIMS = (12, 5, 4)
STEPS = 4


def _global_state(orc, og, seed=4):
    state = []
    tag = 0
    for si, (q, m, ppc, uth, drift) in enumerate(SPECIES):
        p, ids = orc.load_species(og, seed, si, ppc, uth, drift)
        n = ids.size
        # unique weight tags 1 + k 2^-23 (the step never changes w)
        p[6] = (1.0 + (np.arange(n) + tag) * 2.0 ** -23).astype(np.float32)
        tag += n
        state.append((q, m, p, ids))
    return state


def _oracle_run(orc, og, state, f, steps):
    hist = []
    for _ in range(steps):
        orc.step(og, state, f)
        hist.append(([(p.copy(), ids.copy()) for _, _, p, ids in state], f.copy()))
    return hist


def _by_tag(p, ids):
    o = np.argsort(p[6].view(np.uint32), kind="stable")
    return p[:, o], ids[o]


def _compare(geom, parts_per_rank, fields_per_rank, want_parts, want_f, exact):
    for si in range(len(SPECIES)):
        gp = np.concatenate([parts_per_rank[r][si][0] for r in range(geom.world)], axis=1)
        gi = np.concatenate([geom.to_global_ids(r, parts_per_rank[r][si][1]) for r in range(geom.world)])
        gp, gi = _by_tag(gp, gi)
        wp, wi = _by_tag(*want_parts[si])
        assert gp.shape == wp.shape
        assert (gp[6].view(np.uint32) == wp[6].view(np.uint32)).all()
        if exact:
            assert (gi == wi).all(), "voxel ids"
            assert (gp.view(np.uint32) == wp.view(np.uint32)).all(), "particle lanes"
        else:
            assert (gi == wi).mean() > 0.999
            assert np.abs(gp[3:6] - wp[3:6]).max() <= 1e-4 * max(1.0, np.abs(wp[3:6]).max())
    gf = geom.join_fields(fields_per_rank)
    for lane in (0, 1, 2, 4, 5, 6, 8, 9, 10):
        a = gf[lane].reshape(geom.NZ + 2, geom.NY + 2, geom.NX + 2)[1:-1, 1:-1, 1:-1]
        b = want_f[lane].reshape(geom.NZ + 2, geom.NY + 2, geom.NX + 2)[1:-1, 1:-1, 1:-1]
        scale = max(np.abs(b).max(), 1e-12)
        assert np.abs(a - b).max() <= 1e-4 * scale, f"field lane {lane}"


def test_geometry_split_join():
    from oracle.bindings import Orc
    geom = SlabGeometry(*DIMS, world=3, dt=0.25)
    g = geom.global_grid()
    rng = np.random.default_rng(0)
    n = 500
    ix = rng.integers(1, g.nx + 1, n)
    iy = rng.integers(1, g.ny + 1, n)
    iz = rng.integers(1, g.nz + 1, n)
    ids = (ix + (g.nx + 2) * (iy + (g.ny + 2) * iz)).astype(np.int32)
    p = rng.standard_normal((7, n)).astype(np.float32)
    parts = geom.split(p, ids)
    assert sum(q.shape[1] for q, _ in parts) == n
    back = np.concatenate([geom.to_global_ids(r, parts[r][1]) for r in range(3)])
    assert sorted(back.tolist()) == sorted(ids.tolist())
    for r, (_, lid) in enumerate(parts):
        lix = lid % (geom.nx + 2)
        assert lix.min() >= 1 and lix.max() <= geom.nx
    f = rng.standard_normal((16, g.padded)).astype(np.float32)
    Orc().ghost_sync(_og(g), f)
    fs = geom.split_fields(f)
    j = geom.join_fields(fs)
    G = f.reshape(16, g.nz + 2, g.ny + 2, g.nx + 2)
    J = j.reshape(16, g.nz + 2, g.ny + 2, g.nx + 2)
    assert (G[:, :, :, 1:-1] == J[:, :, :, 1:-1]).all()
    with pytest.raises(Exception):
        SlabGeometry(10, 4, 4, world=3)


def _og(g):
    from oracle.bindings import Grid
    return Grid(g.nx, g.ny, g.nz, g.hx, g.hy, g.hz, g.dt)


def _run_numpy(geom, ranks, transport, state, steps):
    from tests.numpy_slab import NumpySlab
    slabs = {r: NumpySlab(geom.local_grid(), r, r == 0) for r in ranks}
    sim = DecomposedSim(geom, slabs, transport)
    for si, (q, m, p, ids) in enumerate(state):
        sid = sim.add_species(f"s{si}", q, m, 1 << 20)
        parts = geom.split(p, ids)
        for r in ranks:
            slabs[r].upload(sid, *parts[r])
    out = []
    for _ in range(steps):
        sim.step()
        out.append(({r: [(s[2].copy(), s[3].copy()) for s in slabs[r].sp] for r in ranks},
                    {r: slabs[r].f.copy() for r in ranks}))
    return sim, out


@pytest.mark.parametrize("world", [1, 3])
def test_numpy_slabs_local_transport(world):
    from oracle.bindings import Orc
    orc = Orc()
    geom = SlabGeometry(*DIMS, world=world, dt=0.25)
    og = _og(geom.global_grid())
    state = _global_state(orc, og)
    f = np.zeros((16, geom.global_grid().padded), np.float32)
    want = _oracle_run(orc, og, [(q, m, p.copy(), i.copy()) for q, m, p, i in state], f, STEPS)
    _, got = _run_numpy(geom, list(range(world)), LocalTransport(), state, STEPS)
    for k in range(STEPS):
        parts, fields = got[k]
        _compare(geom, parts, [fields[r] for r in range(world)], want[k][0], want[k][1], exact=(k == 0))


def _gloo_worker(rank, world, port, tmp):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.bindings import Orc
        orc = Orc()
        geom = SlabGeometry(*DIMS, world=world, dt=0.25)
        state = _global_state(orc, _og(geom.global_grid()))
        sim, got = _run_numpy(geom, [rank], DistTransport(rank, world), state, STEPS)
        d = sim.diagnostics()
        np.savez(os.path.join(tmp, f"r{rank}.npz"),
                 **{f"p{k}_{si}": got[k][0][rank][si][0] for k in range(STEPS) for si in range(len(SPECIES))},
                 **{f"i{k}_{si}": got[k][0][rank][si][1] for k in range(STEPS) for si in range(len(SPECIES))},
                 **{f"f{k}": got[k][1][rank] for k in range(STEPS)},
                 diag=np.array([d["e_energy"], d["b_energy"], d["particle_count"]] + list(d["kinetic"])))
    finally:
        dist.destroy_process_group()


def test_gloo_world2():
    """Two processes, one slab each, exchanges over torch.distributed (gloo)."""
    import socket

    import torch.multiprocessing as mp
    from oracle.bindings import Orc
    world = 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_gloo_worker, args=(world, port, tmp), nprocs=world, join=True)
        res = [np.load(os.path.join(tmp, f"r{r}.npz")) for r in range(world)]
        orc = Orc()
        geom = SlabGeometry(*DIMS, world=world, dt=0.25)
        og = _og(geom.global_grid())
        state = _global_state(orc, og)
        f = np.zeros((16, geom.global_grid().padded), np.float32)
        want = _oracle_run(orc, og, [(q, m, p.copy(), i.copy()) for q, m, p, i in state], f, STEPS)
        for k in range(STEPS):
            parts = {r: [(res[r][f"p{k}_{si}"], res[r][f"i{k}_{si}"]) for si in range(len(SPECIES))]
                     for r in range(world)}
            _compare(geom, parts, [res[r][f"f{k}"] for r in range(world)], want[k][0], want[k][1], exact=(k == 0))
        # diagnostics reduce across ranks: every rank holds the global sums
        d0, d1 = res[0]["diag"], res[1]["diag"]
        assert np.array_equal(d0, d1)
        wf = want[-1][1].copy()
        we, wb = orc.field_energy(og, wf)
        assert abs(d0[0] - we) <= 1e-4 * abs(we) + 1e-12
        assert abs(d0[1] - wb) <= 1e-4 * abs(wb) + 1e-12
        assert d0[2] == sum(p.shape[1] for p, _ in want[-1][0])


# --------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 4])
def test_cuda_slabs_match_global_oracle(world):
    """sm_100a slabs on one GPU (in-process transport) vs the oracle's
    single-domain run of the global box."""
    import paper_2102_13133_b200 as pic
    from oracle.bindings import Orc
    from paper_2102_13133_b200.domain import CudaSlab
    orc = Orc()
    geom = SlabGeometry(16, 6, 5, world=world, dt=0.25)
    og = _og(geom.global_grid())
    state = _global_state(orc, og, seed=9)
    f = np.zeros((16, geom.global_grid().padded), np.float32)
    want = _oracle_run(orc, og, [(q, m, p.copy(), i.copy()) for q, m, p, i in state], f, STEPS)
    slabs = {r: CudaSlab(geom.local_grid(), r, r == 0) for r in range(world)}
    sim = DecomposedSim(geom, slabs, LocalTransport())
    for si, (q, m, p, ids) in enumerate(state):
        sid = sim.add_species(f"s{si}", q, m, ids.size)
        parts = geom.split(p, ids)
        for r in range(world):
            slabs[r].ctx.upload_species(sid, *parts[r])
    for k in range(STEPS):
        sim.step()
        parts = {r: [slabs[r].ctx.download_species(si) for si in range(len(SPECIES))] for r in range(world)}
        fields = [slabs[r].ctx.download_fields() for r in range(world)]
        _compare(geom, parts, fields, want[k][0], want[k][1], exact=(k == 0))
    d = sim.diagnostics()
    assert d["particle_count"] == sum(ids.size for _, _, _, ids in state)
    for e in slabs.values():
        e.ctx.close()
    del pic


@pytest.mark.gpu
def test_cuda_slab_deterministic_mode_runs():
    from oracle.bindings import Orc
    from paper_2102_13133_b200.domain import CudaSlab
    orc = Orc()
    geom = SlabGeometry(9, 4, 4, world=3, dt=0.25)
    state = _global_state(orc, _og(geom.global_grid()), seed=5)
    slabs = {r: CudaSlab(geom.local_grid(), r, r == 0) for r in range(3)}
    sim = DecomposedSim(geom, slabs, LocalTransport())
    for si, (q, m, p, ids) in enumerate(state):
        sid = sim.add_species(f"s{si}", q, m, ids.size)
        for r, part in enumerate(geom.split(p, ids)):
            slabs[r].ctx.upload_species(sid, *part)
    for _ in range(3):
        sim.step(deterministic=True)
    sim.synchronize()
    n = sum(e.ctx.species_count(s) for e in slabs.values() for s in range(len(SPECIES)))
    assert n == sum(ids.size for _, _, _, ids in state)


# --------------------------------------------------------------- global x walls
def _run_numpy_walls(geom, ranks, transport, state, steps):
    from tests.numpy_slab import NumpySlab
    slabs = {r: NumpySlab(geom.local_grid(), r, r == 0, walls=geom.walls, world=geom.world) for r in ranks}
    sim = DecomposedSim(geom, slabs, transport)
    for si, (q, m, p, ids) in enumerate(state):
        sid = sim.add_species(f"s{si}", q, m, 1 << 20)
        parts = geom.split(p, ids)
        for r in ranks:
            slabs[r].upload(sid, *parts[r])
    for _ in range(steps):
        sim.step()
    parts = {r: [(s[2].copy(), s[3].copy()) for s in slabs[r].sp] for r in ranks}
    return sim, parts, {r: slabs[r].f.copy() for r in ranks}


def _gloo_walls_worker(rank, world, port, tmp):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.bindings import Orc
        geom = SlabGeometry(*DIMS, world=world, dt=0.25, walls=(1, 1))
        state = _global_state(Orc(), _og(geom.global_grid()))
        sim, parts, fields = _run_numpy_walls(geom, [rank], DistTransport(rank, world), state, STEPS)
        np.savez(os.path.join(tmp, f"r{rank}.npz"),
                 **{f"p{si}": parts[rank][si][0] for si in range(len(SPECIES))},
                 **{f"i{si}": parts[rank][si][1] for si in range(len(SPECIES))},
                 f=fields[rank], absorbed=np.array(sim.absorbed))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_global_walls():
    """Absorbing / conducting global x walls (pic_set_x_boundary on the outer
    slabs): two processes over gloo against one slab holding the whole box —
    nothing crosses a wall, the leavers are dropped on the owning rank, and
    fields and particles agree."""
    import socket

    import torch.multiprocessing as mp
    from oracle.bindings import Orc
    world = 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_gloo_walls_worker, args=(world, port, tmp), nprocs=world, join=True)
        res = [np.load(os.path.join(tmp, f"r{r}.npz")) for r in range(world)]
    geom2 = SlabGeometry(*DIMS, world=world, dt=0.25, walls=(1, 1))
    geom1 = SlabGeometry(*DIMS, world=1, dt=0.25, walls=(1, 1))
    state = _global_state(Orc(), _og(geom1.global_grid()))
    sim1, parts1, fields1 = _run_numpy_walls(geom1, [0], LocalTransport(), state, STEPS)
    absorbed2 = res[0]["absorbed"] + res[1]["absorbed"]
    assert list(absorbed2) == sim1.absorbed and sum(sim1.absorbed) > 0
    for si in range(len(SPECIES)):
        gp = np.concatenate([res[r][f"p{si}"] for r in range(world)], axis=1)
        gi = np.concatenate([geom2.to_global_ids(r, res[r][f"i{si}"]) for r in range(world)])
        gp, gi = _by_tag(gp, gi)
        wp, wi = _by_tag(parts1[0][si][0], geom1.to_global_ids(0, parts1[0][si][1]))
        assert gp.shape == wp.shape
        assert (gi == wi).mean() > 0.999
        assert np.abs(gp[3:6] - wp[3:6]).max() <= 1e-4 * max(1.0, np.abs(wp[3:6]).max())
    gf = geom2.join_fields([res[r]["f"] for r in range(world)])
    wf = geom1.join_fields([fields1[0]])
    for lane in (0, 1, 2, 4, 5, 6):
        a = gf[lane].reshape(DIMS[2] + 2, DIMS[1] + 2, DIMS[0] + 2)[1:-1, 1:-1, 1:-1]
        b = wf[lane].reshape(DIMS[2] + 2, DIMS[1] + 2, DIMS[0] + 2)[1:-1, 1:-1, 1:-1]
        assert np.abs(a - b).max() <= 1e-4 * max(np.abs(b).max(), 1e-12), lane


def _cuda_gloo_worker(rank, world, port, tmp):
    """One process per slab on the same GPU, the CUDA engine, exchanges over
    gloo through host memory."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.bindings import Orc
        from paper_2102_13133_b200.domain import CudaSlab, HostStagedTransport
        geom = SlabGeometry(16, 6, 5, world=world, dt=0.25)
        state = _global_state(Orc(), _og(geom.global_grid()), seed=9)
        slab = CudaSlab(geom.local_grid(), rank, rank == 0, device=0)
        sim = DecomposedSim(geom, {rank: slab}, HostStagedTransport(rank, world))
        for si, (q, m, p, ids) in enumerate(state):
            sid = sim.add_species(f"s{si}", q, m, ids.size)
            slab.ctx.upload_species(sid, *geom.split(p, ids)[rank])
        out = {}
        for k in range(STEPS):
            sim.step()
            for si in range(len(SPECIES)):
                out[f"p{k}_{si}"], out[f"i{k}_{si}"] = slab.ctx.download_species(si)
            out[f"f{k}"] = slab.ctx.download_fields()
        d = sim.diagnostics()
        out["diag"] = np.array([d["e_energy"], d["b_energy"], d["particle_count"]])
        np.savez(os.path.join(tmp, f"r{rank}.npz"), **out)
        slab.ctx.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_cuda_engine_world2_gloo_host_staged():
    """Two processes on one GPU, each with its sm_100a slab, the exchanges
    over torch.distributed (gloo, host-staged): the global oracle's run."""
    import socket

    import torch.multiprocessing as mp
    from oracle.bindings import Orc
    world = 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_cuda_gloo_worker, args=(world, port, tmp), nprocs=world, join=True)
        res = [np.load(os.path.join(tmp, f"r{r}.npz")) for r in range(world)]
        orc = Orc()
        geom = SlabGeometry(16, 6, 5, world=world, dt=0.25)
        og = _og(geom.global_grid())
        state = _global_state(orc, og, seed=9)
        f = np.zeros((16, geom.global_grid().padded), np.float32)
        want = _oracle_run(orc, og, [(q, m, p.copy(), i.copy()) for q, m, p, i in state], f, STEPS)
        for k in range(STEPS):
            parts = {r: [(res[r][f"p{k}_{si}"], res[r][f"i{k}_{si}"]) for si in range(len(SPECIES))]
                     for r in range(world)}
            _compare(geom, parts, [res[r][f"f{k}"] for r in range(world)], want[k][0], want[k][1], exact=(k == 0))
        assert np.array_equal(res[0]["diag"], res[1]["diag"])
        assert res[0]["diag"][2] == sum(ids.size for _, _, _, ids in state)
