"""The decomposed fast step in C++ over NCCL (pic_dd, csrc/dd.cu): at world 1
every exchange is an NCCL send / receive to self through the same code path
as at world N.  Checked against the oracle's single-domain run of the global
box (the first step's particles bit-exact as a set, then fp32 tolerance:
the x-face fold order differs), against the host-sequenced Python
decomposition, for the count kept on the device across migrations, and for
graph replay."""
import numpy as np
import pytest

from tests.test_domain import SPECIES, STEPS, _by_tag, _compare, _global_state, _og, _oracle_run
from paper_2102_13133_b200.domain import SlabGeometry

pytestmark = pytest.mark.gpu


def _slab(geom, state, graphs=True):
    import paper_2102_13133_b200 as pic
    ctx = pic.Context(geom.local_grid())
    ctx.set_x_open(True, True)  # rank 0 of world 1: its low face is the global periodic boundary
    for si, (q, m, p, ids) in enumerate(state):
        sid = ctx.add_species(f"s{si}", q, m, ids.size + 4096)
        ctx.upload_species(sid, *geom.split(p, ids)[0])
    dd = pic.DecomposedStep(ctx, 0, 1, pic.dd_unique_id())
    return ctx, dd


def test_dd_world1_matches_global_oracle():
    from oracle.bindings import Orc
    orc = Orc()
    geom = SlabGeometry(16, 6, 5, world=1, dt=0.25)
    og = _og(geom.global_grid())
    state = _global_state(orc, og, seed=9)
    f = np.zeros((16, geom.global_grid().padded), np.float32)
    want = _oracle_run(orc, og, [(q, m, p.copy(), i.copy()) for q, m, p, i in state], f, STEPS)
    ctx, dd = _slab(geom, state)
    try:
        for k in range(STEPS):
            dd.step()
            parts = {0: [ctx.download_species(si) for si in range(len(SPECIES))]}
            _compare(geom, parts, [ctx.download_fields()], want[k][0], want[k][1], exact=(k == 0))
    finally:
        dd.close()
        ctx.close()


@pytest.mark.parametrize("prepared", [False, True])
def test_dd_many_steps_conserve_particles_and_match_python_path(prepared):
    """Twenty graphed steps with heavy x migration, reordering pushes every
    fifth step and after a sort: every particle kept (the device count and
    the voxel counts through the migration), and the state tracks the
    host-sequenced decomposition (domain.py) within fp32 tolerance."""
    from oracle.bindings import Orc
    from paper_2102_13133_b200.domain import CudaSlab, DecomposedSim, LocalTransport
    orc = Orc()
    geom = SlabGeometry(8, 6, 5, world=1, dt=0.25)
    state = _global_state(orc, _og(geom.global_grid()), seed=13)
    ctx, dd = _slab(geom, state)
    slab = CudaSlab(geom.local_grid(), 0, True)
    sim = DecomposedSim(geom, {0: slab}, LocalTransport())
    for si, (q, m, p, ids) in enumerate(state):
        sid = sim.add_species(f"s{si}", q, m, ids.size + 4096)
        slab.ctx.upload_species(sid, *geom.split(p, ids)[0])
    try:
        for k in range(1, 21):
            if prepared and k == 2:  # graphs of steps 2..20 captured ahead (sorts after 8 and 16)
                assert dd.prepare_graphs(19, 8, 1) > 0
            dd.step()
            sim.step()
            if k % 8 == 0:  # a blocked sort: a reordering push next (physical voxel order)
                for s in range(len(SPECIES)):
                    ctx.sort_particles(s)
                    slab.ctx.sort_particles(s)
        total = sum(ids.size for _, _, _, ids in state)
        assert sum(ctx.species_count(s) for s in range(len(SPECIES))) == total
        for si in range(len(SPECIES)):
            # the same particles (matched by their unique weight tags: the
            # fast path refills holes in any order), momenta within the fp32
            # drift of 20 fast steps
            a, ai = _by_tag(*ctx.download_species(si))
            b, bi = _by_tag(*slab.ctx.download_species(si))
            assert a.shape == b.shape and (a[6] == b[6]).all()
            assert (ai == bi).mean() > 0.99
            assert np.abs(a[3:6] - b[3:6]).max() <= 1e-3 * max(1.0, np.abs(b[3:6]).max())
        fa, fb = ctx.download_fields(), slab.ctx.download_fields()
        for lane in (0, 1, 2, 4, 5, 6):
            assert np.abs(fa[lane] - fb[lane]).max() <= 1e-3 * max(np.abs(fb[lane]).max(), 1e-12), lane
    finally:
        dd.close()
        ctx.close()
        slab.ctx.close()


def test_dd_migration_capacity_overflow_is_run_abort():
    import paper_2102_13133_b200 as pic
    from oracle.bindings import Orc
    geom = SlabGeometry(8, 4, 4, world=1, dt=0.25)
    g = geom.local_grid()
    ctx = pic.Context(g)
    ctx.set_x_open(True, True)
    n = 200000
    rng = np.random.default_rng(2)
    p = np.zeros((7, n), np.float32)
    p[0] = 0.99  # every particle at the high face of ...
    p[3] = 5.0   # ... moving fast in +x: all cross
    p[6] = 1.0
    ids = np.full(n, g.voxel(8, 2, 2), np.int32)
    sid = ctx.add_species("e", -1e-20, 1.0, n)
    ctx.upload_species(sid, p, ids)
    dd = pic.DecomposedStep(ctx, 0, 1, pic.dd_unique_id(), mig_frac=1e-6)  # 4096-record buffers
    try:
        with pytest.raises(pic.RunAbort):
            dd.step()
            ctx.synchronize()
    finally:
        dd.close()
        ctx.close()
    del rng, Orc


@pytest.mark.parametrize("m", [1, 2, 5])
def test_dd_reorder_intervals_keep_every_particle(m):
    """Reordering pushes at every m-th step with migration in between: the
    chunk reservations stay exact (no hole, no overwrite: the particle set
    is intact, matched by unique weight tags)."""
    import paper_2102_13133_b200 as pic
    from oracle.bindings import Orc
    orc = Orc()
    geom = SlabGeometry(6, 5, 4, world=1, dt=0.25)
    state = _global_state(orc, _og(geom.global_grid()), seed=21)
    ctx, dd = _slab(geom, state)
    ctx._set_reorder_interval(m)
    dd.close()
    dd = pic.DecomposedStep(ctx, 0, 1, pic.dd_unique_id())
    try:
        for _ in range(12):
            dd.step()
        for si, (q, mm, p, ids) in enumerate(state):
            gp, gi = _by_tag(*ctx.download_species(si))
            wp, _ = _by_tag(p, ids)
            assert gp.shape == wp.shape
            assert (gp[6] == wp[6]).all()  # every tag once
            assert ((gi % (geom.nx + 2)) >= 1).all() and ((gi % (geom.nx + 2)) <= geom.nx).all()
    finally:
        dd.close()
        ctx.close()
