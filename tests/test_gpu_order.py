"""Continuous voxel order of the fast push (csrc/order.cu): the store is kept
one step from sorted physically while every caller observes the reference's
order — the push sequence with blocked / interleaved sorts and downloads in
between gives the oracle's particle state bit for bit (fixed interpolators,
so the particle update does not depend on the accumulator's summation
order), the accumulator stays within the fast-mode tolerance, and the
graphed step (captured buffer swaps re-applied on replay) matches the
oracle's SimState::step + sort cadence."""
import numpy as np
import pytest

from tests.helpers import assert_bitwise, assert_close, rand_fields, rand_particles

pytestmark = pytest.mark.gpu

ACC_RTOL = 1e-5


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


# (after push k: action) — "b" blocked sort, "i" interleaved sort, "d" download check
PLAN = {2: "b", 4: "d", 5: "b", 6: "bb", 8: "i", 9: "db", 11: "b"}


@pytest.mark.parametrize("m", [1, 3, 4])  # pushes per reordering of the store
@pytest.mark.parametrize("dims,n,u,sort_first", [
    ((12, 10, 9), 200000, 0.5, False),   # ~185 per voxel: chunks of several warps, many crossers
    ((16, 16, 16), 60000, 0.3, True),     # ~15 per voxel
    ((40, 6, 5), 240000, 0.8, True),      # heavy movers
    ((3, 2, 2), 31, 0.5, True),           # partial slice
])
def test_ordered_push_sequence_matches_oracle(pic, orc, dims, n, u, sort_first, m):
    g = pic.make_grid(dims, 1.0, cfl_frac=0.9)
    o = og(g)
    rng = np.random.default_rng(5)
    f = rand_fields(g, rng, scale=0.3, sync=lambda gg, ff: orc.ghost_sync(o, ff))
    interp = orc.load_interpolators(o, f)
    p, ids = rand_particles(g, rng, n, u_scale=u, sort=False)
    wp, wids = p.copy(), ids.copy()
    with pic.Context(g) as ctx:
        ctx._set_reorder_interval(m)
        sid = ctx.add_species("s", -1.0, 1.0, n)
        ctx.upload_species(sid, p, ids)
        ctx.upload_fields(f)
        ctx.load_interpolators()
        if sort_first:  # enter the order from a deferred sort permutation
            ctx.sort_particles(sid)
            orc.sort(wp, wids, interleaved=False)
        for k in range(1, 13):
            ctx.clear_accumulator()
            ctx.advance_p(sid)
            wacc = np.zeros((g.padded, 12), np.float32)
            orc.advance_particles(o, -1.0, 1.0, wp, wids, interp, wacc, False)
            if k in (1, 7, 12):
                assert ctx._species_ordered(sid)
                assert_close(ctx.download_accumulator(), wacc, ACC_RTOL, what=f"accumulator push {k}")
            for a in PLAN.get(k, ""):
                if a == "b":
                    ctx.sort_particles(sid, pic.SORT_BLOCKED)
                    orc.sort(wp, wids, interleaved=False)
                elif a == "i":
                    ctx.sort_particles(sid, pic.SORT_INTERLEAVED)
                    orc.sort(wp, wids, interleaved=True)
                else:
                    gp, gids = ctx.download_species(sid)
                    assert_bitwise(gids, wids, f"ids after push {k}")
                    assert_bitwise(gp, wp, f"lanes after push {k}")
        gp, gids = ctx.download_species(sid)
    assert_bitwise(gids, wids, "final ids")
    assert_bitwise(gp, wp, "final lanes")
    assert (wids != ids).mean() > 0.05 or n < 100


def test_order_off_switch_and_empty_species(pic, orc):
    g = pic.make_grid((6, 5, 4), 1.0, cfl_frac=0.9)
    o = og(g)
    rng = np.random.default_rng(9)
    f = rand_fields(g, rng, scale=0.3, sync=lambda gg, ff: orc.ghost_sync(o, ff))
    interp = orc.load_interpolators(o, f)
    p, ids = rand_particles(g, rng, 5000, u_scale=0.5)
    wp, wids = p.copy(), ids.copy()
    with pic.Context(g) as ctx:
        e = ctx.add_species("empty", 1.0, 1.0, 10)
        sid = ctx.add_species("s", -1.0, 1.0, 5000)
        ctx.upload_species(sid, p, ids)
        ctx.upload_fields(f)
        ctx.load_interpolators()
        for k in range(3):
            ctx.advance_p(e)
            ctx.advance_p(sid)
            orc.advance_particles(o, -1.0, 1.0, wp, wids, interp, np.zeros((g.padded, 12), np.float32), False)
        ctx.sort_particles(sid)
        orc.sort(wp, wids)
        assert ctx._species_ordered(sid)
        ctx._set_voxel_order(False)  # leaves the order (and applies the owed sort)
        assert not ctx._species_ordered(sid)
        ctx.advance_p(sid)
        orc.advance_particles(o, -1.0, 1.0, wp, wids, interp, np.zeros((g.padded, 12), np.float32), False)
        assert not ctx._species_ordered(sid)
        gp, gids = ctx.download_species(sid)
        assert ctx.species_count(e) == 0
    assert_bitwise(gids, wids, "ids")
    assert_bitwise(gp, wp, "lanes")


@pytest.mark.parametrize("m,prepared", [(1, False), (4, False), (4, True), (5, True)])
def test_graphed_ordered_steps_match_oracle(pic, orc, m, prepared):
    """pic_step captured as CUDA graphs while the ordered push swaps buffers
    every step (two alternating graphs, plus the relabelling step): a
    ballistic deck (q ~ 1e-20: currents far below the fields' ulp) keeps the
    fields identical, so particles and fields are bitwise over 25 steps with
    a blocked sort every 5."""
    g = pic.make_grid((10, 8, 6), 1.0, cfl_frac=0.9)
    o = og(g)
    rng = np.random.default_rng(3)
    f = rand_fields(g, rng, scale=0.3, sync=lambda gg, ff: orc.ghost_sync(o, ff))
    species = [(-1e-20, 1.0, 0.4), (1e-20, 4.0, 0.2)]
    state = []
    with pic.Context(g) as ctx:
        ctx._set_reorder_interval(m)
        sids = []
        for si, (q, m, us) in enumerate(species):
            p, ids = rand_particles(g, rng, 40000, u_scale=us)
            sid = ctx.add_species(f"s{si}", q, m, 40000)
            ctx.upload_species(sid, p, ids)
            sids.append(sid)
            state.append((q, m, p.copy(), ids.copy()))
        ctx.upload_fields(f)
        wf = f.copy()
        for k in range(1, 26):
            if prepared and k == 2:
                # the graphs of steps 2..25 (sort after every 5th) captured
                # ahead without running: every later step is a replay
                assert ctx.prepare_graphs(24, 5, 1) > 0
                g0 = ctx._graph_stats()
            ctx.step()
            orc.step(o, state, wf)
            if k == 13:  # a mid-cycle host download reads the logical order without regrouping
                for sid, (_, _, p, ids) in zip(sids, state):
                    assert ctx._species_ordered(sid)
                    gp, gids = ctx.download_species(sid)
                    assert ctx._species_ordered(sid)
                    assert_bitwise(gids, ids, f"ids s{sid} step {k}")
                    assert_bitwise(gp, p, f"lanes s{sid} step {k}")
            if k % 5 == 0:
                for sid in sids:
                    ctx.sort_particles(sid)
                for (_, _, p, ids) in state:
                    orc.sort(p, ids)
        assert all(ctx._species_ordered(s) for s in sids)
        if prepared:
            g1 = ctx._graph_stats()
            assert (g1[0] - g0[0], g1[1] - g0[1], g1[2] - g0[2]) == (0, 24, 0), (g0, g1)
        gf = ctx.download_fields()
        for sid, (_, _, p, ids) in zip(sids, state):
            gp, gids = ctx.download_species(sid)
            assert_bitwise(gids, ids, f"ids s{sid}")
            assert_bitwise(gp, p, f"lanes s{sid}")
    assert_bitwise(gf[[0, 1, 2, 4, 5, 6]], wf[[0, 1, 2, 4, 5, 6]], "E/B")


@pytest.mark.parametrize("nspecies", [3, 4, 5])
def test_batched_species_mixed_forms_match_oracle(pic, orc, nspecies):
    """Every species of a fast step in one advance_p_lean launch per push
    form (launch_advance_p_batch): species sorted at different steps sit at
    different points of their reorder cycles, so a step mixes in-place,
    counting and reordering pushes (one launch per form, several species per
    launch); five species exceed the batch (kMaxBatch 4) and take the
    per-species path.  Ballistic deck: particles and fields bitwise against
    the oracle after 23 steps (graph captures and replays included: a
    configuration seen twice is captured)."""
    g = pic.make_grid((9, 8, 7), 1.0, cfl_frac=0.9)
    o = og(g)
    rng = np.random.default_rng(11)
    f = rand_fields(g, rng, scale=0.3, sync=lambda gg, ff: orc.ghost_sync(o, ff))
    species = [(-1e-20, 1.0, 0.5), (1e-20, 4.0, 0.2), (-2e-20, 1.5, 0.4), (1e-20, 9.0, 0.1),
               (-1e-20, 2.0, 0.3)][:nspecies]
    sizes = [30000, 17000, 25000, 9000, 12000]
    state = []
    with pic.Context(g) as ctx:
        ctx._set_reorder_interval(4)
        sids = []
        for si, (q, m, us) in enumerate(species):
            p, ids = rand_particles(g, rng, sizes[si], u_scale=us)
            sid = ctx.add_species(f"s{si}", q, m, sizes[si])
            ctx.upload_species(sid, p, ids)
            sids.append(sid)
            state.append((q, m, p.copy(), ids.copy()))
        ctx.upload_fields(f)
        wf = f.copy()
        # species si sorted after step k when (k + si) % (3 + si) == 0
        for k in range(1, 24):
            ctx.step()
            orc.step(o, state, wf)
            for si, sid in enumerate(sids):
                if (k + si) % (3 + si) == 0:
                    ctx.sort_particles(sid)
                    orc.sort(state[si][2], state[si][3])
        batched = ctx._batched_launches()
        gf = ctx.download_fields()
        for sid, (_, _, p, ids) in zip(sids, state):
            gp, gids = ctx.download_species(sid)
            assert_bitwise(gids, ids, f"ids s{sid}")
            assert_bitwise(gp, p, f"lanes s{sid}")
    assert_bitwise(gf[[0, 1, 2, 4, 5, 6]], wf[[0, 1, 2, 4, 5, 6]], "E/B")
    assert (batched > 0) == (nspecies <= 4), batched


@pytest.mark.parametrize("relabel_variant", [0, 1])
def test_clustered_store_relabel(pic, orc, relabel_variant, monkeypatch):
    """Blocked sorts of a store with a few crowded voxels (a voxel block
    holding far more records than the relabel's shared-memory staging, so
    it ranks from global memory) and many empty ones: the download after
    each sort is the oracle's stable order."""
    monkeypatch.setenv("PIC_RELABEL_VARIANT", str(relabel_variant))
    g = pic.make_grid((8, 6, 5), 1.0, cfl_frac=0.9)
    o = og(g)
    rng = np.random.default_rng(11)
    f = rand_fields(g, rng, scale=0.3, sync=lambda gg, ff: orc.ghost_sync(o, ff))
    interp = orc.load_interpolators(o, f)
    n = 30000
    p, ids = rand_particles(g, rng, n, u_scale=0.4, sort=False)
    crowd = rng.choice(np.unique(ids), 3, replace=False)
    pick = rng.random(n) < 0.8
    ids[pick] = crowd[rng.integers(0, 3, int(pick.sum()))]
    wp, wids = p.copy(), ids.copy()
    with pic.Context(g) as ctx:
        ctx._set_reorder_interval(3)
        sid = ctx.add_species("s", -1.0, 1.0, n)
        ctx.upload_species(sid, p, ids)
        ctx.upload_fields(f)
        ctx.load_interpolators()
        for k in range(1, 8):
            ctx.advance_p(sid)
            orc.advance_particles(o, -1.0, 1.0, wp, wids, interp, np.zeros((g.padded, 12), np.float32), False)
            if k in (1, 4, 6):
                ctx.sort_particles(sid, pic.SORT_BLOCKED)
                orc.sort(wp, wids, interleaved=False)
            if k in (2, 5, 7):
                gp, gids = ctx.download_species(sid)
                assert_bitwise(gids, wids, f"ids after push {k}")
                assert_bitwise(gp, wp, f"lanes after push {k}")
