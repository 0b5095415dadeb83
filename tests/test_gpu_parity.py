"""GPU parity: the sm_100a kernels (called through the C-ABI) against the
plain-C oracle (oracle/pic_oracle.c, itself pinned bitwise to the reference by
tests/test_oracle_vs_ref.py).

Bar: bit-exact for everything whose reference order is deterministic
(interpolators, push state, ids, mover, fold, unload, field stencils, ghost
sync, sorts, and the accumulator in PIC_DETERMINISTIC mode); the fast-mode
accumulator (hardware float atomics, order not fixed) within
ACC_RTOL x max|acc|.
"""
import numpy as np
import pytest

from tests.helpers import assert_bitwise, assert_close, rand_fields, rand_particles, rel_err_percentiles

pytestmark = pytest.mark.gpu

ACC_RTOL = 1e-5  # fp32 tolerance for reordered current sums (north_star: 1e-5)


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


GRIDS = [((6, 5, 4), (1.0, 1.0, 1.0), 0.5), ((8, 8, 8), (0.7, 1.1, 0.9), 0.9), ((3, 2, 7), (1.0, 0.5, 2.0), 0.95)]


@pytest.mark.parametrize("dims,h,cfl", GRIDS)
def test_load_interpolators_bitwise(pic, orc, dims, h, cfl):
    g = pic.make_grid(dims, h, cfl_frac=cfl)
    rng = np.random.default_rng(1)
    f = rand_fields(g, rng, sync=lambda gg, ff: orc.ghost_sync(og(gg), ff))
    with pic.Context(g) as ctx:
        ctx.upload_fields(f)
        ctx.load_interpolators()
        got = ctx.download_interpolators()
    want = orc.load_interpolators(og(g), f)
    assert_bitwise(got, want, "interp18")


@pytest.mark.parametrize("dims,h,cfl", GRIDS)
def test_field_stencils_bitwise(pic, orc, dims, h, cfl):
    g = pic.make_grid(dims, h, cfl_frac=cfl)
    rng = np.random.default_rng(2)
    f = rand_fields(g, rng)
    f[8:11] = rng.standard_normal((3, g.padded)).astype(np.float32)
    o = og(g)
    with pic.Context(g) as ctx:
        ctx.upload_fields(f)
        ctx.ghost_sync_fields()
        want = f.copy()
        orc.ghost_sync(o, want)
        assert_bitwise(ctx.download_fields(), want, "ghost_sync")
        ctx.advance_b(0.5)
        orc.advance_b(o, want, 0.5)
        assert_bitwise(ctx.download_fields(), want, "advance_b")
        ctx.advance_e()
        orc.advance_e(o, want)
        assert_bitwise(ctx.download_fields(), want, "advance_e")
        ctx.advance_b(0.25)
        orc.advance_b(o, want, 0.25)
        assert_bitwise(ctx.download_fields(), want, "advance_b(0.25)")


@pytest.mark.parametrize("dims", [(5, 4, 3), (2, 2, 2), (7, 3, 5)])
def test_fold_and_unload_bitwise(pic, orc, dims):
    g = pic.make_grid(dims, (1.0, 0.8, 1.3), cfl_frac=0.6)
    rng = np.random.default_rng(3)
    acc = rng.standard_normal((g.padded, 12)).astype(np.float32)
    f = rand_fields(g, rng)
    f[8:11] = rng.standard_normal((3, g.padded)).astype(np.float32)  # unload adds onto existing jf
    o = og(g)
    with pic.Context(g) as ctx:
        ctx.upload_accumulator(acc)
        ctx.upload_fields(f)
        ctx.ghost_fold_currents()
        want_acc = acc.copy()
        orc.ghost_fold(o, want_acc)
        assert_bitwise(ctx.download_accumulator(), want_acc, "ghost_fold")
        ctx.unload_currents()
        want_f = f.copy()
        orc.unload(o, want_acc, want_f)
        assert_bitwise(ctx.download_fields(), want_f, "unload")
        # fused unload + advance_e == unload then advance_e
        ctx.upload_fields(f)
        ctx.unload_advance_e()
        want_f = f.copy()
        orc.unload(o, want_acc, want_f)
        orc.advance_e(o, want_f)
        assert_bitwise(ctx.download_fields(), want_f, "unload_advance_e")


def _push_case(pic, orc, g, n, seed, q, m, u_scale, deterministic, exact=False, variant=None):
    rng = np.random.default_rng(seed)
    o = og(g)
    f = rand_fields(g, rng, scale=0.3, sync=lambda gg, ff: orc.ghost_sync(o, ff))
    interp = orc.load_interpolators(o, f)
    p, ids = rand_particles(g, rng, n, u_scale=u_scale)
    with pic.Context(g) as ctx:
        sid = ctx.add_species("s", q, m, n)
        if variant is not None:
            ctx._set_push_variant(variant)
        ctx.upload_species(sid, p, ids)
        ctx.upload_fields(f)
        ctx.load_interpolators()
        ctx.clear_accumulator()
        ctx.advance_p(sid, exact_gyration=exact, deterministic=deterministic)
        ctx.synchronize()
        gp, gids = ctx.download_species(sid)
        gacc = ctx.download_accumulator()
    wp, wids = p.copy(), ids.copy()
    wacc = np.zeros((g.padded, 12), np.float32)
    orc.advance_particles(o, q, m, wp, wids, interp, wacc, exact)
    _push_case.ids0 = ids
    return (gp, gids, gacc), (wp, wids, wacc)


@pytest.mark.parametrize("deterministic", [False, True])
@pytest.mark.parametrize("dims,n,u", [((6, 5, 4), 5000, 0.6), ((16, 16, 16), 200000, 0.3), ((3, 2, 2), 777, 2.0)])
def test_advance_p_parity(pic, orc, dims, n, u, deterministic):
    g = pic.make_grid(dims, 1.0, cfl_frac=0.9)
    (gp, gids, gacc), (wp, wids, wacc) = _push_case(pic, orc, g, n, 7, -1.0, 1.0, u, deterministic)
    assert_bitwise(gids, wids, "ids")
    assert_bitwise(gp, wp, "particle lanes")
    if deterministic:
        assert_bitwise(gacc, wacc, "accumulator (deterministic)")
    else:
        assert_close(gacc, wacc, ACC_RTOL, what="accumulator (fast)")
    # the case exercises the face-crossing tail and the periodic wrap
    assert (wids != _push_case.ids0).mean() > 0.02


# the product library's advance_p strategies: 52 = advance_p_lean (default),
# 42 = advance_p_run (exact_gyration / out-of-range decks); the measured
# ablations live in libpic_b200_ablate.so (tests/test_gpu_ablations.py)
PUSH_VARIANTS = [42, 52]


@pytest.mark.parametrize("variant", PUSH_VARIANTS)
def test_advance_p_strategies(pic, orc, variant):
    """Every advance_p deposit/tail strategy gives the bitwise particle state
    and the accumulator within tolerance."""
    g = pic.make_grid((10, 9, 8), 1.0, cfl_frac=0.9)
    (gp, gids, gacc), (wp, wids, wacc) = _push_case(pic, orc, g, 60000, 13, -1.0, 1.0, 0.5, False,
                                                    variant=variant)
    assert_bitwise(gids, wids, "ids")
    assert_bitwise(gp, wp, "particle lanes")
    assert_close(gacc, wacc, ACC_RTOL, what="accumulator")


@pytest.mark.parametrize("variant", PUSH_VARIANTS)
@pytest.mark.parametrize("dims,n,u,sort", [((40, 6, 5), 240000, 0.4, True), ((7, 6, 5), 30000, 1.2, False),
                                           ((4, 3, 2), 31, 0.5, True)])
def test_advance_p_strategies_layouts(pic, orc, variant, dims, n, u, sort):
    """Sorted, unsorted (every particle a new voxel: slot evictions and a
    full crossing queue) and tiny (partial TMA slices) stores."""
    g = pic.make_grid(dims, 1.0, cfl_frac=0.9)
    rng = np.random.default_rng(21)
    o = og(g)
    f = rand_fields(g, rng, scale=0.3, sync=lambda gg, ff: orc.ghost_sync(o, ff))
    interp = orc.load_interpolators(o, f)
    p, ids = rand_particles(g, rng, n, u_scale=u, sort=sort)
    with pic.Context(g) as ctx:
        sid = ctx.add_species("s", -1.0, 1.0, n)
        ctx._set_push_variant(variant)
        ctx.upload_species(sid, p, ids)
        ctx.upload_fields(f)
        ctx.load_interpolators()
        ctx.clear_accumulator()
        ctx.advance_p(sid)
        ctx.synchronize()
        gp, gids = ctx.download_species(sid)
        gacc = ctx.download_accumulator()
    wacc = np.zeros((g.padded, 12), np.float32)
    orc.advance_particles(o, -1.0, 1.0, p, ids, interp, wacc, False)
    assert_bitwise(gids, ids, "ids")
    assert_bitwise(gp, p, "particle lanes")
    assert_close(gacc, wacc, ACC_RTOL, what="accumulator")


def test_product_library_rejects_ablations_and_probes(pic):
    """Timing probes (90-93, 99: not valid pushes) and ablations are not in
    the product library: selecting one raises instead of running it."""
    g = pic.make_grid((4, 4, 4))
    with pic.Context(g) as ctx:
        for v in (0, 7, 43, 55, 90, 93, 99, 1000):
            with pytest.raises(pic.UsageError):
                ctx._set_push_variant(v)
        for v in (1, 2, 3, 4):
            with pytest.raises(pic.UsageError):
                ctx._set_sort_variant(v)
        ctx._set_push_variant(42)
        ctx._set_push_variant(52)


def test_advance_p_unsorted_and_heavy_ions(pic, orc):
    g = pic.make_grid((9, 7, 5), (1.0, 0.9, 1.2), cfl_frac=0.8)
    rng = np.random.default_rng(11)
    o = og(g)
    f = rand_fields(g, rng, scale=2.0, sync=lambda gg, ff: orc.ghost_sync(o, ff))
    interp = orc.load_interpolators(o, f)
    n = 30000
    p, ids = rand_particles(g, rng, n, u_scale=1.0, sort=False)
    with pic.Context(g) as ctx:
        sid = ctx.add_species("i", 1.0, 100.0, n)
        ctx.upload_species(sid, p, ids)
        ctx.upload_fields(f)
        ctx.load_interpolators()
        ctx.clear_accumulator()
        ctx.advance_p(sid, deterministic=True)
        gp, gids = ctx.download_species(sid)
        gacc = ctx.download_accumulator()
    wacc = np.zeros((g.padded, 12), np.float32)
    orc.advance_particles(o, 1.0, 100.0, p, ids, interp, wacc, False)
    assert_bitwise(gids, ids, "ids")
    assert_bitwise(gp, p, "lanes")
    assert_bitwise(gacc, wacc, "acc")


def test_exact_gyration_tolerance(pic, orc):
    # std::tan vs CUDA tanf is not bit-reproducible: tolerance.
    g = pic.make_grid((6, 6, 6), 1.0, cfl_frac=0.5)
    (gp, gids, gacc), (wp, wids, wacc) = _push_case(pic, orc, g, 4000, 5, -1.0, 1.0, 0.3, True, exact=True)
    assert_close(gp[3:6], wp[3:6], 1e-5, what="momenta (exact gyration)")
    assert_close(gp[0:3], wp[0:3], 1e-5, atol_scale=1.0, what="offsets (exact gyration)")
    assert (gids == wids).mean() > 0.999


def test_cfl_violation_raises_run_abort(pic):
    """A validated grid bounds |d| < 2 for |v| < 1, so the device CFL guard
    (particles.cpp:190-194) is reached by a non-finite displacement; it must
    surface as run_abort at the next quiescence point."""
    g = pic.make_grid((4, 4, 4), 1.0, cfl_frac=0.5)
    p = np.zeros((7, 2), np.float32)
    p[6] = 1
    p[3, 1] = np.nan
    ids = np.array([g.voxel(2, 2, 2), g.voxel(3, 2, 2)], np.int32)
    with pic.Context(g) as ctx:
        sid = ctx.add_species("s", 1.0, 1.0, 2)
        ctx.upload_species(sid, p[:, :1].copy(), ids[:1].copy())
        ctx.load_interpolators()
        ctx.advance_p(sid)
        ctx.synchronize()  # finite: no error
        ctx.upload_species(sid, p, ids)
        ctx.advance_p(sid)
        with pytest.raises(pic.RunAbort):
            ctx.synchronize()
        ctx.synchronize()  # the latch is cleared once raised


def test_species_upload_rejects_ghost_ids(pic):
    g = pic.make_grid((4, 4, 4))
    with pic.Context(g) as ctx:
        sid = ctx.add_species("s", -1.0, 1.0, 2)
        p = np.zeros((7, 2), np.float32)
        with pytest.raises(pic.UsageError):
            ctx.upload_species(sid, p, np.array([0, g.voxel(1, 1, 1)], np.int32))


@pytest.mark.parametrize("order", [0, 1])
@pytest.mark.parametrize("dims,n", [((5, 4, 3), 3000), ((20, 20, 20), 300000), ((2, 2, 2), 1)])
@pytest.mark.parametrize("variant", [0])
def test_sort_bitwise(pic, orc, order, dims, n, variant):
    """The sort (LSD radix, 9-bit digits, match.any digit grouping) gives the
    reference's stable permutation (the other strategies: the ablation
    library)."""
    g = pic.make_grid(dims)
    rng = np.random.default_rng(21 + order)
    p, ids = rand_particles(g, rng, n, sort=False)
    # skewed occupancy so the interleaved rounds are ragged
    ids[: n // 3] = ids[0]
    with pic.Context(g) as ctx:
        ctx._set_sort_variant(variant)
        sid = ctx.add_species("s", -1.0, 1.0, n)
        ctx.upload_species(sid, p, ids)
        ctx.sort_particles(sid, order)
        gp, gids = ctx.download_species(sid)
    orc.sort(p, ids, interleaved=bool(order))
    assert_bitwise(gids, ids, "sorted ids")
    assert_bitwise(gp, p, "sorted lanes")


def _deck_state(orc, g, species, seed):
    out = []
    for si, (q, m, ppc, uth, drift) in enumerate(species):
        p, ids = orc.load_species(og(g), seed, si, ppc, uth, drift)
        out.append((q, m, p, ids))
    return out


@pytest.mark.parametrize("deterministic", [True, False])
def test_full_step_parity(pic, orc, deterministic):
    """SimState::step over several steps: bitwise in deterministic mode;
    fast mode: the first step's particle state is bitwise (fields identical
    before it), later steps and fields within fp32 tolerance."""
    from oracle.bindings import make_grid as omake
    g = pic.make_grid((12, 10, 8), 1.0, dt=0.25)
    o = og(g)
    species = [(-1.0, 1.0, 6, 0.2, (0.05, 0.0, 0.0)), (1.0, 100.0, 4, 0.02, (0.0, 0.0, 0.0))]
    state = _deck_state(orc, g, species, seed=4)
    f = np.zeros((16, g.padded), np.float32)
    nsteps = 6
    with pic.Context(g) as ctx:
        sids = []
        for name, (q, m, p, ids) in zip(("electron", "ion"), state):
            sid = ctx.add_species(name, q, m, ids.size)
            ctx.upload_species(sid, p, ids)
            sids.append(sid)
        ctx.upload_fields(f)
        for k in range(nsteps):
            ctx.step(deterministic=deterministic)
            orc.step(o, [(q, m, p, ids) for q, m, p, ids in state], f)
            gf = ctx.download_fields()
            for sid, (q, m, p, ids) in zip(sids, state):
                gp, gids = ctx.download_species(sid)
                if deterministic or k == 0:
                    assert_bitwise(gids, ids, f"step {k} ids")
                    assert_bitwise(gp, p, f"step {k} lanes")
                else:
                    assert (gids == ids).mean() > 0.999
                    assert_close(gp[3:6], p[3:6], 1e-4, what=f"step {k} momenta")
                    # per element (north_star: 1e-5 per step): the median and the
                    # 99th percentile of the relative error grow at most 1e-5 / step
                    p50, p99, pmax = rel_err_percentiles(gp[:6], p[:6])
                    assert p50 <= 1e-5 * k and p99 <= 1e-5 * k, (k, "offsets/momenta", p50, p99, pmax)
            if deterministic:
                assert_bitwise(gf, f, f"step {k} fields")
            else:
                for lane in (0, 1, 2, 4, 5, 6, 8, 9, 10):
                    assert_close(gf[lane], f[lane], 1e-4, what=f"step {k} lane {lane}")
                    # fields sum the atomically accumulated (cancelling) currents:
                    # the median element within 1e-5 per step, the 99th
                    # percentile (elements near a zero crossing) within 1e-4
                    p50, p99, pmax = rel_err_percentiles(gf[lane], f[lane])
                    assert p50 <= 1e-5 * (k + 1) and p99 <= 1e-4 * (k + 1), (k, lane, p50, p99, pmax)


def test_step_host_matches_device_step(pic, orc):
    g = pic.make_grid((8, 8, 8), 1.0, dt=0.25)
    state = _deck_state(orc, g, [(-1.0, 1.0, 4, 0.1, (0, 0, 0))], seed=9)
    q, m, p, ids = state[0]
    with pic.Context(g) as a, pic.Context(g) as b:
        sa = a.add_species("e", q, m, ids.size)
        sb = b.add_species("e", q, m, ids.size)
        a.upload_species(sa, p, ids)
        b.upload_species(sb, p, ids)
        hp, hid = p.copy(), ids.copy()
        for _ in range(3):
            a.step(deterministic=True)
            b.step_host([hp], [hid], deterministic=True)
        dp, did = a.download_species(sa)
        assert_bitwise(hp, dp, "step_host lanes")
        assert_bitwise(hid, did, "step_host ids")
        assert_bitwise(a.download_fields(), b.download_fields(), "step_host fields")


@pytest.mark.parametrize("chunk", [997, 4096, 1 << 25])
def test_step_host_pipeline_fast(pic, orc, chunk):
    """The chunked 3-stream host-buffer step equals the device-resident step
    (particle state bitwise: both see the same fields; fields within
    tolerance: the atomic accumulation order differs)."""
    g = pic.make_grid((10, 8, 6), 1.0, dt=0.25)
    state = _deck_state(orc, g, [(-1.0, 1.0, 5, 0.15, (0.02, 0, 0)), (1.0, 50.0, 3, 0.02, (0, 0, 0))], seed=3)
    with pic.Context(g) as a, pic.Context(g) as b:
        b._set_host_chunk(chunk)
        hosts = []
        for q, m, p, ids in state:
            sa = a.add_species("s", q, m, ids.size)
            sb = b.add_species("s", q, m, ids.size)
            a.upload_species(sa, p, ids)
            b.upload_species(sb, p, ids)
            hosts.append((p.copy(), ids.copy()))
        a.step()
        b.step_host([h[0] for h in hosts], [h[1] for h in hosts])
        for sid, (hp, hid) in enumerate(hosts):
            dp, did = a.download_species(sid)
            assert_bitwise(hid, did, "ids")
            assert_bitwise(hp, dp, "lanes")
        fa, fb = a.download_fields(), b.download_fields()
        for lane in (0, 1, 2, 4, 5, 6, 8, 9, 10):
            assert_close(fb[lane], fa[lane], 1e-5, what=f"lane {lane}")


def test_empty_species_and_zero_particles(pic):
    g = pic.make_grid((4, 4, 4))
    with pic.Context(g) as ctx:
        sid = ctx.add_species("none", -1.0, 1.0, 0)
        ctx.upload_species(sid, np.zeros((7, 0), np.float32), np.zeros(0, np.int32))
        ctx.step()
        ctx.step(deterministic=True)
        ctx.sort_particles(sid, 0)
        ctx.synchronize()
        assert ctx.species_count(sid) == 0
        f = ctx.download_fields()
        assert not f.any()


def test_graph_step_matches_plain_launches(pic, orc):
    """pic_step replays a captured CUDA graph from the third step of a
    configuration on (and a second graph after the sort swaps the record
    buffers): particle state and fields match plain launches within the fast
    mode's atomic-order tolerance; the launch counter keeps counting."""
    g = pic.make_grid((16, 12, 10), 1.0, dt=0.25)
    species = [(-1.0 / 8, 1.0 / 8, 8, 0.1, (0.05, 0.0, 0.0)), (1.0 / 8, 100.0 / 8, 4, 0.01, (0.0, 0.0, 0.0))]
    outs = []
    for graphs in (False, True):
        with pic.Context(g) as ctx:
            ctx._set_graphs(graphs)
            sids = []
            for si, (q, m, ppc, uth, drift) in enumerate(species):
                sid = ctx.add_species(f"s{si}", q, m, ppc * g.interior)
                ctx.load_synthetic(sid, ppc, uth, drift, seed=3)
                sids.append(sid)
            l0 = ctx.launch_count()
            for k in range(12):
                ctx.step()
                if k == 5:
                    for s in sids:
                        ctx.sort_particles(s)
            ctx.synchronize()
            launches = ctx.launch_count() - l0
            outs.append(([ctx.download_species(s) for s in sids], ctx.download_fields(), launches))
    (pa, fa, la), (pb, fb, lb) = outs
    for (p1, i1), (p2, i2) in zip(pa, pb):
        assert (i1 == i2).mean() > 0.999
        same = i1 == i2
        assert np.abs(p1[:, same] - p2[:, same]).max() <= 1e-4 * max(1.0, np.abs(p1).max())
    assert np.abs(fa - fb).max() <= 1e-3 * max(np.abs(fa).max(), 1e-12)
    assert la == lb


def test_deferred_sort_permutation(pic, orc):
    """A blocked sort leaves its permutation to the next default push, which
    gathers through it: the state after sort + push equals sort (applied) +
    push, and a download between them sees the sorted order."""
    g = pic.make_grid((14, 9, 7), 1.0, dt=0.25)
    rng = np.random.default_rng(5)
    p, ids = rand_particles(g, rng, 20000, sort=False)
    p[3:6] *= 0.3
    res = []
    for mode in ("materialized", "deferred", "peek"):
        with pic.Context(g) as ctx:
            sid = ctx.add_species("s", -1.0 / 16, 1.0 / 16, ids.size)
            ctx.upload_species(sid, p, ids)
            ctx.sort_particles(sid)
            if mode == "materialized":
                ctx.download_species(sid)  # any entry point applies the permutation
            if mode == "peek":
                sp, sids = ctx.download_species(sid)
                q, qi = p.copy(), ids.copy()
                orc.sort(q, qi)
                assert_bitwise(sids, qi, "sorted ids")
                assert_bitwise(sp, q, "sorted lanes")
            ctx.advance_p(sid)
            res.append(ctx.download_species(sid))
    for (a, ai), (b, bi) in zip(res[:-1], res[1:]):
        assert_bitwise(ai, bi, "ids after push")
        assert_bitwise(a, b, "lanes after push")
