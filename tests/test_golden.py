"""Golden vectors made by the unmodified reference (tests/golden/make_golden.py)
reproduced bit-for-bit by the oracle (CPU) and by the sm_100a path (GPU)."""
import os

import numpy as np
import pytest

from oracle.bindings import Grid, Orc
from tests.helpers import assert_bitwise

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLD, name)))


def grid_of(d):
    n, h = d["grid"], d["h_dt"]
    return Grid(int(n[0]), int(n[1]), int(n[2]), float(h[0]), float(h[1]), float(h[2]), float(h[3]))


SPECIES = [(-1.0, 1.0, 4, 0.3, (0.05, 0.0, 0.0), 0.02, 2, 3, False),
           (1.0, 25.0, 2, 0.05, (0.0, 0.0, 0.0), 0.0, 1, 4, True)]


@pytest.fixture(scope="module")
def orc():
    return Orc()


def test_oracle_reproduces_simstate_golden(orc):
    d = load("simstate_small.npz")
    g = grid_of(d)
    state = []
    for si, (q, m, ppc, uth, drift, pert, kmode, sint, inter) in enumerate(SPECIES):
        p, ids = orc.load_species(g, 17, si, ppc, uth, drift, pert, kmode)
        assert_bitwise(p, d[f"p0_{si}"], f"load {si}")
        assert_bitwise(ids, d[f"id0_{si}"], f"load ids {si}")
        state.append([q, m, p, ids, sint, inter])
    f = d["fields0"].copy()
    for step in range(1, 7):
        orc.step(g, [(s[0], s[1], s[2], s[3]) for s in state], f)
        for s in state:
            if step % s[4] == 0:
                orc.sort(s[2], s[3], s[5])
    assert_bitwise(f, d["fields6"], "fields after 6 steps")
    for si, s in enumerate(state):
        assert_bitwise(s[2], d[f"p6_{si}"], f"lanes {si}")
        assert_bitwise(s[3], d[f"id6_{si}"], f"ids {si}")


def test_oracle_reproduces_advance_golden(orc):
    d = load("advance_small.npz")
    g = grid_of(d)
    assert_bitwise(orc.load_interpolators(g, d["fields"]), d["interp"], "interp")
    p, ids = d["p_in"].copy(), d["id_in"].copy()
    acc = np.zeros((g.padded, 12), np.float32)
    orc.advance_particles(g, -1.0, 1.0, p, ids, d["interp"], acc)
    assert_bitwise(p, d["p_out"], "lanes")
    assert_bitwise(ids, d["id_out"], "ids")
    assert_bitwise(acc, d["acc"], "acc")
    orc.ghost_fold(g, acc)
    assert_bitwise(acc, d["acc_folded"], "fold")
    f = d["fields"].copy()
    orc.clear_currents(g, f)
    orc.unload(g, acc, f)
    assert_bitwise(f, d["fields_unloaded"], "unload")


def test_oracle_reproduces_sort_golden(orc):
    d = load("sort_small.npz")
    for inter, key in ((False, "blocked"), (True, "inter")):
        p, ids = d["p_in"].copy(), d["id_in"].copy()
        orc.sort(p, ids, inter)
        assert_bitwise(p, d[f"p_{key}"], key)
        assert_bitwise(ids, d[f"id_{key}"], key)


# ---- the sm_100a path against the same vectors --------------------------------
@pytest.fixture(scope="module")
def pic():
    import paper_2102_13133_b200 as pic
    pic.lib()
    return pic


def pgrid(pic, d):
    n, h = d["grid"], d["h_dt"]
    return pic.Grid(int(n[0]), int(n[1]), int(n[2]), float(h[0]), float(h[1]), float(h[2]), float(h[3]))


@pytest.mark.gpu
def test_gpu_reproduces_simstate_golden(pic, orc):
    d = load("simstate_small.npz")
    g = pgrid(pic, d)
    with pic.Context(g) as ctx:
        for si, (q, m, *_rest) in enumerate(SPECIES):
            sid = ctx.add_species(f"s{si}", q, m, d[f"id0_{si}"].size)
            ctx.upload_species(sid, d[f"p0_{si}"], d[f"id0_{si}"])
        ctx.upload_fields(d["fields0"])
        for step in range(1, 7):
            ctx.step(deterministic=True)
            for si, s in enumerate(SPECIES):
                if step % s[7] == 0:
                    ctx.sort_particles(si, 1 if s[8] else 0)
        assert_bitwise(ctx.download_fields(), d["fields6"], "fields after 6 steps")
        for si in range(2):
            p, ids = ctx.download_species(si)
            assert_bitwise(p, d[f"p6_{si}"], f"lanes {si}")
            assert_bitwise(ids, d[f"id6_{si}"], f"ids {si}")


@pytest.mark.gpu
def test_gpu_reproduces_advance_golden(pic):
    d = load("advance_small.npz")
    g = pgrid(pic, d)
    with pic.Context(g) as ctx:
        sid = ctx.add_species("e", -1.0, 1.0, d["id_in"].size)
        ctx.upload_species(sid, d["p_in"], d["id_in"])
        ctx.upload_fields(d["fields"])
        ctx.load_interpolators()
        assert_bitwise(ctx.download_interpolators(), d["interp"], "interp")
        ctx.clear_accumulator()
        ctx.advance_p(sid, deterministic=True)
        p, ids = ctx.download_species(sid)
        assert_bitwise(p, d["p_out"], "lanes")
        assert_bitwise(ids, d["id_out"], "ids")
        assert_bitwise(ctx.download_accumulator(), d["acc"], "acc")
        ctx.ghost_fold_currents()
        assert_bitwise(ctx.download_accumulator(), d["acc_folded"], "fold")
        ctx.clear_currents()
        ctx.unload_currents()
        assert_bitwise(ctx.download_fields(), d["fields_unloaded"], "unload")


@pytest.mark.gpu
def test_gpu_reproduces_sort_golden(pic):
    d = load("sort_small.npz")
    n = d["grid"]
    g = pic.make_grid((int(n[0]), int(n[1]), int(n[2])))
    for order, key in ((0, "blocked"), (1, "inter")):
        with pic.Context(g) as ctx:
            sid = ctx.add_species("s", -1.0, 1.0, d["id_in"].size)
            ctx.upload_species(sid, d["p_in"], d["id_in"])
            ctx.sort_particles(sid, order)
            p, ids = ctx.download_species(sid)
        assert_bitwise(p, d[f"p_{key}"], key)
        assert_bitwise(ids, d[f"id_{key}"], key)
