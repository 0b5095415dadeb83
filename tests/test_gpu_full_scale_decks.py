"""Full-size sampled push parity for the other benchmark configs:
thermal e/i at 256^3 (`weak`, 2^30 particles, u_th 0.1 electrons: multi-face
movers), the double Harris sheet (256 x 64 x 256, four species, sheared
fields) and the laser-plasma deck (2048 x 64 x 64, walls + laser).  After a
few steps, 2^20 random particles of every species are pushed by the device
and by the oracle through the same downloaded interpolators; the records
must agree bit for bit (see test_gpu_full_scale.py for the two-stream deck).
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu


def _build(name):
    import paper_2102_13133_b200 as pic
    from bench import CONFIGS
    cfg = CONFIGS[name]
    deck = cfg.get("deck")
    if deck is not None:
        g = deck.grid()
        ctx = pic.Context(g)
        sids = deck.load(ctx, seed=1234)
    else:
        g = pic.make_grid(cfg["n"], cfg["h"], dt=cfg["dt"])
        ctx = pic.Context(g)
        sids = []
        for sname, q, m, ppc, uth, drift in cfg["species"]:
            sid = ctx.add_species(sname, q, m, ppc * g.interior)
            ctx.load_synthetic(sid, ppc, uth, drift, seed=1234)
            sids.append(sid)
    return ctx, g, cfg, sids


@pytest.mark.parametrize("name", ["weak", "harris", "lpi"])
def test_full_scale_push_sample_bitwise_decks(name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    if torch.cuda.get_device_properties(0).total_memory < 150e9:
        pytest.skip("needs a 180 GB B200")
    from oracle.bindings import Grid as OGrid
    from oracle.bindings import Orc
    ctx, g, cfg, sids = _build(name)
    try:
        for s in sids:
            ctx.sort_particles(s)  # the bench's first sort (deferred permutation pending)
        for _ in range(3):
            ctx.step()
        orc = Orc()
        og = OGrid(g.nx, g.ny, g.nz, g.hx, g.hy, g.hz, g.dt)
        ctx.clear_accumulator()
        ctx.clear_currents()
        ctx.load_interpolators()
        i18 = ctx.download_interpolators()
        rng = np.random.default_rng(11)
        for sid, (sname, q, m, *_rest) in zip(sids, cfg["species"]):
            n = ctx.species_count(sid)
            pos = torch.empty((n, 4), dtype=torch.float32, device="cuda")
            mom = torch.empty((n, 4), dtype=torch.float32, device="cuda")
            torch.cuda.synchronize()
            ctx.download_records(sid, pos, mom)
            torch.cuda.synchronize()
            idx = torch.from_numpy(np.sort(rng.choice(n, min(n, 1 << 20), replace=False))).cuda()
            p0, u0 = pos[idx].cpu().numpy(), mom[idx].cpu().numpy()
            ctx.advance_p(sid)
            torch.cuda.synchronize()
            ctx.download_records(sid, pos, mom)
            torch.cuda.synchronize()
            p1, u1 = pos[idx].cpu().numpy(), mom[idx].cpu().numpy()
            del pos, mom
            torch.cuda.empty_cache()
            p7 = np.ascontiguousarray(np.concatenate([p0[:, 0:3].T, u0[:, 0:4].T]), np.float32)
            ids = np.ascontiguousarray(p0[:, 3].view(np.int32))
            acc = np.zeros((g.padded, 12), np.float32)
            orc.advance_particles(og, q, m, p7, ids, i18, acc)
            got = np.concatenate([p1[:, 0:3].T, u1[:, 0:4].T])
            assert (p1[:, 3].view(np.int32) == ids).all(), f"{name}/{sname}: voxel ids"
            assert (got.view(np.uint32) == p7.view(np.uint32)).all(), f"{name}/{sname}: particle lanes"
    finally:
        ctx.close()
        torch.cuda.empty_cache()


@pytest.mark.parametrize("name,sorted_first", [("weak", False), ("weak", True), ("harris", True)])
def test_full_scale_step_sample_bitwise_decks(name, sorted_first):
    """The step's own push at full size — every species in one launch
    (interleaved for the two thermal species, contiguous for Harris' four),
    in place, or reordering with the relabel of a blocked sort just before
    it: 2^20 sampled particles per species against the oracle's push
    through the interpolators of the step's fields (after a sort, the
    samples are found at their stable-counting-sort positions)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    if torch.cuda.get_device_properties(0).total_memory < 150e9:
        pytest.skip("needs a 180 GB B200")
    from oracle.bindings import Grid as OGrid
    from oracle.bindings import Orc
    ctx, g, cfg, sids = _build(name)
    try:
        for _ in range(3):
            ctx.step()
        orc = Orc()
        og = OGrid(g.nx, g.ny, g.nz, g.hx, g.hy, g.hz, g.dt)
        f = ctx.download_fields()
        i18 = orc.load_interpolators(og, f)
        del f
        rng = np.random.default_rng(13)
        before = []
        for sid in sids:
            n = ctx.species_count(sid)
            pos = torch.empty((n, 4), dtype=torch.float32, device="cuda")
            mom = torch.empty((n, 4), dtype=torch.float32, device="cuda")
            torch.cuda.synchronize()
            ctx.download_records(sid, pos, mom)
            torch.cuda.synchronize()
            idx = torch.from_numpy(np.sort(rng.choice(n, min(n, 1 << 20), replace=False))).cuda()
            at = idx
            if sorted_first:  # where the blocked sort puts them: the stable argsort's inverse
                perm = torch.sort(pos[:, 3].contiguous().view(torch.int32), stable=True).indices
                inv = torch.empty_like(perm)
                inv[perm] = torch.arange(n, device="cuda")
                at = inv[idx]
                del perm, inv
            before.append((at, pos[idx].cpu().numpy(), mom[idx].cpu().numpy()))
            del pos, mom
            torch.cuda.empty_cache()
        if sorted_first:
            for sid in sids:  # a blocked sort: the step's push reorders and relabels
                ctx.sort_particles(sid)
        b0 = ctx._batched_launches()
        ctx.step()
        assert ctx._batched_launches() > b0
        for sid, (sname, q, m, *_rest), (at, p0, u0) in zip(sids, cfg["species"], before):
            n = ctx.species_count(sid)
            pos = torch.empty((n, 4), dtype=torch.float32, device="cuda")
            mom = torch.empty((n, 4), dtype=torch.float32, device="cuda")
            torch.cuda.synchronize()
            ctx.download_records(sid, pos, mom)
            torch.cuda.synchronize()
            p1, u1 = pos[at].cpu().numpy(), mom[at].cpu().numpy()
            del pos, mom
            torch.cuda.empty_cache()
            p7 = np.ascontiguousarray(np.concatenate([p0[:, 0:3].T, u0[:, 0:4].T]), np.float32)
            ids = np.ascontiguousarray(p0[:, 3].view(np.int32))
            acc = np.zeros((g.padded, 12), np.float32)
            orc.advance_particles(og, q, m, p7, ids, i18, acc)
            got = np.concatenate([p1[:, 0:3].T, u1[:, 0:4].T])
            assert (p1[:, 3].view(np.int32) == ids).all(), f"{name}/{sname}: voxel ids"
            assert (got.view(np.uint32) == p7.view(np.uint32)).all(), f"{name}/{sname}: particle lanes"
    finally:
        ctx.close()
        torch.cuda.empty_cache()
