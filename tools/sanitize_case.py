"""A small workload that launches every product kernel family, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

  python tools/sanitize_case.py            # plain run (sanity)
  compute-sanitizer --tool racecheck python tools/sanitize_case.py

Covers: the default push in voxel order (in-place, counting and reordering
pushes, the relabelling sort, the scatter back to logical order), the
in-place push with the deferred radix sort and the gathering push, the
interleaved sort, deterministic mode (stage / emit / segment sort / ordered
reduce), exact_gyration (advance_p_run), the field kernels, diagnostics in
both summation orders, walls (reflect / absorb / PEC / Mur), the laser and
the emitter, and the x-decomposed pieces (emigrant lists, migration pack /
append, halo pack / unpack) on two in-process slabs."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2102_13133_b200 as pic  # noqa: E402
from tests.helpers import rand_fields, rand_particles  # noqa: E402


def deck(ctx, g, rng, n=6000, species=((-1.0, 1.0, 0.4), (1.0, 25.0, 0.1))):
    sids = []
    for k, (q, m, u) in enumerate(species):
        p, ids = rand_particles(g, rng, n, u_scale=u)
        sid = ctx.add_species(f"s{k}", q, m, n + 4096)
        ctx.upload_species(sid, p, ids)
        sids.append(sid)
    ctx.upload_fields(rand_fields(g, rng, scale=0.05))
    ctx.ghost_sync_fields()
    return sids


def main():
    rng = np.random.default_rng(1)
    g = pic.make_grid((10, 8, 6), 1.0, dt=0.25)
    # default fast step: voxel order, reorder every 5th push, relabel at sorts
    with pic.Context(g) as ctx:
        sids = deck(ctx, g, rng)
        for k in range(1, 13):
            ctx.step()
            if k % 4 == 0:
                for s in sids:
                    ctx.sort_particles(s)
        ctx.download_species(0)
        ctx.sort_particles(1, pic.SORT_INTERLEAVED)
        d = ctx.diagnostics()
        ctx.refresh_charge_diagnostics()
        ctx.diagnostics_order(True)
        ctx.diagnostics()
        ctx.step(deterministic=True)
        ctx.step(exact_gyration=True)
        ctx.synchronize()
    # in-place push + deferred radix sort + gathering push (voxel order off)
    with pic.Context(g) as ctx:
        ctx._set_voxel_order(False)
        sids = deck(ctx, g, rng)
        for k in range(1, 6):
            ctx.step()
            for s in sids:
                ctx.sort_particles(s)
        ctx.download_species(0)
        ctx.synchronize()
    # walls, laser, emitter
    with pic.Context(g) as ctx:
        ctx.set_x_boundary(0, pic.PBC_REFLECT, pic.FBC_PEC)
        ctx.set_x_boundary(1, pic.PBC_ABSORB, pic.FBC_MUR)
        sids = deck(ctx, g, rng)
        ctx.set_laser(2, 0.05, 1.0, pol=1, ramp_steps=4.0)
        ctx.set_emitter(sids[0], 0, 1, 0.05)
        for _ in range(4):
            ctx.step()
        ctx.synchronize()
    # x-decomposition on two in-process slabs
    import torch  # noqa: F401
    from paper_2102_13133_b200.domain import CudaSlab, DecomposedSim, LocalTransport, SlabGeometry
    geom = SlabGeometry(16, 6, 6, 2, h=(1.0, 1.0, 1.0), dt=0.25)
    slabs = {r: CudaSlab(geom.local_grid(), r, r == 0, device=0) for r in range(2)}
    sim = DecomposedSim(geom, slabs, LocalTransport())
    for name, q, m in (("e", -1.0, 1.0), ("i", 1.0, 25.0)):
        sid = sim.add_species(name, q, m, 20000)
        for r, sl in slabs.items():
            sl.ctx.load_synthetic(sid, 8, 0.2, (0.1, 0.0, 0.0), seed=3 + r)
    for _ in range(3):
        sim.step()
    for sl in slabs.values():
        sl.ctx.synchronize()
        sl.ctx.close()
    print("sanitize_case: ok", d["particle_count"])


if __name__ == "__main__":
    main()
