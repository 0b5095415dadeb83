"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref,
minipic fp32 compiled from /root/reference/proj sources).  Run here (where
/root/reference exists):  python tests/golden/make_golden.py
The fixtures pin the oracle restatement on machines without the reference."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.bindings import Ref, make_grid  # noqa: E402
from tests.helpers import rand_particles  # noqa: E402

DECK = """[grid]
nx = 6
ny = 5
nz = 4
lx = 6
ly = 5
lz = 4
dt = 0.25
steps = 6
[species.electron]
q = -1
m = 1
ppc = 4
u_th = 0.3
drift = 0.05 0 0
perturb_ux = 0.02
perturb_kmode = 2
sort_interval = 3
[species.ion]
q = 1
m = 25
ppc = 2
u_th = 0.05
sort_interval = 4
sort_order = interleaved
[run]
seed = 17
diag_interval = 2
"""


def main():
    ref = Ref()
    # 1. SimState: initial load, then 6 steps of step()+sort cadence
    sim = ref.sim(DECK)
    g = sim.grid
    out = {"grid": np.array([g.nx, g.ny, g.nz], np.int32), "h_dt": np.array([g.hx, g.hy, g.hz, g.dt], np.float32),
           "fields0": sim.fields()}
    for s in range(2):
        out[f"p0_{s}"], out[f"id0_{s}"] = sim.species(s)
    sim.step_and_sort(6)
    out["fields6"] = sim.fields()
    for s in range(2):
        out[f"p6_{s}"], out[f"id6_{s}"] = sim.species(s)
    np.savez_compressed(os.path.join(HERE, "simstate_small.npz"), **out)
    # the run-loop diagnostics CSV of the same deck (fresh state)
    with open(os.path.join(HERE, "simstate_small_diagnostics.csv"), "w") as fh:
        fh.write(ref.sim(DECK).run_csv())

    # 2. one advance_particles call with random fields and movers
    g = make_grid((5, 4, 3), (1.0, 0.9, 1.2), cfl_frac=0.9)
    rng = np.random.default_rng(2024)
    f = np.zeros((16, g.padded), np.float32)
    for lane in (0, 1, 2, 4, 5, 6):
        f[lane] = (rng.standard_normal(g.padded) * 0.4).astype(np.float32)
    ref.ghost_sync(g, f)
    interp = ref.load_interpolators(g, f)
    p, ids = rand_particles(g, rng, 1500, u_scale=0.8)
    sb = ref.scatter(g, backend=2)
    p1, i1 = p.copy(), ids.copy()
    ref.advance_particles(g, -1.0, 1.0, p1, i1, interp, sb)
    acc = sb.reduce()
    folded = acc.copy()
    ref.ghost_fold(g, folded)
    f2 = f.copy()
    ref.clear_currents(g, f2)
    ref.unload(g, folded, f2)
    np.savez_compressed(os.path.join(HERE, "advance_small.npz"),
                        grid=np.array([g.nx, g.ny, g.nz], np.int32),
                        h_dt=np.array([g.hx, g.hy, g.hz, g.dt], np.float32),
                        fields=f, interp=interp, p_in=p, id_in=ids, p_out=p1, id_out=i1, acc=acc,
                        acc_folded=folded, fields_unloaded=f2)

    # 3. both sort orders on a ragged store
    rng = np.random.default_rng(77)
    g = make_grid((4, 3, 3))
    p, ids = rand_particles(g, rng, 600, sort=False)
    ids[:150] = ids[0]
    pb, ib = p.copy(), ids.copy()
    ref.sort(pb, ib, interleaved=False)
    pi, ii = p.copy(), ids.copy()
    ref.sort(pi, ii, interleaved=True)
    np.savez_compressed(os.path.join(HERE, "sort_small.npz"), grid=np.array([g.nx, g.ny, g.nz], np.int32),
                        p_in=p, id_in=ids, p_blocked=pb, id_blocked=ib, p_inter=pi, id_inter=ii)
    print("golden fixtures written")


if __name__ == "__main__":
    main()
