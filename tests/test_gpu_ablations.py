"""The measured advance_p / sort ablations live in the
tools-only library libpic_b200_ablate.so (python
paper_2102_13133_b200/build.py --ablate).  Each valid push strategy must
still give the bitwise particle state and the accumulator within tolerance,
and each sort strategy the reference's permutation; the timing probes
(90-93, 99) are not pushes and are not checked.  Runs in a subprocess so the
product library stays the one this process loads."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ABLATE = os.path.join(ROOT, "paper_2102_13133_b200", "libpic_b200_ablate.so")

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, ROOT)
import paper_2102_13133_b200 as pic
from oracle.bindings import Orc, Grid
from tests.helpers import assert_bitwise, assert_close, rand_fields, rand_particles
orc = Orc()
g = pic.make_grid((10, 9, 8), 1.0, cfl_frac=0.9)
o = Grid(g.nx, g.ny, g.nz, g.hx, g.hy, g.hz, g.dt)
rng = np.random.default_rng(13)
f = rand_fields(g, rng, scale=0.3, sync=lambda gg, ff: orc.ghost_sync(o, ff))
interp = orc.load_interpolators(o, f)
p, ids = rand_particles(g, rng, 60000, u_scale=0.5, sort=True)
wp, wids = p.copy(), ids.copy()
wacc = np.zeros((g.padded, 12), np.float32)
orc.advance_particles(o, -1.0, 1.0, wp, wids, interp, wacc, False)
for v in list(range(56)):
    with pic.Context(g) as ctx:
        sid = ctx.add_species("s", -1.0, 1.0, ids.size)
        ctx._set_push_variant(v)
        ctx.upload_species(sid, p, ids)
        ctx.upload_fields(f)
        ctx.load_interpolators()
        ctx.clear_accumulator()
        ctx.advance_p(sid)
        ctx.synchronize()
        gp, gids = ctx.download_species(sid)
        gacc = ctx.download_accumulator()
    assert_bitwise(gids, wids, f"ids v{v}")
    assert_bitwise(gp, wp, f"lanes v{v}")
    assert_close(gacc, wacc, 1e-5, what=f"accumulator v{v}")
ps, idss = rand_particles(g, rng, 30000, sort=False)
for order in (0, 1):
    sp, sids_ = ps.copy(), idss.copy()
    orc.sort(sp, sids_, interleaved=bool(order))
    for v in range(5):
        with pic.Context(g) as ctx:
            ctx._set_sort_variant(v)
            sid = ctx.add_species("s", -1.0, 1.0, idss.size)
            ctx.upload_species(sid, ps, idss)
            ctx.sort_particles(sid, order)
            gp, gids = ctx.download_species(sid)
        assert_bitwise(gids, sids_, f"sort ids v{v}")
        assert_bitwise(gp, sp, f"sort lanes v{v}")
print("ablations ok")
"""


def _ablate_current():
    from paper_2102_13133_b200 import build
    return build.up_to_date(ABLATE)


@pytest.mark.skipif(not os.path.exists(ABLATE) or not _ablate_current(),
                    reason="libpic_b200_ablate.so not built or older than the sources (build.py --ablate)")
def test_ablation_strategies_in_tools_library():
    env = dict(os.environ, PIC_LIB_PATH=ABLATE)
    r = subprocess.run([sys.executable, "-c", f"ROOT = {ROOT!r}\n" + SCRIPT], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "ablations ok" in r.stdout
