import numpy as np, sys
sys.path.insert(0, '.')
import paper_2102_13133_b200 as pic
from paper_2102_13133_b200 import F
from paper_2102_13133_b200.decks import LPI
for omega0, e0, steps in [(0.5, 1e-3, 1000), (0.5, 0.0, 1000), (0.5, 1e-3, 400)]:
    d = LPI(omega0=omega0, e0=e0, ramp_steps=3 * 2 * np.pi / omega0 / 0.1)
    g = d.grid()
    with pic.Context(g) as ctx:
        d.load(ctx)
        for _ in range(steps):
            ctx.step()
        f = ctx.download_fields()
        ey = f[F["ey"]].reshape(g.nz + 2, g.ny + 2, g.nx + 2)[1, 1, 1:-1]
        ex = f[F["ex"]].reshape(g.nz + 2, g.ny + 2, g.nx + 2)[1, 1, 1:-1]
    seg = lambda a, b: float(np.abs(ey[a:b]).max())
    print(omega0, e0, steps, "vac", seg(25, 140), "slab-front", seg(150, 170), "slab-mid", seg(180, 230), "beyond", seg(275, 375), "ex-max", float(np.abs(ex).max()))
    print(" profile", np.round(np.abs(ey[::20]) * 1e4, 2).tolist())
