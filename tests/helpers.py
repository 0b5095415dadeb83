"""Shared fixtures for the parity tests: seeded random states in the
reference's field-major conventions, and bitwise comparison helpers."""
from __future__ import annotations

import numpy as np


def rand_fields(g, rng, scale=0.5, sync=None):
    """Random E/B (and zero J/rho) on the padded lattice."""
    f = np.zeros((16, g.padded), np.float32)
    for lane in (0, 1, 2, 4, 5, 6):
        f[lane] = (rng.standard_normal(g.padded) * scale).astype(np.float32)
    if sync is not None:
        sync(g, f)
    return f


def interior_ids(g, rng, n):
    ix = rng.integers(1, g.nx + 1, n)
    iy = rng.integers(1, g.ny + 1, n)
    iz = rng.integers(1, g.nz + 1, n)
    return (ix + (g.nx + 2) * (iy + (g.ny + 2) * iz)).astype(np.int32)


def rand_particles(g, rng, n, u_scale=0.5, sort=True, w_random=True):
    """n particles with interior ids (sorted by voxel if requested), offsets
    in [-1, 1], momenta ~ N(0, u_scale)."""
    ids = interior_ids(g, rng, n)
    if sort:
        ids.sort(kind="stable")
    p = np.zeros((7, n), np.float32)
    p[0:3] = rng.uniform(-1, 1, (3, n)).astype(np.float32)
    p[3:6] = (rng.standard_normal((3, n)) * u_scale).astype(np.float32)
    p[6] = rng.uniform(0.5, 2.0, n).astype(np.float32) if w_random else 1.0
    return p, ids


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32) if a.dtype == np.float32 else a


def assert_bitwise(a, b, what=""):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, f"{what}: shape {a.shape} vs {b.shape}"
    if a.dtype == np.float32:
        eq = bits(a) == bits(b)
    else:
        eq = a == b
    if not eq.all():
        idx = np.argwhere(~eq)[:5]
        samples = [(tuple(i), a[tuple(i)], b[tuple(i)]) for i in idx]
        raise AssertionError(f"{what}: {int((~eq).sum())} of {eq.size} differ; first {samples}")


def assert_close(a, b, rtol, atol_scale=None, what=""):
    """|a - b| <= rtol * max(|b|.max(), tiny) elementwise (fp32 tolerance
    relative to the array's scale)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    scale = atol_scale if atol_scale is not None else max(np.abs(b).max(), 1e-30)
    err = np.abs(a - b).max() if a.size else 0.0
    assert err <= rtol * scale, f"{what}: max |diff| {err:.3e} > {rtol:g} * {scale:.3e}"


def rel_err_percentiles(a, b, floor_frac=1e-3):
    """Per-element relative error |a - b| / (|b| + floor), floor = floor_frac x
    rms(b) (elements at the array's zero crossings are compared at that
    floor), as (p50, p99, max)."""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    if a.size == 0:
        return 0.0, 0.0, 0.0
    floor = floor_frac * max(float(np.sqrt(np.mean(b * b))), 1e-30)
    e = np.abs(a - b) / (np.abs(b) + floor)
    return float(np.percentile(e, 50)), float(np.percentile(e, 99)), float(e.max())
