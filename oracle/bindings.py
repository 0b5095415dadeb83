"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU checkers.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  The product package
(``paper_2102_13133_b200``) never imports, links or calls anything here.

Two checkers:

* ``Orc`` — ``oracle/liborc.so``, the plain-C restatement (oracle/pic_oracle.c);
* ``Ref`` — ``oracle/_ref/libminipic_ref.so``, the unmodified reference compiled
  from ``/root/reference/proj`` sources plus the marshalling shim
  (oracle/ref_shim.cpp).  Present only where it was built.

All arrays follow the reference's field-major convention (lane-major):
fields ``(16, V)``, interpolators ``(18, V)``, particles ``(7, n)`` + ids ``(n,)``;
the accumulator is ``(V, 12)`` (the ScatterBuffer dense form).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "liborc.so")
REF_PATH = os.path.join(HERE, "_ref", "libminipic_ref.so")

F32P = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
I32P = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


class Grid(C.Structure):
    """GridDescriptor (proj/include/minipic/grid.hpp:15-38), fp32 build."""

    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("hx", C.c_float), ("hy", C.c_float), ("hz", C.c_float),
                ("dt", C.c_float)]

    @property
    def padded(self) -> int:
        return (self.nx + 2) * (self.ny + 2) * (self.nz + 2)

    def voxel(self, ix, iy, iz) -> int:
        return ix + (self.nx + 2) * (iy + (self.ny + 2) * iz)

    def coords(self, v):
        v = np.asarray(v)
        ix = v % (self.nx + 2)
        rest = v // (self.nx + 2)
        return ix, rest % (self.ny + 2), rest // (self.ny + 2)


def make_grid(n, h=1.0, dt=None, cfl_frac=0.5) -> Grid:
    nx, ny, nz = (n, n, n) if np.isscalar(n) else n
    hx, hy, hz = (h, h, h) if np.isscalar(h) else h
    g = Grid(nx, ny, nz, hx, hy, hz, 0.0)
    if dt is None:
        f32 = np.float32
        s = f32(1) / (f32(hx) * f32(hx)) + f32(1) / (f32(hy) * f32(hy)) + f32(1) / (f32(hz) * f32(hz))
        dt = f32(cfl_frac) * (f32(1) / np.sqrt(s, dtype=np.float32))
    g.dt = float(np.float32(dt))
    return g


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class UsageError(OracleError):
    pass


class RunAbort(OracleError):
    pass


def _raise(code, msg):
    if code == 1:
        raise UsageError(code, msg)
    if code == 2:
        raise RunAbort(code, msg)
    raise OracleError(code, msg)


class Orc:
    """Plain-C restatement (oracle/pic_oracle.c)."""

    def __init__(self, path: str = ORC_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle orc`")
        L = self.lib = C.CDLL(path)
        G = C.POINTER(Grid)
        L.orc_last_error.restype = C.c_char_p
        L.orc_cfl_limit.argtypes = [G]
        L.orc_cfl_limit.restype = C.c_float
        L.orc_load_interpolators.argtypes = [G, F32P, F32P]
        L.orc_advance_particles.argtypes = [G, C.c_float, C.c_float, C.c_long, F32P, I32P, F32P, F32P, C.c_int]
        L.orc_ghost_fold.argtypes = [G, F32P]
        L.orc_clear_currents.argtypes = [G, F32P]
        L.orc_unload.argtypes = [G, F32P, F32P]
        L.orc_advance_b.argtypes = [G, F32P, C.c_float]
        L.orc_advance_e.argtypes = [G, F32P]
        L.orc_ghost_sync.argtypes = [G, F32P]
        L.orc_sort.argtypes = [C.c_long, F32P, I32P, C.c_int]
        L.orc_load_species.argtypes = [G, C.c_uint64, C.c_int, C.c_int, C.c_float, F32P, C.c_float, C.c_int, F32P, I32P]
        L.orc_deposit_rho.argtypes = [G, C.c_float, C.c_long, F32P, I32P, F32P]
        L.orc_compute_div_errors.argtypes = [G, F32P]
        L.orc_field_energy.argtypes = [G, F32P, F32P]
        L.orc_kinetic_energy_centered.argtypes = [G, C.c_float, C.c_float, C.c_long, F32P, I32P, F32P]
        L.orc_kinetic_energy_centered.restype = C.c_float
        L.orc_max_abs_lane.argtypes = [G, F32P, C.c_int]
        L.orc_max_abs_lane.restype = C.c_float

    def _chk(self, rc):
        if rc:
            _raise(rc, self.lib.orc_last_error().decode())

    def load_interpolators(self, g, f16):
        out = np.zeros((18, g.padded), np.float32)
        self.lib.orc_load_interpolators(C.byref(g), f16, out)
        return out

    def advance_particles(self, g, q, m, p7, ids, i18, acc, exact_gyration=False):
        self._chk(self.lib.orc_advance_particles(C.byref(g), q, m, ids.size, p7, ids, i18, acc, int(exact_gyration)))

    def ghost_fold(self, g, acc):
        self.lib.orc_ghost_fold(C.byref(g), acc)

    def clear_currents(self, g, f16):
        self.lib.orc_clear_currents(C.byref(g), f16)

    def unload(self, g, acc, f16):
        self.lib.orc_unload(C.byref(g), acc, f16)

    def advance_b(self, g, f16, frac):
        self.lib.orc_advance_b(C.byref(g), f16, frac)

    def advance_e(self, g, f16):
        self.lib.orc_advance_e(C.byref(g), f16)

    def ghost_sync(self, g, f16):
        self.lib.orc_ghost_sync(C.byref(g), f16)

    def sort(self, p7, ids, interleaved=False):
        self._chk(self.lib.orc_sort(ids.size, p7, ids, int(interleaved)))

    def load_species(self, g, seed, si, ppc, u_th, drift=(0, 0, 0), perturb_ux=0.0, perturb_kmode=1):
        n = ppc * g.nx * g.ny * g.nz
        p = np.zeros((7, n), np.float32)
        ids = np.zeros(n, np.int32)
        self.lib.orc_load_species(C.byref(g), seed, si, ppc, u_th, np.asarray(drift, np.float32),
                                  perturb_ux, perturb_kmode, p, ids)
        return p, ids

    def step(self, g, species, f16, exact_gyration=False):
        """species: list of (q, m, p7, ids) mutated in place."""
        acc = np.zeros((g.padded, 12), np.float32)
        interp = np.zeros((18, g.padded), np.float32)
        self.clear_currents(g, f16)
        interp[:] = self.load_interpolators(g, f16)
        for q, m, p7, ids in species:
            self.advance_particles(g, q, m, p7, ids, interp, acc, exact_gyration)
        self.ghost_fold(g, acc)
        self.unload(g, acc, f16)
        self.advance_b(g, f16, 0.5)
        self.ghost_sync(g, f16)
        self.advance_e(g, f16)
        self.ghost_sync(g, f16)
        self.advance_b(g, f16, 0.5)
        self.ghost_sync(g, f16)
        return acc

    # diagnostics
    def deposit_rho(self, g, q, p7, ids, f16):
        self.lib.orc_deposit_rho(C.byref(g), q, ids.size, p7, ids, f16)

    def compute_div_errors(self, g, f16):
        self.lib.orc_compute_div_errors(C.byref(g), f16)

    def field_energy(self, g, f16):
        out = np.zeros(2, np.float32)
        self.lib.orc_field_energy(C.byref(g), f16, out)
        return out

    def kinetic_energy_centered(self, g, q, m, p7, ids, i18):
        return self.lib.orc_kinetic_energy_centered(C.byref(g), q, m, ids.size, p7, ids, i18)

    def max_abs_lane(self, g, f16, lane):
        return self.lib.orc_max_abs_lane(C.byref(g), f16, lane)


def ref_available(path: str = REF_PATH) -> bool:
    return os.path.exists(path)


class Ref:
    """The unmodified reference (fp32 build) behind oracle/ref_shim.cpp."""

    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        G = C.POINTER(Grid)
        L.mref_last_error.restype = C.c_char_p
        L.mref_scatter_new.argtypes = [G, C.c_int, C.c_int]
        L.mref_scatter_new.restype = C.c_void_p
        L.mref_scatter_free.argtypes = [C.c_void_p]
        L.mref_scatter_clear.argtypes = [C.c_void_p]
        L.mref_scatter_reduce.argtypes = [C.c_void_p, F32P]
        L.mref_load_interpolators.argtypes = [G, F32P, F32P, C.c_int]
        L.mref_advance_particles.argtypes = [G, C.c_float, C.c_float, C.c_long, F32P, I32P, F32P, C.c_void_p,
                                             C.c_long, C.c_int, C.c_int, C.c_int]
        L.mref_ghost_fold.argtypes = [G, F32P]
        L.mref_unload.argtypes = [G, F32P, F32P]
        L.mref_clear_currents.argtypes = [G, F32P]
        L.mref_advance_b.argtypes = [G, F32P, C.c_float, C.c_int]
        L.mref_advance_e.argtypes = [G, F32P, C.c_int]
        L.mref_ghost_sync.argtypes = [G, F32P]
        L.mref_sort.argtypes = [C.c_long, F32P, I32P, C.c_int]
        L.mref_deposit_rho.argtypes = [G, C.c_float, C.c_long, F32P, I32P, F32P]
        L.mref_compute_div_errors.argtypes = [G, F32P]
        L.mref_field_energy.argtypes = [G, F32P, F32P]
        L.mref_kinetic_energy_centered.argtypes = [G, C.c_float, C.c_float, C.c_long, F32P, I32P, F32P,
                                                   C.POINTER(C.c_float)]
        L.mref_max_abs_lane.argtypes = [G, F32P, C.c_int, C.POINTER(C.c_float)]
        L.mref_deck_roundtrip.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_long]
        L.mref_sim_new.argtypes = [C.c_char_p]
        L.mref_sim_new.restype = C.c_void_p
        L.mref_sim_free.argtypes = [C.c_void_p]
        L.mref_sim_grid.argtypes = [C.c_void_p, G]
        L.mref_sim_nspecies.argtypes = [C.c_void_p]
        L.mref_sim_species_size.argtypes = [C.c_void_p, C.c_int]
        L.mref_sim_species_size.restype = C.c_long
        L.mref_sim_species_get.argtypes = [C.c_void_p, C.c_int, F32P, I32P]
        L.mref_sim_species_set.argtypes = [C.c_void_p, C.c_int, F32P, I32P]
        L.mref_sim_fields_get.argtypes = [C.c_void_p, F32P]
        L.mref_sim_fields_set.argtypes = [C.c_void_p, F32P]
        L.mref_sim_step.argtypes = [C.c_void_p, C.c_long]
        L.mref_sim_step_and_sort.argtypes = [C.c_void_p, C.c_long]
        L.mref_sim_step_count.argtypes = [C.c_void_p]
        L.mref_sim_step_count.restype = C.c_long
        L.mref_sim_run_csv.argtypes = [C.c_void_p, C.c_char_p, C.c_long]
        L.mref_sim_timings.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        L.mref_sim_diagnostics.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.c_int]

    def _chk(self, rc):
        if rc:
            _raise(rc, self.lib.mref_last_error().decode())

    def load_interpolators(self, g, f16, workers=1):
        out = np.zeros((18, g.padded), np.float32)
        self._chk(self.lib.mref_load_interpolators(C.byref(g), f16, out, workers))
        return out

    def advance_particles(self, g, q, m, p7, ids, i18, scatter, chunk=2048, workers=1, exact_gyration=False,
                          deterministic=False):
        self._chk(self.lib.mref_advance_particles(C.byref(g), q, m, ids.size, p7, ids, i18, scatter.h, chunk, workers,
                                                  int(exact_gyration), int(deterministic)))

    def scatter(self, g, backend=2, workers=1):
        return _Scatter(self, g, backend, workers)

    def ghost_fold(self, g, acc):
        self._chk(self.lib.mref_ghost_fold(C.byref(g), acc))

    def unload(self, g, acc, f16):
        self._chk(self.lib.mref_unload(C.byref(g), acc, f16))

    def clear_currents(self, g, f16):
        self._chk(self.lib.mref_clear_currents(C.byref(g), f16))

    def advance_b(self, g, f16, frac, workers=1):
        self._chk(self.lib.mref_advance_b(C.byref(g), f16, frac, workers))

    def advance_e(self, g, f16, workers=1):
        self._chk(self.lib.mref_advance_e(C.byref(g), f16, workers))

    def ghost_sync(self, g, f16):
        self._chk(self.lib.mref_ghost_sync(C.byref(g), f16))

    def sort(self, p7, ids, interleaved=False):
        self._chk(self.lib.mref_sort(ids.size, p7, ids, int(interleaved)))

    def deposit_rho(self, g, q, p7, ids, f16):
        self._chk(self.lib.mref_deposit_rho(C.byref(g), q, ids.size, p7, ids, f16))

    def compute_div_errors(self, g, f16):
        self._chk(self.lib.mref_compute_div_errors(C.byref(g), f16))

    def field_energy(self, g, f16):
        out = np.zeros(2, np.float32)
        self._chk(self.lib.mref_field_energy(C.byref(g), f16, out))
        return out

    def kinetic_energy_centered(self, g, q, m, p7, ids, i18):
        out = C.c_float()
        self._chk(self.lib.mref_kinetic_energy_centered(C.byref(g), q, m, ids.size, p7, ids, i18, C.byref(out)))
        return out.value

    def max_abs_lane(self, g, f16, lane):
        out = C.c_float()
        self._chk(self.lib.mref_max_abs_lane(C.byref(g), f16, lane, C.byref(out)))
        return out.value

    def deck_roundtrip(self, text: str, override: str | None = None) -> str:
        """serialize_deck(parse_deck(text) [+ apply_override]); raises on
        parse errors with the reference's message."""
        buf = C.create_string_buffer(1 << 16)
        self._chk(self.lib.mref_deck_roundtrip(text.encode(), override.encode() if override else None, buf,
                                               len(buf)))
        return buf.value.decode()

    def sim(self, deck_text: str) -> "RefSim":
        return RefSim(self, deck_text)


class _Scatter:
    def __init__(self, ref, g, backend, workers):
        self.ref, self.g = ref, g
        self.h = ref.lib.mref_scatter_new(C.byref(g), backend, workers)

    def reduce(self):
        out = np.zeros((self.g.padded, 12), np.float32)
        self.ref._chk(self.ref.lib.mref_scatter_reduce(self.h, out))
        return out

    def clear(self):
        self.ref._chk(self.ref.lib.mref_scatter_clear(self.h))

    def __del__(self):
        try:
            self.ref.lib.mref_scatter_free(self.h)
        except Exception:
            pass


class RefSim:
    """minipic::SimState built from deck text (proj/src/sim.cpp)."""

    def __init__(self, ref: Ref, deck_text: str):
        self.ref = ref
        self.h = ref.lib.mref_sim_new(deck_text.encode())
        if not self.h:
            raise OracleError(3, ref.lib.mref_last_error().decode())
        self.grid = Grid()
        ref._chk(ref.lib.mref_sim_grid(self.h, C.byref(self.grid)))

    @property
    def nspecies(self):
        return self.ref.lib.mref_sim_nspecies(self.h)

    def species(self, s):
        n = self.ref.lib.mref_sim_species_size(self.h, s)
        p = np.zeros((7, n), np.float32)
        ids = np.zeros(n, np.int32)
        self.ref._chk(self.ref.lib.mref_sim_species_get(self.h, s, p, ids))
        return p, ids

    def set_species(self, s, p, ids):
        self.ref._chk(self.ref.lib.mref_sim_species_set(self.h, s, np.ascontiguousarray(p, np.float32),
                                                        np.ascontiguousarray(ids, np.int32)))

    def fields(self):
        out = np.zeros((16, self.grid.padded), np.float32)
        self.ref._chk(self.ref.lib.mref_sim_fields_get(self.h, out))
        return out

    def set_fields(self, f16):
        self.ref._chk(self.ref.lib.mref_sim_fields_set(self.h, np.ascontiguousarray(f16, np.float32)))

    def step(self, n=1):
        self.ref._chk(self.ref.lib.mref_sim_step(self.h, n))

    def step_and_sort(self, n=1):
        self.ref._chk(self.ref.lib.mref_sim_step_and_sort(self.h, n))

    @property
    def step_count(self):
        return self.ref.lib.mref_sim_step_count(self.h)

    def diagnostics(self, refresh=False) -> dict:
        """SimState::current_diagnostics (after refresh_charge_diagnostics if
        asked), as floats."""
        out = np.zeros(6 + self.nspecies, np.float64)
        self.ref._chk(self.ref.lib.mref_sim_diagnostics(self.h, int(refresh), out.ctypes.data_as(C.POINTER(C.c_double)),
                                                        out.size))
        return {"e_energy": out[0], "b_energy": out[1], "total_energy": out[2], "max_div_e_err": out[3],
                "max_div_b_err": out[4], "particle_count": int(out[5]), "kinetic": list(out[6:])}

    def run_csv(self, cap=1 << 22) -> str:
        buf = C.create_string_buffer(cap)
        self.ref._chk(self.ref.lib.mref_sim_run_csv(self.h, buf, cap))
        return buf.value.decode()

    def timings(self):
        out = (C.c_double * 4)()
        self.ref._chk(self.ref.lib.mref_sim_timings(self.h, out))
        return list(out)

    def __del__(self):
        try:
            self.ref.lib.mref_sim_free(self.h)
        except Exception:
            pass
