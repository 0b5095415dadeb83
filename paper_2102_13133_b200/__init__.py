"""paper_2102_13133_b200 — B200-native (sm_100a CUDA) particle-in-cell step.

A from-scratch re-implementation of the hot path of arXiv 2102.13133 (VPIC
2.0; reference implementation "minipic", /root/reference/proj) behind the C-ABI
declared in ``include/pic_b200.h``.  This module is a thin ctypes binding over
``libpic_b200.so``: every call goes to hand-written sm_100a kernels; there is
no CPU fallback.  Importing on a machine without the built library raises.

Array conventions are the reference's field-major ones (see pic_b200.h):
fields ``(16, V)``, interpolators ``(18, V)``, particles ``(7, n)`` float32 +
``(n,)`` int32 ids, accumulator ``(V, 12)``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PIC_LIB_PATH") or os.path.join(HERE, "libpic_b200.so")  # override: A/B builds

PIC_EXACT_GYRATION = 0x1
PIC_DETERMINISTIC = 0x2
SORT_BLOCKED = 0
SORT_INTERLEAVED = 1

# field lanes (proj/include/minipic/lanes.hpp:23-43)
FIELD_LANES = ["ex", "ey", "ez", "div_e_err", "cbx", "cby", "cbz", "div_b_err",
               "jfx", "jfy", "jfz", "rhof", "tcax", "tcay", "tcaz", "rhob"]
F = {name: i for i, name in enumerate(FIELD_LANES)}

# halo plane kinds (pic_b200.h)
HALO_ACCUMULATOR = 0
HALO_FIELDS = 1
HALO_RHO = 2


class PicError(RuntimeError):
    code = 5


class UsageError(PicError):
    """minipic::usage_error (proj/include/minipic/types.hpp:27-30)."""
    code = 1


class RunAbort(PicError):
    """minipic::run_abort (proj/include/minipic/types.hpp:33-36)."""
    code = 2


class DeckParseError(PicError):
    """minipic::deck_parse_error (proj/include/minipic/sim.hpp:66-69)."""
    code = 3


class CudaError(PicError):
    code = 4


_ERRS = {1: UsageError, 2: RunAbort, 3: DeckParseError, 4: CudaError}


class Grid(C.Structure):
    """pic_grid == GridDescriptor (proj/include/minipic/grid.hpp:15-38), fp32."""

    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("hx", C.c_float), ("hy", C.c_float), ("hz", C.c_float), ("dt", C.c_float)]

    @property
    def padded(self) -> int:
        return (self.nx + 2) * (self.ny + 2) * (self.nz + 2)

    @property
    def interior(self) -> int:
        return self.nx * self.ny * self.nz

    def voxel(self, ix, iy, iz):
        return ix + (self.nx + 2) * (iy + (self.ny + 2) * iz)

    def __repr__(self):
        return (f"Grid(nx={self.nx}, ny={self.ny}, nz={self.nz}, hx={self.hx}, hy={self.hy}, "
                f"hz={self.hz}, dt={self.dt})")


class Diag(C.Structure):
    """pic_diag == DiagnosticsRecord (proj/include/minipic/sim.hpp:88-100) minus wall clock."""

    _fields_ = [("e_energy", C.c_float), ("b_energy", C.c_float), ("total_energy", C.c_float),
                ("max_div_e_err", C.c_float), ("max_div_b_err", C.c_float), ("particle_count", C.c_uint64)]


_lib = None


class Laser(C.Structure):
    """pic_laser (include/pic_b200.h)."""

    _fields_ = [("ix", C.c_int), ("pol", C.c_int), ("e0", C.c_float), ("omega", C.c_float),
                ("ramp_steps", C.c_float), ("y0", C.c_float), ("z0", C.c_float), ("waist", C.c_float)]


PBC_PERIODIC, PBC_ABSORB, PBC_REFLECT = 0, 1, 2
STAGE_FOLD, STAGE_AFTER_B, STAGE_BEFORE_E, STAGE_AFTER_E, STAGE_EMIT = 0, 1, 2, 3, 4
FBC_PERIODIC, FBC_PEC, FBC_MUR = 0, 1, 2


class Sheet(C.Structure):
    """pic_sheet (include/pic_b200.h)."""

    _fields_ = [("z1", C.c_float), ("z2", C.c_float), ("half_width", C.c_float),
                ("background", C.c_float), ("amplitude", C.c_float), ("flip_drift", C.c_int)]


def lib() -> C.CDLL:
    """Loads libpic_b200.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    F32 = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
    I32 = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
    G = C.POINTER(Grid)
    L.pic_last_error.restype = C.c_char_p
    sigs = {
        "pic_context_create": [C.c_int, G, C.POINTER(P)],
        "pic_context_destroy": [P],
        "pic_context_grid": [P, G],
        "pic_synchronize": [P],
        "pic_host_register": [P, C.c_size_t],
        "pic_host_unregister": [P],
        "pic_species_create": [P, C.c_char_p, C.c_float, C.c_float, C.c_size_t, C.POINTER(C.c_int)],
        "pic_species_count": [P, C.c_int, C.POINTER(C.c_size_t)],
        "pic_species_upload": [P, C.c_int, C.c_size_t, F32, I32],
        "pic_species_download": [P, C.c_int, F32, I32],
        "pic_species_upload_records": [P, C.c_int, C.c_size_t, P, P],
        "pic_species_download_records": [P, C.c_int, P, P],
        "pic_species_load_synthetic": [P, C.c_int, C.c_int, C.c_float, F32, C.c_uint64],
        "pic_species_load_harris": [P, C.c_int, C.c_int, C.c_float, F32, C.c_uint64, C.POINTER(Sheet)],
        "pic_species_load_slab": [P, C.c_int, C.c_int, C.c_float, F32, C.c_uint64, C.c_int, C.c_int],
        "pic_set_x_boundary": [P, C.c_int, C.c_int, C.c_int],
        "pic_set_boundary": [P, C.c_int, C.c_int, C.c_int],
        "pic_wall_stage": [P, C.c_int, C.c_float],
        "pic_absorbed_counts": [P, C.POINTER(C.c_uint64), C.c_int],
        "pic_set_laser": [P, C.POINTER(Laser)],
        "pic_set_emitter": [P, C.c_int, C.c_int, C.c_int, C.c_float, F32, C.c_uint64],
        "pic_fields_upload": [P, F32],
        "pic_fields_download": [P, F32],
        "pic_interpolators_download": [P, F32],
        "pic_interpolators_upload": [P, F32],
        "pic_accumulator_download": [P, F32],
        "pic_accumulator_upload": [P, F32],
        "pic_clear_accumulator": [P],
        "pic_clear_currents": [P],
        "pic_load_interpolators": [P],
        "pic_advance_p": [P, C.c_int, C.c_uint],
        "pic_ghost_fold_currents": [P],
        "pic_unload_currents": [P],
        "pic_advance_b": [P, C.c_float],
        "pic_advance_e": [P],
        "pic_unload_advance_e": [P],
        "pic_ghost_sync_fields": [P],
        "pic_sort_particles": [P, C.c_int, C.c_int],
        "pic_step": [P, C.c_uint],
        "pic_prepare_step_graphs": [P, C.c_uint, C.c_int, C.c_int, C.c_longlong, C.POINTER(C.c_int)],
        "pic_step_host": [P, C.c_uint, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)],
        "pic_event_record": [P, C.c_int],
        "pic_event_elapsed_ms": [P, C.c_int, C.c_int, C.POINTER(C.c_float)],
        "pic_launch_count": [P, C.POINTER(C.c_uint64)],
        "pic_phase_timing": [P, C.c_int],
        "pic_phase_timings": [P, C.POINTER(C.c_double), C.c_int],
        "pic_clear_rho": [P],
        "pic_deposit_rho": [P, C.c_int],
        "pic_compute_div_errors": [P],
        "pic_refresh_charge_diagnostics": [P],
        "pic_field_energy": [P, C.POINTER(C.c_float)],
        "pic_max_abs_lane": [P, C.c_int, C.POINTER(C.c_float)],
        "pic_kinetic_energy": [P, C.c_int, C.c_int, C.POINTER(C.c_float)],
        "pic_diagnostics": [P, C.POINTER(Diag), C.POINTER(C.c_float), C.c_size_t],
        "pic_diagnostics_order": [P, C.c_int],
        "pic_set_x_open": [P, C.c_int, C.c_int],
        "pic_set_stream": [P, P],
        "pic_halo_plane_bytes": [P, C.c_int, C.POINTER(C.c_size_t)],
        "pic_halo_pack": [P, C.c_int, C.c_int, P, C.c_int],
        "pic_halo_unpack": [P, C.c_int, C.c_int, P, C.c_int],
        "pic_migrate_counts": [P, C.c_int, C.POINTER(C.c_size_t)],
        "pic_migrate_pack": [P, C.c_int, P, P],
        "pic_migrate_append": [P, C.c_int, P, C.c_size_t],
        "pic_deck_parse": [C.c_char_p, C.POINTER(P)],
        "pic_deck_destroy": [P],
        "pic_deck_override": [P, C.c_char_p],
        "pic_deck_serialize": [P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)],
        "pic_deck_grid": [P, G],
        "pic_deck_steps": [P, C.POINTER(C.c_long)],
        "pic_sim_create": [C.c_int, P, C.POINTER(P)],
        "pic_sim_destroy": [P],
        "pic_sim_context": [P, C.POINTER(P)],
        "pic_sim_step": [P],
        "pic_sim_step_count": [P, C.POINTER(C.c_long)],
        "pic_sim_refresh_charge_diagnostics": [P],
        "pic_sim_emit_diagnostics": [P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)],
        "pic_sim_run": [P, C.c_char_p],
        "pic_sim_dump_fields": [P, C.c_char_p],
        "pic_sim_warnings": [P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)],
    }
    for name, argtypes in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = argtypes
        fn.restype = C.c_int
    _lib = L
    return L


def check(rc: int):
    if rc:
        msg = lib().pic_last_error().decode()
        raise _ERRS.get(rc, PicError)(msg)


def make_grid(n, h=1.0, dt=None, cfl_frac=0.5) -> Grid:
    """Grid with dt = cfl_frac * cfl_limit (computed in fp32) unless given."""
    nx, ny, nz = (n, n, n) if np.isscalar(n) else n
    hx, hy, hz = (h, h, h) if np.isscalar(h) else h
    if dt is None:
        f32 = np.float32
        s = f32(1) / (f32(hx) * f32(hx)) + f32(1) / (f32(hy) * f32(hy)) + f32(1) / (f32(hz) * f32(hz))
        dt = f32(cfl_frac) * (f32(1) / np.sqrt(s, dtype=np.float32))
    return Grid(int(nx), int(ny), int(nz), float(hx), float(hy), float(hz), float(np.float32(dt)))


class Context:
    """Device-resident PIC state on one GPU (pic_context)."""

    def __init__(self, grid: Grid, device: int = 0):
        self.grid = grid
        self._h = C.c_void_p()
        self._borrowed = False
        check(lib().pic_context_create(device, C.byref(grid), C.byref(self._h)))
        self.species_names = []

    @classmethod
    def _borrow(cls, handle: C.c_void_p, grid: Grid, species_names):
        """A view of a context owned elsewhere (a SimState's)."""
        ctx = cls.__new__(cls)
        ctx.grid, ctx._h, ctx._borrowed, ctx.species_names = grid, handle, True, list(species_names)
        return ctx

    def close(self):
        if self._h and not self._borrowed:
            check(lib().pic_context_destroy(self._h))
        self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def V(self) -> int:
        return self.grid.padded

    # --- species -----------------------------------------------------------
    def add_species(self, name: str, q: float, m: float, capacity: int) -> int:
        sid = C.c_int()
        check(lib().pic_species_create(self._h, name.encode(), q, m, capacity, C.byref(sid)))
        self.species_names.append(name)
        return sid.value

    def species_count(self, sid: int) -> int:
        n = C.c_size_t()
        check(lib().pic_species_count(self._h, sid, C.byref(n)))
        return n.value

    def upload_species(self, sid: int, lanes7: np.ndarray, ids: np.ndarray):
        lanes7 = np.ascontiguousarray(lanes7, np.float32)
        ids = np.ascontiguousarray(ids, np.int32)
        assert lanes7.shape == (7, ids.size)
        check(lib().pic_species_upload(self._h, sid, ids.size, lanes7, ids))

    def download_species(self, sid: int):
        n = self.species_count(sid)
        p = np.zeros((7, n), np.float32)
        ids = np.zeros(n, np.int32)
        check(lib().pic_species_download(self._h, sid, p, ids))
        return p, ids

    @staticmethod
    def _addr(a):
        """Address of a numpy array or a (host or CUDA) torch tensor."""
        return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data

    def upload_records(self, sid: int, pos16, mom16, n: int):
        """Native 32-byte records: pos/mom float32 arrays of shape (>= n, 4),
        numpy or torch (host or CUDA: device copies stay on the GPU)."""
        for a in (pos16, mom16):
            assert str(a.dtype).endswith("float32") and a.shape[0] >= n and a.shape[1] == 4
        check(lib().pic_species_upload_records(self._h, sid, n, self._addr(pos16), self._addr(mom16)))

    def download_records(self, sid: int, pos16, mom16) -> int:
        n = self.species_count(sid)
        for a in (pos16, mom16):
            assert str(a.dtype).endswith("float32") and a.shape[0] >= n and a.shape[1] == 4
        check(lib().pic_species_download_records(self._h, sid, self._addr(pos16), self._addr(mom16)))
        return n

    def load_synthetic(self, sid: int, ppc: int, u_th: float, drift=(0.0, 0.0, 0.0), seed: int = 1):
        check(lib().pic_species_load_synthetic(self._h, sid, ppc, u_th, np.asarray(drift, np.float32), seed))

    def load_harris(self, sid: int, ppc: int, u_th: float, drift=(0.0, 0.0, 0.0), seed: int = 1, *,
                    z1: float, z2: float, half_width: float, background: float = 0.0,
                    amplitude: float = 1.0, flip_drift: bool = True):
        """Synthetic load with double-Harris-sheet weights (pic_species_load_harris)."""
        sh = Sheet(z1, z2, half_width, background, amplitude, int(flip_drift))
        check(lib().pic_species_load_harris(self._h, sid, ppc, u_th, np.asarray(drift, np.float32), seed,
                                            C.byref(sh)))

    def load_slab(self, sid: int, ppc: int, u_th: float, drift=(0.0, 0.0, 0.0), seed: int = 1, *,
                  ix_lo: int, ix_hi: int):
        """Synthetic load of the cells with x index in [ix_lo, ix_hi] (pic_species_load_slab)."""
        check(lib().pic_species_load_slab(self._h, sid, ppc, u_th, np.asarray(drift, np.float32), seed,
                                          ix_lo, ix_hi))

    # --- non-periodic x boundaries, laser, emitter (pic_set_x_boundary ...) ---
    def set_x_boundary(self, side: int, particle_bc: int, field_bc: int):
        check(lib().pic_set_x_boundary(self._h, side, particle_bc, field_bc))

    def set_boundary(self, face: int, particle_bc: int, field_bc: int):
        """face 0-5: x low, x high, y low, y high, z low, z high (pic_set_boundary)."""
        check(lib().pic_set_boundary(self._h, face, particle_bc, field_bc))

    def wall_stage(self, stage: int, frac: float = 0.0):
        """pic_wall_stage: STAGE_FOLD / AFTER_B / BEFORE_E / AFTER_E / EMIT."""
        check(lib().pic_wall_stage(self._h, stage, frac))

    def absorbed_counts(self, reset: bool = False):
        out = (C.c_uint64 * 2)()
        check(lib().pic_absorbed_counts(self._h, out, int(reset)))
        return int(out[0]), int(out[1])

    def set_laser(self, ix: int, e0: float, omega: float, pol: int = 1, ramp_steps: float = 0.0,
                  y0: float = 0.0, z0: float = 0.0, waist: float = 0.0):
        check(lib().pic_set_laser(self._h, C.byref(Laser(ix, pol, e0, omega, ramp_steps, y0, z0, waist))))

    def set_emitter(self, sid: int, side: int, per_cell: int, u_th: float, drift=(0.0, 0.0, 0.0), seed: int = 1):
        check(lib().pic_set_emitter(self._h, sid, side, per_cell, u_th, np.asarray(drift, np.float32), seed))

    # --- fields ------------------------------------------------------------
    def upload_fields(self, f16: np.ndarray):
        f16 = np.ascontiguousarray(f16, np.float32)
        assert f16.shape == (16, self.V)
        check(lib().pic_fields_upload(self._h, f16))

    def download_fields(self) -> np.ndarray:
        out = np.zeros((16, self.V), np.float32)
        check(lib().pic_fields_download(self._h, out))
        return out

    def download_interpolators(self) -> np.ndarray:
        out = np.zeros((18, self.V), np.float32)
        check(lib().pic_interpolators_download(self._h, out))
        return out

    def upload_interpolators(self, i18: np.ndarray):
        check(lib().pic_interpolators_upload(self._h, np.ascontiguousarray(i18, np.float32)))

    def download_accumulator(self) -> np.ndarray:
        out = np.zeros((self.V, 12), np.float32)
        check(lib().pic_accumulator_download(self._h, out))
        return out

    def upload_accumulator(self, acc: np.ndarray):
        check(lib().pic_accumulator_upload(self._h, np.ascontiguousarray(acc, np.float32)))

    # --- hot path ------------------------------------------------------------
    def clear_accumulator(self):
        check(lib().pic_clear_accumulator(self._h))

    def clear_currents(self):
        check(lib().pic_clear_currents(self._h))

    def load_interpolators(self):
        check(lib().pic_load_interpolators(self._h))

    def advance_p(self, sid: int, exact_gyration=False, deterministic=False):
        flags = (PIC_EXACT_GYRATION if exact_gyration else 0) | (PIC_DETERMINISTIC if deterministic else 0)
        check(lib().pic_advance_p(self._h, sid, flags))

    def ghost_fold_currents(self):
        check(lib().pic_ghost_fold_currents(self._h))

    def unload_currents(self):
        check(lib().pic_unload_currents(self._h))

    def advance_b(self, frac: float):
        check(lib().pic_advance_b(self._h, frac))

    def advance_e(self):
        check(lib().pic_advance_e(self._h))

    def unload_advance_e(self):
        check(lib().pic_unload_advance_e(self._h))

    def ghost_sync_fields(self):
        check(lib().pic_ghost_sync_fields(self._h))

    def sort_particles(self, sid: int, order: int = SORT_BLOCKED):
        check(lib().pic_sort_particles(self._h, sid, order))

    def step(self, exact_gyration=False, deterministic=False):
        flags = (PIC_EXACT_GYRATION if exact_gyration else 0) | (PIC_DETERMINISTIC if deterministic else 0)
        check(lib().pic_step(self._h, flags))

    def prepare_graphs(self, steps, sort_interval=0, steps_taken=0, exact_gyration=False):
        """Capture (without running) the CUDA graphs of the next `steps` fast
        steps, a blocked sort of every species following each step whose
        count (steps_taken + k) is a multiple of sort_interval.  Returns the
        number of graphs captured (0 unless every store is voxel-ordered)."""
        out = C.c_int(0)
        check(lib().pic_prepare_step_graphs(self._h, PIC_EXACT_GYRATION if exact_gyration else 0, int(steps),
                                            int(sort_interval), int(steps_taken), C.byref(out)))
        return out.value

    def step_host(self, lanes7_list, ids_list, exact_gyration=False, deterministic=False):
        """SimState::step with host-resident species buffers (copied in and out)."""
        flags = (PIC_EXACT_GYRATION if exact_gyration else 0) | (PIC_DETERMINISTIC if deterministic else 0)
        k = len(lanes7_list)
        ns = len(self.species_names)
        if k != ns or len(ids_list) != ns:
            raise UsageError(f"step_host: {k} lane arrays / {len(ids_list)} id arrays for {ns} species")
        for s, (a, i) in enumerate(zip(lanes7_list, ids_list)):
            n = self.species_count(s)
            if not (isinstance(a, np.ndarray) and a.dtype == np.float32 and a.flags.c_contiguous
                    and a.shape == (7, n)):
                raise UsageError(f"step_host: species {s} lanes must be C-contiguous float32 (7, {n})")
            if not (isinstance(i, np.ndarray) and i.dtype == np.int32 and i.flags.c_contiguous and i.shape == (n,)):
                raise UsageError(f"step_host: species {s} ids must be C-contiguous int32 ({n},)")
        lp = (C.c_void_p * k)(*[a.ctypes.data for a in lanes7_list])
        ip = (C.c_void_p * k)(*[a.ctypes.data for a in ids_list])
        check(lib().pic_step_host(self._h, flags, lp, ip))

    def synchronize(self):
        check(lib().pic_synchronize(self._h))

    # --- domain decomposition in x (device pointers) ------------------
    def set_x_open(self, x_open: bool = True, low_wraps: bool = False):
        check(lib().pic_set_x_open(self._h, int(x_open), int(low_wraps)))

    def set_stream(self, cuda_stream_ptr):
        """Run on a caller's cudaStream_t (an int handle, e.g.
        torch.cuda.current_stream().cuda_stream); None restores our own."""
        check(lib().pic_set_stream(self._h, C.c_void_p(cuda_stream_ptr) if cuda_stream_ptr else None))

    def halo_plane_bytes(self, kind: int) -> int:
        n = C.c_size_t()
        check(lib().pic_halo_plane_bytes(self._h, kind, C.byref(n)))
        return n.value

    def halo_pack(self, kind: int, ix: int, dst_ptr: int, zero_after: bool = False):
        check(lib().pic_halo_pack(self._h, kind, ix, C.c_void_p(dst_ptr), int(zero_after)))

    def halo_unpack(self, kind: int, ix: int, src_ptr: int, accumulate: bool = False):
        check(lib().pic_halo_unpack(self._h, kind, ix, C.c_void_p(src_ptr), int(accumulate)))

    def migrate_counts(self, sid: int):
        out = (C.c_size_t * 2)()
        check(lib().pic_migrate_counts(self._h, sid, out))
        return int(out[0]), int(out[1])

    def migrate_pack(self, sid: int, low_ptr: int, high_ptr: int):
        check(lib().pic_migrate_pack(self._h, sid, C.c_void_p(low_ptr), C.c_void_p(high_ptr)))

    def migrate_append(self, sid: int, src_ptr: int, count: int):
        check(lib().pic_migrate_append(self._h, sid, C.c_void_p(src_ptr), count))

    # --- diagnostics (proj/src/sim.cpp:230-266) ---------------------------------
    def clear_rho(self):
        check(lib().pic_clear_rho(self._h))

    def deposit_rho(self, sid: int):
        check(lib().pic_deposit_rho(self._h, sid))

    def compute_div_errors(self):
        check(lib().pic_compute_div_errors(self._h))

    def refresh_charge_diagnostics(self):
        check(lib().pic_refresh_charge_diagnostics(self._h))

    def field_energy(self):
        out = (C.c_float * 2)()
        check(lib().pic_field_energy(self._h, out))
        return float(out[0]), float(out[1])

    def max_abs_lane(self, lane: int) -> float:
        out = C.c_float()
        check(lib().pic_max_abs_lane(self._h, lane, C.byref(out)))
        return out.value

    def kinetic_energy(self, sid: int, centered: bool = True) -> float:
        out = C.c_float()
        check(lib().pic_kinetic_energy(self._h, sid, int(centered), C.byref(out)))
        return out.value

    def diagnostics_order(self, reference_order: bool):
        """Energies summed in the reference's fp32 order (bit-identical in
        deterministic mode) or as fp64 device sums (default)."""
        check(lib().pic_diagnostics_order(self._h, int(reference_order)))

    def diagnostics(self) -> dict:
        """SimState::current_diagnostics (sim.cpp:236-266) on the device."""
        d = Diag()
        k = max(1, len(self.species_names))
        kin = (C.c_float * k)()
        check(lib().pic_diagnostics(self._h, C.byref(d), kin, k))
        return {"e_energy": d.e_energy, "b_energy": d.b_energy,
                "kinetic": [kin[i] for i in range(len(self.species_names))],
                "total_energy": d.total_energy, "max_div_e_err": d.max_div_e_err,
                "max_div_b_err": d.max_div_b_err, "particle_count": int(d.particle_count)}

    # --- timing ----------------------------------------------------------------
    def event(self, slot: int):
        check(lib().pic_event_record(self._h, slot))

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_float()
        check(lib().pic_event_elapsed_ms(self._h, a, b, C.byref(ms)))
        return ms.value

    def phase_timing(self, enable: bool = True):
        check(lib().pic_phase_timing(self._h, int(enable)))

    def phase_timings(self, reset: bool = False) -> dict:
        """Cumulative device ms per phase (PhaseTimings, sim.hpp:129-136)."""
        out = (C.c_double * 5)()
        check(lib().pic_phase_timings(self._h, out, int(reset)))
        return dict(zip(("interpolate", "push", "scatter", "field", "sort"), list(out)))

    def _set_push_variant(self, variant: int):
        """Benchmarking hook (not in the public C header): advance_p strategy."""
        fn = lib().pic_internal_set_push_variant
        fn.argtypes = [C.c_void_p, C.c_int]
        check(fn(self._h, variant))

    def _set_voxel_order(self, on: bool):
        """A/B hook (not in the public C header): continuous voxel order of the
        fast push (default on); off returns every species to logical order."""
        fn = lib().pic_internal_set_voxel_order
        fn.argtypes = [C.c_void_p, C.c_int]
        check(fn(self._h, int(on)))

    def _set_reorder_interval(self, m: int):
        """Tuning hook (not in the public C header): every m-th ordered push
        reorders the store."""
        fn = lib().pic_internal_set_reorder_interval
        fn.argtypes = [C.c_void_p, C.c_int]
        check(fn(self._h, m))

    def _species_ordered(self, sid: int) -> bool:
        """Test hook: whether the species is held in continuous voxel order."""
        fn = lib().pic_internal_species_ordered
        out = C.c_int()
        check(fn(self._h, sid, C.byref(out)))
        return bool(out.value)

    def _download_physical(self, sid: int):
        """Test hook: (pos, mom) float32 (n, 4) records as they lie in memory
        and, in continuous voxel order, their logical indices."""
        n = self.species_count(sid)
        pos = np.zeros((n, 4), np.float32)
        mom = np.zeros((n, 4), np.float32)
        lidx = np.zeros(n, np.uint32)
        fn = lib().pic_internal_download_physical
        fn.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        check(fn(self._h, sid, pos.ctypes.data, mom.ctypes.data, lidx.ctypes.data))
        return pos, mom, lidx

    def _push_kernel_ms(self, reset: bool = False):
        """(cumulative device ms, launches) of the push kernels alone while
        phase timing is on (events on each launch's own stream)."""
        fn = lib().pic_internal_push_kernel_ms
        fn.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.c_int]
        ms, n = C.c_double(), C.c_uint64()
        check(fn(self._h, C.byref(ms), C.byref(n), int(reset)))
        return ms.value, n.value

    def _batched_launches(self) -> int:
        """advance_p launches that pushed several species at once (host
        count of captured and plain steps)."""
        fn = lib().pic_internal_batched_launches
        out = C.c_uint64()
        fn.argtypes = [C.c_void_p, C.c_void_p]
        check(fn(self._h, C.byref(out)))
        return out.value

    def _graph_stats(self):
        """(captures, replays, plain steps) of pic_step's CUDA graphs."""
        fn = lib().pic_internal_graph_stats
        out = (C.c_uint64 * 3)()
        fn.argtypes = [C.c_void_p, C.c_void_p]
        check(fn(self._h, out))
        return tuple(out)

    def _set_graphs(self, on: bool):
        """Benchmarking hook (not in the public C header): pic_step as CUDA graphs."""
        fn = lib().pic_internal_set_graphs
        fn.argtypes = [C.c_void_p, C.c_int]
        check(fn(self._h, int(on)))

    def _set_sort_variant(self, variant: int):
        """Benchmarking hook (not in the public C header): sort strategy."""
        fn = lib().pic_internal_set_sort_variant
        fn.argtypes = [C.c_void_p, C.c_int]
        check(fn(self._h, variant))

    def _set_host_chunk(self, particles: int):
        """Testing hook (not in the public C header): pic_step_host chunk size."""
        fn = lib().pic_internal_set_host_chunk
        fn.argtypes = [C.c_void_p, C.c_size_t]
        check(fn(self._h, particles))

    def launch_count(self) -> int:
        n = C.c_uint64()
        check(lib().pic_launch_count(self._h, C.byref(n)))
        return n.value


def host_register(arr: np.ndarray):
    check(lib().pic_host_register(arr.ctypes.data, arr.nbytes))


def host_unregister(arr: np.ndarray):
    check(lib().pic_host_unregister(arr.ctypes.data))


# --- the decomposed fast step in C++ over NCCL (pic_dd) ----------------
def dd_unique_id() -> bytes:
    """ncclGetUniqueId (rank 0; broadcast it to the other ranks)."""
    import torch  # noqa: F401  (loads the process's NCCL; the library binds to it)
    buf = C.create_string_buffer(128)
    fn = lib().pic_dd_unique_id
    fn.argtypes = [C.c_void_p]
    check(fn(buf))
    return buf.raw


class DecomposedStep:
    """pic_dd: SimState::step over this rank's x-open slab with the x
    exchanges (migration, accumulator halo-add, E/B halo) as NCCL send /
    receive inside the library, no host synchronisation, graph-captured."""

    def __init__(self, ctx: "Context", rank: int, world: int, unique_id: bytes, mig_frac: float = 0.0):
        import torch  # noqa: F401  (loads the process's NCCL; the library binds to it)
        self.ctx = ctx
        self._h = C.c_void_p()
        fn = lib().pic_dd_create
        fn.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_char_p, C.c_double, C.POINTER(C.c_void_p)]
        check(fn(ctx._h, rank, world, unique_id, mig_frac, C.byref(self._h)))

    def step(self, exact_gyration: bool = False):
        fn = lib().pic_dd_step
        fn.argtypes = [C.c_void_p, C.c_uint]
        check(fn(self._h, PIC_EXACT_GYRATION if exact_gyration else 0))

    def prepare_graphs(self, steps, sort_interval=0, steps_taken=0, exact_gyration=False):
        """pic_dd_prepare_graphs: capture the next `steps` decomposed steps'
        graphs ahead (same call on every rank); returns graphs captured."""
        fn = lib().pic_dd_prepare_graphs
        fn.argtypes = [C.c_void_p, C.c_uint, C.c_int, C.c_int, C.c_longlong, C.POINTER(C.c_int)]
        out = C.c_int(0)
        check(fn(self._h, PIC_EXACT_GYRATION if exact_gyration else 0, int(steps), int(sort_interval),
                 int(steps_taken), C.byref(out)))
        return out.value

    def close(self):
        if self._h:
            fn = lib().pic_dd_destroy
            fn.argtypes = [C.c_void_p]
            check(fn(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
