"""The reference's run surface (minipic Deck + SimState) over the C-ABI.

Mirrors proj/include/minipic/sim.hpp:23-200: ``parse_deck`` /
``Deck.serialize`` / ``Deck.override`` (proj/src/deck.cpp) and
``SimState.initialize`` / ``step`` / ``run`` / ``emit_diagnostics``
(proj/src/sim.cpp), executed by the C++ host in csrc/sim.cu on the sm_100a
kernels.  Deck errors raise ``DeckParseError`` with the reference's message.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import Context, Grid, check, lib


class HookFlags(C.Structure):
    """HookFlags (proj/include/minipic/sim.hpp:102-110)."""
    _fields_ = [("particles_to_host", C.c_int), ("fields_to_host", C.c_int), ("particles_back", C.c_int),
                ("fields_back", C.c_int)]

    @classmethod
    def legacy(cls):
        return cls(1, 1, 1, 1)

    @classmethod
    def none(cls):
        return cls(0, 0, 0, 0)


class _HookView(C.Structure):
    _fields_ = [("sim", C.c_void_p), ("step", C.c_long), ("fields16", C.POINTER(C.c_float)),
                ("nspecies", C.c_size_t), ("lanes7", C.POINTER(C.POINTER(C.c_float))),
                ("ids", C.POINTER(C.POINTER(C.c_int32))), ("counts", C.POINTER(C.c_size_t))]


_HOOK_FN = C.CFUNCTYPE(C.c_int, C.POINTER(_HookView), C.c_void_p)


class HookContext:
    """HookContext (sim.hpp:113-119): the step and the host mirrors as numpy
    views (fields (16, V), per species lanes (7, n) and ids (n,)); writes go
    back to the device when the hook's flags say so."""

    def __init__(self, sim, v, padded):
        self.state = sim
        self.step = v.step
        self.host_fields = np.ctypeslib.as_array(v.fields16, shape=(16, padded))
        self.host_particles = []
        for i in range(v.nspecies):
            n = v.counts[i]
            lanes = np.ctypeslib.as_array(v.lanes7[i], shape=(7, n)) if n else np.zeros((7, 0), np.float32)
            ids = np.ctypeslib.as_array(v.ids[i], shape=(n,)) if n else np.zeros(0, np.int32)
            self.host_particles.append((lanes, ids))


class Deck:
    """pic_deck: a parsed, validated deck."""

    def __init__(self, text: str):
        self._h = C.c_void_p()
        check(lib().pic_deck_parse(text.encode(), C.byref(self._h)))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().pic_deck_destroy(self._h)
            self._h = None

    def override(self, key_eq_value: str) -> "Deck":
        check(lib().pic_deck_override(self._h, key_eq_value.encode()))
        return self

    def serialize(self) -> str:
        n = C.c_size_t()
        check(lib().pic_deck_serialize(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(lib().pic_deck_serialize(self._h, buf, len(buf), C.byref(n)))
        return buf.value.decode()

    def grid(self) -> Grid:
        g = Grid()
        check(lib().pic_deck_grid(self._h, C.byref(g)))
        return g

    @property
    def steps(self) -> int:
        n = C.c_long()
        check(lib().pic_deck_steps(self._h, C.byref(n)))
        return n.value


def parse_deck(text: str) -> Deck:
    return Deck(text)


def _text(fn, *args) -> str:
    n = C.c_size_t()
    check(fn(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(fn(*args, buf, len(buf), C.byref(n)))
    return buf.value.decode()


class SimState:
    """pic_sim: SimState on one GPU."""

    def __init__(self, deck: Deck, device: int = 0):
        self._h = C.c_void_p()
        self.deck = deck
        check(lib().pic_sim_create(device, deck._h, C.byref(self._h)))
        ch = C.c_void_p()
        check(lib().pic_sim_context(self._h, C.byref(ch)))
        names = [line.split(".", 1)[1].strip("[] ") for line in deck.serialize().splitlines()
                 if line.startswith("[species.")]
        self.context = Context._borrow(ch, deck.grid(), names)

    @classmethod
    def initialize(cls, deck: Deck, device: int = 0) -> "SimState":
        return cls(deck, device)

    def close(self):
        if self._h:
            check(lib().pic_sim_destroy(self._h))
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

    def step(self):
        """SimState::step + sort_due_species."""
        check(lib().pic_sim_step(self._h))

    def register_hook(self, action, interval=1, flags=None, name="hook"):
        """SimState::register_hook (sim.cpp:185-188): action(HookContext) runs
        in run() every interval steps; an exception in it aborts the run."""
        padded = self.deck.grid().padded
        errors = []

        def trampoline(view, user):
            try:
                if action is not None:
                    action(HookContext(self, view.contents, padded))
                return 0
            except Exception as e:  # reported by the C side as run_abort
                errors.append(e)
                return 1

        cb = _HOOK_FN(trampoline)
        if not hasattr(self, "_hooks"):
            self._hooks = []
        self._hooks.append((cb, errors))
        fn = lib().pic_sim_register_hook
        fn.argtypes = [C.c_void_p, C.c_char_p, C.c_long, C.POINTER(HookFlags), _HOOK_FN, C.c_void_p]
        check(fn(self._h, name.encode(), int(interval), C.byref(flags) if flags is not None else None, cb, None))

    def copies_performed(self) -> int:
        """SimState::copies_performed (sim.hpp:175)."""
        out = C.c_uint64()
        fn = lib().pic_sim_copies_performed
        fn.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
        check(fn(self._h, C.byref(out)))
        return out.value

    @property
    def step_count(self) -> int:
        n = C.c_long()
        check(lib().pic_sim_step_count(self._h, C.byref(n)))
        return n.value

    def refresh_charge_diagnostics(self):
        check(lib().pic_sim_refresh_charge_diagnostics(self._h))

    def emit_diagnostics(self) -> str:
        return _text(lib().pic_sim_emit_diagnostics, self._h)

    def run(self, csv_path: str | None = None):
        check(lib().pic_sim_run(self._h, csv_path.encode() if csv_path else None))

    def dump_fields(self, path: str):
        check(lib().pic_sim_dump_fields(self._h, path.encode()))

    @property
    def warnings(self):
        return [w for w in _text(lib().pic_sim_warnings, self._h).splitlines() if w]
