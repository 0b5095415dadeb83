"""The reference's run surface (minipic Deck + SimState) over the C-ABI.

Mirrors proj/include/minipic/sim.hpp:23-200: ``parse_deck`` /
``Deck.serialize`` / ``Deck.override`` (proj/src/deck.cpp) and
``SimState.initialize`` / ``step`` / ``run`` / ``emit_diagnostics``
(proj/src/sim.cpp), executed by the C++ host in csrc/sim.cu on the sm_100a
kernels.  Deck errors raise ``DeckParseError`` with the reference's message.
"""
from __future__ import annotations

import ctypes as C

from . import Context, Grid, check, lib


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
