"""bench.py's contract on the CPU side: the JSON line is the only thing on
stdout, decks the reference cannot express report the reference arm as
unavailable, and the configs describe the workloads DESIGN.md names."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout  # exactly one JSON line on stdout
    return json.loads(lines[0])


def test_reference_arm_unavailable_for_api_decks():
    for cfg in ("harris", "lpi"):
        d = _run("--impl", "reference", "--config", cfg)
        assert d["impl"] == "reference" and "unavailable" in d


def test_reference_arm_runs_the_compiled_reference():
    from oracle.bindings import ref_available
    if not ref_available():
        import pytest
        pytest.skip("oracle/_ref not built")
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "1", "--cpu-sample-n", "12")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_configs():
    sys.path.insert(0, ROOT)
    import bench
    ts = bench.CONFIGS["two_stream"]
    assert ts["n"] == 256 and sum(s[3] for s in ts["species"]) == 64
    assert 256 ** 3 * 64 == 1073741824
    h = bench.CONFIGS["harris"]["deck"]
    assert h.n == (256, 64, 256) and 4 * h.ppc * 256 * 64 * 256 == 1073741824
    lpi = bench.CONFIGS["lpi"]["deck"]
    lo, hi = lpi.slab
    assert 1 <= lpi.laser_ix < lo <= hi <= lpi.n[0]
    assert "[species.beam_p]" in bench.deck_text(ts, n=8)
