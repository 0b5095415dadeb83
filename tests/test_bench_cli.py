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
    d = _run("--impl", "reference", "--steps", "3", "--warmup", "2", "--cpu-sample-n", "12")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    # the line reports the steps it timed and names its bounded sample
    assert d["steps"] == 3 and d["warmup"] == 2
    assert d["config"]["sample_cells"] == "12^3" and d["config"]["same_config"] is False
    assert d["config"]["workload"] == "two_stream" and d["config"]["cells"] == "256^3"
    assert d["metric"].startswith("particle pushes/sec summed over all GPUs")


def test_reference_arm_sort_cadence_inside_window():
    """With a sort point among the timed steps the reference's own run-loop
    sort is timed (nothing amortised separately)."""
    from oracle.bindings import ref_available
    if not ref_available():
        import pytest
        pytest.skip("oracle/_ref not built")
    d = _run("--impl", "reference", "--steps", "20", "--warmup", "1", "--cpu-sample-n", "8")
    assert d["steps"] == 20 and "amortised" not in d["config"]["sample"]


def test_aggregate_value_and_per_gpu(monkeypatch):
    """value is the whole-job sum over ranks and value_per_gpu = value / N
    (BASELINE.json's per-GPU metric), for the kernel line and e2e alike."""
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert '"value_per_gpu": value / world' in src
    assert 'npart_all * k / dt / world' in src
    assert 'float(tn.item()) * k / dt / world' in src


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
