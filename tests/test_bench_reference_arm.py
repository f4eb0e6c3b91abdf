"""The bench's reference arm on the CPU (no GPU needed): one JSON line with the
contract's keys; ``kind`` is "reference" when the unmodified reference is
installed under baseline/_ref (``__graft_entry__.build()`` in the build
container), else "port" (the C restatement)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["higher_is_better"] is True and d["value"] > 0
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    cpu = d["cpu_baseline"]
    assert cpu["value"] == d["value"] and cpu["cores"] >= 1
    have_ref = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "tilemesh"))
    try:
        import numba  # noqa: F401
    except ImportError:
        have_ref = False
    if have_ref:
        assert cpu["kind"] == "reference" and cpu["port"]["kind"] == "port" and cpu["port"]["value"] > 0
    else:
        assert cpu["kind"] == "port"
