"""bench.py contract on CPU: the reference arm (the unmodified reference package
from baseline/_ref, numba, on the host cores) prints one JSON line with the
driver's keys, times exactly K steps, and maps none of this repo's libraries."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_json_line():
    import pytest
    if not (ROOT / "baseline" / "_ref" / "sparseconv").is_dir():
        pytest.skip("reference not installed into baseline/_ref (DESIGN.md: reference arm)")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--batch", "16", "--ref-seconds", "60"], capture_output=True,
                         text=True, timeout=600, cwd=ROOT, check=True).stdout
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1
    assert d["value"] > 0 and d["unit"] == "images/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert not [l for l in d["repo_native_libs_loaded"] if l.startswith("paper_2011_06295_b200")], d
    assert d["config"]["workload"].startswith("VGG-16 CIFAR-10") and d["config"]["images_per_step"] == 16
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
