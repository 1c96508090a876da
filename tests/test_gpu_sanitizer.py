"""compute-sanitizer memcheck / racecheck / synccheck over every kernel family
(race detection on the small config in CI).  The workload
is tools/sanitize_smoke.py: parity + fast renders with the field, the path
tracer, photon tracing + KNN build / queries (K <= 64 and K > 64) / targets,
the photon-map render and a train step."""
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not Path(exe).exists():
        pytest.skip("compute-sanitizer not installed")
    r = subprocess.run([exe, "--tool", tool, "--error-exitcode", "3", sys.executable,
                        str(ROOT / "tools" / "sanitize_smoke.py")], capture_output=True, text=True, timeout=600)
    tail = (r.stdout + r.stderr)[-3000:]
    if "sanitize workload done" not in r.stdout and "compute-sanitizer is closed" in tail:
        # some GPU pools replace the tool with a stub that refuses to run
        pytest.skip("compute-sanitizer unavailable on this GPU pool: " + tail.strip().splitlines()[0][:200])
    assert r.returncode == 0, tail
    assert "sanitize workload done" in r.stdout, tail
    assert ("0 errors" in tail) or ("0 hazards" in tail), tail
