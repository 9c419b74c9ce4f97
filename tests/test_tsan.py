"""CPU: ThreadSanitizer over the host-side C++ (SURVEY.md §5 race detection):
scripts/tsan.sh builds the offsim core + C ABI with -fsanitize=thread and
runs the reference's own unit, C ABI and acceptance suites on it. Needs the
reference sources (build container); skipped elsewhere."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_host_core_is_tsan_clean(tmp_path):
    if not Path("/root/reference/proj/src").is_dir():
        pytest.skip("reference sources not present")
    r = subprocess.run(["bash", str(ROOT / "scripts" / "tsan.sh"), str(tmp_path)], capture_output=True,
                       text=True, timeout=1800)
    assert r.returncode == 0, r.stderr[-2000:]
    for t in ("unit", "capi", "acc"):
        log = (tmp_path / f"tsan_{t}.log").read_text()
        assert "WARNING: ThreadSanitizer" not in log, log[-3000:]
        assert "rc=0" in log
