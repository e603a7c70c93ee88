"""Every kernel path (tools/all_paths_smoke.py: RK4/RKF45 scene kernels,
table mode, mode R, the ray-batch trace, unfused shading, banded frames) run
against the debug build libbhrt_b200_debug.so, whose device bounds checks
(BHRT_ASSERT: record/pixel indices, sphere slots and indices, controller
table index, b-table entries) trap on any out-of-range access — the
substitute for compute-sanitizer, which the GPU pool does not offer."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEBUG_LIB = os.path.join(ROOT, "paper_2507_16165_b200", "libbhrt_b200_debug.so")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(DEBUG_LIB), reason="debug library not built")]


def test_all_paths_pass_device_bounds_checks():
    env = dict(os.environ, BHRT_B200_LIB=DEBUG_LIB)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "all_paths_smoke.py")], env=env,
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "done" in r.stdout
