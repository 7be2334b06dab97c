"""Memory / race checks of every kernel family (tools/sanitize_cases.py) under NYS_DEBUG_GUARD=1:
NaN-poisoned workspaces with canaries verified after every ABI call, sentinel-guarded caller outputs,
and bitwise run-to-run determinism (compute-sanitizer is closed on the GPU pool)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("guard", ["1", None])
def test_guarded_cases_clean_and_deterministic(guard):
    env = dict(os.environ)
    if guard:
        env["NYS_DEBUG_GUARD"] = guard
    else:
        env.pop("NYS_DEBUG_GUARD", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")], capture_output=True,
                       text=True, timeout=900, cwd=ROOT, env=env)
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "failures: 0" in r.stdout
