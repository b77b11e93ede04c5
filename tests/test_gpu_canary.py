"""Our own bounds check (compute-sanitizer is closed on this pool): with
SIP_CANARY=1 every device field is allocated with guard bands filled with a
canary pattern, checked after each solve; any kernel writing outside a
field's storage makes the solve fail with SIP_ERR_CUDA.  Runs every kernel
family of the path on small cases (tools/sanitize_case.py).  Marked gpu."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_guard_bands_intact():
    env = dict(os.environ, SIP_CANARY="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py")],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    assert r.stdout.count("ok ") >= 8, r.stdout
