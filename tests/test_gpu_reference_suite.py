"""Run the reference's own backend-parametrised tests with the `sm100` backend registered.

Needs oracle/_ref (the unmodified reference + its tests, built by
oracle/build_ref.sh in the build container; the built tree travels to the GPU box).
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tests")),
                    reason="oracle/_ref not built (run oracle/build_ref.sh)")
def test_reference_suite_with_sm100_backend():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT, env.get("PYTHONPATH", "")])
    files = [os.path.join(REF, "tests", f) for f in ("test_multivec.py", "test_kernels.py")]
    out = subprocess.run(
        [sys.executable, "-m", "pytest", "-v", "-p", "paper_2111_06552_b200.refbackend_plugin",
         "-k", "sm100 or backends", "-o", "cache_dir=/tmp/.ref_cache", *files],
        capture_output=True, text=True, env=env, cwd=REF, timeout=600)
    tail = out.stdout[-3000:] + out.stderr[-2000:]
    assert out.returncode == 0, tail
    ran = [ln for ln in out.stdout.splitlines() if "[sm100" in ln and "PASSED" in ln]
    assert len(ran) >= 10, tail
