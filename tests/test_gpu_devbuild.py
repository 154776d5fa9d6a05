"""Backend cross-checks under the development build.

The production library (libmolr_b200.so) has one backend per shape and reads no environment; the
alternative SIMT scans / generic MoL kernel / pilot-size switches that the `devknobs` tests compare
against exist only in libmolr_b200_dev.so (-DMOLR_DEV_KNOBS, same sources).  This test runs those
tests in a subprocess with MOLR_LIB_PATH pointing at the dev build, so every tensor-core path is
also checked bit-for-bit (or within tolerance for the MoL kernel) against its SIMT counterpart."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEV = os.path.join(ROOT, "paper_2306_04039_b200", "libmolr_b200_dev.so")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(os.path.basename(os.environ.get("MOLR_LIB_PATH", "")) == "libmolr_b200_dev.so",
                    reason="already running under the dev build")
def test_devknobs_crosschecks_under_dev_build():
    assert os.path.exists(DEV), "build the dev library (make in paper_2306_04039_b200/csrc)"
    env = dict(os.environ, MOLR_LIB_PATH=DEV)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu and devknobs", "tests"], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=3000)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
