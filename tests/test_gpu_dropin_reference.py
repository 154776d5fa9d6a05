"""The reference's OWN hot-path test suite run against the B200 path.

`tools/install_reference.sh` installs the unmodified reference package into the git-ignored
`baseline/_ref/` (which travels to the GPU box) together with its tests.  Here those tests run with
`paper_2306_04039_b200.dropin.install()` applied before collection (tests/dropin_plugin.py), so
molr.mol / molr.hindexer / molr.quant — and every molr module that imported from them, e.g.
RetrievalEngine (engine.py:17-28) — execute on libmolr_b200.so: test_mol.py, test_hindexer.py,
test_quant.py, test_engine.py and the acceptance criteria C7-C9 (test_acceptance.py:149-222)."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tests")),
                                 reason="reference not installed (tools/install_reference.sh)")]


def _run(args):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT]), MOLR_DROPIN_CHECK="1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "tests.dropin_plugin",
           "--rootdir", REF, "-c", os.devnull, *args]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    print(r.stdout[-4000:])
    print(r.stderr[-2000:])
    return r


def test_reference_hot_path_suite_on_b200():
    files = [os.path.join(REF, "tests", f) for f in ("test_mol.py", "test_hindexer.py", "test_quant.py",
                                                     "test_engine.py")]
    r = _run(files)
    assert r.returncode == 0, r.stdout[-3000:]
    assert " passed" in r.stdout


def test_reference_acceptance_c7_c8_c9_on_b200():
    f = os.path.join(REF, "tests", "test_acceptance.py")
    r = _run([f"{f}::test_criterion_07_hindexer_recall", f"{f}::test_criterion_08_two_stage_fidelity",
              f"{f}::test_criterion_09_int8_fidelity"])
    assert r.returncode == 0, r.stdout[-3000:]
    assert "3 passed" in r.stdout


def test_dropin_actually_routes_to_the_library():
    """The patched reference names are this package's objects and the calls launch our kernels."""
    code = (
        "import numpy as np, molr.mol, molr.engine, molr.hindexer, molr.numerics\n"
        "from paper_2306_04039_b200 import dropin, _lib as L\n"
        "import paper_2306_04039_b200.mol as M, paper_2306_04039_b200.hindexer as Hx\n"
        "h = dropin.install()\n"
        "assert molr.mol.mol_top_k is M.mol_top_k and molr.engine.mol_top_k is M.mol_top_k\n"
        "assert molr.engine.h_indexer is Hx.h_indexer and molr.engine.build_item_cache is M.build_item_cache\n"
        "n0 = L.launch_count()\n"
        "v = np.random.default_rng(0).standard_normal((5000, 64)).astype(np.float32)\n"
        "c = molr.hindexer.h_indexer(v, v[3], molr.hindexer.HIndexerConfig(k_prime=50, lam=5000), molr.numerics.make_rng(0))\n"
        "assert 3 in c.indices and L.launch_count() > n0\n"
        "h.uninstall()\n"
        "import molr.mol as R\n"
        "assert molr.mol.mol_top_k is not M.mol_top_k\n"
        "print('routed OK')\n")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT]))
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "routed OK" in r.stdout
