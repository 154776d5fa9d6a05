"""pytest plugin: route the reference package's MoL / h-indexer / quant modules to the B200 path
before the reference's own tests are collected (they bind names with `from molr.mol import ...`
at import time).  Used by tests/test_gpu_dropin_reference.py as `-p tests.dropin_plugin`."""


def pytest_configure(config):
    from paper_2306_04039_b200 import dropin

    config._molr_b200_dropin = dropin.install()
