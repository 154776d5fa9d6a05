"""CPU oracle for the MoL + h-indexer hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in NumPy, the reference algorithm of arXiv 2306.04039's
`molr` package (`/root/reference/pkg/src/molr/{mol,hindexer,quant,numerics}.py`),
function by function, each citing the reference file:line it follows.

Who may import it: `tests/`, `__graft_entry__.smoke()` (as the checker) and
`bench.py` (the `cpu_baseline` leg and `--impl reference`).  The product package
`paper_2306_04039_b200` never imports it: the GPU path has no CPU fallback.

Pinning: `tests/test_oracle_golden.py` checks this restatement against the golden
vectors in `tests/golden/` that `tests/golden/make_golden.py` produced by importing
the reference itself (`PYTHONPATH=/root/reference/pkg/src`).  Parity is pinned.
"""

from oracle.molr_oracle import *  # noqa: F401,F403
