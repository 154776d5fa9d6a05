"""Route the reference package's hot path (molr.mol, molr.hindexer, molr.quant) to this package.

`install()` is the integration a maintainer would add to the reference: it
rebinds every public name of the three reference modules — the functions and the dataclasses —
and the exception classes of molr.errors
to this package's implementation, in those modules AND in every other loaded `molr.*` module
that imported the name (molr.engine, molr.model, molr.cli, ... bind them at import time with
`from molr.mol import ...`), so `RetrievalEngine.query` (engine.py:117-138) and everything else
above the path run on libmolr_b200.so.  Objects the caller built before the switch (a reference
`ItemCache`, `QuantizedRows`, `Mlp`, `HIndexerConfig`) are accepted duck-typed.

    import molr
    from paper_2306_04039_b200 import dropin
    handle = dropin.install()          # molr.* now routes to the B200 path
    ...
    handle.uninstall()                 # restore the reference bindings
"""

from __future__ import annotations

import importlib
import sys

# module -> the public names it exports on the path (mol.py:30-408, hindexer.py:24-214, quant.py:17-90)
SURFACE = {
    "mol": ["MoLConfig", "Mlp", "GatingNetwork", "QueryState", "ItemCache", "component_logits", "decomposed_gating",
            "mol_score", "build_item_cache", "score_candidates", "batch_score_all", "mol_top_k"],
    "hindexer": ["HIndexerConfig", "CandidateSet", "nth_largest", "stage1_scores", "estimate_threshold", "h_indexer",
                 "exact_top_k", "index_select", "stage1_view", "with_k_prime"],
    "quant": ["MAX_DOT_LENGTH", "QuantizedRows", "quantize_rowwise", "quantize_vector", "int8_dot", "int8_matvec"],
    # the exception taxonomy (errors.py:4-63): the path raises this package's classes, so every molr
    # module must raise / catch the same ones
    "errors": ["MolrError", "ZeroNormError", "DimensionMismatchError", "OutOfRangeError", "LengthOverflowError",
               "EmptyCandidatesError", "EmptyCorpusError", "EmptyEvalSetError", "EmptyInputError", "ParseError",
               "EmptyAfterFilterError", "TooFewInteractionsError"],
}
# molr modules that import path names at module level (engine.py:17-28, cli.py:22, train.py:22, ...)
CALLERS = ["engine", "model", "cli", "train", "evaluation", "service", "lineserver", "snapshot", "data", "runconfig"]


class Installed:
    def __init__(self, undo):
        self._undo = undo

    def uninstall(self) -> None:
        for mod, name, old in reversed(self._undo):
            setattr(mod, name, old)
        self._undo = []


def install(package: str = "molr") -> Installed:
    """Rebind the reference's path surface to the B200 implementation; returns an undo handle."""
    ref = {m: importlib.import_module(f"{package}.{m}") for m in SURFACE}
    ours = {m: importlib.import_module(f"paper_2306_04039_b200.{m}") for m in SURFACE}
    originals = {}  # id(reference object) -> replacement
    for m, names in SURFACE.items():
        for n in names:
            if hasattr(ref[m], n):
                originals[id(getattr(ref[m], n))] = (getattr(ref[m], n), getattr(ours[m], n))
    for c in CALLERS:
        try:
            importlib.import_module(f"{package}.{c}")
        except Exception:  # optional modules (e.g. the HTTP service's dependencies) may be absent
            pass
    undo = []
    for name, mod in list(sys.modules.items()):
        if mod is None or not (name == package or name.startswith(package + ".")):
            continue
        for attr, val in list(vars(mod).items()):
            hit = originals.get(id(val))
            if hit is not None and hit[0] is val and hit[1] is not val:
                undo.append((mod, attr, val))
                setattr(mod, attr, hit[1])
    return Installed(undo)


__all__ = ["install", "Installed", "SURFACE"]
