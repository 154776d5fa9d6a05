"""ctypes wrapper of oracle/molr_oracle.c (TEST INFRASTRUCTURE ONLY — the C restatement of the
reference's MoL scoring, mol.py:139-205 / 329-408, multithreaded over items).  Used by tests/ and by
bench.py's parity leg to recompute exact full-corpus scores at BASELINE's sizes; pinned against the
reference-produced golden vectors and the NumPy restatement in tests/test_oracle_c.py."""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "libmolr_oracle.so")
_lib = None


def build() -> str:
    subprocess.check_call(["make", "-s"], cwd=_HERE)
    return LIB


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        lib = C.CDLL(LIB)
        P, I, L, F = C.c_void_p, C.c_int, C.c_int64, C.c_float
        lib.molo_scores.argtypes = [L, I, I, I, I, P, I, P, I, I, P, P, P, P, P, F, P, L, I]
        lib.molo_score_candidates.argtypes = [I, I, I, I, P, I, P, I, I, P, P, P, P, P, F, P, P, P, I]
        lib.molo_topk_merge.argtypes = [I, L, P, L, L, I, P, P, I]
        lib.molo_num_threads.argtypes = []
        _lib = lib
    return _lib


def num_threads() -> int:
    return int(load().molo_num_threads())


def _items(a):
    """(pointer-owner array, dtype flag): f32 arrays as is, bf16 given as uint16 bit patterns."""
    a = np.asarray(a)
    if a.dtype == np.uint16:
        return np.ascontiguousarray(a), 1
    return np.ascontiguousarray(a, dtype=np.float32), 0


class Net:
    """The cross net (W1 (G,H), b1 (H,), W2 (H,G)) in the layout the C oracle reads."""

    def __init__(self, w1, b1, w2):
        self.w1 = np.ascontiguousarray(w1, dtype=np.float32)
        self.b1 = np.ascontiguousarray(b1, dtype=np.float32)
        self.w2 = np.ascontiguousarray(w2, dtype=np.float32)
        self.G, self.H = self.w1.shape


def scores(item_embs, gate_pre, user_embs, uw, cross: Net, tau: float, *, threads: int = 0) -> np.ndarray:
    """(B, n) exact MoL scores of B queries (user_embs (B,k_u,d), uw = user_net(feat) (B,G))
    against every item (item_embs (n,k_x,d), gate_pre (n,G); f32 or bf16 bits)."""
    e, edt = _items(item_embs)
    g, gdt = _items(gate_pre)
    ue = np.ascontiguousarray(user_embs, dtype=np.float32)
    uwf = np.ascontiguousarray(uw, dtype=np.float32)
    n, k_x, d = e.shape
    B, k_u, _ = ue.shape
    out = np.empty((B, n), dtype=np.float32)
    st = load().molo_scores(n, k_u, k_x, d, cross.H, e.ctypes.data, edt, g.ctypes.data, gdt, B, ue.ctypes.data,
                            uwf.ctypes.data, cross.w1.ctypes.data, cross.b1.ctypes.data, cross.w2.ctypes.data,
                            float(tau), out.ctypes.data, n, int(threads))
    if st != 0:
        raise ValueError("molo_scores: unsupported shape")
    return out


def score_candidates(item_embs, gate_pre, user_embs, uw, cross: Net, tau: float, lists, *, threads: int = 0):
    """Per query b, the scores of its candidate ids lists[b] (score_candidates, mol.py:329-345)."""
    e, edt = _items(item_embs)
    g, gdt = _items(gate_pre)
    ue = np.ascontiguousarray(user_embs, dtype=np.float32)
    uwf = np.ascontiguousarray(uw, dtype=np.float32)
    n, k_x, d = e.shape
    B, k_u, _ = ue.shape
    lists = [np.asarray(x, dtype=np.int64).reshape(-1) for x in lists]
    offs = np.zeros(B + 1, dtype=np.int64)
    offs[1:] = np.cumsum([x.size for x in lists])
    ids = np.ascontiguousarray(np.concatenate(lists) if lists else np.zeros(0, np.int64))
    if ids.size and (ids.min() < 0 or ids.max() >= n):
        raise IndexError("candidate id outside the items")
    out = np.empty(ids.size, dtype=np.float32)
    st = load().molo_score_candidates(k_u, k_x, d, cross.H, e.ctypes.data, edt, g.ctypes.data, gdt, B,
                                      ue.ctypes.data, uwf.ctypes.data, cross.w1.ctypes.data, cross.b1.ctypes.data,
                                      cross.w2.ctypes.data, float(tau), offs.ctypes.data, ids.ctypes.data,
                                      out.ctypes.data, int(threads))
    if st != 0:
        raise ValueError("molo_score_candidates: unsupported shape")
    return [out[offs[b]:offs[b + 1]] for b in range(B)]


class TopK:
    """Running exact top-k per query by (score desc, id asc) — np.lexsort((ids, -s)) (mol.py:407) —
    over a corpus scored chunk by chunk."""

    def __init__(self, B: int, k: int):
        self.k = k
        self.ids = np.full((B, k), -1, dtype=np.int64)
        self.scores = np.full((B, k), -np.inf, dtype=np.float32)

    def add(self, scores, id_offset: int, *, threads: int = 0):
        s = np.ascontiguousarray(scores, dtype=np.float32)
        B, n = s.shape
        load().molo_topk_merge(B, n, s.ctypes.data, n, int(id_offset), self.k, self.ids.ctypes.data,
                               self.scores.ctypes.data, int(threads))
        return self


def exact_top_k_streamed(read_rows, n_items: int, user_embs, uw, cross: Net, tau: float, k: int, *,
                         chunk: int = 1 << 21, threads: int = 0):
    """The reference's exhaustive MoL top-k (RetrievalEngine.full_top_k, engine.py:140-147: every
    item scored by mol.py:329-345, ranked by np.lexsort((ids, -s)), mol.py:407) over a corpus too
    large to hold on the host in f32: `read_rows(row0, n)` returns (item_embs (n,k_x,d),
    gate_pre (n,G)) for rows [row0, row0 + n) (f32 or bf16 bits).  Returns (ids (B,k), scores (B,k))."""
    ue = np.ascontiguousarray(user_embs, dtype=np.float32)
    tk = TopK(ue.shape[0], k)
    for lo in range(0, n_items, chunk):
        hi = min(n_items, lo + chunk)
        e, g = read_rows(lo, hi - lo)
        tk.add(scores(e, g, ue, uw, cross, tau, threads=threads), lo, threads=threads)
    return tk.ids, tk.scores
