"""Serving micro-batching: concurrent single-user queries -> device batches.

The reference serves one query per request thread (`lineserver.py:25-86` with up to
`MOLR_THREADS` handler threads, `service.py:38-51`), each running the whole CPU path.  On the GPU
the path only pays off in batches, so `MicroBatcher` collects concurrent requests for up to
`max_wait_ms` (the paper's ~10 ms batching window) or `max_batch` requests, runs ONE
batched query, and hands every caller its own rows.

Determinism (the reference's contract: 100 concurrent identical queries return identical bytes,
`test_lineserver.py:90-107`): every batch is run with the engine's fixed seed, and a query's
candidates depend only on its own stage-1 scores and that seed (the device sample is shared by
the batch, not drawn per position), so a result never depends on which other requests happened
to share its batch.

`run_batch` is any callable (features (n, d_u), k) -> (ids (n, k), scores (n, k)); the default
binds `BatchedRetrievalEngine.query_features`.
"""

from __future__ import annotations

import queue
import threading
import time
from concurrent.futures import Future

import numpy as np


class MicroBatcher:
    def __init__(self, run_batch, *, max_batch: int = 1024, max_wait_ms: float = 10.0, k: int = 100):
        if max_batch < 1:
            raise ValueError("max_batch must be >= 1")
        self._run = run_batch
        self.max_batch = int(max_batch)
        self.max_wait = float(max_wait_ms) / 1e3
        self.k = int(k)
        self._q: "queue.Queue" = queue.Queue()
        self._stop = threading.Event()
        self.batches = 0  # number of device batches run (observability)
        self._t = threading.Thread(target=self._loop, name="molr-microbatcher", daemon=True)
        self._t.start()

    @classmethod
    def for_engine(cls, engine, **kw):
        k = kw.pop("k", 100)
        return cls(lambda feats, kk: engine.query_features(feats, kk)[:2], k=k, **kw)

    def submit(self, user_feats) -> Future:
        """Queue one query (raw user features, shape (d_u,)); the Future yields (ids, scores)."""
        if self._stop.is_set():
            raise RuntimeError("batcher is closed")
        f: Future = Future()
        self._q.put((np.asarray(user_feats, dtype=np.float32).reshape(-1), f))
        return f

    def query(self, user_feats, timeout: float | None = None):
        """Blocking single query: [(item id, score)] like RetrievalEngine.query (engine.py:117-138)."""
        ids, sc = self.submit(user_feats).result(timeout)
        return [(int(i), float(s)) for i, s in zip(ids, sc)]

    def close(self):
        self._stop.set()
        self._q.put(None)
        self._t.join(timeout=5)

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _loop(self):
        while not self._stop.is_set():
            item = self._q.get()
            if item is None:
                break
            reqs = [item]
            deadline = time.perf_counter() + self.max_wait
            while len(reqs) < self.max_batch:
                left = deadline - time.perf_counter()
                if left <= 0:
                    break
                try:
                    nxt = self._q.get(timeout=left)
                except queue.Empty:
                    break
                if nxt is None:
                    self._stop.set()
                    break
                reqs.append(nxt)
            feats = np.stack([r[0] for r in reqs])
            try:
                ids, sc = self._run(feats, self.k)
                self.batches += 1
                for i, (_, f) in enumerate(reqs):
                    f.set_result((np.array(ids[i]), np.array(sc[i])))
            except BaseException as e:  # every waiter sees the failure
                for _, f in reqs:
                    if not f.done():
                        f.set_exception(e)
        # drain: fail whatever is still queued
        while True:
            try:
                item = self._q.get_nowait()
            except queue.Empty:
                break
            if item is not None and not item[1].done():
                item[1].set_exception(RuntimeError("batcher closed"))
