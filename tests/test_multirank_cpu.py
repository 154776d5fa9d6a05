"""World-size-2 gloo test of the sharded retrieval plumbing (CPU): each rank scores its item
shard (oracle arithmetic), all-gathers (score, global id) top-k lists over torch.distributed, and
the rank-major merge equals the single-process top-k over the whole corpus (mol.py:407 order)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2306_04039_b200.sharding import local_k_prime, local_lambda, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _merge(ids, scores, k):
    """Host restatement of molr_merge_top_k's order: (score desc, id asc)."""
    ids = ids.reshape(-1)
    scores = scores.reshape(-1)
    order = np.lexsort((ids, -scores))[:k]
    return ids[order], scores[order]


def _worker(rank, world, port, out):
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    syn = O.init_synthetic(4, 3000, k_u=2, k_x=2, d=8, gating_hidden=16, d_u=12, d_x=12, proj_hidden=16, seed=3)
    cache = O.build_item_cache(syn.item_table, syn.item_proj, syn.gating.item_net, 2, 8, 20.0, 2)
    ue = O.user_components(syn, np.arange(4), 2, 8)
    X, k = cache.item_embs.shape[0], 20
    lo, hi = shard_range(X, world, rank)
    shard = O.index_select(cache, np.arange(lo, hi))
    res_ids, res_sc = [], []
    for u in range(4):
        ids, sc = O.full_top_k(shard, syn.gating, ue[u], syn.user_table[u], k)
        res_ids.append(ids + lo)
        res_sc.append(sc)
    t_ids = torch.tensor(np.stack(res_ids), dtype=torch.int64)
    t_sc = torch.tensor(np.stack(res_sc), dtype=torch.float32)
    g_ids = [torch.empty_like(t_ids) for _ in range(world)]
    g_sc = [torch.empty_like(t_sc) for _ in range(world)]
    dist.all_gather(g_ids, t_ids)
    dist.all_gather(g_sc, t_sc)
    if rank == 0:
        ok = True
        for u in range(4):
            mi, ms = _merge(np.stack([g[u].numpy() for g in g_ids]), np.stack([g[u].numpy() for g in g_sc]), k)
            fi, fs = O.full_top_k(cache, syn.gating, ue[u], syn.user_table[u], k)
            ok &= mi.tolist() == fi.tolist()
        out.put(ok)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_merge_equals_global_topk_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert ok


def test_shard_math():
    assert shard_range(100_000_000, 8, 7) == (87_500_000, 100_000_000)
    assert [shard_range(10, 3, r) for r in range(3)] == [(0, 3), (3, 6), (6, 10)]
    assert local_k_prime(100_000, 8) == 12_500
    assert local_lambda(12_500_000, sample_ratio=0.01) == 125_000
    assert local_lambda(10, lam=100, world=2) == 10
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)
