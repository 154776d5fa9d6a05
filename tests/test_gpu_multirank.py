"""Two ranks (torch.distributed, gloo for the exchange, both on cuda:0) run the sharded product
path end to end — item-range shard, local K'/P and lambda/P, device two-stage top-k with global
ids, all-gather of (ids, scores), molr_merge_top_k — and the merged top-k must match the exact
MoL top-k over the whole corpus (recall >= 0.99, scores within tolerance).  This is the code path
bench.py runs with one rank per GPU under NCCL."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), MOLR_DEVICE="0")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from paper_2306_04039_b200.engine import merge_top_k, two_stage_top_k
    from paper_2306_04039_b200.hindexer import HIndexerConfig
    from paper_2306_04039_b200.mol import ItemCache
    from paper_2306_04039_b200.quant import quantize_rowwise
    from paper_2306_04039_b200.sharding import local_k_prime, local_lambda, shard_range
    from tests.test_gpu_parity import _prod_gating, _synthetic_prod_cache

    cache, syn, ue, feats = _synthetic_prod_cache(60_000, seed=41, n_users=24)
    gating, og = _prod_gating(syn)
    X, k, kp = cache.num_items, 50, 3000
    lo, hi = shard_range(X, world, rank)
    s1 = cache.stage1_embs[lo:hi]
    shard = ItemCache(config=cache.config, item_embs=cache.item_embs[lo:hi], item_gate_pre=cache.item_gate_pre[lo:hi],
                      stage1_embs=s1, stage1_q=quantize_rowwise(s1))
    h = HIndexerConfig(k_prime=local_k_prime(kp, world), lam=local_lambda(hi - lo, sample_ratio=0.05), quantized=True)
    uw = gating.user_net(feats)
    ids, sc, _ = two_stage_top_k(shard, gating, ue, uw, k, h, seed=9, id_offset=lo)
    g_ids = [torch.empty(ids.shape, dtype=torch.int64) for _ in range(world)]
    g_sc = [torch.empty(sc.shape, dtype=torch.float32) for _ in range(world)]
    dist.all_gather(g_ids, torch.from_numpy(ids))
    dist.all_gather(g_sc, torch.from_numpy(sc))
    if rank == 0:
        mi, ms = merge_top_k(np.stack([t.numpy() for t in g_ids]), np.stack([t.numpy() for t in g_sc]), k)
        oc = O.Cache(cache.item_embs, cache.item_gate_pre, cache.stage1_embs, None, 20.0, 8)
        rec, close = [], True
        for u in range(ue.shape[0]):
            ei, es = O.full_top_k(oc, og, ue[u], feats[u], k)
            rec.append(len(set(ei.tolist()) & set(mi[u].tolist())) / k)
            ref = O.score_candidates(oc, og, mi[u], ue[u], feats[u])
            close &= bool(O.score_close(ms[u], ref).all())
        out.put((float(np.mean(rec)), close, bool(np.all(mi >= 0)) and bool(np.all(mi < X))))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_path_matches_exact():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    rec, close, in_range = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    print("merged recall", rec)
    assert in_range and close and rec >= 0.99
