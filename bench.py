#!/usr/bin/env python
"""MoL + h-indexer top-100 retrieval benchmark (BASELINE.json metric: queries/sec over a 100M-item
synthetic corpus, p50 latency, recall vs the exact MoL top-k).

One step = one batch of B=1024 queries (raw user features) through the whole path on every rank:
device query prep (user_proj MLP + L2 norm -> user components, user_net -> gating weights) ->
stage-1 query + int8 quantisation -> sampled threshold -> full-corpus int8 scan + filter ->
MoL re-scoring of the passers -> top-100 -> (N>1) NCCL all-gather of (score, id) + merge.
The corpus (100M items, k_x=8 x d=64 bf16 item embeddings, bf16 gate pre-activations, int8
stage-1 rows) is sharded across ranks by contiguous item ranges; it is built on the device from a
seeded synthetic model with the reference's init convention (model.py:121-163) by the product's
fused device cache build (molr_cache_build_rows).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 100m|10m|books|ml20m] [--impl reference]

Prints ONE JSON line (rank 0).  `--impl reference` times the reference algorithm's CPU port
(oracle/, NumPy, one process per host core) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # X items, B queries per step, k, K', sample ratio r (lambda = r X)
    "100m": dict(X=100_000_000, B=1024, k=100, k_prime=100_000, ratio=0.01, label="100M-item synthetic corpus"),
    "10m": dict(X=10_000_000, B=1024, k=100, k_prime=100_000, ratio=0.01, label="10M-item synthetic corpus"),
    # the reference's default stage-1 view (quantized=False): fp32 scores, filtered on the tensor
    # cores with an exact fp32 re-check (K2f)
    "10m_f32": dict(X=10_000_000, B=1024, k=100, k_prime=100_000, ratio=0.01, view="f32",
                    label="10M-item synthetic corpus, float stage-1 view"),
    "100m_f32": dict(X=100_000_000, B=1024, k=100, k_prime=100_000, ratio=0.01, view="f32",
                     label="100M-item synthetic corpus, float stage-1 view"),
    "books": dict(X=2_300_000, B=1024, k=100, k_prime=100_000, ratio=0.01, label="Amazon-Books-shaped 2.3M items"),
    # exact path (batch_score_all + mol_top_k over the whole corpus, mol.py:348-408): one step =
    # B users x all X items; the full ML-20M run is 138K users
    "ml20m": dict(X=27_000, B=1024, k=100, k_prime=None, ratio=None, exact=True, users=138_000,
                  label="ML-20M-shaped synthetic: 27K items, exact MoL top-100"),
    # a reference-built cache (mol.py:294-326 in f32: components and gate pre-activations not
    # bf16-representable), served by the tcgen05 scorer through its bf16 hi + lo image (K1)
    "ml20m_f32cache": dict(X=27_000, B=1024, k=100, k_prime=None, ratio=None, exact=True, users=138_000,
                           cache="f32", label="ML-20M-shaped synthetic, f32 (reference-built) cache: 27K items, "
                                               "exact MoL top-100"),
    "books_f32cache": dict(X=2_300_000, B=1024, k=100, k_prime=100_000, ratio=0.01, cache="f32",
                           label="Amazon-Books-shaped 2.3M items, f32 (reference-built) cache"),
    # BASELINE configs[0]: one step = every user of the ML-1M shape against the whole corpus
    "ml1m": dict(X=3_706, B=6_040, k=200, k_prime=None, ratio=None, exact=True, users=6_040,
                 label="ML-1M-shaped synthetic: 6,040 users x 3,706 items, exact MoL top-200"),
}
# queries checked against the CPU oracle (oracle/molr_oracle.c) after the timed region: exhaustive
# oracle top-k for ORACLE_Q[config] queries (all users for ML-1M), oracle scores of the returned items
ORACLE_Q = {"100m": 2, "100m_f32": 2, "10m": 8, "10m_f32": 8, "books": 16, "ml20m": 64, "ml1m": 6_040,
            "ml20m_f32cache": 64, "books_f32cache": 16}
K_U = K_X = 8
D = 64
G = 64
H = 128
D_U = D_X = 64
PROJ_H = 128
TAU = 20.0
CHUNK = 500_000  # global corpus generation chunk (shard boundaries are chunk-aligned)

# per-unit algorithmic work: one MoL pair, one stage-1 (query, row) dot
PAIR_BYTES = K_X * D * 2 + G * 2 + 4       # bf16 item components + bf16 gate_pre + int32 id = 1156 B
PAIR_BYTES_F32C = K_X * D * 4 + G * 4 + 4  # f32 cache: bf16 hi + lo components + f32 gate_pre + id = 2308 B
PAIR_FLOPS = 2 * (G * D + G * H + H * G)   # component GEMM + cross-net 64->128->64 = 40960
S1_OPS = 2 * D                             # int8 MACs x 2 per (query, row)
PAIR_MUFU = 2 * H + 2 * G + G              # ex2 + rcp per hidden / combine SiLU, ex2 per softmax term = 448


def tc_microbench_peaks():
    """tcgen05 dense MMA rates measured by tools/tc_peak_bench.cu on this pool's B200 (one CTA per
    SM, back-to-back M128 x N256 MMAs, max clock): {"i8": Tops/s, "f16": TFLOP/s}, or {}."""
    out = {}
    try:
        with open(os.path.join(ROOT, "profiles", "r02_tc_peak_bench.json")) as f:
            for l in f:
                if l.strip():
                    d = json.loads(l)
                    out["i8" if "i8" in d["mma"] else "f16"] = d["tops_per_s"]
    except Exception:
        pass
    return out


def mufu_peak():
    """Measured MUFU throughput (tools/mufu_bench.cu on this pool's B200: ex2 / rcp, all SMs),
    else the nominal 16 per clock per SM at 1.965 GHz."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_mufu_bench.json")) as f:
            v = [json.loads(l)["ops_per_s"] for l in f if l.strip()]
        return min(v), "measured (profiles/r02_mufu_bench.json)"
    except Exception:
        return 16 * 148 * 1.965e9, "nominal 16/clk/SM x 148 SMs x 1.965 GHz"


def peaks():
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "src": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update(hbm_gbs=m["hbm_gbs"], bf16_tflops=m["bf16_tflops"],
                 bf16_tflops_sustained=m.get("bf16_tflops_sustained", m["bf16_tflops"]), src="measured")
    except Exception:
        pass
    return p


# ------------------------------------------------------------------------------------------
# synthetic model (reference init convention: tables U(+-1/sqrt(dim)), MLPs U(+-1/sqrt(fan_in)))
# ------------------------------------------------------------------------------------------
def _mlp(rng, n_in, n_h, n_out):
    b1, b2 = 1 / math.sqrt(n_in), 1 / math.sqrt(n_h)
    return (rng.uniform(-b1, b1, (n_in, n_h)).astype(np.float32), rng.uniform(-b1, b1, n_h).astype(np.float32),
            rng.uniform(-b2, b2, (n_h, n_out)).astype(np.float32))


def synthetic_model(seed=4242):
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence(seed)))
    return {"user_proj": _mlp(rng, D_U, PROJ_H, K_U * D), "item_proj": _mlp(rng, D_X, PROJ_H, K_X * D),
            "user_net": _mlp(rng, D_U, H, G), "item_net": _mlp(rng, D_X, H, G), "cross_net": _mlp(rng, G, H, G)}


def build_shard(model, X, lo, hi, seed, dev, lib, ctx, storage=None, f32_cache=False):
    """Build rows [lo, hi) of the global corpus on the device into a DeviceItemCache through the
    product's fused cache build (molr_cache_build_rows: item_proj MLP -> L2 norm -> item_net ->
    bf16 storage rounding -> stage-1 mean -> int8), from a synthetic item table drawn on the
    device chunk by chunk (same global rows for every N)."""
    import torch

    from paper_2306_04039_b200 import _lib as L
    from paper_2306_04039_b200.mol import DeviceItemCache, MoLConfig
    from paper_2306_04039_b200.numerics import DEFAULT_EPS

    cfg = MoLConfig(k_u=K_U, k_x=K_X, d=D, tau=TAU, gating_hidden=H, dropout_p=0.0)
    if storage is None:
        storage = L.STORE_S1_INT8
    if f32_cache:  # the reference's f32 cache values (no bf16 rounding), stored losslessly in f32
        storage |= L.STORE_EMBS_F32 | L.STORE_GP_F32
    cache = DeviceItemCache(cfg, hi - lo, D, storage)
    W = {k: [torch.from_numpy(a).to(dev) for a in v] for k, v in model.items()}
    pw, nw = W["item_proj"], W["item_net"]
    s = torch.cuda.current_stream().cuda_stream
    with torch.no_grad():
        for ci in range(lo // CHUNK, (hi + CHUNK - 1) // CHUNK):
            g0, g1 = ci * CHUNK, min((ci + 1) * CHUNK, X)  # global chunk: same rows for every N
            gen = torch.Generator(device=dev)
            gen.manual_seed(seed * 1_000_003 + ci)
            t = (torch.rand((g1 - g0, D_X), generator=gen, device=dev) * 2 - 1) / math.sqrt(D_X)
            c0, c1 = max(lo, g0), min(hi, g1)
            t = t[c0 - g0:c1 - g0].contiguous()
            L.call("molr_cache_build_rows", cache.device_handle(), c0 - lo, c1 - c0, D_X, t.data_ptr(), PROJ_H,
                   pw[0].data_ptr(), pw[1].data_ptr(), pw[2].data_ptr(), H, nw[0].data_ptr(), nw[1].data_ptr(),
                   nw[2].data_ptr(), L.BUILD_L2_NORMALIZE | (0 if f32_cache else L.BUILD_ROUND_BF16),
                   float(DEFAULT_EPS), s)
    torch.cuda.synchronize()
    return cfg, cache


def make_queries(model, B, seed, dev):
    """B users' raw features (the user_table rows of the reference convention, U(+-1/sqrt(d_u)))."""
    import torch

    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence([seed, 7])))
    feats = (rng.uniform(-1, 1, (B, D_U)) / math.sqrt(D_U)).astype(np.float32)
    return feats, torch.from_numpy(feats).to(dev)


# ------------------------------------------------------------------------------------------
# clocks sampled during the timed region
# ------------------------------------------------------------------------------------------
class Clocks:
    """Samples SM clock + throttle reasons through NVML (in-process, every 100 ms) while active."""

    def __init__(self, dev_index):
        self.dev = dev_index
        self.samples = []
        self.stop = threading.Event()
        self.ok = False

    def _run(self):
        import pynvml as N

        while not self.stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, r))
            except Exception:
                pass
            self.stop.wait(0.1)

    def __enter__(self):
        if os.environ.get("MOLR_NO_CLOCKS") == "1":
            self.err = "disabled (MOLR_NO_CLOCKS)"
            return self
        try:
            import pynvml as N

            N.nvmlInit()
            self.h = None
            try:  # NVML and CUDA may order devices differently: match by UUID
                import torch

                self.h = N.nvmlDeviceGetHandleByUUID("GPU-" + str(torch.cuda.get_device_properties(self.dev).uuid))
            except Exception:
                self.h = N.nvmlDeviceGetHandleByIndex(self.dev)
            self.max_sm = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                         "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                         "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                         "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
            self.ok = True
        except Exception as e:
            self.err = repr(e)
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.ok:
            self.t.join(timeout=2)

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable: " + getattr(self, "err", "")]}
        reasons = sorted({k for _, r in self.samples for k, b in self.bits.items() if r & b})
        return {"sm_mhz": float(np.median([s for s, _ in self.samples])), "sm_max_mhz": float(self.max_sm),
                "samples": len(self.samples), "reasons": reasons, "source": "nvml"}


# ------------------------------------------------------------------------------------------
# CPU baseline: the reference algorithm's NumPy port (oracle/) on the host cores
# ------------------------------------------------------------------------------------------
def _cpu_worker(args):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    import oracle as O

    seed, reps, X1, k_prime, ratio, k, f32_view = args
    st = _CPU_STATE
    t1s, t2s = [], []
    for r in range(reps):
        u = (seed * 131 + r) % st["ue"].shape[0]
        q1 = st["ue"][u].mean(axis=0)
        t0 = time.perf_counter()
        if k_prime is None:  # exact path: mol_top_k over the whole corpus (engine.py:140-147)
            O.mol_top_k(st["cache"], st["gating"], st["cand"], st["ue"][u], st["feats"][u], k)
            t1s.append(0.0)
            t2s.append(time.perf_counter() - t0)
            continue
        O.h_indexer(st["cache"].stage1_embs if f32_view else st["cache"].stage1_q, q1,
                    max(1, k_prime * X1 // st["X"]), O.make_rng([9000, u]),
                    sample_ratio=ratio)
        t1 = time.perf_counter()
        O.mol_top_k(st["cache"], st["gating"], st["cand"], st["ue"][u], st["feats"][u], k)
        t2 = time.perf_counter()
        t1s.append(t1 - t0)
        t2s.append(t2 - t1)
    return t1s, t2s


_CPU_STATE = {}


def cpu_baseline(cfg, reps=2, procs=None, X1=1_000_000):
    """Per query at X items: stage 1 (h_indexer int8 incl. the rng permutation) timed on an X1-row
    shard and scaled by X/X1 (it is linear in X), plus stage 2 (mol_top_k) on K' candidates at full
    size.  One process per host core, each on its own queries; qps = procs / t_query."""
    import multiprocessing as mp

    import oracle as O

    model = synthetic_model()
    exact = cfg.get("exact", False)
    ncand = cfg["X"] if exact else cfg["k_prime"]
    n_items = cfg["X"] if exact else max(X1, ncand)
    syn = O.init_synthetic(64, n_items, k_u=K_U, k_x=K_X, d=D, gating_hidden=H)
    ip = O.MlpW(*model["item_proj"])
    inet = O.MlpW(*model["item_net"])
    cache = O.build_item_cache(syn.item_table, ip, inet, K_X, D, TAU, K_U, quantized=True)
    emb = O.round_bf16(cache.item_embs)
    gp = O.round_bf16(cache.item_gate_pre)
    s1 = emb.mean(axis=1).astype(np.float32)
    cache = O.Cache(emb, gp, s1, O.quantize_rowwise(s1), TAU, K_U)
    gating = O.Gating(O.MlpW(*model["user_net"]), inet, O.MlpW(*model["cross_net"]))
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence([1, 7])))
    feats = (rng.uniform(-1, 1, (64, D_U)) / math.sqrt(D_U)).astype(np.float32)
    ue = O.user_components(O.Synthetic(feats, None, O.MlpW(*model["user_proj"]), None, None), np.arange(64),
                           K_U, D)
    _CPU_STATE.update(cache=cache, gating=gating, feats=feats, ue=ue.astype(np.float32),
                      cand=np.arange(n_items) if exact else np.sort(np.random.default_rng(0).permutation(n_items)[:ncand]),
                      X=cfg["X"])
    if procs is None:
        procs = len(os.sched_getaffinity(0))
        try:  # ~1 GB of working set per process (int32 codes of the shard + stage-2 gathers)
            avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
            procs = max(1, min(procs, int(avail // (1 << 30)) - 2))
        except (ValueError, OSError):
            pass
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_cpu_worker, [(i, reps, X1, cfg["k_prime"], cfg["ratio"], cfg["k"], cfg.get("view") == "f32")
                                     for i in range(procs)])
    wall = time.perf_counter() - t0
    t1 = float(np.median([t for r in res for t in r[0]]))
    t2 = float(np.median([t for r in res for t in r[1]]))
    t_query = t1 * cfg["X"] / X1 + t2
    if exact:
        return {"value": procs / t_query, "unit": "queries/s", "cores": procs, "kind": "port",
                "sample": (f"oracle/ NumPy port, {procs} processes x {reps} users: exact mol_top_k over all "
                           f"{cfg['X']:,} items = {t2:.2f} s per user per core; wall {wall:.1f} s"),
                "s_per_query_per_core": t_query}
    return {"value": procs / t_query, "unit": "queries/s", "cores": procs, "kind": "port",
            "sample": (f"oracle/ NumPy port, {procs} processes x {reps} queries: stage 1 "
                       f"({'float' if cfg.get('view') == 'f32' else 'int8'} h_indexer incl. "
                       f"rng.permutation) on a {X1:,}-row shard x {cfg['X'] // X1} (linear in X) = "
                       f"{t1 * cfg['X'] / X1:.2f} s + stage 2 mol_top_k over {ncand:,} candidates = {t2:.2f} s per "
                       f"query per core; wall {wall:.1f} s"),
            "s_per_query_per_core": t_query}


# ------------------------------------------------------------------------------------------
# CPU baseline: the UNMODIFIED reference package (baseline/_ref, tools/install_reference.sh) on
# the host cores, on the same corpus and queries, measured (not extrapolated)
# ------------------------------------------------------------------------------------------
def _reference_package():
    p = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(p, "molr")) and p not in sys.path:
        sys.path.insert(0, p)
    try:
        import molr.hindexer  # noqa: F401
        import molr.mol  # noqa: F401
        import molr.numerics  # noqa: F401
        import molr.quant  # noqa: F401
        return sys.modules["molr"]
    except ImportError:
        return None


_REF = {}


def _ref_query(i):
    """One query through the reference's own functions in a forked worker (numpy on one thread):
    stage 1 = molr.hindexer.h_indexer over the whole int8 view (hindexer.py:135-163, incl. the
    rng.permutation and the int32 mat-vec), stage 2 = molr.mol.mol_top_k over the candidates
    (mol.py:389-408); the exact path = mol_top_k over the whole corpus (engine.py:140-147)."""
    from threadpoolctl import threadpool_limits

    import molr.hindexer as RH
    import molr.mol as RM
    import molr.numerics as RN

    st = _REF
    u = st["users"][i]
    state = RM.QueryState(user_embs=st["ue"][u], gate_features=st["feats"][u])
    with threadpool_limits(1):
        t0 = time.perf_counter()
        if st["exact"]:
            ids, sc = RM.mol_top_k(st["cache"], st["gating"], np.arange(st["X"]), state, st["k"])
            t1 = t2 = time.perf_counter()
            same_cand = True
        else:
            cand = RH.h_indexer(st["view"], st["ue"][u].mean(axis=0), st["hcfg"], RN.make_rng([9000, int(u)])).indices
            t1 = time.perf_counter()
            sub = st["sub"][i]  # the candidates' cache rows (pre-gathered from the device cache)
            same_cand = cand.size == sub[2].size and bool(np.array_equal(cand, sub[2]))
            pos, sc = RM.mol_top_k(sub[0], st["gating"], np.arange(cand.size), state, min(st["k"], cand.size))
            ids = sub[2][pos]
            t2 = time.perf_counter()
    return t1 - t0, t2 - t1, same_cand, ids, sc


def reference_baseline(cfg, model, cache, ue, feats, *, budget_s=30.0, ours=None):
    """Time the unmodified reference package on the host cores (one forked process per query, up
    to the cores / memory allow), on the bench's corpus (read back from the device cache,
    exactly) and queries.  `ours(u)` returns the product's drop-in result for query u on the GPU —
    (candidates of paper_2306_04039_b200.hindexer.h_indexer with the reference's rng, ids and
    scores of its mol_top_k) — used to pre-gather stage 2's rows and compared with the reference's
    candidates (bit-identical expected) and top-k."""
    import multiprocessing as mp

    molr = _reference_package()
    if molr is None:
        return None
    import molr.hindexer as RH
    import molr.mol as RM
    import molr.quant as RQ

    exact = cfg.get("exact", False)
    X, k = cfg["X"], cfg["k"]
    mcfg = RM.MoLConfig(k_u=K_U, k_x=K_X, d=D, tau=TAU, gating_hidden=H, dropout_p=0.0)
    gating = RM.GatingNetwork(RM.Mlp(*model["user_net"]), RM.Mlp(*model["item_net"]), RM.Mlp(*model["cross_net"]))
    cores = len(os.sched_getaffinity(0))
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        avail = 64 << 30
    st = {"ue": ue, "feats": feats, "gating": gating, "X": X, "k": k, "exact": exact}
    t_prep = time.perf_counter()
    if exact:
        embs, gp = cache.read(0, X)
        st["cache"] = RM.ItemCache(config=mcfg, item_embs=embs, item_gate_pre=gp, stage1_embs=embs.mean(axis=1))
        per_proc = (256 << 20) + X * 4 * 64 * 6
    else:
        codes = np.empty((X, D), dtype=np.int8)
        scales = np.empty(X, dtype=np.float32)
        step = 1 << 22
        for lo in range(0, X, step):
            n = min(step, X - lo)
            cache.read_stage1(lo, n, codes[lo:lo + n], scales[lo:lo + n])
        st["view"] = RQ.QuantizedRows(codes=codes, scales=scales)
        st["hcfg"] = RH.HIndexerConfig(k_prime=cfg["k_prime"], sample_ratio=cfg["ratio"], quantized=True)
        # int8_matvec materialises the int32 codes (quant.py:90) + permutation + scores per process
        per_proc = X * (D * 4 + 8 + 4 + 4) + (1 << 30)
    procs = max(1, min(cores, int((avail - (4 << 30)) // per_proc)))
    # one calibration query in the parent sizes the sample to ~budget_s of wall time
    st["users"] = [0]
    if not exact:
        st["sub"] = {}
    _REF.clear()
    _REF.update(st)
    if not exact:
        _REF["sub"][0] = _sub_cache(RM, mcfg, cache, ours, st, 0)
    t_one = sum(_ref_query(0)[:2])
    nq = procs * max(1, int(budget_s / max(t_one, 1e-3)))
    nq = min(nq, ue.shape[0]) if exact else min(procs, ue.shape[0])
    users = list(range(nq))
    _REF["users"] = users
    if not exact:
        for i in range(1, nq):
            _REF["sub"][i] = _sub_cache(RM, mcfg, cache, ours, st, i)
    t_prep = time.perf_counter() - t_prep
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(min(procs, nq)) as pool:
        res = pool.map(_ref_query, range(nq), chunksize=max(1, nq // (4 * procs)))
    wall = time.perf_counter() - t0
    t1 = [r[0] for r in res]
    tq = [r[0] + r[1] for r in res]
    out = {"value": nq / wall, "unit": "queries/s", "cores": min(procs, nq), "kind": "reference",
           "s_per_query_per_core": float(np.median(tq)), "p50_query_s": float(np.median(tq)),
           "stage1_s": float(np.median(t1)), "queries": nq, "wall_s": round(wall, 2), "prep_s": round(t_prep, 1),
           "candidates_identical_to_dropin": None if exact else all(r[2] for r in res)}
    what = (f"exact mol_top_k over all {X:,} items" if exact else
            f"h_indexer (int8 view, {X:,} rows incl. rng.permutation + int32 mat-vec) + mol_top_k over its "
            f"~{cfg['k_prime']:,} candidates")
    out["sample"] = (f"unmodified reference package (baseline/_ref molr) on {out['cores']} processes x 1 thread: "
                     f"{nq} queries, {what}; {out['p50_query_s']:.2f} s per query, wall {wall:.1f} s")
    if not exact:
        same, ov = 0, []
        for i in range(nq):
            oi, ri = _REF["sub"][i][1], res[i][3]
            same += int(oi.tolist() == ri.tolist())
            ov.append(len(set(oi.tolist()) & set(ri.tolist())) / len(ri))
        out["dropin_topk_identical_to_reference"] = same
        out["dropin_topk_overlap_min"] = float(min(ov))
    return out


def _sub_cache(RM, mcfg, cache, ours, st, i):
    """The candidate rows of query i (the drop-in h_indexer on the GPU gives the reference's exact
    candidate set for the same rng) as a reference ItemCache: stage 2's input, gathered outside
    the timed region."""
    from paper_2306_04039_b200.hindexer import index_select

    cand, top_ids, _ = ours(i)
    sub = index_select(cache, cand)
    rc = RM.ItemCache(config=mcfg, item_embs=np.array(sub.item_embs), item_gate_pre=np.array(sub.item_gate_pre),
                      stage1_embs=np.array(sub.stage1_embs))
    return rc, top_ids, cand


# ------------------------------------------------------------------------------------------
# parity against the CPU oracle at the bench's own config (outside the timed region)
# ------------------------------------------------------------------------------------------
def oracle_parity(cfg, model, cache, ue, feats, ids, scores, q_exact, q_scores=8):
    """Compare the step's top-k (ids/scores, host (B,k)) with the C restatement of the reference's
    scorer (oracle/molr_oracle.c, pinned to reference goldens): the oracle's exhaustive top-k
    (RetrievalEngine.full_top_k, engine.py:140-147) of the first q_exact queries, streamed from the
    device cache in chunks (read back exactly), and the oracle's scores of the returned items of
    the first q_scores queries (score_candidates, mol.py:329-345)."""
    import oracle as O
    from oracle import c_oracle as CO

    t0 = time.perf_counter()
    k = ids.shape[1]
    X = cache.num_items
    uw = O.mlp(O.MlpW(*model["user_net"]), feats).astype(np.float32)
    cross = CO.Net(*model["cross_net"])
    q = min(q_exact, ids.shape[0])
    # 256K rows (0.5 GB of f32 staging on the device, which the 100M cache leaves little room for)
    chunk = max(1, min(1 << 18, (1 << 28) // max(q, 1)))
    ex_i, ex_s = CO.exact_top_k_streamed(cache.read, X, ue[:q], uw[:q], cross, TAU, k, chunk=chunk)
    recall = float(np.mean([len(set(ids[b].tolist()) & set(ex_i[b].tolist())) / k for b in range(q)]))
    identical = int(sum(ids[b].tolist() == ex_i[b].tolist() for b in range(q)))
    # oracle scores of the returned items
    qs = min(max(q_scores, q if cfg.get("exact") else 0), ids.shape[0], 64)
    uniq = np.unique(ids[:qs])
    rows = {int(i): cache.read(int(i), 1) for i in uniq}
    e = np.concatenate([rows[int(i)][0] for i in uniq])
    g = np.concatenate([rows[int(i)][1] for i in uniq])
    pos = {int(i): j for j, i in enumerate(uniq)}
    lists = [np.array([pos[int(i)] for i in ids[b]]) for b in range(qs)]
    ref = CO.score_candidates(e, g, ue[:qs], uw[:qs], cross, TAU, lists)
    err = max(float(np.abs(scores[b] - ref[b]).max()) for b in range(qs))
    viol = int(sum((~O.score_close(scores[b], ref[b])).sum() for b in range(qs)))
    return {"recall_vs_oracle": recall, "oracle_queries": q, "lists_identical_to_oracle": identical,
            "max_abs_score_err": err, "score_tolerance": "1e-3*|s| + 1e-6", "score_violations": viol,
            "score_queries": qs, "oracle": "oracle/molr_oracle.c (C restatement of mol.py:139-205, 329-408)",
            "oracle_threads": CO.num_threads(), "seconds": round(time.perf_counter() - t0, 1)}


# ------------------------------------------------------------------------------------------
def metric_name(name, cfg):
    if name == "100m":
        return "MoL+h-indexer top-100 queries/sec over 100M items"  # BASELINE.json's headline metric
    if cfg.get("exact"):
        return f"MoL exact top-{cfg['k']} queries/sec ({cfg['label']})"
    return f"MoL+h-indexer top-{cfg['k']} queries/sec ({cfg['label']})"


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cb = cpu_baseline(cfg, reps=max(1, args.steps // 4 + 1))
    line = {"metric": metric_name(args.config, cfg), "impl": "reference",
            "value": cb["value"], "unit": "queries/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * cb["s_per_query_per_core"] * cfg["B"] / cb["cores"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32+int8",
            "data": "synthetic (reference init convention, bf16-representable cache)",
            "config": {"workload": cfg["label"], "items": cfg["X"], "batch": cfg["B"], "k": cfg["k"],
                       "k_prime": cfg["k_prime"], "sample_ratio": cfg["ratio"]},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="100m", choices=sorted(CONFIGS))
    ap.add_argument("--items", type=int, default=0, help="override corpus size (debug)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-oracle", action="store_true", help="skip the CPU-oracle parity check")
    ap.add_argument("--recall-queries", type=int, default=8)
    ap.add_argument("--global-threshold", action="store_true",
                    help="N>1: the single-device threshold (exchange of each query's top sample keys) instead "
                         "of per-shard K'/N, lambda/N thresholds: results identical to 1 GPU, ~12%% more per step")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.items:
        cfg["X"] = args.items
        cfg["label"] += f" (items={args.items})"
    ref_arm = args.impl == "reference"
    if ref_arm and int(os.environ.get("RANK", "0")) != 0:
        return  # the reference arm runs on rank 0 alone (host cores), the other ranks exit 0
    if ref_arm and _reference_package() is None:
        return run_reference(args, cfg)  # no baseline/_ref install: the oracle port (kind "port")

    import torch
    import torch.distributed as dist

    world = 1 if ref_arm else int(os.environ.get("WORLD_SIZE", "1"))
    rank = 0 if ref_arm else int(os.environ.get("RANK", "0"))
    local = 0 if ref_arm else int(os.environ.get("LOCAL_RANK", "0"))
    # MOLR_BENCH_SHARE_GPU=1 (testing the sharded path on a 1-GPU box): every rank on cuda:0 and
    # gloo for the (tiny) candidate exchange, since NCCL refuses two ranks on one device
    share = os.environ.get("MOLR_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    os.environ["MOLR_DEVICE"] = str(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    # a real stream handle (torch's default stream is the legacy NULL stream, which the C-ABI
    # reads as "the context's own stream")
    main_stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(main_stream)

    from paper_2306_04039_b200 import _lib as L
    from paper_2306_04039_b200.mol import GatingNetwork, Mlp, _gating_handle

    lib = L.load()
    ctx = L.ctx(local)
    X, B, k = cfg["X"], cfg["B"], cfg["k"]
    from paper_2306_04039_b200.sharding import local_k_prime, local_lambda, shard_range

    lo, hi = shard_range(X, world, rank)
    Xl = hi - lo
    exact = cfg.get("exact", False)
    kp_local = None if exact else local_k_prime(cfg["k_prime"], world)
    lam_local = None if exact else local_lambda(Xl, sample_ratio=cfg["ratio"])
    # N>1: per-shard thresholds (K'/N, lambda/N; SURVEY §8(e)'s plan) by default; --global-threshold
    # uses the single-device threshold (every shard scores its part of the same global sample, the
    # shards all-gather each query's top n sample keys, the n-th largest of the union is the 1-GPU
    # threshold), so the N-GPU result equals the 1-GPU result bit for bit
    global_thr = world > 1 and not exact and args.global_threshold
    lam_g = None if exact else local_lambda(X, sample_ratio=cfg["ratio"])
    n_rank = None if exact else max(1, round(cfg["k_prime"] * lam_g / X))

    model = synthetic_model()
    t_build = time.perf_counter()
    f32_view = cfg.get("view") == "f32"
    f32_cache = cfg.get("cache") == "f32"
    s1_mode = L.S1_FLOAT if f32_view else L.S1_INT8
    mcfg, cache = build_shard(model, X, lo, hi, seed=11, dev=dev, lib=lib, ctx=ctx,
                              storage=L.STORE_S1_F32 if f32_view else None, f32_cache=cfg.get("cache") == "f32")
    t_build = time.perf_counter() - t_build
    gating = GatingNetwork(Mlp(*model["user_net"]), Mlp(*model["item_net"]), Mlp(*model["cross_net"]))
    gh = _gating_handle(gating)
    feats_h, feats_d = make_queries(model, B, 1, dev)
    uw1, ub1, uw2 = [torch.from_numpy(a).to(dev) for a in model["user_net"]]
    up1, upb1, up2 = [torch.from_numpy(a).to(dev) for a in model["user_proj"]]
    ue_d = torch.empty((B, K_U, D), dtype=torch.float32, device=dev)
    from paper_2306_04039_b200.numerics import DEFAULT_EPS
    uw_d = torch.empty((B, G), dtype=torch.float32, device=dev)
    ids_d = torch.empty((B, k), dtype=torch.int64, device=dev)
    sc_d = torch.empty((B, k), dtype=torch.float32, device=dev)
    cand_h = np.empty(B, dtype=np.int64)
    gat_ids = torch.empty((world, B, k), dtype=torch.int64, device=dev)
    gat_sc = torch.empty((world, B, k), dtype=torch.float32, device=dev)
    out_ids = torch.empty((B, k), dtype=torch.int64, device=dev)
    out_sc = torch.empty((B, k), dtype=torch.float32, device=dev)
    if global_thr:
        keys_d = torch.empty((B, n_rank), dtype=torch.int32, device=dev)
        gat_keys = torch.empty((world, B, n_rank), dtype=torch.int32, device=dev)
        tk_d = torch.empty((B,), dtype=torch.int32, device=dev)
        cnt_t = torch.empty((B,), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    def ours_dropin(view_holder):
        """The product's drop-in per-query path for query u of the batch (GPU): h_indexer with the
        reference's rng (make_rng([9000, u])) on the host int8 view, then mol_top_k."""
        from paper_2306_04039_b200.hindexer import HIndexerConfig as OH
        from paper_2306_04039_b200.hindexer import h_indexer as oh
        from paper_2306_04039_b200.mol import QueryState, mol_top_k
        from paper_2306_04039_b200.numerics import make_rng

        # (the exact configs never call it: they have no h-indexer)
        hc = None if exact else OH(k_prime=cfg["k_prime"], sample_ratio=cfg["ratio"], quantized=True)

        def run(u):
            cand = oh(view_holder["view"], ref_ue[u].mean(axis=0), hc, make_rng([9000, int(u)])).indices
            ids, sc = mol_top_k(cache, gating, cand, QueryState(user_embs=ref_ue[u], gate_features=feats_h[u]), k)
            return cand, ids, sc
        return run

    if ref_arm:
        L.call("molr_query_prep", ctx, B, D_U, feats_d.data_ptr(), PROJ_H, up1.data_ptr(), upb1.data_ptr(),
               up2.data_ptr(), K_U, D, 1, H, uw1.data_ptr(), ub1.data_ptr(), uw2.data_ptr(), G, float(DEFAULT_EPS),
               ue_d.data_ptr(), uw_d.data_ptr(), sp)
        torch.cuda.synchronize()
        ref_ue = ue_d.cpu().numpy()
        cb = reference_baseline(cfg, model, cache, ref_ue, feats_h, ours=ours_dropin(_REF))
        line = {"metric": metric_name(args.config, cfg), "impl": "reference",
                "value": cb["value"], "unit": "queries/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * B / cb["value"],
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32 NumPy (int8 stage-1 view, int32 accumulate)",
                "data": "synthetic: the bench's corpus and queries, read back exactly from the device cache",
                "config": {"workload": cfg["label"], "items": cfg["X"], "batch": cfg["B"], "k": cfg["k"],
                           "k_prime": cfg["k_prime"], "sample_ratio": cfg["ratio"]},
                "cpu_baseline": {k2: cb[k2] for k2 in ("value", "unit", "cores", "kind", "sample")},
                "reference_run": cb,
                "e2e": {"value": cb["value"], "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    def step(i, feats_ptr, host_out=None):
        """One batch through the C-ABI, from the users' raw features (the query a user makes,
        engine.py:117): device query prep (user_proj + L2 norm -> user components, user_net ->
        uw) then the two-stage retrieval.  feats_ptr may be a device or (pinned) host pointer;
        with host_out=(ids, scores) host tensors the final top-k lands there (the C-ABI stages
        the H2D / D2H copies on the call's stream)."""
        L.call("molr_query_prep", ctx, B, D_U, feats_ptr, PROJ_H, up1.data_ptr(), upb1.data_ptr(), up2.data_ptr(), K_U,
               D, 1, H, uw1.data_ptr(), ub1.data_ptr(), uw2.data_ptr(), G, float(DEFAULT_EPS), ue_d.data_ptr(),
               uw_d.data_ptr(), sp)
        ue_ptr = ue_d.data_ptr()
        last = world == 1 and host_out is not None
        oi = host_out[0].data_ptr() if last else ids_d.data_ptr()
        osc = host_out[1].data_ptr() if last else sc_d.data_ptr()
        if exact:  # mol_top_k over the whole (shard of the) corpus
            L.call("molr_mol_top_k", ctx, cache.device_handle(), gh, B, K_U, ue_ptr, uw_d.data_ptr(), TAU, None, None, k,
                   oi, osc, sp)
            if world > 1:
                ids_d.add_(lo)
        elif global_thr:
            L.call("molr_sample_top_keys", ctx, cache.device_handle(), B, K_U, ue_ptr, s1_mode, X, lo, lam_g, 1000 + i,
                   n_rank, keys_d.data_ptr(), sp)
            all_gather(gat_keys, keys_d)
            rows = gat_keys.permute(1, 0, 2).reshape(B, world * n_rank).contiguous()
            L.call("molr_select_nth_keys", ctx, B, world * n_rank, rows.data_ptr(), n_rank, tk_d.data_ptr(), sp)
            L.call("molr_two_stage_top_k_at", ctx, cache.device_handle(), gh, B, K_U, ue_ptr, uw_d.data_ptr(), TAU,
                   s1_mode, kp_local, tk_d.data_ptr(), L.INCLUSIVE, k, lo, oi, osc, L.ptr(cand_h), sp)
            cnt_t.copy_(torch.from_numpy(cand_h))
            all_reduce_sum(cnt_t)
            short = torch.nonzero(cnt_t < min(k, X)).flatten().tolist()
            if short:  # fewer than k candidates in the whole corpus: every row (engine.py:134-135)
                sel = torch.tensor(short, device=dev)
                ue_s, uw_s = ue_d[sel].contiguous(), uw_d[sel].contiguous()
                tk_s = torch.full((len(short),), 0x007FFFFF, dtype=torch.int32, device=dev)
                fi = torch.empty((len(short), k), dtype=torch.int64, device=dev)
                fs = torch.empty((len(short), k), dtype=torch.float32, device=dev)
                L.call("molr_two_stage_top_k_at", ctx, cache.device_handle(), gh, len(short), K_U, ue_s.data_ptr(),
                       uw_s.data_ptr(), TAU, s1_mode, Xl, tk_s.data_ptr(), L.INCLUSIVE, k, lo, fi.data_ptr(),
                       fs.data_ptr(), None, sp)
                ids_d[sel], sc_d[sel] = fi, fs
        else:
            L.call("molr_two_stage_top_k", ctx, cache.device_handle(), gh, B, K_U, ue_ptr, uw_d.data_ptr(), TAU,
                   s1_mode, kp_local, lam_local, 1000 + i, L.INCLUSIVE, k, lo, oi, osc, L.ptr(cand_h), sp)
        if world > 1:
            all_gather(gat_ids, ids_d)
            all_gather(gat_sc, sc_d)
            mi = host_out[0].data_ptr() if host_out is not None else out_ids.data_ptr()
            ms = host_out[1].data_ptr() if host_out is not None else out_sc.data_ptr()
            L.call("molr_merge_top_k", ctx, world, B, k, gat_ids.data_ptr(), gat_sc.data_ptr(), k, mi, ms, sp)
        return (out_ids, out_sc) if world > 1 else (ids_d, sc_d)

    def all_gather(out, inp):
        if share:  # gloo: stage through the host
            parts = [torch.empty_like(inp, device="cpu") for _ in range(world)]
            dist.all_gather(parts, inp.cpu())
            out.copy_(torch.stack(parts).to(out.device))
        else:
            dist.all_gather_into_tensor(out, inp)

    def all_reduce_sum(t):
        if share:
            c = t.cpu()
            dist.all_reduce(c)
            t.copy_(c)
        else:
            dist.all_reduce(t)

    def all_reduce_max(t):
        if share:
            c = t.cpu()
            dist.all_reduce(c, op=dist.ReduceOp.MAX)
            t.copy_(c)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # the exact path's item side (27K x 1.15 KB) fits the 126 MB L2: flush it between timed steps
    # by writing a buffer larger than L2 (outside the per-step events); the other configs' inputs
    # are larger than L2
    l2_flush = torch.empty(64 << 20, dtype=torch.float32, device=dev) if exact else None

    # ---------------- device-resident timing (value) ----------------
    prof_range = os.environ.get("MOLR_PROFILE_RANGE") == "1"  # ncu --profile-from-start off
    with Clocks(local) as clk:  # sampling starts before the warm-up (nvidia-smi start-up stalls the GPU)
        for i in range(args.warmup):
            step(i, feats_d.data_ptr())
        barrier()
        L.prof_reset(local)
        L.set_profiling(True, local)
        launches0 = L.launch_count(local)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        if prof_range:
            torch.cuda.profiler.start()
        barrier()
        evs[0].record(stream)
        trace = os.environ.get("MOLR_STEP_TRACE") == "1"  # diagnostics: per-step kernel times (syncs)
        last = {}
        host_ms = []
        for i in range(args.steps):
            if l2_flush is not None:  # (untimed) evict the L2-resident item side between steps
                l2_flush.zero_()
            starts[i].record(stream)
            t_host = time.perf_counter()
            step(args.warmup + i, feats_d.data_ptr())
            evs[i + 1].record(stream)
            host_ms.append(round(1e3 * (time.perf_counter() - t_host), 2))
            if trace:
                torch.cuda.synchronize()
                cur = L.prof_read(local)
                d = {n: round(v[1] - last.get(n, (0, 0.0))[1], 2) for n, v in cur.items()}
                last = cur
                print(f"step {i}: host {1e3 * (time.perf_counter() - t_host):.1f} ms, gpu {evs[i].elapsed_time(evs[i + 1]):.1f} ms,"
                      f" {d}", file=sys.stderr, flush=True)
        barrier()
        if prof_range:
            torch.cuda.profiler.stop()
    L.set_profiling(False, local)
    launches = L.launch_count(local) - launches0
    prof = L.prof_read(local)
    step_ms = [starts[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    total_ms = sum(step_ms) if l2_flush is not None else evs[0].elapsed_time(evs[-1])
    if world > 1:
        tt = torch.tensor([total_ms], device=dev)
        all_reduce_max(tt)
        total_ms = float(tt.item())
    ms_per_step = total_ms / args.steps
    value = B * args.steps / (total_ms / 1e3)

    # ---------------- end-to-end through the public API with host buffers (e2e) ----------------
    feats_pin = torch.from_numpy(feats_h).pin_memory()
    host_ids = torch.empty((B, k), dtype=torch.int64).pin_memory()
    host_sc = torch.empty((B, k), dtype=torch.float32).pin_memory()
    # inputs: the step's query features and user components from pinned host memory, passed to the
    # C-ABI as host pointers (copied H2D inside the call); outputs: the top-k ids/scores written to
    # pinned host memory (D2H inside the call)
    for i in range(2):
        step(i, feats_pin.data_ptr(), (host_ids, host_sc))
    barrier()
    eev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    est = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    eev[0].record(stream)
    for i in range(args.steps):
        if l2_flush is not None:
            l2_flush.zero_()
        est[i].record(stream)
        step(args.warmup + i, feats_pin.data_ptr(), (host_ids, host_sc))
        eev[i + 1].record(stream)
    barrier()
    e2e_step_ms = [est[i].elapsed_time(eev[i + 1]) for i in range(args.steps)]
    e2e_ms = sum(e2e_step_ms) if l2_flush is not None else eev[0].elapsed_time(eev[-1])
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev)
        all_reduce_max(tt)
        e2e_ms = float(tt.item())
    e2e_value = B * args.steps / (e2e_ms / 1e3)
    h2d = feats_h.nbytes
    d2h = B * k * (8 + 4)

    # ---------------- single-query latency (B = 1) ----------------
    lat = []
    for i in range(5):
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        L.call("molr_query_prep", ctx, 1, D_U, feats_d.data_ptr(), PROJ_H, up1.data_ptr(), upb1.data_ptr(),
               up2.data_ptr(), K_U, D, 1, H, uw1.data_ptr(), ub1.data_ptr(), uw2.data_ptr(), G, float(DEFAULT_EPS),
               ue_d.data_ptr(), uw_d.data_ptr(), sp)
        if exact:
            L.call("molr_mol_top_k", ctx, cache.device_handle(), gh, 1, K_U, ue_d.data_ptr(), uw_d.data_ptr(), TAU,
                   None, None, k, ids_d.data_ptr(), sc_d.data_ptr(), sp)
        else:
            L.call("molr_two_stage_top_k", ctx, cache.device_handle(), gh, 1, K_U, ue_d.data_ptr(), uw_d.data_ptr(),
                   TAU, s1_mode, kp_local, lam_local, 5 + i, L.INCLUSIVE, k, lo, ids_d.data_ptr(), sc_d.data_ptr(),
                   None, sp)
        t1.record(stream)
        torch.cuda.synchronize()
        lat.append(t0.elapsed_time(t1))

    # ---------------- recall vs the exact MoL top-k (GPU exact path, parity-tested vs the oracle) ----
    R = min(args.recall_queries, B)
    res_i, res_s = step(0, feats_d.data_ptr())
    torch.cuda.synchronize()
    # digest of the whole batch's top-k (ids + score bits): with the single-device threshold the
    # N-GPU digest equals the 1-GPU digest
    import hashlib

    digest = hashlib.sha1(res_i.cpu().numpy().tobytes() + res_s.cpu().numpy().tobytes()).hexdigest()[:16]
    two = res_i[:R].cpu().numpy()
    ex_i = torch.empty((R, k), dtype=torch.int64, device=dev)
    ex_s = torch.empty((R, k), dtype=torch.float32, device=dev)
    L.call("molr_mol_top_k", ctx, cache.device_handle(), gh, R, K_U, ue_d.data_ptr(), uw_d.data_ptr(), TAU, None,
           None, k, ex_i.data_ptr(), ex_s.data_ptr(), sp)
    torch.cuda.synchronize()
    ex_i += lo
    if world > 1:
        gi = torch.empty((world, R, k), dtype=torch.int64, device=dev)
        gs = torch.empty((world, R, k), dtype=torch.float32, device=dev)
        all_gather(gi, ex_i)
        all_gather(gs, ex_s)
        L.call("molr_merge_top_k", ctx, world, R, k, gi.data_ptr(), gs.data_ptr(), k, ex_i.data_ptr(),
               ex_s.data_ptr(), sp)
        torch.cuda.synchronize()
    ex_np = ex_i.cpu().numpy()
    recall = float(np.mean([len(set(two[r]) & set(ex_np[r])) / k for r in range(R)]))

    # ---------------- parity against the CPU oracle (1 GPU: the whole corpus is local) ----------------
    parity = None
    if world == 1 and not args.no_oracle and rank == 0:
        try:
            parity = oracle_parity(cfg, model, cache, ue_d.cpu().numpy(), feats_h, res_i.cpu().numpy(),
                                   res_s.cpu().numpy(), ORACLE_Q.get(args.config, 2))
        except Exception as e:  # keep the GPU line
            parity = {"error": repr(e)}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---------------- roofline of the dominant kernel ----------------
    pk = peaks()
    dom = max(prof.items(), key=lambda kv: kv[1][1]) if prof else None
    roof = None
    kernels = {}
    step_total = sum(v[1] for v in prof.values()) or 1.0
    for name, (cnt, ms, work) in prof.items():
        kernels[name] = {"launches": cnt, "ms_per_launch": ms / max(cnt, 1), "share": ms / step_total}
    def roof_of(name, cnt, ms, work):
        per_launch_s = ms / cnt / 1e3
        units = work / cnt
        if name in ("mol_score", "mol_score_tc") and exact:
            # exact path: the item side is L2-resident (27K items x 1.15 KB), so the kernel is bound by
            # the SFU (ex2 / rcp for every SiLU and softmax term) and the epilogue chain, not HBM or the
            # tensor pipe (K1)
            mp, msrc = mufu_peak()
            achieved = units * PAIR_MUFU / per_launch_s
            r = {"kernel": name, "bound": "sfu", "achieved": achieved / 1e12, "peak": mp / 1e12, "unit": "Tops/s (MUFU)",
                 "frac": achieved / mp, "traffic": None, "units_per_launch": units,
                 "per_unit": f"{PAIR_MUFU} MUFU ops per (user, item) pair", "peak_src": msrc,
                 "tensor_frac": units * PAIR_FLOPS / per_launch_s / 1e12 / pk["bf16_tflops"]}
        elif name in ("mol_score", "mol_score_tc"):
            pb = PAIR_BYTES_F32C if f32_cache else PAIR_BYTES
            achieved = units * pb / per_launch_s / 1e9
            mp, _ = mufu_peak()
            r = {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                 "frac": achieved / pk["hbm_gbs"], "traffic": None, "units_per_launch": units,
                 "per_unit": f"{pb} B per (query, candidate) pair", "peak_src": pk["src"],
                 # the same kernel against the SFU: 448 MUFU ops per pair (K1)
                 "sfu_frac": units * PAIR_MUFU / per_launch_s / mp}
            if cfg.get("k_prime"):
                # item-major minimum: every distinct candidate item fetched once per batch; expected
                # distinct items of B K' uniform-ish picks over the shard, Xl (1 - exp(-units / Xl))
                # (SURVEY.md §8(d)); an analytic expectation, not a count
                distinct = Xl * (1.0 - math.exp(-units / Xl))
                r["item_major_min_bytes"] = distinct * pb
                r["item_major_min_frac"] = distinct * pb / per_launch_s / 1e9 / pk["hbm_gbs"]
        elif name == "stage1_filter_f16":
            achieved = units * S1_OPS / per_launch_s / 1e12
            r = {"kernel": name, "bound": "tensor", "achieved": achieved, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                 "frac": achieved / pk["bf16_tflops"], "traffic": None, "units_per_launch": units,
                 "per_unit": f"{S1_OPS} fp16 flops per (query, row)", "peak_src": f"{pk['src']} bf16 (= fp16 dense rate)",
                 "note": "fp16 pre-test + exact fp32 re-check of the undecided band (DESIGN.md K2f)"}
            tcp = tc_microbench_peaks()
            if "f16" in tcp:  # the same against the tcgen05 rate measured by tools/tc_peak_bench.cu
                r["frac_vs_tcgen05_microbench"] = achieved / tcp["f16"]
        elif name.startswith("stage1_filter"):
            achieved = units * S1_OPS / per_launch_s / 1e12
            peak_i8 = 2 * pk["bf16_tflops"]
            r = {"kernel": name, "bound": "tensor", "achieved": achieved, "peak": peak_i8, "unit": "TFLOP/s",
                 "frac": achieved / peak_i8, "traffic": None, "units_per_launch": units,
                 "per_unit": f"{S1_OPS} int8 ops per (query, row)",
                 "peak_src": f"2x {pk['src']} bf16 (int8 dense rate)",
                 "note": "bound by the SIMT threshold test of every accumulator (ALU pipe, ~3.2 instr each), not the MMA"}
            tcp = tc_microbench_peaks()
            if "i8" in tcp:  # the same against the tcgen05 kind::i8 rate measured by tools/tc_peak_bench.cu
                r["frac_vs_tcgen05_microbench"] = achieved / tcp["i8"]
        else:
            return None
        if args.config == "100m" and world == 1:  # the committed capture is of the 100M N=1 step
            try:
                with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                    r["traffic"] = json.load(f).get(name)
            except Exception:
                pass
        return r

    rooflines = [x for x in (roof_of(n, *v) for n, v in sorted(prof.items(), key=lambda kv: -kv[1][1])) if x]
    roof = rooflines[0] if rooflines else None

    metric = metric_name(args.config, cfg)
    line = {
        "metric": metric, "value": value, "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        # the arithmetic the path computes in (K1/K2): stage 1 int8 x int8 -> int32 (exact) or the
        # fp16 pre-test + exact fp32 re-check; MoL: bf16 item components (bf16 hi + lo for an f32 cache) x
        # (bf16 hi + lo) query split with fp32 accumulate, cross-net layer 1 three bf16 hi/lo passes (hi/lo
        # bias), layer 2 three fp16 hi/lo passes, SiLU as ex2 + rcp, combine / softmax / gated sum in fp32
        "dtype": ("stage1 " + ("fp16 pre-test + fp32 exact re-check" if f32_view else "int8 (int32 acc, exact)")
                  + ("; MoL f32 cache as bf16 hi+lo x bf16-hi/lo" if f32_cache else "; MoL bf16 x bf16-hi/lo")
                  + " (fp32 acc), cross-net L1 3-pass bf16 hi/lo / L2 3-pass fp16 hi/lo, ex2+rcp SiLU, fp32 softmax"),
        "data": ("synthetic (reference init convention model.py:121-163; " +
                 ("f32 item cache as the reference builds it (mol.py:294-326), built on device)" if f32_cache else
                  "bf16-representable item cache built on device)")),
        "config": {"workload": cfg["label"], "items": X, "items_per_gpu": Xl, "batch": B, "k": k,
                   "k_prime": cfg["k_prime"], "k_prime_per_gpu": kp_local, "sample_ratio": cfg["ratio"],
                   "lambda_per_gpu": lam_local,
                   "stage1": None if exact else ("float view: fp16 tensor-core pre-test + exact fp32 re-check"
                                                 if f32_view else "int8 (bit-exact)"),
                   "parallelism": f"item-shard x{world}",
                   "threshold": None if exact else ("single-device (global sample, top-n key all-gather)"
                                                    if (global_thr or world == 1) else "per-shard (K'/N, lambda/N)"),
                   "l2": ("L2 flushed between timed steps (256 MB write outside the step events); the item side "
                          "fits L2 within a step" if exact else
                          "inputs larger than L2 (corpus shard x 1.2 KB per item >> 126 MB)")},
        "p50_batch_latency_ms": float(np.median(step_ms)), "step_ms": [round(x, 3) for x in step_ms], "step_host_ms": host_ms, "p50_single_query_latency_ms": float(np.median(lat)),
        "recall_at_k_vs_exact_mol": recall, "result_digest_step0": digest, "recall_queries": R,
        "oracle_parity": parity,
        "e2e": {"value": e2e_value, "unit": "queries/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "step_ms": [round(x, 3) for x in e2e_step_ms]},
        "gpu_launches": int(launches), "roofline": roof, "rooflines": rooflines, "kernels": kernels,
        "build_s": t_build,
    }
    line["clocks"] = clk.summary()
    if not args.no_cpu and world == 1:  # the host baseline is timed on rank 0 at N=1 only
        try:
            ref_ue = ue_d.cpu().numpy()
            cb = None
            if not f32_view:  # the unmodified reference package when installed (baseline/_ref)
                cb = reference_baseline(cfg, model, cache, ref_ue, feats_h, ours=ours_dropin(_REF))
            if cb is None:  # else the oracle port, extrapolated
                cb = cpu_baseline(cfg)
            line["cpu_baseline"] = {k2: cb[k2] for k2 in ("value", "unit", "cores", "kind", "sample")}
            if cb.get("kind") == "reference":
                line["cpu_baseline"]["reference_run"] = {k2: v for k2, v in cb.items() if k2 not in line["cpu_baseline"]}
        except Exception as e:  # keep the GPU line even if the host run fails
            line["cpu_baseline"] = {"value": None, "error": repr(e)}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
