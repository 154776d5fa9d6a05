"""Reference-compatible snapshot I/O for item caches, and the device loader.

The on-disk format is the reference's (`snapshot.py:1-16`), restated here so files written by
either side load on the other:

    matrix blob    "MOLR" | version u16 | rows u64 | cols u64 | dtype u8 | payload
                   dtype 0: rows*cols f32;  dtype 1: rows*cols i8 then rows f32 row scales
    container      "MOLC" | version u16 | manifest_len u64 | manifest JSON
                   | (blob_len u64 | MOLR blob) per section
    manifest       {"meta": {...}, "sections": [{"name", "shape", "dtype": "f32"|"i8"}, ...]}

An item cache (`ItemCache.save`, `mol.py:253-273`) has sections item_embs, item_gate_pre,
stage1_embs and optionally stage1_q (i8), meta {"kind": "item_cache", "config": MoLConfig fields}.

Reading memory-maps the file: every section comes back as a zero-copy view, so a 100M-item
snapshot (256 GB of f32) streams into device memory chunk by chunk
(`load_device_item_cache`) without ever being resident on the host.
"""

from __future__ import annotations

import json
import struct
from typing import Mapping

import numpy as np

MATRIX_MAGIC = b"MOLR"
CONTAINER_MAGIC = b"MOLC"
VERSION = 1
DTYPE_F32 = 0
DTYPE_I8_ROWSCALED = 1
_HEADER = struct.Struct("<4sHQQB")


def _blob(arr=None, codes=None, scales=None) -> bytes:
    if codes is not None:
        codes = np.ascontiguousarray(codes, dtype=np.int8)
        scales = np.ascontiguousarray(scales, dtype="<f4")
        if codes.ndim != 2 or scales.shape != (codes.shape[0],):
            raise ValueError("codes must be 2-D with one scale per row")
        return (_HEADER.pack(MATRIX_MAGIC, VERSION, codes.shape[0], codes.shape[1], DTYPE_I8_ROWSCALED)
                + codes.tobytes() + scales.tobytes())
    a = np.ascontiguousarray(arr, dtype="<f4")
    if a.ndim != 2:
        raise ValueError(f"expected 2-D array, got shape {a.shape}")
    return _HEADER.pack(MATRIX_MAGIC, VERSION, a.shape[0], a.shape[1], DTYPE_F32) + a.tobytes()


def _as_2d(a: np.ndarray) -> np.ndarray:
    if a.ndim == 0:
        return a.reshape(1, 1)
    if a.ndim == 1:
        return a.reshape(1, -1)
    return a if a.ndim == 2 else a.reshape(-1, a.shape[-1])


def write_container(path, sections: Mapping[str, object], meta: Mapping | None = None) -> None:
    """Named sections -> container (float arrays as dtype 0 with their original shape in the
    manifest; (codes, scales) pairs as dtype 1), byte-identical to the reference writer."""
    entries, blobs = [], []
    for name, value in sections.items():
        if isinstance(value, tuple):
            codes, scales = value
            blobs.append(_blob(codes=codes, scales=scales))
            entries.append({"name": name, "shape": list(np.shape(codes)), "dtype": "i8"})
        else:
            a = np.asarray(value)
            blobs.append(_blob(_as_2d(a)))
            entries.append({"name": name, "shape": list(a.shape), "dtype": "f32"})
    manifest = json.dumps({"meta": dict(meta or {}), "sections": entries}).encode("utf-8")
    with open(path, "wb") as f:
        f.write(CONTAINER_MAGIC + struct.pack("<H", VERSION) + struct.pack("<Q", len(manifest)) + manifest)
        for b in blobs:
            f.write(struct.pack("<Q", len(b)))
            f.write(b)


def read_container(path):
    """Container -> (sections, meta).  Float sections are read-only memmap views with the
    manifest shape; quantized sections are (codes, scales) memmap views."""
    mm = np.memmap(path, dtype=np.uint8, mode="r")
    if bytes(mm[:4]) != CONTAINER_MAGIC:
        raise ValueError(f"{path}: not a snapshot container")
    (version,) = struct.unpack("<H", bytes(mm[4:6]))
    if version != VERSION:
        raise ValueError(f"unsupported container version {version}")
    (mlen,) = struct.unpack("<Q", bytes(mm[6:14]))
    manifest = json.loads(bytes(mm[14:14 + mlen]).decode("utf-8"))
    off = 14 + mlen
    sections = {}
    for entry in manifest["sections"]:
        (blen,) = struct.unpack("<Q", bytes(mm[off:off + 8]))
        off += 8
        magic, ver, rows, cols, tag = _HEADER.unpack(bytes(mm[off:off + _HEADER.size]))
        if magic != MATRIX_MAGIC:
            raise ValueError(f"bad magic {magic!r}")
        if ver != VERSION:
            raise ValueError(f"unsupported snapshot version {ver}")
        p = off + _HEADER.size
        if tag == DTYPE_F32:
            v = np.ndarray((rows, cols), dtype="<f4", buffer=mm, offset=p)
            sections[entry["name"]] = v.reshape(entry["shape"]) if entry["dtype"] == "f32" else v
        elif tag == DTYPE_I8_ROWSCALED:
            codes = np.ndarray((rows, cols), dtype=np.int8, buffer=mm, offset=p)
            scales = np.ndarray((rows,), dtype="<f4", buffer=mm, offset=p + rows * cols)
            sections[entry["name"]] = (codes, scales)
        else:
            raise ValueError(f"unknown dtype tag {tag}")
        off += blen
    return sections, manifest["meta"]


# ---- item caches -------------------------------------------------------------------------------
def _config_meta(cfg) -> dict:
    return {"k_u": cfg.k_u, "k_x": cfg.k_x, "d": cfg.d, "tau": cfg.tau, "gating_hidden": cfg.gating_hidden,
            "dropout_p": cfg.dropout_p, "l2_normalized": cfg.l2_normalized}


def save_item_cache(cache, path) -> None:
    """ItemCache.save (mol.py:253-273) for a host ItemCache."""
    sections = {"item_embs": cache.item_embs, "item_gate_pre": cache.item_gate_pre,
                "stage1_embs": cache.stage1_embs}
    if cache.stage1_q is not None:
        sections["stage1_q"] = (cache.stage1_q.codes, cache.stage1_q.scales)
    write_container(path, sections, {"kind": "item_cache", "config": _config_meta(cache.config)})


def _open_item_cache(path):
    from paper_2306_04039_b200.mol import MoLConfig

    sections, meta = read_container(path)
    if meta.get("kind") != "item_cache":
        raise ValueError(f"{path}: not an item cache snapshot")
    return MoLConfig(**meta["config"]), sections


def load_item_cache(path):
    """ItemCache.load (mol.py:275-291): a host ItemCache (arrays copied out of the file)."""
    from paper_2306_04039_b200.mol import ItemCache
    from paper_2306_04039_b200.quant import QuantizedRows

    cfg, sec = _open_item_cache(path)
    q = None
    if "stage1_q" in sec:
        codes, scales = sec["stage1_q"]
        q = QuantizedRows(codes=np.array(codes), scales=np.array(scales))
    return ItemCache(config=cfg, item_embs=np.array(sec["item_embs"]), item_gate_pre=np.array(sec["item_gate_pre"]),
                     stage1_embs=np.array(sec["stage1_embs"]), stage1_q=q)


def _bf16_exact(a) -> bool:
    return not np.any(np.ascontiguousarray(a, dtype=np.float32).view(np.uint32) & 0xFFFF)


def load_device_item_cache(path, *, chunk_rows: int = 1 << 18, storage: str = "auto", keep_stage1_f32: bool = True):
    """Stream a snapshot straight into a device-resident cache (DeviceItemCache), chunk by chunk
    from the memory-mapped file.  storage: "auto" picks bf16 for item_embs / item_gate_pre when
    every value is bf16-representable (one scan of the file) and f32 otherwise — lossless either
    way; "bf16" asserts representability per chunk; "f32" always stores f32."""
    from paper_2306_04039_b200 import _lib as L
    from paper_2306_04039_b200.mol import DeviceItemCache

    cfg, sec = _open_item_cache(path)
    embs, gp, s1 = sec["item_embs"], sec["item_gate_pre"], sec["stage1_embs"]
    q = sec.get("stage1_q")
    X = embs.shape[0]
    if storage not in ("auto", "bf16", "f32"):
        raise ValueError(f"storage {storage!r}")
    e_f32 = g_f32 = storage == "f32"
    if storage == "auto":
        e_f32 = any(not _bf16_exact(embs[r:r + chunk_rows]) for r in range(0, X, chunk_rows))
        g_f32 = any(not _bf16_exact(gp[r:r + chunk_rows]) for r in range(0, X, chunk_rows))
    flags = (L.STORE_EMBS_F32 if e_f32 else 0) | (L.STORE_GP_F32 if g_f32 else 0)
    flags |= (L.STORE_S1_F32 if keep_stage1_f32 else 0) | (L.STORE_S1_INT8 if q is not None else 0)
    dev = DeviceItemCache(cfg, X, s1.shape[1], flags)
    for r in range(0, X, chunk_rows):
        n = min(chunk_rows, X - r)
        dev.fill(r, n, item_embs=np.ascontiguousarray(embs[r:r + n], dtype=np.float32),
                 item_gate_pre=np.ascontiguousarray(gp[r:r + n], dtype=np.float32),
                 stage1_embs=np.ascontiguousarray(s1[r:r + n], dtype=np.float32) if keep_stage1_f32 else None,
                 stage1_codes=np.ascontiguousarray(q[0][r:r + n]) if q is not None else None,
                 stage1_scales=np.ascontiguousarray(q[1][r:r + n], dtype=np.float32) if q is not None else None)
    return dev


def save_device_item_cache(dev, path, *, chunk_rows: int = 1 << 18) -> None:
    """Write a device-resident cache (DeviceItemCache, e.g. from build_device_item_cache) as a
    reference-format item-cache container, streaming rows back in chunks (molr_cache_read)."""
    import ctypes as C

    from paper_2306_04039_b200 import _lib as L

    cfg = dev.config
    X, kd, G, d1 = dev.num_items, cfg.k_x * cfg.d, cfg.num_logits, dev.stage1_dim
    storage = C.c_int()
    L.call("molr_cache_info", dev.device_handle(), None, C.byref(storage), None)
    has_s1 = bool(storage.value & L.STORE_S1_F32)
    has_q = bool(storage.value & L.STORE_S1_INT8)
    if not has_s1:
        raise ValueError("saving needs the f32 stage-1 view (build with keep_stage1_f32=True)")
    # blob rows/cols follow the reference's 2-D view (_as_2d: leading dims flattened)
    specs = [("item_embs", [X, cfg.k_x, cfg.d], "f32", X * cfg.k_x, cfg.d), ("item_gate_pre", [X, G], "f32", X, G),
             ("stage1_embs", [X, d1], "f32", X, d1)]
    if has_q:
        specs.append(("stage1_q", [X, d1], "i8", X, d1))
    entries = [{"name": n, "shape": sh, "dtype": dt} for n, sh, dt, _, _ in specs]
    manifest = json.dumps({"meta": {"kind": "item_cache", "config": _config_meta(cfg)}, "sections": entries}).encode()

    def chunks(field):
        for r in range(0, X, chunk_rows):
            n = min(chunk_rows, X - r)
            out = {"item_embs": np.empty((n, kd), np.float32), "item_gate_pre": np.empty((n, G), np.float32),
                   "stage1_embs": np.empty((n, d1), np.float32), "codes": np.empty((n, d1), np.int8),
                   "scales": np.empty(n, np.float32)}
            ptrs = [L.ptr(out["item_embs"]) if field == "item_embs" else None,
                    L.ptr(out["item_gate_pre"]) if field == "item_gate_pre" else None,
                    L.ptr(out["stage1_embs"]) if field == "stage1_embs" else None,
                    L.ptr(out["codes"]) if field in ("codes", "scales") else None,
                    L.ptr(out["scales"]) if field in ("codes", "scales") else None]
            L.call("molr_cache_read", dev.device_handle(), r, n, *ptrs, None)
            yield out[field]

    with open(path, "wb") as f:
        f.write(CONTAINER_MAGIC + struct.pack("<H", VERSION) + struct.pack("<Q", len(manifest)) + manifest)
        for name, _, dt, rows, cols in specs:
            if dt == "f32":
                f.write(struct.pack("<Q", _HEADER.size + rows * cols * 4))
                f.write(_HEADER.pack(MATRIX_MAGIC, VERSION, rows, cols, DTYPE_F32))
                for a in chunks(name):
                    f.write(a.astype("<f4", copy=False).tobytes())
            else:
                f.write(struct.pack("<Q", _HEADER.size + rows * cols + rows * 4))
                f.write(_HEADER.pack(MATRIX_MAGIC, VERSION, rows, cols, DTYPE_I8_ROWSCALED))
                for a in chunks("codes"):
                    f.write(a.tobytes())
                for a in chunks("scales"):
                    f.write(a.astype("<f4", copy=False).tobytes())
