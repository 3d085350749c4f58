"""Per-rank DP-KFAC checkpoints in the reference's ``KFACLAB\\0`` v1 file layout.

Layout (kfaclab trainer.py:35-36, 249-271 write / 274-296 read):

    b"KFACLAB\\0" | u32 LE version (1) | u64 LE header length | header JSON
    (sort_keys) | every array as little-endian float64, C order, in header order

with header ``{"meta": {iteration, epoch, algorithm, workers, factor_states},
"arrays": [{"name", "shape", "dtype": "<f8"}, ...]}`` and arrays sorted by
name: ``layer{i}/weight`` (the [W | b] matrix, bias last, model.py:250),
``layer{i}/momentum`` and ``worker{p}/layer{i}/{a_cov, g_cov, a_damped_inv,
g_damped_inv, a_eig_q, a_eig_v, g_eig_q, g_eig_v}`` (trainer.py:218-246).

The reference's cluster lives in one process, so one file holds every
worker's factor states.  Here each rank owns only its layers (DP-KFAC), so
each rank writes ITS file -- same layout, its own ``worker{rank}/...`` prefixes
-- and ``merge`` concatenates the per-rank files into the reference's
whole-cluster file.  ``exact_factors=True`` additionally stores the held
inverse factors X = L^-1 (``a_inv_factor``/``g_inv_factor``) so an inverse-mode
run resumes bit-exactly; the reference reader ignores unknown arrays
(trainer.py:311-324 looks names up).  Pure host code (file I/O is not on the
GPU path).
"""

from __future__ import annotations

import json
import os
import struct
from pathlib import Path
from typing import Optional

import numpy as np

from .errors import ArgumentError, DataFormatError

MAGIC = b"KFACLAB\0"
VERSION = 1


def encode(meta: dict, arrays: dict) -> bytes:
    """Header + payload bytes exactly as trainer.save_checkpoint builds them."""
    names = sorted(arrays)
    header = {"meta": meta,
              "arrays": [{"name": n, "shape": list(np.shape(arrays[n])), "dtype": "<f8"} for n in names]}
    blob = json.dumps(header, sort_keys=True).encode()
    out = bytearray()
    out += MAGIC
    out += struct.pack("<I", VERSION)
    out += struct.pack("<Q", len(blob))
    out += blob
    for n in names:
        out += np.ascontiguousarray(arrays[n], dtype="<f8").tobytes()
    return bytes(out)


def decode(data: bytes, path: str = "<bytes>"):
    """-> (meta, arrays); errors worded like trainer.load_checkpoint."""
    if data[:8] != MAGIC:
        raise DataFormatError(f"{path}: bad checkpoint magic at byte offset 0")
    version = struct.unpack("<I", data[8:12])[0]
    if version != VERSION:
        raise DataFormatError(f"{path}: unsupported checkpoint version {version}")
    header_len = struct.unpack("<Q", data[12:20])[0]
    header = json.loads(data[20:20 + header_len].decode())
    offset = 20 + header_len
    arrays = {}
    for entry in header["arrays"]:
        shape = tuple(entry["shape"])
        count = int(np.prod(shape)) if shape else 1
        nbytes = count * 8
        if offset + nbytes > len(data):
            raise DataFormatError(f"{path}: truncated array data at byte offset {offset}")
        arrays[entry["name"]] = np.frombuffer(data, dtype="<f8", count=count, offset=offset).reshape(shape).copy()
        offset += nbytes
    return header["meta"], arrays


def write(path, meta: dict, arrays: dict):
    path = Path(path)
    tmp = path.with_name(path.name + ".tmp")
    tmp.write_bytes(encode(meta, arrays))
    os.replace(tmp, path)  # atomic, like trainer.atomic_write_bytes


def read(path):
    return decode(Path(path).read_bytes(), str(path))


def merge(paths, out_path=None):
    """Per-rank files -> the reference's whole-cluster checkpoint (weights and
    momentum from the first file; every rank's worker{p}/ entries)."""
    metas, arrs = zip(*(read(p) for p in paths))
    meta = dict(metas[0])
    meta["factor_states"] = {}
    arrays = {}
    for m, a in zip(metas, arrs):
        meta["factor_states"].update(m["factor_states"])
        for k, v in a.items():
            if k.startswith("worker") or k not in arrays:
                arrays[k] = v
    if out_path is not None:
        write(out_path, meta, arrays)
    return meta, arrays


# ------------------------------------------------------------------ DPKFAC <-> file
def _wb(ly):
    w = ly.module.weight.detach().reshape(ly.d_out, -1).double().cpu().numpy()
    if ly.has_bias:
        w = np.hstack([w, ly.module.bias.detach().double().cpu().numpy()[:, None]])
    return w


def _momentum(ly, optimizer):
    if optimizer is None:
        return np.zeros((ly.d_out, ly.d_in))
    st = optimizer.state.get(ly.module.weight, {})
    mw = st.get("momentum_buffer")
    m = mw.detach().reshape(ly.d_out, -1).double().cpu().numpy() if mw is not None else np.zeros((ly.d_out, ly.d_in - ly.has_bias))
    if ly.has_bias:
        mb = optimizer.state.get(ly.module.bias, {}).get("momentum_buffer")
        mb = mb.detach().double().cpu().numpy() if mb is not None else np.zeros(ly.d_out)
        m = np.hstack([m, mb[:, None]])
    return m


def save(path, kf, optimizer=None, iteration: Optional[int] = None, epoch: int = 0,
         algorithm: str = "dp_kfac", exact_factors: bool = True):
    """Write this rank's checkpoint of ``kf`` (a DPKFAC) in the v1 layout."""
    sd = kf.state_dict()
    arrays, fmeta = {}, {}
    for ly in kf.layers:
        arrays[f"layer{ly.index}/weight"] = _wb(ly)
        arrays[f"layer{ly.index}/momentum"] = _momentum(ly, optimizer)
    names = ("a_cov", "g_cov", "a_damped_inv", "g_damped_inv", "a_eig_q", "a_eig_v", "g_eig_q", "g_eig_v")
    if exact_factors:
        names += ("a_inv_factor", "g_inv_factor")
    for i, d in sd["layers"].items():
        prefix = f"worker{kf.rank}/layer{i}"
        fmeta[prefix] = {"initialized": bool(d["initialized"]),
                         "last_factor_update": int(d["last_factor_update"]),
                         "last_inverse_update": int(d["last_inverse_update"])}
        for n in names:
            if n in d:
                arrays[f"{prefix}/{n}"] = d[n].double().cpu().numpy()
    meta = {"iteration": int(kf.t if iteration is None else iteration), "epoch": int(epoch),
            "algorithm": algorithm, "workers": int(kf.world), "factor_states": fmeta}
    write(path, meta, arrays)
    return meta


def load(path, kf, optimizer=None, restore_weights: bool = True, algorithm: str = "dp_kfac"):
    """Restore ``kf`` (this rank's factor states), and optionally the model
    weights and SGD momentum, from a v1 checkpoint (trainer.restore_cluster,
    trainer.py:299-324).  Accepts a per-rank file or a merged cluster file."""
    import torch
    from .errors import OrderingError
    if kf.assignment is None:
        raise OrderingError("the balanced assignment is fixed at the first step(); load after it "
                            "or pass the checkpoint's assignment explicitly")
    meta, arrays = read(path)
    if meta["algorithm"] != algorithm or meta["workers"] != kf.world:
        raise ArgumentError("checkpoint was produced with a different algorithm/worker configuration")
    dev = kf.device
    if restore_weights:
        with torch.no_grad():
            for ly in kf.layers:
                w = torch.from_numpy(arrays[f"layer{ly.index}/weight"]).float().to(dev)
                k = ly.d_in - ly.has_bias
                ly.module.weight.copy_(w[:, :k].reshape(ly.module.weight.shape))
                if ly.has_bias:
                    ly.module.bias.copy_(w[:, k])
                if optimizer is not None and f"layer{ly.index}/momentum" in arrays:
                    m = torch.from_numpy(arrays[f"layer{ly.index}/momentum"]).float().to(dev)
                    buf = torch.empty_like(ly.module.weight)
                    buf.copy_(m[:, :k].reshape(ly.module.weight.shape))
                    optimizer.state[ly.module.weight]["momentum_buffer"] = buf
                    if ly.has_bias:
                        optimizer.state[ly.module.bias]["momentum_buffer"] = m[:, k].clone()
    layers = {}
    for i in kf.assignment[kf.rank]:
        prefix = f"worker{kf.rank}/layer{i}"
        fm = meta["factor_states"].get(prefix)
        if fm is None:
            continue
        d = dict(fm)
        for n in ("a_cov", "g_cov", "a_damped_inv", "g_damped_inv", "a_eig_q", "a_eig_v", "g_eig_q", "g_eig_v",
                  "a_inv_factor", "g_inv_factor"):
            if f"{prefix}/{n}" in arrays:
                d[n] = torch.from_numpy(arrays[f"{prefix}/{n}"]).float()
        layers[i] = d
    kf.load_state_dict({"t": meta["iteration"], "assignment": kf.assignment, "layers": layers})
    return meta
