"""The reference's operator: ``forward(weights, tokens, positions, past, valid)``.

Drop-in for ``kvrerank.model.forward`` (model.py:332-403) -- the function the
reference's operator switch ``_forward_fn(path)`` (reranker.py:146-151)
returns and ``doc_prefill`` / ``_query_block`` / ``score_full`` call once per
sequence.  Same signature, validation and errors (``_check_call``,
model.py:191-224; all-masked input -> zeros, :225-230), same outputs:
``(hidden f32 [T, d] after the final RMSNorm, KVTensorSet f32 [L, KVH, T, HD]
at position_offset = positions[0])``.  One call is one krr_forward over a
single sequence on the device (layer-split mode: every layer runs in full and
the pre-norm residual comes back, then krr_rmsnorm applies the final norm).

``weights`` may be this package's ``DeviceWeights`` / ``RerankModel``, or the
reference's numpy ``Weights`` -- uploaded once per object (``precision``:
"f32" = the f32 CUDA-core debug build, parity 1e-4; "f16"/"bf16" = tensor
cores).  ``past`` may be a host ``KVTensorSet`` or a ``DeviceKV`` page.

Deviation: the past-key mask ``valid[:P]`` must be a non-pad prefix followed by
pads (what every reference caller passes: ``_doc_valid`` enforces trailing
document pads, reranker.py:154-167); other patterns raise ShapeError.
"""

from __future__ import annotations

import weakref

import numpy as np

from . import _lib, engine
from .errors import PositionError, ShapeError
from .model import DeviceWeights, KVTensorSet, RerankModel, torch_dtype

_UPLOADED: dict = {}


def _device_weights(weights, precision: str) -> DeviceWeights:
    if isinstance(weights, DeviceWeights):
        return weights
    if isinstance(weights, RerankModel):
        return weights.weights
    key = (id(weights), precision)
    w = _UPLOADED.get(key)
    if w is None:
        w = DeviceWeights.from_host(weights, precision)
        _UPLOADED[key] = w
        try:
            weakref.finalize(weights, _UPLOADED.pop, key, None)
        except TypeError:          # not weak-referenceable: keep for the process
            pass
    return w


def _check_call(cfg, tokens, positions, past, valid):
    """model.py:191-224 restated (same messages, same error classes)."""
    tokens = np.asarray(tokens, dtype=np.int64)
    positions = np.asarray(positions, dtype=np.int64)
    if tokens.ndim != 1 or tokens.size == 0:
        raise ShapeError("tokens must be a non-empty 1-D sequence")
    if positions.shape != tokens.shape:
        raise ShapeError("positions must match tokens in length")
    if np.any(np.diff(positions) <= 0):
        raise ShapeError("positions must be strictly increasing")
    if tokens.min() < 0 or tokens.max() >= cfg.vocab_size:
        raise ShapeError("token id out of vocabulary range")
    if positions[0] < 0 or positions[-1] >= cfg.max_position:
        raise PositionError(
            f"positions [{positions[0]}, {positions[-1]}] exceed "
            f"max_position {cfg.max_position}")
    P = 0 if past is None else int(past.token_count)
    if past is not None:
        expected = (cfg.layers, cfg.kv_heads, P, cfg.head_dim)
        shape = tuple(past.shape) if hasattr(past, "pool") else tuple(past.keys.shape)
        if shape != expected:
            raise ShapeError(f"past KV shape {shape} != expected {expected}")
        if P and positions[0] != past.position_offset + P:
            raise ShapeError(
                f"positions must continue the past span: expected start "
                f"{past.position_offset + P}, got {positions[0]}")
    total = P + tokens.size
    if valid is None:
        valid = np.ones(total, dtype=bool)
    else:
        valid = np.asarray(valid, dtype=bool)
        if valid.shape != (total,):
            raise ShapeError(
                f"valid mask must cover past+current tokens ({total}), got {valid.shape}")
    return tokens, positions, P, valid


def forward(weights, tokens, positions, past=None, valid=None, *, precision: str = "f32"):
    """model.py:332-403 ``forward`` on the B200; see the module docstring."""
    import torch
    w = _device_weights(weights, precision)
    cfg = w.config
    tokens, positions, P, valid = _check_call(cfg, tokens, positions, past, valid)
    T = tokens.size
    L, KVH, HD, d = cfg.layers, cfg.kv_heads, cfg.head_dim, cfg.model_dim
    if not valid.any():                                   # model.py:225-230
        shape = (L, KVH, T, HD)
        return (np.zeros((T, d), np.float32),
                KVTensorSet(np.zeros(shape, np.float32), np.zeros(shape, np.float32),
                            int(positions[0])))
    pv = valid[:P]
    vl = int(pv.sum())
    if P and not pv[:vl].all():
        raise ShapeError("past-key mask must be a non-pad prefix followed by pads "
                         "(trailing document pads, reranker.py:154-167)")
    dev = w.device
    tdt = torch_dtype(w.code)
    with engine.device_lock(dev):
        tok = torch.as_tensor(tokens.astype(np.int32), device=dev).view(1, T)
        tv = torch.as_tensor(valid[P:].astype(np.uint8), device=dev).view(1, T)
        pos = torch.as_tensor(positions.astype(np.int32), device=dev)
        cur = torch.empty((1, L, 2, KVH, T, HD), dtype=tdt, device=dev)
        cur_ptrs = torch.tensor([cur.data_ptr()], dtype=torch.int64, device=dev)
        pre = pre_ptrs = pre_valid = None
        if P:
            if hasattr(past, "pool") and past.pool.code == w.code:
                pre = past.pool.slab                      # DeviceKV: read the page in place
                pre_ptrs = past.pool.slot_ptrs([past.slot])
            else:
                if hasattr(past, "pool"):
                    past = past.to_host()
                kv = np.stack([np.asarray(past.keys, np.float32),
                               np.asarray(past.values, np.float32)], axis=1)
                pre = torch.from_numpy(np.ascontiguousarray(kv)).to(dev).to(tdt).view(
                    1, L, 2, KVH, P, HD)
                pre_ptrs = torch.tensor([pre.data_ptr()], dtype=torch.int64, device=dev)
            pre_valid = torch.tensor([vl], dtype=torch.int32, device=dev)
        x = torch.empty((T, d), dtype=torch.float32, device=dev)
        engine.run_forward(w, tok, tv, int(positions[0]), P, pre_valid, pre_ptrs, cur_ptrs, L,
                           prefix_pool=pre, cur_pool=cur, x_out=x, positions=pos)
        hidden = torch.empty_like(x)
        stream = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(_lib.lib().krr_rmsnorm(x.data_ptr(), w.final_gain.data_ptr(), T, d, _lib.F32,
                                          hidden.data_ptr(), stream))
        kv = cur[0].float().cpu().numpy()
        h = hidden.cpu().numpy()
    return h, KVTensorSet(np.ascontiguousarray(kv[:, 0]), np.ascontiguousarray(kv[:, 1]),
                          int(positions[0]))


def forward_fn(precision: str = "f32"):
    """A ``_forward_fn(path)``-compatible callable bound to a precision."""
    def fwd(weights, tokens, positions, past=None, valid=None):
        return forward(weights, tokens, positions, past=past, valid=valid, precision=precision)
    return fwd
