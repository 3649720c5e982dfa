"""Paged KV storage: an HBM pool plus a pinned host-DRAM tier.

HBM layout (one slab, allocated once):

    pool[slot][layer][K|V][kv_head][token][head_dim]   (16-bit, or f32 debug)

One slot holds one document chunk's whole fixed-length cache (the static
[doc | query] layout of reranker.py:1-16 makes every chunk the same size), so
the page table is simply ``chunk_id -> slot``.  Kernels receive per-pair slot
base pointers (device int64 array) and index ``layer``/``kv_head`` inside.
The per-(layer, K|V, kv_head) page is ``D*HD`` contiguous elements, the same
order as the reference's HRKV payload (codec.py:8-9), so HRKV import/export
is a straight cast.

HostKVTier is the stand-in for the paper's SSD tier:
same slot layout in pinned host memory, streamed into an HBM staging pool
with cudaMemcpyAsync on a side stream, event-gated against compute.
"""

from __future__ import annotations

import threading

import numpy as np

from . import _lib
from .config import ModelConfig
from .errors import ShapeError, StoreError
from .model import torch_dtype


def to_device(arr, device, dtype=None):
    """Host array -> device tensor without a stream synchronisation: staged
    through pinned memory and copied non-blocking (a pageable source makes
    torch block the host until the stream drains, which serialises host-side
    scheduling with device work, e.g. between host-tier groups)."""
    import torch
    t = torch.from_numpy(np.ascontiguousarray(arr))
    if dtype is not None:
        t = t.to(dtype)
    if torch.device(device).type != "cuda":
        return t.to(device)
    return t.pin_memory().to(device, non_blocking=True)


class KVPool:
    def __init__(self, config: ModelConfig, document_len: int, capacity: int,
                 dtype: str = "f16", device=None):
        import torch
        if capacity < 1:
            raise StoreError("pool capacity must be >= 1")
        self.config = config
        self.document_len = document_len
        self.capacity = capacity
        self.dtype = dtype
        self.code = _lib.DTYPE_CODES[dtype]
        self.device = torch.device(device if device is not None else "cuda")
        L, KVH, HD = config.layers, config.kv_heads, config.head_dim
        self.page_shape = (L, 2, KVH, document_len, HD)
        self.slab = torch.empty((capacity, *self.page_shape), dtype=torch_dtype(self.code),
                                device=self.device)
        self.slot_elems = int(np.prod(self.page_shape))
        self.slot_bytes = self.slot_elems * self.slab.element_size()
        self.valid_len = torch.zeros(capacity, dtype=torch.int32, device=self.device)
        self._valid_host = np.zeros(capacity, dtype=np.int64)
        self._by_id: dict[str, int] = {}
        self._id_of: dict[int, str] = {}
        self._free = list(range(capacity - 1, -1, -1))
        self._owned: set[int] = set()
        self._lock = threading.Lock()
        self.generation = 0

    def grow(self, capacity: int, min_capacity: int | None = None) -> None:
        """Re-home the slab with more slots (slot ids and handles stay valid).

        The copy needs old + new slab at once, so the target is clamped to what
        the device can hold (keeping 1 GiB of headroom); below ``min_capacity``
        (default: ``capacity``) it fails with StoreError instead of driving the
        device out of memory.  Pointers into the old slab (CUDA graphs, cached
        pointer tables) are invalidated; ``generation`` counts re-homes."""
        import torch
        with self._lock:
            if capacity <= self.capacity:
                return
            need = capacity if min_capacity is None else max(min_capacity, self.capacity + 1)
            free, _ = torch.cuda.mem_get_info(self.device)
            fits = self.capacity + max(0, (free - (1 << 30)) // self.slot_bytes)
            if fits < need:
                raise StoreError(
                    f"KV pool full ({self.capacity} slots of {self.slot_bytes} B); growing to "
                    f"{need} slots needs {(need - self.capacity) * self.slot_bytes >> 20} MiB "
                    f"more than the {free >> 20} MiB free on {self.device}")
            capacity = int(min(capacity, fits))
            slab = torch.empty((capacity, *self.page_shape), dtype=self.slab.dtype,
                               device=self.device)
            slab[:self.capacity].copy_(self.slab)
            vl = torch.zeros(capacity, dtype=torch.int32, device=self.device)
            vl[:self.capacity].copy_(self.valid_len)
            hv = np.zeros(capacity, dtype=np.int64)
            hv[:self.capacity] = self._valid_host
            self._free = list(range(capacity - 1, self.capacity - 1, -1)) + self._free
            self.slab, self.valid_len, self._valid_host = slab, vl, hv
            self.capacity = capacity
            self.generation += 1

    @property
    def free_slots(self) -> int:
        return len(self._free)

    # ---------------------------------------------------------- page table
    def __len__(self) -> int:
        """Slots in use: page-table entries plus caller-owned slots."""
        return len(self._by_id) + len(self._owned)

    def __contains__(self, chunk_id: str) -> bool:
        return chunk_id in self._by_id

    def allocate(self, chunk_ids) -> np.ndarray:
        """Slots for new chunk ids (an existing id keeps its slot, like a put)."""
        with self._lock:
            out = np.empty(len(chunk_ids), dtype=np.int64)
            for i, cid in enumerate(chunk_ids):
                slot = self._by_id.get(cid)
                if slot is None:
                    if not self._free:
                        raise StoreError(f"KV pool full ({self.capacity} slots)")
                    slot = self._free.pop()
                    self._by_id[cid] = slot
                    self._id_of[slot] = cid
                out[i] = slot
            return out

    def release(self, chunk_id: str) -> None:
        with self._lock:
            slot = self._by_id.pop(chunk_id, None)
            if slot is not None:
                self._id_of.pop(slot, None)
                self._free.append(slot)

    def allocate_owned(self, n: int) -> np.ndarray:
        """n slots outside the page table, owned by the caller (e.g. a
        DeviceKV lease) and returned with ``free_owned``."""
        with self._lock:
            if len(self._free) < n:
                raise StoreError(f"KV pool full ({self.capacity} slots)")
            out = np.array([self._free.pop() for _ in range(n)], dtype=np.int64)
            self._owned.update(int(s) for s in out)
            return out

    def free_owned(self, slots) -> None:
        with self._lock:
            for s in np.atleast_1d(np.asarray(slots, dtype=np.int64)):
                s = int(s)
                if s in self._owned:
                    self._owned.discard(s)
                    self._free.append(s)

    @property
    def entries(self) -> int:
        """Page-table entries (keyed slots)."""
        return len(self._by_id)

    @property
    def owned(self) -> int:
        return len(self._owned)

    def lookup(self, chunk_ids) -> np.ndarray:
        """chunk ids -> slots (-1 for a miss)."""
        return np.array([self._by_id.get(c, -1) for c in chunk_ids], dtype=np.int64)

    def chunk_ids(self) -> list[str]:
        return sorted(self._by_id)

    def slot_ptrs(self, slots):
        """Device int64 tensor of slot base addresses for the kernels."""
        import torch
        s = slots if isinstance(slots, torch.Tensor) else to_device(
            np.asarray(slots, dtype=np.int64), self.device)
        s = s.to(torch.int64)
        return s * self.slot_bytes + self.slab.data_ptr()

    def set_valid_len(self, slots, valid_len) -> None:
        import torch
        slots = np.asarray(slots, dtype=np.int64)
        vl = np.asarray(valid_len, dtype=np.int64)
        self._valid_host[slots] = vl
        self.valid_len[to_device(slots, self.device)] = to_device(vl, self.device, torch.int32)

    def host_valid_len(self, slot: int) -> int:
        return int(self._valid_host[slot])

    # ---------------------------------------------------------- host I/O
    def write_host_kv(self, slot: int, keys: np.ndarray, values: np.ndarray,
                      valid_len: int) -> None:
        """Store f32 [L, KVH, D, HD] keys/values (e.g. a decoded HRKV entry)."""
        import torch
        L, _, KVH, D, HD = self.page_shape
        if keys.shape != (L, KVH, D, HD) or values.shape != keys.shape:
            raise ShapeError(f"cached KV shape {keys.shape} does not match pool "
                             f"{(L, KVH, D, HD)}")
        page = np.stack([np.asarray(keys, np.float32), np.asarray(values, np.float32)], axis=1)
        self.slab[slot].copy_(torch.from_numpy(np.ascontiguousarray(page)).to(
            self.device, non_blocking=False).to(self.slab.dtype))
        self.set_valid_len([slot], [valid_len])

    def read_host_kv(self, slot: int):
        """(keys, values) as f32 numpy [L, KVH, D, HD]."""
        page = self.slab[slot].float().cpu().numpy()
        return np.ascontiguousarray(page[:, 0]), np.ascontiguousarray(page[:, 1])


class PinnedRows:
    """``n`` rows of ``row_shape`` in pinned host memory, allocated in chunks of
    at most ``chunk_bytes`` (a tier larger than HBM -- hundreds of GB -- is not
    one cudaHostAlloc).  ``rows[h]`` is row h as a tensor view."""

    def __init__(self, n: int, row_shape, dtype, chunk_bytes: int = 4 << 30):
        import torch
        self.n, self.row_shape, self.dtype = n, tuple(row_shape), dtype
        row_bytes = int(np.prod(row_shape)) * torch.empty((), dtype=dtype).element_size()
        self.per_chunk = max(1, min(n, chunk_bytes // max(row_bytes, 1)))
        self.chunks = []
        for c0 in range(0, n, self.per_chunk):
            rows = min(self.per_chunk, n - c0)
            self.chunks.append(torch.empty((rows, *self.row_shape), dtype=dtype,
                                           pin_memory=True))
        self.nbytes = n * row_bytes

    def __getitem__(self, h: int):
        if not 0 <= h < self.n:
            raise IndexError(h)
        return self.chunks[h // self.per_chunk][h % self.per_chunk]


class HostKVTier:
    """Pinned host-DRAM tier with the pool's slot layout, streamed into an HBM
    staging pool on a side stream (cudaMemcpyAsync via torch copy_).

    ``quant="int8"|"int4"`` stores pages in the HRKV quantised form instead
    (codec.py:58-115: per-(kv_head, channel) scales, one tensor per (layer,
    K|V)): the GPU quantises on put (krr_quant_pages, bit-identical to the
    host codec), 2x / 4x fewer bytes cross PCIe, and the staging copy is
    expanded back to 16-bit by krr_dequant_pages on the copy stream."""

    BITS = {None: 16, "int8": 8, "int4": 4}

    def __init__(self, pool_like: KVPool, capacity: int, quant: str | None = None):
        import torch
        if quant not in self.BITS:
            raise StoreError(f"unknown host-tier quantisation {quant!r}")
        self.page_shape = pool_like.page_shape
        self.dtype = pool_like.slab.dtype
        self.code = pool_like.code
        self.capacity = capacity
        self.quant = quant
        L, _, KVH, D, HD = self.page_shape
        self.n_tensors, self.tensor_elems = 2 * L, KVH * D * HD
        if quant is None:
            self.slab = PinnedRows(capacity, self.page_shape, self.dtype)
            self.slot_bytes = pool_like.slot_bytes
        else:
            bits = self.BITS[quant]
            tb = self.tensor_elems if bits == 8 else (self.tensor_elems + 1) // 2
            self.code_bytes = self.n_tensors * tb
            self.scale_elems = self.n_tensors * KVH * HD
            self.codes = PinnedRows(capacity, (self.code_bytes,), torch.uint8)
            self.scales = PinnedRows(capacity, (self.scale_elems,), torch.float32)
            self.slot_bytes = self.code_bytes + 4 * self.scale_elems   # bytes over PCIe
        self.valid_len = np.zeros(capacity, dtype=np.int64)
        self._by_id: dict[str, int] = {}
        self._next = 0
        self._dev = {}

    @property
    def bits(self) -> int:
        return self.BITS[self.quant]

    def _device_bufs(self, device, n: int):
        """Device landing buffers for n quantised pages (codes, scales)."""
        import torch
        key = (str(device), n)
        if key not in self._dev:
            self._dev = {key: (torch.empty((n, self.code_bytes), dtype=torch.uint8, device=device),
                               torch.empty((n, self.scale_elems), dtype=torch.float32,
                                           device=device))}
        return self._dev[key]

    def put_from_pool(self, chunk_id: str, pool: KVPool, slot: int) -> int:
        if chunk_id not in self._by_id:
            if self._next >= self.capacity:
                raise StoreError("host tier full")
            self._by_id[chunk_id] = self._next
            self._next += 1
        h = self._by_id[chunk_id]
        if self.quant is None:
            self.slab[h].copy_(pool.slab[slot])
        else:
            import torch
            codes, scales = self._device_bufs(pool.device, 1)
            L_, KVH, D, HD = self.page_shape[0], *self.page_shape[2:]
            stream = torch.cuda.current_stream(pool.device).cuda_stream
            _lib.check(_lib.lib().krr_quant_pages(
                pool.slab[slot].data_ptr(), pool.code, self.n_tensors, KVH, D, HD, self.bits,
                codes.data_ptr(), scales.data_ptr(), stream))
            self.codes[h].copy_(codes[0])
            self.scales[h].copy_(scales[0])
        self.valid_len[h] = pool.host_valid_len(slot)
        return h

    def copy_in(self, h: int, staging: KVPool, s: int, k: int = 0) -> None:
        """Queue the H2D transfer of host page h into staging slot s on the
        current stream (plus the dequant kernel for a quantised tier; k picks
        the device landing buffer)."""
        self.h2d(h, staging, s, k)
        self.expand(staging, s, k)

    def h2d(self, h: int, staging: KVPool, s: int, k: int = 0) -> None:
        """The PCIe half of copy_in: page h -> staging slot s (16-bit tier) or
        -> landing buffer k (quantised tier), on the current stream."""
        if self.quant is None:
            staging.slab[s].copy_(self.slab[h], non_blocking=True)
            return
        codes, scales = self._device_bufs(staging.device, staging.capacity)
        codes[k].copy_(self.codes[h], non_blocking=True)
        scales[k].copy_(self.scales[h], non_blocking=True)

    def expand(self, staging: KVPool, s: int, k: int = 0) -> None:
        """The HBM half of copy_in: dequantise landing buffer k into staging
        slot s on the current stream (no-op for a 16-bit tier)."""
        if self.quant is None:
            return
        import torch
        codes, scales = self._device_bufs(staging.device, staging.capacity)
        KVH, D, HD = self.page_shape[2:]
        stream = torch.cuda.current_stream(staging.device).cuda_stream
        _lib.check(_lib.lib().krr_dequant_pages(
            codes[k].data_ptr(), scales[k].data_ptr(), self.bits, self.n_tensors, KVH, D, HD,
            staging.code, staging.slab[s].data_ptr(), stream))

    def lookup(self, chunk_ids) -> np.ndarray:
        return np.array([self._by_id.get(c, -1) for c in chunk_ids], dtype=np.int64)

    def __len__(self) -> int:
        """Slots in use: page-table entries plus caller-owned slots."""
        return len(self._by_id) + len(self._owned)

    def __contains__(self, chunk_id: str) -> bool:
        return chunk_id in self._by_id

    def stream_in(self, host_slots, staging: KVPool, staging_slots, stream) -> None:
        """Queue H2D copies of host pages into staging pool slots on ``stream``."""
        import torch
        with torch.cuda.stream(stream):
            for h, s in zip(host_slots, staging_slots):
                self.copy_in(int(h), staging, int(s), int(s))
        staging.set_valid_len(staging_slots, self.valid_len[np.asarray(host_slots)])


class CodePages:
    """The quantised host tier's device landing buffers seen as attention
    prefix pages: slot k = codes [2L][KVH][D][HD] (INT8, or INT4 low nibble
    first; codec.py:58-115) + scales [2L][KVH][HD] f32, dequantised inside the
    attention kernel (krr_batch_t.prefix_bits / prefix_scales).  Quacks like a
    KVPool for engine.score_slots; valid lengths come from the staging pool."""

    def __init__(self, tier: "HostKVTier", staging: KVPool):
        self.codes, self.scales = tier._device_bufs(staging.device, staging.capacity)
        self.slab = self.codes
        self.bits = tier.bits
        self.code = staging.code
        self.dtype = staging.dtype
        self.document_len = staging.document_len
        self.valid_len = staging.valid_len
        self.slot_bytes = tier.code_bytes

    def slot_ptrs(self, slots_t):
        return slots_t * self.slot_bytes + self.codes.data_ptr()

