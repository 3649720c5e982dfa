"""KV-store interface (reference store.py:1-324) plus the HBM-paged backend.

The reference routes encoded HRKV entries to one backend per shard by
``centroid_id % num_shards`` (store.py:27-32, 271-324); backends duck-type
``put/get/exists/keys/stats/close`` (store.py:58-177).  This module keeps
that interface unchanged (memory and directory backends; the TCP backend is
out of scope) and adds ``DevicePagedKVStore``, a backend whose
entries live as 16-bit pages of an HBM ``KVPool``:

* ``put`` decodes the HRKV bytes straight into a pool slot on the GPU
  (F32 cast or INT8/INT4 dequant kernel, codec.decode_entry_to_pool);
* ``get`` re-encodes the page as an F32 entry (bytes-in/bytes-out contract;
  values are the 16-bit page widened, so not byte-identical to the input —
  SURVEY §8(b) b2);
* ``lookup(chunk_ids) -> slots`` is what the rerank kernels consume, and
  ``put_from_device`` registers a GPU-prefilled slot without any bytes.

An optional ``HostKVTier`` behind the same keys holds pages in pinned host
DRAM (the paper's SSD tier stand-in) and streams them into HBM on demand.
"""

from __future__ import annotations

import os
import re
import tempfile
import threading
from dataclasses import dataclass
from pathlib import Path

from .errors import ShapeError, StoreError

KEY_RE = re.compile(r"^[A-Za-z0-9._\-]+(/[A-Za-z0-9._\-]+)*$")   # store.py:23
ENTRY_SUFFIX = ".hrkv"


def shard_of(centroid_id: int, num_shards: int) -> int:
    """Placement rule (store.py:27-32)."""
    if num_shards < 1:
        raise StoreError("num_shards must be >= 1")
    if centroid_id < 0:
        raise StoreError("centroid_id must be nonnegative")
    return centroid_id % num_shards


def check_key(key: str) -> str:
    if not KEY_RE.match(key) or ".." in key.split("/"):
        raise StoreError(f"unsafe key {key!r}")
    return key


@dataclass
class StoreStats:
    """Per-backend counters (store.py:35-55), same text form."""

    entries: int = 0
    bytes: int = 0
    gets: int = 0
    puts: int = 0
    bytes_served: int = 0

    def as_text(self) -> str:
        return "".join(f"{k}={getattr(self, k)}\n"
                       for k in ("entries", "bytes", "gets", "puts", "bytes_served"))

    @classmethod
    def from_text(cls, text: str) -> "StoreStats":
        kv = {}
        for line in text.splitlines():
            if line.strip():
                k, _, v = line.partition("=")
                kv[k.strip()] = int(v)
        return cls(**kv)


class _Counted:
    def __init__(self):
        self._lock = threading.Lock()
        self._gets = self._puts = self._served = 0

    def _count_get(self, value):
        with self._lock:
            self._gets += 1
            if value is not None:
                self._served += len(value)


class MemoryBackend(_Counted):
    """Process-local dict backend (store.py:58-97)."""

    def __init__(self):
        super().__init__()
        self._data: dict[str, bytes] = {}

    def put(self, key: str, value: bytes) -> None:
        with self._lock:
            self._data[key] = bytes(value)
            self._puts += 1

    def get(self, key: str):
        with self._lock:
            v = self._data.get(key)
        self._count_get(v)
        return v

    def exists(self, key: str) -> bool:
        with self._lock:
            return key in self._data

    def keys(self) -> list[str]:
        with self._lock:
            return sorted(self._data)

    def stats(self) -> StoreStats:
        with self._lock:
            return StoreStats(len(self._data), sum(map(len, self._data.values())),
                              self._gets, self._puts, self._served)

    def close(self) -> None:
        pass


class DirectoryBackend(_Counted):
    """One file per entry, written to a temp file then renamed into place so a
    reader sees the old or the new bytes, never a mix (store.py:100-177)."""

    def __init__(self, root, create: bool = True):
        super().__init__()
        self.root = Path(root)
        if create:
            self.root.mkdir(parents=True, exist_ok=True)
        elif not self.root.is_dir():
            raise StoreError(f"store root {self.root} does not exist")

    def _path(self, key: str) -> Path:
        return self.root / (check_key(key) + ENTRY_SUFFIX)

    def put(self, key: str, value: bytes) -> None:
        path = self._path(key)
        path.parent.mkdir(parents=True, exist_ok=True)
        fd, tmp = tempfile.mkstemp(dir=path.parent, prefix=".tmp-")
        try:
            with os.fdopen(fd, "wb") as f:
                f.write(value)
            os.replace(tmp, path)
        except OSError as e:
            try:
                os.unlink(tmp)
            except OSError:
                pass
            raise StoreError(f"write failed for {key!r}: {e}") from e
        with self._lock:
            self._puts += 1

    def get(self, key: str):
        try:
            v = self._path(key).read_bytes()
        except FileNotFoundError:
            v = None
        except OSError as e:
            raise StoreError(f"read failed for {key!r}: {e}") from e
        self._count_get(v)
        return v

    def exists(self, key: str) -> bool:
        return self._path(key).exists()

    def keys(self) -> list[str]:
        n = len(ENTRY_SUFFIX)
        return sorted(p.relative_to(self.root).as_posix()[:-n]
                      for p in self.root.rglob("*" + ENTRY_SUFFIX))

    def stats(self) -> StoreStats:
        files = list(self.root.rglob("*" + ENTRY_SUFFIX))
        with self._lock:
            return StoreStats(len(files), sum(p.stat().st_size for p in files), self._gets,
                              self._puts, self._served)

    def close(self) -> None:
        pass


class DevicePagedKVStore(_Counted):
    """Backend whose entries are HBM pool pages.

    Same duck type as the reference backends, plus ``lookup`` (chunk ids ->
    pool slots, -1 for a miss), ``put_from_device`` and ``doc_kv``.  With a
    ``host_tier`` attached, entries evicted from HBM (``spill``) stay
    addressable and are streamed back by ``ensure_resident``."""

    def __init__(self, pool, host_tier=None, export_scheme=None):
        from .codec import QuantScheme
        super().__init__()
        self.pool = pool
        self.host_tier = host_tier
        # scheme of the bytes get() returns: F32 (reference-readable, default)
        # or F16 (the page's own bytes, half the size; this build only)
        self.export_scheme = export_scheme if export_scheme is not None else QuantScheme.F32
        self._entry_bytes: dict[str, int] = {}

    # -- reference duck type
    def put(self, key: str, value: bytes) -> None:
        from .codec import decode_entry_to_pool, parse_entry
        check_key(key)
        v = parse_entry(value)                # reject bad bytes before taking a slot
        L, KVH, D, HD = v.shape
        if (L, 2, KVH, D, HD) != tuple(self.pool.page_shape):
            raise ShapeError(f"entry shape {v.shape} does not match pool {self.pool.page_shape}")
        fresh = key not in self.pool
        slot = int(self.pool.allocate([key])[0])
        try:
            decode_entry_to_pool(value, self.pool, slot)
        except BaseException:
            if fresh:                           # no half-written page stays mapped
                self.pool.release(key)
            raise
        with self._lock:
            self._puts += 1
            self._entry_bytes[key] = len(value)

    def get(self, key: str):
        from .codec import encode_pool_page
        slot = int(self.pool.lookup([key])[0])
        if slot < 0:
            self._count_get(None)
            return None
        data = encode_pool_page(key, self.pool, slot, self.export_scheme)
        self._count_get(data)
        return data

    def exists(self, key: str) -> bool:
        return key in self.pool or (self.host_tier is not None and
                                    self.host_tier.lookup([key])[0] >= 0)

    def keys(self) -> list[str]:
        return self.pool.chunk_ids()

    def stats(self) -> StoreStats:
        n = self.pool.entries
        with self._lock:
            return StoreStats(n, n * self.pool.slot_bytes, self._gets, self._puts, self._served)

    def close(self) -> None:
        pass

    # -- device extensions
    def lookup(self, chunk_ids):
        return self.pool.lookup(chunk_ids)

    def put_from_device(self, chunk_ids, slots) -> None:
        """Register slots a GPU prefill already wrote (no bytes cross PCIe)."""
        with self._lock:
            self._puts += len(chunk_ids)

    def doc_kv(self, chunk_id: str):
        from .reranker import DeviceKV, DocKV
        slot = int(self.pool.lookup([chunk_id])[0])
        if slot < 0:
            return None
        return DocKV(chunk_id, DeviceKV(self.pool, slot), self.pool.host_valid_len(slot))


class ShardedStore:
    """Routes entries to one backend per shard by centroid id (store.py:271-324)."""

    def __init__(self, backends: list):
        if not backends:
            raise StoreError("need at least one shard backend")
        self.backends = list(backends)
        self.num_shards = len(self.backends)

    @classmethod
    def in_memory(cls, num_shards: int) -> "ShardedStore":
        return cls([MemoryBackend() for _ in range(num_shards)])

    @classmethod
    def local(cls, root, num_shards: int, create: bool = True) -> "ShardedStore":
        return cls([DirectoryBackend(Path(root) / f"shard{k}", create=create)
                    for k in range(num_shards)])

    @classmethod
    def remote(cls, address, num_shards: int) -> "ShardedStore":
        raise StoreError("the TCP shard server is out of scope for the B200 build "
                         "(SURVEY.md §2); use in_memory, local or device")

    @classmethod
    def device(cls, pools) -> "ShardedStore":
        """One DevicePagedKVStore per pool (e.g. one per GPU or per precision)."""
        return cls([DevicePagedKVStore(p) for p in pools])

    def shard_for(self, centroid_id: int) -> int:
        return shard_of(centroid_id, self.num_shards)

    def _call(self, centroid_id: int, op: str, *args):
        shard = self.shard_for(centroid_id)
        try:
            return getattr(self.backends[shard], op)(*args)
        except StoreError as e:
            raise StoreError(f"shard {shard}: {e}") from e

    def put_entry(self, chunk_id: str, centroid_id: int, data: bytes) -> None:
        self._call(centroid_id, "put", chunk_id, data)

    def get_entry(self, chunk_id: str, centroid_id: int):
        return self._call(centroid_id, "get", chunk_id)

    def exists_entry(self, chunk_id: str, centroid_id: int) -> bool:
        return self._call(centroid_id, "exists", chunk_id)

    def stats(self) -> list[StoreStats]:
        return [b.stats() for b in self.backends]

    def close(self) -> None:
        for b in self.backends:
            b.close()
