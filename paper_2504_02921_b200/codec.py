"""HRKV cache-entry format (reference codec.py:1-211), with a device import path.

Byte layout (little-endian), identical to the reference so entries written by
``kvrerank build`` load here and vice versa:

    header  <4sHB6H : "HRKV" | version=1 | scheme | layers | kv_heads |
                      document_len | head_dim | valid_len | chunk_id_len
    chunk id bytes (UTF-8)
    [INT8/INT4] f32 scales [kv_heads*head_dim] per (layer, K|V)
    payload [layer][K|V][kv_head][token][channel]  (f32 | int8 | int4 packed)

Host side: ``encode_entry`` / ``decode_entry`` give the reference's exact
bytes and F32 zero-copy views (codec.py:128-211).  Device side:
``decode_entry_to_pool`` moves the payload into an HBM ``KVPool`` slot —
F32 pages are cast on the GPU, INT8/INT4 pages are dequantised by the
``krr_dequant_kv`` kernel (the quantised bytes are what crosses PCIe).
"""

from __future__ import annotations

import enum
import struct

import numpy as np

from .errors import CodecError, FormatError

MAGIC = b"HRKV"
VERSION = 1
HEADER = struct.Struct("<4sHB6H")      # codec.py:29-31


class QuantScheme(enum.Enum):
    """Scheme codes 0/2/3 as in codec.py:34-56.  Code 1 is unused by the
    reference; this build assigns it to F16 (IEEE binary16 payload, the HBM
    pool's own page format, half the bytes of F32, no scales).  The reference
    decoder rejects code 1 (codec.py:170-173), so F16 entries are for stores
    this build reads; export F32/INT8/INT4 for reference interop."""

    F32 = 0
    F16 = 1
    INT8_PER_CHANNEL = 2
    INT4_PER_CHANNEL = 3

    @classmethod
    def from_name(cls, name: str) -> "QuantScheme":
        table = {"F32": cls.F32, "FLOAT32": cls.F32, "F16": cls.F16, "FLOAT16": cls.F16,
                 "HALF": cls.F16, "INT8": cls.INT8_PER_CHANNEL,
                 "KV8": cls.INT8_PER_CHANNEL, "INT4": cls.INT4_PER_CHANNEL,
                 "KV4": cls.INT4_PER_CHANNEL}
        try:
            return table[name.strip().upper()]
        except KeyError:
            raise CodecError(f"unknown quantization scheme {name!r}") from None

    @property
    def short_name(self) -> str:
        return {0: "f32", 1: "f16", 2: "int8", 3: "int4"}[self.value]

    @property
    def bits(self) -> int:
        return {0: 32, 1: 16, 2: 8, 3: 4}[self.value]

    @property
    def quantised(self) -> bool:
        return self.value >= 2

    @property
    def level(self) -> int:
        return {2: 127, 3: 7}[self.value]


def payload_nbytes(layers: int, kv_heads: int, document_len: int, head_dim: int,
                   scheme: QuantScheme) -> int:
    """Payload bytes of one entry, header and scales excluded (codec.py:118-125)."""
    n = kv_heads * document_len * head_dim
    per = {32: 4 * n, 16: 2 * n, 8: n, 4: (n + 1) // 2}[scheme.bits]
    return 2 * layers * per


# ------------------------------------------------------------ quantisation
def quantize_tensor(t: np.ndarray, scheme: QuantScheme) -> tuple[bytes, np.ndarray]:
    """Symmetric per-(head, channel) quantisation of a [heads, tokens, channels]
    f32 tensor (codec.py:58-79): scale = amax/level (1.0 for an all-zero
    channel), code = clamp(round-half-away(t/scale), +-level); INT4 packs two
    codes per byte, low nibble first."""
    if not scheme.quantised:
        raise CodecError(f"{scheme.name} stores raw floats; nothing to quantize")
    t = np.asarray(t, np.float32)
    if t.ndim != 3:
        raise CodecError("expected a [heads, tokens, channels] tensor")
    if not np.isfinite(t).all():
        raise CodecError("non-finite element in tensor")
    lv = np.float32(scheme.level)
    amax = np.max(np.abs(t), axis=1)                                  # [heads, channels]
    scales = np.where(amax == 0, np.float32(1.0), amax / lv).astype(np.float32)
    ratio = t / scales[:, None, :]
    mag = np.floor(np.abs(ratio) + np.float32(0.5))
    codes = np.clip(np.copysign(mag, ratio), -lv, lv).astype(np.int8)
    if scheme is QuantScheme.INT4_PER_CHANNEL:
        return pack_int4(codes.reshape(-1)), scales
    return codes.tobytes(), scales


def pack_int4(codes: np.ndarray) -> bytes:
    low = codes.astype(np.uint8) & np.uint8(0x0F)
    if low.size & 1:
        low = np.append(low, np.uint8(0))
    return (low[0::2] | (low[1::2] << np.uint8(4))).tobytes()


def unpack_int4(data: bytes, count: int) -> np.ndarray:
    if len(data) != (count + 1) // 2:
        raise CodecError(f"int4 payload has {len(data)} bytes, expected {(count + 1) // 2}")
    raw = np.frombuffer(data, np.uint8)
    nib = np.stack([raw & 0x0F, raw >> 4], axis=1).reshape(-1)[:count].astype(np.int8)
    return np.where(nib >= 8, nib - 16, nib).astype(np.int8)


def dequantize_tensor(qdata: bytes, scales: np.ndarray, scheme: QuantScheme,
                      shape: tuple[int, int, int]) -> np.ndarray:
    """code * scale[head, channel] in f32 (codec.py:82-95)."""
    count = int(np.prod(shape))
    if scheme is QuantScheme.INT4_PER_CHANNEL:
        codes = unpack_int4(qdata, count)
    elif scheme is QuantScheme.INT8_PER_CHANNEL:
        if len(qdata) != count:
            raise CodecError(f"int8 payload has {len(qdata)} bytes, expected {count}")
        codes = np.frombuffer(qdata, np.int8)
    else:
        raise CodecError(f"{scheme.name} stores raw floats; nothing to dequantize")
    return codes.reshape(shape).astype(np.float32) * np.asarray(scales, np.float32)[:, None, :]


# ------------------------------------------------------------ entries
class EntryView:
    """Parsed header plus offsets into the entry bytes (no payload copy)."""

    __slots__ = ("data", "scheme", "layers", "kv_heads", "document_len", "head_dim",
                 "valid_len", "chunk_id", "scales_off", "payload_off", "tensor_bytes")

    @property
    def shape(self):
        return (self.layers, self.kv_heads, self.document_len, self.head_dim)

    def scales(self) -> np.ndarray:
        """[layers, 2, kv_heads, head_dim] f32 (quantised schemes)."""
        n = 2 * self.layers * self.kv_heads * self.head_dim
        return np.frombuffer(self.data, "<f4", n, self.scales_off).reshape(
            self.layers, 2, self.kv_heads, self.head_dim)

    def payload(self) -> memoryview:
        return memoryview(self.data)[self.payload_off:]


def parse_entry(data) -> EntryView:
    """Validate an entry and locate its sections (codec.py:160-188)."""
    if len(data) < HEADER.size:
        raise FormatError("entry shorter than header")
    magic, version, code, L, KVH, D, HD, vl, idn = HEADER.unpack_from(data)
    if magic != MAGIC:
        raise FormatError(f"bad magic {magic!r}")
    if version != VERSION:
        raise FormatError(f"unsupported version {version} (this build reads {VERSION})")
    try:
        scheme = QuantScheme(code)
    except ValueError:
        raise FormatError(f"unknown scheme code {code}") from None
    off = HEADER.size
    if len(data) < off + idn:
        raise CodecError("truncated chunk id")
    v = EntryView()
    v.data = data
    v.scheme, v.layers, v.kv_heads, v.document_len, v.head_dim, v.valid_len = \
        scheme, L, KVH, D, HD, vl
    v.chunk_id = bytes(data[off:off + idn]).decode("utf-8")
    off += idn
    n_t = 2 * L
    scale_bytes = KVH * HD * 4 if scheme.quantised else 0
    v.tensor_bytes = payload_nbytes(1, KVH, D, HD, scheme) // 2
    v.scales_off = off
    v.payload_off = off + n_t * scale_bytes
    expected = v.payload_off + n_t * v.tensor_bytes
    if len(data) != expected:
        raise CodecError(f"entry is {len(data)} bytes, expected {expected}")
    return v


def encode_arrays(chunk_id: str, keys: np.ndarray, values: np.ndarray, valid_len: int,
                  scheme: QuantScheme = QuantScheme.F32) -> bytes:
    """Serialise f32 [L, KVH, D, HD] keys/values (codec.py:128-157)."""
    L, KVH, D, HD = keys.shape
    for name, val in (("layers", L), ("kv_heads", KVH), ("document_len", D),
                      ("head_dim", HD), ("valid_len", valid_len)):
        if not 0 <= val <= 0xFFFF:
            raise CodecError(f"{name}={val} does not fit in u16")
    cid = chunk_id.encode("utf-8")
    if len(cid) > 0xFFFF:
        raise CodecError("chunk id longer than u16")
    if not (np.isfinite(keys).all() and np.isfinite(values).all()):
        raise CodecError("non-finite element in KV tensors")
    head = [HEADER.pack(MAGIC, VERSION, scheme.value, L, KVH, D, HD, valid_len, len(cid)), cid]
    if scheme is QuantScheme.F32:
        kv = np.stack([np.asarray(keys, "<f4"), np.asarray(values, "<f4")], axis=1)
        return b"".join(head) + np.ascontiguousarray(kv).tobytes()
    if scheme is QuantScheme.F16:
        kv = np.stack([np.asarray(keys, np.float32), np.asarray(values, np.float32)], axis=1)
        with np.errstate(over="ignore"):
            h = kv.astype("<f2")                          # round to nearest even
        if not np.isfinite(h).all():
            raise CodecError("KV element outside the f16 range")
        return b"".join(head) + np.ascontiguousarray(h).tobytes()
    scales, payload = [], []
    for li in range(L):
        for t in (keys[li], values[li]):
            q, s = quantize_tensor(np.ascontiguousarray(t, np.float32), scheme)
            scales.append(s.astype("<f4").tobytes())
            payload.append(q)
    return b"".join(head + scales + payload)


def encode_entry(doc_kv, scheme: QuantScheme = QuantScheme.F32) -> bytes:
    """Serialise a DocKV (host KVTensorSet or device pool page); identical inputs
    give identical bytes."""
    kv = doc_kv.kv
    if hasattr(kv, "to_host"):
        kv = kv.to_host()
    return encode_arrays(doc_kv.chunk_id, kv.keys, kv.values, doc_kv.valid_len, scheme)


def encode_pool_page(chunk_id: str, pool, slot: int,
                     scheme: QuantScheme = QuantScheme.F32) -> bytes:
    """Serialise an HBM pool page.  F16 from an f16 pool is the page's own
    bytes behind the header (one D2H copy, no f32 round trip); other schemes
    go through f32 arrays as encode_arrays."""
    import torch
    if scheme is QuantScheme.F16 and pool.slab.dtype == torch.float16:
        L, _, KVH, D, HD = pool.page_shape
        cid = chunk_id.encode("utf-8")
        head = HEADER.pack(MAGIC, VERSION, scheme.value, L, KVH, D, HD,
                           pool.host_valid_len(slot), len(cid))
        page = pool.slab[slot].cpu().numpy()
        if not np.isfinite(page).all():
            raise CodecError("non-finite element in KV page")
        return head + cid + page.tobytes()
    k, v = pool.read_host_kv(slot)
    return encode_arrays(chunk_id, k, v, pool.host_valid_len(slot), scheme)


def decode_arrays(data):
    """(chunk_id, keys, values, valid_len) as f32; F32 entries give read-only
    views over ``data`` (codec.py:190-195)."""
    v = parse_entry(data)
    L, KVH, D, HD = v.shape
    if v.scheme is QuantScheme.F32:
        arr = np.frombuffer(data, "<f4", 2 * L * KVH * D * HD, v.payload_off)
        arr = arr.reshape(L, 2, KVH, D, HD)
        return v.chunk_id, arr[:, 0], arr[:, 1], v.valid_len
    if v.scheme is QuantScheme.F16:
        arr = np.frombuffer(data, "<f2", 2 * L * KVH * D * HD, v.payload_off)
        arr = arr.reshape(L, 2, KVH, D, HD).astype(np.float32)
        return v.chunk_id, np.ascontiguousarray(arr[:, 0]), np.ascontiguousarray(arr[:, 1]), \
            v.valid_len
    sc = v.scales()
    keys = np.empty((L, KVH, D, HD), np.float32)
    values = np.empty_like(keys)
    off = v.payload_off
    for li in range(L):
        for j, out in enumerate((keys, values)):
            out[li] = dequantize_tensor(bytes(data[off:off + v.tensor_bytes]), sc[li, j],
                                        v.scheme, (KVH, D, HD))
            off += v.tensor_bytes
    return v.chunk_id, keys, values, v.valid_len


def decode_entry(data):
    """Parse an entry into a host f32 DocKV ready for scoring (codec.py:160-211)."""
    from .model import KVTensorSet
    from .reranker import DocKV
    cid, k, vals, vl = decode_arrays(data)
    return DocKV(chunk_id=cid, kv=KVTensorSet(k, vals, 0), valid_len=vl)


def decode_entry_to_pool(data, pool, slot: int | None = None, stream=None):
    """Decode an entry straight into an HBM pool page; returns the DocKV handle.

    F32 / F16: the payload bytes are copied H2D once and cast to the pool
    dtype on the GPU (F16 into an f16 pool is a plain copy).  INT8/INT4: codes + scales are copied H2D and expanded by the
    krr_dequant_kv kernel, one launch per (layer, K|V) page."""
    import torch

    from . import _lib
    from .reranker import DeviceKV, DocKV
    v = parse_entry(data)
    L, KVH, D, HD = v.shape
    if (L, 2, KVH, D, HD) != tuple(pool.page_shape):
        from .errors import ShapeError
        raise ShapeError(f"entry shape {v.shape} does not match pool {pool.page_shape}")
    if slot is None:
        slot = int(pool.allocate([v.chunk_id])[0])
    dev = pool.device
    page = pool.slab[slot]
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.stream(st):
        if not v.scheme.quantised:
            dt = torch.float32 if v.scheme is QuantScheme.F32 else torch.float16
            src = torch.frombuffer(bytearray(v.payload()), dtype=dt)
            page.copy_(src.to(dev, non_blocking=False).view(page.shape))
        else:
            codes = torch.frombuffer(bytearray(v.payload()), dtype=torch.uint8).to(dev)
            scales = torch.from_numpy(np.array(v.scales(), dtype=np.float32)).to(dev)
            L_ = _lib.lib()
            for li in range(L):
                for j in range(2):
                    t = li * 2 + j
                    _lib.check(L_.krr_dequant_kv(
                        codes.data_ptr() + t * v.tensor_bytes, scales[li, j].data_ptr(),
                        v.scheme.bits, KVH, D, HD, pool.code, page[li, j].data_ptr(),
                        st.cuda_stream))
    pool.set_valid_len([slot], [v.valid_len])
    return DocKV(chunk_id=v.chunk_id, kv=DeviceKV(pool, slot), valid_len=v.valid_len)
