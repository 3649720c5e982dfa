"""Host-side FNV-1a 64 (hashing.py:23-31): per-tensor stream seeds and the
word tokenizer.  The SplitMix64 weight streams themselves run on the device
(krr_init_uniform)."""

from __future__ import annotations

_M64 = (1 << 64) - 1


def fnv1a64(data) -> int:
    if isinstance(data, str):
        data = data.encode("utf-8")
    h = 0xCBF29CE484222325
    for byte in data:
        h = ((h ^ byte) * 0x100000001B3) & _M64
    return h
