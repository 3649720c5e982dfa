"""Host-side KV-store interface and HRKV codec against the reference's bytes.

tests/golden/codec_c1.npz holds entries written by the reference codec itself
(make_golden.py codec_fixture).  Byte layout is integer/byte work, so the bar
is bit-exact: re-encoding the decoded tensors must reproduce the reference's
bytes for F32, INT8 and INT4.
"""

import os
import threading

import numpy as np
import pytest

from paper_2504_02921_b200 import codec, store
from paper_2504_02921_b200.errors import CodecError, FormatError, StoreError

S = codec.QuantScheme


@pytest.fixture(scope="module")
def g(golden_dir):
    return np.load(os.path.join(golden_dir, "codec_c1.npz"))


@pytest.mark.parametrize("name", ["f32", "int8", "int4"])
def test_decode_matches_reference(g, name):
    data = g[f"entry_{name}"].tobytes()
    cid, k, v, vl = codec.decode_arrays(data)
    assert cid == "doc-00042" and vl == 90
    assert np.array_equal(k, g[f"decoded_keys_{name}"])
    assert np.array_equal(v, g[f"decoded_values_{name}"])


@pytest.mark.parametrize("name", ["f32", "int8", "int4"])
def test_encode_bit_exact_vs_reference(g, name):
    f32 = g["entry_f32"].tobytes()
    cid, k, v, vl = codec.decode_arrays(f32)
    data = codec.encode_arrays(cid, np.array(k), np.array(v), vl, codec.QuantScheme.from_name(name))
    assert data == g[f"entry_{name}"].tobytes()


def test_f32_decode_is_zero_copy_view(g):
    data = g["entry_f32"].tobytes()
    _, k, _, _ = codec.decode_arrays(data)
    assert not k.flags.writeable and k.base is not None


def test_f16_scheme_roundtrip(g):
    """Scheme code 1 (this build's F16 extension): payload = the f16-rounded
    tensors, no scales; decode gives them back exactly as f32."""
    cid, k, v, vl = codec.decode_arrays(g["entry_f32"].tobytes())
    data = codec.encode_arrays(cid, np.array(k), np.array(v), vl, S.F16)
    L, KVH, D, HD = k.shape
    assert len(data) == codec.HEADER.size + len(cid) + codec.payload_nbytes(L, KVH, D, HD, S.F16)
    assert data[6] == 1
    cid2, k2, v2, vl2 = codec.decode_arrays(data)
    assert (cid2, vl2) == (cid, vl)
    assert np.array_equal(k2, np.asarray(k).astype(np.float16).astype(np.float32))
    assert np.array_equal(v2, np.asarray(v).astype(np.float16).astype(np.float32))
    # f16-exact inputs survive unchanged; out-of-range values are refused
    assert codec.encode_arrays(cid, k2, v2, vl, S.F16) == data
    big = np.array(k); big[0, 0, 0, 0] = 1e6
    with pytest.raises(CodecError):
        codec.encode_arrays(cid, big, np.array(v), vl, S.F16)
    with pytest.raises(CodecError):
        codec.quantize_tensor(np.zeros((1, 2, 2), np.float32), S.F16)


@pytest.mark.parametrize("name", ["int8", "int4"])
def test_quantize_edge_cases_vs_reference(g, name):
    q, sc = codec.quantize_tensor(g["edge_tensor"], codec.QuantScheme.from_name(name))
    assert np.frombuffer(q, np.uint8).tobytes() == g[f"edge_codes_{name}"].tobytes()
    assert np.array_equal(sc, g[f"edge_scales_{name}"])
    assert sc[0, 0] == 1.0            # all-zero channel -> scale 1.0


@pytest.mark.parametrize("scheme", [S.INT8_PER_CHANNEL, S.INT4_PER_CHANNEL])
def test_quant_error_bound(scheme):
    """|x - dequant(quant(x))| <= scale/2."""
    t = np.random.default_rng(0).standard_normal((3, 50, 17)).astype(np.float32)
    q, sc = codec.quantize_tensor(t, scheme)
    back = codec.dequantize_tensor(q, sc, scheme, t.shape)
    assert np.all(np.abs(back - t) <= sc[:, None, :] / 2 * (1 + 1e-6))


def test_payload_sizes():
    # SURVEY §4 closed forms (default config L=4, KVH=2, D=256, HD=16)
    assert codec.payload_nbytes(4, 2, 256, 16, S.F32) == 262144
    assert codec.payload_nbytes(4, 2, 256, 16, S.F16) == 131072
    assert codec.payload_nbytes(4, 2, 256, 16, S.INT8_PER_CHANNEL) == 65536
    assert codec.payload_nbytes(4, 2, 256, 16, S.INT4_PER_CHANNEL) == 32768
    assert codec.payload_nbytes(1, 1, 3, 1, S.INT4_PER_CHANNEL) == 4   # odd count pads


def test_format_errors(g):
    data = bytearray(g["entry_int8"].tobytes())
    with pytest.raises(FormatError):
        codec.decode_arrays(b"HRK")
    bad = bytearray(data); bad[0:4] = b"XXXX"
    with pytest.raises(FormatError):
        codec.decode_arrays(bytes(bad))
    bad = bytearray(data); bad[4] = 9
    with pytest.raises(FormatError):
        codec.decode_arrays(bytes(bad))
    bad = bytearray(data); bad[6] = 7          # no such scheme code
    with pytest.raises(FormatError):
        codec.decode_arrays(bytes(bad))
    bad = bytearray(data); bad[6] = 1          # F16 header over an INT8-sized body
    with pytest.raises(CodecError):
        codec.decode_arrays(bytes(bad))
    with pytest.raises(CodecError):
        codec.decode_arrays(bytes(data[:-1]))
    with pytest.raises(CodecError):
        codec.QuantScheme.from_name("fp8")
    k = np.zeros((1, 1, 2, 2), np.float32); k[0, 0, 0, 0] = np.nan
    with pytest.raises(CodecError):
        codec.encode_arrays("x", k, np.zeros_like(k), 1)


def test_scheme_names():
    assert S.from_name("kv8") is S.INT8_PER_CHANNEL and S.from_name(" INT4 ") is S.INT4_PER_CHANNEL
    assert [s.short_name for s in S] == ["f32", "f16", "int8", "int4"]
    assert S.from_name("half") is S.F16 and not S.F16.quantised and S.INT4_PER_CHANNEL.quantised


# ------------------------------------------------------------------ store
@pytest.fixture(params=["memory", "directory"])
def sharded(request, tmp_path):
    if request.param == "memory":
        return store.ShardedStore.in_memory(3)
    return store.ShardedStore.local(tmp_path / "kv", 3)


def test_store_roundtrip_and_placement(sharded, g):
    data = g["entry_int4"].tobytes()
    sharded.put_entry("doc-00042", 7, data)
    assert sharded.exists_entry("doc-00042", 7)
    assert not sharded.exists_entry("doc-00042", 8)       # other shard
    assert sharded.get_entry("doc-00042", 7) == data
    assert sharded.get_entry("nope", 7) is None
    st = sharded.stats()
    assert [s.entries for s in st] == [0, 1, 0]            # 7 % 3 == 1
    assert st[1].bytes == len(data) and st[1].gets == 2 and st[1].bytes_served == len(data)
    assert sharded.backends[1].keys() == ["doc-00042"]
    assert store.StoreStats.from_text(st[1].as_text()) == st[1]


def test_store_errors(tmp_path):
    with pytest.raises(StoreError):
        store.shard_of(1, 0)
    with pytest.raises(StoreError):
        store.shard_of(-1, 2)
    with pytest.raises(StoreError):
        store.ShardedStore([])
    d = store.ShardedStore.local(tmp_path / "s", 1)
    for key in ("../x", "a//b", "a b", ""):
        with pytest.raises(StoreError):
            d.put_entry(key, 0, b"x")
    with pytest.raises(StoreError):
        store.ShardedStore.local(tmp_path / "missing", 1, create=False)
    d.put_entry("ns/a.b-c_1", 0, b"123")                    # namespaced keys allowed
    assert d.backends[0].keys() == ["ns/a.b-c_1"]


def test_directory_put_is_atomic(tmp_path):
    """Concurrent readers see the old or the new value, never a mix."""
    b = store.DirectoryBackend(tmp_path / "a")
    old, new = b"A" * 200000, b"B" * 200000
    b.put("k", old)
    seen, stop = set(), threading.Event()

    def reader():
        while not stop.is_set():
            v = b.get("k")
            seen.add(v[:1] + v[-1:])

    th = threading.Thread(target=reader)
    th.start()
    for _ in range(30):
        b.put("k", new)
        b.put("k", old)
    stop.set()
    th.join()
    assert seen <= {b"AA", b"BB"}
    assert not [p for p in (tmp_path / "a").iterdir() if p.name.startswith(".tmp-")]
