"""CPU tests of the host layer: the C-ABI library's symbol table, the
reference-mirroring config/validation logic, counters and the no-fallback rule."""

import ctypes
import os
import re
import sys

import numpy as np
import pytest

import oracle
import paper_2504_02921_b200 as krr
from paper_2504_02921_b200 import _lib, reranker
from paper_2504_02921_b200.errors import ConfigError, KvRerankError, ShapeError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    syms = set()
    inc = os.path.join(ROOT, "include")
    for f in os.listdir(inc):
        if f.endswith(".h"):
            src = open(os.path.join(inc, f)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            syms |= set(re.findall(r"\b(krr_[a-z0-9_]+)\s*\(", src))
    return syms


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(_lib.LIB_PATH)
    declared = _declared_symbols()
    assert declared, "no krr_* declarations found in include/"
    missing = [s for s in sorted(declared) if not hasattr(L, s)]
    assert not missing, missing
    assert declared == set(_lib.EXPORTS)


def test_library_metadata_without_gpu():
    L = _lib.lib()
    assert L.krr_version().startswith(b"kvrerank_b200")
    assert _lib.launch_count() >= 0


def test_library_is_sm100a_only():
    """The .so carries sm_100a SASS (no PTX JIT fallback, no other arch)."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_error_code_mapping():
    for rc, exc in ((1, ConfigError), (2, ShapeError), (3, KvRerankError), (4, ConfigError)):
        with pytest.raises(exc):
            _lib.check(rc)
    _lib.check(0)


def test_model_config_validation_mirrors_reference():
    with pytest.raises(ConfigError):
        krr.ModelConfig(heads=6, kv_heads=4, model_dim=96, head_dim=16).validate()
    with pytest.raises(ConfigError):
        krr.ModelConfig(model_dim=100).validate()
    with pytest.raises(ConfigError):
        krr.ModelConfig(layers=0).validate()
    with pytest.raises(ConfigError):
        krr.LayoutConfig(document_len=0).validate()
    with pytest.raises(ConfigError):
        krr.LayoutConfig(pad_id=3).validate()
    for name, (cfg, lay) in krr.PRESETS.items():
        cfg.validate()
        lay.validate()
        assert lay.total_len <= cfg.max_position, name


def test_no_cpu_fallback():
    """Without a CUDA device the product path refuses to run (it never
    routes to a CPU implementation)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(ConfigError, match="CUDA"):
        krr.RerankModel.build(krr.ModelConfig(layers=1), krr.LayoutConfig(64, 8))


def test_tokenize_matches_reference_rule():
    text = "the quick brown fox jumps over the lazy dog"
    t = krr.tokenize(text, 12, vocab_size=32768)
    words = text.split()
    want = [1 + oracle.fnv1a64(w) % 32767 for w in words] + [0, 0, 0]
    assert t.tolist() == want and t.dtype == np.int64
    assert krr.tokenize(text, 3).tolist() == want[:3]
    with pytest.raises(ConfigError):
        krr.tokenize("x", 0)


def test_pair_count_vectorised_matches_oracle():
    rng = np.random.default_rng(0)
    v = rng.random((20, 176)) > 0.2
    got = reranker.pair_count(v, 128)
    assert got.tolist() == [oracle.pair_count(row, 128) for row in v]
    assert reranker.pair_count(np.ones(304, bool), 256).tolist() == [13464]


def test_counter_report_merge():
    a = krr.CounterReport(3, 10, 3, 100)
    a.merge(krr.CounterReport(5, 1, 2, 50))
    assert a.as_dict() == {"linear_token_count": 8, "attn_mac_pairs": 11,
                           "peak_activation_tokens": 3, "kv_bytes_loaded": 150}


def test_id_ranks_follow_chunk_id_order():
    from paper_2504_02921_b200.pipeline import _id_ranks, select
    cands = [["doc-3", "doc-1"], ["doc-2", "doc-3"]]
    assert _id_ranks(cands).tolist() == [[2, 0], [1, 2]]
    s = [krr.ScoredPair("b", "q", 1.0), krr.ScoredPair("a", "q", 1.0),
         krr.ScoredPair("c", "q", 2.0)]
    assert [p.chunk_id for p in select(s, 2)] == ["c", "a"]


def test_header_enums_match_host_constants():
    """The C-ABI enum values (include/kvrerank_b200.h) and the ctypes host layer
    agree: dtypes, epilogues, MLP kinds, backends."""
    import re
    src = open(os.path.join(ROOT, "include", "kvrerank_b200.h")).read()
    vals = {m.group(1): int(m.group(2)) for m in re.finditer(r"\b(KRR_[A-Z0-9_]+)\s*=\s*(\d+)", src)}
    want = {"KRR_F32": _lib.F32, "KRR_F16": _lib.F16, "KRR_BF16": _lib.BF16,
            "KRR_EPI_STORE": _lib.EPI_STORE, "KRR_EPI_GELU": _lib.EPI_GELU,
            "KRR_EPI_RESIDUAL": _lib.EPI_RESIDUAL, "KRR_EPI_QKV_ROPE": _lib.EPI_QKV_ROPE,
            "KRR_EPI_GLU_GELU": _lib.EPI_GLU_GELU, "KRR_EPI_GLU_SILU": _lib.EPI_GLU_SILU,
            "KRR_MLP_GELU": _lib.MLP_GELU, "KRR_MLP_GEGLU": _lib.MLP_GEGLU,
            "KRR_MLP_SWIGLU": _lib.MLP_SWIGLU, "KRR_GEMM_AUTO": _lib.GEMM_AUTO,
            "KRR_GEMM_TCGEN05": _lib.GEMM_TCGEN05, "KRR_GEMM_SIMT": _lib.GEMM_SIMT,
            "KRR_ATTN_AUTO": _lib.ATTN_AUTO, "KRR_ATTN_MMA": _lib.ATTN_MMA,
            "KRR_ATTN_SIMT": _lib.ATTN_SIMT, "KRR_ATTN_TCGEN05": _lib.ATTN_TCGEN05}
    for name, v in want.items():
        assert vals.get(name) == v, (name, vals.get(name), v)


def test_bench_rejects_gpus_world_mismatch():
    """bench.py --gpus N under a launcher must match WORLD_SIZE (no silent
    single-process run reporting N GPUs)."""
    import subprocess
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"],
                       env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr


def test_rerank_graph_cache_policy(monkeypatch):
    """pipeline._graph_for: a shape is scored eagerly the first time, captured
    the second, replayed afterwards; at most GRAPH_CACHE graphs per pool (LRU),
    keyed by the weights object and the batch shape."""
    from paper_2504_02921_b200 import engine, pipeline

    made = []

    class FakeGraph:
        def __init__(self, w, pool, n_q, n_c, Q, k):
            made.append((n_q, n_c, Q, k))

    monkeypatch.setattr(engine, "GraphedScorer", FakeGraph)

    class Pool:
        pass

    pool, w = Pool(), object()
    assert pipeline._graph_for(pool, w, 1, 100, 48, 20) is None        # first sight: eager
    g1 = pipeline._graph_for(pool, w, 1, 100, 48, 20)                    # second: capture
    assert isinstance(g1, FakeGraph) and made == [(1, 100, 48, 20)]
    assert pipeline._graph_for(pool, w, 1, 100, 48, 20) is g1            # replay
    for shape in [(2, 50, 48, 20), (4, 25, 48, 20)]:
        assert pipeline._graph_for(pool, w, *shape) is None
        assert pipeline._graph_for(pool, w, *shape) is not None
    assert len(pool._rerank_graphs) == pipeline.GRAPH_CACHE
    assert (id(w), 1, 100, 48, 20) not in pool._rerank_graphs           # least recently used
    assert pipeline._graph_for(pool, object(), 1, 100, 48, 20) is None  # other weights


def test_bench_work_accounting():
    """bench.py's per-pair work model at the C3 shape: 554.67
    GFLOP per pair (541.17 GEMM + 13.50 attention) and 67.1 MB of cached KV;
    the attention term is the part attention_flops_per_pair reports."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2504_02921_b200.config import PRESETS
    cfg, lay = PRESETS["c3_mistral7b"]
    D, Q = lay.document_len, lay.query_len
    f = bench.suffix_flops_per_pair(cfg, D, Q)
    a = bench.attention_flops_per_pair(cfg, D, Q)
    assert abs(f / 1e9 - 554.67) < 0.01 and abs(a / 1e9 - 13.50) < 0.01
    d, H, KVH, HD, L = 4096, 32, 8, 128, 32
    gemm = 2 * L * Q * (d * (H + 2 * KVH) * HD + H * HD * d + 2 * d * 4 * d)
    assert f - a == gemm
    assert bench.kv_bytes_per_pair(cfg, D) == 2 * L * KVH * D * HD * 2 == 67108864


def test_balanced_pass_split():
    """Scoring/prefill passes: the fewest passes of <= cap units, sized evenly
    (C3: 6,400 pairs at 682 per pass -> 10 passes of 640, not 9 + a 262 tail)."""
    from paper_2504_02921_b200.engine import _balanced_step
    assert _balanced_step(6400, 682) == 640
    assert _balanced_step(100, 682) == 100
    assert _balanced_step(1, 1) == 1
    assert _balanced_step(0, 5) == 1
    for n in (1, 7, 683, 1364, 1365, 6400):
        for cap in (1, 3, 64, 682):
            s = _balanced_step(n, cap)
            assert s <= cap and -(-n // s) == -(-n // cap)
