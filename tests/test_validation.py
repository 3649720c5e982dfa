"""Host-side input validation of the scoring entry points (CPU): the same
error classes and conditions as the reference's reranker.py:154-179 (_doc_valid,
_query_valid), :146-151 (_forward_fn path switch), :132-143 (tokenize)."""

from types import SimpleNamespace

import numpy as np
import pytest

from paper_2504_02921_b200 import reranker
from paper_2504_02921_b200.config import LayoutConfig, ModelConfig
from paper_2504_02921_b200.errors import ConfigError, DegenerateInputError, ShapeError

M = SimpleNamespace(config=ModelConfig(vocab_size=100), layout=LayoutConfig(document_len=6,
                                                                          query_len=4))


def test_doc_validation():
    valid, vl = reranker._doc_valid(M, [5, 6, 7, 0, 0, 0])
    assert vl == 3 and valid.tolist() == [True] * 3 + [False] * 3
    with pytest.raises(ShapeError):                      # wrong length
        reranker._doc_valid(M, [1, 2, 3])
    with pytest.raises(DegenerateInputError):            # all padding
        reranker._doc_valid(M, [0] * 6)
    with pytest.raises(ShapeError):                      # interior pad
        reranker._doc_valid(M, [1, 0, 2, 3, 0, 0])
    with pytest.raises(ShapeError):                      # out of vocabulary
        reranker._doc_valid(M, [1, 2, 100, 0, 0, 0])
    with pytest.raises(ShapeError):
        reranker._doc_valid(M, [1, -2, 3, 0, 0, 0])


def test_query_validation():
    # interior query pads are allowed (only the document must be a prefix)
    assert reranker._query_valid(M, [3, 0, 4, 0]).tolist() == [True, False, True, False]
    with pytest.raises(ShapeError):
        reranker._query_valid(M, [1, 2, 3, 4, 5])
    with pytest.raises(DegenerateInputError):
        reranker._query_valid(M, [0, 0, 0, 0])
    with pytest.raises(ShapeError):
        reranker._query_valid(M, [1, 2, 3, 999])


def test_path_switch():
    reranker._check_path("fast")
    reranker._check_path("reference")
    with pytest.raises(ConfigError):
        reranker._check_path("fused")


def test_pair_count_closed_form():
    """attn_mac_pairs closed form (SPEC: D=256, Q=48 reuse = 48*256 + 48*49/2)."""
    valid = np.ones(256 + 48, bool)
    assert int(reranker.pair_count(valid, 256)[0]) == 48 * 256 + 48 * 49 // 2 == 13464
    assert int(reranker.pair_count(valid, 0)[0]) == 304 * 305 // 2 == 46360
    v = valid.copy(); v[250:256] = False                 # padded document: pads never count
    assert int(reranker.pair_count(v, 256)[0]) == 48 * 250 + 48 * 49 // 2
