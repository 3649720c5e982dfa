"""CPU oracle for the KV-reuse rerank hot path — TEST INFRASTRUCTURE ONLY.

This package is a plain numpy restatement of the reference package
``kvrerank`` 0.1.0 (``/root/reference/pkg/src/kvrerank``) for the functions
on the hot path (SURVEY.md §8(a) rows a1–a13).  It is the *checker*:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* the product package ``paper_2504_02921_b200`` never imports it and has no
  CPU fallback — its compute path is the CUDA library only.

Parity is PINNED: ``tests/golden/*.npz`` were produced by running the
reference package itself in the build container
(``tests/golden/make_golden.py``), and ``tests/test_oracle.py`` checks this
restatement against those vectors (weights bit-exact, scores to <=1e-5 of the
reference's own fast path, counters exact).
"""

from .kvrerank_np import (  # noqa: F401
    OracleConfig, OracleWeights, fnv1a64, splitmix64_array, uniform_signed,
    init_tensor, init_weights, rope_tables, forward, doc_prefill, score_reuse,
    score_full, pair_count, select_topk, score_head, round_weights, init_rows,
    LazyEmbedding,
)
