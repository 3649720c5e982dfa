"""B200-native KV-reuse decoder-reranker hot path (HyperRAG, arXiv 2504.02921).

Drop-in for the reference package ``kvrerank``'s hot path: document-KV
precompute (``doc_prefill`` / ``populate_store``), the KV-store interface
(``ShardedStore`` + HRKV entries) and the rerank entry points
(``score_reuse`` / ``score_batch``).  Compute runs in hand-written sm_100a
CUDA kernels behind a C ABI (``include/kvrerank_b200.h``); there is no CPU
fallback.
"""

from .codec import (QuantScheme, decode_entry, decode_entry_to_pool, dequantize_tensor,
                    encode_entry, payload_nbytes, quantize_tensor)
from .config import PRESETS, LayoutConfig, ModelConfig
from .errors import (CodecError, ConfigError, DegenerateInputError, DuplicateChunkError,
                     FormatError, KvRerankError, PositionError, ShapeError, StoreError)
from .forward import forward, forward_fn
from .kvpool import HostKVTier, KVPool
from .model import KVTensorSet, RerankModel
from .reranker import (CounterReport, DeviceKV, DocKV, ScoredPair, doc_prefill,
                       doc_prefill_batch, pool_for, score_batch, score_full, score_reuse,
                       tokenize)
from .pipeline import populate_store, rerank, select
from .store import (DevicePagedKVStore, DirectoryBackend, MemoryBackend, ShardedStore,
                    StoreStats, shard_of)

__version__ = "0.1.0"
