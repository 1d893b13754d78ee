"""B200-native Intergrams top-k n-gram counter (arxiv 2511.14955).

The product path is the C-ABI library built from csrc/ (sm_100a CUDA) and the
Python mirror of the reference API in :mod:`.intergrams`.
"""
from .intergrams import (ConfigError, CountMode, Corpus, GramCount, IntergramConfig,  # noqa: F401
                         IntergramsResult, InternalError, IoError, MergeStrategy, PassResult,
                         Session, candidate_gram, candidate_id, count_dense, count_trigrams,
                         dense_capacity, dense_gram, extend_pass, gram_to_key, key_to_gram,
                         make_memory_corpus, run_intergrams, shard_range, top_k, topk_to_tsv)

__version__ = "0.1.0"
