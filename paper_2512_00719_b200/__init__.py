"""B200-native decision plane (sampling epilogue) of SIMPLE, arXiv 2512.00719.

Public names mirror the reference package `decplane` (decplane/__init__.py:1-35)
where the concept carries over; the compute runs in hand-written sm_100a CUDA
kernels behind the C ABI in include/decplane_b200.h.
"""

from .core import (
    DEFAULT_MAX_GENERATED,
    LogitsShardBlock,
    TOP_K_DISABLED,
    DegenerateRowError,
    RangeError,
    SamplingParams,
    SequenceState,
    TokenDecision,
    new_sequence_state,
    validate_params,
)
from .penalty import PenaltyState, update_output_histogram
from .sampler import VARIANT_FULL, VARIANT_SHVS, DecisionPlane, Decisions
from .service import (VARIANTS, ShvsRowContext, Sampler, _Sampler, make_shard_blocks, sample_full,
                      shvs_sample)
from .shvs import HotVocab, acceptance_rate, build_hot_vocab, load_hot_vocab_trace, save_hot_vocab_trace
from .transport import AssembledLogitsView, DecisionBatch, assemble_view, partition_batch

__version__ = "0.1.0"

__all__ = [
    "DEFAULT_MAX_GENERATED", "TOP_K_DISABLED", "DegenerateRowError", "RangeError", "SamplingParams",
    "SequenceState", "TokenDecision", "new_sequence_state", "validate_params", "PenaltyState",
    "update_output_histogram", "VARIANT_FULL", "VARIANT_SHVS", "DecisionPlane", "Decisions", "sample_full",
    "shvs_sample", "HotVocab", "acceptance_rate", "build_hot_vocab", "load_hot_vocab_trace",
    "save_hot_vocab_trace", "partition_batch", "__version__", "LogitsShardBlock", "VARIANTS", "ShvsRowContext",
    "Sampler", "_Sampler", "make_shard_blocks", "AssembledLogitsView", "DecisionBatch", "assemble_view",
]
