"""B200-native hot path of the sparse cross-encoder (arXiv 2312.17649).

Drop-in for the reference package's attention module and encoder forward
(``sparsecross.attention`` / ``sparsecross.encoder``), plus GPU fine-tuning
(``sparsecross.training``, backward kernels): same names, argument
meaning and error classes, computed by sm_100a CUDA kernels behind the C ABI
in ``include/sparsecross_b200.h``.  No CPU fallback exists.
"""

from .attention import (
    FULL,
    GROUPS,
    PADDING_MODES,
    AttentionError,
    AttentionPattern,
    apply_pattern,
    attend_packed,
    attend_segments,
    attend_segments_backward,
    full_pattern,
    full_attention,
    group_attention,
    group_attention_backward,
    longformer_pattern,
    make_pattern,
    SegmentScores,
    masked_segment_softmax,
    segment_softmax,
    masked_segment_softmax_backward,
    qds_band_exclusions,
    qds_pattern,
    sparse_pattern,
    windowed_cross_attention,
)
from .band import (
    MASKED,
    BandMatrix,
    BandShapeError,
    band_apply,
    band_apply_backward,
    band_pv,
    band_pv_backward,
    band_qk,
    band_qk_backward,
    band_scores,
    band_scores_backward,
    band_to_dense,
    band_validity,
    dense_band_oracle,
)
from .benchmark import (
    BenchConfigError,
    BenchRecord,
    BenchSpec,
    FlopBreakdown,
    default_model_config,
    emit_report,
    flop_count,
    gen_random_batch,
    measure,
    run_bench,
)
from .encoder import (
    CrossEncoder,
    EncoderConfig,
    EncoderError,
    NonFiniteActivationError,
    PackedBatch,
    SubsequencePartition,
    TokenSequence,
    assemble_input,
    encoder_forward,
    gelu,
    gelu_grad,
    init_weights,
    interpolate_positions,
    layer_backward,
    layer_forward,
    layer_norm,
    layer_norm_backward,
    qds_global_positions,
    relevance_score,
    resolve_pattern,
    weight_nbytes,
)
from .layout import PackedLayout
from .serialize import SerializationError, load_model, save_model
from .training import (
    AdamW,
    SyntheticTask,
    TrainableCrossEncoder,
    TrainingDivergedError,
    TrainingError,
    Triple,
    grad_check,
    margin_mse_grad,
    margin_mse_loss,
    ranknet_grad,
    ranknet_loss,
    train_toy,
    validation_ndcg,
    write_trace_csv,
)

__version__ = "0.1.0"
from .rerank import EvaluationError, RunEntry, ndcg_at_k, rerank  # noqa: E402  (R/evaluation.py; shadows the submodule attribute as the reference's top-level name does)
