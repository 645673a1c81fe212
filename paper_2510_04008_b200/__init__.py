"""B200-native RACE attention (arXiv 2510.04008): forward + backward, causal and
non-causal, as hand-written sm_100a CUDA behind the reference package's API.

Drop-in names (same meaning as ``race_attention`` in the reference):
``SketchConfig, AttnInputs, RaceOutput, RaceGradients, race_attention,
race_attention_vjp, accumulate_num_den, row_normalize, table_hyperplanes,
derive_table_rng, gaussian_matrix`` plus the validation-side names of
``ra/__init__.py:58-98`` (soft/hard hashing, theory sweeps, exact attention,
``bench_scaling``).  Device-level: ``race_forward``, ``race_backward``,
``RaceAttentionFunction``, ``RaceAttention`` (nn.Module), and the
sequence-sharded ``sharded_forward`` / ``sharded_backward``.
"""

from .attention import (
    DEGENERATE_DEN_EPS,
    ZERO_ROW_EPS,
    AttnInputs,
    PrecisionWarning,
    RaceGradients,
    RaceOutput,
    SketchConfig,
    accumulate_num_den,
    all_hyperplanes,
    derive_table_rng,
    gaussian_matrix,
    race_attention,
    race_attention_vjp,
    row_normalize,
    row_normalize_vjp,
    table_hyperplanes,
)
from .functional import (
    RaceAttentionFunction,
    SketchParams,
    race_attention_torch,
    race_backward,
    race_forward,
)
from .module import RaceAttention, head_hyperplanes
from .sharded import sharded_backward, sharded_forward, shard_bounds
from .sketch import (
    BucketStats,
    HashTable,
    bucket_stats,
    corner_matrix,
    corner_vector,
    dominant_corner_mass,
    hard_hash,
    make_hash_table,
    soft_features,
)
from .exact import (
    angular_attention,
    angular_attention_vjp,
    angular_kernel_matrix,
    angular_similarity,
    softmax_attention,
    softmax_attention_vjp,
)
from .benchmark import BenchMethod, BenchRecord, bench_scaling, demo_kernel_heatmap
from .theory import (
    CollisionReport,
    RowSumReport,
    ScalingExperiment,
    bias_sweep,
    collision_identity_check,
    hard_race_attention,
    kernel_deviation,
    output_rms_error,
    race_kernel,
    row_sum_stability,
    variance_sweep,
)

__version__ = "0.1.0"

__all__ = [
    "AttnInputs", "DEGENERATE_DEN_EPS", "RaceAttention", "RaceAttentionFunction", "RaceGradients",
    "RaceOutput", "SketchConfig", "SketchParams", "ZERO_ROW_EPS", "accumulate_num_den",
    "all_hyperplanes", "derive_table_rng", "gaussian_matrix", "head_hyperplanes", "race_attention",
    "race_attention_torch", "race_attention_vjp", "race_backward", "race_forward", "shard_bounds",
    "sharded_backward", "sharded_forward", "table_hyperplanes",
    # validation side (sketch.py, exact.py, theory.py, benchmark.py)
    "BucketStats", "HashTable", "angular_attention", "angular_attention_vjp", "angular_kernel_matrix",
    "angular_similarity", "bias_sweep", "bucket_stats", "collision_identity_check", "corner_matrix",
    "corner_vector", "dominant_corner_mass", "hard_hash", "hard_race_attention", "kernel_deviation",
    "make_hash_table", "output_rms_error", "race_kernel", "row_sum_stability", "soft_features",
    "softmax_attention", "softmax_attention_vjp", "variance_sweep",
    # the rest of the reference's top-level names (ra/__init__.py:58-98)
    "BenchMethod", "BenchRecord", "CollisionReport", "RowSumReport", "ScalingExperiment", "bench_scaling",
    "demo_kernel_heatmap", "row_normalize", "row_normalize_vjp", "PrecisionWarning",
]
