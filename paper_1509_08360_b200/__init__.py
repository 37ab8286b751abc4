"""B200-native compressive spectral embedding (arXiv 1509.08360) -- the hot path.

A drop-in for the reference `csemb` package's embedding path: the order-L
Legendre matrix polynomial E = f_L(S) Omega computed on the GPU by a fused
SpMM-recurrence kernel (sm_100a), behind the reference's public signatures.
Host-side pieces (coefficients, spectral functions, CSR container, input
builders) mirror the reference; the recurrence, the projection block, the
power-iteration norm estimate and the row normalisation run on the device
through the C ABI in include/csemb_cuda.h.  The embedding's downstream
consumers (k-means, modularity, sampled-pair distortion: `cluster`,
`distortion`) run on the device as well.
"""

from .engine import (
    COLUMN_CHUNK,
    DeviceMatrix,
    EmbedConfig,
    EmbeddingMatrix,
    Plan,
    SpmvCounter,
    apply_expansion,
    default_dimension,
    device_matrix,
    release_device_copy,
    estimate_spectral_norm,
    fast_embed_cascaded,
    fast_embed_eig,
    fast_embed_general,
    fold_seed,
    install,
    jl_dimension,
    norm_start_block,
    sample_projection,
)
from .cluster import (
    ClusterAssignment,
    ClusterExperiment,
    DeviceKMeans,
    DeviceRows,
    ModularityScore,
    cluster_experiment,
    kmeans,
    modularity,
    plan_rows,
)
from .distortion import (
    DistortionReport,
    distance_bound_audit,
    distortion_percentiles,
    exact_embedding,
    pair_correlations,
    sample_pairs,
)
from .errors import CsembError, CudaUnavailableError, DivergenceError, InputFormatError
from .functions import (
    SpectralFunction,
    commute_time,
    constant,
    identity,
    indicator_above,
    odd_extension,
    parse_function,
    remapped,
    root_function,
    tabulated,
)
from .legendre import (
    LegendreExpansion,
    QuadratureSpec,
    approximation_report,
    expansion_eval,
    legendre_coefficients,
    legendre_eval,
    legendre_table,
)
from .sparse import SparseMatrix, dilate, normalized_adjacency, scale_values, simple_edges

__version__ = "0.1.0"

__all__ = [
    "COLUMN_CHUNK", "CsembError", "CudaUnavailableError", "DeviceMatrix", "DivergenceError",
    "EmbedConfig", "EmbeddingMatrix", "InputFormatError", "LegendreExpansion", "Plan",
    "QuadratureSpec", "SparseMatrix", "SpectralFunction", "SpmvCounter", "apply_expansion",
    "approximation_report", "commute_time", "constant", "default_dimension", "device_matrix", "release_device_copy",
    "dilate", "estimate_spectral_norm", "expansion_eval", "fast_embed_cascaded", "fast_embed_eig",
    "fast_embed_general", "fold_seed", "identity", "indicator_above", "install", "jl_dimension",
    "legendre_coefficients", "legendre_eval", "legendre_table", "norm_start_block",
    "normalized_adjacency", "odd_extension", "parse_function", "remapped", "root_function",
    "sample_projection", "scale_values", "simple_edges", "tabulated",
    # downstream consumers (cluster.py, oracle.py:88-186)
    "ClusterAssignment", "ClusterExperiment", "DeviceKMeans", "DeviceRows", "DistortionReport",
    "ModularityScore", "cluster_experiment", "distortion_percentiles", "kmeans", "modularity",
    "pair_correlations", "plan_rows", "sample_pairs", "distance_bound_audit", "exact_embedding",
]
