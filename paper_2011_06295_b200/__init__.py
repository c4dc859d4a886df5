"""B200-native (sm_100a) direct sparse convolution engine.

Drop-in for the hot path of the reference package ``sparseconv``
(arXiv 2011.06295): the unified-sparsity CSR weight format and the
``conv_sparse`` operator, re-exported under the reference's names
(sparseconv/__init__.py:6-24).  Compute runs in libsparseconv_b200.so
(hand-written CUDA for sm_100a behind a C ABI, include/sparseconv_b200.h);
there is no CPU fallback.
"""
from .engine import (SUB_BATCH_CANDIDATES, EnginePlan, conv_sparse, conv_sparse_1d,
                     conv_sparse_reference, dense_mac_count, sparse_mac_count,
                     tune_sub_batch)
from .benchmark import BenchRecord, SweepResult, bench_layer, emit_report, sparsity_sweep
from .configure import NetworkConfig, configure_network
from .errors import FormatError, IntegrityError, ShapeError, SparseConvError, TrainingError
from .geometry import ConvShape, check_nchw, compute_dtype, output_shape, pad_input
from .weights import (CsrKernel, SparsityReport, analyze_sparsity, build_csr, decompress,
                      select_padding_zeros)

__version__ = "0.1.0"

__all__ = [
    "BenchRecord", "SweepResult", "bench_layer", "emit_report", "sparsity_sweep",
    "ConvShape", "CsrKernel", "EnginePlan", "NetworkConfig", "configure_network", "FormatError", "IntegrityError", "ShapeError",
    "SparseConvError", "SparsityReport", "SUB_BATCH_CANDIDATES", "TrainingError",
    "analyze_sparsity", "build_csr", "check_nchw", "compute_dtype", "conv_sparse",
    "conv_sparse_1d", "conv_sparse_reference", "decompress", "dense_mac_count",
    "output_shape", "pad_input", "select_padding_zeros", "sparse_mac_count", "tune_sub_batch",
]
