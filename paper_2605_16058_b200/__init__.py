"""B200-native t-SVDM (arxiv 2605.16058): drop-in for the reference
``starm`` hot path.

The public names and signatures follow ``starm.__all__``
(/root/reference/pkg/src/starm/__init__.py:78-146) for the compression
path: transforms, mode-k TTM, slice SVDs, global thresholding, fixed-rank
and tolerance t-SVDM, reconstruction and the *_M product.  Compute runs in
``libstarm.so`` (hand-written sm_100a kernels, C ABI in include/starm.h);
there is no CPU fallback.  Host inputs (DenseTensor) come back as host
outputs; DeviceTensor inputs stay in HBM end to end.
"""

from .codec import (BadMagicError, BenchRow, CodecError, FormatError, TruncatedPayloadError,
                    UnsupportedDtypeError, UnsupportedVersionError, read_compressed, read_tensor,
                    write_bench_csv, write_compressed, write_tensor)
from .compress import (COMPUTE_EFFICIENT, MEMORY_EFFICIENT, METHOD_FIXED_RANK, METHOD_TOLERANCE,
                       TOLERANCE_STRATEGIES, TRUNCATE, CompressedTensor, StageClock,
                       ThresholdResult, TSVDMResult, compression_ratio, compute_threshold,
                       full_tsvdm, reconstruct, reconstruct_fused, relative_error_device,
                       starm_product,
                       tsvdm_fixed_rank, tsvdm_tolerance, tsvdm_tolerance_stream)
from .mode_product import (BATCHED, LOOP, PARFOR, TTMPlan, from_transform_domain,
                           to_transform_domain, ttm, ttm_inverse)
from .slice_svd import (SLICES_PARALLEL, SVD_PARALLEL, DeviceFactors, SliceSVDSet,
                        VariableRankFactors, svd_all_slices, svd_truncated_slices,
                        svd_values_only)
from .tensors import DenseTensor, DeviceTensor, SliceIndex, linear_index, multi_index, refold
from .transform_set import (CUSTOM, DATA_DRIVEN, DCT, IDENTITY, Transform, TransformSet,
                            data_driven_transform, dct_matrix, identity_transform,
                            orthonormality_residual, validate_transform)

__version__ = "0.1.0"

__all__ = [
    "BadMagicError", "BenchRow", "CodecError", "FormatError", "TruncatedPayloadError",
    "UnsupportedDtypeError", "UnsupportedVersionError", "read_compressed", "read_tensor",
    "write_bench_csv", "write_compressed", "write_tensor",
    "BATCHED", "COMPUTE_EFFICIENT", "CUSTOM", "CompressedTensor", "DATA_DRIVEN", "DCT",
    "DenseTensor", "DeviceFactors", "DeviceTensor", "IDENTITY", "LOOP", "MEMORY_EFFICIENT",
    "METHOD_FIXED_RANK", "METHOD_TOLERANCE", "PARFOR", "SLICES_PARALLEL", "SVD_PARALLEL",
    "SliceIndex", "SliceSVDSet", "StageClock", "TOLERANCE_STRATEGIES", "TRUNCATE", "TSVDMResult",
    "TTMPlan", "ThresholdResult", "Transform", "TransformSet", "VariableRankFactors",
    "compression_ratio", "compute_threshold", "data_driven_transform", "dct_matrix",
    "from_transform_domain", "full_tsvdm", "identity_transform", "linear_index", "multi_index",
    "orthonormality_residual", "reconstruct", "reconstruct_fused", "refold", "relative_error_device", "starm_product",
    "svd_all_slices", "svd_truncated_slices", "svd_values_only", "to_transform_domain",
    "tsvdm_fixed_rank", "tsvdm_tolerance", "tsvdm_tolerance_stream", "ttm", "ttm_inverse", "validate_transform",
]
