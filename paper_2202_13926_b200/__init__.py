"""B200-native Frequency Selective Reconstruction (Regensky et al., arXiv 2202.13926).

Drop-in for the reference package ``fsrkit`` on its hot path: the same public
names and signatures, with reconstruction running in hand-written sm_100a
CUDA kernels (libfsr.so, C ABI in include/fsr.h).
"""

from .engine import (BlockResult, BlockState, Trace, init_residual, reconstruct,
                     reconstruct_batch, reconstruct_block, reconstruct_block_full,
                     reconstruct_image, run_iterations)
from .frames import (BlockDescriptor, FsrParams, GrayImage, SampledBlock, SampledImage,
                     block_partition, extract_support_block, mean_fill, quarter_sample,
                     quarter_sample_mask, splitmix64)
from .quality import QualityReport, psnr, time_block
from .spectra import WeightSet, build_weight_set, frequency_weight, spatial_weight

__version__ = "0.1.0"

__all__ = [
    "BlockDescriptor", "BlockResult", "BlockState", "FsrParams", "GrayImage", "QualityReport",
    "SampledBlock", "SampledImage", "Trace", "WeightSet", "block_partition", "build_weight_set",
    "extract_support_block", "frequency_weight", "init_residual", "mean_fill", "psnr",
    "quarter_sample", "quarter_sample_mask", "reconstruct", "reconstruct_batch",
    "reconstruct_block", "reconstruct_block_full", "reconstruct_image", "run_iterations",
    "spatial_weight", "splitmix64", "time_block",
]
