"""paper_2505_21728_b200 -- B200-native batched Hypercube-Givens Transform (HyGT).

The drop-in for the data-parallel hot path of the reference toolkit (arXiv 2505.21728,
/root/reference/proj): batched hygt::forward / hygt::inverse with per-class models, the
bit-exact forward_fixed / inverse_fixed, the per-class energy reduction and the dense KLT
comparison path, and the coordinate-descent trainer (optimize), all computed by hand-written sm_100a kernels in libhygt_gpu.so behind the C ABI
of include/hygt_gpu.h. There is no CPU fallback.
"""
from .errors import (ArgumentError, CudaError, IoError, NumericalError,  # noqa: F401
                     OverflowError)
from .model import (HyGTModel, ModelBundle, QuantizedHyGTModel, TransformKind,  # noqa: F401
                    TrigTable, build_trig_table, dequantize_model, hypercube_indices,
                    memory_footprint, num_parameters, quantize_model, validate_permutation)
from .plan import (FixedPlan, HyGTPlan, KLTPlan, correlation, finalize_correlation,  # noqa: F401
                   forward, forward_fixed, inverse, inverse_fixed)
from .train import (OptimizerConfig, TrainingReport, optimize, optimize_batch,  # noqa: F401
                    train_classes, variance_permutation)

__all__ = [
    "ArgumentError", "IoError", "NumericalError", "OverflowError", "CudaError",
    "HyGTModel", "QuantizedHyGTModel", "TrigTable", "ModelBundle", "TransformKind",
    "build_trig_table", "quantize_model", "dequantize_model", "hypercube_indices",
    "memory_footprint", "num_parameters", "validate_permutation",
    "HyGTPlan", "FixedPlan", "KLTPlan", "forward", "inverse", "forward_fixed", "inverse_fixed",
    "correlation", "finalize_correlation",
    "OptimizerConfig", "TrainingReport", "optimize", "optimize_batch", "variance_permutation",
    "train_classes",
]
