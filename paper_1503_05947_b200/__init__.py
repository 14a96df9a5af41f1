"""paper_1503_05947_b200 — B200-native Reduced Basis Decomposition greedy loop.

A drop-in for the hot path of the reference (arXiv 1503.05947, proj/): the
``decompose`` greedy loop and out-of-sample ``project``, executed by
hand-written sm_100a CUDA kernels behind the C ABI ``include/rbd_cuda.h``.
"""
from ._lib import (CudaError, DegenerateInput, DimensionMismatch, IncompatibleWeight,
                   IndexOutOfRange, InvalidArgument, IoError, NoConvergence, NotPositive,
                   ParseError, RbdError, UnsupportedFormat, Context, default_context,
                   load_library)
from .api import (Classifier, Model, ResidentModel, Workspace, decompose, decompose_many, fit, load, make_config,
                  mgs_project, project, project_batch, project_batch_f32, reconstruct, save)

__all__ = [
    "RbdError", "InvalidArgument", "IncompatibleWeight", "DegenerateInput", "IndexOutOfRange",
    "DimensionMismatch", "NotPositive", "NoConvergence", "UnsupportedFormat", "IoError",
    "ParseError", "CudaError", "Context", "default_context", "load_library", "Model",
    "Workspace", "ResidentModel", "Classifier", "fit", "decompose", "decompose_many", "load", "make_config", "mgs_project", "project", "project_batch",
    "project_batch_f32", "reconstruct", "save",
]
