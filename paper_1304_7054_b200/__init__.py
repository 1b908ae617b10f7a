"""kronbatch-b200: batched Kronecker-product action on NVIDIA B200 (sm_100a).

B200-native implementation of the hot path of arXiv:1304.7054 / the reference
``kronbatch`` library: ``kron2`` (Y = alpha op(A) op(X) op(B)^T + beta Y) and
``kron3`` (vec Y = alpha (C (x) B (x) A) vec X + beta vec Y) over large batches,
fp32 / fp64, behind the reference's own API -- plus the umbrella API's other two
batched operators, ``kron1`` (shared-A GEMV) and ``gemm_a`` (varying-A GEMM).
See DESIGN.md.
"""
from ._lib import ABI_SYMBOLS, LIB_PATH, lib  # noqa: F401  (raises if the .so is missing)
from .api import (  # noqa: F401
    Array3View,
    BatchView,
    Exec,
    KronProblem2D,
    KronProblem3D,
    MatrixOp,
    MatrixView,
    Part,
    VectorView,
    Workspace,
    footprint,
    gemm_a,
    is_transposed,
    kron1,
    kron2,
    kron2_parts,
    kron3,
    kron3_parts,
    kron3_workspace_size,
    last_path,
    launch_count,
    op_dims,
    pooled_bytes,
    release_buffers,
    validate,
    validate_batch,
    version,
)

__all__ = [
    "Array3View", "BatchView", "Exec", "KronProblem2D", "KronProblem3D", "MatrixOp", "MatrixView", "Part", "VectorView",
    "Workspace", "footprint", "gemm_a", "is_transposed", "kron1", "kron2", "kron2_parts", "kron3", "kron3_parts", "kron3_workspace_size", "last_path", "launch_count", "op_dims",
    "pooled_bytes", "release_buffers", "validate", "validate_batch", "version",
]
