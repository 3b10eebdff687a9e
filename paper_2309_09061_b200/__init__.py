"""B200-native adaptive H^2 x H^2 product (arXiv 2309.09061).

Drop-in for the hot path of the reference package h2mul: the same container names
(ClusterTree, BlockTree, ClusterBasis, H2Matrix) and the same entry points (multiply, coarsen,
recompress, build_product_block_tree), computed by hand-written FP64 CUDA kernels for sm_100a
behind the C ABI in include/h2g.h.
"""

from .errors import CudaError, InvalidInputError, StructureError
from .h2 import BasisProduct, ClusterBasis, H2Matrix, expand_basis, h2_matvec_host, storage_bytes, to_dense
from .trees import (BlockTree, ClusterTree, ColumnTree, build_block_tree, build_cluster_tree,
                    build_product_block_tree, same_cluster_tree, sparsity_constant)

# stage-level drop-ins (stages.py; reference h2mul/__init__.py:11-32), loaded with the native library
_STAGES = ("cluster_basis_product", "basis_weights", "total_weights", "compress_induced_row_basis",
           "compress_induced_col_basis", "assemble_product", "build_coarse_row_basis", "build_coarse_col_basis",
           "project_final", "coupling_norms", "nearfield_norms", "block_norms", "InducedBasisResult",
           "CoarsenState", "BasisWeights", "TotalWeights", "DeviceBasis", "DeviceMats")

__version__ = "0.1.0"


def __getattr__(name):
    # GPU entry points import the native binding lazily (the CPU test tier imports this package)
    if name in ("multiply", "coarsen", "recompress", "multiply_coarsen", "multiply_coarsen_packed"):
        from . import api
        return getattr(api, name)
    if name in ("estimate_relative_spectral_error", "h2_matvec", "h2_matvec_adjoint"):
        from . import errest
        return getattr(errest, name)
    if name in _STAGES:
        from . import stages
        return getattr(stages, name)
    if name in ("Context", "DeviceH2", "default_context"):
        from . import device
        return getattr(device, name)
    raise AttributeError(name)
