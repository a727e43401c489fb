"""paper_1704_02457_b200: B200-native batched FP64 small-matrix BLAS/LAPACK
on BLASFEO's panel-major format (arXiv 1704.02457).

Drop-in for the reference ``panelblas`` hot path -- ``level3.gemm_nt /
syrk_ln / trsm_rltn / potrf_l`` and the ``pack`` conversions -- with a
leading batch dimension.  Device memory and streams come from PyTorch; all
arithmetic runs in hand-written sm_100a CUDA kernels behind the C ABI in
``include/pb_b200.h`` (``lib/libpb_b200.so``).  There is no CPU fallback.
"""
from . import fixtures, level3, pack
from ._native import lib_path, load as load_native
from .errors import (DimensionError, FactorizationError, MemoryLayoutError,
                     NotPositiveDefiniteError, PanelBlasError, SingularMatrixError)
from .matstore import (ALIGN, PS, DenseVectorBatch, PanelBatch, SubRef, allocate_panel_batch,
                       allocate_vector_batch, create_panel_batch, create_vector_batch, element_offset,
                       memsize_panel_batch, memsize_panel_matrix, memsize_split_batch, memsize_vector,
                       panel_data_elems)
from .pack import ColBatch

__version__ = "0.1.0"


def backend_name():
    """The reference exposes 'c' or 'py' (_backend/__init__.py:31-32); this engine has one backend."""
    return "cuda-sm100a"


__all__ = [
    "ALIGN", "PS", "ColBatch", "DenseVectorBatch", "PanelBatch", "SubRef", "allocate_panel_batch",
    "allocate_vector_batch", "backend_name", "create_panel_batch", "create_vector_batch", "element_offset",
    "fixtures", "level3", "lib_path", "load_native", "memsize_panel_batch", "memsize_panel_matrix",
    "memsize_split_batch", "memsize_vector", "pack", "panel_data_elems",
    "DimensionError", "FactorizationError", "MemoryLayoutError", "NotPositiveDefiniteError",
    "PanelBlasError", "SingularMatrixError",
]
