"""ctsm-b200: B200-native consistent fan/cone-beam CT system matrix
(arXiv 2511.12235), a drop-in for the reference's projector hot path.

Host mirror of the reference API (``ctsm::`` in /root/reference/proj/include)
over the C-ABI library libctsm_b200.so (include/ctsm_b200.h).
"""
from .geometry import CONFIGS, TEST_GEOMETRIES, CtsmError, ScanGeometry  # noqa: F401
from .projector import (  # noqa: F401
    Context,
    MatrixMode,
    SparseSystemMatrix,
    angle_block_entries,
    angle_column_sums,
    back_project,
    back_project_matrix_free,
    build_system_matrix,
    build_transpose,
    drop_transpose,
    forward_project,
    forward_project_matrix_free,
    matrix_mode_name,
    parse_matrix_mode,
    pixel_area_factors,
    scale_values,
    sirt,
    spectral_norm_power,
    voxel_volume_factors,
    weights_batch,
)

__version__ = "0.1.0"
