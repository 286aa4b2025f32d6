"""paper_2407_07058_b200 -- all-points minimax path distance (APPD) on B200.

The hot path of arxiv 2407.07058 (Algorithm 4, "MMJ distance by Calculation and
Copy") re-designed for sm_100a: MST by Boruvka rounds -> edge sort ->
dendrogram (leaf order + merge heights) -> HBM-bandwidth-bound fill.  The work
runs in libappd.so (hand-written CUDA, C ABI in include/appd.h); this package
is the thin Python binding.
"""
from .binding import (  # noqa: F401
    AppdError,
    Context,
    VARIANT_AUTO,
    VARIANT_BORUVKA,
    VARIANT_PRIM,
    appd_create,
    appd_destroy,
    appd_get_nccl_unique_id,
    appd_row_range_of,
    appd_solve_points,
    appd_solve_weights,
    appd_version,
    load,
)
