"""B200-native FSOFT / iFSOFT -- drop-in for the hot path of the reference `so3fft`.

Public names follow the reference's export table (pkg/src/so3fft/__init__.py:17-94)
for the transform path: containers and layouts (core), grid/weights, clusters and the
sigma / kappa work-index maps, make_plan / fsoft_* / ifsoft_*, the direct route and the
benchmark harness.  Compute runs in libso3fft_b200.so (hand-written
sm_100a CUDA, include/so3fft_b200.h); there is no CPU fallback.
"""

from __future__ import annotations

from .core import (
    FORMAT_VERSION,
    SOFC_MAGIC,
    SOFG_MAGIC,
    So3Coefficients,
    So3SampleGrid,
    coeff_count,
    coeff_index,
    container_info,
    degree_of_slots,
    grid_size,
    order_pair_slots,
    read_coefficients,
    read_samples,
    read_samples_slab,
    validate_bandwidth,
    write_coefficients,
    write_samples,
    write_samples_slab,
)
from .soft import (
    DIRECT_BANDWIDTH_CAP,
    fsoft_direct,
    ifsoft_direct,
    OrderPair,
    QuadratureWeights,
    SampleAngles,
    SymmetryCluster,
    TransformPlan,
    cluster_for_base,
    cluster_schedule,
    dwt_analysis,
    dwt_synthesis,
    enumerate_clusters,
    fft_analysis,
    fft_synthesis,
    fsoft_batch,
    fsoft_parallel,
    fsoft_sequential,
    ifsoft_batch,
    ifsoft_parallel,
    ifsoft_sequential,
    kappa_count,
    kappa_split,
    kappa_to_orders,
    make_plan,
    quadrature_weights,
    rect_to_orders,
    sample_angles,
    sigma_index,
    sigma_inverse,
    wigner_rows,
)
from .wigner import (
    SYMMETRY_RELATIONS,
    SymmetryRelation,
    WignerColumn,
    apply_symmetry,
    jacobi_poly,
    wigner_D,
    wigner_d_column,
    wigner_d_direct,
    wigner_d_seed,
)
from .dwt import (
    DwtScalers,
    WignerMatrix,
    build_wigner_matrix,
    derive_cluster_matrices,
    dwt_apply,
    idwt_apply,
    make_scalers,
)
from .report import (
    BenchConfig,
    BenchRecord,
    OracleMismatchError,
    error_metrics,
    random_coefficients,
    run_benchmark,
    write_report,
)

__version__ = "0.1.0"
