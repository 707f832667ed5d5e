"""B200-native MPM-2P / MRCM velocity-update and saturation-update path.

Host mirror of the reference's C++ driver/solver API (arxiv/paper_2103_11050,
proj/include/mrcmflow/*.hpp) over the C ABI in include/mpm2p_b200.h, backed by
hand-written sm_100a CUDA kernels in csrc/.
"""
from .api import (  # noqa: F401
    ALPHA_ADAPTIVE, ALPHA_UNIFORM, EPS_ABSOLUTE, EPS_MOBILITY, EPS_RELATIVE, FINE_REFERENCE, FLUX,
    HBAR_HALF, HBAR_PER_EDGE, HBAR_SEGMENT, HBAR_WHOLE, MPM2P, MPM2P_NO_UPDATES, MRCM_EVERY_STEP,
    PRESSURE, SPACE_CONSTANT, SPACE_LINEAR, AlphaSpec, BoundarySpec, CapacityError, ConfigError,
    CudaError, GlobalSolution, NumericError, Problem, RunRecord, RunResult, Simulator,
    SplittingConfig, pressure_drop, product_lib, rcr, unit_inflow,
)
