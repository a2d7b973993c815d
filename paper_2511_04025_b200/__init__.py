"""B200-native shellular hot path: field -> shell mask -> six-load-case PCG -> C^H.

Host code over libshellular_cuda.so (hand-written sm_100a kernels behind the C
ABI in include/shellular_cuda.h).  ``api`` mirrors the reference's
``shellular`` namespace (proj/include/shellular/*.hpp).
"""
from .api import *  # noqa: F401,F403
from .api import (BaseMaterial, Context, DesignParams, GridSolver, HomogenizeOptions,  # noqa: F401
                  RandomDesignSpec, ShellParams, build_reduced_mesh, classify_surface_elements,
                  default_context, element_stiffness, expand_symmetry, homogenize,
                  homogenize_batch, random_design, sample_grid, sample_grid_fn)

__version__ = "0.1.0"
