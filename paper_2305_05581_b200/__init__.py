"""B200-native H_eff·ψ / renormalization path of the sector-sparse two-site DMRG
(arxiv 2305.05581, reference package ``sector_dmrg``).

The product is the sm_100a C-ABI library ``lib/libsdmrg_b200.so``
(include/sdmrg_b200.h); this package is the host side mirroring the
reference's interfaces for that path:

  build_plan / apply_plan / DevicePlan   blocks.py:503, dmrg.py:107
  lanczos_ground                         dmrg.py:43
  sbmm4s, CudaGemm                       sbmm4s.py:167, gemm.py:53
  renormalize_store, rotate_operators,   dmrg.py:335, dmrg.py:254,
  reduced_density_matrix                 dmrg.py:221
"""

__version__ = "0.1.0"

from ._lib import LibraryError, SdmrgError, WorkspaceError, launch_count, load  # noqa: F401
from .plan_input import PlanInput, compile_reference_plan  # noqa: F401


def __getattr__(name):
    # torch-dependent modules load lazily so the CPU test-suite stays light
    if name in ("DevicePlan", "build_plan", "apply_plan", "apply_effective_hamiltonian"):
        from . import plan
        return getattr(plan, name)
    if name in ("lanczos_ground", "LanczosResult"):
        from . import lanczos
        return getattr(lanczos, name)
    if name in ("CudaGemm", "KernelCounter"):
        from . import gemm
        return getattr(gemm, name)
    if name in ("sbmm4s", "DeviceProblem", "flops_fused"):
        from . import sbmm4s
        return getattr(sbmm4s, name)
    if name in ("renormalize_store", "renormalize_blocks", "rotate_operators",
                "reduced_density_matrix", "rdm_eigensystem", "truncate"):
        from . import renorm
        return getattr(renorm, name)
    raise AttributeError(name)
