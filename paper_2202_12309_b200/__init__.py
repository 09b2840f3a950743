"""B200-native Parthenon-hydro hot path (arXiv 2202.12309, §4.1): a C-ABI CUDA library
(``libph.so``, built from ``csrc/`` for sm_100a) and its thin ctypes binding.

Every step of the per-cycle update runs in the library's kernels; this package only
marshals arguments and provides PyTorch plumbing (device allocator, stream, process group).
There is no CPU fallback: if ``libph.so`` is missing the import fails loudly.
"""
from .ph import Mesh, PhError, lib, PERIODIC, OUTFLOW, REFLECT, MINMOD, VANLEER, MC, PPM, WENOZ, RK2, VL2  # noqa: F401
from .ph import LINEAR_WAVE, SOD, BLAST, KH, REF_NONE, REF_STATIC, REF_ADAPTIVE  # noqa: F401
from .ph import HALO_AUTO, HALO_NCCL, HALO_PEER, DAVIS, EINFELDT  # noqa: F401
