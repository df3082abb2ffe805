"""B200-native (sm_100a) temporally fused LIF neurons -- arXiv 2408.00280.

Product path: ``libsnn_lif.so`` (include/snn_lif.h C ABI, CUDA kernels in csrc/) and the
thin Python layers over it (``lif`` functional API, ``autograd`` FusedLIF / LIFLayer,
``dist`` multi-GPU sharding and time-split).  Importing this package loads the CUDA
library and raises if it is missing: there is no CPU fallback.
"""
from . import _lib  # noqa: F401  (fails loudly when libsnn_lif.so is absent)
from .lif import LIFForward, LIFParams, lif_backward, lif_forward, unpack_bits  # noqa: F401
from .autograd import AffineLIFLayer, FusedAffineLIF, FusedLIF, LIFLayer  # noqa: F401
from .lif import AffineSpec, lif_backward_affine, lif_forward_affine  # noqa: F401
from .lif import host_workspace, lif_fwd_bwd_host  # noqa: F401
from .lif import LIFPlan  # noqa: F401

__all__ = ["LIFPlan", "LIFParams", "LIFForward", "lif_forward", "lif_backward", "unpack_bits",
           "FusedLIF", "LIFLayer", "FusedAffineLIF", "AffineLIFLayer", "AffineSpec",
           "lif_forward_affine", "lif_backward_affine", "host_workspace", "lif_fwd_bwd_host"]
