"""B200-native hot path of arXiv 1504.03151 (per-pixel iterative ray tracing of spheres and
planes). The compute path is libb200rt.so (CUDA, sm_100a) behind the C ABI in include/rt.h;
`rt` is its ctypes binding and `multigpu` the torch.distributed (NCCL) sharding driver."""
from . import rt  # noqa: F401

__all__ = ["rt"]
