"""B200-native GRCA hot path (arxiv 2605.10457): CUDA kernels behind a C ABI.

``paper_2605_10457_b200.grca`` is the thin ctypes binding of include/grca.h;
``paper_2605_10457_b200.dist`` holds the multi-GPU sharding and merge plumbing
(torch.distributed, NCCL on GPU / gloo in CPU tests).
"""
from .grca import Grca, GrcaError, load, tris_to_float4, version  # noqa: F401
