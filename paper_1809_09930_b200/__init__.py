"""B200-native epsilon self-join (arxiv 1809.09930, GPU-Join).

Layout:
  csrc/          CUDA kernels (sm_100a) + the C ABI (include/gpujoin.h)
  gpujoin.py     ctypes binding (argument marshalling only)
  distributed.py entity partitioning over torch.distributed (NCCL)
  _build.py      in-tree nvcc build of libgpujoin.so
"""
from .gpujoin import Index, GpuJoinError, abi_version, lib, num_batches  # noqa: F401

__all__ = ["Index", "GpuJoinError", "abi_version", "lib", "num_batches"]
