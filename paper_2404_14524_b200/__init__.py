"""paper_2404_14524_b200 — B200-native (sm_100a) hot path of Nys-IP-PMM (arXiv 2404.14524).

The product is the C-ABI library libnysipm.so (include/nysipm.h); this package holds its
CUDA sources (csrc/), the in-tree build script and a thin ctypes binding with the same
call names as the ABI.  It never imports the CPU oracle (oracle/), and has no CPU fallback.
"""
from ._lib import (Context, LoopbackComm, NysError, colmajor_device, load_library, LIB_PATH, EXPORTED,  # noqa: F401
                   SketchInfo, PcgInfo, nccl_unique_id)
