"""B200-native fused warp + loss step (LNCC / Mattes MI) of FFDP (arXiv 2509.25044),
a drop-in for the voxreg reference's hot path. The compute path is libffdp.so
(sm_100a CUDA kernels behind the C ABI in include/ffdp.h); this package is the host
side: a mirror of voxreg's operator API (``voxreg``), the z-slab sharded driver
(``dist``) and the build recipe (``build``)."""
from ._lib import (CudaError, FabricError, FfdpError, InvalidArgument, LogicError)  # noqa: F401

__version__ = "0.1.0"
