"""B200-native MERF baked-scene renderer (arXiv 2302.12249): C-ABI libmerf.so (hand-written
sm_100a CUDA) + a thin ctypes binding.  See include/merf.h and DESIGN.md."""
from .merf import *  # noqa: F401,F403
from .merf import Scene, MerfError, lib, LIB_PATH  # noqa: F401
