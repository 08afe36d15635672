"""B200-native balanced butterfly counting (arXiv 2308.07932 hot path).

The compute path is libbbf.so (CUDA, sm_100a, C ABI in include/bbf.h); `bbf` is its thin
ctypes binding.  Importing this package never imports the CPU oracle."""
from . import bbf  # noqa: F401
from .bbf import (  # noqa: F401
    BBFError, Comm, Graph, BBF_SIDE_U, BBF_SIDE_V, BBF_PTR_DEVICE, BBF_FORCE_SPARSE,
    BBF_FORCE_DENSE,
)
