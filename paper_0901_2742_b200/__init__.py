"""B200-native k-mer-rank domain decomposition of Sample-Align-D (arXiv 0901.2742).

The product is libsad.so (include/sad.h: hand-written sm_100a CUDA kernels behind a
C ABI); this package holds its ctypes binding (`_lib`) and the torch-based driver
(`runtime.Context`). There is no CPU fallback: without the built library or a GPU,
the calls raise.
"""
from ._lib import SadError, lib  # noqa: F401

__all__ = ["Context", "SadError", "lib"]


def __getattr__(name):
    if name == "Context":
        from .runtime import Context
        return Context
    raise AttributeError(name)
