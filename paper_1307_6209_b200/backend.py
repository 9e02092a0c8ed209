"""Kernel backend selection, drop-in for ``sellkit.backend``
(/root/reference/pkg/src/sellkit/backend.py:12-47).

This package ships exactly one kernels module, ``kernels_cuda`` (NAME
"cuda"), which implements the reference's seven-attribute protocol on the
GPU.  There is no CPU fallback: ``get_kernels()`` raises ResourceError when
the CUDA library or a device is unavailable, and asking for the reference's
CPU backends ("compiled", "python") is a ResourceError too -- use the
reference package itself for those.

``SELLKIT_BACKEND`` is honoured for the values this package can serve
("auto", "", "cuda"); anything else raises at selection time.
"""

import os

from .errors import ParameterError, ResourceError

_requested = os.environ.get("SELLKIT_BACKEND", "auto").strip().lower()

NAME_CUDA = "cuda"
BACKEND_NAME = NAME_CUDA


def cuda_kernels():
    from . import kernels_cuda
    return kernels_cuda


def _has_cuda():
    try:
        from . import _lib
        return _lib.device_count() > 0
    except ResourceError:
        return False


def __getattr__(name):
    # HAS_COMPILED / HAS_CUDA are evaluated lazily: loading the library must
    # not be a side effect of importing the package on a CPU-only host.
    if name in ("HAS_COMPILED", "HAS_CUDA"):
        return _has_cuda()
    raise AttributeError(name)


def kernels():
    """The default kernels module (backend.py:27)."""
    if _requested not in ("auto", "", "cuda"):
        raise ResourceError(
            f"SELLKIT_BACKEND={_requested!r} is not served by the sell-b200 "
            "package (only 'cuda')")
    return cuda_kernels()


def get_kernels(name=None):
    """Kernel module by name (backend.py:32-47): None / 'auto' / 'cuda'."""
    if name in (None, "auto", NAME_CUDA):
        from . import _lib
        _lib.require_device()
        return cuda_kernels()
    if name in ("python", "pure", "compiled"):
        raise ResourceError(
            f"the {name!r} CPU backend is not part of the sell-b200 package; "
            "this backend runs on the GPU only")
    raise ParameterError(f"unknown backend name: {name!r}")
