"""B200-native Flash HE-convolution hot path (arxiv 2401.16732).

Drop-in for the reference package `privinfer` (params, ring, bfv, conv,
errors) plus the SPEC's x^2+x share protocol (act2pc). All arithmetic runs
in hand-written sm_100a kernels in `libflashhe.so` behind a C ABI
(include/flashhe.h); the Python modules keep the reference's API.
"""

from . import errors, params  # noqa: F401  (host-only, importable without a GPU)

__all__ = ["errors", "params", "ring", "bfv", "conv", "act2pc"]


def __getattr__(name):
    if name in ("ring", "bfv", "conv", "act2pc", "device"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
