"""GESR MoA candidate scoring on B200 (arxiv 2511.21095): the hot path behind libgesr.so.

Python binding layer only (argument marshalling); every step of the path runs in the CUDA
kernels of ``csrc/`` behind the C ABI declared in ``include/gesr.h``.  The CUDA library is
loaded lazily on first use and its absence raises -- there is no CPU fallback.
"""
from .configs import CONFIGS, Config, get as get_config  # noqa: F401


def __getattr__(name):
    # lazy: importing configs/inputs must not require the CUDA library
    if name in ("kv_project", "tasa_score", "hma_count", "tasa_workspace_bytes", "lib",
                "GesrError", "status_string", "score_step"):
        from . import binding
        return getattr(binding, name)
    raise AttributeError(name)
