"""B200-native sparse-grid time-discontinuous Galerkin streamline-diffusion solver.

Thin Python binding of libsg.so (include/sg.h): argument marshalling only.
Every step of the method runs in the CUDA kernels of libsg.so; if the library
is missing or no CUDA device is present the calls raise (there is no CPU
fallback).  PyTorch is used for device memory and the stream only.
"""
from .binding import (  # noqa: F401
    SGError,
    Problem,
    config_from_dict,
    lib_path,
    load_library,
)
