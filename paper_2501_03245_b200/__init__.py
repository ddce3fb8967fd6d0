"""gecc-b200: batched elliptic-curve engine for NVIDIA B200 (sm_100a).

Python is only a thin ctypes view of ``lib/libgecc_b200.so`` (the product is the
CUDA library behind the C ABI in ``include/gecc_b200.h``).  There is no CPU
implementation here: importing works anywhere, but creating a Context needs the
compiled library and a CUDA device and raises loudly otherwise.
"""
from .capi import (BaseTable, Context, GeccError, LIB_PATH, SM2, SECP256K1, BLS12_381, BLS12_377, STATUS,
                   SECRET_FAST, SECRET_UNIFORM, COMM_ID_BYTES, lib, lib_available, cols_from_ints, ints_from_cols,
                   comm_unique_id, set_batch_form, set_msm_form, field_params_make, field_params_get)

__all__ = ["BaseTable", "Context", "GeccError", "LIB_PATH", "SM2", "SECP256K1", "BLS12_381", "BLS12_377", "STATUS",
           "SECRET_FAST", "SECRET_UNIFORM", "COMM_ID_BYTES", "lib", "lib_available", "cols_from_ints",
           "ints_from_cols", "comm_unique_id", "set_batch_form", "set_msm_form", "field_params_make", "field_params_get"]
__version__ = "0.1.0"
