"""paper_2605_29232_b200 -- B200-native (sm_100a) batched CVR scoring hot path.

The compute path lives in ``libcvr.so`` (CUDA C++, C ABI in ``include/cvr.h``); this package is
a thin ctypes binding (argument marshalling only, same names as the C entry points) plus the
host-side serving logic (``serving``: dynamic batcher, load generator) and the sharded-table
driver (``sharded``).  PyTorch is used only for device memory, streams and process groups.
There is no CPU fallback: if the extension is missing or no CUDA device is present the calls
raise.
"""
from ._cvr import (  # noqa: F401
    CVR_BF16, CVR_DCN_FULL, CVR_DCN_LOWRANK, CVR_ENSEMBLE, CVR_F16, CVR_F32, CVR_MASKNET, CvrError, CvrModel, gemm_bf16,
    lib, lib_path, status_string, text_ngram_keys, truncate_bags,
)

__all__ = ["CvrModel", "CvrError", "lib", "lib_path", "status_string", "text_ngram_keys", "truncate_bags"]
