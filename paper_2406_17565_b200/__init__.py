"""paper_2406_17565_b200 -- B200-native KV-block migration for MemServe's MemPool.

The hot path (§4 "Elastic Memory Pool", arXiv 2406.17565) lives in
``_lib/libmempool.so`` (C-ABI declared in ``include/mempool.h``): a device
bitmap block allocator, a host prompt (radix) index, sm_100a gather/scatter
kernels and the transfer / swap engines.  ``mempool`` is a thin ctypes
binding with the paper's API names.
"""
from .mempool import (  # noqa: F401
    HBM, DRAM, MIXED, XFER_DST_GIVEN, XFER_DEDUP, XFER_ASYNC, XFER_PIPELINE, INS_ERR_ON_CONFLICT, MATCH_PIN,
    PATH_AUTO, PATH_FUSED, PATH_STAGED, PATH_CE, SWAP_ZERO_COPY, SWAP_CE,
    MempoolError, Pool, connect, make_addr, addr_inst, addr_medium, addr_index,
    addr_indices, addr_media, LIB_PATH, SIGNATURES,
)
