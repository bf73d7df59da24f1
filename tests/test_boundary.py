"""CPU checks of the C-ABI boundary: libmempool.so loads, exports every symbol
include/mempool.h declares, the binding covers exactly that set, and calls
that need no GPU behave (status strings; pool creation fails cleanly with no
device).  No compute calls -- those are the -m gpu parity tests."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mempool.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mp_[a-z0-9_]+)\s*\(", src)) - {"mp_addr"})


def test_header_declares_paper_api():
    names = declared()
    for api in ("alloc_mem", "free_mem", "insert", "match", "delete", "swap_out", "swap_in",
                "transfer", "transfer_with_insert", "evict"):
        assert f"mp_{api}" in names


def test_library_exports_every_declared_symbol():
    from paper_2406_17565_b200 import mempool as M
    lib = ctypes.CDLL(M.LIB_PATH)
    for name in declared():
        assert hasattr(lib, name), name
    assert sorted(M.SIGNATURES) == declared()


def test_status_strings_and_no_device():
    import torch
    from paper_2406_17565_b200 import mempool as M
    assert M._lib.mp_status_str(0) == b"MP_OK"
    assert M._lib.mp_status_str(-10) == b"MP_ERR_PREFIX_MISSING"
    for k, v in M.STATUS.items():
        assert M._lib.mp_status_str(k).decode().endswith(v)
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by -m gpu")
    with pytest.raises(M.MempoolError) as e:
        M.Pool(0, 0, 2, 2, 64, 16, 64)
    assert e.value.name in ("CUDA", "CONFIG")


def test_bad_config_rejected_before_cuda():
    from paper_2406_17565_b200 import mempool as M
    with pytest.raises(M.MempoolError) as e:
        M.Pool(0, 0, 0, 2, 64, 16, 64)            # zero layers
    assert e.value.name == "CONFIG"
    with pytest.raises(M.MempoolError) as e:
        M.Pool(0, 0, 2, 1, 1, 1, 64, elem_bytes=1)  # chunk 1 byte: not 16-B aligned
    assert e.value.name == "CONFIG"


def test_fast_binding_loads_and_reports_status():
    """The CPython binding of the per-request calls (csrc/pyfast.c) is built
    next to the library, links the same copy, and maps a non-OK status to
    MempoolError (a NULL pool handle is rejected before any CUDA call)."""
    import numpy as np
    from paper_2406_17565_b200 import mempool as M
    F = M._F
    for name in ("alloc_mem", "free_mem", "insert", "match", "unpin", "delete", "transfer",
                 "transfer_with_insert", "record_event", "wait_event", "sync"):
        assert callable(getattr(F, name)), name
    toks = np.arange(40, dtype=np.int32)
    calls = [
        lambda: F.alloc_mem(0, 4, M.HBM, 0),
        lambda: F.free_mem(0, np.zeros(2, np.uint64)),
        lambda: F.insert(0, toks, np.zeros(2, np.uint64), 0),
        lambda: F.match(0, toks, 0, 16),
        lambda: F.unpin(0, [1, 2]),
        lambda: F.delete(0, toks),
        lambda: F.transfer(0, 1, [1], None, 0, 0, 2, None),
        lambda: F.transfer_with_insert(0, 1, toks, [1, 2, 3], None, 0, b"x", 16),
        lambda: F.sync(0),
        # a non-positive block size sizes no output: rejected, no division
        lambda: F.match(0, toks, 0, 0),
        lambda: F.transfer_with_insert(0, 1, toks, [1], None, 0, None, -16),
    ]
    for c in calls:
        with pytest.raises(M.MempoolError) as e:
            c()
        assert e.value.name == "CONFIG"
    with pytest.raises((TypeError, ValueError)):
        F.free_mem(0, "not an addr list")
    with pytest.raises(M.MempoolError) as e:       # a handle that is not an int
        F.free_mem("not a pool", [1])
    assert e.value.name == "CONFIG"


def test_fast_binding_converts_inputs():
    """Lists, other integer dtypes, non-contiguous and 2-D arrays are
    converted (flattened, cast) before the C call -- the NULL handle then
    yields CONFIG, not a conversion error."""
    import numpy as np
    from paper_2406_17565_b200 import mempool as M
    F = M._F
    toks64 = np.arange(0, 96, dtype=np.int64)
    strided = np.arange(0, 192, dtype=np.int32)[::2]
    addrs = np.arange(12, dtype=np.uint64).reshape(3, 4)
    for toks in (list(range(48)), toks64, strided, toks64.reshape(6, 16)):
        for a in (addrs, addrs.T, [1, 2, 3], np.arange(3, dtype=np.int64)):
            with pytest.raises(M.MempoolError) as e:
                F.insert(0, toks, a, 0)
            assert e.value.name == "CONFIG"
    with pytest.raises(M.MempoolError) as e:
        F.transfer_with_insert(0, 1, strided, addrs.T, list(range(5, 17)), 0,
                               bytearray(b"pv"), 16)
    assert e.value.name == "CONFIG"
    # a given destination list names exactly one block per source block
    # (ADDR_COUNT, before the handle is looked at); no list: DST_GIVEN is
    # cleared, not read from an uninitialised buffer
    with pytest.raises(M.MempoolError) as e:
        F.transfer_with_insert(0, 1, strided, addrs.T, [5, 6], 0, None, 16)
    assert e.value.name == "ADDR_COUNT"
    with pytest.raises(M.MempoolError) as e:
        F.transfer(0, 1, [1, 2, 3], [7], 0, 0, 1, None)
    assert e.value.name == "ADDR_COUNT"
    for d in (None,):
        with pytest.raises(M.MempoolError) as e:
            F.transfer(0, 1, [1, 2, 3], d, M.XFER_DST_GIVEN, 0, 1, None)
        assert e.value.name == "CONFIG"


def test_nccl_arm_exports_every_declared_symbol():
    """libmempool_nccl.so (the paper's NCCL transport, comparison arm) loads
    without a GPU and exports what include/mempool_nccl.h declares."""
    src = open(os.path.join(ROOT, "include", "mempool_nccl.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = sorted(set(re.findall(r"\b(mp_nccl_[a-z0-9_]+)\s*\(", src)))
    from paper_2406_17565_b200 import nccl_arm as N
    lib = N.lib()
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(N.SIGNATURES) == names
    assert N.version() >= 22000
