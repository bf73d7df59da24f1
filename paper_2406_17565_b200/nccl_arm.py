"""ctypes binding of libmempool_nccl.so (include/mempool_nccl.h): the paper's
NCCL send/recv transport as a comparison arm beside the
fused one-sided path.  Argument marshalling only.

    comm = NcclComm.create_single(device)           # one rank: self send/recv
    comm = NcclComm.create(world, rank, device, uid)  # uid from rank 0, any bootstrap
    comm.exchange(peer, send_ptrs, send_bytes, peer, recv_ptrs, recv_bytes, stream)
"""
import contextlib
import ctypes as C
import os
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libmempool_nccl.so")

SIGNATURES = {
    "mp_nccl_unique_id": (C.c_int, [C.c_void_p, C.c_int64]),
    "mp_nccl_comm_init": (C.c_int, [C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                    C.POINTER(C.c_void_p)]),
    "mp_nccl_comm_destroy": (None, [C.c_void_p]),
    "mp_nccl_exchange": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64,
                                   C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "mp_nccl_last_error": (C.c_char_p, []),
    "mp_nccl_version": (C.c_int32, []),
}


def load_library(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"{path} not found; build it with "
                          "`python paper_2406_17565_b200/build.py`")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = load_library()
    return _lib


class NcclError(RuntimeError):
    pass


def _check(r: int, where: str):
    if r != 0:
        raise NcclError(f"{where}: {lib().mp_nccl_last_error().decode()} ({r})")


def unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().mp_nccl_unique_id(buf, 128), "unique_id")
    return buf.raw


def version() -> int:
    return int(lib().mp_nccl_version())


@contextlib.contextmanager
def _stdout_to_stderr():
    """NCCL may print its version banner on stdout at communicator init;
    bench.py's stdout must carry exactly one JSON line."""
    sys.stdout.flush()
    saved = os.dup(1)
    try:
        os.dup2(2, 1)
        yield
    finally:
        libc = C.CDLL(None)
        libc.fflush(None)
        os.dup2(saved, 1)
        os.close(saved)


class NcclComm:
    def __init__(self, world: int, rank: int, device: int, uid: bytes):
        h = C.c_void_p()
        b = C.create_string_buffer(bytes(uid), 128)
        with _stdout_to_stderr():
            r = lib().mp_nccl_comm_init(world, rank, b, device, C.byref(h))
        _check(r, "comm_init")
        self._h = h
        self.rank = rank
        self.world = world

    @classmethod
    def create(cls, world: int, rank: int, device: int, uid: bytes):
        return cls(world, rank, device, uid)

    @classmethod
    def create_single(cls, device: int):
        return cls(1, 0, device, unique_id())

    def close(self):
        if getattr(self, "_h", None):
            lib().mp_nccl_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def exchange(self, peer_send: int, send_ptrs, send_bytes, peer_recv: int, recv_ptrs,
                 recv_bytes, stream: int = 0):
        """One NCCL group of sends to peer_send and recvs from peer_recv."""
        sp = np.ascontiguousarray(np.asarray(send_ptrs, dtype=np.uint64))
        sb = np.ascontiguousarray(np.asarray(send_bytes, dtype=np.int64))
        rp = np.ascontiguousarray(np.asarray(recv_ptrs, dtype=np.uint64))
        rb = np.ascontiguousarray(np.asarray(recv_bytes, dtype=np.int64))
        assert len(sp) == len(sb) and len(rp) == len(rb)
        _check(lib().mp_nccl_exchange(self._h, peer_send, sp.ctypes.data, sb.ctypes.data,
                                      len(sp), peer_recv, rp.ctypes.data, rb.ctypes.data,
                                      len(rp), C.c_void_p(stream)), "exchange")
