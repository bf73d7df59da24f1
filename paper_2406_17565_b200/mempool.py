"""Thin binding of libmempool.so (include/mempool.h): the per-request calls
through the CPython extension _mpfast (csrc/pyfast.c), the rest through ctypes.

Argument marshalling only: every step of the hot path runs in the library's
C++ runtime and sm_100a kernels.  There is no fallback -- importing this
module fails loudly when the library is missing.

Names follow the paper's MemPool API (PAPER.md Table tbl-mempool-api,
P:261-290): alloc_mem, free_mem, insert, match, delete, swap_out, swap_in,
transfer, transfer_with_insert (+ evict).
"""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libmempool.so")

HBM, DRAM, MIXED = 0, 1, 2
ALLOC_STREAM_ORDERED = 1 << 8

XFER_DST_GIVEN = 1 << 0
XFER_DEDUP = 1 << 1
XFER_ASYNC = 1 << 2
XFER_PIPELINE = 1 << 3
INS_ERR_ON_CONFLICT = 1 << 4
MATCH_PIN = 1 << 5
PATH_AUTO = 0 << 8
PATH_FUSED = 1 << 8
PATH_STAGED = 2 << 8
PATH_CE = 3 << 8
SWAP_ZERO_COPY = 1
SWAP_CE = 2

STATUS = {
    0: "OK", -1: "OOM", -2: "DOUBLE_FREE", -3: "INVALID_ADDR", -4: "ADDR_COUNT",
    -5: "CONFLICT", -6: "NO_DRAM", -7: "DST_OOM", -8: "DST_UNREACHABLE",
    -9: "PRECONDITION", -10: "PREFIX_MISSING", -11: "CONFIG", -12: "BUFFER_TOO_SMALL",
    -13: "CUDA", -14: "NCCL", -15: "INTERNAL",
}


class MempoolError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{where}: MP_ERR_{self.name}" + (f" ({detail})" if detail else ""))


def make_addr(inst: int, medium: int, idx: int) -> int:
    return (inst << 40) | ((medium & 0xFF) << 32) | (idx & 0xFFFFFFFF)


def addr_inst(a) -> int:
    return int(a) >> 40


def addr_medium(a) -> int:
    return (int(a) >> 32) & 0xFF


def addr_index(a) -> int:
    return int(a) & 0xFFFFFFFF


def addr_indices(addrs) -> np.ndarray:
    return (np.asarray(addrs, np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.int64)


def addr_media(addrs) -> np.ndarray:
    return ((np.asarray(addrs, np.uint64) >> np.uint64(32)) & np.uint64(0xFF)).astype(np.int64)


class PoolConfig(C.Structure):
    _fields_ = [
        ("instance_id", C.c_int32), ("device", C.c_int32), ("layers", C.c_int32),
        ("kv_heads", C.c_int32), ("head_dim", C.c_int32), ("elem_bytes", C.c_int32),
        ("block_tokens", C.c_int32), ("verify", C.c_int32),
        ("hbm_blocks", C.c_int64), ("dram_blocks", C.c_int64),
        ("slabs", C.POINTER(C.c_void_p)), ("dram_base", C.c_void_p),
        ("staging_bytes", C.c_int64), ("staging_slots", C.c_int32), ("max_ctas", C.c_int32),
        ("copy_kernel", C.c_int32), ("coalesce_mib", C.c_int32),
        ("peer_engine", C.c_int32), ("peer_sched", C.c_int32), ("force_peer", C.c_int32),
    ]


class PoolInfo(C.Structure):
    _fields_ = [
        ("chunk_bytes", C.c_int64), ("block_bytes", C.c_int64), ("hbm_blocks", C.c_int64),
        ("dram_blocks", C.c_int64), ("hbm_free", C.c_int64), ("dram_free", C.c_int64),
        ("index_blocks", C.c_int64), ("clock", C.c_uint64), ("epoch", C.c_uint64),
        ("instance_id", C.c_int32), ("device", C.c_int32), ("layers", C.c_int32),
        ("block_tokens", C.c_int32),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("kernel_launches", C.c_uint64), ("bytes_moved", C.c_uint64),
        ("blocks_moved", C.c_uint64), ("kernel_ms", C.c_double),
        ("timed_launches", C.c_uint64), ("timed_bytes", C.c_uint64),
        ("aux_launches", C.c_uint64), ("gap_ms", C.c_double),
        ("profiled_launches", C.c_uint64), ("profiled_bytes", C.c_uint64),
        ("overlapped_launches", C.c_uint64),
    ]


class RecvMsg(C.Structure):
    _fields_ = [("kind", C.c_int32), ("src_instance", C.c_int32), ("n_addrs", C.c_int64),
                ("priv_len", C.c_int64)]


_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_U32 = C.c_uint32
_U64 = C.c_uint64
# array arguments travel as plain addresses (c_void_p): numpy's
# `a.ctypes.data` is half the cost of building a typed ctypes pointer
_PU64 = C.c_void_p
_PI32 = C.c_void_p
_PI64 = C.POINTER(C.c_int64)

# name -> (restype, argtypes); the list is also the export check of the tests.
SIGNATURES = {
    "mp_pool_create": (_I32, [C.POINTER(PoolConfig), C.POINTER(_P)]),
    "mp_pool_destroy": (None, [_P]),
    "mp_connect": (_I32, [_P, _P]),
    "mp_pool_info_get": (_I32, [_P, C.POINTER(PoolInfo)]),
    "mp_sync": (_I32, [_P]),
    "mp_wait_event": (_I32, [_P, _P]),
    "mp_record_event": (_I32, [_P, _P]),
    "mp_status_str": (C.c_char_p, [_I32]),
    "mp_last_error": (C.c_char_p, []),
    "mp_alloc_mem": (_I32, [_P, _I64, _I32, _I32, _PU64]),
    "mp_free_mem": (_I32, [_P, _PU64, _I64]),
    "mp_insert": (_I32, [_P, _PI32, _I64, _PU64, _I64, _U32, _PI64]),
    "mp_match": (_I32, [_P, _PI32, _I64, _U32, _PU64, _I64, _PI64]),
    "mp_unpin": (_I32, [_P, _PU64, _I64]),
    "mp_delete": (_I32, [_P, _PI32, _I64]),
    "mp_evict": (_I32, [_P, _I64, _I32, _PU64, _PI64]),
    "mp_swap_out": (_I32, [_P, _I64, _U32, _PU64, _PU64, _PI64]),
    "mp_swap_in": (_I32, [_P, _PU64, _I64, _U32, _PU64]),
    "mp_transfer": (_I32, [_P, _I32, _PU64, _I64, _PU64, _U32, _I32, _I32, _P, _I64]),
    "mp_transfer_with_insert": (_I32, [_P, _I32, _PI32, _I64, _PU64, _I64, _PU64, _U32, _P,
                                       _I64, _PI64]),
    "mp_recv_poll": (_I32, [_P, C.POINTER(RecvMsg), _P, _I64, _PU64, _I64]),
    "mp_transfer_heads": (_I32, [_P, _I32, _PU64, _I64, _PU64, _U32, _I32, _I32, _I32, _I32,
                                 _I32]),
    "mp_tp_plan": (_I32, [_I32, _I32, _I32, _PI32, _I64, _PI64]),
    "mp_gs_create": (_I32, [_I32, C.c_double, C.POINTER(_P)]),
    "mp_gs_destroy": (None, [_P]),
    "mp_gs_register": (_I32, [_P, _I32, _I32]),
    "mp_gs_set_load": (_I32, [_P, _I32, C.c_double]),
    "mp_gs_update": (_I32, [_P, _I32, _PI32, _I64, C.c_double]),
    "mp_gs_route": (_I32, [_P, _I32, _PI32, _I64, C.c_double, _PI32, _PI64, _PI32, _PI64, _I64,
                           _PI64]),
    "mp_export_handle": (_I32, [_P, _P, _I64, _PI64]),
    "mp_import_peer": (_I32, [_P, _P, _I64]),
    "mp_serve": (_I32, [_P, _I64, _I32, _PI64, _PI32]),
    "mp_send_mark": (_I32, [_P, _I32, _I32]),
    "mp_debug_channel_selftest": (_I32, [C.c_char_p, _I32, _I64, _I64]),
    "mp_pack": (_I32, [_P, _PU64, _I64, _I32, _I32, _P]),
    "mp_unpack": (_I32, [_P, _P, _PU64, _I64, _I32, _I32]),
    "mp_profile": (_I32, [_P, _I32]),
    "mp_stats_get": (_I32, [_P, C.POINTER(Stats)]),
    "mp_stats_reset": (_I32, [_P]),
    "mp_debug_fill": (_I32, [_P, _PU64, _I64, _U64]),
    "mp_debug_read_block": (_I32, [_P, _U64, _P, _I64]),
    "mp_debug_dump_index": (_I32, [_P, C.c_char_p, _I64, _PI64]),
    "mp_debug_block_states": (_I32, [_P, _I32, C.POINTER(C.c_uint8), _I64]),
    "mp_debug_bitmap": (_I32, [_P, C.POINTER(C.c_uint32), _I64]),
}


def load_library(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"libmempool.so not found at {path}; build it with "
            "`python paper_2406_17565_b200/build.py` (there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = load_library()


def load_fast(libdir: str = os.path.dirname(LIB_PATH)):
    """The CPython binding of the per-request calls (csrc/pyfast.c); built
    next to the library by build.py.  No ctypes fallback: a missing binding
    fails loudly like a missing library."""
    import importlib.machinery
    import importlib.util
    for suffix in importlib.machinery.EXTENSION_SUFFIXES:
        path = os.path.join(libdir, "_mpfast" + suffix)
        if os.path.exists(path):
            spec = importlib.util.spec_from_file_location("_mpfast", path)
            mod = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(mod)
            return mod
    raise ImportError(f"_mpfast binding not found in {libdir}; build it with "
                      "`python paper_2406_17565_b200/build.py`")


_F = load_fast()


def _check(st: int, where: str):
    if st != 0:
        detail = _lib.mp_last_error().decode() if st in (-13, -14, -15) else ""
        raise MempoolError(st, where, detail)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64).reshape(-1))


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(-1))


def _pu64(a: np.ndarray):
    return a.ctypes.data


def _pi32(a: np.ndarray):
    return a.ctypes.data


def _event_handle(event) -> int:
    """cudaEvent_t of a torch.cuda.Event (created on first record) or an int."""
    if isinstance(event, int):
        return event
    if not getattr(event, "cuda_event", 0):
        event.record()      # torch creates the CUDA event lazily, on first record
    return int(event.cuda_event)


def _raise_factory(status: int, where: str):
    detail = _lib.mp_last_error().decode() if status in (-13, -14, -15) else ""
    return MempoolError(status, where, detail)


_F.set_error_factory(_raise_factory)


class Pool:
    """One serving instance's MemPool."""

    def __init__(self, instance_id: int, device: int, layers: int, kv_heads: int,
                 head_dim: int, block_tokens: int, hbm_blocks: int, dram_blocks: int = 0,
                 elem_bytes: int = 2, slabs=None, dram_base=None, staging_bytes: int = 0,
                 staging_slots: int = 0, max_ctas: int = 0, verify: bool = False,
                 copy_kernel: int = 0, coalesce_mib: int = 0, peer_engine: int = 0,
                 peer_sched: int = 0, force_peer: bool = False):
        self.inst = instance_id
        self.B = block_tokens
        self.L = layers
        self._slab_arr = None
        cfg = PoolConfig(instance_id, device, layers, kv_heads, head_dim, elem_bytes,
                         block_tokens, int(verify), hbm_blocks, dram_blocks, None,
                         dram_base, staging_bytes, staging_slots, max_ctas, copy_kernel,
                         coalesce_mib, peer_engine, peer_sched, int(force_peer))
        if slabs is not None:
            assert len(slabs) == 2 * layers
            self._slab_arr = (C.c_void_p * len(slabs))(*[int(s) for s in slabs])
            cfg.slabs = C.cast(self._slab_arr, C.POINTER(C.c_void_p))
        h = C.c_void_p()
        _check(_lib.mp_pool_create(C.byref(cfg), C.byref(h)), "mp_pool_create")
        self._h = h
        self._hv = h.value      # the handle as an int, for the _mpfast calls
        info = self.info()
        self.chunk_bytes = info.chunk_bytes
        self.block_bytes = info.block_bytes
        self.hbm_blocks = info.hbm_blocks
        self.dram_blocks = info.dram_blocks

    def close(self):
        if getattr(self, "_h", None):
            _lib.mp_pool_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def sync(self):
        """Wait for all device work issued on this pool (mp_sync)."""
        _F.sync(self._hv)

    def wait_event(self, event):
        """Later device work of this pool waits for a CUDA event (e.g. a
        torch.cuda.Event recorded after the engine wrote the KV)."""
        _F.wait_event(self._hv, _event_handle(event))

    def record_event(self, event):
        """Record a CUDA event after all work issued on this pool so far."""
        _F.record_event(self._hv, _event_handle(event))

    def info(self) -> PoolInfo:
        o = PoolInfo()
        _check(_lib.mp_pool_info_get(self._h, C.byref(o)), "mp_pool_info_get")
        return o

    # -------------------------------------------------------------- memory API
    def alloc_mem(self, n: int, medium: int = HBM, requester: int = None,
                  stream_ordered: bool = False) -> np.ndarray:
        """stream_ordered: no drain; order the caller's writes after an event
        from record_event (MP_ALLOC_STREAM_ORDERED, include/mempool.h)."""
        return _F.alloc_mem(self._hv, n, medium | (ALLOC_STREAM_ORDERED if stream_ordered else 0),
                            self.inst if requester is None else requester)

    def free_mem(self, addrs):
        _F.free_mem(self._hv, addrs)

    # --------------------------------------------------------------- index API
    def insert(self, tokens, addrs, flags: int = 0) -> int:
        return _F.insert(self._hv, tokens, addrs, flags)

    def match(self, tokens, flags: int = 0):
        return _F.match(self._hv, tokens, flags, self.B)

    def unpin(self, addrs):
        _F.unpin(self._hv, addrs)

    def delete(self, tokens):
        _F.delete(self._hv, tokens)

    def evict(self, n: int, medium: int = HBM) -> np.ndarray:
        out = np.zeros(max(n, 1), np.uint64)
        k = C.c_int64(0)
        _check(_lib.mp_evict(self._h, n, medium, _pu64(out), C.byref(k)), "evict")
        return out[: k.value]

    # ---------------------------------------------------------------- swap API
    def swap_out(self, n: int, flags: int = 0):
        old = np.zeros(max(n, 1), np.uint64)
        new = np.zeros(max(n, 1), np.uint64)
        k = C.c_int64(0)
        _check(_lib.mp_swap_out(self._h, n, flags, _pu64(old), _pu64(new), C.byref(k)),
               "swap_out")
        return old[: k.value], new[: k.value]

    def swap_in(self, addrs, flags: int = 0) -> np.ndarray:
        a = _u64(addrs)
        out = np.zeros(max(len(a), 1), np.uint64)
        _check(_lib.mp_swap_in(self._h, _pu64(a), len(a), flags, _pu64(out)), "swap_in")
        return out[: len(a)]

    # --------------------------------------------------------- distributed API
    def transfer(self, dst_instance: int, src_addrs, dst_addrs=None, flags: int = 0,
                 layer_begin: int = 0, layer_end: int = None, priv: bytes = b"") -> np.ndarray:
        return _F.transfer(self._hv, dst_instance, src_addrs, dst_addrs, flags, layer_begin,
                           self.L if layer_end is None else layer_end, priv or None)

    def transfer_with_insert(self, dst_instance: int, tokens, src_addrs, dst_addrs=None,
                             flags: int = 0, priv: bytes = b""):
        return _F.transfer_with_insert(self._hv, dst_instance, tokens, src_addrs, dst_addrs, flags,
                                       priv or None, self.B)

    def recv_poll(self):
        """Oldest delivered message (kind, src_instance, private, addrs) or None."""
        return _F.recv_poll(self._hv)

    def transfer_heads(self, dst_instance: int, src_addrs, dst_addrs, src_head0: int,
                       dst_head0: int, n_heads: int, layer_begin: int = 0,
                       layer_end: int = None, flags: int = 0):
        """Head-range copy between tensor-parallel shards."""
        s, d = _u64(src_addrs), _u64(dst_addrs)
        le = self.L if layer_end is None else layer_end
        _check(_lib.mp_transfer_heads(self._h, dst_instance, _pu64(s), len(s), _pu64(d), flags,
                                      src_head0, dst_head0, n_heads, layer_begin, le),
               "transfer_heads")

    # ------------------------------------------- multi-process (one per GPU)
    def export_handle(self) -> bytes:
        n = C.c_int64(0)
        _lib.mp_export_handle(self._h, None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value)
        _check(_lib.mp_export_handle(self._h, buf, n.value, C.byref(n)), "export_handle")
        return buf.raw[: n.value]

    def import_peer(self, blob: bytes):
        b = C.create_string_buffer(bytes(blob), len(blob))
        _check(_lib.mp_import_peer(self._h, b, len(blob)), "import_peer")

    def serve(self, timeout_ms: int = -1, until_mark: bool = True):
        """Run the receiver's half of remote transfers; returns (served, mark)."""
        served = C.c_int64(0)
        mark = C.c_int32(-1)
        _check(_lib.mp_serve(self._h, timeout_ms, int(until_mark), C.byref(served),
                             C.byref(mark)), "serve")
        return served.value, (None if mark.value < 0 else mark.value)

    def send_mark(self, dst_instance: int, tag: int):
        _check(_lib.mp_send_mark(self._h, dst_instance, tag), "send_mark")

    # ----------------------------------------------------- building blocks
    def pack(self, addrs, layer_begin: int, layer_end: int, staging_ptr: int):
        a = _u64(addrs)
        _check(_lib.mp_pack(self._h, _pu64(a), len(a), layer_begin, layer_end,
                            C.c_void_p(staging_ptr)), "pack")

    def unpack(self, staging_ptr: int, addrs, layer_begin: int, layer_end: int):
        a = _u64(addrs)
        _check(_lib.mp_unpack(self._h, C.c_void_p(staging_ptr), _pu64(a), len(a), layer_begin,
                              layer_end), "unpack")

    # ---------------------------------------------------- measurement / debug
    def profile(self, enable: bool = True, every: int = 1):
        """Time every `every`-th migration launch with CUDA events (mp_profile)."""
        _check(_lib.mp_profile(self._h, int(every) if enable else 0), "profile")

    def stats(self) -> dict:
        s = Stats()
        _check(_lib.mp_stats_get(self._h, C.byref(s)), "stats")
        return {k: getattr(s, k) for k, _ in Stats._fields_}

    def stats_reset(self):
        _check(_lib.mp_stats_reset(self._h), "stats_reset")

    def debug_fill(self, addrs, seed: int):
        a = _u64(addrs)
        _check(_lib.mp_debug_fill(self._h, _pu64(a), len(a), seed), "debug_fill")

    def debug_read_block(self, addr) -> np.ndarray:
        out = np.zeros(self.block_bytes // 8, np.uint64)
        _check(_lib.mp_debug_read_block(self._h, int(addr), out.ctypes.data_as(C.c_void_p),
                                        self.block_bytes), "debug_read_block")
        return out.reshape(2 * self.L, -1)

    def dump_index(self):
        n = C.c_int64(0)
        _lib.mp_debug_dump_index(self._h, None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value + 1)
        _check(_lib.mp_debug_dump_index(self._h, buf, n.value + 1, C.byref(n)), "dump_index")
        rows = []
        for line in buf.value.decode().splitlines():
            depth, med, idx, la, ref, term, toks = line.split("\t")
            rows.append((tuple(int(x) for x in toks.split(",")), int(med), int(idx), int(la),
                         int(ref), term == "1"))
        return sorted(rows)

    def block_states(self, medium: int = HBM) -> np.ndarray:
        n = self.hbm_blocks if medium == HBM else self.dram_blocks
        out = np.zeros(max(n, 1), np.uint8)
        _check(_lib.mp_debug_block_states(self._h, medium,
                                          out.ctypes.data_as(C.POINTER(C.c_uint8)), len(out)),
               "block_states")
        return out[:n]

    def bitmap(self) -> np.ndarray:
        nw = (self.hbm_blocks + 31) // 32
        out = np.zeros(nw, np.uint32)
        _check(_lib.mp_debug_bitmap(self._h, out.ctypes.data_as(C.POINTER(C.c_uint32)), nw),
               "bitmap")
        return out


def connect(a: Pool, b: Pool):
    _check(_lib.mp_connect(a.handle, b.handle), "connect")


class GlobalScheduler:
    """Global prompt trees + locality-aware routing, mp_gs_*."""

    PREFILL, DECODE, COLOCATED = 0, 1, 2

    def __init__(self, block_tokens: int, ttl_seconds: float):
        h = C.c_void_p()
        _check(_lib.mp_gs_create(block_tokens, ttl_seconds, C.byref(h)), "mp_gs_create")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _lib.mp_gs_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def register(self, instance: int, kind: int):
        _check(_lib.mp_gs_register(self._h, instance, kind), "gs_register")
        self._n_inst = getattr(self, "_n_inst", 0) + 1

    def set_load(self, instance: int, load: float):
        _check(_lib.mp_gs_set_load(self._h, instance, load), "gs_set_load")

    def update(self, instance: int, tokens, now: float):
        t = _i32(tokens)
        _check(_lib.mp_gs_update(self._h, instance, _pi32(t), len(t), now), "gs_update")

    def route(self, kind: int, tokens, now: float):
        """-> (instance, matched_tokens, [(extra_instance, its_prefix_tokens), ...])"""
        t = _i32(tokens)
        inst = C.c_int32(-1)
        mt = C.c_int64(0)
        n = C.c_int64(0)
        cap = max(getattr(self, "_n_inst", 0), 1)   # extra holders <= registered instances
        ei = np.zeros(cap, np.int32)
        et = np.zeros(cap, np.int64)
        _check(_lib.mp_gs_route(self._h, kind, _pi32(t), len(t), now, C.byref(inst),
                                C.byref(mt), _pi32(ei), et.ctypes.data_as(_PI64), cap,
                                C.byref(n)), "gs_route")
        return inst.value, mt.value, [(int(ei[i]), int(et[i])) for i in range(n.value)]


def tp_plan(H: int, p: int, q: int):
    """Pieces (src_rank, dst_rank, src_head0, dst_head0, n_heads) of a TP=p ->
    TP=q repartition of H KV heads (mp_tp_plan)."""
    k = C.c_int64(0)
    _check(_lib.mp_tp_plan(H, p, q, None, 0, C.byref(k)), "tp_plan")
    out = np.zeros(5 * max(k.value, 1), np.int32)
    _check(_lib.mp_tp_plan(H, p, q, out.ctypes.data, k.value, C.byref(k)), "tp_plan")
    return [tuple(int(x) for x in out[5 * i: 5 * i + 5]) for i in range(k.value)]


def repartition(src_shards, dst_shards, src_addrs_per_shard, dst_addrs_per_shard, H: int,
                layer_begin: int = 0, layer_end: int = None, flags: int = 0):
    """TP=p -> TP=q move of the same blocks ("the sender partitions its
    local cache and invokes the appropriate network primitives"): one
    transfer_heads per plan piece.  Block ids are per shard (each shard's own
    allocation); addrs lists are aligned block by block."""
    for r, s, h0, g0, k in tp_plan(H, len(src_shards), len(dst_shards)):
        src_shards[r].transfer_heads(dst_shards[s].inst, src_addrs_per_shard[r],
                                     dst_addrs_per_shard[s], h0, g0, k, layer_begin,
                                     layer_end, flags)


def channel_selftest(name: str, role: int, n_msgs: int, payload: int):
    """Mailbox self-test (no GPU): run role 0 and role 1 in two processes."""
    _check(_lib.mp_debug_channel_selftest(name.encode(), role, n_msgs, payload),
           "channel_selftest")


def exchange_handles(pool: Pool, group=None) -> dict:
    """Bootstrap over torch.distributed: every rank exports its pool and
    gathers everyone's blob (plumbing only; returns {rank: blob})."""
    import torch.distributed as dist
    blob = pool.export_handle()
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, (pool.inst, blob), group=group)
    return {r: v for r, v in enumerate(out)}
