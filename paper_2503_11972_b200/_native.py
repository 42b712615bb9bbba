"""ctypes binding of libmodmcache.so (the C ABI in include/modmcache.h).

There is no fallback: if the shared library is missing or no sm_100 device is
present, every call raises ``NativeError``.  ``DeviceRing`` is the thin
object the drop-in ``SemanticCache`` drives; it holds one native handle.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libmodmcache.so"

MC_FLAG_HIT = 0x01
MC_FLAG_EMPTY = 0x02
MC_FLAG_TIE = 0x04
MC_FLAG_NEAR_TIE = 0x08
MC_FLAG_NEAR_TAU = 0x10
MC_FLAG_FALLBACK = 0x20
MC_FLAG_NONFINITE = 0x40
MC_FLAG_NEED_RESCAN = 0x80  # merge of mc_retrieve_local_submit records: run rescan_local, gather, merge again

PATH_AUTO, PATH_GEMV, PATH_GEMM, PATH_STREAM8 = 0, 1, 2, 6

RECORD_DTYPE = np.dtype([("sim", "<f8"), ("second", "<f8"), ("pos", "<i8"), ("flags", "<u4"), ("reserved", "<i4")])
# struct mc_decision (include/modmcache.h)
DECISION_DTYPE = np.dtype([("live", "<i8"), ("similarity", "<f8"), ("sigma", "<f8"), ("k", "<i4"), ("steps", "<i4"),
                           ("flags", "<u4"), ("route", "<i4")])

EXPORTED = (
    "mc_create", "mc_destroy", "mc_set_thresholds", "mc_append", "mc_evict_front", "mc_size",
    "mc_retrieve_batch", "mc_set_path", "mc_configure_shard", "mc_retrieve_local_async",
    "mc_merge_records", "mc_stats", "mc_last_error", "mc_version", "mc_profile_steps", "mc_profile_rotate",
    "mc_debug_gemv_timing", "mc_retrieve_submit", "mc_retrieve_wait", "mc_debug_read_row",
    "mc_retrieve_decisions", "mc_set_sigma_schedule", "mc_generate_rows", "mc_read_rows", "mc_register_host",
    "mc_unregister_host", "mc_retrieve_local_device", "mc_merge_records_submit", "mc_merge_records_wait",
    "mc_retrieve_local_submit", "mc_rescan_local",
)


class NativeError(RuntimeError):
    """Raised for any failure inside libmodmcache (message from mc_last_error)."""


_lib = None


def _declare(lib):
    vp, i32, i64, dp = C.c_void_p, C.c_int32, C.c_int64, C.c_void_p
    lib.mc_create.argtypes = [C.POINTER(vp), i64, i32, i32]
    lib.mc_destroy.argtypes = [vp]
    lib.mc_set_thresholds.argtypes = [vp, dp, dp, i32, i32]
    lib.mc_append.argtypes = [vp, dp, i64]
    lib.mc_evict_front.argtypes = [vp, i64]
    lib.mc_size.argtypes = [vp]
    lib.mc_size.restype = i64
    lib.mc_retrieve_batch.argtypes = [vp, dp, i32, dp, dp, dp, dp]
    lib.mc_set_path.argtypes = [vp, i32]
    lib.mc_configure_shard.argtypes = [vp, i32, i32]
    lib.mc_retrieve_local_async.argtypes = [vp, dp, i32, vp, vp]
    lib.mc_merge_records.argtypes = [vp, vp, i32, i32, i64, vp, dp, dp, dp, dp]
    lib.mc_stats.argtypes = [vp, dp]
    lib.mc_profile_steps.argtypes = [vp, dp, dp, i32, i32, i64, dp, dp]
    lib.mc_profile_rotate.argtypes = [dp, i32, dp, dp, i32, i32, dp, dp]
    lib.mc_retrieve_submit.argtypes = [vp, dp, i32, dp]
    lib.mc_debug_read_row.argtypes = [vp, i64, dp]
    lib.mc_retrieve_wait.argtypes = [vp, C.c_uint32, dp, dp, dp, dp]
    lib.mc_debug_gemv_timing.argtypes = [dp, i32]
    lib.mc_retrieve_decisions.argtypes = [vp, dp, i32, dp]
    lib.mc_set_sigma_schedule.argtypes = [vp, dp, i32]
    lib.mc_generate_rows.argtypes = [vp, i64, dp, i32, C.c_double, C.c_double, C.c_uint64, i64]
    lib.mc_read_rows.argtypes = [vp, i64, i64, dp]
    lib.mc_register_host.argtypes = [vp, i64]
    lib.mc_retrieve_local_device.argtypes = [vp, vp, i32, vp, vp]
    lib.mc_unregister_host.argtypes = [vp]
    lib.mc_merge_records_submit.argtypes = [vp, vp, i32, i32, i64, vp, i32]
    lib.mc_merge_records_wait.argtypes = [vp, i32, dp, dp, dp, dp]
    lib.mc_retrieve_local_submit.argtypes = [vp, dp, i32, vp, vp]
    lib.mc_rescan_local.argtypes = [vp, dp, i32, vp, vp]
    lib.mc_last_error.restype = C.c_char_p
    lib.mc_version.restype = C.c_char_p
    return lib


def load(path: str | os.PathLike | None = None):
    """Load (once) and return the native library; raises NativeError if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # MODMCACHE_LIB: an alternative build of the same library (A/B kernel measurements only)
    p = Path(path) if path else Path(os.environ.get("MODMCACHE_LIB") or LIB_PATH)
    if not p.exists():
        raise NativeError(
            f"{p} is missing: build it with `python -m paper_2503_11972_b200.build` "
            "(there is no CPU fallback for the retrieval path)"
        )
    try:
        lib = _declare(C.CDLL(str(p)))
    except OSError as exc:
        raise NativeError(f"cannot load {p}: {exc}") from exc
    if path is None:
        _lib = lib
    return lib


def _check(lib, rc: int) -> None:
    if rc != 0:
        raise NativeError(f"libmodmcache error {rc}: {lib.mc_last_error().decode(errors='replace')}")


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


_registered: dict = {}  # buffer address -> the array (kept alive while registered)


def register_host(arr: np.ndarray) -> None:
    """Page-lock a C-contiguous float64 array so batched lookups DMA straight from it
    (mc_register_host); idempotent."""
    if not arr.flags["C_CONTIGUOUS"]:
        raise ValueError("register_host needs a C-contiguous array")
    addr = arr.ctypes.data
    if addr in _registered:
        return
    lib = load()
    _check(lib, lib.mc_register_host(addr, arr.nbytes))
    _registered[addr] = arr


def unregister_host(arr: np.ndarray) -> None:
    addr = arr.ctypes.data
    if _registered.pop(addr, None) is not None:
        lib = load()
        _check(lib, lib.mc_unregister_host(addr))


class DeviceRing:
    """One device-resident FIFO ring (fp16 scan copy + float64 master) on one GPU."""

    def __init__(self, capacity: int, dim: int, device: int = 0):
        self.lib = load()
        self.capacity = int(capacity)
        self.dim = int(dim)
        self.device = int(device)
        h = C.c_void_p()
        _check(self.lib, self.lib.mc_create(C.byref(h), self.capacity, self.dim, self.device))
        self._h = h
        self._hv = h.value  # plain int handle for the per-call fast paths
        self._append = self.lib.mc_append
        self._retrieve = self.lib.mc_retrieve_batch
        self._submit = self.lib.mc_retrieve_submit
        self._wait = self.lib.mc_retrieve_wait
        self._ticket = np.zeros(1, dtype=np.uint32)
        self._ticket_ptr = self._ticket.ctypes.data  # .ctypes costs ~1 us per access
        self._rowbuf = np.zeros(self.dim, dtype=np.float64)
        self._rowptr = self._rowbuf.ctypes.data
        self._bcap = 0
        self._ensure_out(1)
        self._table_key = None
        # The query / result buffers below are shared by every call on this ring, and ctypes
        # releases the GIL during the native call: one lock spans each buffer write -> native
        # call -> copy-out, so concurrent readers ("many readers or one writer", cache.py:144)
        # never see each other's queries or answers.
        self._lock = threading.Lock()
        self._merge_B = {}  # merge slot -> batch of the merge submitted into it

    # -- lifecycle -----------------------------------------------------------
    def close(self) -> None:
        h, self._h = getattr(self, "_h", None), None
        if h is not None and h.value:
            self.lib.mc_destroy(h)

    def __del__(self):  # pragma: no cover - interpreter teardown order varies
        try:
            self.close()
        except Exception:
            pass

    # -- configuration -------------------------------------------------------
    def set_table(self, pairs, total_steps: int) -> None:
        key = (tuple(pairs), int(total_steps))
        if key == self._table_key:
            return
        ks = np.array([k for k, _ in pairs], dtype=np.int32)
        taus = np.array([t for _, t in pairs], dtype=np.float64)
        _check(self.lib, self.lib.mc_set_thresholds(self._h, _ptr(ks), _ptr(taus), len(ks), int(total_steps)))
        self._table_key = key

    def set_sigma_schedule(self, schedule) -> None:
        """sigma over timesteps 0..T for the decision epilogue (None clears it)."""
        key = None if schedule is None else np.asarray(schedule, dtype=np.float64).tobytes()
        if key == getattr(self, "_sched_key", None):
            return
        s = np.zeros(0) if schedule is None else np.ascontiguousarray(schedule, dtype=np.float64)
        _check(self.lib, self.lib.mc_set_sigma_schedule(self._h, _ptr(s) if s.size else None, int(s.size)))
        self._sched_key = key

    def decisions(self, Q: np.ndarray) -> np.ndarray:
        """Q: float64 [B, dim] -> B serving decisions (DECISION_DTYPE), from the device epilogue."""
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        out = np.empty(Q.shape[0], dtype=DECISION_DTYPE)
        if Q.shape[0]:
            _check(self.lib, self.lib.mc_retrieve_decisions(self._h, _ptr(Q), Q.shape[0], _ptr(out)))
        return out

    def set_path(self, path: int) -> None:
        _check(self.lib, self.lib.mc_set_path(self._h, int(path)))

    def configure_shard(self, n_shards: int, shard_id: int) -> None:
        _check(self.lib, self.lib.mc_configure_shard(self._h, int(n_shards), int(shard_id)))

    # -- ring maintenance ----------------------------------------------------
    def append(self, rows: np.ndarray) -> None:
        rows = np.ascontiguousarray(rows, dtype=np.float64)
        n = rows.shape[0] if rows.ndim == 2 else 1
        _check(self.lib, self.lib.mc_append(self._h, _ptr(rows), n))

    def append1(self, row: np.ndarray) -> None:
        """One row (the per-insert path): copied into a fixed float64 buffer, whose pointer is
        computed once (cheaper than a per-call .ctypes on the caller's array)."""
        self._rowbuf[...] = row
        rc = self._append(self._hv, self._rowptr, 1)
        if rc:
            _check(self.lib, rc)

    def evict_front(self, n: int) -> None:
        if n:
            _check(self.lib, self.lib.mc_evict_front(self._h, int(n)))

    def __len__(self) -> int:
        return int(self.lib.mc_size(self._h))

    # -- lookups -------------------------------------------------------------
    def _ensure_out(self, B: int) -> None:
        if B <= self._bcap:
            return
        cap = max(B, 2 * self._bcap, 4)
        self._live = np.empty(cap, dtype=np.int64)
        self._sim = np.empty(cap, dtype=np.float64)
        self._k = np.empty(cap, dtype=np.int32)
        self._flags = np.empty(cap, dtype=np.uint32)
        self._qbuf = np.zeros((cap, self.dim), dtype=np.float64)
        self._out_ptrs = tuple(a.ctypes.data for a in (self._live, self._sim, self._k, self._flags))
        self._qptr = self._qbuf.ctypes.data
        self._bcap = cap

    def retrieve(self, Q: np.ndarray):
        """Q: float64 [B, dim] -> (live[B], sim[B], k[B], flags[B]) arrays."""
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        B = Q.shape[0]
        with self._lock:
            self._ensure_out(B)
            _check(self.lib, self.lib.mc_retrieve_batch(self._h, _ptr(Q), B, *self._out_ptrs))
            return self._live[:B].copy(), self._sim[:B].copy(), self._k[:B].copy(), self._flags[:B].copy()

    def retrieve1(self, q: np.ndarray):
        """One query (1-d, length dim) -> (live, sim, k, flags) as Python scalars."""
        with self._lock:
            self._qbuf[0] = q  # copies and converts; the buffer pointer never changes
            rc = self._retrieve(self._hv, self._qptr, 1, *self._out_ptrs)
            if rc:
                _check(self.lib, rc)
            return int(self._live[0]), float(self._sim[0]), int(self._k[0]), int(self._flags[0])

    def submit1(self, q: np.ndarray) -> int:
        """Enqueue one lookup (mc_retrieve_submit); returns its ticket."""
        with self._lock:
            self._qbuf[0] = q
            rc = self._submit(self._hv, self._qptr, 1, self._ticket_ptr)
            if rc:
                _check(self.lib, rc)
            return int(self._ticket[0])

    def submit(self, Q: np.ndarray) -> int:
        """Enqueue a batch of lookups (mc_retrieve_submit) and return its ticket at once; a
        registered query array must stay untouched until wait()."""
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        with self._lock:
            _check(self.lib, self._submit(self._hv, _ptr(Q), Q.shape[0], self._ticket_ptr))
            return int(self._ticket[0])

    def wait(self, ticket: int, B: int):
        """(live, sim, k, flags) arrays of the submitted batch (mc_retrieve_wait)."""
        live = np.empty(B, dtype=np.int64)
        sim = np.empty(B, dtype=np.float64)
        k = np.empty(B, dtype=np.int32)
        flags = np.empty(B, dtype=np.uint32)
        with self._lock:
            _check(self.lib, self._wait(self._hv, ticket, _ptr(live), _ptr(sim), _ptr(k), _ptr(flags)))
        return live, sim, k, flags

    def wait1(self, ticket: int):
        """The submitted lookup's (live, sim, k, flags) as Python scalars (mc_retrieve_wait)."""
        with self._lock:
            rc = self._wait(self._hv, ticket, *self._out_ptrs)
            if rc:
                _check(self.lib, rc)
            return int(self._live[0]), float(self._sim[0]), int(self._k[0]), int(self._flags[0])

    def records_device(self):
        """Device that holds this ring's records (for the collective's buffers)."""
        import torch

        return torch.device("cuda", self.device)

    @staticmethod
    def _addr(buf) -> int:
        return buf if isinstance(buf, int) else buf.data_ptr()

    def retrieve_local_async(self, Q: np.ndarray, dev_records, stream_ptr: int = 0) -> None:
        """This shard's certified best per query -> B mc_records in device memory (a torch
        uint8 tensor of B*32 bytes, or a raw pointer), ordered before `stream`."""
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        _check(self.lib, self.lib.mc_retrieve_local_async(self._h, _ptr(Q), Q.shape[0], self._addr(dev_records),
                                                          stream_ptr or None))

    def retrieve_local_submit(self, Q: np.ndarray, dev_records, stream_ptr: int = 0) -> None:
        """retrieve_local_async without the exhaustive rescan behind the scan: records whose
        certificate failed surface as MC_FLAG_NEED_RESCAN in the merge (mc_retrieve_local_submit)."""
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        _check(self.lib, self.lib.mc_retrieve_local_submit(self._h, _ptr(Q), Q.shape[0], self._addr(dev_records),
                                                           stream_ptr or None))

    def rescan_local(self, Q: np.ndarray, dev_records, stream_ptr: int = 0) -> None:
        """Exhaustive float64 rescan of the records that ask for it, in place (mc_rescan_local)."""
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        _check(self.lib, self.lib.mc_rescan_local(self._h, _ptr(Q), Q.shape[0], self._addr(dev_records),
                                                  stream_ptr or None))

    def retrieve_local_device(self, dev_queries, B: int, dev_records, stream_ptr: int = 0) -> None:
        """retrieve_local_async for B float64 query rows already on this ring's device (a torch
        tensor or raw pointer, row stride dim), written on `stream` (mc_retrieve_local_device)."""
        _check(self.lib, self.lib.mc_retrieve_local_device(self._h, self._addr(dev_queries), int(B),
                                                           self._addr(dev_records), stream_ptr or None))

    def merge_records(self, dev_records, G: int, B: int, p0: int, stream_ptr: int = 0):
        """Merge G x B gathered records (shard-major) into decisions; p0 = oldest live global position."""
        with self._lock:
            self._ensure_out(B)
            _check(self.lib, self.lib.mc_merge_records(
                self._h, self._addr(dev_records), int(G), int(B), int(p0), stream_ptr or None, *self._out_ptrs))
            return self._live[:B].copy(), self._sim[:B].copy(), self._k[:B].copy(), self._flags[:B].copy()

    MERGE_SLOTS = 2  # MC_MERGE_SLOTS

    def merge_submit(self, dev_records, G: int, B: int, p0: int, stream_ptr: int, slot: int) -> None:
        """Enqueue the merge of G x B records on `stream` into result slot `slot` and return at once
        (mc_merge_records_submit); merge_wait(slot) collects it."""
        _check(self.lib, self.lib.mc_merge_records_submit(self._h, self._addr(dev_records), int(G), int(B), int(p0),
                                                          stream_ptr or None, int(slot)))
        self._merge_B[slot] = int(B)

    def merge_wait(self, slot: int):
        """(live, sim, k, flags) arrays of the merge submitted into `slot` (mc_merge_records_wait)."""
        B = self._merge_B.get(slot, 0)
        live = np.empty(B, dtype=np.int64)
        sim = np.empty(B, dtype=np.float64)
        k = np.empty(B, dtype=np.int32)
        flags = np.empty(B, dtype=np.uint32)
        _check(self.lib, self.lib.mc_merge_records_wait(self._h, int(slot), _ptr(live), _ptr(sim), _ptr(k),
                                                        _ptr(flags)))
        self._merge_B[slot] = 0
        return live, sim, k, flags

    def profile_steps(self, Q: np.ndarray, rows: np.ndarray | None, iters: int, flush_bytes: int):
        """Device-timed steps (see mc_profile_steps). Q: [iters, B, dim]; rows: [iters, dim] or None."""
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        B = Q.shape[1]
        r = None if rows is None else np.ascontiguousarray(rows, dtype=np.float64)
        ms = np.zeros(4, dtype=np.float64)
        cnt = np.zeros(2, dtype=np.int64)
        _check(self.lib, self.lib.mc_profile_steps(self._h, _ptr(Q), None if r is None else _ptr(r), B, int(iters),
                                                   int(flush_bytes), _ptr(ms), _ptr(cnt)))
        return {"step_ms": ms[0], "scan_ms": ms[1], "merge_ms": ms[2], "append_ms": ms[3],
                "launches_per_step": int(cnt[0]), "would_fallback": int(cnt[1])}

    @staticmethod
    def profile_rotate(rings, Q: np.ndarray, rows: np.ndarray | None, iters: int):
        """Back-to-back device-timed steps rotating over `rings` (see mc_profile_rotate).
        Q: [iters, B, dim]; rows: [iters, dim] or None."""
        lib = load()
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        B = Q.shape[1]
        r = None if rows is None else np.ascontiguousarray(rows, dtype=np.float64)
        hs = (C.c_void_p * len(rings))(*[ring._hv for ring in rings])
        ms = np.zeros(1, dtype=np.float64)
        cnt = np.zeros(2, dtype=np.int64)
        _check(lib, lib.mc_profile_rotate(C.cast(hs, C.c_void_p), len(rings), _ptr(Q), None if r is None else _ptr(r),
                                          B, int(iters), _ptr(ms), _ptr(cnt)))
        return {"step_ms": float(ms[0]), "launches_per_step": int(cnt[0]), "would_fallback": int(cnt[1])}

    def generate(self, n: int, centers: np.ndarray, spread: float, beta: float, seed: int, row0: int = 0) -> None:
        """Append n device-generated synthetic rows (mc_generate_rows; measurement infrastructure)."""
        c = np.ascontiguousarray(centers, dtype=np.float64)
        if c.ndim != 2 or c.shape[1] != self.dim:
            raise ValueError(f"centers must be [K, {self.dim}]")
        _check(self.lib, self.lib.mc_generate_rows(self._h, int(n), _ptr(c), c.shape[0], float(spread), float(beta),
                                                   int(seed) & (2**64 - 1), int(row0)))

    def read_rows(self, first: int, n: int) -> np.ndarray:
        """float64 master rows of live indices [first, first + n) (mc_read_rows)."""
        out = np.empty((int(n), self.dim), dtype=np.float64)
        _check(self.lib, self.lib.mc_read_rows(self._h, int(first), int(n), _ptr(out)))
        return out

    def debug_read_row(self, live: int) -> np.ndarray:
        """The device's float64 copy of live row `live` (debugging)."""
        out = np.empty(3 * self.dim, dtype=np.float64)
        _check(self.lib, self.lib.mc_debug_read_row(self._h, int(live), _ptr(out)))
        return out[: self.dim] if not os.environ.get("MC_DEBUG_COPIES") else out.reshape(3, self.dim)

    def stats(self) -> dict:
        out = np.zeros(8, dtype=np.int64)
        _check(self.lib, self.lib.mc_stats(self._h, _ptr(out)))
        keys = ("lookups", "fallbacks", "nonfinite", "ties", "candidates", "gemv_launches", "gemm_launches",
                "kernel_launches")
        return dict(zip(keys, (int(x) for x in out)))
