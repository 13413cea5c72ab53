"""paper_2507_19845_b200 — B200-native MegaScan trace-analysis hot path (arXiv 2507.19845 §3.2).

Thin ctypes binding over the C ABI in ``include/megascan/scan.h`` (``libmegascan.so``, built
in-tree for sm_100a). Argument marshalling only: every analysis step runs in the CUDA kernels.
There is no CPU fallback — if the library or a CUDA device is missing, calls raise.

Same names as the C ABI: ``scan_create``, ``scan_load_events``, ``scan_match_collectives``,
``scan_detect``, ``scan_localize``, ``scan_export``; plus the ``Scan`` convenience class.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _build

_HERE = os.path.dirname(os.path.abspath(__file__))

SCAN_OK, SCAN_PARTIAL = 0, 1
SCAN_HOST_PTRS, SCAN_DEVICE_PTRS, SCAN_STRICT = 0, 1, 2
_STATUS = {0: "SCAN_OK", 1: "SCAN_PARTIAL", -1: "SCAN_E_INVALID_ARG", -2: "SCAN_E_SCHEMA", -3: "SCAN_E_INTEGRITY",
           -4: "SCAN_E_ORDER", -5: "SCAN_E_CUDA", -6: "SCAN_E_NCCL", -7: "SCAN_E_OOM", -8: "SCAN_E_UNSUPPORTED"}

# export names, in scan_output enum order, with dtypes
OUTPUTS = [
    ("ev_inst", np.uint32), ("ev_wait", np.uint32), ("ev_slow", np.uint8), ("ev_ref", np.uint32),
    ("ch_kind", np.uint8), ("ch_a", np.uint32), ("ch_b", np.uint32), ("ch_nmem", np.uint32), ("ch_nmax", np.uint32),
    ("ch_nmin", np.uint32), ("ch_base", np.uint64),
    ("in_channel", np.uint32), ("in_k", np.uint32), ("in_flags", np.uint8), ("in_dmin", np.uint32),
    ("in_dmax", np.uint32), ("in_last", np.uint32), ("in_npresent", np.uint32), ("in_payload", np.uint32),
    ("rk_sum_compute", np.uint64), ("rk_sum_wait", np.uint64), ("rk_sum_transfer", np.uint64),
    ("cl_J", np.uint32), ("cl_mismatch", np.uint8),
    ("wd_total", np.uint32), ("wd_slow", np.uint32), ("wd_cand", np.uint8), ("wd_frac", np.float64),
    ("wl_joined", np.uint32), ("wl_late", np.uint32), ("wl_late_frac", np.float64), ("wl_verdict", np.uint8),
    ("wl_link_slow", np.uint8),
    ("lk_window", np.uint32), ("lk_src", np.uint32), ("lk_dst", np.uint32), ("lk_n", np.uint32),
    ("lk_med_payload", np.uint32), ("lk_med_transfer", np.uint32), ("lk_used_warm", np.uint8), ("lk_slow", np.uint8),
    ("lk_dir", np.uint8), ("lk_eligible", np.uint8), ("lk_med_bw", np.float64),
    ("lb_label", np.uint8), ("lb_root_kind", np.uint8), ("lb_root_rank", np.uint32), ("lb_root_src", np.uint32),
    ("lb_depth", np.uint32), ("lb_total_wait", np.uint64),
    ("eg_window", np.uint32), ("eg_src", np.uint32), ("eg_dst", np.uint32), ("eg_weight", np.uint64),
    ("comm_inst", np.uint32), ("comm_wait", np.uint32), ("slow_bits", np.uint32),
    ("ch_shard_k0", np.uint64), ("ch_shard_n", np.uint32),
    ("al_start", np.int64), ("al_level", np.int32), ("al_nanchor", np.uint32), ("al_residual", np.uint64),
    ("bl_root", np.uint64), ("bl_inflicted", np.uint64), ("bl_self", np.uint64), ("bl_unattributed", np.uint64),
    ("bl_suffered", np.uint64),
]
ALIGN_OUTPUTS = ("al_start", "al_level", "al_nanchor", "al_residual")
BLAME_OUTPUTS = ("bl_root", "bl_inflicted", "bl_self", "bl_unattributed", "bl_suffered")
NATIVE_ONLY = ("comm_inst", "comm_wait", "slow_bits", "ch_shard_k0", "ch_shard_n") + ALIGN_OUTPUTS + BLAME_OUTPUTS
OUT_INDEX = {n: i for i, (n, _) in enumerate(OUTPUTS)}
OUT_DTYPE = dict(OUTPUTS)


class ScanError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class _Topo(ctypes.Structure):
    _fields_ = [("tp", ctypes.c_int32), ("pp", ctypes.c_int32), ("dp", ctypes.c_int32), ("rank_order", ctypes.c_uint32)]


class _Comms(ctypes.Structure):
    _fields_ = [("n_comms", ctypes.c_uint32), ("offsets", ctypes.c_void_p), ("members", ctypes.c_void_p)]


class _JsonRes(ctypes.Structure):
    _fields_ = [("n_events", ctypes.c_uint64), ("n_skipped", ctypes.c_uint64), ("n_comms", ctypes.c_uint32),
                ("err_kind", ctypes.c_int32), ("err_field", ctypes.c_int32), ("reserved", ctypes.c_uint32),
                ("err_offset", ctypes.c_uint64)]


class JsonTraceError(RuntimeError):
    """scan_ingest_json rejected the input: ``kind`` 1 syntax / 2 schema, ``field`` (SCAN_JF_*),
    ``offset`` (byte offset into the concatenated documents)."""

    def __init__(self, status: int, msg: str, kind: int, field: int, offset: int):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status, self.kind, self.field, self.offset = status, kind, field, offset


class _BlameRes(ctypes.Structure):
    _fields_ = [("n_waiting", ctypes.c_uint64), ("n_cyclic", ctypes.c_uint64), ("total_wait_ns", ctypes.c_uint64),
                ("rounds", ctypes.c_uint32), ("top_rank", ctypes.c_uint32), ("n_active", ctypes.c_uint64)]


class _AlignCfg(ctypes.Structure):
    _fields_ = [("reference", ctypes.c_int32), ("reserved", ctypes.c_uint32)]


class _AlignRes(ctypes.Structure):
    _fields_ = [("n_anchors", ctypes.c_uint64), ("n_aligned_ranks", ctypes.c_uint32), ("n_unaligned_ranks", ctypes.c_uint32),
                ("max_level", ctypes.c_uint32), ("reserved", ctypes.c_uint32), ("max_residual_ns", ctypes.c_uint64)]


class _Cols(ctypes.Structure):
    _fields_ = [("n_events", ctypes.c_uint64), ("rank_offsets", ctypes.c_void_p), ("start_ns", ctypes.c_void_p),
                ("dur_ns", ctypes.c_void_p), ("kind_op", ctypes.c_void_p), ("meta", ctypes.c_void_p),
                ("comm", ctypes.c_void_p), ("payload_bytes", ctypes.c_void_p)]


class _MatchRes(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in ("n_events", "n_comm_events", "n_compute_events", "n_channels",
                                               "n_p2p_channels", "n_instances", "n_incomplete", "n_kind_mismatch",
                                               "n_payload_mismatch", "n_iters")]


class _DetectCfg(ctypes.Structure):
    _fields_ = [("slow_num", ctypes.c_uint32), ("slow_den", ctypes.c_uint32), ("slow_margin_ns", ctypes.c_uint64),
                ("cand_num", ctypes.c_uint32), ("cand_den", ctypes.c_uint32), ("min_samples", ctypes.c_uint32),
                ("window_iters", ctypes.c_uint32), ("want_ref", ctypes.c_uint32), ("pad", ctypes.c_uint32)]


class _DetectRes(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in ("n_windows", "n_compared", "n_slow", "n_candidates", "n_class_mismatch")]


class _LocCfg(ctypes.Structure):
    _fields_ = [("late_margin_ns", ctypes.c_uint64), ("late_num", ctypes.c_uint32), ("late_den", ctypes.c_uint32),
                ("bw_num", ctypes.c_uint32), ("bw_den", ctypes.c_uint32), ("min_samples", ctypes.c_uint32),
                ("stage2_classes", ctypes.c_uint32), ("stage2_mode", ctypes.c_uint32), ("pad", ctypes.c_uint32),
                ("wait_margin_ns", ctypes.c_uint64)]


class _LocRes(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in ("n_windows", "n_links", "n_link_slow", "n_compute_slow",
                                               "n_link_slow_ranks", "n_both", "n_exonerated", "n_insufficient",
                                               "n_roots", "n_victims", "n_unattributed", "n_edges")]


_lib = None


def library_path() -> str:
    """The in-tree libmegascan.so (MEGASCAN_LIB may name another in-tree build, for A/B runs)."""
    return os.environ.get("MEGASCAN_LIB") or _build.SO


def _load_lib():
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if path == _build.SO and (not os.path.exists(_build.SO) or _build.stale()):
        _build.build()
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    lib.scan_create.argtypes = [ctypes.POINTER(P), ctypes.c_int, P]
    lib.scan_destroy.argtypes = [P]
    lib.scan_last_error.argtypes = [P]
    lib.scan_last_error.restype = ctypes.c_char_p
    lib.scan_load_events.argtypes = [P, ctypes.POINTER(_Topo), ctypes.POINTER(_Comms), ctypes.POINTER(_Cols), ctypes.c_uint32]
    lib.scan_match_collectives.argtypes = [P, ctypes.POINTER(_MatchRes)]
    lib.scan_detect.argtypes = [P, ctypes.POINTER(_DetectCfg), ctypes.POINTER(_DetectRes)]
    lib.scan_localize.argtypes = [P, ctypes.POINTER(_LocCfg), ctypes.POINTER(_LocRes)]
    lib.scan_output_size.argtypes = [P, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)]
    lib.scan_export.argtypes = [P, ctypes.c_int, P, ctypes.c_uint64, ctypes.c_int]
    lib.scan_output_device_ptr.argtypes = [P, ctypes.c_int]
    lib.scan_output_device_ptr.restype = P
    lib.scan_kernel_launches.argtypes = [P]
    lib.scan_kernel_launches.restype = ctypes.c_uint64
    lib.scan_set_timing.argtypes = [P, ctypes.c_int]
    lib.scan_set_timing.restype = ctypes.c_int32
    lib.scan_timing_reset.argtypes = [P]
    lib.scan_kernel_timing.argtypes = [P, ctypes.c_int, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(ctypes.c_uint64)]
    lib.scan_kernel_timing.restype = ctypes.c_int
    lib.scan_analyze.argtypes = [P, ctypes.POINTER(_DetectCfg), ctypes.POINTER(_LocCfg), ctypes.POINTER(_MatchRes),
                                 ctypes.POINTER(_DetectRes), ctypes.POINTER(_LocRes)]
    lib.scan_used_fused.argtypes = [P]
    lib.scan_used_fused.restype = ctypes.c_int
    lib.scan_force_general.argtypes = [P, ctypes.c_int]
    lib.scan_fused_variant.argtypes = [P, ctypes.c_int]
    lib.scan_nccl_unique_id.argtypes = [P]
    lib.scan_align.argtypes = [P, ctypes.POINTER(_AlignCfg), ctypes.POINTER(_AlignRes)]
    lib.scan_stream_open.argtypes = [P, ctypes.POINTER(_Topo), ctypes.POINTER(_Comms), ctypes.c_uint32,
                                     ctypes.POINTER(_DetectCfg), ctypes.POINTER(_LocCfg)]
    lib.scan_stream_push.argtypes = [P, ctypes.POINTER(_Cols), ctypes.c_uint32, ctypes.POINTER(_LocRes)]
    lib.scan_stream_window.argtypes = [P]
    lib.scan_stream_window.restype = ctypes.c_uint64
    lib.scan_create_sharded.argtypes = [ctypes.POINTER(P), ctypes.c_int, P, ctypes.c_int, ctypes.c_int, P]
    lib.scan_local_group_create.argtypes = [ctypes.POINTER(P), ctypes.c_int]
    lib.scan_local_group_destroy.argtypes = [P]
    lib.scan_create_sharded_local.argtypes = [ctypes.POINTER(P), ctypes.c_int, P, P, ctypes.c_int]
    lib.scan_blame.argtypes = [P, ctypes.POINTER(_BlameRes)]
    lib.scan_ingest_json.argtypes = [P, ctypes.POINTER(_Topo), P, ctypes.c_uint64, P, ctypes.c_uint32, ctypes.c_uint32,
                                     ctypes.POINTER(_JsonRes)]
    lib.scan_loaded_column.argtypes = [P, ctypes.c_int, P, ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)]
    lib.scan_emit_chrome.argtypes = [P, ctypes.c_uint32, P, ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)]
    for f in ("scan_create", "scan_load_events", "scan_match_collectives", "scan_detect", "scan_localize",
              "scan_output_size", "scan_export", "scan_analyze", "scan_force_general", "scan_fused_variant",
              "scan_nccl_unique_id", "scan_create_sharded", "scan_align", "scan_stream_open", "scan_stream_push",
              "scan_ingest_json", "scan_loaded_column", "scan_emit_chrome", "scan_blame", "scan_local_group_create",
              "scan_create_sharded_local"):
        getattr(lib, f).restype = ctypes.c_int32
    _lib = lib
    return lib


EXPORTED_SYMBOLS = ["scan_create", "scan_destroy", "scan_last_error", "scan_load_events", "scan_match_collectives",
                    "scan_detect", "scan_localize", "scan_output_size", "scan_export", "scan_output_device_ptr",
                    "scan_kernel_launches", "scan_set_timing", "scan_timing_reset", "scan_kernel_timing",
                    "scan_analyze", "scan_used_fused", "scan_force_general", "scan_fused_variant",
                    "scan_nccl_unique_id", "scan_create_sharded", "scan_align", "scan_stream_open", "scan_stream_push",
                    "scan_stream_window", "scan_ingest_json", "scan_loaded_column", "scan_emit_chrome",
                    "scan_blame", "scan_local_group_create", "scan_local_group_destroy", "scan_create_sharded_local"]


@dataclass
class DetectConfig:
    """Stage-1 thresholds (SPEC S:L313 defaults as exact rationals)."""
    slow_num: int = 3
    slow_den: int = 2
    slow_margin_ns: int = 50_000
    cand_num: int = 3
    cand_den: int = 10
    min_samples: int = 10
    window_iters: int = 0
    want_ref: bool = False


@dataclass
class LocalizeConfig:
    """Stage-2/3 + walk thresholds."""
    late_margin_ns: int = 100_000
    late_num: int = 7
    late_den: int = 10
    bw_num: int = 7
    bw_den: int = 10
    min_samples: int = 10
    stage2_classes: int = 3
    stage2_mode: int = 0
    wait_margin_ns: int = 100_000


def _check(ctx, st):
    if st < 0:
        raise ScanError(st, _load_lib().scan_last_error(ctx).decode())
    return st


def _ptr(x):
    """Pointer of a numpy array or a torch tensor (host or device)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    return x.ctypes.data


# ---- C-ABI mirrors ------------------------------------------------------------------------
def scan_create(device: int = 0, stream: int | None = None):
    lib = _load_lib()
    h = ctypes.c_void_p()
    st = lib.scan_create(ctypes.byref(h), device, stream)
    if st < 0:
        raise ScanError(st, "scan_create failed (no CUDA device?)")
    return h


def scan_nccl_unique_id() -> bytes:
    lib = _load_lib()
    buf = (ctypes.c_uint8 * 128)()
    st = lib.scan_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p))
    if st < 0:
        raise ScanError(st, "ncclGetUniqueId failed")
    return bytes(buf)


def scan_create_sharded(device: int, stream, n_shards: int, shard: int, unique_id: bytes | None):
    lib = _load_lib()
    h = ctypes.c_void_p()
    idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(unique_id) if unique_id is not None else None
    st = lib.scan_create_sharded(ctypes.byref(h), device, stream, n_shards, shard,
                                 ctypes.cast(idbuf, ctypes.c_void_p) if idbuf is not None else None)
    if st < 0:
        msg = lib.scan_last_error(h).decode() if h else "scan_create_sharded failed"
        if h:
            lib.scan_destroy(h)
        raise ScanError(st, msg)
    return h


# ABI width of every event column (scan.h scan_event_columns): the library copies / reads exactly
# n_events * itemsize bytes per column, so a column of another width would be misread.
COLUMN_DTYPES = {"dur_ns": np.uint32, "kind_op": np.uint16, "meta": np.uint16, "comm": np.uint32, "payload": np.uint32,
                 "start_ns": np.int64}


def _column(name: str, x, n: int, device: bool):
    """Marshal one event column to the ABI width. Host arrays are converted (value-checked: a value that
    does not fit the ABI width raises); device tensors must already have the width (any signedness of
    that size), be contiguous and hold n elements, else ValueError (no silent copy on the device path)."""
    if x is None:
        return None
    want = np.dtype(COLUMN_DTYPES[name])
    if device:
        if not hasattr(x, "data_ptr"):
            raise ValueError(f"{name}: device_ptrs=True needs a CUDA tensor")
        if x.element_size() != want.itemsize or not x.is_contiguous() or x.numel() != n:
            raise ValueError(f"{name}: need a contiguous {want.itemsize}-byte-element tensor of {n} elements, got "
                             f"{x.dtype} shape {tuple(x.shape)} contiguous={x.is_contiguous()}")
        return x
    a = np.asarray(x)
    if a.shape != (n,):
        raise ValueError(f"{name}: need shape ({n},), got {a.shape}")
    if a.dtype != want:
        if a.size and (a.dtype.kind not in "iub" or int(a.min()) < np.iinfo(want).min or int(a.max()) > np.iinfo(want).max):
            raise ValueError(f"{name}: values of dtype {a.dtype} do not fit the ABI type {want}")
        a = a.astype(want)
    return np.ascontiguousarray(a)


class LocalGroup:
    """In-process shard group (scan.h scan_local_group_create): G sharded contexts of this process,
    one host thread per shard, exchanging through the library's in-process back-end (no NCCL). For
    testing the sharded path on one GPU; the group must outlive its Scan objects."""

    def __init__(self, n_shards: int):
        lib = _load_lib()
        h = ctypes.c_void_p()
        st = lib.scan_local_group_create(ctypes.byref(h), int(n_shards))
        if st < 0:
            raise ScanError(st, "scan_local_group_create failed")
        self.h, self.n = h, int(n_shards)

    def close(self):
        if self.h:
            _load_lib().scan_local_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def scan_create_sharded_local(device: int, stream, group: LocalGroup, shard: int):
    lib = _load_lib()
    h = ctypes.c_void_p()
    st = lib.scan_create_sharded_local(ctypes.byref(h), device, stream, group.h, int(shard))
    if st < 0:
        raise ScanError(st, "scan_create_sharded_local failed")
    return h


def scan_load_events(ctx, tp, pp, dp, rank_offsets, comm_offsets, comm_members, dur, kind_op, meta, comm, payload,
                     flags: int = SCAN_HOST_PTRS, keep: list | None = None, start_ns=None):
    lib = _load_lib()
    ro = np.ascontiguousarray(rank_offsets, dtype=np.uint64)
    n = int(ro[-1]) if len(ro) else 0
    dev = bool(flags & SCAN_DEVICE_PTRS)
    dur, kind_op, meta, comm, payload, start_ns = (
        _column(k, v, n, dev) for k, v in (("dur_ns", dur), ("kind_op", kind_op), ("meta", meta), ("comm", comm),
                                           ("payload", payload), ("start_ns", start_ns)))
    co = np.ascontiguousarray(comm_offsets, dtype=np.uint64)
    cm = np.ascontiguousarray(comm_members, dtype=np.uint32)
    if keep is not None:
        keep += [ro, co, cm]
    topo = _Topo(tp, pp, dp, 0)
    comms = _Comms(len(co) - 1, co.ctypes.data, cm.ctypes.data if len(cm) else None)
    if keep is not None:
        keep += [dur, kind_op, meta, comm, payload, start_ns]
    cols = _Cols(n, ro.ctypes.data, _ptr(start_ns), _ptr(dur), _ptr(kind_op), _ptr(meta), _ptr(comm), _ptr(payload))
    return _check(ctx, lib.scan_load_events(ctx, ctypes.byref(topo), ctypes.byref(comms), ctypes.byref(cols), flags))


def scan_align(ctx, reference: int = 0) -> dict:
    """NEXT-1 timeline alignment (scan.h): needs start_ns at load and a completed analysis."""
    r = _AlignRes()
    _check(ctx, _load_lib().scan_align(ctx, ctypes.byref(_AlignCfg(int(reference), 0)), ctypes.byref(r)))
    return {n: getattr(r, n) for n, _ in r._fields_ if n != "reserved"}


LOADED_COLUMNS = (("start_ns", np.int64), ("dur_ns", np.uint32), ("kind_op", np.uint16), ("meta", np.uint16),
                  ("comm", np.uint32), ("payload", np.uint32), ("rank_offsets", np.uint64),
                  ("comm_offsets", np.uint64), ("comm_members", np.uint32))
SCAN_EMIT_ALIGNED = 1


def scan_ingest_json(ctx, tp, pp, dp, data, doc_offsets, flags: int = SCAN_HOST_PTRS) -> dict:
    """NEXT-2 (scan.h): parse JSON documents on the device and load them. ``data``: bytes / uint8
    numpy array (host) or a uint8 CUDA tensor with ``flags=SCAN_DEVICE_PTRS``."""
    lib = _load_lib()
    if isinstance(data, (bytes, bytearray, memoryview)):
        data = np.frombuffer(bytes(data), dtype=np.uint8)
    n = int(data.numel() if hasattr(data, "numel") else data.size)
    off = np.ascontiguousarray(doc_offsets, dtype=np.uint64)
    r = _JsonRes()
    st = lib.scan_ingest_json(ctx, ctypes.byref(_Topo(tp, pp, dp, 0)), _ptr(data) if n else None, n, off.ctypes.data,
                              len(off) - 1, flags, ctypes.byref(r))
    if st < 0:
        raise JsonTraceError(st, lib.scan_last_error(ctx).decode(), r.err_kind, r.err_field, r.err_offset)
    return {n_: getattr(r, n_) for n_, _ in r._fields_ if n_ != "reserved"}


def scan_loaded_column(ctx, name: str) -> np.ndarray:
    lib = _load_lib()
    idx = [n for n, _ in LOADED_COLUMNS].index(name)
    nb = ctypes.c_uint64()
    _check(ctx, lib.scan_loaded_column(ctx, idx, None, 0, 0, ctypes.byref(nb)))
    dt = dict(LOADED_COLUMNS)[name]
    out = np.empty(nb.value // np.dtype(dt).itemsize, dtype=dt)
    _check(ctx, lib.scan_loaded_column(ctx, idx, out.ctypes.data if out.size else None, nb.value, 0, ctypes.byref(nb)))
    return out


def scan_emit_chrome(ctx, aligned: bool = False, dst=None, as_bytes: bool = True):
    """Merged, annotated Chrome Tracing document (scan.h). Returns bytes; with ``as_bytes=False`` a
    uint8 numpy array in pinned host memory (one D2H copy, no further copy); or the byte count when
    ``dst`` (a uint8 CUDA tensor / numpy array large enough) receives it."""
    lib = _load_lib()
    flags = SCAN_EMIT_ALIGNED if aligned else 0
    nb = ctypes.c_uint64()
    _check(ctx, lib.scan_emit_chrome(ctx, flags, None, 0, 0, ctypes.byref(nb)))
    if dst is not None:
        dev = hasattr(dst, "is_cuda") and dst.is_cuda
        _check(ctx, lib.scan_emit_chrome(ctx, flags, _ptr(dst), int(dst.numel() if hasattr(dst, "numel") else dst.size),
                                         1 if dev else 0, ctypes.byref(nb)))
        return nb.value
    out = None
    if not as_bytes:
        try:
            import torch
            out = torch.empty(max(nb.value, 1), dtype=torch.uint8, pin_memory=True).numpy()[:nb.value]
        except Exception:
            out = None
    if out is None:
        out = np.empty(nb.value, dtype=np.uint8)
    _check(ctx, lib.scan_emit_chrome(ctx, flags, out.ctypes.data if nb.value else None, nb.value, 0, ctypes.byref(nb)))
    return out.tobytes() if as_bytes else out


def scan_blame(ctx) -> dict:
    """NEXT-4 event-level blame (scan.h): needs a completed analysis."""
    r = _BlameRes()
    _check(ctx, _load_lib().scan_blame(ctx, ctypes.byref(r)))
    return {n: getattr(r, n) for n, _ in r._fields_}


def scan_match_collectives(ctx) -> tuple[int, dict]:
    r = _MatchRes()
    st = _check(ctx, _load_lib().scan_match_collectives(ctx, ctypes.byref(r)))
    return st, {n: getattr(r, n) for n, _ in r._fields_}


def scan_detect(ctx, cfg: DetectConfig | None = None) -> dict:
    cfg = cfg or DetectConfig()
    c = _DetectCfg(cfg.slow_num, cfg.slow_den, cfg.slow_margin_ns, cfg.cand_num, cfg.cand_den, cfg.min_samples,
                   cfg.window_iters, 1 if cfg.want_ref else 0, 0)
    r = _DetectRes()
    _check(ctx, _load_lib().scan_detect(ctx, ctypes.byref(c), ctypes.byref(r)))
    return {n: getattr(r, n) for n, _ in r._fields_}


def scan_localize(ctx, cfg: LocalizeConfig | None = None) -> dict:
    cfg = cfg or LocalizeConfig()
    c = _LocCfg(cfg.late_margin_ns, cfg.late_num, cfg.late_den, cfg.bw_num, cfg.bw_den, cfg.min_samples,
                cfg.stage2_classes, cfg.stage2_mode, 0, cfg.wait_margin_ns)
    r = _LocRes()
    _check(ctx, _load_lib().scan_localize(ctx, ctypes.byref(c), ctypes.byref(r)))
    return {n: getattr(r, n) for n, _ in r._fields_}


def _dcfg(cfg):
    cfg = cfg or DetectConfig()
    return _DetectCfg(cfg.slow_num, cfg.slow_den, cfg.slow_margin_ns, cfg.cand_num, cfg.cand_den, cfg.min_samples,
                      cfg.window_iters, 1 if cfg.want_ref else 0, 0)


def _lcfg(cfg):
    cfg = cfg or LocalizeConfig()
    return _LocCfg(cfg.late_margin_ns, cfg.late_num, cfg.late_den, cfg.bw_num, cfg.bw_den, cfg.min_samples,
                   cfg.stage2_classes, cfg.stage2_mode, 0, cfg.wait_margin_ns)


def scan_analyze(ctx, dcfg: DetectConfig | None = None, lcfg: LocalizeConfig | None = None) -> dict:
    """A1-A8 in one call (fused SPMD stage-tile pass when applicable, else the general path)."""
    m, d, l_ = _MatchRes(), _DetectRes(), _LocRes()
    st = _check(ctx, _load_lib().scan_analyze(ctx, ctypes.byref(_dcfg(dcfg)), ctypes.byref(_lcfg(lcfg)), ctypes.byref(m),
                                              ctypes.byref(d), ctypes.byref(l_)))
    return {"status": st, "match": {n: getattr(m, n) for n, _ in m._fields_},
            "detect": {n: getattr(d, n) for n, _ in d._fields_}, "localize": {n: getattr(l_, n) for n, _ in l_._fields_},
            "fused": bool(_load_lib().scan_used_fused(ctx))}


def scan_export(ctx, name: str) -> np.ndarray:
    lib = _load_lib()
    idx = OUT_INDEX[name]
    nb = ctypes.c_uint64()
    _check(ctx, lib.scan_output_size(ctx, idx, ctypes.byref(nb)))
    dt = np.dtype(OUT_DTYPE[name])
    out = np.empty(nb.value // dt.itemsize, dtype=dt)
    if nb.value:
        _check(ctx, lib.scan_export(ctx, idx, out.ctypes.data, nb.value, 0))
    return out


def scan_export_device(ctx, name: str, dst) -> int:
    """Export a result array into a caller-owned CUDA tensor (device to device, no host copy); returns
    the bytes written. ``dst`` must hold at least ``scan_output_size`` bytes."""
    lib = _load_lib()
    idx = OUT_INDEX[name]
    nb = ctypes.c_uint64()
    _check(ctx, lib.scan_output_size(ctx, idx, ctypes.byref(nb)))
    if nb.value > dst.numel() * dst.element_size():
        raise ValueError(f"{name}: destination holds {dst.numel() * dst.element_size()} bytes, need {nb.value}")
    if nb.value:
        _check(ctx, lib.scan_export(ctx, idx, dst.data_ptr(), nb.value, 1))
    return int(nb.value)


def scan_output_bytes(ctx, name: str) -> int:
    nb = ctypes.c_uint64()
    _check(ctx, _load_lib().scan_output_size(ctx, OUT_INDEX[name], ctypes.byref(nb)))
    return int(nb.value)


def scan_destroy(ctx):
    if ctx:
        _load_lib().scan_destroy(ctx)


# ---- convenience ----------------------------------------------------------------------------
class Scan:
    """One analysis context on one GPU. ``load`` accepts a trace with numpy host columns
    (copied H2D by the library) or torch CUDA tensors (``device_ptrs=True``, zero-copy)."""

    def __init__(self, device: int = 0, stream=None, shards: tuple | None = None):
        """``shards=(n_shards, shard, nccl_unique_id)``: one iteration-window shard of a multi-GPU
        analysis (scan.h "multi-GPU"); ``analyze`` is then a collective call over the shards."""
        if stream is None:
            try:
                import torch
                if torch.cuda.is_available():
                    stream = torch.cuda.current_stream(device).cuda_stream
            except Exception:
                stream = None
        if shards is not None and isinstance(shards[2], LocalGroup):
            self.ctx = scan_create_sharded_local(device, stream, shards[2], int(shards[1]))
        elif shards is not None and shards[0] > 1:
            self.ctx = scan_create_sharded(device, stream, int(shards[0]), int(shards[1]), shards[2])
        else:
            self.ctx = scan_create(device, stream)
        self._keep: list = []

    def close(self):
        if self.ctx:
            scan_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load(self, trace, device_ptrs: bool = False, strict: bool = False, cols: dict | None = None,
             start: bool = False):
        """``start=True`` also hands over ``start_ns`` (only the timeline alignment reads it)."""
        self._keep = [trace]
        names = ("dur_ns", "kind_op", "meta", "comm", "payload") + (("start_ns",) if start else ())
        c = cols or {k: getattr(trace, k) for k in names}
        self._keep.append(c)
        flags = (SCAN_DEVICE_PTRS if device_ptrs else SCAN_HOST_PTRS) | (SCAN_STRICT if strict else 0)
        return scan_load_events(self.ctx, trace.tp, trace.pp, trace.dp, trace.rank_offsets, trace.comm_offsets,
                                trace.comm_members, c["dur_ns"], c["kind_op"], c["meta"], c["comm"], c["payload"],
                                flags, keep=self._keep, start_ns=c.get("start_ns"))

    def match(self):
        return scan_match_collectives(self.ctx)

    def detect(self, cfg: DetectConfig | None = None):
        return scan_detect(self.ctx, cfg)

    def localize(self, cfg: LocalizeConfig | None = None):
        return scan_localize(self.ctx, cfg)

    def run(self, dcfg: DetectConfig | None = None, lcfg: LocalizeConfig | None = None) -> dict:
        st, m = self.match()
        d = self.detect(dcfg)
        l_ = self.localize(lcfg)
        return {"status": st, "match": m, "detect": d, "localize": l_}

    def analyze(self, dcfg: DetectConfig | None = None, lcfg: LocalizeConfig | None = None) -> dict:
        return scan_analyze(self.ctx, dcfg, lcfg)

    def align(self, reference: int = 0) -> dict:
        """Timeline alignment onto ``reference``'s clock (load with ``start=True`` first)."""
        return scan_align(self.ctx, reference)

    def blame(self) -> dict:
        """Event-level blame of every wait (after ``analyze``); outputs ``BLAME_OUTPUTS``."""
        return scan_blame(self.ctx)

    # ---- NEXT-2 Chrome-trace JSON ingest / emit (scan.h)
    def ingest_json(self, docs, tp: int, pp: int, dp: int, device: bool = False) -> dict:
        """Parse JSON documents (a list of per-rank files' bytes, or one bytes object) on the GPU
        and load the job; ``device=True`` stages the bytes in a CUDA tensor first (zero-copy ingest)."""
        docs = [docs] if isinstance(docs, (bytes, bytearray)) else list(docs)
        off = np.zeros(len(docs) + 1, dtype=np.uint64)
        for i, d in enumerate(docs):
            off[i + 1] = off[i] + len(d)
        data = np.frombuffer(b"".join(docs), dtype=np.uint8)
        if device:
            import torch
            data = torch.from_numpy(data.copy()).cuda()
        self._keep = [data]
        return scan_ingest_json(self.ctx, tp, pp, dp, data, off, SCAN_DEVICE_PTRS if device else SCAN_HOST_PTRS)

    def loaded(self, name: str) -> np.ndarray:
        """A loaded input column (``LOADED_COLUMNS``), e.g. after ``ingest_json``."""
        return scan_loaded_column(self.ctx, name)

    def emit_chrome(self, aligned: bool = False, dst=None, as_bytes: bool = True):
        return scan_emit_chrome(self.ctx, aligned, dst, as_bytes)

    # ---- NEXT-3 sliding-window streaming (scan.h)
    STREAM_OUTPUTS = tuple(n for n, _ in OUTPUTS if n.startswith(("rk_sum", "wd_", "wl_", "lk_", "lb_", "eg_")))

    def stream_open(self, trace, window_iters: int, dcfg: DetectConfig | None = None, lcfg: LocalizeConfig | None = None):
        """Open a sliding window of ``window_iters`` iterations on ``trace``'s topology / comm table."""
        lib = _load_lib()
        co = np.ascontiguousarray(trace.comm_offsets, dtype=np.uint64)
        cm = np.ascontiguousarray(trace.comm_members, dtype=np.uint32)
        self._stream_keep = [co, cm]
        dcfg, lcfg = dcfg or DetectConfig(), lcfg or LocalizeConfig()
        d = _DetectCfg(dcfg.slow_num, dcfg.slow_den, dcfg.slow_margin_ns, dcfg.cand_num, dcfg.cand_den, dcfg.min_samples,
                       0, 1 if dcfg.want_ref else 0, 0)
        l_ = _LocCfg(lcfg.late_margin_ns, lcfg.late_num, lcfg.late_den, lcfg.bw_num, lcfg.bw_den, lcfg.min_samples,
                     lcfg.stage2_classes, lcfg.stage2_mode, 0, lcfg.wait_margin_ns)
        _check(self.ctx, lib.scan_stream_open(self.ctx, ctypes.byref(_Topo(trace.tp, trace.pp, trace.dp, 0)),
                                              ctypes.byref(_Comms(len(co) - 1, co.ctypes.data, cm.ctypes.data if len(cm) else None)),
                                              int(window_iters), ctypes.byref(d), ctypes.byref(l_)))

    def stream_push(self, iteration, device_ptrs: bool = False, cols: dict | None = None) -> dict:
        """Push one whole iteration (a trace holding exactly one iteration of every rank)."""
        lib = _load_lib()
        ro = np.ascontiguousarray(iteration.rank_offsets, dtype=np.uint64)
        src = cols or {k: getattr(iteration, k) for k in ("dur_ns", "kind_op", "meta", "comm", "payload")}
        c = {k: _column(k, v, int(ro[-1]), device_ptrs) for k, v in src.items()}
        self._stream_cols = c  # alive until the call returns (the push copies them)
        cs = _Cols(int(ro[-1]), ro.ctypes.data, None, _ptr(c["dur_ns"]), _ptr(c["kind_op"]), _ptr(c["meta"]), _ptr(c["comm"]),
                   _ptr(c["payload"]))
        r = _LocRes()
        st = _check(self.ctx, lib.scan_stream_push(self.ctx, ctypes.byref(cs), SCAN_DEVICE_PTRS if device_ptrs else SCAN_HOST_PTRS,
                                                   ctypes.byref(r)))
        out = {n: getattr(r, n) for n, _ in r._fields_}
        out["status"] = st
        out["window"] = int(lib.scan_stream_window(self.ctx))
        return out

    def fused_variant(self, variant: int):
        """-1 automatic, 0 generic tile kernel, 1 transposed warp-per-position kernel, 2 persistent TMA-fed
        stage kernel (next load; falls back to the automatic choice where not applicable)."""
        _check(self.ctx, _load_lib().scan_fused_variant(self.ctx, variant))

    def force_general(self, on: bool = True):
        _check(self.ctx, _load_lib().scan_force_general(self.ctx, 1 if on else 0))

    def export(self, name: str) -> np.ndarray:
        return scan_export(self.ctx, name)

    def export_all(self, names=None) -> dict:
        names = names or [n for n, _ in OUTPUTS if n not in NATIVE_ONLY]
        return {n: self.export(n) for n in names}

    def device_ptr(self, name: str) -> int:
        return _load_lib().scan_output_device_ptr(self.ctx, OUT_INDEX[name]) or 0

    def kernel_launches(self) -> int:
        return int(_load_lib().scan_kernel_launches(self.ctx))

    def set_timing(self, on: bool):
        lib = _load_lib()
        lib.scan_set_timing(self.ctx, 1 if on else 0)
        lib.scan_timing_reset(self.ctx)

    def kernel_timing(self) -> dict:
        """{kernel name: (total ms, launches)} accumulated since set_timing(True)."""
        lib = _load_lib()
        n = lib.scan_kernel_timing(self.ctx, -1, None, None, None)
        out = {}
        for i in range(n):
            nm, ms_, cnt = ctypes.c_char_p(), ctypes.c_double(), ctypes.c_uint64()
            lib.scan_kernel_timing(self.ctx, i, ctypes.byref(nm), ctypes.byref(ms_), ctypes.byref(cnt))
            out[nm.value.decode()] = (ms_.value, cnt.value)
        return out


# ---- multi-GPU plumbing (host side) -------------------------------------------------------------
def shard_iterations(n_iters: int, n_shards: int, shard: int) -> tuple[int, int]:
    """Iteration block [b, e) of ``shard``: contiguous, ordered, sizes differ by at most one."""
    q, r = divmod(n_iters, n_shards)
    b = shard * q + min(shard, r)
    return b, b + q + (1 if shard < r else 0)


def slice_iterations(trace, b: int, e: int):
    """The events of iterations [b, e) of every rank of a host trace (iteration = events up to and
    including an iter_end-flagged event), as a trace with the same topology and comm table."""
    from dataclasses import replace
    W = trace.world
    ro = np.asarray(trace.rank_offsets, dtype=np.uint64)
    ends = (np.asarray(trace.kind_op) & 8) != 0
    lo = np.zeros(W, np.uint64)
    hi = np.zeros(W, np.uint64)
    for r in range(W):
        a0, a1 = int(ro[r]), int(ro[r + 1])
        cut = np.flatnonzero(ends[a0:a1]) + 1  # event index after each iteration end
        starts = np.concatenate([[0], cut])
        lo[r] = a0 + (starts[b] if b < len(starts) else a1 - a0)
        hi[r] = a0 + (starts[e] if e < len(starts) else a1 - a0)
    idx = np.concatenate([np.arange(int(lo[r]), int(hi[r]), dtype=np.int64) for r in range(W)]) if W else np.zeros(0, np.int64)
    nro = np.zeros(W + 1, np.uint64)
    nro[1:] = np.cumsum(hi - lo)
    cols = {k: np.ascontiguousarray(getattr(trace, k)[idx]) for k in ("dur_ns", "kind_op", "meta", "comm", "payload")}
    st = getattr(trace, "start_ns", None)
    return replace(trace, rank_offsets=nro, start_ns=(np.ascontiguousarray(st[idx]) if st is not None else None),
                   gt_inst=None, gt_true_start=None, **cols)


def shard_unique_id(group=None) -> bytes:
    """NCCL unique id made on rank 0 of a torch.distributed group and broadcast to its ranks."""
    import torch.distributed as dist
    obj = [scan_nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return obj[0]
