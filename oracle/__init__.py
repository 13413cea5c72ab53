"""oracle — plain single-threaded CPU reference of MegaScan's analysis pass.

TEST INFRASTRUCTURE ONLY: may be imported by ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs, nothing else. It shares no code
with the CUDA path (``paper_2507_19845_b200``); see ``oracle.cpp`` for the procedure
(§3.2).

Parity status per function (DESIGN.md §Oracle pins):
  A1-A2 matching ...... pinned (SPEC examples, brute-force enumeration, DES ground truth)
  A3 decomposition .... pinned (closed form vs DES true clock, invariants)
  A4 stage 1 .......... pinned (SPEC examples, small-dp closed forms, injected throttle)
  A5 stage 2 .......... pinned (SPEC examples, injected throttle / collateral victims)
  A6 stage 3 .......... pinned (SPEC arithmetic example, injected degraded link)
  A7-A8 walk .......... parity unpinned by the paper (definition is ours, reading R17);
                        pinned by hand-built chains and cycles only.
  NEXT-4 blame ........ parity unpinned by the paper (definition is ours, readings EB1-EB6);
                        pinned by hand-built chains / a cycle, wait conservation, DES throttles.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", _SRC, "-o", _SO])
    return _SO


class _Input(ctypes.Structure):
    _fields_ = [("tp", ctypes.c_int32), ("pp", ctypes.c_int32), ("dp", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("n_events", ctypes.c_uint64), ("rank_offsets", ctypes.c_void_p), ("dur", ctypes.c_void_p),
                ("kind_op", ctypes.c_void_p), ("meta", ctypes.c_void_p), ("comm", ctypes.c_void_p),
                ("payload", ctypes.c_void_p), ("n_comms", ctypes.c_uint32), ("pad2", ctypes.c_uint32),
                ("comm_offsets", ctypes.c_void_p), ("comm_members", ctypes.c_void_p)]


class _Config(ctypes.Structure):
    _fields_ = [("slow_num", ctypes.c_uint32), ("slow_den", ctypes.c_uint32), ("slow_margin_ns", ctypes.c_uint64),
                ("cand_num", ctypes.c_uint32), ("cand_den", ctypes.c_uint32), ("min_samples", ctypes.c_uint32),
                ("late_num", ctypes.c_uint32), ("late_den", ctypes.c_uint32), ("late_margin_ns", ctypes.c_uint64),
                ("bw_num", ctypes.c_uint32), ("bw_den", ctypes.c_uint32), ("wait_margin_ns", ctypes.c_uint64),
                ("window_iters", ctypes.c_uint32), ("stage2_classes", ctypes.c_uint32),
                ("stage2_mode", ctypes.c_uint32), ("pad", ctypes.c_uint32)]


@dataclass
class Config:
    """Thresholds (SPEC S:L313 defaults as exact rationals; readings R8-R14)."""
    slow_num: int = 3
    slow_den: int = 2
    slow_margin_ns: int = 50_000
    cand_num: int = 3
    cand_den: int = 10
    min_samples: int = 10
    late_num: int = 7
    late_den: int = 10
    late_margin_ns: int = 100_000
    bw_num: int = 7
    bw_den: int = 10
    wait_margin_ns: int = 100_000
    window_iters: int = 0
    stage2_classes: int = 3
    stage2_mode: int = 0  # 0 CONDITIONAL, 1 UNCONDITIONAL (SPEC S:L342 literal)


_ARRAYS = {
    "scalars": np.uint64,
    "ev_inst": np.uint32, "ev_wait": np.uint32, "ev_ref": np.uint32, "ev_slow": np.uint8,
    "ch_kind": np.uint8, "ch_a": np.uint32, "ch_b": np.uint32, "ch_nmem": np.uint32, "ch_nmax": np.uint32,
    "ch_nmin": np.uint32, "ch_base": np.uint64,
    "in_channel": np.uint32, "in_k": np.uint32, "in_dmin": np.uint32, "in_dmax": np.uint32, "in_last": np.uint32,
    "in_npresent": np.uint32, "in_payload": np.uint32, "in_flags": np.uint8,
    "rk_sum_compute": np.uint64, "rk_sum_wait": np.uint64, "rk_sum_transfer": np.uint64,
    "cl_J": np.uint32, "cl_mismatch": np.uint8,
    "wd_total": np.uint32, "wd_slow": np.uint32, "wd_cand": np.uint8, "wd_frac": np.float64,
    "wl_joined": np.uint32, "wl_late": np.uint32, "wl_late_frac": np.float64, "wl_verdict": np.uint8,
    "wl_link_slow": np.uint8,
    "lk_window": np.uint32, "lk_src": np.uint32, "lk_dst": np.uint32, "lk_n": np.uint32,
    "lk_med_payload": np.uint32, "lk_med_transfer": np.uint32, "lk_used_warm": np.uint8, "lk_slow": np.uint8,
    "lk_dir": np.uint8, "lk_eligible": np.uint8, "lk_med_bw": np.float64,
    "lb_label": np.uint8, "lb_root_kind": np.uint8, "lb_root_rank": np.uint32, "lb_root_src": np.uint32,
    "lb_depth": np.uint32, "lb_total_wait": np.uint64,
    "eg_window": np.uint32, "eg_src": np.uint32, "eg_dst": np.uint32, "eg_weight": np.uint64,
}
_SCALARS = ["status", "bad_event", "n_instances", "n_incomplete", "n_kind_mismatch", "n_payload_mismatch",
            "n_windows", "n_iters", "n_channels", "n_links", "n_edges"]

_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        lib.orc_run.restype = ctypes.c_void_p
        lib.orc_run.argtypes = [ctypes.POINTER(_Input), ctypes.POINTER(_Config), ctypes.POINTER(ctypes.c_int32)]
        lib.orc_free.argtypes = [ctypes.c_void_p]
        lib.orc_run_align.restype = ctypes.c_void_p
        lib.orc_run_align.argtypes = [ctypes.POINTER(_Input), ctypes.POINTER(_Config), ctypes.c_void_p, ctypes.c_int32,
                                      ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
        lib.orc_run_blame.restype = ctypes.c_void_p
        lib.orc_run_blame.argtypes = [ctypes.POINTER(_Input), ctypes.POINTER(_Config), ctypes.POINTER(ctypes.c_int32)]
        lib.orc_array.restype = ctypes.c_int
        lib.orc_array.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p),
                                  ctypes.POINTER(ctypes.c_uint64)]
        _lib = lib
    return _lib


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


_AL_ARRAYS = {"al_start": np.int64, "al_level": np.int32, "al_nanchor": np.uint32, "al_residual": np.uint64}


def align(trace, reference: int = 0, cfg: Config | None = None) -> dict:
    """run() plus the NEXT-1 timeline alignment (oracle.cpp ``align``, SPEC
    S:L243-300; readings AL1-AL6). Needs ``trace.start_ns``. Adds al_start (i64 per event),
    al_level (i32 per rank, -1 = not reached), al_nanchor, al_residual and al_status."""
    cfg = cfg or Config()
    lib = _load()
    start = _c(trace.start_ns, np.int64)
    return run(trace, cfg, _align=(start, int(reference)))


_BL_ARRAYS = {"bl_root": np.uint64, "bl_inflicted": np.uint64, "bl_self": np.uint64, "bl_unattributed": np.uint64,
              "bl_suffered": np.uint64}


def blame(trace, cfg: Config | None = None) -> dict:
    """run() plus the NEXT-4 event-level blame (oracle.cpp ``blame``; DESIGN.md §10e EB1-EB6).
    Adds bl_root (u64 per event: root event of a waiting event; 2^64-1 not waiting, 2^64-2 on a
    cycle), per-rank bl_inflicted / bl_self / bl_unattributed / bl_suffered (ns) and the counts
    bl_n_waiting / bl_n_cyclic."""
    return run(trace, cfg, _blame=True)


def run(trace, cfg: Config | None = None, _align=None, _blame: bool = False) -> dict:
    """Analyse ``trace`` (a tracegen.Trace or any object with the same columns). Returns a dict of
    numpy arrays (keys of ``_ARRAYS``) plus the scalar counters."""
    cfg = cfg or Config()
    lib = _load()
    keep = [_c(trace.rank_offsets, np.uint64), _c(trace.dur_ns, np.uint32), _c(trace.kind_op, np.uint16),
            _c(trace.meta, np.uint16), _c(trace.comm, np.uint32), _c(trace.payload, np.uint32),
            _c(trace.comm_offsets, np.uint64), _c(trace.comm_members, np.uint32)]
    inp = _Input(trace.tp, trace.pp, trace.dp, 0, int(trace.rank_offsets[-1]), keep[0].ctypes.data,
                 keep[1].ctypes.data, keep[2].ctypes.data, keep[3].ctypes.data, keep[4].ctypes.data,
                 keep[5].ctypes.data, len(trace.comm_offsets) - 1, 0, keep[6].ctypes.data, keep[7].ctypes.data)
    c = _Config(cfg.slow_num, cfg.slow_den, cfg.slow_margin_ns, cfg.cand_num, cfg.cand_den, cfg.min_samples,
                cfg.late_num, cfg.late_den, cfg.late_margin_ns, cfg.bw_num, cfg.bw_den, cfg.wait_margin_ns,
                cfg.window_iters, cfg.stage2_classes, cfg.stage2_mode, 0)
    st = ctypes.c_int32(0)
    ast = ctypes.c_int32(0)
    if _blame:
        h = lib.orc_run_blame(ctypes.byref(inp), ctypes.byref(c), ctypes.byref(st))
    elif _align is None:
        h = lib.orc_run(ctypes.byref(inp), ctypes.byref(c), ctypes.byref(st))
    else:
        keep.append(_align[0])
        h = lib.orc_run_align(ctypes.byref(inp), ctypes.byref(c), _align[0].ctypes.data, _align[1],
                              ctypes.byref(st), ctypes.byref(ast))
    try:
        out = {}
        for name, dt in _ARRAYS.items():
            p = ctypes.c_void_p()
            nb = ctypes.c_uint64()
            if lib.orc_array(h, name.encode(), ctypes.byref(p), ctypes.byref(nb)) != 0:
                raise KeyError(name)
            n = nb.value // np.dtype(dt).itemsize
            out[name] = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_uint8)), shape=(nb.value,)).view(dt)[:n].copy() if n else np.zeros(0, dt)
        if _align is not None:
            for name, dt in _AL_ARRAYS.items():
                p = ctypes.c_void_p()
                nb = ctypes.c_uint64()
                if lib.orc_array(h, name.encode(), ctypes.byref(p), ctypes.byref(nb)) != 0:
                    raise KeyError(name)
                n = nb.value // np.dtype(dt).itemsize
                out[name] = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_uint8)), shape=(nb.value,)).view(dt)[:n].copy() if n else np.zeros(0, dt)
            out["al_status"] = int(ast.value)
        if _blame and st.value >= 0:
            for name, dt in _BL_ARRAYS.items():
                p = ctypes.c_void_p()
                nb = ctypes.c_uint64()
                if lib.orc_array(h, name.encode(), ctypes.byref(p), ctypes.byref(nb)) != 0:
                    raise KeyError(name)
                n = nb.value // np.dtype(dt).itemsize
                out[name] = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_uint8)), shape=(nb.value,)).view(dt)[:n].copy() if n else np.zeros(0, dt)
        sc = out.pop("scalars")
        if _blame and st.value >= 0:
            out["bl_n_waiting"], out["bl_n_cyclic"] = int(sc[len(_SCALARS)]), int(sc[len(_SCALARS) + 1])
        for i, k in enumerate(_SCALARS):
            out[k] = int(np.int64(sc[i])) if k == "status" else int(sc[i])
        return out
    finally:
        lib.orc_free(h)
