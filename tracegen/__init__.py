"""tracegen — seeded synthetic trace generator (TEST INFRASTRUCTURE, shared input source).

Serves both the oracle (``oracle/``) and the CUDA path. Holds none of MegaScan's
analysis arithmetic: it simulates a TP x PP x DP Megatron 1F1B job (see gen.cpp header
and DESIGN.md "Input recipe") and returns the per-rank event columns the paper's tracer
records (§3.2), plus the DES ground truth.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libtracegen.so")
_SRC = os.path.join(_HERE, "gen.cpp")

THROTTLE, LINK_JITTER, LINK_DEGRADE = 1, 2, 3


class _Fault(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int32), ("a", ctypes.c_int32), ("b", ctypes.c_int32),
                ("it0", ctypes.c_int32), ("it1", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("factor", ctypes.c_double), ("prob", ctypes.c_double)]


class _Config(ctypes.Structure):
    _fields_ = [("tp", ctypes.c_int32), ("pp", ctypes.c_int32), ("dp", ctypes.c_int32),
                ("layers_per_stage", ctypes.c_int32), ("microbatches", ctypes.c_int32),
                ("iterations", ctypes.c_int32), ("seed", ctypes.c_uint64), ("hidden", ctypes.c_int64),
                ("jitter", ctypes.c_double), ("clock_skew", ctypes.c_int32), ("n_faults", ctypes.c_int32),
                ("faults", ctypes.POINTER(_Fault)), ("n_threads", ctypes.c_int32), ("it_begin", ctypes.c_int32),
                ("it_end", ctypes.c_int32), ("pad", ctypes.c_int32)]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread", _SRC, "-o", _SO])
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        lib.gen_count.restype = ctypes.c_int64
        lib.gen_count.argtypes = [ctypes.POINTER(_Config), ctypes.c_void_p]
        lib.gen_comm_table.restype = ctypes.c_int64
        lib.gen_comm_table.argtypes = [ctypes.POINTER(_Config), ctypes.c_void_p, ctypes.c_void_p]
        lib.gen_fill.restype = ctypes.c_int
        lib.gen_fill.argtypes = [ctypes.POINTER(_Config)] + [ctypes.c_void_p] * 9
        _lib = lib
    return _lib


@dataclass
class Fault:
    type: int
    a: int
    b: int = -1
    it0: int = 0
    it1: int = 1 << 30
    factor: float = 1.0
    prob: float = 1.0


@dataclass
class GenConfig:
    tp: int
    pp: int
    dp: int
    layers_per_stage: int
    microbatches: int
    iterations: int
    seed: int = 1
    hidden: int = 12288
    jitter: float = 0.05
    clock_skew: bool = True
    faults: list = field(default_factory=list)
    threads: int = 0

    @property
    def world(self) -> int:
        return self.tp * self.pp * self.dp


@dataclass
class Trace:
    """A trace in the columnar layout the C-ABI consumes (events grouped by rank, program order)."""
    tp: int
    pp: int
    dp: int
    rank_offsets: np.ndarray  # u64 [W+1]
    comm_offsets: np.ndarray  # u64 [n_comms+1]
    comm_members: np.ndarray  # u32
    start_ns: np.ndarray      # i64
    dur_ns: np.ndarray        # u32
    kind_op: np.ndarray       # u16
    meta: np.ndarray          # u16
    comm: np.ndarray          # u32
    payload: np.ndarray       # u32
    gt_inst: np.ndarray | None = None
    gt_true_start: np.ndarray | None = None

    @property
    def world(self) -> int:
        return self.tp * self.pp * self.dp

    @property
    def n_events(self) -> int:
        return int(self.rank_offsets[-1])

    @property
    def n_comms(self) -> int:
        return len(self.comm_offsets) - 1


def _cfg_struct(cfg: GenConfig, iter_range=None):
    arr = (_Fault * max(1, len(cfg.faults)))()
    for i, f in enumerate(cfg.faults):
        arr[i] = _Fault(f.type, f.a, f.b, f.it0, f.it1, 0, f.factor, f.prob)
    b, e = iter_range if iter_range is not None else (0, 0)
    c = _Config(cfg.tp, cfg.pp, cfg.dp, cfg.layers_per_stage, cfg.microbatches, cfg.iterations,
                cfg.seed, cfg.hidden, cfg.jitter, 1 if cfg.clock_skew else 0, len(cfg.faults),
                ctypes.cast(arr, ctypes.POINTER(_Fault)), cfg.threads, b, e, 0)
    return c, arr


def count(cfg: GenConfig, iter_range=None) -> np.ndarray:
    """Per-rank event offsets [W+1] of the whole trace, or of iterations [b, e) when ``iter_range``."""
    lib = _load()
    c, keep = _cfg_struct(cfg, iter_range)
    ro = np.zeros(cfg.world + 1, dtype=np.uint64)
    n = lib.gen_count(ctypes.byref(c), ro.ctypes.data)
    if n < 0:
        raise ValueError("bad generator config")
    return ro


def _ptr(a):
    return None if a is None else a.ctypes.data


def generate(cfg: GenConfig, ground_truth: bool = False, out: dict | None = None, with_start: bool = True,
             iter_range: tuple[int, int] | None = None) -> Trace:
    """Run the DES. ``out`` may supply preallocated (e.g. pinned) column arrays.

    ``iter_range=(b, e)`` emits only iterations [b, e) of the same job: per rank, exactly the events
    the full trace holds for those iterations (iterations are simulated independently from
    (seed, iteration, ...)-keyed draws), without start times or ground truth.
    """
    lib = _load()
    if iter_range is not None and (with_start or ground_truth):
        raise ValueError("an iteration range carries durations only: pass with_start=False, ground_truth=False")
    c, keep = _cfg_struct(cfg, iter_range)
    ro = count(cfg, iter_range)
    n = int(ro[-1])
    nc = lib.gen_comm_table(ctypes.byref(c), None, None)
    coff = np.zeros(nc + 1, dtype=np.uint64)
    lib.gen_comm_table(ctypes.byref(c), coff.ctypes.data, None)
    mem = np.zeros(int(coff[-1]), dtype=np.uint32)
    lib.gen_comm_table(ctypes.byref(c), coff.ctypes.data, mem.ctypes.data if len(mem) else None)
    out = out or {}
    cols = {
        "start_ns": out.get("start_ns", np.empty(n, dtype=np.int64)) if with_start else None,
        "dur_ns": out.get("dur_ns", np.empty(n, dtype=np.uint32)),
        "kind_op": out.get("kind_op", np.empty(n, dtype=np.uint16)),
        "meta": out.get("meta", np.empty(n, dtype=np.uint16)),
        "comm": out.get("comm", np.empty(n, dtype=np.uint32)),
        "payload": out.get("payload", np.empty(n, dtype=np.uint32)),
    }
    gt_inst = np.empty(n, dtype=np.uint64) if ground_truth else None
    gt_ts = np.empty(n, dtype=np.int64) if ground_truth else None
    rc = lib.gen_fill(ctypes.byref(c), ro.ctypes.data, _ptr(cols["start_ns"]), _ptr(cols["dur_ns"]),
                      _ptr(cols["kind_op"]), _ptr(cols["meta"]), _ptr(cols["comm"]), _ptr(cols["payload"]),
                      _ptr(gt_inst), _ptr(gt_ts))
    if rc != 0:
        raise RuntimeError(f"generator failed rc={rc} (-1 = schedule deadlock)")
    return Trace(cfg.tp, cfg.pp, cfg.dp, ro, coff, mem, gt_inst=gt_inst, gt_true_start=gt_ts, **cols)


# --- hand-built traces ------------------------------------------------------------------

COMPUTE, ALLREDUCE, ALLGATHER, REDUCESCATTER, BROADCAST, SEND, RECV = range(7)


def kind_op(kind: int, op: int = 0, iter_end: bool = False) -> int:
    return (kind & 7) | (8 if iter_end else 0) | ((op & 0xFFF) << 4)


def meta(mb: int = 0, chunk: int = 0, bwd: int = 0, warmup: int = 0) -> int:
    return (mb & 1023) | ((chunk & 7) << 10) | ((bwd & 1) << 13) | ((warmup & 1) << 14)


def from_events(tp: int, pp: int, dp: int, comms: list[list[int]], per_rank: list[list[tuple]]) -> Trace:
    """Build a Trace from per-rank lists of (kind, op, dur, comm_or_peer, payload, meta, iter_end)."""
    W = tp * pp * dp
    assert len(per_rank) == W
    ro = np.zeros(W + 1, dtype=np.uint64)
    for r in range(W):
        ro[r + 1] = ro[r] + len(per_rank[r])
    n = int(ro[-1])
    cols = dict(start_ns=np.zeros(n, np.int64), dur_ns=np.zeros(n, np.uint32), kind_op=np.zeros(n, np.uint16),
                meta=np.zeros(n, np.uint16), comm=np.zeros(n, np.uint32), payload=np.zeros(n, np.uint32))
    i = 0
    for r in range(W):
        t = 0
        for ev in per_rank[r]:
            kind, op, dur, cm, pl, me, ie = (list(ev) + [0, 0, 0, 0, 0, 0, False])[:7]
            cols["start_ns"][i] = t
            cols["dur_ns"][i] = dur
            cols["kind_op"][i] = kind_op(kind, op, bool(ie))
            cols["meta"][i] = me
            cols["comm"][i] = cm
            cols["payload"][i] = pl
            t += dur
            i += 1
    coff = np.zeros(len(comms) + 1, dtype=np.uint64)
    for c, m in enumerate(comms):
        coff[c + 1] = coff[c] + len(m)
    mem = np.array([x for m in comms for x in sorted(m)], dtype=np.uint32)
    return Trace(tp, pp, dp, ro, coff, mem, **cols)
