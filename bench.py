#!/usr/bin/env python
"""bench.py — trace events analysed per second on B200 (BASELINE.json metric), with the HBM
roofline fraction and the CPU oracle beside it.

One step = one pass of the whole hot path (scan_match_collectives + scan_detect + scan_localize,
SURVEY.md §8(a) rows A1-A8) over one synthetic trace resident in HBM.
Default workload (N=1): configs[2] "C3" — 1024 ranks TP8xPP8xDP16, 1000 iterations,
960,768,000 events, mixed throttling + link jitter (the north-star target workload).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--iters I] [--impl reference]

N>1 (torchrun): the SAME job is split into N iteration-window shards (strong scaling): rank g
generates iterations shard_iterations(I, N, g) of every rank and analyses them through one sharded
context (scan_create_sharded; NCCL all-gather / all-to-all / all-reduce inside scan_analyze), so
every rank ends with the job-wide verdicts. value = all events / max-over-ranks step time.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "trace events analysed/sec (1/2/4/8 B200) and % of HBM roofline vs CPU oracle"
WORKLOADS = {
    "c1": "C1 8-rank TP2xPP2xDP2, L_s=12, M=8, 10 it, rank 5 throttled x2.0",
    "c2": "C2 64-rank TP8xPP4xDP2, L_s=8, M=16, 200 it, jitter on the 16 fwd links leaving stage 1",
    "c3": "C3 1024-rank TP8xPP8xDP16, L_s=8, M=8, 1000 it, rank 299 x1.6 [200,600), rank 862 x2.5 [500,900), "
          "jitter on the 128 fwd links leaving stage 4",
    "c4": "C4 3072-rank TP8xPP64xDP6, L_s=2, M=16, 500 it, one rank x1.5 + one link x0.5",
    "c5": "C5 512-rank TP8xPP8xDP8, L_s=8, M=8, 100 it, cascading victims (whole trace)",
}


def alg_bytes_per_event(comm_frac: float) -> float:
    """read dur 4 + kind_op 2 + meta 2 + comm 4 + payload 4 = 16 B/event; write
    inst_id 4 + wait 4 per comm event and a 1 B slow flag per compute event."""
    return 16.0 + 8.0 * comm_frac + 1.0 * (1.0 - comm_frac)


def needed_bytes_per_event(comm_frac: float, p2p_frac: float) -> float:
    """What the fused pass must move at least: dense reads of dur 4 + kind_op 2 +
    comm 4 = 10 B/event; payload 4 + meta 2 only at P2P events; writes inst_id 4 + wait 4 per comm
    event and one slow bit per compute event."""
    return 10.0 + 6.0 * p2p_frac + 8.0 * comm_frac + (1.0 - comm_frac) / 8.0


def peak_of() -> float:
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json), else the profiling guide's fallback."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return float(json.load(open(path)).get("hbm_gbs", 6650.0)) if os.path.exists(path) else 6650.0


def bpe_of(comm_frac: float) -> float:
    return alg_bytes_per_event(comm_frac)


def host_cpu() -> dict:
    """The host the oracle baseline ran on: logical CPUs, this process's affinity, CPU model."""
    model = None
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        model = None
    return {"nproc": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)), "cpu_model": model}


def event_fractions(kind_op: np.ndarray) -> tuple[float, float]:
    """Communication and P2P fractions over the WHOLE trace (chunked: no 1 GB temporaries)."""
    n = len(kind_op)
    comm = p2p = 0
    for a in range(0, n, 1 << 26):
        k = kind_op[a:a + (1 << 26)] & 7
        comm += int(np.count_nonzero(k))
        p2p += int(np.count_nonzero(k >= 5))
    return (comm / n, p2p / n) if n else (0.0, 0.0)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev = dev
        self.rows: list[list[str]] = []
        self.p = None
        self.i0, self.i1 = 0, None

    def wait_ready(self, timeout: float = 10.0):
        """nvidia-smi takes a while to start: wait for its first sample before the timed region."""
        t0 = time.time()
        while self.p and not self.rows and time.time() - t0 < timeout:
            time.sleep(0.02)

    def mark_start(self):
        self.i0 = len(self.rows)

    def mark_end(self):
        self.i1 = len(self.rows)

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "20"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None
        return self

    def _read(self):
        for line in self.p.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.p.wait(timeout=2)
            except Exception:
                self.p.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        # the samples taken during the timed region (at least the first one after it began)
        i1 = len(self.rows) if self.i1 is None else max(self.i1, self.i0 + 1)
        for r in self.rows[self.i0:i1]:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
                for n, v in zip(names, r[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
            except Exception:
                pass
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_trace(name: str, iters: int | None, seed: int, pinned: bool, it_range=None, with_start: bool = False):
    import tracegen as tg
    from tracegen import configs
    cfg = configs.CONFIGS[name](seed=seed) if iters is None else configs.CONFIGS[name](seed=seed, iterations=iters)
    ro = tg.count(cfg, it_range)
    n = int(ro[-1])
    out = None
    if pinned:
        import torch
        out = {}
        for k, dt in (("dur_ns", torch.int32), ("kind_op", torch.int16), ("meta", torch.int16), ("comm", torch.int32),
                      ("payload", torch.int32)):
            t = torch.empty(n, dtype=dt, pin_memory=True)
            out[k] = t.numpy().view({torch.int32: np.uint32, torch.int16: np.uint16}[dt])
    return tg.generate(cfg, out=out, with_start=with_start, iter_range=it_range), cfg


def streaming_c5(ms, torch, local, stream) -> dict:
    """C5: a 100-iteration stream of the 512-rank TP8xPP8xDP8 job; after every new
    iteration the last 50 iterations are re-analysed from scratch (51 windows). Reports the window
    analysis latency (device-resident window, CUDA events around scan_analyze) and the steps to
    detection of the injected source (rank 208 x2.5 from iteration 30) as ComputeSlow."""
    from dataclasses import replace
    import tracegen as tg
    from tracegen import configs
    cfg = configs.c5(seed=1)
    K, src, onset = 50, 208, 30
    full = tg.generate(cfg, with_start=False)
    W, ro = full.world, full.rank_offsets.astype(np.int64)
    ends = (full.kind_op & 8) != 0
    first = [np.concatenate([[0], np.flatnonzero(ends[ro[r]:ro[r + 1]]) + 1]) for r in range(W)]
    dev = {k: torch.from_numpy(np.ascontiguousarray(getattr(full, k)).view(np.int16 if getattr(full, k).dtype == np.uint16
                                                                          else np.int32)).cuda(local)
           for k in ("dur_ns", "kind_op", "meta", "comm", "payload")}
    s = ms.Scan(local, stream.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lat, det, nev = [], None, 0
    for wi_, w0 in enumerate([0] + list(range(cfg.iterations - K + 1))):  # window 0 twice: the first (module
        # load, first allocations) is untimed
        lo = np.array([ro[r] + first[r][w0] for r in range(W)])
        hi = np.array([ro[r] + first[r][w0 + K] for r in range(W)])
        idx = torch.from_numpy(np.concatenate([np.arange(a, b) for a, b in zip(lo, hi)])).cuda(local)
        cols = {k: v.index_select(0, idx) for k, v in dev.items()}  # window layout (untimed gather)
        wro = np.zeros(W + 1, np.uint64)
        wro[1:] = np.cumsum(hi - lo)
        s.load(replace(full, rank_offsets=wro), device_ptrs=True, cols=cols)
        torch.cuda.synchronize()
        e0.record(stream)
        s.analyze()
        e1.record(stream)
        torch.cuda.synchronize()
        if wi_ == 0:
            continue
        lat.append(e0.elapsed_time(e1))
        nev = int(wro[-1])
        v = int(s.export("wl_verdict")[src])
        if det is None and v in (1, 3):  # SCAN_V_COMPUTE_SLOW, SCAN_V_BOTH
            det = w0 + K - 1
    s.close()
    lat = np.array(lat)
    # NEXT-3: the same stream pushed one iteration at a time into a sliding-window context
    import time as _t
    si = ms.Scan(local, stream.cuda_stream)
    si.stream_open(full, K)
    plat, pdet = [], None
    for it in range(cfg.iterations):
        lo = np.array([ro[r] + first[r][it] for r in range(W)])
        hi = np.array([ro[r] + first[r][it + 1] for r in range(W)])
        idx = torch.from_numpy(np.concatenate([np.arange(a, b) for a, b in zip(lo, hi)])).cuda(local)
        cols = {k: v.index_select(0, idx) for k, v in dev.items()}
        iro = np.zeros(W + 1, np.uint64)
        iro[1:] = np.cumsum(hi - lo)
        torch.cuda.synchronize()
        t0 = _t.perf_counter()
        si.stream_push(replace(full, rank_offsets=iro), device_ptrs=True, cols=cols)
        plat.append((_t.perf_counter() - t0) * 1e3)
        if it >= K - 1:
            v = int(si.export("wl_verdict")[src])
            if pdet is None and v in (1, 3):
                pdet = it
    si.close()
    plat = np.array(plat[K - 1:])  # full windows
    incremental = {"latency_ms_median": float(np.median(plat)), "latency_ms_p99": float(np.percentile(plat, 99)),
                   "detected_at_iteration": pdet, "steps_to_detection": (pdet - onset + 1) if pdet is not None else None,
                   "timing": "wall clock per scan_stream_push (synchronous call; device-resident iteration columns)"}
    return {"incremental": incremental,
            "workload": "C5 512-rank TP8xPP8xDP8, L_s=8, M=8, 100-it stream, 50-it window re-analysed per iteration "
                        "(51 windows); rank 208 x2.5 from it 30, its 7 TP peers x1.8 on 40% of ops",
            "window_events": nev, "windows": len(lat), "latency_ms_median": float(np.median(lat)),
            "latency_ms_p99": float(np.percentile(lat, 99)), "value": nev / (float(np.median(lat)) / 1e3),
            "unit": "events/s (window analysis)", "detected_at_iteration": det,
            "steps_to_detection": (det - onset + 1) if det is not None else None,
            "note": "every window analysed from scratch (scan_analyze); incremental streaming is SURVEY NEXT-3"}


def json_io(ms, torch, local, stream, steps: int, warmup: int, cpu: bool) -> dict:
    """NEXT-2 (scan_ingest_json / scan_emit_chrome): the per-rank Chrome-trace JSON files of the C2
    job (TP8xPP4xDP2, 64 ranks, 40 iterations) parsed on the GPU into the event columns (device-
    resident bytes, CUDA events around the call), then the merged, annotated document emitted."""
    import ctypes
    import tracegen as tg
    from tracegen import chrome, configs
    cfg = configs.c2(seed=1, iterations=40)
    tr = tg.generate(cfg)
    data, off = chrome.rank_documents_fast(tr)
    nbytes = len(data)
    host = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
    dbuf = host.cuda(local)
    lib = ms._load_lib()
    s = ms.Scan(local, stream.cuda_stream)
    topo = (cfg.tp, cfg.pp, cfg.dp)
    for _ in range(max(1, warmup)):
        res = ms.scan_ingest_json(s.ctx, *topo, dbuf, off, ms.SCAN_DEVICE_PTRS)
    torch.cuda.synchronize()
    s.set_timing(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        res = ms.scan_ingest_json(s.ctx, *topo, dbuf, off, ms.SCAN_DEVICE_PTRS)
    e1.record(stream)
    torch.cuda.synchronize()
    ims = e0.elapsed_time(e1) / steps
    ik = s.kernel_timing()
    s.set_timing(False)
    # e2e: pinned host bytes -> H2D inside the call -> parse -> load
    t0 = time.perf_counter()
    ms.scan_ingest_json(s.ctx, *topo, host.numpy(), off, ms.SCAN_HOST_PTRS)
    e2e_s = time.perf_counter() - t0
    # emit: analysis once (untimed), then the document build (size query) per step
    s.analyze()
    nb = ctypes.c_uint64()
    for _ in range(max(1, warmup)):
        ms._check(s.ctx, lib.scan_emit_chrome(s.ctx, 0, None, 0, 0, ctypes.byref(nb)))
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(steps):
        ms._check(s.ctx, lib.scan_emit_chrome(s.ctx, 0, None, 0, 0, ctypes.byref(nb)))
    e1.record(stream)
    torch.cuda.synchronize()
    ems = e0.elapsed_time(e1) / steps
    out = torch.empty(int(nb.value), dtype=torch.uint8, pin_memory=True).numpy()  # caller-owned, allocated once
    s.emit_chrome(dst=out)
    t0 = time.perf_counter()
    s.emit_chrome(dst=out)  # build on the device + one D2H into the pinned host buffer
    emit_e2e_s = time.perf_counter() - t0
    s.close()
    base = None
    if cpu:  # oracle (Python json) on the first two ranks' files
        from oracle import chrome_json as cj
        docs = [data[int(off[r]):int(off[r + 1])] for r in range(2)]
        t0 = time.perf_counter()
        t_, _ = cj.parse(docs, *topo)
        dt = time.perf_counter() - t0
        nb_s = sum(len(d) for d in docs)
        base = {"value": nb_s / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
                "sample": f"oracle.chrome_json.parse of ranks 0-1's files ({nb_s / 1e6:.1f} MB, {t_.n_events} events), "
                          "Python json module, one core"}
    kern = {k: {"ms_per_call": round(v[0] / steps, 4), "launches": v[1]} for k, v in sorted(ik.items(), key=lambda kv: -kv[1][0])}
    pk_j = float((json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}).get("hbm_gbs", 6650.0))
    jp = ik.get("k_j_parse")
    jp_ms = jp[0] / steps if jp else None
    # k_j_parse reads every event object's text once and writes its columns (dur, kind_op, meta, comm,
    # payload: 16 B, start_ns: 8 B)
    jp_bytes = nbytes + 24 * int(res["n_events"])
    roof = ({"bound": "hbm", "kernel": "k_j_parse", "bytes_per_call": jp_bytes, "achieved": jp_bytes / (jp_ms / 1e3) / 1e9,
             "peak": pk_j, "unit": "GB/s", "frac": jp_bytes / (jp_ms / 1e3) / 1e9 / pk_j,
             "call_frac": nbytes / (ims / 1e3) / 1e9 / pk_j,
             "note": "k_j_parse: one thread per event object walking its bytes (latency-bound); call_frac: the "
                     "whole call's JSON bytes over its time"} if jp_ms else None)
    return {"metric": "Chrome-trace JSON parsed into event columns per second (scan_ingest_json)",
            "roofline": roof,
            "value": nbytes / (ims / 1e3) / 1e9, "unit": "GB/s",
            "events_per_s": res["n_events"] / (ims / 1e3), "ms_per_call": ims, "json_bytes": nbytes,
            "events": int(res["n_events"]), "docs": int(len(off) - 1),
            "workload": "C2 TP8xPP4xDP2 (64 per-rank files), 40 iterations, clean tracer format",
            "kernels": kern,
            "e2e": {"value": nbytes / e2e_s / 1e9, "unit": "GB/s", "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": 0,
                    "path": "pinned host bytes -> scan_ingest_json(SCAN_HOST_PTRS), wall clock"},
            "emit": {"value": len(out) / (ems / 1e3) / 1e9, "unit": "GB/s (merged document built on the device)",
                     "ms_per_call": ems, "bytes": len(out),
                     "e2e_gb_s": len(out) / emit_e2e_s / 1e9,
                     "e2e_path": "scan_emit_chrome build + D2H into a caller-owned pinned buffer (s.emit_chrome(dst=...)), wall clock"},
            "cpu_baseline": base}


def cpu_oracle_rate(name: str, sample_iters: int, seed: int) -> dict:
    import oracle
    tr, _ = make_trace(name, sample_iters, seed, pinned=False)
    t0 = time.perf_counter()
    oracle.run(tr)
    dt = time.perf_counter() - t0
    return {"value": tr.n_events / dt, "unit": "events/s", "cores": 1, "kind": "oracle",
            "sample": f"{name} shape, iterations [0,{sample_iters}) = {tr.n_events} events, single-threaded C++ oracle, "
                      f"{dt:.2f} s", "seconds": dt, "host": host_cpu()}


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    sample_iters = args.ref_iters
    rates = []
    for i in range(args.warmup + args.steps):
        r = cpu_oracle_rate(args.config, sample_iters, args.seed)
        if i >= args.warmup:
            rates.append(r)
    v = float(np.median([r["value"] for r in rates]))
    secs = float(np.median([r["seconds"] for r in rates]))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "events/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config] + f" (sample: iterations [0,{sample_iters}))"},
            "cpu_baseline": {"value": v, "unit": "events/s", "cores": 1, "kind": "oracle", "sample": rates[0]["sample"],
                             "host": rates[0]["host"]},
            "e2e": {"value": v, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--iters", type=int, default=None, help="override the config's iteration count")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cpu-iters", type=int, default=64, help="oracle sample (iterations) for cpu_baseline (~16 s)")
    ap.add_argument("--ref-iters", type=int, default=16, help="oracle sample per step for --impl reference")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--breakdown", action="store_true", default=True)
    ap.add_argument("--no-align", action="store_true", help="skip the timeline-alignment measurement (N=1 only)")
    ap.add_argument("--no-stream", action="store_true", help="skip the C5 sliding-window measurement (N=1 only)")
    ap.add_argument("--no-json", action="store_true", help="skip the JSON ingest / emit measurement (N=1 only)")
    ap.add_argument("--no-blame", action="store_true", help="skip the event-level blame measurement (N=1 only)")
    ap.add_argument("--no-general", action="store_true", help="skip the general-path measurement (N=1 only)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import paper_2507_19845_b200 as ms
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    # ---- synthetic trace: host (pinned) -> device columns; N>1: this rank's iteration block ----
    from tracegen import configs as _cf
    iters = args.iters
    total_iters = iters if iters is not None else _cf.CONFIGS[args.config]().iterations
    blk = ms.shard_iterations(total_iters, world, rank) if world > 1 else None
    uid = ms.shard_unique_id() if world > 1 else None
    t_gen = time.perf_counter()
    do_align = world == 1 and not args.no_align
    tr, cfg = make_trace(args.config, iters, args.seed, pinned=True, it_range=blk, with_start=do_align)
    t_gen = time.perf_counter() - t_gen
    N = tr.n_events
    comm_frac, p2p_frac = event_fractions(tr.kind_op)
    host = {k: getattr(tr, k) for k in ("dur_ns", "kind_op", "meta", "comm", "payload")}
    dev = {k: torch.from_numpy(v.view(np.int16 if v.dtype == np.uint16 else np.int32)).cuda(local, non_blocking=True)
           for k, v in host.items()}
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(local)
    s = ms.Scan(local, stream.cuda_stream, shards=(world, rank, uid) if world > 1 else None)
    s.load(tr, device_ptrs=True, cols=dev)

    def step():
        s.analyze()

    clk = ClockSampler(local).__enter__()  # started before the warm-up, so it samples from the timed region's start
    clk.wait_ready()
    for _ in range(args.warmup):
        step()
    import gc
    gc.collect()
    gc.disable()  # no collector pauses inside the timed steps (a late rank stalls every other at the first exchange)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if True:
        clk.mark_start()
        # the step time: K steps with nothing but the analysis between the two events
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        launches = s.kernel_launches()
        # the kernel breakdown: another K steps with the library's per-kernel CUDA events (recorded on the
        # launch stream around every launch), so their cost never enters the step time above
        kernels, ms_total_ev = {}, None
        if args.breakdown:
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            s.set_timing(True)
            e2a, e2b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e2a.record(stream)
            for _ in range(args.steps):
                step()
            e2b.record(stream)
            torch.cuda.synchronize()
            kernels = s.kernel_timing()
            s.set_timing(False)
            ms_total_ev = e2a.elapsed_time(e2b)
            if os.environ.get("MS_BENCH_RANK_KERNELS"):  # diagnostics: every rank's fused-pass and exchange times
                print(f"[rank {rank}] " + " ".join(f"{k}={v[0] / max(v[1], 1):.3f}" for k, v in kernels.items()
                                                   if k in ("k_fused", "x3_alltoall", "k_cross_reduce", "k_link_median")),
                      file=sys.stderr, flush=True)
        clk.mark_end()
    time.sleep(0.05)
    clk.__exit__(None, None, None)
    gc.enable()
    ms_total = ev0.elapsed_time(ev1)
    t_local = torch.tensor([ms_total], dtype=torch.float64, device=f"cuda:{local}")
    n_tot = torch.tensor([float(N)], dtype=torch.float64, device=f"cuda:{local}")
    if dist:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
        dist.all_reduce(n_tot, op=dist.ReduceOp.SUM)
    ms_step = float(t_local.item()) / args.steps
    value = float(n_tot.item()) / (ms_step / 1e3)

    # per-event outputs (comm-order waits and instance ids, event-order waits): device-to-device exports
    # after a fresh analysis, timed with CUDA events (they include the deferred scatter of the cross-stage
    # members' waits, k_xwait_scatter, which the analysis step leaves to the first export that needs it)
    exports = None
    if world == 1:
        s.analyze()
        torch.cuda.synchronize()
        names = ("comm_wait", "comm_inst", "ev_wait")
        bufs = {n: torch.empty(ms.scan_output_bytes(s.ctx, n), dtype=torch.uint8, device=f"cuda:{local}") for n in names}
        ex = {}
        for n in names:
            x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            x0.record(stream)
            nb = ms.scan_export_device(s.ctx, n, bufs[n])
            x1.record(stream)
            torch.cuda.synchronize()
            ex[n] = {"ms": x0.elapsed_time(x1), "bytes": nb}
        exports = {"per_event_exports": ex,
                   "note": "first export after an analysis; comm_wait / ev_wait include k_xwait_scatter (cross-stage "
                           "members' waits from instance-slot order to comm order)"}
        del bufs
    # verdicts for the record
    fused = bool(s.analyze()["fused"])
    verdict = s.export("wl_verdict")
    flagged = {int(r): int(v) for r, v in enumerate(verdict) if v}

    # ---- e2e: host pinned columns through the public API, H2D + analysis + D2H of the verdicts ----
    e2e = None
    if not args.no_e2e:
        s2 = ms.Scan(local, stream.cuda_stream, shards=(world, rank, ms.shard_unique_id()) if world > 1 else None)
        h2d = sum(v.nbytes for v in host.values())
        times = []
        for i in range(2):
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            t0 = time.perf_counter()
            s2.load(tr)
            s2.analyze()
            out_v = s2.export("wl_verdict")
            out_l = s2.export("lb_label")
            times.append(time.perf_counter() - t0)
        s2.close()
        d2h = out_v.nbytes + out_l.nbytes
        t_e2e = torch.tensor([min(times)], dtype=torch.float64, device=f"cuda:{local}")
        h2d_t = torch.tensor([float(h2d)], dtype=torch.float64, device=f"cuda:{local}")
        if dist:
            dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
            dist.all_reduce(h2d_t, op=dist.ReduceOp.SUM)
        e2e = {"value": float(n_tot.item()) / float(t_e2e.item()), "unit": "events/s",
               "h2d_bytes_per_step": int(h2d_t.item()), "d2h_bytes_per_step": int(d2h) * world,
               "seconds_per_step": float(t_e2e.item()),
               "path": "pinned host columns -> scan_load_events(SCAN_HOST_PTRS) -> scan_analyze -> scan_export"
                       " (verdicts + labels), wall clock" + (", max over ranks" if dist else "")}

    # ---- NEXT-1 timeline alignment (scan_align) on the same resident trace, N=1 only ----
    alignment = None
    if do_align:
        dev["start_ns"] = torch.from_numpy(tr.start_ns).cuda(local)
        torch.cuda.synchronize()
        s.load(tr, device_ptrs=True, cols=dev)
        s.analyze()  # instances (untimed here: the analysis is the main metric)
        for _ in range(max(1, args.warmup)):
            res_al = s.align(0)
        torch.cuda.synchronize()
        s.set_timing(True)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(args.steps):
            res_al = s.align(0)
        a1.record(stream)
        torch.cuda.synchronize()
        akern = s.kernel_timing()
        s.set_timing(False)
        ams = a0.elapsed_time(a1) / args.steps
        al_k = {k: v for k, v in akern.items() if k.startswith("k_al_")}
        apply_ms = al_k["k_al_apply"][0] / max(al_k["k_al_apply"][1], 1) if "k_al_apply" in al_k else None
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
        pk = float(peaks.get("hbm_gbs", 6650.0))
        alignment = {
            "metric": "trace events aligned/sec (scan_align, reference rank 0)", "value": N / (ams / 1e3),
            "unit": "events/s", "ms_per_call": ams, "result": {k: int(v) for k, v in res_al.items()},
            "kernels": {k: {"ms_per_call": round(v[0] / args.steps, 4), "launches": v[1]}
                        for k, v in sorted(al_k.items(), key=lambda kv: -kv[1][0])},
            "roofline": ({"bound": "hbm", "kernel": "k_al_apply", "bytes_per_event": 16,
                          "achieved": 16 * N / (apply_ms / 1e3) / 1e9, "peak": pk, "unit": "GB/s",
                          "frac": 16 * N / (apply_ms / 1e3) / 1e9 / pk} if apply_ms else None),
            "note": "start_ns resident in HBM; per call: candidate ends, monotonicity, BFS levels, per-level "
                    "anchors + aligned ends, aligned start of every event, residuals",
        }
        del dev["start_ns"]

    # ---- NEXT-4 event-level blame (scan_blame) on the same resident trace, N=1 only ----
    blame = None
    if world == 1 and not args.no_blame:
        s.analyze()
        for _ in range(max(1, args.warmup)):
            res_bl = s.blame()
        torch.cuda.synchronize()
        s.set_timing(True)
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        for _ in range(args.steps):
            res_bl = s.blame()
        b1.record(stream)
        torch.cuda.synchronize()
        bkern = s.kernel_timing()
        s.set_timing(False)
        bms = b0.elapsed_time(b1) / args.steps
        bl_k = {k: v for k, v in bkern.items() if k.startswith("k_bl_")}
        jump = bl_k.get("k_bl_jump")
        pk_b = float((json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}).get("hbm_gbs", 6650.0))
        jump_ms = jump[0] / args.steps if jump else None  # all rounds of one call
        jb_bytes = 4 * N + 12 * res_bl["n_active"]
        blame = {
            "metric": "trace events blamed/sec (scan_blame: root event of every wait, per-rank blame)",
            "value": N / (bms / 1e3), "unit": "events/s", "ms_per_call": bms,
            "result": {k: int(v) for k, v in res_bl.items()},
            "kernels": {k: {"ms_per_call": round(v[0] / args.steps, 4), "launches": v[1]}
                        for k, v in sorted(bl_k.items(), key=lambda kv: -kv[1][0])},
            "roofline": ({"bound": "hbm", "kernel": "k_bl_jump (all rounds of one call)",
                          "bytes_per_call": jb_bytes,
                          "achieved": jb_bytes / (jump_ms / 1e3) / 1e9, "peak": pk_b,
                          "unit": "GB/s", "frac": jb_bytes / (jump_ms / 1e3) / 1e9 / pk_b,
                          "note": "bytes of round 1 only: every event's pointer 4 B, and for the events whose pointer "
                                  "is not a root (n_active) a 4-byte gather, a 4-byte write and a 4-byte list append; "
                                  "later rounds (compacted lists of the pointers still moving) are not counted, so "
                                  "this is a lower bound"}
                         if jump_ms else None),
        }

    # ---- the general path on the same resident trace, N=1 only: forced, and as the fallback after one
    # SPMD violation (an op id changed on one rank: the fused pass rejects the trace, the general path reruns)
    general = None
    if world == 1 and not args.no_general:
        def timed_steps(n):
            s.set_timing(True)
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            for _ in range(n):
                r_ = s.analyze()
            g1.record(stream)
            torch.cuda.synchronize()
            kt = s.kernel_timing()
            s.set_timing(False)
            top = sorted(kt.items(), key=lambda kv: -kv[1][0])[:6]
            return g0.elapsed_time(g1) / n, r_, {k: round(v[0] / n, 4) for k, v in top}
        gsteps = max(2, min(args.steps, 3))
        s.force_general(True)
        s.analyze()
        gms, gres, gk = timed_steps(gsteps)
        s.force_general(False)
        e_bad = int(tr.rank_offsets[min(300, tr.world - 1)]) + 5000
        old_k = dev["kind_op"][e_bad].item()
        new_k = ((old_k & 0xFFFF) ^ (9 << 4)) & 0xFFFF
        dev["kind_op"][e_bad] = new_k - 0x10000 if new_k >= 0x8000 else new_k
        s.analyze()
        vms, vres, vk = timed_steps(gsteps)
        dev["kind_op"][e_bad] = old_k
        torch.cuda.synchronize()
        general = {
            "metric": "trace events analysed/sec on the general (non-SPMD) path",
            "forced": {"value": N / (gms / 1e3), "unit": "events/s", "ms_per_step": gms,
                       "hbm_frac": bpe_of(comm_frac) * N / (gms / 1e3) / 1e9 / peak_of(), "fused": bool(gres["fused"]),
                       "kernels_ms": gk},
            "one_violation": {"value": N / (vms / 1e3), "unit": "events/s", "ms_per_step": vms,
                              "hbm_frac": bpe_of(comm_frac) * N / (vms / 1e3) / 1e9 / peak_of(), "fused": bool(vres["fused"]),
                              "kernels_ms": vk,
                              "note": f"op id of event {e_bad} (rank {min(300, tr.world - 1)}) changed: the fused pass "
                                      "verifies, rejects, and the call reruns the general path (both inside the time)"},
        }

    streaming = streaming_c5(ms, torch, local, stream) if (world == 1 and not args.no_stream) else None
    json_ingest = json_io(ms, torch, local, stream, args.steps, args.warmup, not args.no_cpu) if (
        world == 1 and not args.no_json) else None

    if rank != 0:
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    bpe = alg_bytes_per_event(comm_frac)
    nbpe = needed_bytes_per_event(comm_frac, p2p_frac)
    dom = max(kernels.items(), key=lambda kv: kv[1][0]) if kernels else None
    kern_ms = sum(v[0] for v in kernels.values()) if kernels else None
    # dominant kernel (k_fused: reads every event column once and writes every per-event output, so
    # its algorithmic bytes per launch are the path's bpe x this GPU's events) / its mean launch time
    dom_ms = dom[1][0] / max(dom[1][1], 1) if dom else ms_step
    achieved = bpe * N / (dom_ms / 1e3) / 1e9
    step_achieved = bpe * N / (ms_step / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            if tj.get("config") == args.config and tj.get("iters") == total_iters and tj.get("n_gpus", 1) == world:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    cpu = None
    if not args.no_cpu and world == 1:
        cpu = cpu_oracle_rate(args.config, args.cpu_iters, args.seed)
        cpu.pop("seconds", None)
    line = {
        "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config] + (f" [{iters} it]" if iters else ""), "events": int(n_tot.item()),
                   "events_per_gpu": N, "comm_fraction": round(comm_frac, 4),
                   "parallelism": (f"{world} iteration-window shards (rank 0: iterations {blk[0]}..{blk[1] - 1}), "
                                   "NCCL all-gather + all-to-all + all-reduce inside scan_analyze") if world > 1
                                  else "1 GPU, whole trace",
                   "l2": "inputs (16 B/event, %.1f GB) >> 126 MB L2: no flush needed" % (16 * N / 1e9),
                   "timing": "step time: K steps between two CUDA events, nothing else recorded; kernel breakdown "
                             "and roofline: a second K steps with per-kernel CUDA events on the launch stream"
                             + (f" ({ms_total_ev / args.steps:.3f} ms/step with them)" if ms_total_ev else ""),
                   "generator_s": round(t_gen, 1)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)",
                     "bytes_per_event": round(bpe, 3),
                     "needed_bytes_per_event": round(nbpe, 3),
                     "frac_needed": nbpe * N / (dom_ms / 1e3) / 1e9 / peak,
                     "needed_note": "the same kernel time against the bytes the pass must move (dense dur + kind_op + comm, "
                                    "payload / meta at P2P events only, per-comm-event outputs, slow bits)",
                     "scope": "dominant kernel: algorithmic bytes per launch / its mean launch time (CUDA events on the "
                              "launch stream over the timed steps)",
                     "step_achieved": step_achieved, "step_frac": step_achieved / peak,
                     "dominant_kernel": ({"name": dom[0], "ms_per_launch": dom_ms, "launches": dom[1][1],
                                          "share": dom[1][0] / kern_ms} if dom else None)},
        "kernels": {k: {"ms_per_step": round(v[0] / args.steps, 4), "launches": v[1]}
                    for k, v in sorted(kernels.items(), key=lambda kv: -kv[1][0])},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches) * args.steps,
        "clocks": clk.summary(),
        "verdicts": {"flagged": flagged},
        "alignment": alignment,
        "streaming_c5": streaming,
        "json_ingest": json_ingest,
        "blame": blame,
        "exports": exports,
        "general_path": general,
        "path": "fused SPMD stage-tile pass (K9)" if fused else "general path",
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
