"""Reassemble per-shard exports of a sharded analysis into the job-wide layout (test plumbing,
no method arithmetic). Shard s holds iterations [b_s, e_s) of every rank (scan.h "multi-GPU"):

* event-indexed outputs (ev_*): rank r's events are shard 0's slice of r, then shard 1's, ...
* instance-indexed outputs (in_*): shard s holds occurrences [ch_shard_k0[c], +ch_shard_n[c])
  of channel c, i.e. rows ch_base[c] + k;
* every other output is job-wide and must be identical on every shard.
"""
from __future__ import annotations

import numpy as np

EV_KEYS = ("ev_inst", "ev_wait", "ev_slow", "ev_ref")


def merge(parts: list[dict]) -> tuple[dict, list[str]]:
    """parts[s] = {"out": export_all() + ch_shard_k0 / ch_shard_n, "ro": rank offsets of shard s,
    "res": analyze() result}. Returns (merged outputs, list of cross-shard inconsistencies)."""
    issues = []
    base = parts[0]["out"]
    merged = {}
    W = len(parts[0]["ro"]) - 1
    for k, v0 in base.items():
        if not isinstance(v0, np.ndarray) or k in ("ch_shard_k0", "ch_shard_n"):
            continue
        if k in EV_KEYS:
            pieces = []
            for r in range(W):
                for p in parts:
                    ro = p["ro"]
                    pieces.append(p["out"][k][int(ro[r]):int(ro[r + 1])])
            merged[k] = np.concatenate(pieces) if pieces else v0[:0]
        elif k.startswith("in_"):
            out = np.zeros_like(v0)
            chb = base["ch_base"].astype(np.int64)
            for p in parts:
                k0 = p["out"]["ch_shard_k0"].astype(np.int64)
                n = p["out"]["ch_shard_n"].astype(np.int64)
                for c in np.nonzero(n)[0]:
                    a = chb[c] + k0[c]
                    out[a:a + n[c]] = p["out"][k][a:a + n[c]]
            merged[k] = out
        else:
            for s, p in enumerate(parts[1:], 1):
                v = p["out"][k]
                same = v.shape == v0.shape and (np.array_equal(v, v0) if v.dtype.kind != "f" else
                                                np.array_equal(v, v0) or np.allclose(v, v0, rtol=0, atol=0))
                if not same:
                    issues.append(f"{k}: shard {s} differs from shard 0")
            merged[k] = v0
    for s, p in enumerate(parts[1:], 1):
        if p["res"]["status"] != parts[0]["res"]["status"]:
            issues.append(f"status: shard {s} differs")
        for sect in ("match", "detect", "localize"):
            if p["res"][sect] != parts[0]["res"][sect]:
                issues.append(f"{sect} result: shard {s} differs")
    return merged, issues


def coverage(parts: list[dict], n_inst: int) -> np.ndarray:
    """How many shards claim each instance id (must be exactly one)."""
    cnt = np.zeros(n_inst, np.int64)
    chb = parts[0]["out"]["ch_base"].astype(np.int64)
    for p in parts:
        k0 = p["out"]["ch_shard_k0"].astype(np.int64)
        n = p["out"]["ch_shard_n"].astype(np.int64)
        for c in np.nonzero(n)[0]:
            cnt[chb[c] + k0[c]:chb[c] + k0[c] + n[c]] += 1
    return cnt
