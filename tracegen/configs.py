"""The five BASELINE.json configs as generator recipes.

C1 is the small parity case; C3 is the bench workload (the north-star target: a
1024-rank x 1000-iteration trace on 1 B200). Faults follow the SURVEY.md §8(d) table.
"""
from __future__ import annotations

from . import Fault, GenConfig, LINK_DEGRADE, LINK_JITTER, THROTTLE


def _rank(tp, dp, t, d, s):
    return t + tp * (d + dp * s)


def _fwd_links(tp, dp, stage):
    """All forward P2P links leaving `stage` (src on `stage`, dst on `stage+1`)."""
    return [(_rank(tp, dp, t, d, stage), _rank(tp, dp, t, d, stage + 1)) for d in range(dp) for t in range(tp)]


def c1(seed: int = 1, iterations: int = 10) -> GenConfig:
    """8-rank TP2xPP2xDP2, 24 layers (L_s=12), M=8, 10 it; rank 5 = (tp1,dp0,pp1) throttled x2.0."""
    return GenConfig(2, 2, 2, 12, 8, iterations, seed=seed,
                     faults=[Fault(THROTTLE, 5, factor=2.0)])


def c2(seed: int = 1, iterations: int = 200) -> GenConfig:
    """64-rank TP8xPP4xDP2, L_s=8, M=16, 200 it; jitter x(1+Exp(1)) on all 16 fwd links leaving stage 1."""
    return GenConfig(8, 4, 2, 8, 16, iterations, seed=seed,
                     faults=[Fault(LINK_JITTER, s, d) for s, d in _fwd_links(8, 2, 1)])


def c3(seed: int = 1, iterations: int = 1000) -> GenConfig:
    """1024-rank TP8xPP8xDP16, L_s=8, M=8, 1000 it; rank 299 x1.6 on [200,600), rank 862 x2.5 on
    [500,900), jitter on the 128 fwd links leaving stage 4."""
    it = iterations
    return GenConfig(8, 8, 16, 8, 8, it, seed=seed,
                     faults=[Fault(THROTTLE, 299, it0=it * 2 // 10, it1=it * 6 // 10, factor=1.6),
                             Fault(THROTTLE, 862, it0=it * 5 // 10, it1=it * 9 // 10, factor=2.5)]
                     + [Fault(LINK_JITTER, s, d) for s, d in _fwd_links(8, 16, 4)])


def c4(seed: int = 1, iterations: int = 500) -> GenConfig:
    """3072-rank TP8xPP64xDP6 (1T-shaped), L_s=2, M=16, 500 it, hidden 25600; one rank x1.5 and one
    link at x0.5 bandwidth."""
    slow = _rank(8, 6, 5, 3, 40)
    src, dst = _rank(8, 6, 2, 1, 20), _rank(8, 6, 2, 1, 21)
    return GenConfig(8, 64, 6, 2, 16, iterations, seed=seed, hidden=25600,
                     faults=[Fault(THROTTLE, slow, factor=1.5), Fault(LINK_DEGRADE, src, dst, factor=0.5)])


def c5(seed: int = 1, iterations: int = 100) -> GenConfig:
    """512-rank TP8xPP8xDP8, L_s=8, M=8, 100 it (50-it sliding window); cascading victims: rank 208 =
    (tp0,dp2,pp3) x2.5 from it 30, its 7 TP peers x1.8 on 40% of their compute ops."""
    src = 208
    peers = [_rank(8, 8, t, 2, 3) for t in range(1, 8)]
    return GenConfig(8, 8, 8, 8, 8, iterations, seed=seed,
                     faults=[Fault(THROTTLE, src, it0=30, factor=2.5)]
                     + [Fault(THROTTLE, p, it0=30, factor=1.8, prob=0.4) for p in peers])


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}
