"""BASELINE.json configurations (codes, schedules, operating points).

C1  (3,6)-regular n=1008 with 4-cycles removed; NDGSBP 8 windows of 84 at
    stride 63 (wrapping, 21-CN overlap), GSBP 8 x 63, flooding; 2.0 dB,
    <=20 iterations with early stop, 10^4 frames.
C2  same code, 1.0-3.0 dB in 0.25 dB steps, 10^6 frames per point.
C3  QC 12x24 base, Z=81 (n=1944), p(-1)=0.65, shifts U[0,80], column degree
    >= 2; 6 groups of 3 block rows at stride 2; 1.5-2.5 dB, <=15 iterations.
C4  irregular n=64800, VN degrees {2:50%, 3:40%, 8:10%}, d_c=6; NDGSBP 45
    windows of 960 at stride 720; 0.9-1.3 dB, <=30 iterations.
C5  throughput: C1 code at 2.0 dB and C4 code at 1.1 dB, NDGSBP, fixed 10
    iterations, no early stop.
"""
from __future__ import annotations

from functools import lru_cache

from .api import DISJOINT, FLOODING, NONDISJOINT, GroupSchedule, TannerGraph

CODE_SEED = 1
CHANNEL_SEED = 1


@lru_cache(maxsize=None)
def c1_code(seed: int = CODE_SEED) -> TannerGraph:
    return TannerGraph.random_regular_girth6(1008, 3, 6, seed)


@lru_cache(maxsize=None)
def c3_code(seed: int = CODE_SEED) -> TannerGraph:
    return TannerGraph.qc(12, 24, 81, 0.65, 2, seed)


@lru_cache(maxsize=None)
def c4_code(seed: int = CODE_SEED) -> TannerGraph:
    return TannerGraph.irregular(64800, [2, 3, 8], [32400, 25920, 6480], 6, seed)


def c1_schedules(g: TannerGraph) -> dict:
    return {
        "ndgsbp": GroupSchedule.windows(g, 8, 84, 63, NONDISJOINT),
        "gsbp": GroupSchedule.windows(g, 8, 63, 63, DISJOINT),
        "bp": GroupSchedule.flooding(g),
    }


def c3_schedules(g: TannerGraph) -> dict:
    z = 81
    return {
        "ndgsbp": GroupSchedule.windows(g, 6, 3 * z, 2 * z, NONDISJOINT),
        "gsbp": GroupSchedule.windows(g, 6, 2 * z, 2 * z, DISJOINT),
        "bp": GroupSchedule.flooding(g),
    }


def c4_schedules(g: TannerGraph) -> dict:
    return {
        "ndgsbp": GroupSchedule.windows(g, 45, 960, 720, NONDISJOINT),
        "gsbp": GroupSchedule.windows(g, 45, 720, 720, DISJOINT),
        "bp": GroupSchedule.flooding(g),
    }


C1 = dict(ebn0_db=2.0, max_iters=20, early_stop=True, frames=10_000)
C2 = dict(ebn0_db=[1.0 + 0.25 * i for i in range(9)], max_iters=20, early_stop=True, frames=1_000_000)
C3 = dict(ebn0_db=[1.5, 2.0, 2.5], max_iters=15, early_stop=True, frames=1 << 22)
C4 = dict(ebn0_db=[0.9, 1.0, 1.1, 1.2, 1.3], max_iters=30, early_stop=True, frames=1 << 18)
C5_SHORT = dict(ebn0_db=2.0, max_iters=10, early_stop=False, frames=1 << 26)
C5_LONG = dict(ebn0_db=1.1, max_iters=10, early_stop=False, frames=1 << 20)

FLOODING_KIND = FLOODING
