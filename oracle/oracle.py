"""ctypes bindings of the CPU ORACLE (test infrastructure only).

  COracle    oracle/lib/libldpc_oracle.so -- plain-C fp64 restatement
             (oracle/ldpc_oracle.c), always available once built
  RefOracle  oracle/_ref/libldpc_ref.so  -- the unmodified reference headers
             compiled through oracle/ref_driver.cpp (only where
             /root/reference existed at build time; the .so travels)

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this
module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
C_LIB = os.path.join(HERE, "lib", "libldpc_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libldpc_ref.so")

vp, i32, i64, u64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double


def build(quiet: bool = True) -> None:
    """make -C oracle (C restatement; the reference build when its headers exist)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{out.stdout}\n{out.stderr}")
    if not quiet:
        print(out.stdout)


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _groups_csr(groups):
    off = np.zeros(len(groups) + 1, np.int32)
    off[1:] = np.cumsum([len(g) for g in groups])
    cns = np.array([c for g in groups for c in g] or [0], np.int32)
    return off, cns


class PerFrame:
    """run_sweep's per-frame grouping (sim.hpp:113-117) in place of explicit
    groups: kind, G, overlap, schedule_seed, regroup_each_iteration."""

    def __init__(self, kind, n_groups, overlap, seed, regroup=True):
        self.kind, self.n_groups, self.overlap, self.seed, self.regroup = kind, n_groups, overlap, seed, regroup


class _Sched(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("n_groups", C.c_int),
        ("overlap", C.c_double),
        ("seed", C.c_uint64),
        ("regroup", C.c_int),
        ("grp_off", C.c_void_p),
        ("grp_cns", C.c_void_p),
        ("per_frame", C.c_int),
    ]


class COracle:
    """The plain-C restatement."""

    kind = "port"

    def __init__(self, path: str = C_LIB):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.orc_last_error.restype = C.c_char_p
        L.orc_mix_seed.restype = u64
        L.orc_mix_seed.argtypes = [u64, u64]
        L.orc_sigma2_from_ebn0.restype = dbl
        L.orc_sigma2_from_ebn0.argtypes = [dbl, dbl]
        L.orc_transmit_all_zero.argtypes = [dbl, u64, C.c_int, u64, vp]
        L.orc_transmit_batch_f32.argtypes = [dbl, u64, C.c_int, u64, i64, vp, C.c_int]
        L.orc_graph_create.restype = vp
        L.orc_graph_create.argtypes = [C.c_int, C.c_int, vp, vp]
        L.orc_graph_destroy.argtypes = [vp]
        L.orc_graph_n_edges.argtypes = [vp]
        L.orc_graph_var_view.argtypes = [vp, vp, vp, vp]
        L.orc_random_regular.argtypes = [C.c_int, C.c_int, C.c_int, u64, vp]
        L.orc_generate_groups.argtypes = [C.c_int, C.c_int, dbl, u64, vp, vp, C.c_int]
        L.orc_iteration_budget.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, dbl]
        L.orc_check_update.argtypes = [C.c_int, vp, vp]
        L.orc_decode.argtypes = [vp, C.POINTER(_Sched), vp, C.c_int, C.c_int, vp, vp, vp, vp, vp, vp]
        L.orc_decode_batch_f32.argtypes = [vp, C.POINTER(_Sched), vp, i64, C.c_int, C.c_int, C.c_int, vp, vp, vp,
                                           vp, vp]
        L.orc_run_subiterations.argtypes = [vp, C.POINTER(_Sched), vp, C.c_int, vp, vp]
        L.orc_simulate.argtypes = [vp, C.POINTER(_Sched), dbl, u64, u64, i64, C.c_int, C.c_int, C.c_int, C.c_int,
                                   vp]

    def err(self) -> str:
        return self.lib.orc_last_error().decode()

    # graphs ---------------------------------------------------------------
    def graph(self, n: int, row_off, cols):
        off = np.ascontiguousarray(row_off, np.int32)
        col = np.ascontiguousarray(cols, np.int32)
        h = self.lib.orc_graph_create(n, len(off) - 1, _p(off), _p(col))
        if not h:
            raise ValueError(self.err())
        return _Graph(self, h, n, len(off) - 1, int(off[-1]))

    def random_regular(self, n, dv, dc, seed) -> np.ndarray:
        out = np.empty(n * dv, np.int32)
        m = self.lib.orc_random_regular(n, dv, dc, seed, _p(out))
        if m < 0:
            raise ValueError(self.err())
        return out

    def generate_groups(self, M, G, overlap, seed_value) -> list[list[int]]:
        off = np.empty(G + 1, np.int32)
        cns = np.empty(2 * M + 1, np.int32)
        r = self.lib.orc_generate_groups(M, G, overlap, seed_value, _p(off), _p(cns), 2 * M + 1)
        if r < 0:
            raise ValueError(self.err())
        return [cns[off[k] : off[k + 1]].tolist() for k in range(G)]

    def mix_seed(self, seed, stream) -> int:
        return int(self.lib.orc_mix_seed(seed, stream))

    def iteration_budget(self, M, i_max, kind, G, group_size, overlap) -> int:
        return int(self.lib.orc_iteration_budget(M, i_max, kind, G, group_size, overlap))

    # channel --------------------------------------------------------------
    def sigma2_from_ebn0(self, ebn0, rate) -> float:
        return float(self.lib.orc_sigma2_from_ebn0(ebn0, rate))

    def transmit_all_zero(self, sigma2, seed, n, frame) -> np.ndarray:
        out = np.empty(n, np.float64)
        if self.lib.orc_transmit_all_zero(sigma2, seed, n, frame, _p(out)):
            raise ValueError(self.err())
        return out

    def transmit_batch_f32(self, sigma2, seed, n, frame0, frames, threads=8) -> np.ndarray:
        out = np.empty((frames, n), np.float32)
        self.lib.orc_transmit_batch_f32(sigma2, seed, n, frame0, frames, _p(out), threads)
        return out

    # decoder --------------------------------------------------------------
    def check_update(self, v2c) -> np.ndarray:
        x = np.ascontiguousarray(v2c, np.float64)
        out = np.empty_like(x)
        self.lib.orc_check_update(len(x), _p(x), _p(out))
        return out

    def _sched(self, groups, kind=2, overlap=0.0, seed=0, regroup=0):
        if isinstance(groups, PerFrame):
            p = groups
            return _Sched(p.kind, p.n_groups, p.overlap, p.seed, int(p.regroup), None, None, 1), None
        off, cns = _groups_csr(groups)
        s = _Sched(kind, len(groups), overlap, seed, regroup, off.ctypes.data, cns.ctypes.data, 0)
        return s, (off, cns)

    def decode(self, g, groups, llr, max_iters, early_stop=True, kind=2, overlap=0.0, seed=0, regroup=0):
        s, keep = self._sched(groups, kind, overlap, seed, regroup)
        x = np.ascontiguousarray(llr, np.float64)
        bits = np.empty(g.n, np.uint8)
        it, cv, cnu = C.c_int32(), C.c_uint8(), C.c_int64()
        post = np.empty(g.n, np.float64)
        trace = np.empty(max_iters, np.int32)
        r = self.lib.orc_decode(g.h, C.byref(s), _p(x), max_iters, int(early_stop), _p(bits), C.byref(it),
                                C.byref(cv), _p(post), _p(trace), C.byref(cnu))
        if r:
            raise ValueError(self.err())
        return dict(bits=bits, iterations=it.value, converged=bool(cv.value), posterior=post,
                    trace=trace, cn_updates=cnu.value)

    def decode_batch(self, g, groups, llr_f32, max_iters, early_stop=True, threads=8, posterior=False, trace=False):
        s, keep = self._sched(groups)
        x = np.ascontiguousarray(llr_f32, np.float32)
        F = x.shape[0]
        bits = np.empty((F, g.n), np.uint8)
        it = np.empty(F, np.int32)
        cv = np.empty(F, np.uint8)
        post = np.empty((F, g.n), np.float32) if posterior else None
        tr = np.empty((F, max_iters), np.int32) if trace else None
        r = self.lib.orc_decode_batch_f32(g.h, C.byref(s), _p(x), F, max_iters, int(early_stop), threads, _p(bits),
                                          _p(it), _p(cv), _p(post), _p(tr))
        if r:
            raise ValueError(self.err())
        out = dict(bits=bits, iterations=it, converged=cv)
        if posterior:
            out["posterior"] = post
        if trace:
            out["syndrome_trace"] = tr
        return out

    def run_subiterations(self, g, groups, llr, n_subiters):
        s, keep = self._sched(groups)
        x = np.ascontiguousarray(llr, np.float64)
        c2v = np.empty(g.E, np.float64)
        v2c = np.empty(g.E, np.float64)
        if self.lib.orc_run_subiterations(g.h, C.byref(s), _p(x), n_subiters, _p(c2v), _p(v2c)):
            raise ValueError(self.err())
        return c2v, v2c

    def simulate(self, g, groups, sigma2, seed, frame0, frames, max_iters, early_stop=True, round_f32=True,
                 threads=8):
        s, keep = self._sched(groups)
        cnt = np.zeros(6, np.int64)
        if self.lib.orc_simulate(g.h, C.byref(s), sigma2, seed, frame0, frames, max_iters, int(early_stop),
                                 int(round_f32), threads, _p(cnt)):
            raise ValueError(self.err())
        return cnt


class RefOracle:
    """The unmodified reference headers behind oracle/ref_driver.cpp."""

    kind = "reference"

    def __init__(self, path: str = REF_LIB):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_graph_create.restype = vp
        L.ref_graph_create.argtypes = [C.c_int, C.c_int, vp, vp]
        L.ref_graph_destroy.argtypes = [vp]
        L.ref_graph_var_view.argtypes = [vp, vp, vp, vp]
        L.ref_random_regular.argtypes = [C.c_int, C.c_int, C.c_int, u64, vp]
        L.ref_parse_alist.argtypes = [C.c_char_p, vp, vp, vp, vp, C.c_int, C.c_int, vp, vp]
        L.ref_serialize_alist.restype = C.c_long
        L.ref_serialize_alist.argtypes = [vp, C.c_char_p, C.c_long]
        L.ref_sigma2_from_ebn0.restype = dbl
        L.ref_sigma2_from_ebn0.argtypes = [dbl, dbl]
        L.ref_transmit_all_zero.argtypes = [dbl, u64, C.c_int, u64, vp]
        L.ref_transmit_batch_f32.argtypes = [dbl, u64, C.c_int, u64, i64, vp, C.c_int]
        L.ref_mix_seed.restype = u64
        L.ref_mix_seed.argtypes = [u64, u64]
        L.ref_rng_draw.argtypes = [u64, C.c_int, u64, C.c_int, vp, vp]
        L.ref_make_schedule.argtypes = [vp, C.c_int, C.c_int, dbl, u64, vp, vp, C.c_int, vp]
        L.ref_iteration_budget.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, dbl]
        L.ref_measure_cocsg.argtypes = [vp, C.c_int, vp, vp, vp]
        L.ref_check_update.argtypes = [C.c_int, vp, vp]
        L.ref_decode.argtypes = [vp, C.c_int, C.c_int, vp, vp, dbl, u64, C.c_int, vp, C.c_int, vp, vp, vp, vp, vp]
        L.ref_decode_composed.argtypes = [vp, C.c_int, C.c_int, vp, vp, dbl, u64, C.c_int, vp, C.c_int, C.c_int, vp,
                                          vp, vp, vp, vp]
        L.ref_run_subiterations.argtypes = [vp, C.c_int, vp, vp, vp, C.c_int, vp, vp]
        L.ref_decode_batch_f32.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp, i64, C.c_int, C.c_int, C.c_int, vp, vp,
                                           vp, vp]
        L.ref_run_sweep.argtypes = [vp, C.c_int, C.c_int, dbl, C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_long,
                                    C.c_int, u64, u64, C.c_int, vp]

    def err(self) -> str:
        return self.lib.ref_last_error().decode()

    def graph(self, n, row_off, cols):
        off = np.ascontiguousarray(row_off, np.int32)
        col = np.ascontiguousarray(cols, np.int32)
        h = self.lib.ref_graph_create(n, len(off) - 1, _p(off), _p(col))
        if not h:
            raise ValueError(self.err())
        return _Graph(self, h, n, len(off) - 1, int(off[-1]))

    def random_regular(self, n, dv, dc, seed) -> np.ndarray:
        out = np.empty(n * dv, np.int32)
        if self.lib.ref_random_regular(n, dv, dc, seed, _p(out)) < 0:
            raise ValueError(self.err())
        return out

    def parse_alist(self, text: str):
        n, m = C.c_int(), C.c_int()
        kind, line = C.c_int(-1), C.c_int(0)
        E = self.lib.ref_parse_alist(text.encode(), C.byref(n), C.byref(m), None, None, 0, 0, C.byref(kind),
                                     C.byref(line))
        if E < 0:
            return dict(error=self.err(), kind=kind.value, line=line.value)
        off = np.empty(m.value + 1, np.int32)
        cols = np.empty(E, np.int32)
        self.lib.ref_parse_alist(text.encode(), C.byref(n), C.byref(m), _p(off), _p(cols), m.value, E, None, None)
        return dict(n=n.value, row_off=off, cols=cols)

    def serialize_alist(self, g) -> str:
        L = self.lib.ref_serialize_alist(g.h, None, 0)
        buf = C.create_string_buffer(L + 1)
        self.lib.ref_serialize_alist(g.h, buf, L + 1)
        return buf.value.decode()

    def sigma2_from_ebn0(self, ebn0, rate) -> float:
        return float(self.lib.ref_sigma2_from_ebn0(ebn0, rate))

    def transmit_all_zero(self, sigma2, seed, n, frame) -> np.ndarray:
        out = np.empty(n, np.float64)
        if self.lib.ref_transmit_all_zero(sigma2, seed, n, frame, _p(out)):
            raise ValueError(self.err())
        return out

    def transmit_batch_f32(self, sigma2, seed, n, frame0, frames, threads=8) -> np.ndarray:
        out = np.empty((frames, n), np.float32)
        self.lib.ref_transmit_batch_f32(sigma2, seed, n, frame0, frames, _p(out), threads)
        return out

    def mix_seed(self, seed, stream) -> int:
        return int(self.lib.ref_mix_seed(seed, stream))

    def rng_draw(self, seed, kind, count, bound=0):
        u = np.zeros(count, np.uint64)
        d = np.zeros(count, np.float64)
        self.lib.ref_rng_draw(seed, kind, bound, count, _p(u), _p(d))
        return d if kind in (1, 2) else u

    def make_schedule(self, g, kind, G=1, overlap=0.0, seed=0):
        off = np.empty(G + 2, np.int32)
        cns = np.empty(2 * g.m + 1, np.int32)
        gs = C.c_int()
        r = self.lib.ref_make_schedule(g.h, kind, G, overlap, seed, _p(off), _p(cns), 2 * g.m + 1, C.byref(gs))
        if r < 0:
            raise ValueError(self.err())
        ng = 1 if kind == 0 else G
        return [cns[off[k] : off[k + 1]].tolist() for k in range(ng)], gs.value

    def iteration_budget(self, M, i_max, kind, G, group_size, overlap) -> int:
        return int(self.lib.ref_iteration_budget(M, i_max, kind, G, group_size, overlap))

    def measure_cocsg(self, g, groups):
        off, cns = _groups_csr(groups)
        out = np.zeros(max(len(groups) - 1, 1), np.int32)
        k = self.lib.ref_measure_cocsg(g.h, len(groups), _p(off), _p(cns), _p(out))
        return out[:k].tolist()

    def check_update(self, v2c) -> np.ndarray:
        x = np.ascontiguousarray(v2c, np.float64)
        out = np.empty_like(x)
        self.lib.ref_check_update(len(x), _p(x), _p(out))
        return out

    def decode(self, g, groups, llr, max_iters, early_stop=True, kind=2, overlap=0.0, seed=0, regroup=0,
               composed=False):
        off, cns = _groups_csr(groups)
        x = np.ascontiguousarray(llr, np.float64)
        bits = np.empty(g.n, np.uint8)
        it, cv = C.c_int32(), C.c_uint8()
        trace = np.empty(max_iters, np.int32)
        if composed or not early_stop:
            post = np.empty(g.n, np.float64)
            r = self.lib.ref_decode_composed(g.h, kind, len(groups), _p(off), _p(cns), overlap, seed, regroup, _p(x),
                                             max_iters, int(early_stop), _p(bits), C.byref(it), C.byref(cv),
                                             _p(post), _p(trace))
            cnu = None
        else:
            post = None
            cnu = C.c_int64()
            r = self.lib.ref_decode(g.h, kind, len(groups), _p(off), _p(cns), overlap, seed, regroup, _p(x),
                                    max_iters, _p(bits), C.byref(it), C.byref(cv), _p(trace), C.byref(cnu))
            cnu = cnu.value
        if r:
            raise ValueError(self.err())
        return dict(bits=bits, iterations=it.value, converged=bool(cv.value), posterior=post, trace=trace,
                    cn_updates=cnu)

    def decode_batch(self, g, groups, llr_f32, max_iters, early_stop=True, threads=8, posterior=False):
        off, cns = _groups_csr(groups)
        x = np.ascontiguousarray(llr_f32, np.float32)
        F = x.shape[0]
        bits = np.empty((F, g.n), np.uint8)
        it = np.empty(F, np.int32)
        cv = np.empty(F, np.uint8)
        post = np.empty((F, g.n), np.float32) if posterior else None
        r = self.lib.ref_decode_batch_f32(g.h, 2, len(groups), _p(off), _p(cns), _p(x), F, max_iters,
                                          int(early_stop), threads, _p(bits), _p(it), _p(cv), _p(post))
        if r:
            raise ValueError(self.err())
        out = dict(bits=bits, iterations=it, converged=cv)
        if posterior:
            out["posterior"] = post
        return out

    def run_subiterations(self, g, groups, llr, n_subiters):
        off, cns = _groups_csr(groups)
        x = np.ascontiguousarray(llr, np.float64)
        c2v = np.empty(g.E, np.float64)
        v2c = np.empty(g.E, np.float64)
        if self.lib.ref_run_subiterations(g.h, len(groups), _p(off), _p(cns), _p(x), n_subiters, _p(c2v), _p(v2c)):
            raise ValueError(self.err())
        return c2v, v2c

    def run_sweep(self, g, kind, n_groups, overlap, regroup, ebn0, i_max, budgeted, max_frames, min_frame_errors,
                  channel_seed, schedule_seed, workers):
        pts = np.ascontiguousarray(ebn0, np.float64)
        out = np.zeros((len(pts), 11), np.float64)
        r = self.lib.ref_run_sweep(g.h, kind, n_groups, overlap, regroup, _p(pts), len(pts), i_max, budgeted,
                                   max_frames, min_frame_errors, channel_seed, schedule_seed, workers, _p(out))
        if r < 0:
            raise ValueError(self.err())
        keys = ("frames", "bit_errors", "frame_errors", "converged_frames", "ber", "fer", "mean_iters_converged",
                "mean_iters_all", "iter_limit", "wall_seconds", "ebn0_db")
        return [dict(zip(keys, row.tolist())) for row in out]


class _Graph:
    def __init__(self, owner, h, n, m, E):
        self.owner, self.h, self.n, self.m, self.E = owner, h, n, m, E

    def __del__(self):
        try:
            if isinstance(self.owner, COracle):
                self.owner.lib.orc_graph_destroy(self.h)
            else:
                self.owner.lib.ref_graph_destroy(self.h)
        except Exception:
            pass

    def var_view(self):
        off = np.empty(self.n + 1, np.int32)
        cns = np.empty(self.E, np.int32)
        eid = np.empty(self.E, np.int32)
        if isinstance(self.owner, COracle):
            self.owner.lib.orc_graph_var_view(self.h, _p(off), _p(cns), _p(eid))
        else:
            self.owner.lib.ref_graph_var_view(self.h, _p(off), _p(cns), _p(eid))
        return off, cns, eid


def best_available():
    """The reference build when present (kind 'reference'), else the C port."""
    if os.path.exists(REF_LIB):
        return RefOracle()
    return COracle()
