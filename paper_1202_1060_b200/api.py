"""Host-side mirror of the reference decoder interface over the C ABI.

Names, argument meaning and error behaviour follow the reference's header API
(arxiv/paper_1202_1060 proj/include/ldpc/*.hpp):

  TannerGraph            tanner.hpp:21-37  (build_from_check_lists :79-114,
                         random_regular_graph :356-393, parse_alist :172-282,
                         serialize_alist :286-317)
  GroupSchedule          schedule.hpp:32-40 (make_*_schedule :129-171,
                         iteration_budget :206-210, measure_cocsg :175-201)
  sigma2_from_ebn0       channel.hpp:21-24
  transmit_all_zero      channel.hpp:38-46  (device generator, fp32 output)
  decode / DecodeOutcome decoder.hpp:31-37, 143-181
  check_update           decoder.hpp:59-87
  run_subiterations      decoder.hpp:39-52 + 112-127

std::invalid_argument becomes ValueError, AlistError keeps .kind / .line.
Every compute call runs the sm_100a kernels of libldpc_b200.so; there is no
CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import AlistError, check, lib

FLOODING, DISJOINT, NONDISJOINT = 0, 1, 2
KIND_NAMES = {FLOODING: "bp", DISJOINT: "gsbp", NONDISJOINT: "ndgsbp"}  # schedule.hpp:18-25
COUNTER_NAMES = ("frames", "bit_errors", "frame_errors", "converged_frames", "iter_sum", "iter_sum_converged")


def _vp(a):
    """ctypes pointer of a numpy array, a torch tensor, or None."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return C.c_void_p(a.ctypes.data)
    return C.c_void_p(a.data_ptr())  # torch.Tensor


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _csr(lists) -> tuple[np.ndarray, np.ndarray]:
    off = np.zeros(len(lists) + 1, dtype=np.int32)
    off[1:] = np.cumsum([len(x) for x in lists])
    flat = _i32([v for row in lists for v in row]) if off[-1] else np.zeros(1, np.int32)
    return off, flat


class TannerGraph:
    """Immutable code graph with CN-major edge ids (tanner.hpp:16-37)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        n, m, e, dc, dv = (C.c_int32() for _ in range(5))
        check(lib.ldpcb_code_dims(self._h, n, m, e, dc, dv))
        self.n_vars, self.n_checks, self.n_edges = n.value, m.value, e.value
        self.max_check_degree, self.max_var_degree = dc.value, dv.value
        self._csr = None
        self._csc = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.ldpcb_code_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    # ---- constructors -------------------------------------------------
    @classmethod
    def _make(cls, fn, *args, what=""):
        h = C.c_void_p()
        check(fn(*args, C.byref(h)), what)
        return cls(h)

    @classmethod
    def from_check_lists(cls, n_vars: int, check_lists) -> "TannerGraph":
        off, flat = _csr(check_lists)
        return cls._make(lib.ldpcb_code_from_check_lists, n_vars, len(check_lists), _vp(off), _vp(flat))

    @classmethod
    def from_csr(cls, n_vars: int, row_off, cols) -> "TannerGraph":
        off, flat = _i32(row_off), _i32(cols)
        return cls._make(lib.ldpcb_code_from_check_lists, n_vars, len(off) - 1, _vp(off), _vp(flat))

    @classmethod
    def random_regular(cls, n_vars: int, dv: int, dc: int, seed: int) -> "TannerGraph":
        return cls._make(lib.ldpcb_code_random_regular, n_vars, dv, dc, seed)

    @classmethod
    def random_regular_girth6(cls, n_vars: int, dv: int, dc: int, seed: int) -> "TannerGraph":
        return cls._make(lib.ldpcb_code_random_regular_girth6, n_vars, dv, dc, seed)

    @classmethod
    def qc(cls, base_rows=12, base_cols=24, z=81, p_empty=0.65, min_col_degree=2, seed=1) -> "TannerGraph":
        return cls._make(lib.ldpcb_code_qc, base_rows, base_cols, z, p_empty, min_col_degree, seed)

    @classmethod
    def irregular(cls, n_vars: int, degrees, counts, dc: int, seed: int) -> "TannerGraph":
        d, c = _i32(degrees), _i32(counts)
        return cls._make(lib.ldpcb_code_irregular, n_vars, len(d), _vp(d), _vp(c), dc, seed)

    @classmethod
    def parse_alist(cls, text: str) -> "TannerGraph":
        h = C.c_void_p()
        kind, line = C.c_int(-1), C.c_int(0)
        st = lib.ldpcb_code_parse_alist(text.encode(), C.byref(h), C.byref(kind), C.byref(line))
        if st == _lib.EALIST:
            raise AlistError(lib.ldpcb_last_error().decode(), kind.value, line.value)
        check(st)
        return cls(h)

    # ---- views ----------------------------------------------------------
    def csr(self) -> tuple[np.ndarray, np.ndarray]:
        if self._csr is None:
            off = np.empty(self.n_checks + 1, np.int32)
            cols = np.empty(max(self.n_edges, 1), np.int32)
            check(lib.ldpcb_code_export(self._h, _vp(off), _vp(cols), None, None, None))
            self._csr = (off, cols[: self.n_edges])
        return self._csr

    def csc(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        if self._csc is None:
            off = np.empty(self.n_vars + 1, np.int32)
            cns = np.empty(max(self.n_edges, 1), np.int32)
            eid = np.empty(max(self.n_edges, 1), np.int32)
            check(lib.ldpcb_code_export(self._h, None, None, _vp(off), _vp(cns), _vp(eid)))
            self._csc = (off, cns[: self.n_edges], eid[: self.n_edges])
        return self._csc

    @property
    def check_edge_offset(self) -> list[int]:
        return self.csr()[0].tolist()

    @property
    def check_adj(self) -> list[list[int]]:
        off, cols = self.csr()
        return [cols[off[r] : off[r + 1]].tolist() for r in range(self.n_checks)]

    @property
    def var_adj(self) -> list[list[int]]:
        off, cns, _ = self.csc()
        return [cns[off[v] : off[v + 1]].tolist() for v in range(self.n_vars)]

    @property
    def var_edge_ids(self) -> list[list[int]]:
        off, _, eid = self.csc()
        return [eid[off[v] : off[v + 1]].tolist() for v in range(self.n_vars)]

    def check_degree(self, m: int) -> int:
        off = self.csr()[0]
        return int(off[m + 1] - off[m])

    def var_degree(self, n: int) -> int:
        off = self.csc()[0]
        return int(off[n + 1] - off[n])

    def edge_id(self, m: int, slot: int) -> int:
        return int(self.csr()[0][m]) + slot

    @property
    def rate(self) -> float:
        """(n - m) / n, the reference harness's rate convention (sim.hpp:103)."""
        return (self.n_vars - self.n_checks) / self.n_vars

    def serialize_alist(self) -> str:
        n = C.c_int64()
        check(lib.ldpcb_code_serialize_alist(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(lib.ldpcb_code_serialize_alist(self._h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def count_4cycles(self) -> int:
        c = C.c_int64()
        check(lib.ldpcb_code_count_4cycles(self._h, C.byref(c)))
        return c.value

    def __eq__(self, other) -> bool:  # tanner.hpp:34-36
        if not isinstance(other, TannerGraph):
            return NotImplemented
        return (
            self.n_vars == other.n_vars
            and self.n_checks == other.n_checks
            and all(np.array_equal(a, b) for a, b in zip(self.csr(), other.csr()))
        )

    __hash__ = None


class GroupSchedule:
    """Ordered CN groups processed one sub-iteration each (schedule.hpp:32-40).

    The device schedule is fixed for the whole decode
    (regroup_each_iteration = false, decoder.hpp:150-157)."""

    regroup_each_iteration = False

    def __init__(self, graph: TannerGraph, handle: C.c_void_p):
        self.graph = graph
        self._h = handle
        kind, G, slots, gsz = (C.c_int32() for _ in range(4))
        ov = C.c_double()
        eu, tu = C.c_int64(), C.c_int64()
        check(lib.ldpcb_schedule_dims(self._h, kind, G, slots, gsz, ov, eu, tu))
        self.kind, self.n_groups, self.n_slots = kind.value, G.value, slots.value
        self.group_size, self.overlap_ratio = gsz.value, ov.value
        self.edge_updates_per_iter, self.touched_per_iter = eu.value, tu.value
        self._groups = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.ldpcb_schedule_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @classmethod
    def _make(cls, g: TannerGraph, fn, *args):
        h = C.c_void_p()
        check(fn(g.handle, *args, C.byref(h)))
        return cls(g, h)

    @classmethod
    def from_groups(cls, g: TannerGraph, kind: int, groups) -> "GroupSchedule":
        off, flat = _csr(groups)
        return cls._make(g, lib.ldpcb_schedule_from_groups, kind, len(groups), _vp(off), _vp(flat))

    @classmethod
    def flooding(cls, g: TannerGraph) -> "GroupSchedule":
        return cls._make(g, lib.ldpcb_schedule_flooding)

    @classmethod
    def disjoint(cls, g: TannerGraph, n_groups: int, seed: int) -> "GroupSchedule":
        return cls._make(g, lib.ldpcb_schedule_disjoint, n_groups, seed)

    @classmethod
    def nondisjoint(cls, g: TannerGraph, n_groups: int, overlap: float, seed: int) -> "GroupSchedule":
        return cls._make(g, lib.ldpcb_schedule_nondisjoint, n_groups, overlap, seed)

    @classmethod
    def per_frame(cls, g: TannerGraph, kind: int, n_groups: int = 1, overlap: float = 0.0, schedule_seed: int = 2,
                  regroup_each_iteration: bool = True) -> "GroupSchedule":
        """The reference harness's grouping (sim.hpp:113-117, decoder.hpp:153-156):
        random groups per frame (and per iteration when regrouping)."""
        s = cls._make(g, lib.ldpcb_schedule_per_frame, kind, n_groups, overlap, schedule_seed,
                      int(regroup_each_iteration))
        s.regroup_each_iteration = bool(regroup_each_iteration) and kind != FLOODING
        s.per_frame_seed = schedule_seed if kind != FLOODING else None
        return s

    @classmethod
    def windows(cls, g: TannerGraph, n_groups: int, window: int, stride: int, kind: int | None = None):
        if kind is None:
            kind = NONDISJOINT if window > stride else DISJOINT
        return cls._make(g, lib.ldpcb_schedule_windows, kind, n_groups, window, stride)

    @property
    def groups(self) -> list[list[int]]:
        if self._groups is None:
            off = np.empty(self.n_groups + 1, np.int32)
            cns = np.empty(max(self.n_slots, 1), np.int32)
            check(lib.ldpcb_schedule_export(self._h, _vp(off), _vp(cns)))
            self._groups = [cns[off[k] : off[k + 1]].tolist() for k in range(self.n_groups)]
        return self._groups

    def frame_groups(self, frame0: int, frames: int, iteration: int = 1) -> "torch.Tensor":
        """Device-generated groups of a per-frame schedule: int32 [frames, n_slots]
        in group order (split at the offsets of ``groups``)."""
        import torch
        out = torch.empty((frames, self.n_slots), dtype=torch.int16, device="cuda")
        check(lib.ldpcb_schedule_per_frame_groups_device(self.graph.handle, self._h, frame0, frames, iteration,
                                                         out.data_ptr(), _stream()))
        return out.view(torch.uint16).to(torch.int32) if hasattr(torch, "uint16") else (out.to(torch.int32) & 0xFFFF)

    def direct_layout(self) -> dict | None:
        """Tables of the posterior-free resident kernel for this schedule (csrc/host.hpp
        DirectTables), or None where that kernel does not apply: frames per thread, cell
        counts, wavefronts per shared-memory access after bank colouring, and the records
        (byte offsets into the cell array)."""
        fv, cells, lb, buf, items = (C.c_int32() for _ in range(5))
        wf = C.c_double()
        check(lib.ldpcb_schedule_direct_layout(self._h, fv, cells, lb, buf, items, wf))
        if fv.value == 0:
            return None
        g = self.graph
        out = {"frames_per_thread": fv.value, "cells": cells.value, "l_base": lb.value, "buffer_cells": buf.value,
               "wavefronts_per_access": wf.value,
               "cn_off": np.empty(self.n_groups + 1, np.int32), "cn_rec": np.empty(12 * items.value, np.int32),
               "vn_rec": np.empty(2 * g.n_vars, np.int32), "vn_hold": np.empty(g.n_vars, np.int32),
               "vn_pos": np.empty(g.n_vars, np.int32), "edge_rec": np.empty(2 * g.n_edges, np.int32)}
        check(lib.ldpcb_schedule_direct_export(self._h, *(_vp(out[k]) for k in
                                                          ("cn_off", "cn_rec", "vn_rec", "vn_hold", "vn_pos", "edge_rec"))))
        return out

    def iteration_budget(self, i_max: int) -> int:
        b = C.c_int32()
        check(lib.ldpcb_schedule_iteration_budget(self._h, i_max, C.byref(b)))
        return b.value

    def measure_cocsg(self) -> list[int]:
        out = np.zeros(max(self.n_groups - 1, 1), np.int32)
        check(lib.ldpcb_schedule_cocsg(self._h, _vp(out)))
        return out[: max(self.n_groups - 1, 0)].tolist()

    @property
    def name(self) -> str:
        return KIND_NAMES[self.kind]


def make_flooding_schedule(g):
    return GroupSchedule.flooding(g)


def make_disjoint_schedule(g, n_groups, seed):
    return GroupSchedule.disjoint(g, n_groups, seed)


def make_nondisjoint_schedule(g, n_groups, overlap, seed):
    return GroupSchedule.nondisjoint(g, n_groups, overlap, seed)


def sigma2_from_ebn0(ebn0_db: float, rate: float) -> float:
    out = C.c_double()
    check(lib.ldpcb_sigma2_from_ebn0(ebn0_db, rate, C.byref(out)))
    return out.value


# --------------------------------------------------------------------------
# device calls (torch provides device memory and the stream)
# --------------------------------------------------------------------------


def _torch():
    import torch

    return torch


def _stream(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def transmit_all_zero(n: int, sigma2: float, seed: int, frame0: int, frames: int, out=None, stream=None):
    """Device transmit_all_zero for frames [frame0, frame0+frames) -> fp32 [frames, n]."""
    torch = _torch()
    if out is None:
        out = torch.empty((frames, n), dtype=torch.float32, device="cuda")
    check(lib.ldpcb_channel_llr_device(n, sigma2, seed, frame0, frames, _vp(out), _stream(stream)), "channel")
    return out


def decode_batch(
    g: TannerGraph,
    s: GroupSchedule,
    llr,
    max_iters: int,
    early_stop: bool = True,
    bits: bool = True,
    packed: bool = False,
    posterior: bool = False,
    trace: bool = False,
    counters=None,
    stream=None,
) -> dict:
    """decode() over a batch of device-resident fp32 LLRs [frames, n].

    Returns a dict of device tensors: bits, iterations, converged and
    optionally posterior, syndrome_trace. `counters` (int64[6] cuda tensor)
    is accumulated into when given."""
    torch = _torch()
    _device_counters(counters)
    if llr.dtype != torch.float32 or not llr.is_cuda or not llr.is_contiguous():
        raise ValueError("llr must be a contiguous float32 CUDA tensor")
    if llr.dim() != 2 or llr.shape[1] != g.n_vars:
        raise ValueError("channel LLR length does not match the code length")
    F = llr.shape[0]
    dev = llr.device
    out = {
        "iterations": torch.empty(F, dtype=torch.int32, device=dev),
        "converged": torch.empty(F, dtype=torch.uint8, device=dev),
    }
    if bits:
        nb = (g.n_vars + 7) // 8 if packed else g.n_vars
        out["bits"] = torch.empty((F, nb), dtype=torch.uint8, device=dev)
    if posterior:
        out["posterior"] = torch.empty((F, g.n_vars), dtype=torch.float32, device=dev)
    if trace:
        out["syndrome_trace"] = torch.empty((F, max_iters), dtype=torch.int32, device=dev)
    check(
        lib.ldpcb_decode_device(
            g.handle,
            s.handle,
            F,
            _vp(llr),
            max_iters,
            int(early_stop),
            _vp(out.get("bits")),
            int(packed),
            _vp(out["iterations"]),
            _vp(out["converged"]),
            _vp(out.get("posterior")),
            _vp(out.get("syndrome_trace")),
            _vp(counters),
            _stream(stream),
        ),
        "decode",
    )
    return out


_NP_OF_TORCH = {"torch.float32": np.float32, "torch.uint8": np.uint8, "torch.int32": np.int32,
                "torch.int64": np.int64}


def _host_check(a, dtype, size, name):
    """Host buffer passed as a raw pointer: C-contiguous, host-resident, the
    given dtype and (when size is not None) exactly `size` elements. Returns
    the leading dimension."""
    if a is None:
        return 0
    if isinstance(a, np.ndarray):
        ok_dtype = a.dtype == np.dtype(dtype)
        contiguous = a.flags["C_CONTIGUOUS"]
        count = a.size
    else:  # torch.Tensor on the host (pinned or pageable)
        if a.is_cuda:
            raise ValueError(f"{name} must be a host buffer")
        ok_dtype = _NP_OF_TORCH.get(str(a.dtype)) is dtype
        contiguous = a.is_contiguous()
        count = a.numel()
    if not ok_dtype:
        raise ValueError(f"{name} must be {np.dtype(dtype).name}, got {a.dtype}")
    if not contiguous:
        raise ValueError(f"{name} must be C-contiguous")
    if size is not None and count != size:
        raise ValueError(f"{name} must hold exactly {size} elements, got {count}")
    return a.shape[0] if a.ndim else 0


def _device_counters(counters, name="counters"):
    if counters is None:
        return
    if not getattr(counters, "is_cuda", False) or str(counters.dtype) != "torch.int64" or counters.numel() != 6 \
            or not counters.is_contiguous():
        raise ValueError(f"{name} must be a contiguous int64[6] CUDA tensor")


def decode_host(
    g: TannerGraph,
    s: GroupSchedule,
    llr: np.ndarray,
    max_iters: int,
    early_stop: bool = True,
    packed: bool = True,
    bits=None,
    iterations=None,
    converged=None,
    posterior=None,
    counters=None,
    syndrome_trace=None,
):
    """decode() from host memory (numpy / pinned torch CPU tensors); blocks.

    The library reads LLRs as fp32 and writes every output with a D2H copy of
    its exact size, so dtypes and sizes are checked here (a float64 array, the
    reference decoder's own LLR type, is rejected instead of being read as
    fp32 garbage)."""
    F = _host_check(llr, np.float32, None, "llr")
    if llr.ndim != 2 or llr.shape[1] != g.n_vars:
        raise ValueError("channel LLR length does not match the code length")
    n = g.n_vars
    _host_check(bits, np.uint8, F * ((n + 7) // 8 if packed else n), "bits")
    _host_check(iterations, np.int32, F, "iterations")
    _host_check(converged, np.uint8, F, "converged")
    _host_check(posterior, np.float32, F * n, "posterior")
    _host_check(syndrome_trace, np.int32, F * max_iters, "syndrome_trace")
    _host_check(counters, np.int64, 6, "counters")
    check(
        lib.ldpcb_decode_host(
            g.handle,
            s.handle,
            F,
            _vp(llr),
            max_iters,
            int(early_stop),
            _vp(bits),
            int(packed),
            _vp(iterations),
            _vp(converged),
            _vp(posterior),
            _vp(syndrome_trace),
            _vp(counters),
        ),
        "decode_host",
    )


def simulate(g, s, sigma2: float, channel_seed: int, frame_begin: int, frames: int, max_iters: int,
             early_stop: bool = True, counters=None, stream=None):
    """Device Monte-Carlo over frames [frame_begin, frame_begin+frames): returns
    (or accumulates into) the int64[6] counters of sim.hpp:162-181."""
    torch = _torch()
    if counters is None:
        counters = torch.zeros(6, dtype=torch.int64, device="cuda")
    _device_counters(counters)
    check(
        lib.ldpcb_simulate_device(
            g.handle, s.handle, sigma2, channel_seed, frame_begin, frames, max_iters, int(early_stop),
            _vp(counters), _stream(stream),
        ),
        "simulate",
    )
    return counters


def simulate_frames(g, s, sigma2: float, channel_seed: int, frame_begin: int, frames: int, max_iters: int,
                    early_stop: bool = True, stream=None):
    """Per-frame outcomes of frames [frame_begin, frame_begin+frames) (run_frame,
    sim.hpp:111-124): device int32 bit_errors, int32 iterations, uint8 converged."""
    torch = _torch()
    be = torch.empty(frames, dtype=torch.int32, device="cuda")
    it = torch.empty(frames, dtype=torch.int32, device="cuda")
    cv = torch.empty(frames, dtype=torch.uint8, device="cuda")
    check(
        lib.ldpcb_simulate_frames_device(
            g.handle, s.handle, sigma2, channel_seed, frame_begin, frames, max_iters, int(early_stop), _vp(be),
            _vp(it), _vp(cv), None, _stream(stream),
        ),
        "simulate_frames",
    )
    return be, it, cv


def run_sweep_native(g, s, ebn0_db, iter_limit: int, max_frames: int, min_frame_errors: int, channel_seed: int = 1,
                     wave_frames: int = 0) -> list[dict]:
    """run_sweep (sim.hpp:96-186) on the current GPU through ldpcb_run_sweep_host:
    one SimResult dict per Eb/N0 point."""
    pts = np.ascontiguousarray(list(ebn0_db), np.float64)
    out = np.zeros((len(pts), 11), np.float64)
    check(lib.ldpcb_run_sweep_host(g.handle, s.handle, _vp(pts), len(pts), iter_limit, max_frames, min_frame_errors,
                                   channel_seed, wave_frames, _vp(out)), "run_sweep")
    keys = ("frames", "bit_errors", "frame_errors", "converged_frames", "ber", "fer", "mean_iters_converged",
            "mean_iters_all", "iter_limit", "wall_seconds", "ebn0_db")
    ints = {"frames", "bit_errors", "frame_errors", "converged_frames", "iter_limit"}
    return [{k: (int(v) if k in ints else float(v)) for k, v in zip(keys, row)} for row in out]


def _sweep_records(out) -> list[dict]:
    keys = ("frames", "bit_errors", "frame_errors", "converged_frames", "ber", "fer", "mean_iters_converged",
            "mean_iters_all", "iter_limit", "wall_seconds", "ebn0_db")
    ints = {"frames", "bit_errors", "frame_errors", "converged_frames", "iter_limit"}
    return [{k: (int(v) if k in ints else float(v)) for k, v in zip(keys, row)} for row in out]


def simulate_multi(g, s, devices, sigma2: float, channel_seed: int, frame_begin: int, frames: int, max_iters: int,
                   early_stop: bool = True) -> np.ndarray:
    """ldpcb_simulate_multi: frames [frame_begin, frame_begin+frames) split in
    contiguous ranges over `devices` (one host thread per entry, a device may
    repeat); returns the summed int64[6] counters (host)."""
    dev = np.ascontiguousarray(list(devices), np.int32)
    cnt = np.zeros(6, np.int64)
    check(lib.ldpcb_simulate_multi(g.handle, s.handle, _vp(dev), len(dev), sigma2, channel_seed, frame_begin, frames,
                                   max_iters, int(early_stop), _vp(cnt)), "simulate_multi")
    return cnt


def run_sweep_multi(g, s, devices, ebn0_db, iter_limit: int, max_frames: int, min_frame_errors: int,
                    channel_seed: int = 1, wave_frames: int = 0) -> list[dict]:
    """run_sweep (sim.hpp:96-186) over several GPUs through ldpcb_run_sweep_multi."""
    dev = np.ascontiguousarray(list(devices), np.int32)
    pts = np.ascontiguousarray(list(ebn0_db), np.float64)
    out = np.zeros((len(pts), 11), np.float64)
    check(lib.ldpcb_run_sweep_multi(g.handle, s.handle, _vp(dev), len(dev), _vp(pts), len(pts), iter_limit,
                                    max_frames, min_frame_errors, channel_seed, wave_frames, _vp(out)),
          "run_sweep_multi")
    return _sweep_records(out)


@dataclass
class DecodeOutcome:
    """decoder.hpp:31-37."""

    bits: np.ndarray
    converged: bool
    iterations: int
    syndrome_weight_trace: list = field(default_factory=list)
    cn_updates: int = 0


def decode(g: TannerGraph, s: GroupSchedule, channel_llr, max_iters: int) -> DecodeOutcome:
    """Single-frame decode() with the reference's signature and outcome."""
    torch = _torch()
    if max_iters < 1:
        raise ValueError("max_iters must be >= 1")
    x = torch.as_tensor(np.asarray(channel_llr, dtype=np.float32)).reshape(1, -1)
    if x.shape[1] != g.n_vars:
        raise ValueError("channel LLR length does not match the code length")
    r = decode_batch(g, s, x.cuda(), max_iters, early_stop=True, trace=True)
    it = int(r["iterations"][0])
    tr = [int(v) for v in r["syndrome_trace"][0, :it].tolist()]
    return DecodeOutcome(
        bits=r["bits"][0].cpu().numpy(),
        converged=bool(r["converged"][0]),
        iterations=it,
        syndrome_weight_trace=tr,
        cn_updates=it * s.n_slots,
    )


def check_update(v2c):
    """check_update (decoder.hpp:59-87) per row of a [rows, degree] CUDA tensor."""
    torch = _torch()
    v2c = v2c.contiguous().to(torch.float32)
    rows, deg = v2c.shape
    c2v = torch.empty_like(v2c)
    check(lib.ldpcb_check_update_device(deg, rows, _vp(v2c), _vp(c2v), _stream()), "check_update")
    return c2v


def run_subiterations(g: TannerGraph, s: GroupSchedule, llr, n_subiters: int):
    """init_state + n_subiters sub-iterations; returns (c2v, v2c) [frames, E]."""
    torch = _torch()
    F = llr.shape[0]
    c2v = torch.empty((F, g.n_edges), dtype=torch.float32, device=llr.device)
    v2c = torch.empty_like(c2v)
    check(
        lib.ldpcb_run_subiterations_device(g.handle, s.handle, F, _vp(llr), n_subiters, _vp(c2v), _vp(v2c), _stream()),
        "run_subiterations",
    )
    return c2v, v2c


def plan(g: TannerGraph, s: GroupSchedule, frames: int) -> dict:
    vals = [C.c_int32() for _ in range(5)]
    check(lib.ldpcb_decode_plan(g.handle, s.handle, frames, *vals))
    return dict(zip(("kernel", "frames_per_cta", "threads", "smem_bytes", "degree_bucket"), (v.value for v in vals)))


def set_tuning(frames_per_cta: int = 0, threads: int = 0, frames_per_thread: int = 0) -> None:
    """Resident-kernel launch shape; 0 = automatic."""
    check(lib.ldpcb_set_tuning(frames_per_cta, threads))
    check(lib.ldpcb_set_frames_per_thread(frames_per_thread))


def set_kernel(kernel: int = 0) -> None:
    """0 automatic, 1 shared-memory resident (posterior-based kernel) only,
    2 HBM-streamed, 3 posterior-free resident kernel (direct.cu)."""
    check(lib.ldpcb_set_kernel(kernel))


def set_lazy_totals(on: bool) -> None:
    check(lib.ldpcb_set_lazy_totals(int(on)))


def kernel_launches() -> int:
    return int(lib.ldpcb_kernel_launches())
