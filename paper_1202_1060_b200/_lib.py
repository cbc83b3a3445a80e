"""ctypes binding of the C ABI in include/ldpc_b200.h (libldpc_b200.so).

The shared library is the product: there is no Python or CPU fallback. If the
library is missing this module raises ImportError immediately.
"""
from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LDPCB_LIBRARY") or os.path.join(_HERE, "libldpc_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "ldpc_b200.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the sm_100a library first "
        "(python -c 'import __graft_entry__ as g; g.build()')"
    )

lib = C.CDLL(LIB_PATH)

i32, i64, u64, dbl = C.c_int32, C.c_int64, C.c_uint64, C.c_double
vp, cp = C.c_void_p, C.c_char_p
P32, P64 = C.POINTER(C.c_int32), C.POINTER(C.c_int64)
PD = C.POINTER(C.c_double)
PI = C.POINTER(C.c_int)

OK, EINVAL, ERUNTIME, EALIST, ECUDA, EUNSUPPORTED = 0, -1, -2, -3, -4, -5

_SIGS = {
    "ldpcb_last_error": (cp, []),
    "ldpcb_abi_version": (C.c_int, []),
    "ldpcb_code_from_check_lists": (C.c_int, [C.c_int, C.c_int, vp, vp, C.POINTER(vp)]),
    "ldpcb_code_random_regular": (C.c_int, [C.c_int, C.c_int, C.c_int, u64, C.POINTER(vp)]),
    "ldpcb_code_random_regular_girth6": (C.c_int, [C.c_int, C.c_int, C.c_int, u64, C.POINTER(vp)]),
    "ldpcb_code_qc": (C.c_int, [C.c_int, C.c_int, C.c_int, dbl, C.c_int, u64, C.POINTER(vp)]),
    "ldpcb_code_irregular": (C.c_int, [C.c_int, C.c_int, vp, vp, C.c_int, u64, C.POINTER(vp)]),
    "ldpcb_code_parse_alist": (C.c_int, [cp, C.POINTER(vp), PI, PI]),
    "ldpcb_code_serialize_alist": (C.c_int, [vp, C.c_char_p, i64, P64]),
    "ldpcb_code_dims": (C.c_int, [vp, P32, P32, P32, P32, P32]),
    "ldpcb_code_export": (C.c_int, [vp, vp, vp, vp, vp, vp]),
    "ldpcb_code_count_4cycles": (C.c_int, [vp, P64]),
    "ldpcb_code_destroy": (None, [vp]),
    "ldpcb_schedule_from_groups": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, C.POINTER(vp)]),
    "ldpcb_schedule_flooding": (C.c_int, [vp, C.POINTER(vp)]),
    "ldpcb_schedule_disjoint": (C.c_int, [vp, C.c_int, u64, C.POINTER(vp)]),
    "ldpcb_schedule_nondisjoint": (C.c_int, [vp, C.c_int, dbl, u64, C.POINTER(vp)]),
    "ldpcb_schedule_windows": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
    "ldpcb_simulate_frames_device": (C.c_int, [vp, vp, dbl, u64, i64, i64, C.c_int, C.c_int, vp, vp, vp, vp, vp]),
    "ldpcb_run_sweep_host": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, i64, C.c_int, u64, i64, vp]),
    "ldpcb_schedule_per_frame": (C.c_int, [vp, C.c_int, C.c_int, dbl, u64, C.c_int, C.POINTER(vp)]),
    "ldpcb_schedule_per_frame_groups_device": (C.c_int, [vp, vp, i64, i64, C.c_int, vp, vp]),
    "ldpcb_schedule_dims": (C.c_int, [vp, P32, P32, P32, P32, PD, P64, P64]),
    "ldpcb_schedule_export": (C.c_int, [vp, vp, vp]),
    "ldpcb_schedule_iteration_budget": (C.c_int, [vp, C.c_int, P32]),
    "ldpcb_schedule_direct_layout": (C.c_int, [vp, P32, P32, P32, P32, P32, PD]),
    "ldpcb_schedule_direct_export": (C.c_int, [vp, vp, vp, vp, vp, vp, vp]),
    "ldpcb_schedule_cocsg": (C.c_int, [vp, vp]),
    "ldpcb_schedule_destroy": (None, [vp]),
    "ldpcb_sigma2_from_ebn0": (C.c_int, [dbl, dbl, PD]),
    "ldpcb_channel_llr_device": (C.c_int, [C.c_int, dbl, u64, i64, i64, vp, vp]),
    "ldpcb_decode_device": (
        C.c_int,
        [vp, vp, i64, vp, C.c_int, C.c_int, vp, C.c_int, vp, vp, vp, vp, vp, vp],
    ),
    "ldpcb_decode_host": (
        C.c_int,
        [vp, vp, i64, vp, C.c_int, C.c_int, vp, C.c_int, vp, vp, vp, vp, vp],
    ),
    "ldpcb_simulate_host": (C.c_int, [vp, vp, dbl, u64, i64, i64, C.c_int, C.c_int, vp]),
    "ldpcb_simulate_multi": (C.c_int, [vp, vp, vp, C.c_int, dbl, u64, i64, i64, C.c_int, C.c_int, vp]),
    "ldpcb_run_sweep_multi": (C.c_int, [vp, vp, vp, C.c_int, vp, C.c_int, C.c_int, i64, C.c_int, u64, i64, vp]),
    "ldpcb_simulate_device": (C.c_int, [vp, vp, dbl, u64, i64, i64, C.c_int, C.c_int, vp, vp]),
    "ldpcb_check_update_device": (C.c_int, [C.c_int, i64, vp, vp, vp]),
    "ldpcb_run_subiterations_device": (C.c_int, [vp, vp, i64, vp, C.c_int, vp, vp, vp]),
    "ldpcb_decode_plan": (C.c_int, [vp, vp, i64, P32, P32, P32, P32, P32]),
    "ldpcb_set_tuning": (C.c_int, [C.c_int, C.c_int]),
    "ldpcb_kernel_launches": (i64, []),
    "ldpcb_set_lazy_totals": (C.c_int, [C.c_int]),
    "ldpcb_set_kernel": (C.c_int, [C.c_int]),
    "ldpcb_set_frames_per_thread": (C.c_int, [C.c_int]),
}

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


class AlistError(RuntimeError):
    """Mirror of ldpc::AlistError (tanner.hpp:61-73): .kind and 1-based .line."""

    KINDS = (
        "malformed_header",
        "bad_token",
        "degree_error",
        "length_mismatch",
        "index_out_of_range",
        "duplicate_entry",
        "edge_count_mismatch",
        "transpose_mismatch",
        "trailing_content",
        "truncated",
    )

    def __init__(self, msg: str, kind: int, line: int):
        super().__init__(msg)
        self.kind = self.KINDS[kind] if 0 <= kind < len(self.KINDS) else str(kind)
        self.line = line


def check(status: int, what: str = "") -> None:
    """Map a C status to the reference's exception types."""
    if status == OK:
        return
    msg = (lib.ldpcb_last_error() or b"").decode()
    if what:
        msg = f"{what}: {msg}"
    if status == EINVAL:
        raise ValueError(msg)  # std::invalid_argument in the reference
    raise RuntimeError(msg)


def header_functions(path: str = HEADER_PATH) -> list[str]:
    """Every function declared in include/ldpc_b200.h."""
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ldpcb_[a-z0-9_]+)\s*\(", text)))
