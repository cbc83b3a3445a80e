"""B200-native batched group-shuffled LDPC decoder (arxiv/paper_1202_1060 hot path).

The compute path is libldpc_b200.so (sm_100a CUDA kernels behind the C ABI in
include/ldpc_b200.h); this package is its host-side mirror of the reference's
decoder interface. Importing fails loudly when the library is not built.
"""
from .api import (  # noqa: F401
    COUNTER_NAMES,
    DISJOINT,
    FLOODING,
    KIND_NAMES,
    NONDISJOINT,
    AlistError,
    DecodeOutcome,
    GroupSchedule,
    TannerGraph,
    check_update,
    decode,
    decode_batch,
    decode_host,
    kernel_launches,
    make_disjoint_schedule,
    make_flooding_schedule,
    make_nondisjoint_schedule,
    plan,
    run_subiterations,
    set_kernel,
    set_lazy_totals,
    set_tuning,
    sigma2_from_ebn0,
    run_sweep_multi,
    run_sweep_native,
    simulate,
    simulate_multi,
    simulate_frames,
    transmit_all_zero,
)
from . import configs  # noqa: F401
