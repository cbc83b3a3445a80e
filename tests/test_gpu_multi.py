"""Several GPUs of one process through the C ABI (ldpcb_simulate_multi,
ldpcb_run_sweep_multi): one host thread per listed device, contiguous
frame-id ranges, host-summed counters. The box has one GPU, so device 0 is
listed several times (independent workers on one GPU); frames are keyed by
id, so the results must equal the one-device results exactly."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0]])
@pytest.mark.parametrize("es", [True, False])
def test_simulate_multi_equals_one_device(P, torch, devices, es):
    g = P.configs.c1_code()
    s = P.configs.c1_schedules(g)["ndgsbp"]
    s2 = P.sigma2_from_ebn0(1.75, g.rate)
    one = P.simulate(g, s, s2, 5, 123, 20_001, 20, early_stop=es).cpu().numpy()
    many = P.simulate_multi(g, s, devices, s2, 5, 123, 20_001, 20, early_stop=es)
    assert np.array_equal(one, many), (one, many)


def test_simulate_multi_streamed_code(P, torch):
    """The HBM-streamed path (C4 code) under two workers."""
    g = P.configs.c4_code()
    s = P.configs.c4_schedules(g)["ndgsbp"]
    s2 = P.sigma2_from_ebn0(1.1, g.rate)
    one = P.simulate(g, s, s2, 1, 0, 96, 10, early_stop=False).cpu().numpy()
    many = P.simulate_multi(g, s, [0, 0], s2, 1, 0, 96, 10, early_stop=False)
    assert np.array_equal(one, many)


def test_run_sweep_multi_equals_one_device(P, torch):
    g = P.configs.c1_code()
    pf = P.GroupSchedule.per_frame(g, P.NONDISJOINT, 8, 0.25, 2, True)
    one = P.run_sweep_native(g, pf, [1.5, 2.0], 20, 100_000, 40, wave_frames=3000)
    for devices, wave in (([0, 0], 3000), ([0, 0, 0], 0)):
        many = P.run_sweep_multi(g, pf, devices, [1.5, 2.0], 20, 100_000, 40, wave_frames=wave)
        for a, b in zip(one, many):
            for k in ("frames", "bit_errors", "frame_errors", "converged_frames", "ber", "fer",
                      "mean_iters_converged", "mean_iters_all", "iter_limit", "ebn0_db"):
                assert a[k] == b[k], (devices, k, a[k], b[k])


def test_multi_rejects_bad_device_lists(P, torch):
    g = P.configs.c1_code()
    s = P.configs.c1_schedules(g)["ndgsbp"]
    with pytest.raises(ValueError):
        P.simulate_multi(g, s, [], 1.0, 1, 0, 10, 5)
    with pytest.raises(ValueError):
        P.simulate_multi(g, s, [0, 4096], 1.0, 1, 0, 10, 5)
