"""The reference's own decoder unit pins (proj/tests/test_decoder.cpp) run
through the sm_100a path and the C ABI: init_state, empty groups, noiseless
input, a saturated codeword fixed point, determinism with per-iteration
regrouping. Messages come back in nats from log2-unit fp32 state, so
equalities the reference checks exactly are checked to fp32 rounding
(relative 1e-6) unless the value is exactly representable through the
round trip (zeros, untouched messages)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIG1 = [[0, 1, 2], [1, 3, 4], [3, 5, 6], [5, 7]]  # test_decoder.cpp:17-19


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def cu(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def state_after_empty_group(P, torch, llr):
    """init_state, then one sub-iteration over an empty group (decoder.hpp:39-52, 112-127)."""
    g = P.TannerGraph.from_check_lists(8, FIG1)
    s = P.GroupSchedule.from_groups(g, P.NONDISJOINT, [[], [0, 1, 2, 3]])
    c2v, v2c = (t.cpu().numpy()[0] for t in P.run_subiterations(g, s, cu(torch, [llr]), 1))
    return g, c2v, v2c


def test_init_state_zero_input(P, torch):
    # test_decoder.cpp:30-34
    _, c2v, v2c = state_after_empty_group(P, torch, [0.0] * 8)
    assert np.all(c2v == 0.0) and np.all(v2c == 0.0)


def test_init_state_huge_inputs_saturate(P, torch):
    # test_decoder.cpp:35-38: 1e12 -> the clamp, 30
    _, c2v, v2c = state_after_empty_group(P, torch, [1e12] * 8)
    assert np.all(c2v == 0.0)
    assert np.allclose(v2c, 30.0, rtol=1e-6, atol=0)


def test_init_state_edges_carry_their_vn_value(P, torch):
    # test_decoder.cpp:39-46: eleven edges, each carrying its VN's LLR
    llr = [0.25 * (n + 1) for n in range(8)]
    g, _, v2c = state_after_empty_group(P, torch, llr)
    assert v2c.shape == (11,)
    for n in range(8):
        for e in g.var_edge_ids[n]:
            assert v2c[e] == pytest.approx(llr[n], rel=1e-6)


def test_empty_group_leaves_state_unchanged(P, torch):
    # test_decoder.cpp:104-112: zero sub-iterations' worth of change
    llr = [0.3, -0.2, 1.0, -1.5, 0.7, 0.1, -0.4, 0.9]
    g, c2v, v2c = state_after_empty_group(P, torch, llr)
    assert np.all(c2v == 0.0)
    for n in range(8):
        for e in g.var_edge_ids[n]:
            assert v2c[e] == pytest.approx(llr[n], rel=1e-6)


def test_init_state_length_mismatch_raises(P, torch):
    # test_decoder.cpp:47-49 (std::invalid_argument -> ValueError)
    g = P.TannerGraph.from_check_lists(8, FIG1)
    with pytest.raises(ValueError):
        P.decode(g, P.make_flooding_schedule(g), [0.0] * 7, 5)


def test_noiseless_input_converges_in_one_iteration(P, torch):
    # test_decoder.cpp:149-156
    g = P.TannerGraph.random_regular(60, 3, 6, 21)
    out = P.decode(g, P.make_flooding_schedule(g), [1e9] * g.n_vars, 10)
    assert out.converged and out.iterations == 1
    assert not out.bits.any()


@pytest.mark.parametrize("kind", ["flooding", "groups"])
def test_saturated_codeword_is_a_fixed_point(P, torch, kind):
    # test_decoder.cpp:158-168 (and the same word under a two-group schedule)
    g = P.TannerGraph.from_check_lists(8, FIG1)
    word = np.array([1, 1, 0, 1, 0, 1, 0, 1], np.uint8)
    llr = np.where(word == 1, -30.0, 30.0)
    s = (P.make_flooding_schedule(g) if kind == "flooding"
         else P.GroupSchedule.from_groups(g, P.NONDISJOINT, [[0, 1], [1, 2, 3]]))
    out = P.decode(g, s, llr, 5)
    assert out.converged and out.iterations == 1
    assert np.array_equal(out.bits, word)
    assert out.syndrome_weight_trace == [0]


def test_determinism_with_per_iteration_regrouping(P, torch):
    # test_decoder.cpp:267-277: identical reruns, groups redrawn every iteration
    g = P.configs.c1_code()
    s = P.GroupSchedule.per_frame(g, P.NONDISJOINT, 8, 0.25, 7, True)
    x = P.transmit_all_zero(g.n_vars, P.sigma2_from_ebn0(1.5, g.rate), 3, 0, 300)
    a = P.decode_batch(g, s, x, 20, posterior=True, trace=True)
    b = P.decode_batch(g, s, x, 20, posterior=True, trace=True)
    for k in a:
        assert torch.equal(a[k], b[k]), k
