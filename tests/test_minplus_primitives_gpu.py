"""The reference's min-plus primitives on plain sequences (proj/include/laxol/minplus.hpp:
conv_naive, decompose, conv_fast incl. eta > 0) on the device against the reference itself,
plus its known answers (proj/tests/unit_minplus.cpp:102-116,203-227,274-335)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _t(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()


def _naive(dev, f, g):
    import torch

    out = torch.empty(len(f) + len(g) - 1, dtype=torch.float64, device="cuda")
    dev.conv_naive(_t(f), _t(g), out)
    return out.cpu().numpy()


def _fast(dev, k, u, eta):
    import torch

    out = torch.empty(len(k) + len(u) - 1, dtype=torch.float64, device="cuda")
    b = dev.conv_fast(_t(k), _t(u), out, eta)
    return out.cpu().numpy(), b


def test_known_answers(dev):
    assert np.array_equal(_naive(dev, [0, 1, 4], [0, 2]), [0, 1, 3, 6])
    assert np.array_equal(_fast(dev, [0, 1, 4], [0, 2], 0.0)[0], [0, 1, 3, 6])
    assert np.array_equal(_fast(dev, [4, 1, 0, 1, 4], [0, -1], 0.0)[0], [4, 1, 0, -1, 0, 3])
    assert np.array_equal(_fast(dev, [4, 1, 0, 1, 4], [0, 2, 2, 0], 0.0)[0], [4, 1, 0, 1, 1, 0, 1, 4])
    x = np.arange(17) / 16.0
    kinds, starts, ends = dev.decompose(_t(np.cos(2 * np.pi * x)))
    assert list(kinds) == [1, 0, 1]  # concave, convex, concave (unit_minplus.cpp:274-293)


@pytest.mark.parametrize("nf,ng,seed", [(1, 1, 0), (5, 9, 1), (200, 37, 2), (513, 1024, 3)])
def test_conv_naive_equals_reference(dev, ref, nf, ng, seed):
    rng = np.random.default_rng(seed)
    f = rng.integers(-4, 5, nf) * 0.5  # tie-heavy
    g = rng.uniform(-1, 1, ng)
    want, _, st = ref.conv(0, f, g)
    assert st == 0 and np.array_equal(_naive(dev, f, g), want)


@pytest.mark.parametrize("eta", [0.0, 1e-6, 1e-3, 1e-1])
@pytest.mark.parametrize("m,seed", [(2, 0), (30, 1), (333, 2), (2000, 3)])
def test_decompose_and_conv_fast_equal_reference(dev, ref, eta, m, seed):
    rng = np.random.default_rng(seed)
    u = np.cumsum(rng.uniform(-1, 1, m)) * 0.1 + 0.01 * np.sin(np.arange(m) * 0.3)
    c, kinds, starts, ends = ref.decompose(u, eta)
    gk, gs, ge = dev.decompose(_t(u), eta)
    assert len(gk) == c and np.array_equal(gk, kinds) and np.array_equal(gs, starts) and np.array_equal(ge, ends)
    v = np.linspace(-3, 3, 121)
    kern = 0.5 * v * v - 0.2 * v
    want, wb, st = ref.conv(3, kern, u, eta)
    assert st == 0
    got, gb = _fast(dev, kern, u, eta)
    assert np.array_equal(got, want) and gb == wb
