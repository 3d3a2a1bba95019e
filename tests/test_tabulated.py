"""Tabulated kinetic conjugates (proj/src/hamiltonian.cpp:30-82 `tabulated`, kstar by linear
interpolation, argmin velocity; proj/src/scheme.cpp:59-105 build_kernel with its monotone slope
repair) against the reference itself: the host window `==`, and the device engines that take
any table — K1 direct and the relaxed fast engine — `==` the reference's kinetic_convolve."""
import numpy as np
import pytest

from paper_1210_4090_b200 import api
from paper_1210_4090_b200._capi import InvalidInput

TABLES = {
    # name: (samples as a function of the velocity grid, v0, dv, count)
    "quadratic": (lambda v: 0.5 * v * v - 0.3 * v, -30.0, 0.25, 241),
    "pow15": (lambda v: np.abs(v) ** 1.5, -25.0, 0.5, 101),
    "flat_bottom": (lambda v: np.maximum(np.abs(v) - 2.0, 0.0) ** 2, -40.0, 1.0, 81),
    "piecewise": (lambda v: np.maximum(np.maximum(-v, 0.5 * v), 0.25 * v + 1.0), -50.0, 2.5, 41),
}


def table(name):
    f, v0, dv, count = TABLES[name]
    v = v0 + np.arange(count) * dv
    return f(v), v0, dv


@pytest.mark.parametrize("name", list(TABLES))
@pytest.mark.parametrize("n,tau", [(16, 0.25), (64, 0.05), (256, 0.02)])
def test_tabulated_kernel_equals_reference(ref, name, n, tau):
    s, v0, dv = table(name)
    want, first, arg, st = ref.kernel_tabulated(n, tau, s, v0, dv)
    if st != 0:
        with pytest.raises(InvalidInput):
            api.Device.build_kernel_tabulated(n, tau, s, v0, dv)
        return
    k = api.Device.build_kernel_tabulated(n, tau, s, v0, dv)
    assert np.array_equal(k.window, want)
    assert k.first == first and k.argmin_index == arg


def test_tabulated_rejects_what_the_reference_rejects(ref):
    s, v0, dv = table("quadratic")
    # window wider than the table (proj/src/scheme.cpp:69-74)
    assert ref.kernel_tabulated(64, 0.005, s, v0, dv)[3] == 1
    with pytest.raises(InvalidInput):
        api.Device.build_kernel_tabulated(64, 0.005, s, v0, dv)
    bad = s.copy()
    bad[10] += 1.0  # not convex
    assert ref.kernel_tabulated(64, 0.05, bad, v0, dv)[3] == 1
    with pytest.raises(InvalidInput):
        api.Device.build_kernel_tabulated(64, 0.05, bad, v0, dv)


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(TABLES))
@pytest.mark.parametrize("eta", [0.0, 1e-4])
@pytest.mark.parametrize("n,tau", [(64, 0.05), (128, 0.25), (256, 0.1)])
def test_tabulated_convolve_on_device_equals_reference(dev, ref, name, eta, n, tau):
    import torch

    s, v0, dv = table(name)
    if ref.kernel_tabulated(n, tau, s, v0, dv)[3] != 0:  # the reference rejects this window too
        with pytest.raises(InvalidInput):
            api.Device.build_kernel_tabulated(n, tau, s, v0, dv)
        return
    k = api.Device.build_kernel_tabulated(n, tau, s, v0, dv)
    rng = np.random.default_rng(len(name))
    u = rng.uniform(-0.05, 0.05, (3, n)).cumsum(axis=1)
    u -= np.linspace(0, 1, n)[None, :] * u[:, -1:]
    du = torch.from_numpy(u).cuda()
    out = torch.empty_like(du)
    kt = torch.from_numpy(k.window).cuda()
    fr = torch.full((3,), k.first, dtype=torch.int64, device="cuda")
    if eta == 0.0:
        dev.direct_f64(du, out, kt, fr)
        got = out.cpu().numpy()
        for l in range(3):
            want, _, st = ref.convolve_tabulated(u[l], tau, s, v0, dv, 0.0, engine=1)
            assert st == 0 and np.array_equal(got[l], want)
    bl = torch.empty(3, dtype=torch.int64, device="cuda")
    dev.relaxed_f64(du, out, kt, fr, eta, blocks=bl)
    got = out.cpu().numpy()
    for l in range(3):
        want, wb, st = ref.convolve_tabulated(u[l], tau, s, v0, dv, eta, engine=0)
        assert st == 0 and np.array_equal(got[l], want)
        assert bl[l].item() == wb
