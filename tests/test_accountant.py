"""Privacy bookkeeping on the host, no GPU needed:

* NoiseSchedule / schedule_noise against the reference's own NoiseSchedule (optimizer.hpp:280-358,
  compiled from /root/reference into oracle/_ref by oracle/Makefile) on the same factories and
  epochs, bit for bit, and its ParameterError texts;
* the RDP accountant against the known-answer tests and properties of SPEC.md:331-389 (the
  reference specifies it but ships no implementation), with an exact rational-arithmetic oracle
  for the binomial sum.
"""
import ctypes
import math

import numpy as np
import pytest

import oracle
from paper_2109_12298_b200 import dpg


def _ref_sigmas(kind, sigma0=1.0, gamma=1.0, factor=1.0, period=1, table=None, epochs=range(12)):
    ref = oracle.reference()
    ep = np.array(list(epochs), dtype=np.uint64)
    out = np.empty(len(ep), dtype=np.float64)
    tab = np.array(table if table is not None else [0.0], dtype=np.float64)
    f = ref.lib.dpgref_schedule_sigmas
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_uint64, ctypes.c_void_p,
                  ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
    rc = f(kind, sigma0, gamma, factor, period, tab.ctypes.data, len(tab), ep.ctypes.data, len(ep), out.ctypes.data)
    return rc, out, ref.lib.dpgref_last_error().decode() if rc else ""


CASES = [
    (dpg.NoiseSchedule.CONSTANT, dict(sigma0=1.3)),
    (dpg.NoiseSchedule.EXPONENTIAL, dict(sigma0=2.0, gamma=0.93)),
    (dpg.NoiseSchedule.STEP, dict(sigma0=1.5, factor=0.5, period=3)),
    (dpg.NoiseSchedule.CUSTOM, dict(table=[1.0, 0.9, 0.7])),
]


@pytest.mark.parametrize("kind,kw", CASES)
def test_schedule_matches_reference(kind, kw):
    if not oracle.reference_available():
        pytest.skip("oracle/_ref not built")
    s = dpg.NoiseSchedule(kind, **kw)
    rc, ref, _ = _ref_sigmas(kind, **kw)
    assert rc == 0
    got = np.array([s.schedule_noise(e) for e in range(12)])
    np.testing.assert_array_equal(got, ref)
    assert s.current == ref[-1]


@pytest.mark.parametrize("kind,kw,msg", [
    (dpg.NoiseSchedule.CONSTANT, dict(sigma0=-1.0), "schedule sigma must be >= 0"),
    (dpg.NoiseSchedule.EXPONENTIAL, dict(sigma0=1.0, gamma=-0.1), "exponential schedule needs gamma >= 0"),
    (dpg.NoiseSchedule.STEP, dict(sigma0=1.0, factor=-1.0, period=2), "step schedule needs factor >= 0"),
    (dpg.NoiseSchedule.STEP, dict(sigma0=1.0, factor=0.5, period=0), "step schedule needs period >= 1"),
    (dpg.NoiseSchedule.CUSTOM, dict(table=[1.0, -0.5]), "schedule sigma must be >= 0"),
])
def test_schedule_errors_match_reference(kind, kw, msg):
    with pytest.raises(dpg.ParameterError, match=msg):
        dpg.NoiseSchedule(kind, **kw)
    if oracle.reference_available():
        rc, _, err = _ref_sigmas(kind, **kw)
        assert rc == 2 and err == msg


def _rdp_exact(q, sigma, alpha):
    """(1/(a-1)) ln sum_k C(a,k)(1-q)^(a-k) q^k exp((k^2-k)/(2 s^2)) by direct summation in
    60-digit decimal arithmetic (SPEC.md:349 'high-precision summation oracle')."""
    from decimal import Decimal, getcontext
    getcontext().prec = 60
    qd, sd = Decimal(q), Decimal(sigma)
    tot = Decimal(0)
    for k in range(alpha + 1):
        w = Decimal(math.comb(alpha, k)) * (1 - qd) ** (alpha - k) * qd ** k
        tot += w * (Decimal(k * k - k) / (2 * sd * sd)).exp()
    return float(tot.ln() / (alpha - 1))


def test_rdp_known_answers():
    assert dpg.rdp_subsampled_gaussian(1.0, 2.0, 7) == pytest.approx(7 / (2 * 4.0), rel=1e-15)
    assert dpg.rdp_subsampled_gaussian(0.0, 1.0, 5) == 0.0
    v = dpg.rdp_subsampled_gaussian(0.01, 1.0, 2)
    assert v == pytest.approx(math.log(0.9801 + 0.0198 + 0.0001 * math.e), rel=1e-12)
    assert v == pytest.approx(1.718e-4, rel=1e-3)
    for q, s, a in [(0.002, 1.1, 2), (0.01, 0.8, 8), (0.05, 1.5, 32), (0.03, 0.3, 12)]:
        assert dpg.rdp_subsampled_gaussian(q, s, a) == pytest.approx(_rdp_exact(q, s, a), rel=1e-9)
    with pytest.raises(dpg.ParameterError):
        dpg.rdp_subsampled_gaussian(0.1, 0.0, 2)
    with pytest.raises(dpg.ParameterError):
        dpg.rdp_subsampled_gaussian(1.5, 1.0, 2)


def test_accountant_composition_and_conversion():
    a = dpg.RdpAccountant()
    orders, curve = a.rdp()
    assert orders[:3] == [2, 3, 4] and orders[-2:] == [128, 256] and all(c == 0 for c in curve)
    eps, best = a.epsilon(1e-5)  # zero curve: ln(1/delta)/(a_max - 1) at the largest order
    assert best == 256 and eps == pytest.approx(math.log(1e5) / 255)
    one = dpg.RdpAccountant([2])
    one.step(1.0, 0.01, 1)
    r = one.rdp()[1][0]
    assert one.epsilon(1e-5)[0] == pytest.approx(r + math.log(1e5))
    # T identical steps = T x one step; heterogeneous history = per-step sum; order independence
    b = dpg.RdpAccountant()
    b.step(1.1, 0.004, 1000)
    c = dpg.RdpAccountant()
    for _ in range(10):
        c.step(1.1, 0.004, 100)
    np.testing.assert_allclose(b.rdp()[1], c.rdp()[1], rtol=1e-12)
    h1, h2 = dpg.RdpAccountant(), dpg.RdpAccountant()
    hist = [(1.0, 0.01, 50), (0.8, 0.02, 20), (1.3, 0.005, 300)]
    for rec in hist:
        h1.step(*rec)
    for rec in reversed(hist):
        h2.step(*rec)
    o1, c1 = h1.rdp()
    _, c2 = h2.rdp()
    np.testing.assert_allclose(c1, c2, rtol=1e-14)
    brute = [sum(n * _rdp_exact(q, s, al) for (s, q, n) in hist) for al in o1[:20]]
    np.testing.assert_allclose(c1[:20], brute, rtol=1e-9)
    # delta monotonicity
    assert h1.epsilon(1e-6)[0] >= h1.epsilon(1e-5)[0]


def test_epsilon_monotone_properties():
    def eps(sigma, q, steps):
        a = dpg.RdpAccountant()
        a.step(sigma, q, steps)
        return a.epsilon(1e-5)[0]
    assert eps(1.0, 0.01, 100) <= eps(1.0, 0.01, 200)
    assert eps(1.2, 0.01, 100) <= eps(1.0, 0.01, 100)
    assert eps(1.0, 0.01, 100) <= eps(1.0, 0.02, 100)


def test_noise_calibration_self_consistent():
    q, steps, delta, target = 1 / 500, 5000, 1e-5, 2.0
    s = dpg.get_noise_multiplier(target, delta, q, steps)

    def eps(sigma):
        a = dpg.RdpAccountant()
        a.step(sigma, q, steps)
        return a.epsilon(delta)[0]
    assert eps(s) <= target < eps(s - 1e-3)
    assert dpg.get_noise_multiplier(target, delta, q, 2 * steps) >= s  # more steps never need less noise
    assert dpg.get_noise_multiplier(1e9, delta, q, steps) == 0.01       # huge budget: the bracket's lower end
    with pytest.raises(dpg.ParameterError, match="infeasible"):
        dpg.get_noise_multiplier(1e-4, delta, 0.5, 10 ** 6)


def test_schedule_drives_the_optimizer_sigma():
    """schedule_noise with an optimizer applies sigma through dpg_set_noise_multiplier (host-side
    state only: no step is run, so this needs no GPU)."""
    s = dpg.NoiseSchedule.step(2.0, 0.5, 2)
    assert [s.schedule_noise(e) for e in (0, 1, 2, 5)] == [2.0, 2.0, 1.0, 0.5]
