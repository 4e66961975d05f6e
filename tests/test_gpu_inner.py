"""GPU sum-space inner product / norm (kernels.py:209-252; SURVEY 8(f) row 4,
the Fejer-monotonicity diagnostics), mirroring the reference's
tests/test_kernels.py:186-248 and test_acceptance.py:150-181."""

import numpy as np
import pytest
from numpy.testing import assert_allclose

import paper_2201_05024_b200 as K
from oracle import kapsm_oracle as O

pytestmark = pytest.mark.gpu
P_HALF = K.KernelParams(0.5, 0.5, 0.05)


def kernel_sum(u, v, p):
    return p.w_l * float(u @ v) + p.w_g * float(np.exp(-np.sum((u - v) ** 2) / (2 * p.sigma_sq)))


def random_expansion(rng, n, dim, p):
    g = rng.standard_normal(n)
    a = rng.standard_normal((n, dim)) * 0.3
    return g, a, K.from_expansion(g, a, p)


def oracle_inner(gf, af, gg, ag, p):
    return float(sum(gf[i] * gg[j] * kernel_sum(af[i], ag[j], p)
                     for i in range(len(gf)) for j in range(len(gg))))


def test_reproducing_property():
    rng = np.random.default_rng(3)
    for _ in range(20):
        u, v = rng.standard_normal(6) * 0.5, rng.standard_normal(6) * 0.5
        fu = K.from_expansion([1.0], [u], P_HALF)
        fv = K.from_expansion([1.0], [v], P_HALF)
        assert_allclose(K.inner_product(fu, fv, P_HALF), kernel_sum(u, v, P_HALF), rtol=1e-12)


def test_unit_norm_zero_filter_symmetry():
    f = K.from_expansion([1.0], [np.array([1.0, 0.0])], P_HALF)
    assert_allclose(K.inner_product(f, f, P_HALF), 1.0, rtol=1e-14)
    assert_allclose(K.norm_sq(f, P_HALF), 1.0, rtol=1e-14)
    rng = np.random.default_rng(4)
    _, _, g = random_expansion(rng, 7, 5, P_HALF)
    assert K.inner_product(K.zero_filter(5), g, P_HALF) == 0.0
    _, _, f = random_expansion(rng, 6, 4, P_HALF)
    _, _, g = random_expansion(rng, 9, 4, P_HALF)
    assert_allclose(K.inner_product(f, g, P_HALF), K.inner_product(g, f, P_HALF), rtol=1e-13)


@pytest.mark.parametrize("p", [P_HALF, K.KernelParams(0.2, 0.8, 0.3)])
def test_against_expansion_oracle(p):
    rng = np.random.default_rng(12)
    for _ in range(30):
        dim = int(rng.integers(2, 9))
        gf, af, f = random_expansion(rng, int(rng.integers(1, 12)), dim, p)
        gg, ag, g = random_expansion(rng, int(rng.integers(1, 12)), dim, p)
        assert_allclose(K.inner_product(f, g, p), oracle_inner(gf, af, gg, ag, p),
                        rtol=1e-10, atol=1e-12)


def test_fejer_monotonicity_on_trained_filter():
    """||f_n - f*||^2 non-increasing along the APSM iterates when the target
    f* interpolates every sample within eps (test_apsm.py:300-320)."""
    rng = np.random.default_rng(21)
    p = P_HALF
    star = K.from_expansion(rng.standard_normal(5) * 0.5, rng.standard_normal((5, 4)) * 0.4, p)
    R = rng.standard_normal((60, 4)) * 0.4
    B = K.batch_evaluate(star, R, p, K.EngineConfig())
    cfg = K.ApsmConfig(window=1, epsilon=0.01, params=p)
    star_norm = K.norm_sq(star, p)
    tr = K.ApsmTrainer(4, cfg)
    prev = star_norm
    for n, (r, b) in enumerate(zip(R, B)):
        tr.observe(r, b)
        if n % 6 == 5:
            f = tr.state()
            d2 = K.norm_sq(f, p) - 2.0 * K.inner_product(f, star, p) + star_norm
            assert d2 <= prev + 1e-9
            prev = d2
