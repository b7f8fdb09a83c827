"""Quadrature weights: SPEC KATs (acceptance 4) and packing."""

from fractions import Fraction

import numpy as np
import pytest

from paper_1209_4297_b200.quadrature import (apply_quadrature, pack_weight_tables,
                                              startup_weights, steady_weights,
                                              weight_table_offsets)


def test_steady_kats():
    assert np.allclose(steady_weights(1, 1.0).weights, [0.5, 0.5], rtol=0, atol=1e-16)
    assert np.allclose(steady_weights(2, 1.0).weights, [5 / 12, 2 / 3, -1 / 12], rtol=0, atol=1e-15)
    assert np.allclose(steady_weights(3, 1.0).weights, [3 / 8, 19 / 24, -5 / 24, 1 / 24], rtol=0, atol=1e-15)


def test_startup_kats():
    assert np.allclose(startup_weights(2, 0, 1.0).weights, [5 / 12, 2 / 3, -1 / 12], atol=1e-15)
    assert np.allclose(startup_weights(3, 0, 1.0).weights, [3 / 8, 19 / 24, -5 / 24, 1 / 24], atol=1e-15)
    assert np.allclose(startup_weights(3, 1, 1.0).weights, [-1 / 24, 13 / 24, 13 / 24, -1 / 24], atol=1e-15)


@pytest.mark.parametrize("j", range(1, 12))
def test_sum_is_dt(j):
    for dt in (1.0, 1e-4, 0.37):
        assert abs(steady_weights(j, dt).weights.sum() - dt) <= 1e-13 * dt
        for n in range(j - 1):
            assert abs(startup_weights(j, n, dt).weights.sum() - dt) <= 1e-13 * dt


@pytest.mark.parametrize("j", [1, 2, 3, 4, 5])
def test_polynomial_exactness_vs_gauss(j):
    """Acceptance 4: exact on t^m, m <= j, vs Gauss-Legendre on random placements."""
    rng = np.random.default_rng(j)
    xg, wg = np.polynomial.legendre.leggauss(j + 2)
    for _ in range(10):
        tn, dt = rng.uniform(-2, 2), rng.uniform(0.05, 1.0)
        for m in range(j + 1):
            f = lambda t: t ** m  # noqa: E731
            a, b = tn, tn + dt
            exact = np.sum(wg * f(0.5 * (b - a) * xg + 0.5 * (a + b))) * 0.5 * (b - a)
            nodes = [tn + dt - k * dt for k in range(j + 1)]   # steady: t_{n+1-k}
            got = apply_quadrature(steady_weights(j, dt), [f(x) for x in nodes])
            assert abs(got - exact) <= 1e-12 * max(1.0, abs(exact))
            for n in range(j - 1):
                t0 = tn - n * dt
                nodes = [t0 + k * dt for k in range(j + 1)]
                got = apply_quadrature(startup_weights(j, n, dt), [f(x) for x in nodes])
                assert abs(got - exact) <= 1e-12 * max(1.0, abs(exact))


def test_pack_layout():
    L = 5
    st, su, total = weight_table_offsets(L)
    packed = pack_weight_tables(L, 0.01)
    assert packed.shape[0] == total == sum(j + 1 for j in range(1, L)) + sum(
        (j - 1) * (j + 1) for j in range(2, L))
    for j in range(1, L):
        assert np.array_equal(packed[st[j]:st[j] + j + 1], steady_weights(j, 0.01).weights)
    for j in range(2, L):
        for n in range(j - 1):
            o = su[(j, n)]
            assert np.array_equal(packed[o:o + j + 1], startup_weights(j, n, 0.01).weights)
        # the native side indexes startup (j, n) as startup_off[j] + n*(j+1)
        assert su[(j, 1)] - su[(j, 0)] == j + 1 if j > 2 else True


def test_invalid():
    with pytest.raises(ValueError):
        steady_weights(0, 1.0)
    with pytest.raises(ValueError):
        steady_weights(12, 1.0)
    with pytest.raises(ValueError):
        startup_weights(3, 2, 1.0)


def test_bitwise_vs_reference(reference):
    from ridc import quadrature as RQ
    for dt in (1.0, 4e-3, 1e-4):
        for j in range(1, 12):
            assert np.array_equal(RQ.steady_weights(j, dt).weights, steady_weights(j, dt).weights)
            for n in range(j - 1):
                assert np.array_equal(RQ.startup_weights(j, n, dt).weights,
                                      startup_weights(j, n, dt).weights)
