"""The closed forms the carry-exchange kernels rely on, checked on the CPU
against the two first-order recurrences of the factored shifted solve
(DESIGN.md §3.1, §3.3 "Early carries"; csrc/ridc_febe_carry.cuh):

* y_end of a chunk (zero carry in) and its local first x (zero carries at
  both ends) are dot products of the chunk's right-hand side, computed per
  lane with the pw[e] = lam^(e+1) table and the lane multipliers M^lane,
  M^(31-lane) (M = lam^K);
* zf[e] = (pw[e] - lam^(K+1) pw[K-1-e]) / (1 - lam^2), so the warp's own carry
  corrections and the neighbours' head / tail corrections are one rank-2
  update in the basis pw[e], pw[K-1-e];
* the dropped lam^(2 CH - j) part of the first-x weight is below lam^CH.
"""
import numpy as np
import pytest


def _lam(r):
    # (I - dt L_S) = (r / lam)(1 - lam E^-1)(1 - lam E): lam + 1/lam = 2 + 1/r
    b = 2.0 + 1.0 / r
    return (b - np.sqrt(b * b - 4.0)) / 2.0


def _local_solve(rhs, lam):
    """Zero-carry forward then backward recurrences over one chunk."""
    y = np.zeros_like(rhs)
    acc = 0.0
    for j in range(rhs.size):
        acc = lam * acc + rhs[j]
        y[j] = acc
    x = np.zeros_like(rhs)
    acc = 0.0
    for j in range(rhs.size - 1, -1, -1):
        acc = lam * acc + y[j]
        x[j] = acc
    return y, x


@pytest.mark.parametrize("r,K", [(110.0, 16), (110.0, 32), (20.0, 16)])
def test_early_carries_are_dot_products(r, K):
    lam = _lam(r)
    CH = 32 * K
    rng = np.random.default_rng(7)
    rhs = rng.standard_normal(CH)
    y, x = _local_solve(rhs, lam)
    pw = lam ** (np.arange(K) + 1.0)
    M = lam ** K
    inv = 1.0 / (1.0 - lam * lam)
    yend = xfirst = 0.0
    for lane in range(32):
        r_l = rhs[K * lane:K * lane + K]
        ml, mr = M ** lane, M ** (31 - lane)
        sa = float(r_l @ pw)          # lam * sum_e lam^e r_e
        sb = float(r_l @ pw[::-1])    # lam * sum_e lam^(K-1-e) r_e = lam * (the lane's last y)
        yend += sb * mr / lam
        xfirst += sa * ml * inv / lam
    assert abs(yend - y[-1]) <= 1e-13 * np.abs(y).max()
    # the dropped lam^(2 CH - j) part: below lam^CH relative (the kernels' truncation)
    assert abs(xfirst - x[0]) <= max(1e-13, 4.0 * lam ** CH) * np.abs(x).max()


@pytest.mark.parametrize("r,K", [(110.0, 16), (20.0, 32)])
def test_zf_is_in_the_rank2_basis(r, K):
    lam = _lam(r)
    pw = lam ** (np.arange(K) + 1.0)
    # zf[e]: the lane's x response at point e to a unit forward carry into the lane
    zf = np.array([sum(lam ** (k - e) * lam ** (k + 1) for k in range(e, K)) for e in range(K)])
    rebuilt = (pw - lam ** (K + 1) * pw[::-1]) / (1.0 - lam * lam)
    assert np.allclose(zf, rebuilt, rtol=1e-13, atol=0.0)


def test_one_hop_tail_carry():
    """Two neighbouring chunks: the left chunk's exact solution near its end
    is its local solution + the right chunk's (local first x + the head
    correction the left chunk's own y_end causes there) times lam^(T - i)."""
    r, K = 110.0, 16
    lam = _lam(r)
    T = 32 * K
    rng = np.random.default_rng(3)
    rhs = rng.standard_normal(3 * T)
    y_all, x_all = _local_solve(rhs, lam)   # the exact non-periodic solve of three chunks
    left, right = rhs[T:2 * T], rhs[2 * T:3 * T]
    yl, xl = _local_solve(left, lam)
    yr, xr = _local_solve(right, lam)
    # the left chunk's exact forward carry in is y_all[T - 1]; correct its local x
    c = y_all[T - 1]
    i = np.arange(T)
    x_head = xl + c * lam ** (i + 1) / (1.0 - lam * lam)
    # tail: d = right's local first x + the head correction my own y_end causes there
    yend = yl[-1] + c * lam ** T   # my y_end with my own carry in (the one-hop rule's value)
    d = xr[0] + yend * lam / (1.0 - lam * lam)
    x_corr = x_head + d * lam ** (T - i)
    exact = x_all[T:2 * T]
    # the right chunk's own backward carry (lam^T) and the third chunk's are dropped
    assert np.max(np.abs(x_corr - exact)) <= 1e-12 * np.abs(exact).max()
