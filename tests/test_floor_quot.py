"""CPU check of the exactness argument behind K1's floor_quot (pgrid_kernels.cuh): the floor of
RN(x * RN(1/c)) equals numpy's floor(RN(x / c)) whenever RN(x * RN(1/c)) is farther than
2^-50 |p| from an integer -- restated in numpy float64 (same IEEE operations, no FMA) and
run over values on, near and between cell boundaries."""
import numpy as np


def floor_quot(x, c):
    rc = 1.0 / c
    p = x * rc
    f = np.floor(p)
    tol = np.abs(p) * 2.0 ** -50
    fast = (np.abs(p) < 2.0 ** 52) & ((p - f) > tol) & (((f + 1.0) - p) > tol)
    with np.errstate(all="ignore"):
        slow = np.floor(x / c)
    return np.where(fast, f, slow), fast


def test_floor_quot_matches_ieee_division():
    rng = np.random.default_rng(5)
    total = fast_total = 0
    for _ in range(20):
        c = rng.uniform(1e-6, 10.0) * 10.0 ** rng.integers(-3, 4)
        k = rng.integers(-5, 2000, size=200_000).astype(np.float64)
        x = k * c                                          # on boundaries (rounded)
        u = rng.integers(-8, 9, size=x.shape)
        for _i in range(8):                                 # up to 8 ulps either side
            x = np.where(u > _i, np.nextafter(x, np.inf), x)
            x = np.where(u < -_i, np.nextafter(x, -np.inf), x)
        x = np.concatenate([x, rng.uniform(-10, 2000, size=200_000) * c, np.array([0.0, -0.0, 1e-310, -1e-310])])
        got, fast = floor_quot(x, c)
        want = np.floor(x / c)
        assert np.array_equal(got, want), (c, x[got != want][:5])
        total += x.size
        fast_total += int(fast.sum())
    assert fast_total > 0.5 * total      # the division is the exception
