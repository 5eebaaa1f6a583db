"""Input generators: determinism, ranges and distribution shape."""
import numpy as np

import zdgen


def test_deterministic_and_prefix_stable():
    a = zdgen.uniform(1000, 3, seed=3)
    b = zdgen.uniform(1000, 3, seed=3)
    c = zdgen.uniform(500, 3, seed=3)
    assert np.array_equal(a, b) and np.array_equal(a[:500], c)
    assert not np.array_equal(a, zdgen.uniform(1000, 3, seed=4))
    assert np.array_equal(zdgen.plummer(3000, 4), zdgen.plummer(3000, 4))


def test_ranges():
    for dim, B in ((2, 30), (3, 21)):
        p = zdgen.uniform(100_000, dim, seed=1)
        assert p.dtype == np.int32 and p.min() >= 0 and p.max() < (1 << B)
        m = p.astype(np.float64).mean(0) / (1 << B)
        assert np.all(np.abs(m - 0.5) < 0.01)
    for f in (zdgen.plummer, zdgen.sphere):
        p = f(100_000, 5)
        assert p.min() >= 0 and p.max() < (1 << 21)


def test_plummer_concentrated():
    p = zdgen.plummer(100_000, 4).astype(np.float64)
    c = (1 << 20)
    r = np.sqrt(((p - c) ** 2).sum(1)) / (1 << 21) * 100.0   # back to model units
    # Plummer cumulative mass M(<r) = r^3 / (1 + r^2)^1.5 ; half-mass radius ~1.305
    frac = (r < 1.305).mean()
    assert abs(frac - 0.5) < 0.01
    assert r.max() <= 50.0 * np.sqrt(3) + 1e-6


def test_sphere_radius():
    p = zdgen.sphere(50_000, 5).astype(np.float64)
    r = np.sqrt(((p + 0.5 - (1 << 20)) ** 2).sum(1)) / (1 << 20)
    assert np.all(np.abs(r - 1.0) < 3.0 / (1 << 20))


def test_delete_ids():
    d = zdgen.delete_ids(100_000, 10_000, seed=8)
    assert d.size == 10_000 and np.unique(d).size == 10_000
    assert np.array_equal(d, zdgen.delete_ids(100_000, 10_000, seed=8))
    assert d.min() >= 0 and d.max() < 100_000
    h = zdgen.words(8, np.arange(100_000), 0)
    assert h[d].max() < np.delete(h, d).min()


def test_kuzmin_radial_cdf():
    """Kuzmin disk: M(<R) = 1 - 1/sqrt(1 + R^2), truncated at R = 100."""
    p = zdgen.kuzmin(200_000, 9).astype(np.float64)
    assert p.shape == (200_000, 2) and p.min() >= 0 and p.max() < 2 ** 30
    c = (p + 0.5) / 2 ** 30 * 200.0 - 100.0
    R = np.sqrt((c ** 2).sum(1))
    mcut = 1 - 1 / np.sqrt(1 + 100.0 ** 2)
    for r0 in (0.5, 1.0, 3.0, 10.0):
        expect = (1 - 1 / np.sqrt(1 + r0 ** 2)) / mcut
        assert abs((R < r0).mean() - expect) < 0.01, (r0, (R < r0).mean(), expect)
    assert np.array_equal(zdgen.kuzmin(1000, 9), zdgen.kuzmin(5000, 9)[:1000])
