"""The seeded generators: reproducible, right sizes and h recipes."""
import numpy as np

from paper_1910_02639_b200 import datagen


def test_reproducible_and_shapes():
    for cfg, n in ((1, None), (2, 5000), (3, 8000), (4, 5000), (5, 6000)):
        a = datagen.make_config(cfg, n=n)
        b = datagen.make_config(cfg, n=n)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        assert a[0].dtype == np.float64 and a[0].flags.c_contiguous and a[0].shape[1] == 3
        assert np.all(a[1] > 0) and np.all(np.isfinite(a[0]))
    assert datagen.make_config(1)[0].shape == (10_000, 3)


def test_recipes():
    pos, h = datagen.make_config(1)
    assert np.all(h == 0.0668) and pos.min() >= 0 and pos.max() < 1
    pos, h = datagen.make_config(4, n=100_000)
    r = np.linalg.norm(pos, axis=1)
    n_r = 100_000 / (2 * np.pi * r)
    assert np.allclose(4.0 / 3.0 * np.pi * (2 * h) ** 3 * n_r, 100.0, rtol=1e-9)
    pos, h = datagen.make_config(3, n=27_000)
    assert pos.shape[0] == 27_000 and np.allclose(h, 1.5 / 30)


def test_near_boundary_places_pairs_at_2h():
    pos, h = datagen.near_boundary(8, 16, 1)
    assert pos.shape[0] == 8 * 17
