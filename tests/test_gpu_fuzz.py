"""Randomised GPU parity sweep: seeded random particle sets (shapes, sizes,
h distributions, tree policies, bucket sizes, beta) through every entry point
of the C ABI, each checked element by element against the oracle's plain
definitions (brute force, symmetric brute force, brute-force density).  The
seeds are fixed, so a failure is reproducible by its case id.

Run with ``pytest -m gpu`` on a B200.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1910_02639_b200 import datagen  # noqa: E402
from test_gpu_parity import DEV, assert_same, sort_rows  # noqa: E402

pytestmark = pytest.mark.gpu

POLICIES = ("btree", "octree", "btree2d", "quadtree")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1910_02639_b200 as P
    P.lib()
    return P


def _case(seed):
    """A random particle set: uniform / clumped / planar / shell / duplicated
    points, n in [1, 12000], h spread over a decade, random (s, beta, policy)."""
    rng = np.random.default_rng(10_000 + seed)
    n = int(rng.choice([1, 2, 3, 17, 64, 65, 500, 2000, 5000, 12000, 30000]))
    kind = rng.integers(0, 5)
    if kind == 0:
        pos = rng.random((n, 3))
    elif kind == 1:  # clumps
        c = rng.random((4, 3))
        pos = c[rng.integers(0, 4, n)] + rng.normal(0, 0.02, (n, 3))
    elif kind == 2:  # planar
        pos = np.zeros((n, 3))
        pos[:, :2] = rng.random((n, 2))
    elif kind == 3:  # thin spherical shell far from the origin
        v = rng.normal(size=(n, 3))
        pos = 1e3 + v / np.linalg.norm(v, axis=1, keepdims=True) * (1 + 1e-3 * rng.random((n, 1)))
    else:  # many exact duplicates
        base = rng.random((max(1, n // 8), 3))
        pos = base[rng.integers(0, len(base), n)]
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    ext = float(np.max(pos.max(0) - pos.min(0))) if n > 1 else 1.0
    ext = ext if ext > 0 else 1.0
    hmean = ext * (30.0 / max(n, 1)) ** (1 / 3) * rng.uniform(0.3, 1.5)
    h = hmean * np.exp(rng.uniform(-1.2, 1.2, n)) if rng.random() < 0.7 else np.full(n, hmean)
    s = int(rng.choice([1, 4, 16, 64, 200]))
    beta = float(rng.choice([0.1, 0.5, 1.0]))
    policy = POLICIES[int(rng.integers(0, 4))]
    return pos, np.ascontiguousarray(h), s, beta, policy


@pytest.mark.parametrize("seed", range(96))
def test_fuzz_gather_symmetric_density(P, oracle, seed):
    pos, h, s, beta, policy = _case(seed)
    n = len(pos)
    t = P.build(torch.from_numpy(pos).to(DEV), s, beta, policy=policy)
    hd = torch.from_numpy(h).to(DEV)
    c, o, nb = t.find_neighbors(hd)
    gpu = (c.cpu().numpy(), o.cpu().numpy(), sort_rows(c, o, nb))
    assert_same(gpu, oracle.brute_force(pos, h))
    cs, os_, ns = t.find_neighbors(hd, symmetric=True)
    assert_same((cs.cpu().numpy(), os_.cpu().numpy(), sort_rows(cs, os_, ns)),
                oracle.brute_force(pos, h, symmetric=True))
    m = np.random.default_rng(seed).uniform(0.5, 2.0, n)
    rho = t.density(hd, torch.from_numpy(m).to(DEV)).cpu().numpy()
    np.testing.assert_allclose(rho, oracle.brute_density(pos, h, m), rtol=2e-5, atol=0)
    # the tree agrees with the oracle's for this policy
    st, ost = t.stats(), oracle.Tree(pos, s, beta, policy=policy).stats()
    for k in ("nodes", "leaves", "halvings", "depth", "root_b", "max_leaf"):
        assert st[k] == ost[k], (k, st[k], ost[k])
    # a random partition is a disjoint cover of the rows
    if n > 1:
        parts = int(np.random.default_rng(seed + 1).integers(2, 6))
        tot = 0
        for p in range(parts):
            t.set_partition(p, parts)
            cp, op = t.count(hd)
            tot += int(op[-1])
        assert tot == int(o[-1])
