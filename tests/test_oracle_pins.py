"""Pins for the CPU oracle (oracle/btree_oracle.c) against what the paper and
the mathematics fix -- not against the oracle itself.

Each test names the passage (P:n = PAPER.md line n) or the closed form it
checks.  CPU only; the whole file runs in well under a minute.
"""
import json
import os

import numpy as np
import pytest

from paper_1910_02639_b200 import datagen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "paper_worked_examples.json")))


# ---- Eq. 2 / Eq. 3 worked example --------------------------------
def test_eq2_eq3_worked_example(oracle):
    g = GOLD["eq2_eq3_worked_example"]
    c = [oracle.cell_coord(x, g["lo"], g["hi"], g["b"]) for x in g["x"]]
    assert c == g["coords"]
    assert oracle.cell_id(*c, g["b"]) == g["j"]
    assert g["b"] ** 3 == g["ncells"]


def test_eq2_clamps_and_faces(oracle):
    # x at the min face -> 0; x at the max face maps to b and is clamped to b-1 (R8)
    assert oracle.cell_coord(0.0, 0.0, 5.0, 10) == 0
    assert oracle.cell_coord(5.0, 0.0, 5.0, 10) == 9
    assert oracle.cell_coord(-1.0, 0.0, 5.0, 10) == 0
    assert oracle.cell_coord(7.0, 0.0, 5.0, 10) == 9
    # monotone in x on a fine sweep straddling every face (lemma L2)
    xs = np.linspace(-0.1, 5.1, 20001)
    cs = [oracle.cell_coord(float(x), 0.0, 5.0, 7) for x in xs]
    assert all(a <= b for a, b in zip(cs, cs[1:]))
    assert set(cs) == set(range(7))
    # zero-extent box (degenerate axis): still monotone, NaN (0/0) -> 0
    assert oracle.cell_coord(1.0, 1.0, 1.0, 4) == 0
    assert oracle.cell_coord(0.5, 1.0, 1.0, 4) == 0
    assert oracle.cell_coord(1.5, 1.0, 1.0, 4) == 3


def test_eq3_corners(oracle):
    for b in (2, 3, 10, 81):
        assert oracle.cell_id(0, 0, 0, b) == 0
        assert oracle.cell_id(b - 1, b - 1, b - 1, b) == b ** 3 - 1
        assert oracle.cell_id(1, 0, 0, b) == 1
        assert oracle.cell_id(0, 1, 0, b) == b
        assert oracle.cell_id(0, 0, 1, b) == b * b


# ---- Eq. 1 ------------------------------------------------------
def test_eq1_branching_factor(oracle):
    for n, s, b in GOLD["eq1_examples"]["cases"]:
        assert oracle.branching_factor(n, s) == b, (n, s)


def test_eq1_is_smallest_integer_root(oracle):
    rng = np.random.default_rng(7)
    for _ in range(2000):
        s = int(rng.integers(1, 200))
        n = int(rng.integers(s + 1, 10 ** 7))
        b = oracle.branching_factor(n, s)
        assert b >= 2
        assert b ** 3 * s >= n
        assert b == 2 or (b - 1) ** 3 * s < n


# ---- Eq. 4 ------------------------------------------------------
def test_eq4_ratio(oracle):
    for c in GOLD["eq4_examples"]["cases"]:
        assert oracle.ratio(c["counts"], c["alpha"], c["s"]) == c["r"]


# ---- Eq. 5 / Fig. 1 ----------------------------------
def test_eq5_fig1_range(oracle):
    g = GOLD["fig1_search_range"]
    rx = oracle.search_range(g["x"][0], g["R"], g["lo"], g["hi"], g["b"])
    ry = oracle.search_range(g["x"][1], g["R"], g["lo"], g["hi"], g["b"])
    assert list(rx) == g["range_x"]
    assert list(ry) == g["range_y"]
    # radius >= box side -> whole range; tiny radius at a cell centre -> one cell
    assert oracle.search_range(3.0, 10.0, 0.0, 6.0, 6) == (0, 5)
    assert oracle.search_range(2.5, 0.1, 0.0, 6.0, 6) == (2, 2)


# ---- root box (reading R9) ---------------------------------------
def test_root_box_strictly_contains(oracle):
    pos = np.array([[0.0, 0.0, 0.0], [1.0, 1.0, 1.0]])
    lo, hi = oracle.root_box(pos)
    assert np.all(lo < 0.0) and np.all(hi > 1.0)
    assert np.allclose(lo, -1e-9, rtol=1e-6) and np.allclose(hi, 1 + 1e-9, rtol=1e-12)
    lo, hi = oracle.root_box(np.zeros((1, 3)))
    assert np.all(hi - lo >= 2e-12)


# ---- predicate and closed forms ---------------------------------------------
def test_boundary_is_strict(oracle):
    pos = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    h = np.array([0.5, 0.5])  # d^2 = 1 = (2h)^2 -> not neighbors (strict <)
    for counts in (oracle.brute_force(pos, h)[0], oracle.Tree(pos, 1).count(h)):
        assert list(counts) == [0, 0]
    h = np.array([np.nextafter(0.5, 1.0), 0.5])  # (2h)^2 = 1 + 2^-51 > 1
    for counts in (oracle.brute_force(pos, h)[0], oracle.Tree(pos, 1).count(h)):
        assert list(counts) == [1, 0]  # gather: asymmetric for unequal h (R13)


def _lattice_expected(m, r2max):
    """Exact neighbor count of every point of an integer m^3 lattice for the
    criterion |d|^2 <= r2max (integers), by enumerating integer offsets."""
    offs = [(a, b, c) for a in range(-3, 4) for b in range(-3, 4) for c in range(-3, 4)
            if 0 < a * a + b * b + c * c <= r2max]
    idx = np.arange(m)
    gx, gy, gz = np.meshgrid(idx, idx, idx, indexing="ij")
    P = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
    cnt = np.zeros(len(P), dtype=np.int64)
    for a, b, c in offs:
        q = P + np.array([a, b, c])
        cnt += np.all((q >= 0) & (q < m), axis=1)
    return cnt


@pytest.mark.parametrize("two_h,r2max,interior", [(2.5, 6, 80), (1.01, 1, 6), (1.9, 3, 26)])
def test_lattice_closed_form(oracle, two_h, r2max, interior):
    m = 9
    pos = datagen.lattice(m, 1.0)
    h = np.full(len(pos), two_h / 2)
    exp = _lattice_expected(m, r2max)
    bf = oracle.brute_force(pos, h)[0]
    assert np.array_equal(bf, exp)
    for s in (1, 8, 64):
        assert np.array_equal(oracle.Tree(pos, s).count(h), exp)
    centre = (m // 2) * (m * m + m + 1)
    assert exp[centre] == interior


def test_brute_force_vs_scipy_ckdtree(oracle):
    """Independent library arithmetic: scipy's cKDTree (<= with its own
    arithmetic).  Sets agree except pairs within a relative band 1e-12 of
    the threshold, which we exclude from the comparison."""
    cKDTree = pytest.importorskip("scipy.spatial").cKDTree
    for seed, hh in ((1, (0.03, 0.08)), (2, (0.05, 0.05))):
        pos, h = datagen.uniform(3000, seed, *hh)
        c, off, idx = oracle.brute_force(pos, h)
        kd = cKDTree(pos)
        for i in range(0, 3000, 7):
            mine = set(idx[off[i]:off[i + 1]].tolist())
            theirs = set(kd.query_ball_point(pos[i], 2 * h[i])) - {i}
            for j in mine ^ theirs:
                d2 = float(np.sum((pos[i] - pos[j]) ** 2))
                assert abs(d2 - (2 * h[i]) ** 2) <= 1e-12 * (2 * h[i]) ** 2, (i, j)


# ---- tree walk vs brute force ----------------------------------------------
def _assert_same(a, b):
    ca, oa, ia = a
    cb, ob, ib = b
    assert np.array_equal(ca, cb)
    assert np.array_equal(oa, ob)
    assert np.array_equal(ia, ib)


@pytest.mark.parametrize("case", ["uniform", "varh", "clustered", "boundary", "lattice"])
def test_tree_walk_equals_brute_force(oracle, case):
    if case == "uniform":
        pos, h = datagen.uniform(4000, 11, 0.04)
    elif case == "varh":
        pos, h = datagen.uniform(4000, 12, 0.01, 0.08)
    elif case == "clustered":
        pos, h = datagen.clustered(5000, 13, h=0.01)
    elif case == "boundary":
        pos, h = datagen.near_boundary(64, 64, 14)
    else:
        pos = datagen.lattice(12, 0.01, 0.005)
        h = np.full(len(pos), 0.015)
    ref = oracle.brute_force(pos, h)
    for s, beta in ((64, 0.5), (8, 0.5), (1, 0.1), (2, 1.0)):
        _assert_same(oracle.Tree(pos, s, beta).neighbors(h), ref)


def test_invariance_over_s_beta_alpha(oracle):
    pos, h = datagen.clustered(6000, 21, h=0.015)
    ref = oracle.Tree(pos, 64).neighbors(h)
    for s in (1, 2, 8, 64, 4096):
        for beta in (0.1, 0.5, 1.0):
            for alpha in (0.0, 0.5):
                _assert_same(oracle.Tree(pos, s, beta, alpha).neighbors(h), ref)


def test_symmetry_constant_h_and_self_excluded(oracle):
    pos, h = datagen.uniform(3000, 31, 0.05)
    c, off, idx = oracle.Tree(pos, 16).neighbors(h)
    rows = np.repeat(np.arange(len(pos)), c)
    assert not np.any(rows == idx)
    pairs = set(zip(rows.tolist(), idx.tolist()))
    assert all((j, i) in pairs for i, j in pairs)
    assert c.sum() == off[-1] == idx.size


def test_permutation_invariance_and_monotone_h(oracle):
    pos, h = datagen.clustered(4000, 41, h=0.02)
    c, off, idx = oracle.Tree(pos, 32).neighbors(h)
    rng = np.random.default_rng(5)
    p = rng.permutation(len(pos))
    c2, off2, idx2 = oracle.Tree(pos[p], 32).neighbors(h[p])
    inv = np.argsort(p)
    for i in range(0, len(pos), 13):
        k = inv[i]
        mapped = np.sort(p[idx2[off2[k]:off2[k + 1]]])
        assert np.array_equal(mapped, idx[off[i]:off[i + 1]])
    cbig = oracle.Tree(pos, 32).count(h * 1.1)
    assert np.all(cbig >= c)


# ---- build structure (Alg. 1, Table II best case) --
def test_partition_and_bucket_bound(oracle):
    pos, h = datagen.clustered(20000, 51, h=0.01)
    for s in (1, 8, 64):
        t = oracle.Tree(pos, s)
        perm, lb, lc, ld = t.order()
        assert np.array_equal(np.sort(perm), np.arange(len(pos)))
        assert lc.sum() == len(pos)
        assert np.all(lc >= 1) and np.all(lc <= s)
        assert np.array_equal(lb[1:], np.cumsum(lc)[:-1])
        for b0, c in zip(lb[:200], lc[:200]):  # leaves keep ascending original index
            seg = perm[b0:b0 + c]
            assert np.all(np.diff(seg) > 0)
        st = t.stats()
        assert st["leaves"] == len(lc) and st["overfull"] == 0


@pytest.mark.parametrize("m", [4, 8, 16])
def test_even_lattice_best_case_depth_one(oracle, m):
    t = oracle.Tree(datagen.lattice(m, 1.0), 8)
    st = t.stats()
    assert st["depth"] == 1 and st["halvings"] == 0 and st["nodes"] == 1
    assert st["root_b"] == m // 2 and st["leaves"] == (m // 2) ** 3
    _, _, lc, _ = t.order()
    assert np.all(lc == 8)


def test_single_leaf_and_empty(oracle):
    pos, _ = datagen.uniform(50, 61, 0.1)
    st = oracle.Tree(pos, 64).stats()
    assert st["depth"] == 0 and st["leaves"] == 1 and st["nodes"] == 0
    st = oracle.Tree(np.zeros((0, 3)), 64).stats()
    assert st["leaves"] == 0


def test_coincident_points_depth_cap(oracle):
    s = 8
    pos = np.tile(np.array([[0.25, 0.5, 0.75]]), (s + 1, 1))
    pos = np.concatenate([pos, [[0.0, 0.0, 0.0], [1.0, 1.0, 1.0]]])
    h = np.full(len(pos), 0.01)
    t = oracle.Tree(pos, s, depth_cap=64)
    st = t.stats()
    assert st["overfull"] == 1 and st["max_leaf"] == s + 1 and st["depth"] == 64
    c = t.count(h)
    assert list(c[: s + 1]) == [s] * (s + 1) and list(c[s + 1:]) == [0, 0]


def test_halving_hand_derived(oracle):
    """1000 points in [0,0.1)^3 plus one at (1,1,1), s=8, beta=0.5:
    Eq. 1 gives b=6 (5^3 < 126 <= 6^3); r = 215/216 >= 0.5 -> b=3;
    r = 26/27 -> b = max(2, 1) = 2; at b=2 the loop stops (octree limit)."""
    rng = np.random.default_rng(3)
    pos = np.concatenate([rng.random((1000, 3)) * 0.1, [[1.0, 1.0, 1.0]]])
    t = oracle.Tree(pos, 8, 0.5)
    st = t.stats()
    assert st["root_b"] == 2
    # with beta = 1.0 the ratio never reaches beta (r < 1): b stays 6
    assert oracle.Tree(pos, 8, 1.0).stats()["root_b"] == 6


def test_uniform_root_needs_no_halving(oracle):
    pos, _ = datagen.uniform(20000, 71, 0.01)
    st = oracle.Tree(pos, 64).stats()
    assert st["root_b"] == oracle.branching_factor(20000, 64) == 7


# ---- FixedOctree policy (the paper's comparison baseline, Sec. II) ----
def test_octree_policy_lattice_depth(oracle):
    # 8^3 lattice, s = 8: the b-tree takes b = 4 at the root (depth 1, Table II
    # best case); the octree halves twice (8 -> 64 -> 8 particles): depth 2.
    pos = datagen.lattice(8, 1.0)
    bt = oracle.Tree(pos, 8).stats()
    oc = oracle.Tree(pos, 8, policy="octree").stats()
    assert bt["depth"] == 1 and bt["root_b"] == 4 and bt["leaves"] == 64
    assert oc["depth"] == 2 and oc["root_b"] == 2 and oc["leaves"] == 64 and oc["nodes"] == 9
    assert oc["halvings"] == 0


def test_octree_same_neighbors_deeper_tree(oracle):
    pos, h = datagen.clustered(8000, 91, h=0.01)
    bt = oracle.Tree(pos, 16)
    oc = oracle.Tree(pos, 16, policy="octree")
    _assert_same(bt.neighbors(h), oc.neighbors(h))
    assert oc.stats()["depth"] >= bt.stats()["depth"]
    perm, lb, lc, _ = oc.order()
    assert np.array_equal(np.sort(perm), np.arange(len(pos))) and np.all(lc <= 16)


# ---- SPH density consumer (reading R21: M4 cubic spline) -----
def test_density_kernel_normalisation_and_shape(oracle):
    """W(r, h) = w(r/h) / (pi h^3) integrates to one over its support 2h (the
    defining normalisation of an SPH kernel), w and w' are continuous at q = 1
    and q = 2, and hand-computed values hold."""
    from scipy.integrate import quad
    for h in (0.3, 1.0, 2.5):
        tot, _ = quad(lambda r: 4.0 * np.pi * r * r * oracle.w_m4(r / h) / (np.pi * h ** 3), 0.0, 2.0 * h,
                      points=[h], epsabs=1e-13)
        assert abs(tot - 1.0) < 1e-10
    e = 1e-7
    for q in (1.0, 2.0):
        assert abs(oracle.w_m4(q - e) - oracle.w_m4(q + e)) < 1e-6
        d_left = (oracle.w_m4(q - e) - oracle.w_m4(q - 2 * e)) / e
        d_right = (oracle.w_m4(q + 2 * e) - oracle.w_m4(q + e)) / e
        assert abs(d_left - d_right) < 1e-5
    assert oracle.w_m4(0.0) == 1.0
    assert abs(oracle.w_m4(0.7) - 0.52225) < 1e-15   # 1 - 1.5*0.49 + 0.75*0.343 (by hand)
    assert oracle.w_m4(1.5) == 0.03125                # 0.25 * 0.5^3
    assert oracle.w_m4(2.0) == 0.0 and oracle.w_m4(3.0) == 0.0


def test_density_closed_forms(oracle):
    # an isolated particle sees only itself: rho = m W(0, h) = m / (pi h^3)
    pos = np.array([[0.1, 0.2, 0.3]])
    rho = oracle.Tree(pos, 8).density(np.array([0.5]), np.array([2.0]))
    assert rho[0] == 2.0 / (np.pi * 0.125)
    # a fine unit lattice, unit masses, h = 3 lattice spacings: an interior
    # particle's kernel sum approximates the continuum density 1 / a^3
    m = 21
    pos = datagen.lattice(m, 1.0)
    h = np.full(len(pos), 3.0)
    centre = (m // 2) * (m * m + m + 1)
    rho = oracle.Tree(pos, 64).density(h, np.ones(len(pos)), queries=np.array([centre]))
    assert abs(rho[0] - 1.0) < 2e-3


def test_density_tree_equals_brute_force(oracle):
    pos, h = datagen.uniform(3000, 17, 0.05, 0.08)
    mass = np.random.default_rng(3).uniform(0.5, 1.5, len(pos))
    a = oracle.Tree(pos, 16).density(h, mass)
    b = oracle.brute_density(pos, h, mass)
    assert np.array_equal(a, b)   # same terms, same (ascending j) order


# ---- symmetric criterion (reading R22) ---------------------
def test_symmetric_hand_values(oracle):
    # d = 1, h = (0.6, 0.1): gather gives 0 -> 1 only (1 < 1.2, 1 >= 0.2); the
    # max(h_i, h_j) criterion gives both directions
    pos = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    h = np.array([0.6, 0.1])
    c, off, idx = oracle.brute_force(pos, h)
    assert c.tolist() == [1, 0] and idx.tolist() == [1]
    c, off, idx = oracle.brute_force(pos, h, symmetric=True)
    assert c.tolist() == [1, 1] and idx.tolist() == [1, 0]
    # strict at d = 2 max(h): d^2 = 1 = (2 * 0.5)^2 -> not neighbors
    h = np.array([0.5, 0.1])
    assert oracle.brute_force(pos, h, symmetric=True)[0].tolist() == [0, 0]
    h = np.array([0.1, np.nextafter(0.5, 1.0)])
    assert oracle.brute_force(pos, h, symmetric=True)[0].tolist() == [1, 1]


def test_symmetric_chain_closed_form(oracle):
    # unit-spaced chain, h alternating 0.3 (2h = 0.6 < 1) and 0.55 (2h = 1.1 < 2):
    # gather: odd points see their two neighbours, even points none; symmetric:
    # every point sees its two neighbours (ends: one)
    m = 101
    pos = np.zeros((m, 3))
    pos[:, 0] = np.arange(m, dtype=np.float64)
    h = np.where(np.arange(m) % 2 == 0, 0.3, 0.55)
    cg = oracle.brute_force(pos, h)[0]
    cs = oracle.brute_force(pos, h, symmetric=True)[0]
    expect_g = np.where(np.arange(m) % 2 == 1, 2, 0)
    expect_s = np.full(m, 2)
    expect_s[0] = expect_s[-1] = 1
    assert np.array_equal(cg, expect_g)
    assert np.array_equal(cs, expect_s)


def test_symmetric_is_gather_union_transpose(oracle):
    # N_sym(i) = N(i) u {j : i in N(j)} (d^2 is the same bits both ways and
    # fl(t^2) is monotone), with N from the tree walk (Alg. 2), an independent
    # code path from the symmetric brute force; constant h: N_sym = N
    pos, h = datagen.clustered(3000, 61, h=0.012)
    h = h * np.random.default_rng(62).uniform(0.5, 2.0, len(h))
    c, off, idx = oracle.Tree(pos, 16).neighbors(h)
    rows = np.repeat(np.arange(len(pos)), c)
    union = set(zip(rows.tolist(), idx.tolist())) | set(zip(idx.tolist(), rows.tolist()))
    cs, offs, idxs = oracle.brute_force(pos, h, symmetric=True)
    rs = np.repeat(np.arange(len(pos)), cs)
    sym = set(zip(rs.tolist(), idxs.tolist()))
    assert sym == union
    assert len(sym) > c.sum()  # variable h: some pairs are one-sided
    assert all((j, i) in sym for i, j in sym)
    hc = np.full(len(pos), 0.02)
    g = oracle.brute_force(pos, hc)
    s = oracle.brute_force(pos, hc, symmetric=True)
    _assert_same(g, s)


# ---- k = 2 (the paper's k-generic b-tree, Table I; reading R23) ---------
def _plane_lattice(m, z=0.0):
    g = np.arange(m, dtype=np.float64)
    gx, gy = np.meshgrid(g, g, indexing="ij")
    return np.ascontiguousarray(np.stack([gx.ravel(), gy.ravel(), np.full(m * m, z)], axis=1))


def test_eq1_two_dimensions(oracle):
    # b = smallest integer >= 2 with b^2 s >= n, by integer arithmetic
    assert oracle.branching_factor_k(10**6, 64, 2) == 125      # 125^2 = 15625 = 10^6 / 64
    assert oracle.branching_factor_k(10**6 + 1, 64, 2) == 126
    assert oracle.branching_factor_k(5, 8, 2) == 2
    assert oracle.branching_factor_k(2**25, 64, 2) == 725    # 724^2 < 524288 <= 725^2
    rng = np.random.default_rng(17)
    for _ in range(500):
        n, s = int(rng.integers(1, 10**9)), int(rng.integers(1, 5000))
        b = oracle.branching_factor_k(n, s, 2)
        m = -(-n // s)
        assert b * b >= m and (b == 2 or (b - 1) ** 2 < m)
        assert oracle.branching_factor_k(n, s, 3) == oracle.branching_factor(n, s)


@pytest.mark.parametrize("m", [4, 8, 16])
def test_plane_lattice_best_case_k2(oracle, m):
    # m^2 plane lattice, s = 4: Eq. 1 (k = 2) gives b = m/2, every cell 2x2 =
    # 4 points = s: depth 1, no halving, (m/2)^2 leaves of 4 -- the 2-D analogue
    # of the Table II best case; the quadtree reaches it only at depth log2(m/2)
    pos = _plane_lattice(m)
    st = oracle.Tree(pos, 4, policy="btree2d").stats()
    assert st["depth"] == 1 and st["halvings"] == 0 and st["nodes"] == 1
    assert st["root_b"] == m // 2 and st["leaves"] == (m // 2) ** 2
    _, _, lc, _ = oracle.Tree(pos, 4, policy="btree2d").order()
    assert np.all(lc == 4)
    q = oracle.Tree(pos, 4, policy="quadtree").stats()
    assert q["root_b"] == 2 and q["leaves"] == (m // 2) ** 2
    assert q["depth"] == int(np.log2(m // 2)) and q["nodes"] == sum(4 ** d for d in range(q["depth"]))


def test_halving_hand_derived_k2(oracle):
    """1000 points in [0,0.01)^2 x [0,1) plus one at (1,1,1), s = 8, k = 2:
    Eq. 1 gives b = 12 (11^2 < 126 <= 12^2); r = 142/144 -> b = 6; r = 34/36 ->
    b = 3; r = 7/9 -> b = 2; at b = 2 the loop stops: 3 halvings at the root."""
    rng = np.random.default_rng(4)
    pts = rng.random((1000, 3)) * np.array([0.01, 0.01, 1.0])
    pos = np.concatenate([pts, [[1.0, 1.0, 1.0]]])
    st = oracle.Tree(pos, 8, 0.5, policy="btree2d").stats()
    assert st["root_b"] == 2
    t = oracle.Tree(pos, 8, 1.0, policy="btree2d")
    assert t.stats()["root_b"] == 12 and t.stats()["halvings"] == 0


def test_k2_trees_same_neighbors(oracle):
    # the neighbor sets do not depend on the tree: k = 2 (slabs through z) and the
    # quadtree give the brute-force sets on 3-D and planar inputs
    pos, h = datagen.clustered(5000, 93, h=0.012)
    ref = oracle.brute_force(pos, h)
    for pol in ("btree2d", "quadtree"):
        for s in (4, 16, 64):
            _assert_same(oracle.Tree(pos, s, 0.5, policy=pol).neighbors(h), ref)
    flat = pos.copy()
    flat[:, 2] = 0.25
    ref = oracle.brute_force(flat, h)
    for pol in ("btree", "btree2d", "quadtree"):
        _assert_same(oracle.Tree(flat, 16, 0.5, policy=pol).neighbors(h), ref)


# ---- Eq. 4 tie r = beta (reading R3: the prose "until r < beta", P:254-256,
# so a ratio equal to beta halves) ---------------------------------------------
def _tie_set():
    """A 4^3 lattice of sites (i + 0.5), s = 8 (alpha s = 4): 32 sites carry 5
    coincident points (over-full), 32 carry 2 (under-full), n = 224.  Eq. 1
    gives b = 4 (3^3 8 = 216 < 224 <= 512); every site is its own root cell
    (cell = i), so Eq. 4 gives r = 32 / 64 = 0.5 exactly."""
    pts = []
    for k in range(64):
        i, j, l = k % 4, (k // 4) % 4, k // 16
        mult = 5 if (i + j + l) % 2 == 0 else 2  # 32 even-parity sites, 32 odd
        pts += [[i + 0.5, j + 0.5, l + 0.5]] * mult
    return np.array(pts, dtype=np.float64)


def test_eq4_tie_halves(oracle):
    pos = _tie_set()
    assert len(pos) == 224 and oracle.branching_factor(224, 8) == 4
    # r = beta = 0.5: halve (4 -> 2); the root then holds 28 points per cell (r = 0)
    st = oracle.Tree(pos, 8, 0.5).stats()
    assert st["root_b"] == 2 and st["halvings"] == 1
    # beta one ulp-scale step above r: r < beta, b stays 4 and every site is a leaf
    st = oracle.Tree(pos, 8, 0.5 + 2.0 ** -20).stats()
    assert st["root_b"] == 4 and st["halvings"] == 0 and st["leaves"] == 64 and st["depth"] == 1
    # beta below r: halves as well
    assert oracle.Tree(pos, 8, 0.5 - 2.0 ** -20).stats()["root_b"] == 2


# ---- depth-first leaf order, children in ascending j (Sec. IV-E, the
# reorder along the tree-walk curve; Eq. 3 j = c1 + c2 b + c3 b^2) -------------
def test_leaf_order_depth_first_ascending_j(oracle):
    """4^3 lattice at (i + 0.5) without root cell 2's eight sites, plus eight
    points at (site + 0.1) inside root cell 5: n = 64, s = 8 -> b = 2 (Eq. 1),
    r = 1/8 (only cell 2 empty).  Root cells 0, 1, 3, 4, 6, 7 are leaves of 8;
    cell 5 (16 points) splits into 2^3 sub-cells of 2 (a lattice site and its
    +0.1 partner; sub-cell faces lie at 2.75 / 1.25 / 2.75 of the cell box
    [2, 3.5] x [0.5, 2] x [2, 3.5]).  The expected order, worked out here from
    the geometry alone: cells 0, 1, 3, 4, then cell 5's sub-cells in ascending
    sub-j, then cells 6, 7; inside a leaf ascending input index."""
    def root_cell(p):
        c = [int(v - 0.5) // 2 for v in p]   # site index i // 2 on every axis
        return c[0] + 2 * c[1] + 4 * c[2]
    sites = [[i + 0.5, j + 0.5, l + 0.5] for l in range(4) for j in range(4) for i in range(4)]
    sites = [s for s in sites if root_cell(s) != 2]
    extra = [[s[0] + 0.1, s[1] + 0.1, s[2] + 0.1] for s in sites if root_cell(s) == 5]
    pos = np.array(sites + extra, dtype=np.float64)
    assert len(pos) == 64
    t = oracle.Tree(pos, 8, 0.5)
    st = t.stats()
    assert st["root_b"] == 2 and st["halvings"] == 0 and st["depth"] == 2
    perm, lb, lc, ld = t.order()

    def sub_cell(p):  # cell 5's sub-cells: faces at x 2.75, y 1.25, z 2.75
        return int(p[0] > 2.75) + 2 * int(p[1] > 1.25) + 4 * int(p[2] > 2.75)
    in_cell = [root_cell(p) for p in pos]  # (the +0.1 partners stay in their site's cell)
    expect = [(1, [k for k in range(64) if in_cell[k] == j]) for j in (0, 1, 3, 4)]
    expect += [(2, [k for k in range(64) if in_cell[k] == 5 and sub_cell(pos[k]) == sj]) for sj in range(8)]
    expect += [(1, [k for k in range(64) if in_cell[k] == j]) for j in (6, 7)]
    assert len(lc) == len(expect)
    for leaf, (depth, members) in enumerate(expect):
        assert ld[leaf] == depth
        assert list(perm[lb[leaf]:lb[leaf] + lc[leaf]]) == sorted(members), leaf
