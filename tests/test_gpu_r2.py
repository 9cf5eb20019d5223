"""GPU tests added in round 2: robustness fixes and the tree-shape
pins of the oracle (Eq. 4 tie, depth-first ascending-j leaf order) carried to
the CUDA build.  Run with ``pytest -m gpu`` on a B200."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1910_02639_b200 import datagen  # noqa: E402

from test_gpu_parity import DEV, assert_same, assert_same_tree, gpu_run, sort_rows  # noqa: E402
from test_oracle_pins import _tie_set  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1910_02639_b200 as P
    P.lib()
    return P


def test_big_coincident_leaves(P, oracle):
    """Clusters of 1500 / 2600 / 4100 identical points (R14: depth-cap leaves
    above the warp-rank limit, ordered by the segmented sort) in a uniform
    background: tree and neighbor sets equal the oracle's."""
    rng = np.random.default_rng(11)
    parts = [rng.random((20000, 3))]
    for m, c in ((1500, 0.2), (2600, 0.5), (4100, 0.8)):
        parts.append(np.tile([[c, c, c]], (m, 1)))
    pos = np.ascontiguousarray(np.concatenate(parts)[rng.permutation(20000 + 8200)])
    h = np.full(len(pos), 0.01)
    for s in (8, 64):
        t, gpu = gpu_run(P, pos, h, s=s, depth_cap=20)
        ot = oracle.Tree(pos, s, depth_cap=20)
        assert_same_tree(t, ot)
        assert_same(gpu, ot.neighbors(h))
        assert t.stats()["max_leaf"] == 4100


def test_fill_only_rejects_foreign_offsets(P):
    """A fill-only call whose offsets are not the scan of this tree's counts
    for this h (another h, another partition) is refused with BT_ERR_ARG
    instead of writing rows past their ends."""
    pos, h = datagen.make_config(2, n=40_000)
    t = P.build(torch.from_numpy(pos).to(DEV))
    hd = torch.from_numpy(h).to(DEV)
    hd_big = hd * 1.3
    _, off_small = t.count(hd)
    c_big, off_big = t.count(hd_big)
    # offsets of the smaller h with the larger h's record: counts grew
    with pytest.raises(P.BtreeError) as e:
        t.fill(hd_big, off_small, out=torch.empty(int(off_big[-1]), dtype=torch.int32, device=DEV))
    assert e.value.code == 1
    # after a rerun of the test pass (h changed at the same pointer) as well
    hd2 = hd.clone()
    t.count(hd2)
    hd2.mul_(1.3)
    with pytest.raises(P.BtreeError) as e:
        t.fill(hd2, off_small, out=torch.empty(int(off_big[-1]), dtype=torch.int32, device=DEV))
    assert e.value.code == 1
    # whole-search offsets on a partitioned tree
    _, off_all = t.count(hd)
    t.set_partition(0, 2)
    with pytest.raises(P.BtreeError) as e:
        t.fill(hd, off_all)
    assert e.value.code == 1
    # the matching offsets still work
    t.set_partition(0, 1)
    c, off = t.count(hd)
    nb = t.fill(hd, off)
    assert nb.numel() == int(off[-1])
    # symmetric fill-only with gather offsets (counts differ where h varies)
    cs, offs = t.count(hd, symmetric=True)
    assert int(offs[-1]) > int(off[-1])
    with pytest.raises(P.BtreeError) as e:
        t.fill(hd, off, out=torch.empty(int(offs[-1]), dtype=torch.int32, device=DEV), symmetric=True)
    assert e.value.code == 1


def test_eq4_tie_and_leaf_order_on_gpu(P, oracle):
    """The oracle pins' hand-derived trees (test_oracle_pins: Eq. 4 tie r = beta
    halves; depth-first ascending-j leaf order) built by the CUDA path."""
    pos = _tie_set()
    h = np.full(len(pos), 0.3)
    for beta in (0.5, 0.5 + 2.0 ** -20, 0.5 - 2.0 ** -20):
        t, gpu = gpu_run(P, pos, h, s=8, beta=beta)
        ot = oracle.Tree(pos, 8, beta)
        assert_same_tree(t, ot)
        assert_same(gpu, ot.neighbors(h))
    assert P.build(torch.from_numpy(pos).to(DEV), 8, 0.5).stats()["root_b"] == 2
    assert P.build(torch.from_numpy(pos).to(DEV), 8, 0.5 + 2.0 ** -20).stats()["root_b"] == 4


def test_binding_rejects_bad_arguments(P):
    pos, h = datagen.make_config(1, n=2000)
    t = P.build(torch.from_numpy(pos).to(DEV))
    with pytest.raises(TypeError):
        t.count(torch.from_numpy(h))                                   # host tensor
    with pytest.raises(TypeError):
        t.count(torch.from_numpy(h).to(DEV).float())                   # float32
    with pytest.raises(ValueError):
        t.count(torch.from_numpy(h[:-1]).to(DEV))                      # wrong length
    with pytest.raises(ValueError):
        t.find_neighbors(torch.from_numpy(h).to(DEV), 4,
                         nbr_idx=torch.empty(10, dtype=torch.int32, device=DEV))  # below n * ngmax
    with pytest.raises(TypeError):
        P.build(torch.from_numpy(pos).to(DEV).reshape(-1))              # not [n, 3]
    with pytest.raises(ValueError):
        P.search_host(torch.from_numpy(pos), torch.from_numpy(h), capacity=100,
                      nbr=torch.empty(10, dtype=torch.int32))          # capacity above the buffer


def _sym_rows(P, pos, h, **kw):
    from test_gpu_parity import sort_rows
    t = P.build(torch.from_numpy(pos).to(DEV), kw.get("s", 64), 0.5)
    c, o, nb = t.find_neighbors(torch.from_numpy(h).to(DEV), symmetric=True)
    torch.cuda.synchronize()
    return t, (c.cpu().numpy(), o.cpu().numpy(), sort_rows(c, o, nb))


@pytest.mark.parametrize("case", ["boundary", "cfg5", "far_origin", "tiny_h", "h_spread"])
def test_symmetric_exact_only_identical(P, oracle, case):
    """Lemma L4s: the symmetric walk's fp32 decisions (two thresholds, one k
    per unit, candidate thresholds that cannot decide set to +inf) give the
    max(h_i, h_j) definition's sets, as the fp64 predicate alone does."""
    rng = np.random.default_rng(41)
    if case == "boundary":
        pos, h = datagen.near_boundary(2048, 64, 43)
        h = h * (1.0 + rng.integers(-2, 3, h.size) * 2.0 ** -50)  # thresholds within ulps of each other
    elif case == "cfg5":
        pos, h = datagen.make_config(5, n=200_000)
    elif case == "far_origin":
        pos, h = datagen.uniform(30_000, 47, 0.01, 0.03)
        pos = np.ascontiguousarray(pos + 1.0e4)
    elif case == "tiny_h":
        pos, h = datagen.uniform(20_000, 53, 1e-5, 3e-5)
        pos = np.ascontiguousarray(pos * 1e-3)
    else:  # a few huge-h particles among small ones: node h_max radii far above the unit's own
        pos, h = datagen.uniform(40_000, 59, 0.005, 0.01)
        h[rng.choice(h.size, 40, replace=False)] = 0.2
    h = np.ascontiguousarray(h)
    ref = oracle.brute_force(pos, h, symmetric=True) if pos.shape[0] <= 50_000 else None
    try:
        P.set_exact_only(True)
        _, g_exact = _sym_rows(P, pos, h)
    finally:
        P.set_exact_only(False)
    _, g_fast = _sym_rows(P, pos, h)
    assert_same(g_fast, g_exact)
    if ref is not None:
        assert_same(g_fast, ref)
    else:  # sampled rows against the symmetric brute force
        q = np.sort(rng.choice(pos.shape[0], 1500, replace=False)).astype(np.int64)
        rc, ro, ri = oracle.brute_force(pos, h, queries=q, symmetric=True)
        gc, go, gi = g_fast
        assert np.array_equal(gc[q], rc)
        for k, i in enumerate(q):
            assert np.array_equal(gi[go[i]:go[i + 1]], ri[ro[k]:ro[k + 1]])


@pytest.mark.parametrize("bad", [float("nan"), float("inf"), 0.0, -1.0, 1e200])
def test_count_rejects_bad_h(P, oracle, bad):
    """The count walk gathers h into tree order inside its descent (no
    separate gather launch): an h outside (0, 1e150] anywhere is still
    BT_ERR_INPUT before any arena grows for r = inf, and the tree stays
    usable (the next call with a valid h equals the oracle)."""
    pos, h = datagen.make_config(2, n=30_000)
    t = P.build(torch.from_numpy(pos).to(DEV))
    hb = h.copy()
    hb[12345] = bad
    with pytest.raises(P.BtreeError) as e:
        t.count(torch.from_numpy(hb).to(DEV))
    assert e.value.code == 2
    with pytest.raises(P.BtreeError) as e:
        t.find_neighbors(torch.from_numpy(hb).to(DEV), ngmax=512)
    assert e.value.code == 2
    c, o, nb = t.find_neighbors(torch.from_numpy(h).to(DEV), ngmax=512)
    assert_same((c.cpu().numpy(), o.cpu().numpy(), sort_rows(c, o, nb)), oracle.Tree(pos, 64).neighbors(h))


def test_fill_after_count_replays_record(P, oracle):
    """A count call (h gathered in the descent) followed by a fill-only call
    with the same h: the fill replays the recorded masks (no second descent
    or test pass), i.e. the fused checksum equals the gather kernel's."""
    pos, h = datagen.make_config(2, n=40_000)
    t = P.build(torch.from_numpy(pos).to(DEV))
    hd = torch.from_numpy(h).to(DEV)
    c, off = t.count(hd)
    P.profile_enable(True)
    try:
        P.profile_reset()
        nb = t.fill(hd, off)
        prof = P.profile()
    finally:
        P.profile_enable(False)
    assert "search.fill" in prof
    assert "search.desc" not in prof and "search.count" not in prof
    oc, ooff, oidx = oracle.Tree(pos, 64).neighbors(h)
    assert np.array_equal(off.cpu().numpy(), ooff)
    assert np.array_equal(sort_rows(c, off, nb), oidx)
