"""GPU tests of the tree-order index space (bt_set_tree_order / bt_reorder):
the paper's walk optimisation (1), "particles are reordered in memory along
this curve".  Expected values are the oracle's caller-order results
mapped through the tree's permutation.  Run with ``pytest -m gpu``."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1910_02639_b200 import datagen  # noqa: E402

from test_gpu_parity import DENSITY_RTOL, DEV, sort_rows, sym_union_ref  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1910_02639_b200 as P
    P.lib()
    return P


def to_tree(ref, perm):
    """Caller-order CSR (counts, offsets, rows ascending) -> tree order: row k
    = {iperm[j] : j in N(perm[k])}, rows ascending."""
    c, _, idx = ref
    n = len(c)
    iperm = np.empty(n, dtype=np.int64)
    iperm[perm] = np.arange(n)
    rows = iperm[np.repeat(np.arange(n), c)]
    key = np.sort(rows * (1 << 32) + iperm[idx.astype(np.int64)])
    ct = np.asarray(c)[perm].astype(np.int32)
    ot = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(ct, out=ot[1:])
    return ct, ot, (key & 0xFFFFFFFF).astype(np.int32)


def tree_run(P, t, h, **kw):
    hd = torch.from_numpy(h).to(DEV)
    ht = t.reorder(hd)
    c, o, nb = t.find_neighbors(ht, **kw)
    torch.cuda.synchronize()
    return c.cpu().numpy(), o.cpu().numpy(), sort_rows(c, o, nb)


def assert_csr(got, exp):
    assert np.array_equal(got[0], exp[0])
    assert np.array_equal(got[1], exp[1])
    assert np.array_equal(got[2], exp[2])


@pytest.mark.parametrize("cfg,n", [(1, None), (2, 100_000), (3, 125_000), (4, 100_000), (5, 200_000)])
def test_tree_order_gather_parity(P, oracle, cfg, n):
    pos, h = datagen.make_config(cfg, n=n)
    t = P.build(torch.from_numpy(pos).to(DEV)).set_tree_order(True)
    perm = t.order()[0].cpu().numpy()
    assert_csr(tree_run(P, t, h), to_tree(oracle.Tree(pos, 64).neighbors(h), perm))


def test_tree_order_is_the_reordered_input(P):
    """Tree order on pos equals the default search of pos[perm] (whose own
    tree has the identity permutation)."""
    pos, h = datagen.make_config(5, n=150_000)
    t = P.build(torch.from_numpy(pos).to(DEV)).set_tree_order(True)
    perm = t.order()[0].cpu().numpy()
    got = tree_run(P, t, h)
    t2 = P.build(torch.from_numpy(np.ascontiguousarray(pos[perm])).to(DEV))
    assert np.array_equal(t2.order()[0].cpu().numpy(), np.arange(len(pos)))
    c, o, nb = t2.find_neighbors(torch.from_numpy(np.ascontiguousarray(h[perm])).to(DEV))
    assert_csr(got, (c.cpu().numpy(), o.cpu().numpy(), sort_rows(c, o, nb)))


def test_tree_order_symmetric_and_density(P, oracle):
    pos, h = datagen.make_config(4, n=100_000)
    mass = np.random.default_rng(5).uniform(0.5, 1.5, len(pos))
    t = P.build(torch.from_numpy(pos).to(DEV))
    hd, md = torch.from_numpy(h).to(DEV), torch.from_numpy(mass).to(DEV)
    rho_caller = t.density(hd, md)
    t.set_tree_order(True)
    perm_d = t.order()[0]
    perm = perm_d.cpu().numpy()
    ht, mt = t.reorder(hd), t.reorder(md)
    # symmetric criterion
    c, o, nb = t.find_neighbors(ht, symmetric=True)
    assert_csr((c.cpu().numpy(), o.cpu().numpy(), sort_rows(c, o, nb)), to_tree(sym_union_ref(oracle, pos, h), perm))
    # density: the same walk in the same order, so bit-identical to caller order mapped
    rho_t = t.density(ht, mt)
    assert torch.equal(rho_t, rho_caller[perm_d.long()])
    ref = oracle.Tree(pos, 64).density(h, mass)[perm]
    assert (np.abs(rho_t.cpu().numpy() - ref) / ref).max() < DENSITY_RTOL


def test_tree_order_fill_only_record_and_mode_switch(P, oracle):
    pos, h = datagen.make_config(2, n=60_000)
    t = P.build(torch.from_numpy(pos).to(DEV))
    perm = t.order()[0].cpu().numpy()
    hd = torch.from_numpy(h).to(DEV)
    ref = oracle.Tree(pos, 64).neighbors(h)
    c_c, off_c = t.count(hd)
    t.set_tree_order(True)
    ht = t.reorder(hd)
    c_t, off_t = t.count(ht)
    assert np.array_equal(c_t.cpu().numpy(), ref[0][perm])
    P.profile_enable(True)
    try:
        P.profile_reset()
        nb = t.fill(ht, off_t)  # replays the tree-order count pass
        prof = P.profile()
    finally:
        P.profile_enable(False)
    assert "search.count" not in prof
    assert_csr((c_t.cpu().numpy(), off_t.cpu().numpy(), sort_rows(c_t, off_t, nb)), to_tree(ref, perm))
    # caller-order offsets in tree order: not this space's scan -> BT_ERR_ARG
    with pytest.raises(P.BtreeError) as e:
        t.fill(ht, off_c)
    assert e.value.code == 1
    # back to caller order: the record of the other space is not reused
    t.set_tree_order(False)
    nb = t.fill(hd, off_c)
    assert_csr((c_c.cpu().numpy(), off_c.cpu().numpy(), sort_rows(c_c, off_c, nb)), ref)


@pytest.mark.parametrize("nparts", [3])
def test_tree_order_partitions(P, oracle, nparts):
    """Parts in tree order: each part's rows are its particles' full rows, and
    a part's particles are a contiguous run of whole units (rows of other
    parts empty)."""
    pos, h = datagen.make_config(5, n=120_000)
    t = P.build(torch.from_numpy(pos).to(DEV)).set_tree_order(True)
    perm = t.order()[0].cpu().numpy()
    exp = to_tree(oracle.Tree(pos, 64).neighbors(h), perm)
    ht = t.reorder(torch.from_numpy(h).to(DEV))
    seen = np.zeros(len(pos), dtype=bool)
    for p in range(nparts):
        t.set_partition(p, nparts)
        c, o, nb = t.find_neighbors(ht)
        cn = c.cpu().numpy()
        mine = cn > 0
        assert not np.any(seen & mine)
        seen |= mine
        assert np.array_equal(cn[mine], exp[0][mine])
        assert np.array_equal(sort_rows(c, o, nb), exp[2][np.repeat(mine, exp[0])])
    assert np.array_equal(seen, exp[0] > 0)


def test_reorder(P):
    pos, h = datagen.make_config(3, n=50_000)
    pd = torch.from_numpy(pos).to(DEV)
    t = P.build(pd)
    perm = t.order()[0].long()
    assert torch.equal(t.reorder(pd), pd[perm])
    hd = torch.from_numpy(h).to(DEV)
    assert torch.equal(t.reorder(hd), hd[perm])
    x = torch.randn(len(pos), 7, dtype=torch.float64, device=DEV)
    assert torch.equal(t.reorder(x), x[perm])
    with pytest.raises(ValueError):
        t.reorder(hd, out=hd)
    with pytest.raises(ValueError):
        t.reorder(hd[:-1])
    with pytest.raises(P.BtreeError):
        t.reorder(torch.zeros(len(pos), 17, dtype=torch.float64, device=DEV))


def test_tree_order_cfg5_full_size_sampled(P, oracle):
    """cfg 5 at full size in tree order (the bench's reordered leg): every
    count against the oracle's mapped through perm, 20k sampled rows."""
    pos, h = datagen.make_config(5)
    n = pos.shape[0]
    t = P.build(torch.from_numpy(pos).to(DEV), 64, 0.5).set_tree_order(True)
    perm = t.order()[0].cpu().numpy()
    ht = t.reorder(torch.from_numpy(h).to(DEV))
    counts, offsets = t.count(ht)
    nbr = t.fill(ht, offsets)
    torch.cuda.synchronize()
    t.free()
    ot = oracle.Tree(pos, 64, 0.5)
    assert np.array_equal(counts.cpu().numpy(), ot.count(h)[perm])
    rng = np.random.default_rng(7)
    k = np.sort(rng.choice(n, 20_000, replace=False))
    q = perm[k].astype(np.int64)
    order = np.argsort(q)
    oc, ooff, oidx = ot.neighbors(h, queries=q[order])
    iperm = np.empty(n, dtype=np.int64)
    iperm[perm] = np.arange(n)
    off = offsets.cpu().numpy()
    for r, kk in enumerate(k[order]):
        row = nbr[int(off[kk]):int(off[kk + 1])].cpu().numpy()
        assert np.array_equal(np.sort(row), np.sort(iperm[oidx[ooff[r]:ooff[r + 1]]]))
