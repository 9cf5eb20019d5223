"""GPU parity: the CUDA path (through the C ABI, libbtree.so) against the CPU
oracle, element by element, on seeded inputs.  Bit-exact: counts, offsets,
per-row-sorted neighbor lists, and the tree itself (leaf partition in
depth-first order, statistics) -- all integer results.

Run with ``pytest -m gpu`` on a B200.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1910_02639_b200 import datagen  # noqa: E402

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1910_02639_b200 as P
    P.lib()
    return P


def sort_rows(counts, offsets, nbr):
    """Sort each CSR row ascending (on the device; harness plumbing only)."""
    n = counts.numel()
    total = int(offsets[-1].item())
    if total == 0:
        return np.zeros(0, dtype=np.int32)
    rows = torch.repeat_interleave(torch.arange(n, device=counts.device, dtype=torch.int64),
                                   counts.to(torch.int64), output_size=total)
    key = rows * (1 << 32) + nbr[:total].to(torch.int64)
    key, _ = torch.sort(key)
    return (key & 0xFFFFFFFF).to(torch.int32).cpu().numpy()


def gpu_run(P, pos, h, s=64, beta=0.5, alpha=None, depth_cap=None, ngmax=None):
    t = P.build(torch.from_numpy(pos).to(DEV), s, beta, alpha=alpha, depth_cap=depth_cap)
    hd = torch.from_numpy(h).to(DEV)
    counts, offsets, nbr = t.find_neighbors(hd, ngmax)
    torch.cuda.synchronize()
    res = (counts.cpu().numpy(), offsets.cpu().numpy(), sort_rows(counts, offsets, nbr))
    return t, res


def assert_same(gpu, ref):
    gc, go, gi = gpu
    rc, ro, ri = ref
    assert gc.shape == rc.shape
    bad = np.nonzero(gc != rc)[0]
    assert bad.size == 0, f"{bad.size} counts differ, first rows {bad[:10]} gpu {gc[bad[:10]]} oracle {rc[bad[:10]]}"
    assert np.array_equal(go, ro)
    assert np.array_equal(gi, ri)


def assert_same_tree(t, otree):
    gs = t.stats()
    os_ = otree.stats()
    for k in ("nodes", "leaves", "halvings", "overfull", "max_leaf", "depth", "root_b"):
        assert gs[k] == os_[k], (k, gs[k], os_[k])
    perm, lb, lc, ld = t.order()
    operm, olb, olc, old = otree.order()
    assert np.array_equal(perm.cpu().numpy(), operm)
    assert np.array_equal(lb.cpu().numpy(), olb)
    assert np.array_equal(lc.cpu().numpy(), olc)
    assert np.array_equal(ld.cpu().numpy(), old)


# ---- the five configurations --------------------------------------------------
@pytest.mark.parametrize("cfg,n", [(1, None), (2, 200_003), (3, 216_000), (4, 300_001), (5, 400_000)])
def test_parity_scaled_configs(P, oracle, cfg, n):
    pos, h = datagen.make_config(cfg, n=n)
    t, gpu = gpu_run(P, pos, h, ngmax=datagen.NGMAX)
    ot = oracle.Tree(pos, 64, 0.5)
    assert_same(gpu, ot.neighbors(h))
    assert_same_tree(t, ot)
    st = t.stats()
    assert st["total_pairs"] == int(gpu[1][-1]) == int(gpu[0].sum())


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_parity_full_size_configs(P, oracle, cfg):
    pos, h = datagen.make_config(cfg)
    t, gpu = gpu_run(P, pos, h, ngmax=datagen.NGMAX)
    ot = oracle.Tree(pos, 64, 0.5)
    assert_same(gpu, ot.neighbors(h))
    assert_same_tree(t, ot)


def test_parity_cfg5_full_size_sampled(P, oracle):
    """cfg 5 at full size (2^25 particles) in the bench's launch configuration:
    counts of 40k sampled rows and their sorted rows against the oracle's own
    tree walk, 2k rows against brute force; invariants at every row."""
    pos, h = datagen.make_config(5)
    n = pos.shape[0]
    t = P.build(torch.from_numpy(pos).to(DEV), 64, 0.5)
    hd = torch.from_numpy(h).to(DEV)
    counts, offsets = t.count(hd)
    nbr = t.fill(hd, offsets)
    torch.cuda.synchronize()
    c = counts.cpu().numpy()
    off = offsets.cpu().numpy()
    assert off[0] == 0 and np.all(np.diff(off) == c) and off[-1] == c.sum()
    rng = np.random.default_rng(99)
    q = np.sort(rng.choice(n, 40_000, replace=False)).astype(np.int64)
    ot = oracle.Tree(pos, 64, 0.5)
    oc, ooff, oidx = ot.neighbors(h, queries=q)
    assert np.array_equal(c[q], oc)
    qd = torch.from_numpy(q).to(DEV)
    starts = offsets[qd]
    for k in range(0, q.size, 97):
        row = nbr[int(starts[k]):int(starts[k]) + int(oc[k])].cpu().numpy()
        assert np.array_equal(np.sort(row), oidx[ooff[k]:ooff[k + 1]])
    bc, _, _ = oracle.brute_force(pos, h, queries=q[:2000])
    assert np.array_equal(c[q[:2000]], bc)
    # the tree statistics of the full-size build equal the oracle's
    assert_same_tree(t, ot)


# ---- invariance, edge cases ------------------------------------------------------
def test_independent_of_bucket_size_and_beta(P, oracle):
    pos, h = datagen.clustered(30_000, 5, h=0.008)
    ref = oracle.Tree(pos, 64).neighbors(h)
    for s in (1, 2, 8, 64, 4096):
        for beta in (0.1, 0.5, 1.0):
            t, gpu = gpu_run(P, pos, h, s=s, beta=beta)
            assert_same(gpu, ref)
            assert_same_tree(t, oracle.Tree(pos, s, beta))
    t, gpu = gpu_run(P, pos, h, s=16, beta=0.5, alpha=0.0)
    assert_same(gpu, ref)
    assert_same_tree(t, oracle.Tree(pos, 16, 0.5, 0.0))


def test_near_boundary_adversarial(P, oracle):
    pos, h = datagen.near_boundary(1024, 64, 17)
    ref = oracle.brute_force(pos, h)
    for s in (8, 64):
        _, gpu = gpu_run(P, pos, h, s=s)
        assert_same(gpu, ref)


@pytest.mark.parametrize("two_h,interior", [(2.5, 80), (1.01, 6)])
def test_lattice_closed_form_gpu(P, oracle, two_h, interior):
    m = 20
    pos = datagen.lattice(m, 1.0)
    h = np.full(len(pos), two_h / 2)
    _, gpu = gpu_run(P, pos, h, s=8)
    assert_same(gpu, oracle.brute_force(pos, h))
    centre = (m // 2) * (m * m + m + 1)
    assert gpu[0][centre] == interior


def test_edge_cases(P, oracle):
    cases = []
    cases.append((np.zeros((1, 3)), np.array([0.1])))                      # n = 1
    p, hh = datagen.uniform(50, 3, 0.2)
    cases.append((p, hh))                                                  # n <= s: root leaf
    cases.append((np.tile([[0.3, 0.3, 0.3]], (300, 1)), np.full(300, 1e-3)))  # coincident, depth cap
    p, hh = datagen.uniform(5000, 4, 0.03)
    p[:, 2] = 0.5
    cases.append((p, hh))                                                  # plane: zero z extent
    p, hh = datagen.uniform(3000, 5, 2.0)
    cases.append((p, hh))                                                  # 2h > domain: n - 1 each
    p, _ = datagen.uniform(4000, 6, 0.01)
    hh = np.where(np.arange(4000) % 2 == 0, 0.2, 0.001)
    cases.append((p, np.ascontiguousarray(hh)))                            # strongly asymmetric h
    p, hh = datagen.uniform(1_000_003 // 10, 7, 0.02, 0.03)
    cases.append((p, hh))                                                  # ragged n
    for k, (p, hh) in enumerate(cases):
        for s in (8, 64):
            t, gpu = gpu_run(P, np.ascontiguousarray(p), np.ascontiguousarray(hh), s=s)
            ref = oracle.Tree(p, s).neighbors(hh)
            assert_same(gpu, ref)
            assert_same_tree(t, oracle.Tree(p, s))
    # 2h > domain -> every particle sees all others
    _, gpu = gpu_run(P, *datagen.uniform(3000, 5, 2.0))
    assert np.all(gpu[0] == 2999)


def test_empty_input(P):
    t = P.build(torch.zeros((0, 3), dtype=torch.float64, device=DEV))
    counts, offsets = t.count(torch.zeros(0, dtype=torch.float64, device=DEV))
    assert counts.numel() == 0 and int(offsets[0]) == 0
    assert t.stats()["leaves"] == 0


def test_count_then_fill_and_determinism(P):
    pos, h = datagen.make_config(2, n=100_000)
    t = P.build(torch.from_numpy(pos).to(DEV))
    hd = torch.from_numpy(h).to(DEV)
    c1, o1, n1 = t.find_neighbors(hd)             # count-only + exact fill
    c2, o2, n2 = t.find_neighbors(hd, ngmax=512)  # single call
    total = int(o1[-1])
    assert torch.equal(c1, c2) and torch.equal(o1, o2)
    assert torch.equal(n1[:total], n2[:total])    # same row order run to run
    t2 = P.build(torch.from_numpy(pos).to(DEV))
    _, _, n3 = t2.find_neighbors(hd, ngmax=512)
    assert torch.equal(n2[:total], n3[:total])


def test_errors(P):
    pos, h = datagen.uniform(2000, 8, 0.05)
    bad = pos.copy()
    bad[5, 1] = np.nan
    with pytest.raises(P.BtreeError) as e:
        P.build(torch.from_numpy(bad).to(DEV))
    assert e.value.code == 2
    with pytest.raises(P.BtreeError) as e:
        P.build(torch.from_numpy(pos).to(DEV), 0)
    assert e.value.code == 1
    with pytest.raises(P.BtreeError) as e:
        P.build(torch.from_numpy(pos).to(DEV), 8, 0.0)
    assert e.value.code == 1
    t = P.build(torch.from_numpy(pos).to(DEV), 8)
    hb = h.copy()
    hb[3] = 0.0
    with pytest.raises(P.BtreeError) as e:
        t.count(torch.from_numpy(hb).to(DEV))
    assert e.value.code == 2
    # capacity: counts/offsets valid, nbr untouched
    hd = torch.from_numpy(h).to(DEV)
    counts = torch.empty(2000, dtype=torch.int32, device=DEV)
    offsets = torch.empty(2001, dtype=torch.int64, device=DEV)
    nbr = torch.full((2000,), -7, dtype=torch.int32, device=DEV)
    with pytest.raises(P.BtreeError) as e:
        t.find_neighbors(hd, ngmax=1, counts=counts, offsets=offsets, nbr_idx=nbr)
    assert e.value.code == 3
    c_ref, o_ref = t.count(hd)
    assert torch.equal(counts, c_ref) and torch.equal(offsets, o_ref)
    assert bool((nbr == -7).all())


def test_search_host_end_to_end(P, oracle):
    pos, h = datagen.make_config(2, n=50_000)
    oc, ooff, oidx = oracle.Tree(pos, 64).neighbors(h)
    cap = int(ooff[-1])
    c, off, nbr = P.search_host(torch.from_numpy(pos), torch.from_numpy(h), capacity=cap)
    assert np.array_equal(c.numpy(), oc) and np.array_equal(off.numpy(), ooff)
    nb = nbr.numpy()
    for i in range(0, 50_000, 37):
        assert np.array_equal(np.sort(nb[off[i]:off[i + 1]]), oidx[ooff[i]:ooff[i + 1]])
    with pytest.raises(P.BtreeError) as e:
        P.search_host(torch.from_numpy(pos), torch.from_numpy(h), capacity=cap - 1)
    assert e.value.code == 3


# ---- the fp32 pre-test (lemma L4) decides nothing the fp64 predicate would not --
@pytest.mark.parametrize("case", ["boundary", "cfg2", "cfg5", "far_origin", "tiny_h"])
def test_exact_only_mode_identical(P, oracle, case):
    if case == "boundary":
        pos, h = datagen.near_boundary(2048, 64, 23)
    elif case == "cfg2":
        pos, h = datagen.make_config(2, n=150_000)
    elif case == "cfg5":
        pos, h = datagen.make_config(5, n=300_000)
    elif case == "far_origin":   # large |x| relative to h: wide fp32 error band
        pos, h = datagen.uniform(40_000, 29, 0.01, 0.02)
        pos = np.ascontiguousarray(pos + 1.0e4)
    else:                        # h so small that the fp32 squares underflow
        pos, h = datagen.uniform(20_000, 31, 1e-5)
        pos = np.ascontiguousarray(pos * 1e-3)
    ref = oracle.brute_force(pos, h) if pos.shape[0] <= 50_000 else oracle.Tree(pos, 64).neighbors(h)
    try:
        P.set_exact_only(True)
        _, g_exact = gpu_run(P, pos, h)
    finally:
        P.set_exact_only(False)
    t, g_fast = gpu_run(P, pos, h)
    assert_same(g_exact, ref)
    assert_same(g_fast, ref)
    st = t.stats()
    assert st["exact_tests"] <= st["tests"]


def test_fill_reuses_or_recomputes_record(P, oracle):
    pos, h = datagen.make_config(2, n=60_000)
    t = P.build(torch.from_numpy(pos).to(DEV))
    hd = torch.from_numpy(h).to(DEV)
    c, off = t.count(hd)
    nb = t.fill(hd, off)                      # reuses the recorded test pass
    ref = oracle.Tree(pos, 64).neighbors(h)
    assert_same((c.cpu().numpy(), off.cpu().numpy(), sort_rows(c, off, nb)), ref)
    h2 = h * 1.05
    hd2 = torch.from_numpy(h2).to(DEV)
    c2, off2 = t.count(hd2)
    hd.copy_(hd2)                             # same pointer, new values: must recompute
    nb2 = t.fill(hd, off2)
    ref2 = oracle.Tree(pos, 64).neighbors(h2)
    assert_same((c2.cpu().numpy(), off2.cpu().numpy(), sort_rows(c2, off2, nb2)), ref2)


@pytest.mark.parametrize("cfg,n", [(2, 100_000), (4, 200_000), (5, 300_000)])
def test_octree_policy_parity(P, oracle, cfg, n):
    pos, h = datagen.make_config(cfg, n=n)
    t = P.build(torch.from_numpy(pos).to(DEV), 64, 0.5, policy="octree")
    hd = torch.from_numpy(h).to(DEV)
    counts, offsets, nbr = t.find_neighbors(hd)
    gpu = (counts.cpu().numpy(), offsets.cpu().numpy(), sort_rows(counts, offsets, nbr))
    ot = oracle.Tree(pos, 64, 0.5, policy="octree")
    assert_same(gpu, ot.neighbors(h))
    assert_same_tree(t, ot)


# ---- rare walk paths: big-unit descent, scratch-full resume ----------------------
def test_big_unit_descent_pass(P, oracle):
    """s = 1 (one particle per leaf) and ~3000 neighbors per particle: units list
    more than 2048 candidate leaves, so the descent's global-frontier pass
    (desc_kernel<true>) redoes them; results must equal brute force."""
    pos, h = datagen.uniform(20_000, 41, 0.17)
    t, gpu = gpu_run(P, pos, h, s=1)
    assert t.stats()["big_units"] > 0
    assert_same(gpu, oracle.brute_force(pos, h))


def test_scratch_full_resume(P, oracle):
    """2h > domain with n = 6000: every unit stages all 6000 particles, more than
    the walk's per-warp scratch (4096), so staging stops, tests the full
    blocks and resumes; every particle sees the other n - 1."""
    pos, h = datagen.uniform(6000, 43, 2.0)
    t, gpu = gpu_run(P, pos, h, s=64)
    assert np.all(gpu[0] == 5999)
    assert_same(gpu, oracle.brute_force(pos, h))
    st = t.stats()
    assert st["staged"] == st["units"] * 6000  # every unit staged every particle


# ---- SPH density consumer (bt_density; reading R21) ------------------------------
# per-term error <= 1.2e-5 of a term's weight (fp32
# unit-relative coordinates, lemma L4's eps; SFU square root); with random
# signs over ~100 terms the relative error of rho is ~1.2e-5 (1.2e-4 if all
# aligned); measured max 4.3e-7, mean 8.5e-8 at cfg 5.  The max gate is the
# random-sign bound with margin; the mean gate (~12x the measured mean)
# catches a systematic accuracy regression.
DENSITY_RTOL = 2e-5
DENSITY_MEAN_RTOL = 1e-6


@pytest.mark.parametrize("cfg,n", [(1, None), (2, 100_000), (4, 100_000), (5, 200_000)])
def test_density_parity(P, oracle, cfg, n):
    pos, h = datagen.make_config(cfg, n=n)
    mass = np.random.default_rng(5).uniform(0.5, 1.5, len(pos))
    t = P.build(torch.from_numpy(pos).to(DEV))
    hd, md = torch.from_numpy(h).to(DEV), torch.from_numpy(mass).to(DEV)
    rho = t.density(hd, md).cpu().numpy()
    ref = oracle.Tree(pos, 64).density(h, mass)
    rel = np.abs(rho - ref) / ref
    assert rel.max() < DENSITY_RTOL, (rel.max(), int(rel.argmax()))
    assert rel.mean() < DENSITY_MEAN_RTOL, rel.mean()
    # the density walk records nothing: a later count + fill is still exact
    c, off, nb = t.find_neighbors(hd)
    ot = oracle.Tree(pos, 64)
    assert_same((c.cpu().numpy(), off.cpu().numpy(), sort_rows(c, off, nb)), ot.neighbors(h))


def test_density_exact_only_and_boundary(P, oracle):
    pos, h = datagen.near_boundary(512, 64, 29)
    mass = np.random.default_rng(6).uniform(0.5, 1.5, len(pos))
    ref = oracle.brute_density(pos, h, mass)
    t = P.build(torch.from_numpy(pos).to(DEV), 8)
    hd, md = torch.from_numpy(h).to(DEV), torch.from_numpy(mass).to(DEV)
    for exact in (False, True):
        try:
            P.set_exact_only(exact)
            rho = t.density(hd, md).cpu().numpy()
        finally:
            P.set_exact_only(False)
        assert (np.abs(rho - ref) / ref).max() < DENSITY_RTOL


def test_density_errors(P):
    pos, h = datagen.uniform(1000, 9, 0.05)
    t = P.build(torch.from_numpy(pos).to(DEV))
    m = np.ones(1000)
    m[7] = np.inf
    with pytest.raises(P.BtreeError) as e:
        t.density(torch.from_numpy(h).to(DEV), torch.from_numpy(m).to(DEV))
    assert e.value.code == 2


# ---- symmetric criterion (reading R22) -----------------------
def sym_union_ref(oracle, pos, h, s=64):
    """Oracle symmetric sets as N u N^T of the oracle's own tree walk (pinned
    equal to the symmetric brute force in test_oracle_pins); rows ascending."""
    c, off, idx = oracle.Tree(pos, s, 0.5).neighbors(h)
    n = len(pos)
    rows = np.repeat(np.arange(n, dtype=np.int64), c)
    cols = idx.astype(np.int64)
    key = np.unique(np.concatenate([rows * (1 << 32) + cols, cols * (1 << 32) + rows]))
    r = key >> 32
    counts = np.bincount(r, minlength=n).astype(np.int32)
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    return counts, offsets, (key & 0xFFFFFFFF).astype(np.int32)


def gpu_sym(P, pos, h, s=64, ngmax=None):
    t = P.build(torch.from_numpy(pos).to(DEV), s, 0.5)
    hd = torch.from_numpy(h).to(DEV)
    counts, offsets, nbr = t.find_neighbors(hd, ngmax, symmetric=True)
    torch.cuda.synchronize()
    return t, (counts.cpu().numpy(), offsets.cpu().numpy(), sort_rows(counts, offsets, nbr))


@pytest.mark.parametrize("cfg,n", [(1, None), (2, 100_000), (4, 100_000), (5, 200_000)])
def test_symmetric_parity(P, oracle, cfg, n):
    pos, h = datagen.make_config(cfg, n=n)
    _, gpu = gpu_sym(P, pos, h)
    ref = sym_union_ref(oracle, pos, h)
    assert_same(gpu, ref)
    if cfg == 1:  # the plain definition itself at cfg 1
        assert_same(gpu, oracle.brute_force(pos, h, symmetric=True))
    # gather sets are a subset; the relation is symmetric
    if cfg in (2, 4, 5):
        assert int(ref[1][-1]) > int(oracle.Tree(pos, 64).count(h).sum())


def test_symmetric_closed_forms_and_edges(P, oracle):
    # hand pair (0.6, 0.1) at d = 1, and the chain of test_symmetric_chain_closed_form
    pos = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    _, gpu = gpu_sym(P, pos, np.array([0.6, 0.1]), s=1)
    assert gpu[0].tolist() == [1, 1] and gpu[2].tolist() == [1, 0]
    m = 101
    pos = np.zeros((m, 3))
    pos[:, 0] = np.arange(m, dtype=np.float64)
    h = np.where(np.arange(m) % 2 == 0, 0.3, 0.55)
    for s in (1, 4, 64):
        _, gpu = gpu_sym(P, pos, h, s=s)
        expect = np.full(m, 2)
        expect[0] = expect[-1] = 1
        assert np.array_equal(gpu[0], expect)
        assert_same(gpu, oracle.brute_force(pos, h, symmetric=True))
    # constant h: identical to the gather result
    pos, h = datagen.make_config(3, n=50_000)
    _, g = gpu_run(P, pos, h)
    _, s_ = gpu_sym(P, pos, h)
    assert_same(s_, g)
    # n = 1 and the adversarial near-boundary set with variable h
    _, gpu = gpu_sym(P, np.zeros((1, 3)), np.array([1.0]))
    assert gpu[0].tolist() == [0]
    pos, h = datagen.near_boundary(64, 64, 77)
    h = h * np.random.default_rng(78).choice([1.0, 1.0 + 2.0 ** -50, 0.5], len(h))
    _, gpu = gpu_sym(P, pos, h)
    assert_same(gpu, oracle.brute_force(pos, h, symmetric=True))


def test_symmetric_one_call_capacity_and_reuse(P, oracle):
    pos, h = datagen.make_config(4, n=60_000)
    t = P.build(torch.from_numpy(pos).to(DEV))
    hd = torch.from_numpy(h).to(DEV)
    c1, o1, n1 = t.find_neighbors(hd, symmetric=True)              # count-only + exact fill
    c2, o2, n2 = t.find_neighbors(hd, ngmax=512, symmetric=True)   # single call
    assert torch.equal(c1, c2) and torch.equal(o1, o2)
    assert np.array_equal(sort_rows(c1, o1, n1), sort_rows(c2, o2, n2))
    # a gather call in between invalidates nothing the symmetric fill relies on
    cs, os_ = t.count(hd, symmetric=True)
    t.find_neighbors(hd, ngmax=512)
    t.density(hd, torch.ones_like(hd))
    n3 = t.fill(hd, os_, symmetric=True)
    assert np.array_equal(sort_rows(cs, os_, n3), sort_rows(c1, o1, n1))
    # capacity: counts/offsets valid, nbr untouched
    n = pos.shape[0]
    counts = torch.empty(n, dtype=torch.int32, device=DEV)
    offsets = torch.empty(n + 1, dtype=torch.int64, device=DEV)
    nbr = torch.full((n,), -7, dtype=torch.int32, device=DEV)
    with pytest.raises(P.BtreeError) as e:
        t.find_neighbors(hd, ngmax=1, counts=counts, offsets=offsets, nbr_idx=nbr, symmetric=True)
    assert e.value.code == 3
    assert torch.equal(counts, c1) and torch.equal(offsets, o1)
    assert bool((nbr == -7).all())
    ref = sym_union_ref(oracle, pos, h)
    assert_same((c1.cpu().numpy(), o1.cpu().numpy(), sort_rows(c1, o1, n1)), ref)


def test_symmetric_cfg5_full_size_sampled(P, oracle):
    """Symmetric criterion at full cfg 5 (2^25): counts of sampled rows and
    their sorted rows against the symmetric brute force; CSR invariants."""
    pos, h = datagen.make_config(5)
    n = pos.shape[0]
    t = P.build(torch.from_numpy(pos).to(DEV), 64, 0.5)
    hd = torch.from_numpy(h).to(DEV)
    counts, offsets = t.count(hd, symmetric=True)
    nbr = t.fill(hd, offsets, symmetric=True)
    torch.cuda.synchronize()
    c = counts.cpu().numpy()
    off = offsets.cpu().numpy()
    assert off[0] == 0 and np.all(np.diff(off) == c) and off[-1] == c.sum()
    cg, _ = t.count(hd)
    assert bool((counts >= cg).all()) and int(offsets[-1]) > int(cg.sum())
    rng = np.random.default_rng(199)
    q = np.sort(rng.choice(n, 300, replace=False)).astype(np.int64)
    bc, boff, bidx = oracle.brute_force(pos, h, queries=q, symmetric=True)
    assert np.array_equal(c[q], bc)
    for k in range(q.size):
        s0 = int(off[q[k]])
        row = nbr[s0:s0 + int(c[q[k]])].cpu().numpy()
        assert np.array_equal(np.sort(row), bidx[boff[k]:boff[k + 1]])


# ---- k = 2 policies (b-tree with b^2 sub-cells, quadtree; reading R23) -----------
def _plane(n, seed):
    rng = np.random.default_rng(seed)
    pos = np.zeros((n, 3))
    pos[:, :2] = rng.random((n, 2))
    h = 0.5 * np.sqrt(100.0 / (np.pi * n)) * rng.uniform(0.8, 1.2, n)  # ~100 neighbours in 2-D
    return pos, h


@pytest.mark.parametrize("policy", ["btree2d", "quadtree"])
@pytest.mark.parametrize("case", ["plane", "cfg2", "cfg5"])
def test_k2_policy_parity(P, oracle, policy, case):
    if case == "plane":
        pos, h = _plane(200_003, 7)
    elif case == "cfg2":
        pos, h = datagen.make_config(2, n=100_000)
    else:
        pos, h = datagen.make_config(5, n=200_000)
    t = P.build(torch.from_numpy(pos).to(DEV), 64, 0.5, policy=policy)
    hd = torch.from_numpy(h).to(DEV)
    counts, offsets, nbr = t.find_neighbors(hd)
    gpu = (counts.cpu().numpy(), offsets.cpu().numpy(), sort_rows(counts, offsets, nbr))
    ot = oracle.Tree(pos, 64, 0.5, policy=policy)
    assert_same(gpu, ot.neighbors(h))
    assert_same_tree(t, ot)


def test_k2_plane_lattice_and_halving(P, oracle):
    # the oracle-pinned shapes: 16^2 plane lattice at s = 4 (depth 1, b = 8) and
    # the 12 -> 6 -> 3 -> 2 halving sequence; 2-D lattice closed form: 2h = 2.5
    # gives the 20 integer offsets with a^2 + b^2 <= 6 in the interior
    g = np.arange(16, dtype=np.float64)
    gx, gy = np.meshgrid(g, g, indexing="ij")
    pos = np.ascontiguousarray(np.stack([gx.ravel(), gy.ravel(), np.zeros(256)], axis=1))
    for pol in ("btree2d", "quadtree"):
        t = P.build(torch.from_numpy(pos).to(DEV), 4, 0.5, policy=pol)
        assert_same_tree(t, oracle.Tree(pos, 4, 0.5, policy=pol))
        hd = torch.full((256,), 1.25, dtype=torch.float64, device=DEV)
        c = t.count(hd)[0].cpu().numpy().reshape(16, 16)
        assert np.all(c[2:-2, 2:-2] == 20)
    rng = np.random.default_rng(4)
    pts = rng.random((1000, 3)) * np.array([0.01, 0.01, 1.0])
    pos = np.concatenate([pts, [[1.0, 1.0, 1.0]]])
    t = P.build(torch.from_numpy(pos).to(DEV), 8, 0.5, policy="btree2d")
    ot = oracle.Tree(pos, 8, 0.5, policy="btree2d")
    assert t.stats()["root_b"] == 2
    assert_same_tree(t, ot)
    with pytest.raises(ValueError):
        P.build(torch.from_numpy(pos).to(DEV), 8, 0.5, policy="k3")


# ---- replicated-tree partition (SURVEY 8(e) variant (i), bt_set_partition) -------
@pytest.mark.parametrize("cfg,n,nparts", [(2, 100_000, 3), (4, 100_000, 2), (5, 200_000, 5)])
def test_partitioned_search_is_a_disjoint_cover(P, oracle, cfg, n, nparts):
    """Each part's search returns exactly the full rows of its particles and
    empty rows elsewhere; the parts are disjoint and cover all particles (the
    density written per part marks membership)."""
    pos, h = datagen.make_config(cfg, n=n)
    t = P.build(torch.from_numpy(pos).to(DEV))
    hd = torch.from_numpy(h).to(DEV)
    mass = torch.ones_like(hd)
    fc, fo, fn = t.find_neighbors(hd)
    full_rows = sort_rows(fc, fo, fn)
    full_rho = t.density(hd, mass)
    sc, so, sn = t.find_neighbors(hd, symmetric=True)
    sym_rows = sort_rows(sc, so, sn)
    scn = sc.cpu().numpy()
    ref = oracle.Tree(pos, 64, 0.5).neighbors(h)
    assert_same((fc.cpu().numpy(), fo.cpu().numpy(), full_rows), ref)
    owner = np.full(n, -1)
    fcn = fc.cpu().numpy()
    for p in range(nparts):
        t.set_partition(p, nparts)
        rho = torch.full_like(hd, float("nan"))
        t.density(hd, mass, out=rho)
        mine = ~torch.isnan(rho).cpu().numpy()
        assert np.all(owner[mine] == -1)
        owner[mine] = p
        torch.testing.assert_close(rho[torch.from_numpy(mine).to(DEV)], full_rho[torch.from_numpy(mine).to(DEV)],
                                   rtol=0, atol=0)
        c, o, nb = t.find_neighbors(hd)
        cn = c.cpu().numpy()
        assert np.array_equal(cn[mine], fcn[mine]) and not np.any(cn[~mine])
        # the part's sorted rows are the full rows of its particles
        rows = sort_rows(c, o, nb)
        keep = np.repeat(mine, fcn)
        assert np.array_equal(rows, full_rows[keep])
        # the symmetric criterion is searched from the query side too: a part
        # returns the full symmetric rows of its particles
        c, o, nb = t.find_neighbors(hd, symmetric=True)
        cn = c.cpu().numpy()
        assert np.array_equal(cn[mine], scn[mine]) and not np.any(cn[~mine])
        assert np.array_equal(sort_rows(c, o, nb), sym_rows[np.repeat(mine, scn)])
    assert np.all(owner >= 0)
    t.set_partition(0, 1)
    c, o, nb = t.find_neighbors(hd)
    assert np.array_equal(sort_rows(c, o, nb), full_rows)
    with pytest.raises(P.BtreeError):
        t.set_partition(2, 2)


def test_parity_cfg5_full_size_every_row(P, oracle):
    """cfg 5 at full size (2^25 particles): every count against the oracle's
    own tree walk (memcmp), and every row, compared sorted in chunks of 2^21
    queries (the oracle recomputes each chunk) -- the whole 4.35e9-pair CSR."""
    pos, h = datagen.make_config(5)
    n = pos.shape[0]
    t = P.build(torch.from_numpy(pos).to(DEV), 64, 0.5)
    hd = torch.from_numpy(h).to(DEV)
    counts, offsets = t.count(hd)
    nbr = t.fill(hd, offsets)
    torch.cuda.synchronize()
    t.free()
    ot = oracle.Tree(pos, 64, 0.5)
    oc = ot.count(h)
    c = counts.cpu().numpy()
    assert np.array_equal(c, oc)
    chunk = 1 << 21
    for q0 in range(0, n, chunk):
        q1 = min(n, q0 + chunk)
        _, ooff, oidx = ot.neighbors(h, queries=np.arange(q0, q1, dtype=np.int64))
        s0, s1 = int(offsets[q0]), int(offsets[q1])
        sub_off = offsets[q0:q1 + 1] - s0
        rows = sort_rows(counts[q0:q1], sub_off, nbr[s0:s1])
        assert np.array_equal(rows, oidx), f"rows {q0}..{q1} differ"


def test_rows_over_ngmax_stat(P, oracle):
    # bt_tree_stats reports the rows above the call's ngmax (counts never clamped)
    pos, h = datagen.make_config(5, n=200_000)
    t = P.build(torch.from_numpy(pos).to(DEV))
    hd = torch.from_numpy(h).to(DEV)
    c, _ = t.count(hd, ngmax=100)
    cn = c.cpu().numpy()
    st = t.stats()
    assert st["rows_over_ngmax"] == int((cn > 100).sum()) and st["max_count"] == int(cn.max())
    t.count(hd, ngmax=int(cn.max()))
    assert t.stats()["rows_over_ngmax"] == 0
    cs, _ = t.count(hd, symmetric=True, ngmax=100)
    assert t.stats()["rows_over_ngmax"] == int((cs.cpu().numpy() > 100).sum())
