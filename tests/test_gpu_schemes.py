"""GPU parity of SURVEY.md §8f row f3: zen_merge_sum, Hierarchical
Centralization, the tensor metrics, profile_sparsity and select_scheme, against
the reference's own outputs (tests/golden/hc.npz from oracle/_ref) and the C
oracle.  Bit-exact: indices, fp32 value bits, the SimNet ledger, and the
double-precision profile."""
import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

KINDS = {1: "coo", 2: "bitmap", 3: "tensor_block"}


def _fmt(zen, k, bs, cb):
    k = KINDS[int(k)]
    if k == "coo":
        return zen.WireFormat.coo(int(cb))
    if k == "bitmap":
        return zen.WireFormat.bitmap()
    return zen.WireFormat.tensor_block(int(bs))


def _case(zen, g, c):
    m, n = (int(x) for x in g[f"c{c}_m"])
    return m, n, [zen.SparseTensor(m, g[f"c{c}_in{w}_idx"], g[f"c{c}_in{w}_val"])
                  for w in range(n)]


def _ledger(rep, n):
    return np.array([[s.sent_bits, s.recv_bits, s.recv_index_bits, s.recv_value_bits]
                     for s in rep.stages], np.uint64).reshape(len(rep.stages), 4, n)


def test_hier_centralization_golden(zen):
    g = load_golden("hc")
    for c in range(int(g["ncases"][0])):
        m, n, ins = _case(zen, g, c)
        for f, row in enumerate(g["formats"]):
            out = zen.run_hier_centralization(ins, zen.SimNet(n, 1.0), _fmt(zen, *row))
            assert len(out.results) == n
            want = zen.SparseTensor(m, g[f"c{c}_f{f}_idx"], g[f"c{c}_f{f}_val"])
            for r in out.results:
                assert r == want, f"case {c} format {f}"
            np.testing.assert_array_equal(_ledger(out.traffic, n), g[f"c{c}_f{f}_ledger"])


def test_merge_sum_golden(zen):
    g = load_golden("hc")
    for c in range(int(g["ncases"][0])):
        m, n, ins = _case(zen, g, c)
        r = zen.merge_sum(ins[0], ins[1])
        assert r == zen.SparseTensor(m, g[f"c{c}_merge_idx"], g[f"c{c}_merge_val"])


def test_metrics_profile_selector_golden(zen):
    g = load_golden("hc")
    for c in range(int(g["ncases"][0])):
        if f"c{c}_profile" not in g:
            continue
        m, n, ins = _case(zen, g, c)
        met = g[f"c{c}_metrics"]
        assert zen.overlap_ratio(ins[0], ins[1]) == met[0]
        assert zen.densification_ratio(ins) == met[1]
        assert zen.skewness_ratio(ins[0], n) == met[2]
        p = zen.profile_sparsity([ins, list(reversed(ins))])
        want = g[f"c{c}_profile"]
        assert p.d == want[0] and p.skew[n] == want[1]
        for j in range(5):
            if not np.isnan(want[3 + j]):
                assert p.gamma[1 << j] == want[3 + j]
        choice = zen.select_scheme(p, n)
        assert choice == (zen.BALANCED_PARALLELISM if want[2] == 0
                          else zen.HIERARCHICAL_CENTRALIZATION)


@pytest.mark.parametrize("seed", range(4))
def test_hier_centralization_random_vs_reference(zen, co, seed):
    """Random power-of-two n, densities and overlaps (schemes_test.cpp:110-119
    style) against the C oracle's restatement."""
    rng = np.random.default_rng(300 + seed)
    n = 1 << int(rng.integers(1, 5))
    m = int(rng.integers(1000, 200_000))
    ins, raw = [], []
    core = rng.choice(m, max(1, m // 200), replace=False)
    for w in range(n):
        own = rng.choice(m, max(1, m // 100), replace=False)
        idx = np.unique(np.concatenate([core, own])).astype(np.uint64)
        val = rng.standard_normal(idx.size).astype(np.float32)
        raw.append((idx, val))
        ins.append(zen.SparseTensor(m, idx, val))
    for kind, fmt in [("coo", zen.WireFormat.coo()), ("tensor_block", zen.WireFormat.tensor_block(256))]:
        out = zen.run_hier_centralization(ins, zen.SimNet(n, 1.0), fmt)
        wi, wv, led = co.hier_centralization(m, raw, kind, 256)
        for r in out.results:
            np.testing.assert_array_equal(r.indices(), wi)
            np.testing.assert_array_equal(r.values().view(np.uint32), wv.view(np.uint32))
        np.testing.assert_array_equal(_ledger(out.traffic, n), led)


def test_hier_centralization_edges(zen):
    m = 1000
    six = [zen.SparseTensor(m, [w], [1.0]) for w in range(6)]
    with pytest.raises(zen.NonPowerOfTwo):
        zen.run_hier_centralization(six, zen.SimNet(6, 1.0))
    empty = [zen.SparseTensor(m) for _ in range(4)]
    out = zen.run_hier_centralization(empty, zen.SimNet(4, 1.0))
    assert all(r.nnz() == 0 for r in out.results)
    assert out.traffic.total_recv_bits == 0
    one = [zen.SparseTensor(m, [7], [1.5])] + [zen.SparseTensor(m) for _ in range(3)]
    out = zen.run_hier_centralization(one, zen.SimNet(4, 1.0))
    assert all(r == one[0] for r in out.results)
    with pytest.raises(zen.UniverseMismatch):
        zen.merge_sum(zen.SparseTensor(10, [1], [1.0]), zen.SparseTensor(11, [1], [1.0]))
    with pytest.raises(zen.Error):
        zen.run_hier_centralization([zen.SparseTensor(5, [1], [1.0])] * 2, zen.SimNet(2, 1.0),
                                    zen.WireFormat.hash_bitmap())
    p = zen.SparsityProfile(0.01, {1: 1.0, 2: 1.5}, {})
    with pytest.raises(zen.MissingProfileEntry):
        zen.select_scheme(p, 4)
    with pytest.raises(zen.NonPowerOfTwo):
        zen.t_hc_coefficient(6, {})


def test_merge_sum_full_size_properties(zen):
    """Two 16M-entry tensors over M = 2^40 (64-bit indices): the union is the
    sorted set union, shared values are the fp32 pair sums (torch reference),
    the others pass through unchanged."""
    import ctypes as C
    import torch
    from paper_2309_13254_b200 import schemes
    g = torch.Generator(device="cuda").manual_seed(3)
    m = 1 << 40
    z = 16 << 20
    a = torch.unique(torch.randint(0, 1 << 26, (z,), device="cuda", generator=g)) << 14
    b = torch.unique(torch.randint(0, 1 << 26, (z,), device="cuda", generator=g)) << 14
    av = torch.randn(a.numel(), device="cuda", generator=g)
    bv = torch.randn(b.numel(), device="cuda", generator=g)
    oi, ov = schemes._merge_dev(a, av, b, bv, m)
    want_i, inv = torch.unique(torch.cat([a, b]), return_inverse=True)
    want_v = torch.zeros(want_i.numel(), device="cuda").index_add_(0, inv, torch.cat([av, bv]))
    assert torch.equal(oi, want_i)
    assert torch.equal(ov.view(torch.int32), want_v.view(torch.int32))
    # out-of-order input is rejected, not merged
    with pytest.raises(zen.Error):
        schemes._merge_dev(a.flip(0), av, b, bv, m)


def test_hc_rank_api_single_rank(zen):
    """zen_hc with n = 1 (no stage): the result is to_sparse of the input; the
    n > 1 NVLink path runs in tests/mgpu_worker.py (test_multi_gpu.py)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(9)
    d = torch.zeros(1 << 20, device="cuda")
    live = torch.randperm(1 << 20, device="cuda", generator=g)[:5000]
    d[live] = torch.randn(5000, device="cuda", generator=g)
    torch.cuda.set_stream(torch.cuda.Stream())
    hc = zen.HCSynchronizer(1, d.numel(), 0, max_nnz=8192)
    hc.connect([hc.ipc_handle()])
    want = zen.to_sparse(d)
    for _ in range(3):
        hc.sync_dense(d)
        i, v = hc.result()
        assert np.array_equal(i.cpu().numpy().view(np.uint64), want.indices())
        assert np.array_equal(v.cpu().numpy(), want.values())
    assert hc.stage_bits() == []
    with pytest.raises(zen.NonPowerOfTwo):
        zen.HCSynchronizer(3, 100, 0, max_nnz=10)
    with pytest.raises(zen.Error):
        hc.sync_sparse(torch.tensor([5, 3], device="cuda"), torch.ones(2, device="cuda"))
        hc.wait()
    torch.cuda.set_stream(torch.cuda.default_stream())


# ---- f4: the baseline schemes on the GPU (run_scheme) ----

def _scheme_cfg(zen, name, comm, kind, bs):
    cfg = zen.scheme_config_from_name(name)
    if comm is not None:
        cfg.communication = comm
    if kind == "coo32":
        cfg.format = zen.WireFormat.coo(32)
    elif kind == "bitmap":
        cfg.format = zen.WireFormat.bitmap()
    elif kind == "tensor_block":
        cfg.format = zen.WireFormat.tensor_block(bs)
    return cfg


def test_baseline_schemes_golden(zen):
    """run_scheme for AGsparse (3 patterns), SparCML, ring centralization and
    OmniReduce-like against the reference's own outputs: every node's result
    (fp32 bits), the SimNet ledger and the balance."""
    from make_golden import SCHEME_RUNS
    g = load_golden("schemes")
    for c in range(int(g["ncases"][0])):
        m, n = (int(x) for x in g[f"c{c}_m"])
        ins = [zen.SparseTensor(m, g[f"c{c}_in{w}_idx"], g[f"c{c}_in{w}_val"]) for w in range(n)]
        for r, (name, comm, kind, bs) in enumerate(SCHEME_RUNS):
            out = zen.run_scheme(_scheme_cfg(zen, name, comm, kind, bs), ins, zen.SimNet(n, 1.0))
            for w in range(n):
                want = zen.SparseTensor(m, g[f"c{c}_r{r}_w{w}_idx"], g[f"c{c}_r{r}_w{w}_val"])
                assert out.results[w] == want, f"case {c} {name} {comm} {kind} node {w}"
            np.testing.assert_array_equal(_ledger(out.traffic, n), g[f"c{c}_r{r}_ledger"])
            key = f"c{c}_r{r}_balance"
            assert (out.balance is None) == (key not in g)
            if out.balance is not None:
                assert (out.balance.push_imbalance, out.balance.pull_imbalance) == tuple(g[key])


def test_scheme_dispatch_and_errors(zen):
    m = 1000
    ins = [zen.SparseTensor(m, [w, 500 + w], [1.0, 2.0]) for w in range(4)]
    assert set(zen.KNOWN_SCHEME_NAMES) == {"agsparse", "sparcml", "ring-centralization",
                                           "omnireduce", "balanced-parallelism"}
    bp = zen.run_scheme(zen.scheme_config_from_name("balanced-parallelism"), ins,
                        zen.SimNet(4, 1.0))
    ag = zen.run_scheme(zen.scheme_config_from_name("agsparse"), ins, zen.SimNet(4, 1.0))
    assert bp.results[0] == ag.results[0]
    with pytest.raises(zen.UnsupportedCombination):
        zen.scheme_config_from_name("nope")
    bad = zen.scheme_config_from_name("agsparse")
    bad.balance = zen.BalancePattern.Balanced
    with pytest.raises(zen.UnsupportedCombination):
        zen.run_scheme(bad, ins, zen.SimNet(4, 1.0))
    p2p_inc = zen.scheme_config_from_name("sparcml")
    p2p_inc.communication = zen.CommPattern.PointToPoint
    with pytest.raises(zen.UnsupportedCombination):
        zen.run_scheme(p2p_inc, ins, zen.SimNet(4, 1.0))
    three = [zen.SparseTensor(m, [w], [1.0]) for w in range(3)]
    for name in ["ring-centralization", "sparcml"]:
        with pytest.raises(zen.NonPowerOfTwo):
            zen.run_scheme(zen.scheme_config_from_name(name), three, zen.SimNet(3, 1.0))
    om = zen.run_omnireduce_like(three, zen.SimNet(3, 1.0), 16)  # any n
    assert om.results[0].nnz() == 3
    with pytest.raises(zen.Error):
        zen.run_omnireduce_like(three, zen.SimNet(3, 1.0), 0)
