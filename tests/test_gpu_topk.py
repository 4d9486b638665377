"""GPU parity of the top-k sparsification (the step
before the sync): zen_sparsify_topk against the reference's own outputs
(tests/golden/topk.npz from oracle/_ref) and the C oracle, bit-exact --
including ties (lower index first), signs, -0.0 and exact zeros."""
import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def test_topk_golden(zen):
    g = load_golden("topk")
    for name in ["gauss", "ints"]:
        d = g[f"{name}_dense"]
        for f in g["fractions"]:
            key = f"{name}_{f}_idx"
            if key not in g:
                continue
            t = zen.sparsify_topk(d, float(f))
            np.testing.assert_array_equal(t.indices(), g[key], err_msg=f"{name} {f}")
            np.testing.assert_array_equal(t.values().view(np.uint32),
                                          g[f"{name}_{f}_val"].view(np.uint32))


@pytest.mark.parametrize("seed", range(6))
def test_topk_random_vs_oracle(zen, co, seed):
    rng = np.random.default_rng(seed)
    m = int(rng.integers(1, 300_000))
    kind = seed % 3
    if kind == 0:
        d = rng.standard_normal(m).astype(np.float32)
    elif kind == 1:  # heavy ties
        d = rng.integers(-3, 4, m).astype(np.float32)
    else:  # sparse rows with zeros and -0.0
        d = np.zeros(m, np.float32)
        nz = rng.choice(m, max(1, m // 50), replace=False)
        d[nz] = rng.standard_normal(nz.size).astype(np.float32)
        d[rng.choice(m, max(1, m // 100))] = -0.0
    for f in [1.0 / m, 0.001, 0.01, 0.2, 0.75, 1.0]:
        t = zen.sparsify_topk(d, f)
        wi, wv = co.sparsify_topk(d, f)
        np.testing.assert_array_equal(t.indices(), wi, err_msg=f"seed {seed} f {f}")
        np.testing.assert_array_equal(t.values().view(np.uint32), wv.view(np.uint32))


def test_topk_misaligned_and_device_input(zen, co):
    import torch
    rng = np.random.default_rng(5)
    base = torch.from_numpy(rng.standard_normal(100_003).astype(np.float32)).cuda()
    d = base[3:]  # 12-byte offset: the scalar path of every pass
    t = zen.sparsify_topk(d, 0.01)
    wi, wv = co.sparsify_topk(d.cpu().numpy(), 0.01)
    np.testing.assert_array_equal(t.indices(), wi)
    np.testing.assert_array_equal(t.values(), wv)


def test_topk_edges(zen):
    z = zen.sparsify_topk(np.zeros(1000, np.float32), 0.5)
    assert z.nnz() == 0 and z.universe() == 1000
    one = zen.sparsify_topk(np.array([0.0, -2.0, 2.0, 1.0], np.float32), 0.25)
    assert one.indices().tolist() == [1] and one.values().tolist() == [-2.0]  # tie -> lower index
    d = np.random.default_rng(1).standard_normal(4097).astype(np.float32)
    full = zen.sparsify_topk(d, 1.0)
    assert full == zen.to_sparse(zen.DenseTensor(d))
    for bad in [0.0, -0.5, 1.5]:
        with pytest.raises(zen.Error):
            zen.sparsify_topk(d, bad)


def test_topk_staging_edges(zen, co):
    """The tile pass stages the whole threshold bucket (top 11 key bits) and the
    lower digits are selected among the staged entries: a rank that falls
    among the zeros of bucket 0 (next to non-zero denormals), every entry in
    one bucket, and equal magnitudes everywhere."""
    rng = np.random.default_rng(23)
    m = 70_001
    den = np.zeros(m, np.float32)
    nz = rng.choice(m, 300, replace=False)
    den[nz] = (rng.integers(1, 1 << 20, nz.size).astype(np.uint32)).view(np.float32)
    den[nz[:50]] *= -1
    one_bucket = ((1.0 + 0.2 * rng.random(m)) * rng.choice([-1, 1], m)).astype(np.float32)
    equal = np.full(m, 0.5, np.float32) * rng.choice([-1, 1], m).astype(np.float32)
    for name, d in [("denormals", den), ("one_bucket", one_bucket), ("equal", equal)]:
        for f in [1.0 / m, 0.002, 0.01, 0.5, 1.0]:
            t = zen.sparsify_topk(d, f)
            wi, wv = co.sparsify_topk(d, f)
            np.testing.assert_array_equal(t.indices(), wi, err_msg=f"{name} {f}")
            np.testing.assert_array_equal(t.values().view(np.uint32), wv.view(np.uint32))


def test_topk_full_size_properties(zen):
    """64M-element embedding gradient (1M x 64, 1% rows live, Gaussian values),
    keep 0.5%: the kept set is exactly {|v| > T} plus the lowest-indexed
    T-ties, ascending."""
    import torch
    rows, width = 1_000_000, 64
    g = torch.zeros(rows, width, device="cuda")
    gen = torch.Generator(device="cuda").manual_seed(7)
    live = torch.randperm(rows, device="cuda", generator=gen)[:10_000]
    g[live] = torch.randn(10_000, width, device="cuda", generator=gen)
    d = g.view(-1)
    f = 0.005
    t = zen.sparsify_topk(d, f)
    keep = int(np.ceil(f * d.numel()))
    assert t.nnz() == keep
    idx = t.indices()
    assert np.all(np.diff(idx.astype(np.int64)) > 0)
    mag = d.abs()
    kept = torch.zeros(d.numel(), dtype=torch.bool, device="cuda")
    kept[torch.from_numpy(idx.view(np.int64)).cuda()] = True
    thr = mag[kept].min()
    assert float(mag[~kept].max()) <= float(thr)
    ties_out = torch.nonzero((~kept) & (mag == thr)).flatten()
    ties_in = torch.nonzero(kept & (mag == thr)).flatten()
    if ties_out.numel():
        assert int(ties_in.max()) < int(ties_out.min())
    np.testing.assert_array_equal(t.values(), d[kept].cpu().numpy())


def test_apply_sgd_after_sync(zen):
    """The step after the sync (f2): param[idx] -= lr * synced value, on the
    device, against a torch fp32 reference of the same update."""
    import torch
    rng = np.random.default_rng(11)
    m, n = 200_000, 3
    torch.cuda.set_stream(torch.cuda.Stream())
    dense = []
    for _ in range(n):
        d = np.zeros(m, np.float32)
        nz = rng.choice(m, 2000, replace=False)
        d[nz] = rng.standard_normal(nz.size).astype(np.float32)
        dense.append(torch.from_numpy(d).cuda())
    bp = zen.BPSynchronizer(n, m, max_nnz=8000)
    bp.sync_dense(dense)
    param = torch.from_numpy(rng.standard_normal(m).astype(np.float32)).cuda()
    want = param.clone()
    bp.apply_sgd(param, 0.05)
    idx, val = bp.result()
    want[idx] -= 0.05 * val  # torch fp32 reference (fma vs mul+sub: <= 1 ulp)
    torch.testing.assert_close(param, want, rtol=1e-6, atol=1e-7)
    torch.cuda.set_stream(torch.cuda.default_stream())


def test_axpy_sparse_many_rounds_and_range_error(zen):
    """zen_axpy_sparse over more entries than one round of the grid (4 per
    thread): param[idx] += alpha * val against torch fp32; an index >= M is
    reported as ZEN_E_INVALID."""
    import ctypes as C
    import torch
    lib, ctx = zen.load(), zen.context()
    m, cnt = 4_000_000, 2_500_001
    g = torch.Generator(device="cuda").manual_seed(3)
    idx = torch.randperm(m, device="cuda", generator=g)[:cnt].sort().values
    val = torch.randn(cnt, device="cuda", generator=g)
    param = torch.randn(m, device="cuda", generator=g)
    want = param.clone()
    want[idx] = torch.addcmul(want[idx], val, torch.full_like(val, -0.5))
    ctx.bind_stream()
    assert lib.zen_axpy_sparse(ctx.h, C.c_void_p(param.data_ptr()), m, C.c_void_p(idx.data_ptr()),
                               C.c_void_p(val.data_ptr()), cnt, C.c_float(-0.5)) == 0
    torch.cuda.synchronize()
    torch.testing.assert_close(param, want, rtol=1e-6, atol=1e-7)
    bad = idx.clone()
    bad[-1] = m
    assert lib.zen_axpy_sparse(ctx.h, C.c_void_p(param.data_ptr()), m, C.c_void_p(bad.data_ptr()),
                               C.c_void_p(val.data_ptr()), cnt, C.c_float(-0.5)) != 0
