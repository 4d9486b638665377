"""Mixed sparse / top-k / dense buckets through the
product API (paper_2309_13254_b200.buckets.MixedBucketSync), checked against
the oracle: the sparse bucket is to_sparse (n = 1), the top-k bucket is
zen::sparsify_topk (zen/workload.hpp:158-178), the dense bucket is the
all-reduced sum, and the SGD step applies the synced gradients."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")


def test_allreduce_dense_time_bits():
    """zen::allreduce_dense_time_bits (experiment.hpp:161-169): 2(n-1)/n * M
    elements at b/32 elements per time unit; 0 for a single node."""
    import paper_2309_13254_b200 as zen
    assert zen.allreduce_dense_time_bits(4, 1000, 32.0) == 1500.0
    assert zen.allreduce_dense_time_bits(1, 1000, 32.0) == 0.0
    assert zen.allreduce_dense_time_bits(8, 64_000_000, 1e9) == pytest.approx(
        2 * 7 / 8 * 64e6 / (1e9 / 32))


@pytest.mark.gpu
def test_mixed_buckets_one_gpu(zen, co):
    rng = np.random.default_rng(31)
    rows, d = 5000, 64
    emb = np.zeros((rows, d), np.float32)
    live = rng.choice(rows, 300, replace=False)
    emb[live] = rng.standard_normal((live.size, d)).astype(np.float32)
    lay = rng.standard_normal(200_000).astype(np.float32)
    lay[rng.choice(lay.size, 5000, replace=False)] = 0.0
    dense = rng.standard_normal(100_000).astype(np.float32)
    grads = [torch.from_numpy(x.ravel()).cuda() for x in (emb, lay, dense)]
    ms = zen.MixedBucketSync([("sparse", emb.size), ("topk", lay.size, 0.01),
                              ("dense", dense.size)])
    ms.step(grads)
    i0, v0 = ms.result(0)
    wi, wv = co.to_sparse(emb.ravel())
    np.testing.assert_array_equal(i0.cpu().numpy().view(np.uint64), wi)
    np.testing.assert_array_equal(v0.cpu().numpy(), wv)
    i1, v1 = ms.result(1)
    ti, tv = co.sparsify_topk(lay, 0.01)
    np.testing.assert_array_equal(i1.cpu().numpy().view(np.uint64), ti)
    np.testing.assert_array_equal(v1.cpu().numpy(), tv)
    np.testing.assert_array_equal(grads[2].cpu().numpy(), dense)  # n = 1: the sum is itself
    params = [torch.ones(x.size, device="cuda") for x in (emb, lay, dense)]
    ms.apply_sgd(params, grads, 0.5)
    torch.cuda.synchronize()
    want0 = np.ones(emb.size, np.float32)
    want0[wi.astype(np.int64)] -= np.float32(0.5) * wv
    np.testing.assert_array_equal(params[0].cpu().numpy(), want0)
    want1 = np.ones(lay.size, np.float32)
    want1[ti.astype(np.int64)] -= np.float32(0.5) * tv
    np.testing.assert_array_equal(params[1].cpu().numpy(), want1)
    np.testing.assert_allclose(params[2].cpu().numpy(), 1.0 - 0.5 * dense, rtol=1e-6)
    with pytest.raises(zen.Error):  # a bf16 gradient is refused, not misread
        ms.step([grads[0].bfloat16(), grads[1], grads[2]])
