"""The device workload generator (zen_generate; zen::generate,
zen/workload.hpp:22-154).

Same spec as the reference, not the same bits (counter-based hashes instead of
libstdc++'s mt19937_64), so the checks are the spec's exact properties --
ceil(d*M) distinct ascending indices per node, the shared core on every node,
integer values in [1, 16], determinism per seed, WorkloadSpec::validate's
InfeasibleSpec cases -- and statistical agreement with the reference's own
generator (oracle/_ref) on the measured workload characteristics.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _spec(zen, **kw):
    base = dict(universe=1_000_000, nodes=4, density=0.01, omega=0.5, hot_fraction=0.125,
                hot_mass=0.125, seed=42)
    base.update(kw)
    return zen.WorkloadSpec(**base)


def test_generate_exact_properties(zen):
    spec = _spec(zen)
    ts = zen.generate(spec)
    z = spec.nnz_per_node()
    core = int(np.ceil(spec.omega * spec.density * spec.universe))
    assert len(ts) == spec.nodes
    for t in ts:
        i = t.indices()
        assert i.size == z and np.all(np.diff(i.astype(np.int64)) > 0) and int(i[-1]) < spec.universe
        v = t.values()
        assert np.all((v >= 1) & (v <= 16)) and np.all(v == np.round(v))
    common = ts[0].indices()
    for t in ts[1:]:
        common = np.intersect1d(common, t.indices())
    assert common.size >= core  # the shared core is on every node
    again = zen.generate(spec)
    assert all(a == b for a, b in zip(ts, again))  # deterministic per seed
    other = zen.generate(_spec(zen, seed=43))
    assert ts[0] != other[0]


def test_generate_matches_reference_statistics(zen, ro):
    """Mean pairwise overlap, hot-tier share and union size vs the reference
    generator on the same spec (tolerances: a few standard errors)."""
    spec = _spec(zen, universe=2_000_000, nodes=4, density=0.01, omega=0.3, hot_mass=0.4)
    ours = [t.indices() for t in zen.generate(spec)]
    ref = [i for i, _ in ro.generate(spec.universe, spec.nodes, spec.density, spec.omega,
                                     spec.seed, spec.hot_fraction, spec.hot_mass)]
    hot = int(round(spec.hot_fraction * spec.universe))

    def stats(ts):
        ov = np.mean([np.intersect1d(a, b).size / a.size for k, a in enumerate(ts)
                      for b in ts[k + 1:]])
        hs = np.mean([(t < hot).mean() for t in ts])
        un = np.unique(np.concatenate(ts)).size
        return ov, hs, un

    (o1, h1, u1), (o2, h2, u2) = stats(ours), stats(ref)
    assert abs(o1 - o2) < 0.01
    assert abs(h1 - h2) < 0.01
    assert abs(u1 - u2) / u2 < 0.01


def test_generate_infeasible_specs(zen):
    with pytest.raises(zen.InfeasibleSpec):
        zen.generate(_spec(zen, density=0.0))
    with pytest.raises(zen.InfeasibleSpec):
        zen.generate(_spec(zen, universe=100, density=0.001))  # d*M < 1
    with pytest.raises(zen.InfeasibleSpec):
        zen.generate(_spec(zen, density=0.5, omega=0.0))  # disjoint remainders do not fit
    with pytest.raises(zen.InfeasibleSpec):
        zen.generate(_spec(zen, hot_mass=1.5))


def test_generate_tier_saturation(zen):
    """hot_mass = 1 with a tiny hot tier: the sampler must spill into the cold
    tier once the hot one is exhausted (TwoTierSampler, workload.hpp:79-100)."""
    spec = _spec(zen, universe=10_000, nodes=2, density=0.05, omega=0.0, hot_fraction=0.01,
                 hot_mass=1.0)
    for t in zen.generate(spec):
        i = t.indices()
        assert i.size == spec.nnz_per_node()
        assert np.count_nonzero(i < 100) == 100  # the whole hot tier, then cold draws
