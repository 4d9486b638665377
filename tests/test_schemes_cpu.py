"""Host-side logic of the scheme layer, no GPU:
the cost model, the selector and the profile's validation against the
reference's formulas (zen/costmodel.hpp) and its costmodel_test.cpp cases,
and the scheme dispatch's rejection rules (zen/schemes.hpp:27-41, 420-470)."""
import math

import pytest

import paper_2309_13254_b200 as zen


def flat(n):
    return {k: 1.0 for k in [1 << j for j in range(n.bit_length())] if k <= n}


def linear(n):
    return {k: float(k) for k in [1 << j for j in range(n.bit_length())] if k <= n}


def test_select_scheme_regimes():  # costmodel_test.cpp:129-150
    assert zen.select_scheme(zen.SparsityProfile(0.01, flat(16)), 16) == zen.BALANCED_PARALLELISM
    lin = zen.SparsityProfile(0.001, linear(16))
    assert zen.select_scheme(lin, 8) == zen.HIERARCHICAL_CENTRALIZATION
    assert zen.select_scheme(lin, 16) == zen.HIERARCHICAL_CENTRALIZATION
    tie = zen.SparsityProfile(0.01, {1: 1.0, 2: 1.0})
    assert zen.select_scheme(tie, 2) == zen.BALANCED_PARALLELISM
    with pytest.raises(zen.MissingProfileEntry):
        zen.select_scheme(zen.SparsityProfile(0.01, {1: 1.0, 4: 2.0}), 4)


def test_selection_is_invariant_to_bandwidth():  # costmodel_test.cpp:152-...
    g = {1: 1.0, 2: 1.9, 4: 3.4, 8: 5.9, 16: 9.5}
    choice = zen.select_scheme(zen.SparsityProfile(0.02, g), 16)
    for b in [0.5, 8.0, 1e9]:
        c = zen.CostInputs(16, 1e6, 0.02, b, g)
        bp_cheaper = zen.t_bp(c) <= zen.t_hc(c)
        assert (choice == zen.BALANCED_PARALLELISM) == bp_cheaper


def test_cost_formulas():
    g = {1: 1.0, 2: 1.5, 4: 2.5, 8: 4.0}
    assert zen.t_bp_coefficient(8, 4.0) == 7.0 / 8.0 * 5.0
    assert zen.t_bp_coefficient(1, 9.0) == 0.0
    assert zen.t_hc_coefficient(8, g) == 1.0 + 1.5 + 2.5
    with pytest.raises(zen.NonPowerOfTwo):
        zen.t_hc_coefficient(6, g)
    with pytest.raises(zen.MissingProfileEntry):
        zen.t_hc_coefficient(8, {1: 1.0, 2: 1.5})
    c = zen.CostInputs(8, 1e6, 0.01, 2.0, g, skew=1.5)
    assert math.isclose(zen.t_bp(c), 7.0 / 8.0 * 5.0 * 2.0 * 1e6 * 0.01 / 2.0)
    assert math.isclose(zen.t_hc(c), 5.0 * 2.0 * 1e6 * 0.01 / 2.0)
    assert zen.t_hierarchy_incremental_lb(c) <= zen.t_hc(c)
    assert math.isclose(zen.t_allreduce_dense(c), 2.0 * 7.0 / 8.0 * 1e6 / 2.0)
    assert zen.t_sparse_ps(c) > 0 and zen.t_sparse_ps_broadcast(c) > 0
    with pytest.raises(zen.MissingProfileEntry):
        zen.t_ring_incremental(c)  # needs gamma at every k < n
    assert zen.t_bp(zen.CostInputs(1)) == 0.0


def test_profile_validation():  # tensor.hpp:221-239
    zen.SparsityProfile(0.01, {1: 1.0, 2: 1.5}, {2: 1.1}).validate()
    for bad in [zen.SparsityProfile(0.0, {1: 1.0}),
                zen.SparsityProfile(0.01, {1: 0.9}),
                zen.SparsityProfile(0.01, {1: 1.0, 2: 0.5}),
                zen.SparsityProfile(0.01, {1: 1.0, 2: 2.5}),
                zen.SparsityProfile(0.6, {1: 1.0, 2: 2.0}),
                zen.SparsityProfile(0.01, {1: 1.0}, {4: 0.5})]:
        with pytest.raises(zen.Error):
            bad.validate()


def test_scheme_configs_and_rejections():
    for name in zen.KNOWN_SCHEME_NAMES:
        zen.scheme_config_from_name(name).validate()
    with pytest.raises(zen.UnsupportedCombination):
        zen.scheme_config_from_name("allreduce")
    cfg = zen.SchemeConfig(balance=zen.BalancePattern.Balanced)
    with pytest.raises(zen.UnsupportedCombination):
        cfg.validate()
    om = zen.scheme_config_from_name("omnireduce")
    assert om.format.kind == "tensor_block" and om.format.block_size == 256
    assert zen.scheme_config_from_name("balanced-parallelism").format.kind == "hash_bitmap"
