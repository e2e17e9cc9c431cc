"""Partition/grouping contracts (bit-exact integer work), mirroring
pkg/tests/test_tree.py and the slab rule of strategies.py:162-164."""
import pytest

from paper_2506_21411_b200.config import (ConfigError, ModelConfig, StrategyConfig, TreeSpec,
                                          build_tree_spec, channel_slabs, max_group_for_depth)
import dchag_oracle as O


def test_reference_tree_cases():
    assert build_tree_spec(256, 128).levels == ((128, 128), (2,))
    assert build_tree_spec(256, 32).levels == ((32,) * 8, (8,))
    assert build_tree_spec(5, 8).levels == ((5,),)
    assert build_tree_spec(1, 2).levels == ((1,),)
    assert build_tree_spec(10, 4).levels == ((4, 3, 3), (3,))
    s = build_tree_spec(64, 2)
    s.validate(64)
    assert s.levels[-1] in ((2,), (1,))


def test_validate_and_bad_args():
    with pytest.raises(ConfigError):
        TreeSpec(((2, 2),)).validate(5)
    with pytest.raises(ConfigError):
        TreeSpec(((2, 2), (2,), (2,))).validate(4)
    with pytest.raises(ConfigError):
        build_tree_spec(0, 4)
    with pytest.raises(ConfigError):
        build_tree_spec(8, 1)


@pytest.mark.parametrize("n", list(range(1, 130)) + [250, 500, 1024])
@pytest.mark.parametrize("g", [2, 3, 4, 8, 16, 64])
def test_tree_matches_oracle_restatement(n, g):
    assert build_tree_spec(n, g).levels == O.build_levels(n, g)


def test_canonical_configs():
    # SURVEY.md section 8(a)/(d) canonical instantiations
    assert build_tree_spec(16, 8).levels == ((8, 8), (2,))
    assert build_tree_spec(128, 64).levels == ((64, 64), (2,))
    assert build_tree_spec(500, 16).depth == 3 and build_tree_spec(500, 16).num_nodes == 35
    assert build_tree_spec(250, 8).num_nodes == 37
    assert build_tree_spec(125, 8).num_nodes == 19
    assert build_tree_spec(63, 4).num_nodes == 21 and build_tree_spec(62, 4).num_nodes == 21
    assert max_group_for_depth(500, 3) == 16
    assert max_group_for_depth(250, 3) == 8
    assert max_group_for_depth(125, 3) == 8
    assert max_group_for_depth([63, 62], 3) == 4
    assert max_group_for_depth(128, 2) == 64


def test_slabs_equal_and_balanced():
    assert channel_slabs(8, 2) == ((0, 4), (4, 4))
    assert channel_slabs(500, 8) == ((0, 63), (63, 63), (126, 63), (189, 63), (252, 62),
                                     (314, 62), (376, 62), (438, 62))
    for c in (16, 500, 128, 1024, 7):
        for tp in (1, 2, 4, 8):
            if tp > c:
                continue
            sl = channel_slabs(c, tp)
            assert sum(n for _, n in sl) == c
            assert [o for o, _ in sl] == [sum(n for _, n in sl[:i]) for i in range(tp)]
            assert sl == tuple(O.slabs(c, tp))
            if c % tp == 0:
                assert sl == tuple((r * c // tp, c // tp) for r in range(tp))


def test_strategy_validation():
    m = ModelConfig(channels=500, image_h=128, image_w=128, patch=8, embed=1024, heads=16,
                    agg_variant="single_query")
    m.validate()
    with pytest.raises(ConfigError, match="divisible"):
        StrategyConfig(tp_degree=8, max_group=4).validate(m)
    StrategyConfig(tp_degree=8, max_group=4, uneven_slabs=True).validate(m)
    s = StrategyConfig(tp_degree=8, max_group=4, uneven_slabs=True)
    assert [s.local_channels(m, r) for r in range(8)] == [63] * 4 + [62] * 4
    with pytest.raises(ConfigError):
        ModelConfig(channels=4, image_h=10, image_w=8, patch=4, embed=8, heads=2).validate()
