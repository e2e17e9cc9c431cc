"""Front-end configuration: channel partition, aggregation tree, model/strategy fields.

Mirrors the reference's config surface for the D-CHAG channel front end
(`/root/reference/pkg/src/dchag/config.py`), restated here with the same
names, argument meaning and error class so existing call sites keep working:

* ``ConfigError``                       -- config.py:8-9
* ``TreeSpec`` (levels/depth/fanout_max/validate) -- config.py:17-45
* ``build_tree_spec(local_channels, max_group)``  -- config.py:48-66
* ``ModelConfig`` front-end fields + validate     -- config.py:69-116
* ``StrategyConfig`` dchag fields + validate      -- config.py:119-162

Extension (declared, not in the reference): ``channel_slabs`` partitions C
channels over tp ranks as balanced contiguous slabs (the first C mod tp ranks
get one extra channel) -- the same rule ``build_tree_spec`` applies to groups
(config.py:59-61).  When tp divides C it reproduces the reference's equal slabs
``[r*C/tp, (r+1)*C/tp)`` (strategies.py:162-164) bit-exactly.
"""

from __future__ import annotations

from dataclasses import dataclass

AGG_VARIANTS = ("single_query", "full_cross")
AGG_LAYER_KINDS = ("cross_attention", "linear")
STRATEGY_KINDS = ("serial", "tp_only", "dist_token", "dchag")


class ConfigError(Exception):
    """Invalid or inconsistent configuration (reference config.py:8-9)."""


def _balanced_split(n: int, parts: int) -> tuple[int, ...]:
    """n items into `parts` contiguous groups whose sizes differ by <= 1, larger first."""
    base, extra = divmod(n, parts)
    return tuple(base + 1 if i < extra else base for i in range(parts))


@dataclass(frozen=True)
class TreeSpec:
    """Grouping plan: levels[0] splits the local channels, each later level
    splits the previous level's group count, the last level is one group."""

    levels: tuple[tuple[int, ...], ...]

    @property
    def depth(self) -> int:
        return len(self.levels)

    @property
    def fanout_max(self) -> int:
        return max(max(lv) for lv in self.levels)

    @property
    def num_nodes(self) -> int:
        return sum(len(lv) for lv in self.levels)

    def validate(self, local_channels: int) -> None:
        want = local_channels
        for li, lv in enumerate(self.levels):
            got = sum(lv)
            if got != want:
                raise ConfigError(
                    f"tree level {li} groups {lv} sum to {got}, expected {want}")
            want = len(lv)
        if want != 1:
            raise ConfigError("tree must terminate in a single group")

    def offsets(self, level: int) -> tuple[int, ...]:
        """Start index of every group of `level` within that level's inputs."""
        out, acc = [], 0
        for g in self.levels[level]:
            out.append(acc)
            acc += g
        return tuple(out)


def build_tree_spec(local_channels: int, max_group: int) -> TreeSpec:
    """Greedy balanced contiguous grouping (reference config.py:48-66):
    k = ceil(n / max_group) groups whose sizes differ by at most one (larger
    groups first), repeated on the group count until one group remains."""
    if local_channels < 1:
        raise ConfigError(f"local_channels must be >= 1, got {local_channels}")
    if max_group < 2:
        raise ConfigError(f"max_group must be >= 2, got {max_group}")
    levels = []
    n = local_channels
    while True:
        k = (n + max_group - 1) // max_group
        levels.append(_balanced_split(n, k))
        if k == 1:
            return TreeSpec(tuple(levels))
        n = k


def channel_slabs(channels: int, tp: int) -> tuple[tuple[int, int], ...]:
    """(offset, count) of every rank's contiguous channel slab, in rank order."""
    if tp < 1:
        raise ConfigError("tp_degree must be >= 1")
    if channels < tp:
        raise ConfigError(f"channels {channels} < tp_degree {tp}: a rank would own no channel")
    out, off = [], 0
    for cnt in _balanced_split(channels, tp):
        out.append((off, cnt))
        off += cnt
    return tuple(out)


def max_group_for_depth(local_channels, depth: int) -> int:
    """Largest power-of-two max_group giving `depth` levels for every slab size
    (the canonical instantiation of SURVEY.md section 8(d))."""
    sizes = [local_channels] if isinstance(local_channels, int) else list(local_channels)
    best = None
    g = 2
    while g <= max(sizes) * 2:
        if all(build_tree_spec(c, g).depth == depth for c in sizes):
            best = g
        g *= 2
    if best is None:
        raise ConfigError(f"no power-of-two max_group gives depth {depth} for slabs {sizes}")
    return best


@dataclass(frozen=True)
class ModelConfig:
    """Front-end subset of the reference ModelConfig (config.py:69-116).

    Trunk-only fields (depth, mlp_ratio, mask_ratio, decoder_*) are accepted
    for signature compatibility and ignored by the front end."""

    channels: int
    image_h: int
    image_w: int
    patch: int
    embed: int
    depth: int = 0
    heads: int = 1
    mlp_ratio: int = 4
    agg_variant: str = "full_cross"
    agg_layer_kind: str = "cross_attention"
    tree_max_group: int = 0
    mask_ratio: float = 0.5
    decoder_depth: int = 1
    decoder_dim: int = 16

    @property
    def seq(self) -> int:
        return (self.image_h // self.patch) * (self.image_w // self.patch)

    @property
    def patch_pixels(self) -> int:
        return self.patch * self.patch

    @property
    def tree(self) -> TreeSpec | None:
        return build_tree_spec(self.channels, self.tree_max_group) if self.tree_max_group else None

    def validate(self) -> None:
        if self.channels < 1:
            raise ConfigError(f"channels must be >= 1, got {self.channels}")
        if self.image_h % self.patch or self.image_w % self.patch:
            raise ConfigError(
                f"image {self.image_h}x{self.image_w} not divisible by patch {self.patch}"
                " (no padding is applied)")
        if self.embed % self.heads:
            raise ConfigError(f"embed {self.embed} not divisible by heads {self.heads}")
        if not (0 <= self.mask_ratio < 1):
            raise ConfigError(f"mask_ratio must be in [0, 1), got {self.mask_ratio}")
        if self.agg_variant not in AGG_VARIANTS:
            raise ConfigError(f"agg_variant must be one of {AGG_VARIANTS}")
        if self.agg_layer_kind not in AGG_LAYER_KINDS:
            raise ConfigError(f"agg_layer_kind must be one of {AGG_LAYER_KINDS}")


@dataclass(frozen=True)
class StrategyConfig:
    """dchag subset of the reference StrategyConfig (config.py:119-162).

    ``uneven_slabs`` is the declared extension: allow tp not dividing C with
    balanced slabs (the reference raises ConfigError, config.py:137-141)."""

    kind: str = "dchag"
    tp_degree: int = 1
    max_group: int = 128
    agg_layer_kind: str = "cross_attention"
    final_layer_tp_split: bool = False
    vit_tp_split: bool = False
    uneven_slabs: bool = False

    def validate(self, model: ModelConfig) -> None:
        if self.kind not in STRATEGY_KINDS:
            raise ConfigError(f"strategy kind must be one of {STRATEGY_KINDS}")
        if self.kind == "serial" and self.tp_degree != 1:
            raise ConfigError("serial strategy requires tp_degree=1")
        if self.tp_degree < 1:
            raise ConfigError("tp_degree must be >= 1")
        if self.agg_layer_kind not in AGG_LAYER_KINDS:
            raise ConfigError(f"agg_layer_kind must be one of {AGG_LAYER_KINDS}")
        if (self.kind in ("dist_token", "dchag") and model.channels % self.tp_degree
                and not self.uneven_slabs):
            raise ConfigError(
                f"channels {model.channels} not divisible by tp_degree {self.tp_degree}"
                " (equal channel slabs required)")
        if self.final_layer_tp_split and model.heads % self.tp_degree:
            raise ConfigError(f"heads {model.heads} not divisible by tp_degree {self.tp_degree}")

    def slabs(self, model: ModelConfig) -> tuple[tuple[int, int], ...]:
        if self.kind in ("dist_token", "dchag"):
            return channel_slabs(model.channels, self.tp_degree)
        return ((0, model.channels),)

    def local_channels(self, model: ModelConfig, rank: int = 0) -> int:
        return self.slabs(model)[rank if self.kind in ("dist_token", "dchag") else 0][1]

    def rank_tree(self, model: ModelConfig, rank: int = 0) -> TreeSpec:
        """Tree applied by `rank` to its slab (reference params.py:94-96)."""
        return build_tree_spec(self.local_channels(model, rank), self.max_group)
