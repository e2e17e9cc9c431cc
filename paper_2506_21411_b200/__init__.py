"""B200-native D-CHAG channel front end (per-channel tokenizer + hierarchical
cross-channel aggregation + partial-aggregate AllGather + final layer)."""
from .config import (ConfigError, ModelConfig, StrategyConfig, TreeSpec, build_tree_spec,
                     channel_slabs)
from .frontend import DchagFrontEnd

__version__ = "0.1.0"
__all__ = ["ConfigError", "ModelConfig", "StrategyConfig", "TreeSpec", "build_tree_spec",
           "channel_slabs", "DchagFrontEnd"]
