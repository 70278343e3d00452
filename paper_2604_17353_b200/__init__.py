"""B200-native Logits-Cache re-sampling path (Hive, arXiv 2604.17353).

Drop-in for the reference's logits-cache interface (pkg/src/agentserve
``logits_cache`` / ``sampling`` / ``errors``; re-exported names follow
__init__.py:8-32 of the reference).  Everything on the path runs in
``_lib/liblcb200.so`` (hand-written sm_100a kernels behind the C ABI in
``include/lc_b200.h``); importing this package fails if that library cannot be
loaded -- there is no CPU fallback.
"""

from . import _capi  # noqa: F401  (loads liblcb200.so or raises)
from .errors import CapacityError, ConfigError
from .logits_cache import (
    TOKEN_OVERHEAD_BYTES,
    CachedTrajectory,
    LogitsCache,
    ReplayOutcome,
    ReplayPolicy,
    StateKey,
)
from .mixing import RngStream, hash_prompts, hash_tokens, mix2, uniforms
from .sampling import (
    HotspotParams,
    SamplingConfig,
    entropy,
    hotspot_score,
    identify_hotspots,
    make_tasks,
    max_prob,
    resample,
    sample,
    select_hotspots,
    softmax,
    truncate,
)

__version__ = "0.1.0"
LIB_PATH = _capi.LIB_PATH

__all__ = [
    "CachedTrajectory",
    "CapacityError",
    "ConfigError",
    "HotspotParams",
    "LogitsCache",
    "ReplayOutcome",
    "ReplayPolicy",
    "RngStream",
    "SamplingConfig",
    "StateKey",
    "TOKEN_OVERHEAD_BYTES",
    "entropy",
    "hash_prompts",
    "hash_tokens",
    "hotspot_score",
    "identify_hotspots",
    "make_tasks",
    "max_prob",
    "mix2",
    "resample",
    "sample",
    "select_hotspots",
    "softmax",
    "truncate",
    "uniforms",
    "__version__",
]
