"""B200-native MoDM cache-retrieval hot path (drop-in for mixserve.cache).

Exports mirror pkg/src/mixserve/__init__.py:15-24 for the cache symbols.
"""
from .cache import SemanticCache
from .records import (
    DEFAULT_DIM,
    DEFAULT_THRESHOLDS,
    LARGE,
    NORM_TOL,
    POLICIES,
    POLICY_ALL,
    POLICY_DISABLED,
    POLICY_LARGE,
    SMALL,
    STEP_CHOICES,
    CacheEntry,
    EmbeddingError,
    RetrievalBatch,
    RetrievalResult,
    ThresholdTable,
    cosine,
    is_normalized,
    linear_sigma_schedule,
    noise_reentry_level,
    normalize,
    validate_sigma_schedule,
)

__version__ = "0.2.0"
