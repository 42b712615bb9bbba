"""Install the GPU cache into a running ``mixserve`` (the reference package) in place.

The reference builds its cache in one place, ``SimConfig.build_cache()``
(pkg/src/mixserve/config.py:98-104, ``from .cache import SemanticCache``), and
every caller — ``scheduler.classify`` (scheduler.py:70-90), the engine's
reclassification (engine.py:329-338), completions (scheduler.py:126-128),
preload (engine.py:116-117) and the tests — reaches it through the
``mixserve.cache`` module.  ``install(mixserve.cache)`` replaces that module's
``SemanticCache`` with a subclass of the drop-in whose answers and errors are
built from the module's own value types: results are the reference's
``RetrievalResult`` (so ``res == RetrievalResult(None, None, None)`` holds),
inserted/imported entries are its ``CacheEntry`` and shape errors raise its
``EmbeddingError``.  Call it before the rest of ``mixserve`` is imported (their
``from .cache import SemanticCache`` lines then bind the GPU class), or patch
those modules too with ``modules=``.
"""
from __future__ import annotations

from .cache import SemanticCache
from .records import _entry_factory, _result_factory


def dropin_class(cache_module, base=SemanticCache):
    """The drop-in SemanticCache speaking `cache_module`'s value types."""
    rr = cache_module.RetrievalResult
    return type("SemanticCache", (base,), {
        "__module__": base.__module__,
        "__doc__": base.__doc__,
        "_Entry": cache_module.CacheEntry,
        "_new_entry": staticmethod(_entry_factory(cache_module.CacheEntry)),
        "_EmbeddingError": cache_module.EmbeddingError,
        "_make": staticmethod(_result_factory(rr)),
        "_MISS": rr(None, None, None),
    })


def install(cache_module, modules=(), base=SemanticCache):
    """Replace ``cache_module.SemanticCache`` (and the name in every module of `modules`)
    with the GPU drop-in.  Returns the previous class, so a caller can restore it."""
    old = cache_module.SemanticCache
    cls = dropin_class(cache_module, base)
    cache_module.SemanticCache = cls
    for m in modules:
        if getattr(m, "SemanticCache", None) is old:
            m.SemanticCache = cls
    return old
