"""Switch the reference package over to the B200 data plane by module aliasing.

The reference (``rolloutlab``) has no FFI and no factory for its store: ``TrajectoryManager``
builds ``SessionTrie`` objects itself (trajectory.py:143), and every other module imports
the data-plane types from ``.core`` / ``.trie`` / ``.trajectory``.  ``install()`` makes
those three module names resolve to this package's drop-ins *before* ``rolloutlab`` is
imported, so the reference's untouched engine, rollout manager, runtime drivers and HTTP
API (engine.py, rollout.py, runtime.py, api.py) run on the GPU store:

    rolloutlab.core        -> paper_2508_11553_b200.core        (core.py:1-228)
    rolloutlab.trie        -> paper_2508_11553_b200.trie        (trie.py:1-265)
    rolloutlab.trajectory  -> paper_2508_11553_b200.trajectory  (trajectory.py:1-375)

``core`` is aliased together with the trie because the reference's ``SpanOrigin`` is a
plain ``Enum``: types produced by one module set must compare identical (``is``) with the
types the callers hold.  Used by tests/test_reference_suite_gpu.py to run the reference's
own hot-path tests against the drop-in (pytest ``-p paper_2508_11553_b200.refalias``).
"""

from __future__ import annotations

import sys

ALIASED = ("core", "trie", "trajectory")


def install() -> None:
    """Alias rolloutlab.{core,trie,trajectory} to this package, then import rolloutlab."""
    from . import core, trajectory, trie

    mods = {"core": core, "trie": trie, "trajectory": trajectory}
    loaded = sys.modules.get("rolloutlab")
    if loaded is not None and sys.modules.get("rolloutlab.trie") is not trie:
        raise RuntimeError("rolloutlab was imported before refalias.install(); install the aliases first")
    for name, mod in mods.items():
        sys.modules[f"rolloutlab.{name}"] = mod
    import rolloutlab

    for name, mod in mods.items():
        setattr(rolloutlab, name, mod)


def pytest_configure(config):  # noqa: ARG001 - pytest plugin hook: alias before test modules import rolloutlab
    install()
