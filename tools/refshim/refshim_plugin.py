"""pytest plugin: run the reference's OWN tests against the B200 drop-in.

Loaded with ``-p refshim_plugin`` before collection, it imports the unmodified
reference package ``citywalk`` (the baseline/_ref install) and rebinds the
hot-path entry points -- the ones SURVEY §8(b) lists -- to the B200 classes and
functions of ``paper_2505_00690_b200``.  Everything else (out-of-scope modules,
stage internals the tests poke at, the reference's dataclasses used as inputs)
stays the reference's own, so a test that fails here fails on the drop-in.

Rebound (reference module -> B200):
  citywalk.crowd{,.field,.step,.routes,.orca}: CrowdField, step_crowd, spawn_agents,
      sample_routes, connected_components, compute_orca_constraints, solve_velocity,
      feasible, orca_halfplane, HalfPlane, write_trace, field._batched_lp
  citywalk.urbangen{,.scene,.occupancy}: generate_scene, rasterize_occupancy
  citywalk.envcore{,.batch,.cache}: BatchedEnv, AssetCache
Each test records which B200 entry points it called (``b200_calls`` in the
junit properties), so the report separates drop-in tests from tests of
reference internals.
"""

import functools

import pytest

_CALLS = set()


def _track(name, fn):
    @functools.wraps(fn)
    def wrapped(*a, **k):
        _CALLS.add(name)
        return fn(*a, **k)
    return wrapped


def _track_class(name, cls):
    orig = cls.__init__

    @functools.wraps(orig)
    def init(self, *a, **k):
        _CALLS.add(name)
        return orig(self, *a, **k)
    return type(cls.__name__, (cls,), {"__init__": init, "__module__": cls.__module__})


def _install():
    # the drop-in raises its own exception classes (same names, same hierarchy); bind
    # them into citywalk.errors before any other reference module imports them
    import citywalk.errors
    from paper_2505_00690_b200 import errors as BX
    for n in dir(BX):
        if isinstance(getattr(BX, n), type) and hasattr(citywalk.errors, n):
            setattr(citywalk.errors, n, getattr(BX, n))
    import citywalk.crowd
    import citywalk.crowd.field
    import citywalk.crowd.orca
    import citywalk.crowd.routes
    import citywalk.crowd.step
    import citywalk.envcore
    import citywalk.envcore.batch
    import citywalk.envcore.cache
    import citywalk.urbangen
    import citywalk.urbangen.occupancy
    import citywalk.urbangen.scene
    from paper_2505_00690_b200 import crowd as BC
    from paper_2505_00690_b200 import envcore as BE
    from paper_2505_00690_b200 import sceneio as BS
    from paper_2505_00690_b200 import urbangen as BU

    crowd = {n: _track(n, getattr(BC, n)) for n in (
        "step_crowd", "spawn_agents", "sample_routes", "connected_components", "compute_orca_constraints",
        "solve_velocity", "feasible", "orca_halfplane", "write_trace", "_batched_lp")}
    crowd["CrowdField"] = _track_class("CrowdField", BC.CrowdField)
    crowd["HalfPlane"] = BC.HalfPlane
    for mod in (citywalk.crowd, citywalk.crowd.field, citywalk.crowd.step, citywalk.crowd.routes,
                citywalk.crowd.orca):
        for n, v in crowd.items():
            if hasattr(mod, n):
                setattr(mod, n, v)
    gen = _track("generate_scene", BU.generate_scene)
    ras = _track("rasterize_occupancy", BU.rasterize_occupancy)
    for mod in (citywalk.urbangen, citywalk.urbangen.scene, citywalk.urbangen.occupancy):
        if hasattr(mod, "generate_scene"):
            mod.generate_scene = gen
        if hasattr(mod, "rasterize_occupancy"):
            mod.rasterize_occupancy = ras
    env = _track_class("BatchedEnv", BE.BatchedEnv)
    cache = _track_class("AssetCache", BS.AssetCache)
    for mod in (citywalk.envcore, citywalk.envcore.batch, citywalk.envcore.cache):
        if hasattr(mod, "BatchedEnv"):
            mod.BatchedEnv = env
        if hasattr(mod, "AssetCache"):
            mod.AssetCache = cache


_install()


@pytest.hookimpl(hookwrapper=True)
def pytest_runtest_call(item):
    _CALLS.clear()
    yield
    item.user_properties.append(("b200_calls", ",".join(sorted(_CALLS))))
