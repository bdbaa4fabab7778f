"""Pin oracle/routes.py (route anchors, spawn pick, clearance) to fixtures from the
unmodified reference (oracle/make_golden_routes.py)."""

import json

import numpy as np
import pytest

from conftest import load_golden

G = None


def _g():
    global G
    if G is None:
        G = load_golden("routes.npz")
    return G


@pytest.mark.parametrize("case", [0, 1, 2, 17, 19])   # 128^2 courtyards, small NavStatic, traverse
def test_route_anchors_match_reference(case):
    from oracle import routes as R
    g = _g()
    spec = json.loads(str(g[f"c{case}_spec"]))
    labels = g[f"c{case}_labels"]
    got = R.sample_route_anchors(labels, spec["res"], spec["seed"], (spec["extent"], spec["extent"]),
                                 spec["task"])
    assert np.array_equal(np.array(got, np.float64).reshape(-1, 2, 2), g[f"c{case}_routes"])
    picks = [R.spawn_pick(spec["seed"], rc, len(got)) for rc in range(3)]
    assert picks == list(g[f"c{case}_spawn_pick"])


@pytest.mark.parametrize("case", range(21))
def test_clearance_matches_reference(case):
    from oracle.scene import chamfer
    g = _g()
    spec = json.loads(str(g[f"c{case}_spec"]))
    walk = g[f"c{case}_labels"] == 2
    assert np.array_equal(chamfer(~walk, spec["res"]), g[f"c{case}_clearance"])
