"""Scene identity / wire format on the host, no GPU.

The oracle (oracle/sceneio.py) is pinned to the reference's own scene JSON texts
and scene hashes (tests/golden/sceneio.json, oracle/make_golden_sceneio.py);
the package's host serializer (paper_2505_00690_b200/sceneio.py) must
reproduce them byte for byte through a load -> dump round trip."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import sceneio as O


def _golden():
    with open(os.path.join(GOLDEN, "sceneio.json"), encoding="utf-8") as fh:
        return json.load(fh)


def _texts():
    return [c for c in _golden()["cases"] if "json" in c]


def test_oracle_matches_reference_texts_and_hashes():
    for c in _texts():
        d = json.loads(c["json"])
        assert O.canonical_dumps(d) == c["json"]
        assert O.content_hash(d) == c["hash"]
        z = O.rle_decode(d["zones"]["rle"])
        assert z.size == d["zones"]["shape"][0] * d["zones"]["shape"][1]
        assert O.rle_encode(z) == d["zones"]["rle"]
        a = O.rle_decode(d["terrain"]["assignment_rle"], dtype=np.int64)
        assert a.size == d["terrain"]["rows"] * d["terrain"]["cols"]
        assert O.rle_encode(a) == d["terrain"]["assignment_rle"]


@pytest.mark.parametrize("k", range(7))
def test_scene_json_round_trip_matches_reference(k, tmp_path):
    from paper_2505_00690_b200 import sceneio as S
    c = _texts()[k]
    sc = S.scene_from_json(c["json"])
    assert S.scene_to_json(sc) == c["json"]
    assert S.scene_hash(sc) == c["hash"]
    # host re-encoding of the decoded grids (no cached run lists) gives the same text
    sc.zones.rle = None
    sc.terrain.assignment_rle = None
    assert S.scene_to_json(sc) == c["json"]
    p = str(tmp_path / "scene.json")
    S.save_scene(sc, p)
    assert S.scene_hash(S.load_scene(p)) == c["hash"]


def test_rle_codec_matches_oracle():
    from paper_2505_00690_b200 import sceneio as S
    rng = np.random.default_rng(0)
    for n in (0, 1, 2, 7, 1000):
        for hi in (1, 2, 6):
            v = rng.integers(0, hi, size=n).astype(np.uint8)
            v = np.repeat(v, rng.integers(1, 4, size=n))
            assert S.rle_encode(v) == O.rle_encode(v)
            assert np.array_equal(S.rle_decode(S.rle_encode(v)), v)


def test_scene_load_errors():
    from paper_2505_00690_b200 import sceneio as S
    from paper_2505_00690_b200.errors import SceneLoadError
    c = _texts()[0]
    d = json.loads(c["json"])
    d["schema_version"] = 2
    with pytest.raises(SceneLoadError):
        S.scene_from_json(json.dumps(d))
    with pytest.raises(SceneLoadError):
        S.scene_from_json("{}")
    with pytest.raises(SceneLoadError):
        S.scene_from_json("[1, 2")


def test_occupancy_export_round_trip(tmp_path):
    from paper_2505_00690_b200 import sceneio as S
    from paper_2505_00690_b200.urbangen import OccupancyGrid
    rng = np.random.default_rng(1)
    g = OccupancyGrid(0.25, rng.integers(0, 4, size=(13, 21)).astype(np.uint8),
                      rng.normal(size=(13, 21)).astype(np.float32))
    pre = str(tmp_path / "occ")
    S.export_occupancy(g, pre)
    with open(pre + ".pgm", "rb") as fh:
        assert fh.read(11) == b"P5\n21 13\n25"
    with open(pre + ".json", encoding="utf-8") as fh:
        assert fh.read() == ('{"elevation_file":"occ.elev.f32","height":13,"origin":[0.0,0.0],'
                             '"resolution":0.25,"width":21}\n')
    h = S.load_occupancy(pre)
    assert np.array_equal(h.labels, g.labels) and np.array_equal(h.elevation, g.elevation)


def test_spec_dict_matches_reference_keys():
    from paper_2505_00690_b200.urbangen import SceneSpec
    for c in _golden()["cases"]:
        assert SceneSpec.from_dict(c["spec"]).to_dict() == c["spec"]
