"""Device scene identity vs the unmodified reference
(tests/golden/sceneio.json, oracle/make_golden_sceneio.py): scene_hash of
device-sampled scenes (all layouts, both splits), canonical JSON texts byte for
byte, BatchedEnv.scene_hashes (Async / Sync / after resampling), and the device
run-length coder (cw_scene_rle) against the oracle on adversarial grids."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import sceneio as O

pytestmark = pytest.mark.gpu


def _golden():
    with open(os.path.join(GOLDEN, "sceneio.json"), encoding="utf-8") as fh:
        return json.load(fh)


def _first_diff(a, b):
    i = next((k for k in range(min(len(a), len(b))) if a[k] != b[k]), min(len(a), len(b)))
    return f"first difference at {i}: ours {a[max(0, i - 60):i + 60]!r} ref {b[max(0, i - 60):i + 60]!r}"


@pytest.mark.parametrize("case", range(16))
def test_scene_hash_matches_reference(case, torch_cuda):
    from paper_2505_00690_b200.urbangen import SceneSampler, SceneSpec
    c = _golden()["cases"][case]
    spec = SceneSpec.from_dict(c["spec"])
    s = SceneSampler(spec, 1)
    s.sample([spec.seed])
    d = s.scene_dicts()[0]
    if "json" in c:
        text = O.canonical_dumps(d)
        assert text == c["json"], _first_diff(text, c["json"])
    assert s.scene_hashes() == [c["hash"]]


def test_batch_hashes_match_reference(torch_cuda):
    """Six cfg1 scenes sampled in one batch, hashed in one device RLE pass, rows
    requested out of order."""
    from paper_2505_00690_b200.urbangen import SceneSampler, SceneSpec
    cs = _golden()["cases"][:6]
    spec = SceneSpec.from_dict(cs[0]["spec"])
    s = SceneSampler(spec, 6)
    s.sample([c["spec"]["seed"] for c in cs])
    order = [4, 0, 5, 2, 1, 3]
    assert s.scene_hashes(order) == [cs[i]["hash"] for i in order]


def test_generate_scene_description_hash(torch_cuda):
    from paper_2505_00690_b200 import sceneio as S
    from paper_2505_00690_b200.urbangen import SceneSpec, generate_scene
    c = _golden()["cases"][8]
    sc = generate_scene(SceneSpec.from_dict(c["spec"]))
    assert S.scene_hash(sc) == c["hash"]
    assert S.scene_to_json(sc) == c["json"]
    assert np.array_equal(sc.zones.grid, O.rle_decode(json.loads(c["json"])["zones"]["rle"]).reshape(
        sc.zones.grid.shape))
    cache = S.AssetCache()
    spec = SceneSpec.from_dict(c["spec"])
    assert cache.scene(spec) is cache.scene(spec) and len(cache) == 1


def test_batched_env_scene_hashes(torch_cuda):
    from paper_2505_00690_b200.envcore import BatchedEnv, Scheme
    from paper_2505_00690_b200.urbangen import SceneSpec
    g = _golden()["batched"]
    spec = SceneSpec.from_dict(g["batch_spec"])
    a = BatchedEnv(spec, Scheme.ASYNC, master_seed=0, k=4)
    assert a.scene_hashes == g["Async"]
    assert len(set(a.scene_hashes)) == 4
    s = BatchedEnv(spec, Scheme.SYNC, master_seed=0, k=4)
    assert s.scene_hashes == g["Sync"] and len(set(s.scene_hashes)) == 1
    a.reset(1, resample=True)
    a.reset(1, resample=False)
    a.reset(1, resample=True)
    assert a.scene_hashes == g["Async_resampled"]


@pytest.mark.parametrize("shape", [(512, 512), (97, 103), (4, 5)])
def test_device_rle_matches_oracle(shape, torch_cuda):
    """Constant, every-cell-alternating (maximum runs), random runs and a single
    odd cell at the end; chunk boundaries (1024 cells) cut runs; rows requested
    out of order."""
    import torch
    from paper_2505_00690_b200 import sceneio as S
    from paper_2505_00690_b200.urbangen import SceneBatch, SceneSpec, TaskKind, scene_params
    ny, nx = shape
    res = 0.125
    spec = SceneSpec(seed=0, extent_m=(nx * res, ny * res), task_kind=TaskKind.NAV_CLEAR,
                     grid_resolution_m=res) if min(nx, ny) * res >= 5.0 else None
    if spec is None:
        spec = SceneSpec(seed=0, extent_m=(5.0, 5.0), task_kind=TaskKind.NAV_CLEAR, grid_resolution_m=1.0)
    p = scene_params(spec)
    b = SceneBatch(p, 5)
    N, NT = p.nx * p.ny, p.trows * p.tcols
    rng = np.random.default_rng(7)
    z = np.zeros((5, N), np.uint8)
    z[1] = np.arange(N) % 2
    z[2] = np.repeat(rng.integers(0, 6, N), rng.integers(1, 2000, N))[:N]
    z[3] = np.repeat(rng.integers(0, 3, N), rng.integers(1, 5, N))[:N]
    z[4, -1] = 5
    a = np.zeros((5, NT), np.int32)
    a[1] = np.arange(NT) % 3
    a[2] = rng.integers(0, 44, NT)
    a[4, 0] = 43
    b.zones.copy_(torch.from_numpy(z.reshape(5, p.ny, p.nx)))
    b.assign.copy_(torch.from_numpy(a.reshape(5, p.trows, p.tcols)))
    rows = [3, 0, 4, 1, 2]
    got = S.device_rle(b, rows)
    for (zr, ar), r in zip(got, rows):
        assert zr == O.rle_encode(z[r]), r
        assert ar == O.rle_encode(a[r]), r
