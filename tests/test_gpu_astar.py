"""Device A* (k_astar) against the oracle A* (oracle/crowd.py astar, pinned to
paths.py:48-87) search by search.

* tests/golden/astar_regress.npz: three long searches on a dense 256^2 scene
  (cfg5 shape) that once came out 2 - sqrt(2) too long -- an insertion into a
  full head lowered the head bound T below a later key of the same expansion.
  Kept as a regression for both search shapes (1 warp / 4 warps per CTA).
* every search of 48 dense cfg5-shape envs over 40 ticks, both shapes.
"""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu
MIX = {"Flat": 0.25, "Slope": 0.25, "Stair": 0.25, "Rough": 0.25}


def _path(f, e, a):
    """The agent's guidance cells (path_cells[head : head + path_n - 1])."""
    hd, n = int(f.path_head_t[e, a]), int(f.path_n_t[e, a])
    return f.path_cells_t[e, a, hd:hd + n - 1].cpu().numpy().tolist()


def _oracle_cells(passable, st, gl):
    from oracle import crowd as C
    ny, nx = passable.shape
    ref = C.astar(passable, divmod(st, nx), divmod(gl, nx))
    return None if ref is None else [r * nx + c for r, c in ref[1:]]


@pytest.mark.parametrize("warps", [1, 4])
def test_astar_regressions(warps, torch_cuda):
    from paper_2505_00690_b200.crowd import CrowdAgent, CrowdConfig, CrowdField
    from paper_2505_00690_b200.urbangen import OccupancyGrid
    g = load_golden("astar_regress.npz")
    res = 0.125
    for k in range(int(g["n"])):
        passable = g[f"c{k}_passable"].astype(bool)
        ny, nx = passable.shape
        st, gl = int(g[f"c{k}_start"]), int(g[f"c{k}_goal"])
        want = _oracle_cells(passable, st, gl)
        occ = OccupancyGrid(res, np.where(passable, 2, 0).astype(np.uint8), np.zeros((ny, nx), np.float32))
        f = CrowdField([occ], CrowdConfig(), [0], astar_warps=warps)
        at = lambda c: np.array([(c % nx + 0.5) * res, (c // nx + 0.5) * res])
        f.set_agents([[CrowdAgent(0, at(st), np.zeros(2), 0.3, 1.0, at(gl))]])
        f.prepare_step()
        f.step_phase(1)
        f.step_phase(2)
        n = int(f.path_n_t[0, 0])
        assert n == len(want) + 1, (k, n, len(want) + 1)
        assert _path(f, 0, 0) == want, k


@pytest.mark.parametrize("warps", [1, 4])
def test_every_search_matches_oracle_dense_scenes(warps, torch_cuda):
    import torch
    from oracle.rng import child_seed
    from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField
    from paper_2505_00690_b200.urbangen import SceneSampler, SceneSpec, TaskKind
    E, T = 48, 40
    seeds = [child_seed(0, "env", 500 + i) for i in range(E)]
    spec = SceneSpec(seed=0, extent_m=(32.0, 32.0), task_kind=TaskKind.NAV_DYNAMIC, pedestrian_count=48,
                     object_density=128 / 41, terrain_mix=MIX, grid_resolution_m=0.125)
    b = SceneSampler(spec, E).sample(seeds, [child_seed(s, "crowd", 0) for s in seeds])
    f = CrowdField(b, CrowdConfig(), [child_seed(s, "crowd-run") for s in seeds], astar_warps=warps)
    f.set_from_spawn(b)
    f.prepare_step()
    nx = b.params.nx
    passable = {}
    checked = 0
    for t in range(T):
        f.step_phase(1)
        torch.cuda.synchronize()
        reqs = f.astar_req_t[:int(f.flags_t[4])].cpu().numpy()
        f.step_phase(2)
        torch.cuda.synchronize()
        paths_n = f.path_n_t.cpu().numpy()
        for e, a, st, gl in reqs:
            if e not in passable:
                passable[e] = b.labels[e].cpu().numpy() != 0
            want = _oracle_cells(passable[e], int(st), int(gl))
            n = int(paths_n[e, a])
            if want is None:
                assert n == 1, (t, e, a)
                continue
            assert n == len(want) + 1, (t, e, a, n, len(want) + 1)
            assert _path(f, e, a) == want, (t, e, a)
            checked += 1
        f.step_phase(4)
    assert checked > 100


@pytest.mark.parametrize("warps", [1, 4])
def test_astar_pool_handover_matches_oracle(warps, torch_cuda):
    """A search that floods a 200 x 200 cup (~40k cells, more tiles than the shared
    pool holds) hands its open set over to the global store mid-search and must
    still pop in the reference order: same path as the oracle."""
    from paper_2505_00690_b200.crowd import CrowdAgent, CrowdConfig, CrowdField
    from paper_2505_00690_b200.urbangen import OccupancyGrid
    ny = nx = 256
    res = 0.125
    passable = np.ones((ny, nx), bool)
    passable[30:231, 30] = False
    passable[30:231, 230] = False
    passable[230, 30:231] = False
    st, gl = 220 * nx + 130, 245 * nx + 131
    want = _oracle_cells(passable, st, gl)
    occ = OccupancyGrid(res, np.where(passable, 2, 0).astype(np.uint8), np.zeros((ny, nx), np.float32))
    f = CrowdField([occ], CrowdConfig(), [0], astar_warps=warps)
    at = lambda c: np.array([(c % nx + 0.5) * res, (c // nx + 0.5) * res])
    f.set_agents([[CrowdAgent(0, at(st), np.zeros(2), 0.3, 1.0, at(gl))]])
    f.prepare_step()
    f.counters_t.zero_()
    f.step_phase(1)
    f.step_phase(2)
    assert int(f.counters_t[10]) == 1, "the search should have outgrown the shared tile pool"
    n = int(f.path_n_t[0, 0])
    assert n == len(want) + 1
    assert _path(f, 0, 0) == want
