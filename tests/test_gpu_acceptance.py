"""The reference's ORCA acceptance sweep on the device (tests/test_acceptance.py:209-253
of the reference): 100 open 26 m arenas x 50 agents x 2000 steps (10 M agent-steps),
safety margin 0.05 m, goals re-sampled inside the spawnable interior.  Every step must
be overlap-free (last_gap_by_env >= 0, full pairwise checks every 200 steps), and since
the trajectories are bit-identical to the reference, the sweep's minimum gap must be
the reference's recorded 0.037 m (test_output.txt:17; reproduced in-container,
SURVEY.md §8c)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_orca_sweep_overlap_free_min_gap_matches_reference(torch_cuda):
    import torch
    from paper_2505_00690_b200.crowd import CrowdAgent, CrowdConfig, CrowdField
    from paper_2505_00690_b200.urbangen import OccupancyGrid
    arena, res = 26.0, 0.1
    n = int(arena / res)
    occ = OccupancyGrid(res, np.full((n, n), 2, np.uint8), np.zeros((n, n), np.float32))
    E, A = 100, 50
    field = CrowdField([occ] * E, CrowdConfig(safety_margin=0.05), [5000 + e for e in range(E)])
    lists = []
    for e in range(E):
        r = np.random.default_rng(e)
        lst = []
        for a in range(A):
            while True:
                p = r.uniform(1.5, arena - 1.5, 2)
                if all(np.hypot(*(p - o.position)) > 1.2 for o in lst):
                    break
            lst.append(CrowdAgent(id=a, position=p, velocity=np.zeros(2), radius=0.3,
                                  preferred_speed=float(r.uniform(0.8, 1.4)),
                                  goal=r.uniform(1.5, arena - 1.5, 2)))
        lists.append(lst)
    field.set_agents(lists)
    # goal re-sampling restricted to the spawnable interior, in walk-list order
    walk = field.walk_t.cpu().numpy()
    wn = field.walk_n_t.cpu().numpy()
    for e in range(E):
        f = walk[e, :wn[e]]
        x, y = (f % n + 0.5) * res, (f // n + 0.5) * res
        keep = f[(x > 1.5) & (x < arena - 1.5) & (y > 1.5) & (y < arena - 1.5)]
        field.walk_t[e, :keep.size] = torch.from_numpy(keep.astype(np.int32)).cuda()
        field.walk_n_t[e] = int(keep.size)
    field.prepare_step()
    iu = np.triu_indices(A, 1)
    rad = field.radius_t.cpu().numpy()
    rr2 = (rad[:, :, None] + rad[:, None, :]) ** 2
    min_gap = np.inf
    for step in range(2000):
        field.step(check=False)
        g = float(field.last_gap_t.min())
        min_gap = min(min_gap, g)
        assert g >= 0.0, f"overlap at step {step}"
        if step % 200 == 199:
            pos = field.pos_t.cpu().numpy()
            d2 = ((pos[:, :, None, :] - pos[:, None, :, :]) ** 2).sum(-1)
            assert not (d2[:, iu[0], iu[1]] < rr2[:, iu[0], iu[1]]).any(), step
    field.check_flags()
    assert f"{min_gap:.3f}" == "0.037", min_gap
