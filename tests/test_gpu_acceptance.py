"""The reference's ORCA acceptance sweep on the device (tests/test_acceptance.py:209-253
of the reference): 100 open 26 m arenas x 50 agents x 2000 steps (10 M agent-steps),
safety margin 0.05 m, goals re-sampled inside the spawnable interior.  Every step must
be overlap-free (last_gap_by_env >= 0, full pairwise checks every 200 steps), and the
trajectories are bit-identical to the reference's: every step's minimum gap, the
sweep's minimum (printed as 0.037 m in test_output.txt:17) and the final positions,
velocities and goals equal the values the unmodified reference wrote
(tests/golden/acceptance_sweep.npz, oracle/make_golden_acceptance.py)."""

import os

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
    # goal re-sampling restricted to the spawnable interior (the reference test writes
    # field._walk_cells, tests/test_acceptance.py:234-238)
    field._walk_cells = [wc[(wc[:, 0] > 1.5) & (wc[:, 0] < arena - 1.5) & (wc[:, 1] > 1.5)
                            & (wc[:, 1] < arena - 1.5)] for wc in field._walk_cells]
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "acceptance_sweep.npz"))
    iu = np.triu_indices(A, 1)
    rad = field.radius_t.cpu().numpy()
    rr2 = (rad[:, :, None] + rad[:, None, :]) ** 2
    min_gap = np.inf
    mins = np.empty(2000)
    for step in range(2000):
        field.step(check=False)
        g = float(field.last_gap_t.min())
        mins[step] = g
        min_gap = min(min_gap, g)
        assert g >= 0.0, f"overlap at step {step}"
        if step % 200 == 199:
            pos = field.pos_t.cpu().numpy()
            d2 = ((pos[:, :, None, :] - pos[:, None, :, :]) ** 2).sum(-1)
            assert not (d2[:, iu[0], iu[1]] < rr2[:, iu[0], iu[1]]).any(), step
    field.check_flags()
    assert f"{min_gap:.3f}" == "0.037", min_gap
    assert min_gap == float(gold["min_gap"])
    assert np.array_equal(mins, gold["step_min_gap"])
    assert np.array_equal(field.pos_t.cpu().numpy(), gold["pos"])
    assert np.array_equal(field.vel_t.cpu().numpy(), gold["vel"])
    assert np.array_equal(field.goal_t.cpu().numpy(), gold["goal"])
