"""Generate tests/golden/acceptance_sweep.npz from the REAL reference (build container only).

Run:  PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_acceptance.py   (~2 min)

The reference's ORCA acceptance sweep (tests/test_acceptance.py:209-249): 100 open
26 m arenas x 50 agents x 2000 steps, safety margin 0.05 m, goals re-sampled inside
the spawnable interior.  Stores the exact minimum gap (printed as 0.037 m in
test_output.txt:17), the per-step minimum of last_gap_by_env, and the final
positions / velocities / goals, so the device sweep is checked bit for bit.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def main():
    sys.path.insert(0, REF)
    from citywalk.crowd import CrowdAgent, CrowdConfig, CrowdField
    from citywalk.urbangen.types import CellLabel, OccupancyGrid
    arena, res = 26.0, 0.1
    n = int(arena / res)
    labels = np.full((n, n), int(CellLabel.WALKABLE), dtype=np.uint8)
    occ = OccupancyGrid(resolution=res, labels=labels, elevation=np.zeros((n, n), dtype=np.float32))
    E, A = 100, 50
    field = CrowdField([occ] * E, CrowdConfig(safety_margin=0.05), env_seeds=[5000 + e for e in range(E)])
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
    field._walk_cells = [wc[(wc[:, 0] > 1.5) & (wc[:, 0] < arena - 1.5) & (wc[:, 1] > 1.5) & (wc[:, 1] < arena - 1.5)]
                         for wc in field._walk_cells]
    mins = np.empty(2000)
    for step in range(2000):
        field.step()
        mins[step] = float(field.last_gap_by_env.min())
    np.savez_compressed(os.path.join(OUT, "acceptance_sweep.npz"), step_min_gap=mins, min_gap=mins.min(),
                        pos=field.pos, vel=field.vel, goal=field.goal, last_gap=field.last_gap_by_env)
    print("min gap", repr(mins.min()))


if __name__ == "__main__":
    main()
