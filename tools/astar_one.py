"""Run single A* searches (start, goal on a label grid; e.g. the cases of
tests/golden/astar_regress.npz exported with np.savez) through the product
k_astar via CrowdField and compare with the oracle (GPU).
Usage: python tools/astar_one.py case.npz [...]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import crowd as C  # noqa: E402
from paper_2505_00690_b200 import _lib  # noqa: E402
from paper_2505_00690_b200.crowd import CrowdAgent, CrowdConfig, CrowdField  # noqa: E402
from paper_2505_00690_b200.urbangen import OccupancyGrid  # noqa: E402

_lib.build()
res = float(os.environ.get("ONE_RES", 0.125))
for path in sys.argv[1:]:
    d = np.load(path)
    passable = d["labels"]
    ny, nx = passable.shape
    labels = np.where(passable, 2, 0).astype(np.uint8)
    st, gl = int(d["start"]), int(d["goal"])
    ref = C.astar(passable, divmod(st, nx), divmod(gl, nx))
    want = [r * nx + c for r, c in ref[1:]] if ref else None
    occ = OccupancyGrid(res, labels, np.zeros((ny, nx), np.float32))
    for w in (1, 4):
        for rep in range(3):
            E = 8
            f = CrowdField([occ] * E, CrowdConfig(), list(range(E)), astar_warps=w)
            ag = [CrowdAgent(0, np.array([(st % nx + 0.5) * res, (st // nx + 0.5) * res]), np.zeros(2), 0.3, 1.0,
                             np.array([(gl % nx + 0.5) * res, (gl // nx + 0.5) * res]))]
            f.set_agents([ag] * E)
            f.prepare_step()
            for ph in (1, 2):
                f.step_phase(ph)
            torch.cuda.synchronize()
            res_ok = []
            for e in range(E):
                n = int(f.path_n_t[e, 0])
                hd = int(f.path_head_t[e, 0])
                cells = f.path_cells_t[e, 0, hd:hd + n - 1].cpu().numpy().tolist()
                res_ok.append(n == len(ref) and cells == want)
            print(f"{os.path.basename(path)} W={w} rep {rep}: oracle n {len(ref)}; device ok per env {res_ok}",
                  flush=True)
