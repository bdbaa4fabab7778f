"""Compare the device A* expansion order (counters[15] trace) of one search with
the oracle's heapq pop order (GPU).  Usage: python tools/astar_trace.py case.npz [W]

The trace is compiled only into debug builds: rebuild the library with the
_lib.NVCC_FLAGS command plus -DCW_ASTAR_TRACE before using this tool."""
import heapq
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_00690_b200 import _lib  # noqa: E402
from paper_2505_00690_b200.crowd import CrowdAgent, CrowdConfig, CrowdField  # noqa: E402
from paper_2505_00690_b200.urbangen import OccupancyGrid  # noqa: E402

SQRT2 = math.sqrt(2.0)


def oracle_pops(passable, start, goal):
    ny, nx = passable.shape
    sr, sc = start
    gr, gc = goal

    def h(r, c):
        dr, dc = abs(r - gr), abs(c - gc)
        return SQRT2 * min(dr, dc) + abs(dr - dc)
    g = {(sr, sc): 0.0}
    heap = [(h(sr, sc), h(sr, sc), sr, sc)]
    pops = []
    moves = ((-1, 0, 1.0), (1, 0, 1.0), (0, -1, 1.0), (0, 1, 1.0),
             (-1, -1, SQRT2), (-1, 1, SQRT2), (1, -1, SQRT2), (1, 1, SQRT2))
    while heap:
        f, hh, r, c = heapq.heappop(heap)
        if f > g[(r, c)] + h(r, c) + 1e-12:
            continue
        pops.append((r * nx + c, g[(r, c)], f, hh))
        if (r, c) == (gr, gc):
            break
        for dr, dc, w in moves:
            rr, cc = r + dr, c + dc
            if not (0 <= rr < ny and 0 <= cc < nx) or not passable[rr, cc]:
                continue
            if dr and dc and not (passable[r, cc] and passable[rr, c]):
                continue
            ng = g[(r, c)] + w
            if ng < g.get((rr, cc), math.inf) - 1e-12:
                g[(rr, cc)] = ng
                heapq.heappush(heap, (ng + h(rr, cc), h(rr, cc), rr, cc))
    return pops


_lib.build()
d = np.load(sys.argv[1])
W = int(sys.argv[2]) if len(sys.argv) > 2 else 1
res = 0.125
passable = d["labels"]
ny, nx = passable.shape
st, gl = int(d["start"]), int(d["goal"])
pops = oracle_pops(passable, divmod(st, nx), divmod(gl, nx))
labels = np.where(passable, 2, 0).astype(np.uint8)
occ = OccupancyGrid(res, labels, np.zeros((ny, nx), np.float32))
f = CrowdField([occ], CrowdConfig(), [0], astar_warps=W)
ag = [CrowdAgent(0, np.array([(st % nx + 0.5) * res, (st // nx + 0.5) * res]), np.zeros(2), 0.3, 1.0,
                 np.array([(gl % nx + 0.5) * res, (gl // nx + 0.5) * res]))]
f.set_agents([ag])
f.prepare_step()
tr = torch.full((2 << 20,), -1, dtype=torch.int64, device="cuda")
evb = torch.zeros((4 + 4 * 4096,), dtype=torch.int64, device="cuda")
watch = os.environ.get("WATCH")
f.step_phase(1)
f.counters_t[15] = tr.data_ptr()
if watch:
    wr, wc = (int(v) for v in watch.split(","))
    f.counters_t[12] = evb.data_ptr()
    f.counters_t[13] = wr * nx + wc
f.step_phase(2)
torch.cuda.synchronize()
f.counters_t[15] = 0
f.counters_t[12] = 0
if watch:
    ev = evb.cpu().numpy()
    names = {10: "split: stale", 12: "split: keep", 13: "split: demote", 20: "far->near stale", 22: "far keep",
             23: "far->near", 30: "near->head stale", 34: "near keep", 35: "near->far", 36: "near->band",
             40: "merge reject->near", 51: "push->head", 52: "push->near", 54: "push->far", 60: "dec-key evict",
             70: "full-head evict->far", 71: "full-head evict->near", 80: "REFILL nn,nf,h", 81: "SPLIT nn,nf,h"}
    for k in range(int(ev[0])):
        c, a, b, d = ev[4 + 4 * k: 8 + 4 * k]
        fa = float(np.int64(a).view(np.float64)) if a >= 0 and c < 80 else a
        fb = float(np.int64(b).view(np.float64)) if b >= 0 and c < 80 else b
        print(f"  ev {names.get(int(c), c)}: f {fa!r} | {fb!r} | {d}")
t = tr.cpu().numpy().reshape(-1, 2)
n = int((t[:, 0] >= 0).sum())
dev = [(int(x), float(np.int64(gb).view(np.float64))) for x, gb in t[:n]]
print(f"oracle pops {len(pops)}, device expansions {n} (incl. goal)")
for i, ((ox, og, of, oh), (dx, dg)) in enumerate(zip(pops, dev)):
    if ox != dx or og != dg:
        print(f"first divergence at pop {i}: oracle cell {divmod(ox, nx)} g {og!r} f {of!r} h {oh!r}; "
              f"device cell {divmod(dx, nx)} g {dg!r}")
        for j in range(max(0, i - 3), min(len(pops), i + 4)):
            print("   oracle", j, divmod(pops[j][0], nx), pops[j][1:], " device",
                  divmod(dev[j][0], nx) if j < n else None, dev[j][1] if j < n else None)
        # is the oracle's cell later expanded by the device?
        later = [k for k in range(i, n) if dev[k][0] == ox]
        print("   oracle cell expanded by the device at", later[:3], [dev[k][1] for k in later[:3]])
        break
else:
    print("same order over the common prefix")
