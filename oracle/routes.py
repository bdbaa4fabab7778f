"""Oracle (TEST INFRASTRUCTURE ONLY): route anchors and the robot spawn they
feed -- SURVEY §8(f) row 2.  Only tests/ may import this module.

  dijkstra_field          paths.py:21-45 (heapq Dijkstra, float64 sums, strict
                          improvement re-pushes; walkable cells, corner rule)
  sample_route_anchors    urbangen/scene.py:102-158 (+ _traverse_anchor :161-178)
  spawn_pose              envcore/batch.py:183-198

Pinned against tests/golden/routes.npz (oracle/make_golden_routes.py).
"""

import heapq
import math

import numpy as np

from .rng import make_rng
from .scene import chamfer

SQRT2 = math.sqrt(2.0)
MOVES = ((-1, 0, 1.0), (1, 0, 1.0), (0, -1, 1.0), (0, 1, 1.0),
         (-1, -1, SQRT2), (-1, 1, SQRT2), (1, -1, SQRT2), (1, 1, SQRT2))
MAX_ROUTE_ANCHORS, MIN_ANCHOR_CLEARANCE_M, WALKABLE = 8, 0.4, 2


def dijkstra_field(passable, source, res):
    ny, nx = passable.shape
    dist = np.full((ny, nx), np.inf)
    r0, c0 = source
    heap = []
    if passable[r0, c0]:
        dist[r0, c0] = 0.0
        heap.append((0.0, r0, c0))
    while heap:
        d, r, c = heapq.heappop(heap)
        if d > dist[r, c]:
            continue
        for dr, dc, w in MOVES:
            rr, cc = r + dr, c + dc
            if not (0 <= rr < ny and 0 <= cc < nx) or not passable[rr, cc]:
                continue
            if dr and dc and not (passable[r, cc] and passable[rr, c]):
                continue
            nd = d + w
            if nd < dist[rr, cc]:
                dist[rr, cc] = nd
                heapq.heappush(heap, (nd, rr, cc))
    return dist * res


def sample_route_anchors(labels, res, seed, extent, task):
    """scene.py:102-158; returns a list of [[sx, sy], [gx, gy]] (None = NoRouteAvailable)."""
    walk = labels == WALKABLE
    clear = walk & (chamfer(~walk, res) >= MIN_ANCHOR_CLEARANCE_M)
    if not clear.any():
        clear = walk
    if not clear.any():
        return None
    rows, cols = np.nonzero(clear)
    xs, ys = (cols + 0.5) * res, (rows + 0.5) * res
    if task == "Traverse":
        ny, nx = labels.shape
        want_sx, want_gx, cy = 1.5, nx * res - 1.5, ny * res / 2.0
        si = int(np.argmin((xs - want_sx) ** 2 + (ys - cy) ** 2))
        geo = dijkstra_field(walk, (rows[si], cols[si]), res)[rows, cols]
        ok = np.isfinite(geo)
        if not ok.any():
            return None
        gi = int(np.argmin((xs - want_gx) ** 2 + (ys - cy) ** 2 + np.where(ok, 0.0, 1e12)))
        return [[[float(xs[si]), float(ys[si])], [float(xs[gi]), float(ys[gi])]]]
    rng = make_rng(seed, "routes")
    d = float(min(extent))
    windows = [(0.5 * d, 0.8 * d, 1.6), (0.35 * d, 0.8 * d, 2.0), (0.2 * d, 0.9 * d, 4.0)]
    fields = []
    for _ in range(4):
        i = int(rng.integers(rows.size))
        fields.append((i, dijkstra_field(walk, (rows[i], cols[i]), res)[rows, cols]))
    pairs = []
    for lo, hi, cap in windows:
        for i, geo in fields:
            eu = np.sqrt((xs - xs[i]) ** 2 + (ys - ys[i]) ** 2)
            ok = (eu >= lo) & (eu <= hi) & np.isfinite(geo) & (geo <= cap * np.maximum(eu, 1e-9))
            idx = np.flatnonzero(ok)
            for _ in range(min(2, idx.size)):
                j = int(idx[int(rng.integers(idx.size))])
                pairs.append([[float(xs[i]), float(ys[i])], [float(xs[j]), float(ys[j])]])
                if len(pairs) >= MAX_ROUTE_ANCHORS:
                    return pairs
        if pairs:
            return pairs
    return None


def spawn_pick(env_seed, reset_count, n_routes):
    """batch.py:184-186: index of the route the robot spawns on."""
    return int(make_rng(env_seed, "spawn", reset_count).integers(n_routes))
