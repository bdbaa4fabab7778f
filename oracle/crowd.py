"""Crowd oracle: per-env prep, spawn/routes, and the batched ORCA step
(test infrastructure only -- see oracle/__init__.py).

Restates /root/reference/pkg/src/citywalk/crowd/{field,orca,routes,step}.py
and paths.astar_path op-for-op in float64 (the fp32 neighbour key included).
Where the reference goes through OpenBLAS (``@`` on 2-vectors, the fp32
Gram matrix) the explicit measured formula is used:
  * 1-D float64 dot of length 2:  fma(a1, b1, a0*b0)
  * fp32 Gram entry:              fma(y_i, y_j, x_i*x_j)
and ``np.hypot`` is glibc's hypot (non-FMA Borges kernel), which numpy calls.
"""

import heapq
import math
from collections import deque

import numpy as np

from .rng import make_rng
from .scene import OBSTACLE, WALKABLE, fma

EPS = 1e-12
GOAL_REACH = 0.3
WAYPOINT_REACH = 0.5
STRAY_LIMIT = 1.0
STALL_BIAS = 0.6
SQRT2 = float(np.sqrt(2.0))
MAX_SPEED = (2.0, 5.0, 4.0)          # crowd/types.py:15-19
PREF_RANGE = ((0.8, 1.4), (2.0, 4.0), (1.5, 3.0))   # types.py:22-26
RADIUS = (0.3, 0.45, 0.4)            # types.py:28-32
NEIGH8 = ((1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (1, -1), (-1, 1), (-1, -1))


class Config:
    """crowd/types.py:59-79 defaults."""

    def __init__(self, time_horizon=2.0, obstacle_time_horizon=1.0, neighbor_distance=5.0,
                 max_neighbors=10, dt=0.05, safety_margin=0.03):
        self.time_horizon = time_horizon
        self.obstacle_time_horizon = obstacle_time_horizon
        self.neighbor_distance = neighbor_distance
        self.max_neighbors = max_neighbors
        self.dt = dt
        self.safety_margin = safety_margin


def dot2(a0, a1, b0, b1):
    """numpy ``a @ b`` for float64 2-vectors (OpenBLAS ddot)."""
    return fma(a1, b1, a0 * b0)


def hypot(x, y):
    """glibc __hypot (the non-FMA kernel numpy reaches through libm)."""
    ax, ay = abs(float(x)), abs(float(y))
    if ax < ay:
        ax, ay = ay, ax
    if ay <= ax * 2.0 ** -54:
        return ax + ay
    if ay < 2.0 ** -511 or ax > 2.0 ** 511:
        return math.hypot(ax, ay)   # never reached on this path's magnitudes
    h = math.sqrt(ax * ax + ay * ay)
    if h <= 2.0 * ay:
        de = h - ay
        t1 = ax * (2.0 * de - ax)
        t2 = (de - 2.0 * (ax - ay)) * de
    else:
        de = h - ax
        t1 = 2.0 * de * (ax - 2.0 * ay)
        t2 = (4.0 * de - ay) * ay + de * de
    return h - (t1 + t2) / (2.0 * h)


# -- per-env preparation (field.py:60-67, 571-593) ----------------------------------

def nearest_obstacle_map(labels):
    """FIFO multi-source BFS over all cells; flat index of the first
    discovering obstacle, or None when there is no obstacle.  field.py:571-593."""
    ny, nx = labels.shape
    obs = labels == OBSTACLE
    if not obs.any():
        return None
    near = np.full(ny * nx, -1, np.int64)
    q = deque()
    for f in np.flatnonzero(obs.ravel()).tolist():
        near[f] = f
        q.append(f)
    while q:
        f = q.popleft()
        r, c = divmod(f, nx)
        src = near[f]
        for dr, dc in NEIGH8:
            rr, cc = r + dr, c + dc
            if 0 <= rr < ny and 0 <= cc < nx and near[rr * nx + cc] < 0:
                near[rr * nx + cc] = src
                q.append(rr * nx + cc)
    return near.reshape(ny, nx)


def walk_cells(labels, res):
    rows, cols = np.nonzero(labels == WALKABLE)
    return np.stack([(cols + 0.5) * res, (rows + 0.5) * res], axis=1)


def components(ok):
    """8-connected component id per cell (-1 elsewhere); routes.py:14-32."""
    ny, nx = ok.shape
    comp = np.full((ny, nx), -1, np.int32)
    nid = 0
    for r0, c0 in zip(*np.nonzero(ok)):
        if comp[r0, c0] >= 0:
            continue
        comp[r0, c0] = nid
        q = deque([(int(r0), int(c0))])
        while q:
            r, c = q.popleft()
            for dr, dc in NEIGH8:
                rr, cc = r + dr, c + dc
                if 0 <= rr < ny and 0 <= cc < nx and ok[rr, cc] and comp[rr, cc] < 0:
                    comp[rr, cc] = nid
                    q.append((rr, cc))
        nid += 1
    return comp


def sample_routes(labels, res, count, seed, max_radius):
    """routes.py:35-87 for pedestrian routing on WALKABLE cells.

    Returns (start (count,2), goal (count,2), start_flat, goal_flat)."""
    if count == 0:
        return np.zeros((0, 2)), np.zeros((0, 2)), [], []
    rng = np.random.Generator(np.random.PCG64(seed))
    ok = labels == WALKABLE
    rows, cols = np.nonzero(ok)
    if rows.size < count:
        raise ValueError("NoRouteAvailable: too few candidate cells")
    comp = components(ok)[rows, cols]
    xs = (cols + 0.5) * res
    ys = (rows + 0.5) * res
    sep2 = (2.0 * max_radius) ** 2
    starts, goals, sf, gf = [], [], [], []
    for idx in rng.permutation(rows.size):
        if len(starts) >= count:
            break
        sx, sy = float(xs[idx]), float(ys[idx])
        if any((sx - ox) ** 2 + (sy - oy) ** 2 < sep2 for ox, oy in starts):
            continue
        cand = np.flatnonzero((comp == comp[idx]) & ((xs - sx) ** 2 + (ys - sy) ** 2 >= sep2))
        if cand.size == 0:
            continue
        j = int(cand[int(rng.integers(cand.size))])
        starts.append((sx, sy))
        goals.append((float(xs[j]), float(ys[j])))
        sf.append(int(rows[idx]) * labels.shape[1] + int(cols[idx]))
        gf.append(int(rows[j]) * labels.shape[1] + int(cols[j]))
    if len(starts) < count:
        raise ValueError("NoRouteAvailable: separation")
    return np.array(starts), np.array(goals), sf, gf


def spawn_agents(labels, res, count, seed):
    """step.py:37-63.  Returns a dict of per-agent arrays."""
    rng = make_rng(seed, "crowd-spawn")
    kinds = []
    for _ in range(count):
        u = rng.random()
        kinds.append(0 if u < 0.7 else (1 if u < 0.9 else 2))
    max_r = max(RADIUS[k] for k in kinds) if kinds else 0.3
    st, gl, sf, gf = sample_routes(labels, res, count, int(rng.integers(2 ** 63)), max_r)
    pref = [float(rng.uniform(*PREF_RANGE[k])) for k in kinds]
    return {
        "pos": st, "goal": gl, "kind": np.array(kinds, np.int8),
        "radius": np.array([RADIUS[k] for k in kinds]),
        "pref": np.array(pref), "max_speed": np.array([MAX_SPEED[k] for k in kinds]),
        "start_flat": np.array(sf, np.int64), "goal_flat": np.array(gf, np.int64),
    }


# -- guidance helpers (field.py:596-625, paths.py:48-87) ------------------------------

def astar(passable, start, goal):
    """paths.py:48-87: 8-connected, no corner cutting, heap on (f, h, r, c)."""
    ny, nx = passable.shape
    sr, sc = start
    gr, gc = goal
    if not (passable[sr, sc] and passable[gr, gc]):
        return None

    def h(r, c):
        dr, dc = abs(r - gr), abs(c - gc)
        return SQRT2 * min(dr, dc) + abs(dr - dc)

    g = {(sr, sc): 0.0}
    parent = {}
    h0 = h(sr, sc)
    heap = [(h0, h0, sr, sc)]
    moves = ((-1, 0, 1.0), (1, 0, 1.0), (0, -1, 1.0), (0, 1, 1.0),
             (-1, -1, SQRT2), (-1, 1, SQRT2), (1, -1, SQRT2), (1, 1, SQRT2))
    while heap:
        f, _, r, c = heapq.heappop(heap)
        if (r, c) == (gr, gc):
            path = [(r, c)]
            while (r, c) in parent:
                r, c = parent[(r, c)]
                path.append((r, c))
            return path[::-1]
        if f > g[(r, c)] + h(r, c) + 1e-12:
            continue
        for dr, dc, w in moves:
            rr, cc = r + dr, c + dc
            if not (0 <= rr < ny and 0 <= cc < nx) or not passable[rr, cc]:
                continue
            if dr and dc and not (passable[r, cc] and passable[rr, c]):
                continue
            ng = g[(r, c)] + w
            if ng < g.get((rr, cc), math.inf) - 1e-12:
                g[(rr, cc)] = ng
                parent[(rr, cc)] = (r, c)
                hh = h(rr, cc)
                heapq.heappush(heap, (ng + hh, hh, rr, cc))
    return None


def linspace01(n):
    """np.linspace(0.0, 1.0, n) for n >= 2."""
    step = 1.0 / (n - 1)
    t = np.arange(n, dtype=np.float64) * step + 0.0
    t[-1] = 1.0
    return t


def line_of_sight(passable, a, b, res):
    """field.py:601-610."""
    ny, nx = passable.shape
    d = hypot(b[0] - a[0], b[1] - a[1])
    n = max(2, int(2.0 * d / res) + 2)
    ts = linspace01(n)
    xs = a[0] + (b[0] - a[0]) * ts
    ys = a[1] + (b[1] - a[1]) * ts
    rr = np.clip((ys / res).astype(np.int64), 0, ny - 1)
    cc = np.clip((xs / res).astype(np.int64), 0, nx - 1)
    return bool(passable[rr, cc].all())


def dist_to_polyline(p, pts):
    """field.py:613-625."""
    px, py = float(p[0]), float(p[1])
    q = (px, py) if len(pts) == 0 else pts[0]
    best = min(math.inf, hypot(q[0] - px, q[1] - py))
    for k in range(1, len(pts)):
        ax, ay = pts[k - 1]
        bx, by = pts[k]
        abx, aby = bx - ax, by - ay
        den = dot2(abx, aby, abx, aby)
        if den < EPS:
            t = 0.0
        else:
            t = float(np.clip(dot2(px - ax, py - ay, abx, aby) / den, 0.0, 1.0))
        best = min(best, hypot(ax + t * abx - px, ay + t * aby - py))
    return best


# -- half-planes and the LP (field.py:448-566, orca.py:155-242) -------------------------

def vo_halfplane(rp, rv, rr, horizon, dt, vs, share):
    """Vectorised VO half-plane, field.py:448-495 (op order preserved).
    rp, rv, vs: (..., 2); rr: (...)."""
    with np.errstate(invalid="ignore", divide="ignore"):
        rp0, rp1 = rp[..., 0], rp[..., 1]
        rv0, rv1 = rv[..., 0], rv[..., 1]
        dsq = rp0 * rp0 + rp1 * rp1
        rsq = rr * rr
        coll = dsq <= rsq
        w0 = rv0 - rp0 / horizon
        w1 = rv1 - rp1 / horizon
        wlsq = w0 * w0 + w1 * w1
        d1 = w0 * rp0 + w1 * rp1
        cut = (d1 < 0.0) & (d1 * d1 > rsq * wlsq)
        wl = np.sqrt(wlsq)
        wsafe = np.maximum(wl, EPS)
        uw0, uw1 = w0 / wsafe, w1 / wsafe
        kc = rr / horizon - wl
        leg = np.sqrt(np.maximum(dsq - rsq, 0.0))
        det = rp0 * w1 - rp1 * w0
        sg = np.where(det > 0.0, 1.0, -1.0)
        sd2 = np.maximum(dsq, EPS)
        ld0 = (rp0 * leg - sg * rp1 * rr) / sd2
        ld1 = (sg * rp0 * rr + rp1 * leg) / sd2
        nl0, nl1 = -sg * ld1, sg * ld0
        d2v = rv0 * ld0 + rv1 * ld1
        ul0, ul1 = d2v * ld0 - rv0, d2v * ld1 - rv1
        wc0 = rv0 - rp0 / dt
        wc1 = rv1 - rp1 / dt
        wcl = np.sqrt(wc0 * wc0 + wc1 * wc1)
        dist = np.sqrt(dsq)
        dsafe = np.maximum(dist, EPS)
        pu0, pu1 = -rp0 / dsafe, -rp1 / dsafe
        wcs = np.maximum(wcl, EPS)
        big = wcl > EPS
        uc0 = np.where(big, wc0 / wcs, pu0)
        uc1 = np.where(big, wc1 / wcs, pu1)
        deg = (wcl <= EPS) & (dist <= EPS)
        uc0 = np.where(deg, 1.0, uc0)
        uc1 = np.where(deg, 0.0, uc1)
        kk = rr / dt - wcl
        uo0, uo1 = kk * uc0, kk * uc1
        u0 = np.where(coll, uo0, np.where(cut, kc * uw0, ul0))
        u1 = np.where(coll, uo1, np.where(cut, kc * uw1, ul1))
        n0 = np.where(coll, uc0, np.where(cut, uw0, nl0))
        n1 = np.where(coll, uc1, np.where(cut, uw1, nl1))
        pt = np.stack([vs[..., 0] + share * u0, vs[..., 1] + share * u1], axis=-1)
        return pt, np.stack([n0, n1], axis=-1)


def batched_lp(points, normals, valid, pref, max_speed, lane_active):
    """field.py:500-566 (row by row; identical arithmetic)."""
    N, L = valid.shape
    out = np.zeros((N, 2))
    for row in range(N):
        out[row] = _lp_row(points[row], normals[row], valid[row], pref[row],
                           float(max_speed[row]), bool(lane_active[row]))
    return out


def _lp_row(P, Nm, V, pref, ms, active):
    p0, p1 = float(pref[0]), float(pref[1])
    pn = math.sqrt(p0 * p0 + p1 * p1)
    sc = ms / max(pn, EPS) if pn > ms else 1.0
    r0, r1 = p0 * sc, p1 * sc
    if not active:
        return r0, r1
    L = len(V)
    for i in range(L):
        if not V[i]:
            continue
        pi0, pi1 = float(P[i, 0]), float(P[i, 1])
        ni0, ni1 = float(Nm[i, 0]), float(Nm[i, 1])
        if not ((r0 - pi0) * ni0 + (r1 - pi1) * ni1 < -EPS):
            continue
        d0, d1 = -ni1, ni0
        dpd = pi0 * d0 + pi1 * d1
        disc = dpd * dpd + ms * ms - (pi0 * pi0 + pi1 * pi1)
        bad = disc < 0.0
        sq = math.sqrt(max(disc, 0.0))
        tl, tr = -dpd - sq, -dpd + sq
        for j in range(i):
            if not V[j]:
                continue
            nj0, nj1 = float(Nm[j, 0]), float(Nm[j, 1])
            den = d0 * nj0 + d1 * nj1
            num = (float(P[j, 0]) - pi0) * nj0 + (float(P[j, 1]) - pi1) * nj1
            par = abs(den) < EPS
            if par:
                bad |= num > EPS
                continue
            t = num / den
            if den > 0.0:
                tl = max(tl, t)
            else:
                tr = min(tr, t)
        bad |= tl > tr
        if bad:
            lanes = [k for k in range(L) if V[k]]
            cons = [(float(P[k, 0]), float(P[k, 1]), float(Nm[k, 0]), float(Nm[k, 1]))
                    for k in lanes]
            return least_violation(cons, lanes.index(i), ms, (r0, r1))
        tb = (p0 - pi0) * d0 + (p1 - pi1) * d1
        tb = min(max(tb, tl), tr)
        r0, r1 = pi0 + tb * d0, pi1 + tb * d1
    return r0, r1


def _viol(hp, v):
    return -dot2(v[0] - hp[0], v[1] - hp[1], hp[2], hp[3])


def _solve_on_line(cons, i, ms, opt, dir_opt):
    """orca.py:155-189."""
    px, py, nx_, ny_ = cons[i]
    dx, dy = -ny_, nx_
    dpd = dot2(px, py, dx, dy)
    disc = dpd * dpd + ms * ms - dot2(px, py, px, py)
    if disc < 0.0:
        return None
    sq = math.sqrt(disc)
    tl, tr = -dpd - sq, -dpd + sq
    for j in range(i):
        qx, qy, mx, my = cons[j]
        den = dot2(dx, dy, mx, my)
        num = dot2(qx - px, qy - py, mx, my)
        if abs(den) < EPS:
            if num > EPS:
                return None
            continue
        t = num / den
        if den > 0.0:
            tl = max(tl, t)
        else:
            tr = min(tr, t)
        if tl > tr:
            return None
    if dir_opt:
        tb = tr if dot2(opt[0], opt[1], dx, dy) > 0.0 else tl
    else:
        tb = float(np.clip(dot2(opt[0] - px, opt[1] - py, dx, dy), tl, tr))
    return (px + tb * dx, py + tb * dy)


def _lp2_toward(cons, ms, od):
    """orca.py:215-224."""
    s = ms / max(hypot(od[0], od[1]), EPS)
    res = (od[0] * s, od[1] * s)
    for i, hp in enumerate(cons):
        if dot2(res[0] - hp[0], res[1] - hp[1], hp[2], hp[3]) < -EPS:
            new = _solve_on_line(cons, i, ms, od, True)
            if new is None:
                return None
            res = new
    return res


def least_violation(cons, begin, ms, result):
    """orca.py:196-212 (3-D lifted fallback)."""
    dist = 0.0
    for i in range(begin, len(cons)):
        pix, piy, nix, niy = cons[i]
        if _viol(cons[i], result) <= dist + EPS:
            continue
        proj = []
        for j in range(i):
            pjx, pjy, njx, njy = cons[j]
            det = nix * njy - niy * njx
            dfx, dfy = njx - nix, njy - niy
            if abs(det) < EPS:
                if dot2(nix, niy, njx, njy) > 0.0:
                    continue
                mx, my = 0.5 * (pix + pjx), 0.5 * (piy + pjy)
            else:
                dix, diy = -niy, nix
                t = dot2(pjx - pix, pjy - piy, njx, njy) / dot2(dix, diy, njx, njy)
                mx, my = pix + t * dix, piy + t * diy
            nrm = hypot(dfx, dfy)
            if nrm < EPS:
                continue
            proj.append((mx, my, dfx / nrm, dfy / nrm))
        new = _lp2_toward(proj, ms, (nix, niy))
        if new is not None:
            result = new
        dist = _viol(cons[i], result)
    return result


# -- the batched field (field.py:26-163, 214-381) ----------------------------------------

class CrowdFieldOracle:
    """CrowdField restated; state arrays share the reference's names/shapes."""

    def __init__(self, grids, cfg, env_seeds, resample_goals=True):
        """grids: list of (labels uint8 (ny,nx), resolution)."""
        self.cfg = cfg
        self.grids = list(grids)
        self.E = len(self.grids)
        self.resample_goals = resample_goals
        self.rngs = [np.random.Generator(np.random.PCG64(int(s))) for s in env_seeds]
        self.walk = [walk_cells(lb, r) for lb, r in self.grids]
        self.passable = [lb != OBSTACLE for lb, _ in self.grids]
        self.nearest = [nearest_obstacle_map(lb) for lb, _ in self.grids]
        self.has_obstacles = any(m is not None for m in self.nearest)
        self.last_gap_by_env = np.full(self.E, np.inf)
        self._alloc(0)

    def _alloc(self, A):
        E = self.E
        self.A = A
        self.pos = np.zeros((E, A, 2))
        self.vel = np.zeros((E, A, 2))
        self.goal = np.zeros((E, A, 2))
        self.waypoint = np.zeros((E, A, 2))
        self.radius = np.full((E, A), 0.3)
        self.pref_speed = np.full((E, A), 1.0)
        self.max_speed = np.full((E, A), 2.0)
        self.kind = np.zeros((E, A), np.int8)
        self.active = np.zeros((E, A), bool)
        self.paths = [[None] * A for _ in range(E)]

    def set_agents(self, per_env):
        """per_env: list of dicts with pos, goal, radius, pref, max_speed, kind (+ vel)."""
        A = max((len(d["pos"]) for d in per_env), default=0)
        self._alloc(A)
        for e, d in enumerate(per_env):
            n = len(d["pos"])
            self.pos[e, :n] = d["pos"]
            self.vel[e, :n] = d.get("vel", np.zeros((n, 2)))
            self.goal[e, :n] = d["goal"]
            self.waypoint[e, :n] = d["goal"]
            self.radius[e, :n] = d["radius"]
            self.pref_speed[e, :n] = d["pref"]
            self.max_speed[e, :n] = d["max_speed"]
            self.kind[e, :n] = d["kind"]
            self.active[e, :n] = True

    # ---------------------------------------------------------------- step
    def step(self, robot_pos=None, robot_vel=None, robot_radius=0.35, env_mask=None):
        if self.A == 0 or self.E == 0:
            return
        act = self.active.copy()
        if env_mask is not None:
            act &= np.asarray(env_mask, bool)[:, None]
        if not act.any():
            return
        cfg = self.cfg
        E, A = self.E, self.A
        self._guidance(act)
        pref = self._pref(act)
        P, Nm, V = self._constraints(act, robot_pos, robot_vel, robot_radius)
        ms = self.max_speed.reshape(-1)
        nv = batched_lp(P, Nm, V, pref, ms, act.reshape(-1))
        spd = np.sqrt(nv[:, 0] * nv[:, 0] + nv[:, 1] * nv[:, 1])
        want = np.sqrt(pref[:, 0] * pref[:, 0] + pref[:, 1] * pref[:, 1])
        stalled = act.reshape(-1) & (spd < 0.2 * want) & (want > 1e-6)
        rows = np.flatnonzero(stalled)
        if rows.size:
            c, s = np.cos(STALL_BIAS), np.sin(STALL_BIAS)
            pr = np.stack([c * pref[rows, 0] + s * pref[rows, 1],
                           -s * pref[rows, 0] + c * pref[rows, 1]], axis=-1)
            nv[rows] = batched_lp(P[rows], Nm[rows], V[rows], pr, ms[rows],
                                  np.ones(rows.size, bool))
        nv = nv.reshape(E, A, 2)
        nv[~act] = self.vel[~act]
        newp = self.pos + nv * cfg.dt
        blocked = np.zeros((E, A), bool)
        for e in range(E):
            lb, res = self.grids[e]
            ny, nx = lb.shape
            x, y = newp[e, :, 0], newp[e, :, 1]
            out = (x < 0) | (y < 0) | (x >= nx * res) | (y >= ny * res)
            rr = np.clip((y / res).astype(np.int64), 0, ny - 1)
            cc = np.clip((x / res).astype(np.int64), 0, nx - 1)
            blocked[e] = out | ~self.passable[e][rr, cc]
        commit = act & ~blocked
        self.pos[commit] = newp[commit]
        self.vel[act] = nv[act]
        self.vel[act & blocked] = 0.0
        if self.resample_goals:
            d2 = ((self.goal - self.pos) ** 2).sum(-1)
            hit = act & (d2 < GOAL_REACH ** 2)
            for e in range(E):
                for a in np.flatnonzero(hit[e]):
                    k = int(self.rngs[e].integers(len(self.walk[e])))
                    self.goal[e, a] = self.walk[e][k]
                    self.paths[e][a] = None

    def _guidance(self, act):
        """field.py:165-212."""
        for e in range(self.E):
            if self.nearest[e] is None:
                self.waypoint[e][act[e]] = self.goal[e][act[e]]
                continue
            lb, res = self.grids[e]
            ps = self.passable[e]
            ny, nx = ps.shape
            for a in range(self.A):
                if not act[e, a]:
                    continue
                p = self.pos[e, a]
                path = self.paths[e][a]
                if path is not None and len(path) > 0:
                    wp = path[0]
                    if hypot(wp[0] - p[0], wp[1] - p[1]) < WAYPOINT_REACH and len(path) > 1:
                        path.pop(0)
                    if dist_to_polyline(p, path) <= STRAY_LIMIT:
                        self.waypoint[e, a] = path[0]
                        continue
                g = self.goal[e, a]
                gt = (float(g[0]), float(g[1]))
                if line_of_sight(ps, p, g, res):
                    self.paths[e][a] = [gt]
                    self.waypoint[e, a] = g
                    continue
                st = (int(np.clip(p[1] / res, 0, ny - 1)), int(np.clip(p[0] / res, 0, nx - 1)))
                en = (int(np.clip(g[1] / res, 0, ny - 1)), int(np.clip(g[0] / res, 0, nx - 1)))
                cells = astar(ps, st, en)
                if cells is None or len(cells) < 2:
                    self.paths[e][a] = [gt]
                    self.waypoint[e, a] = g
                    continue
                pts = [((c + 0.5) * res, (r + 0.5) * res) for r, c in cells[1:]]
                pts.append(gt)
                self.paths[e][a] = pts
                self.waypoint[e, a] = pts[0]

    def _pref(self, act):
        """field.py:214-227."""
        tw = self.waypoint - self.pos
        dist = np.sqrt(tw[..., 0] * tw[..., 0] + tw[..., 1] * tw[..., 1])
        safe = np.maximum(dist, EPS)
        sp = self.pref_speed
        pref = tw / safe[..., None] * sp[..., None]
        tg = self.goal - self.pos
        dg = np.sqrt(tg[..., 0] * tg[..., 0] + tg[..., 1] * tg[..., 1])
        scale = np.minimum(1.0, dg / np.maximum(sp * self.cfg.dt * 4, EPS))
        pref = pref * scale[..., None]
        pref[~act] = 0.0
        return pref.reshape(-1, 2)

    def neighbour_keys(self, act):
        """fp32 Gram key (field.py:246-254): fma(y_i,y_j,x_i*x_j) in fp32."""
        p32 = self.pos.astype(np.float32)
        x, y = p32[..., 0], p32[..., 1]
        sq = x * x + y * y
        xl, yl = x.astype(np.longdouble), y.astype(np.longdouble)
        xx = (xl[:, :, None] * xl[:, None, :]).astype(np.float32)
        dot = (yl[:, :, None] * yl[:, None, :] + xx.astype(np.longdouble)).astype(np.float32)
        d2 = sq[:, :, None] + sq[:, None, :] - np.float32(2.0) * dot
        inf32 = np.float32(np.inf)
        d2 = d2 + np.where(act, np.float32(0), inf32)[:, None, :]
        d2 = d2 + np.where(act, np.float32(0), inf32)[:, :, None]
        i = np.arange(self.A)
        d2[:, i, i] = inf32
        return d2

    def _constraints(self, act, robot_pos, robot_vel, robot_radius):
        """field.py:229-350."""
        cfg = self.cfg
        E, A = self.E, self.A
        N = E * A
        pos, vel, rad = self.pos, self.vel, self.radius
        K = min(cfg.max_neighbors, max(A - 1, 0))
        nb = None
        if K > 0:
            d2 = self.neighbour_keys(act)
            inr = d2 < np.float32(cfg.neighbor_distance ** 2)
            K = min(K, int(inr.sum(-1).max(initial=0)))
            if K > 0:
                key = np.where(inr, d2, np.float32(np.inf))
                order = np.argsort(key, axis=-1, kind="stable")[..., :K]
                ok = np.isfinite(np.take_along_axis(key, order, axis=-1))
                ie = np.arange(E)[:, None, None]
                npos, nvel, nrad = pos[ie, order], vel[ie, order], rad[ie, order]
                dx = npos[:, :, 0, 0] - pos[..., 0]
                dy = npos[:, :, 0, 1] - pos[..., 1]
                gap = np.where(ok[:, :, 0], np.sqrt(dx * dx + dy * dy) - (rad + nrad[:, :, 0]), np.inf)
                self.last_gap_by_env[:] = gap.min(axis=1)
                rp = npos - pos[:, :, None, :]
                rv = vel[:, :, None, :] - nvel
                rr = rad[:, :, None] + nrad + cfg.safety_margin
                vs = np.broadcast_to(vel[:, :, None, :], rp.shape)
                pt, nm = vo_halfplane(rp, rv, rr, cfg.time_horizon, cfg.dt, vs, 0.5)
                pt = np.where(ok[..., None], pt, 0.0)
                nm = np.where(ok[..., None], nm, np.array([1.0, 0.0]))
                nb = (pt.reshape(N, K, 2), nm.reshape(N, K, 2), ok.reshape(N, K))
        use_robot = robot_pos is not None
        use_static = self.has_obstacles
        L = max(K + int(use_robot) + int(use_static), 1)
        P = np.zeros((N, L, 2))
        Nm = np.zeros((N, L, 2))
        Nm[..., 0] = 1.0
        V = np.zeros((N, L), bool)
        if nb is not None:
            P[:, :K], Nm[:, :K], V[:, :K] = nb
        lane = K
        if use_robot:
            rpp = np.asarray(robot_pos, np.float64).reshape(E, 1, 2)
            rvv = (np.zeros((E, 1, 2)) if robot_vel is None
                   else np.asarray(robot_vel, np.float64).reshape(E, 1, 2))
            rp = rpp - pos
            d2r = rp[..., 0] * rp[..., 0] + rp[..., 1] * rp[..., 1]
            ok = act & (d2r < cfg.neighbor_distance ** 2)
            rr = rad + robot_radius + cfg.safety_margin
            pt, nm = vo_halfplane(rp, vel - rvv, rr, cfg.obstacle_time_horizon, cfg.dt, vel, 1.0)
            P[:, lane], Nm[:, lane], V[:, lane] = pt.reshape(N, 2), nm.reshape(N, 2), ok.reshape(N)
            lane += 1
        if use_static:
            opt = np.zeros((E, A, 2))
            ook = np.zeros((E, A), bool)
            for e in range(E):
                near = self.nearest[e]
                if near is None:
                    continue
                lb, res = self.grids[e]
                ny, nx = lb.shape
                ri = np.clip((pos[e, :, 1] / res).astype(np.int64), 0, ny - 1)
                ci = np.clip((pos[e, :, 0] / res).astype(np.int64), 0, nx - 1)
                flat = near[ri, ci]
                orow, ocol = np.divmod(np.maximum(flat, 0), nx)
                opt[e, :, 0] = (ocol + 0.5) * res
                opt[e, :, 1] = (orow + 0.5) * res
                ook[e] = (flat >= 0) & act[e]
            rp = opt - pos
            d2o = rp[..., 0] * rp[..., 0] + rp[..., 1] * rp[..., 1]
            ook &= d2o < cfg.neighbor_distance ** 2
            margin = 0.5 * np.sqrt(2.0) * self.grids[0][1]
            rr = rad + margin + cfg.safety_margin
            pt, nm = vo_halfplane(rp, vel, rr, cfg.obstacle_time_horizon, cfg.dt, vel, 1.0)
            P[:, lane], Nm[:, lane], V[:, lane] = pt.reshape(N, 2), nm.reshape(N, 2), ook.reshape(N)
        return P, Nm, V
