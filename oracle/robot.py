"""Oracle (TEST INFRASTRUCTURE ONLY): numpy restatement of the reference's robot
step, traversability gating, reward and observations -- SURVEY §8(f) row 1.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module; the product path never does.  Pinned against tests/golden/robot_*.npz
(generated from the unmodified reference by oracle/make_golden_robot.py).

  integrate_motion     envcore/robot.py:94-124
  traversability_maps  envcore/robot.py:127-179
  reward_batch         bench/reward.py:29-53
  observe_batch        envcore/observe.py:39-129
  RobotBatch.step      envcore/batch.py:205-302 (robot part; the crowd is stepped
                       by the caller with the pre-step robot pos/vel, batch.py:216-221)
"""

from dataclasses import dataclass

import numpy as np

TWO_PI = 2.0 * np.pi
YAW_RATE_LIMIT = TWO_PI
L_OBSTACLE, L_WALKABLE = 0, 2


@dataclass(frozen=True)
class Model:
    body_radius: float
    max_speed: float
    holonomic: bool
    wheelbase: float = 0.0
    max_steer: float = 0.0
    max_step_rise: float = 0.25
    max_grade: float = 0.60
    max_roughness: float = 0.15


# robot.py:56-80
MODELS = {
    "wheeled": Model(0.35, 2.0, False, 0.4, 0.6, 0.05, 0.15, 0.03),
    "quadruped": Model(0.35, 2.0, True, 0.0, 0.0, 0.25, 0.60, 0.15),
    "wheeled_legged": Model(0.45, 2.0, True, 0.0, 0.0, 0.25, 0.60, 0.18),
    "humanoid": Model(0.35, 1.2, True, 0.0, 0.0, 0.20, 0.45, 0.12),
}


def integrate_motion(x, y, yaw, a0, a1, m, dt):
    """robot.py:94-124 (vectorised over envs)."""
    if m.holonomic:
        ex = a0 * m.max_speed
        ey = a1 * m.max_speed
        c, s = np.cos(yaw), np.sin(yaw)
        vx = c * ex - s * ey
        vy = s * ex + c * ey
        nx = x + vx * dt
        ny = y + vy * dt
        speed = np.hypot(vx, vy)
        target = np.where(speed > 1e-9, np.arctan2(vy, vx), yaw)
        dyaw = np.arctan2(np.sin(target - yaw), np.cos(target - yaw))
        lim = YAW_RATE_LIMIT * dt
        dyaw = np.clip(dyaw, -lim, lim)
        return nx, ny, yaw + dyaw, vx, vy
    v = a0 * m.max_speed
    steer = a1 * m.max_steer
    nyaw = yaw + v * np.tan(steer) / m.wheelbase * dt
    vx = v * np.cos(yaw)
    vy = v * np.sin(yaw)
    return x + vx * dt, y + vy * dt, nyaw, vx, vy


def traversability_maps(labels, elevation, res, m):
    """robot.py:127-179: step rise to the 4 neighbours, 5x5 box mean via a column-
    then-row float64 cumulative sum of the edge-padded grid, grade of the box
    surface (central differences, hypot), roughness |elev - box|."""
    e = elevation.astype(np.float64)
    ny, nx = e.shape
    step = np.zeros_like(e)
    for dr, dc in ((1, 0), (-1, 0), (0, 1), (0, -1)):
        nb = np.full_like(e, np.nan)
        rs, re_ = max(dr, 0), ny + min(dr, 0)
        cs, ce = max(dc, 0), nx + min(dc, 0)
        nb[rs:re_, cs:ce] = e[rs - dr:re_ - dr, cs - dc:ce - dc]
        with np.errstate(invalid="ignore"):
            step = np.fmax(step, np.abs(e - nb))
    p = np.pad(e, 2, mode="edge")
    cum = np.zeros((ny + 5, nx + 5))
    cum[1:, 1:] = np.cumsum(np.cumsum(p, axis=0), axis=1)
    box = (cum[5:, 5:] - cum[:-5, 5:] - cum[5:, :-5] + cum[:-5, :-5]) / 25
    rough = np.abs(e - box)
    gx = np.zeros_like(e)
    gy = np.zeros_like(e)
    gx[:, 1:-1] = (box[:, 2:] - box[:, :-2]) / (2 * res)
    gy[1:-1, :] = (box[2:, :] - box[:-2, :]) / (2 * res)
    grade = np.hypot(gx, gy)
    obstacle = labels == L_OBSTACLE
    passable = ~(obstacle | (step > m.max_step_rise) | (grade > m.max_grade) | (rough > m.max_roughness))
    return dict(passable=passable, obstacle=obstacle, step=step.astype(np.float32),
                grade=grade.astype(np.float32), rough=rough.astype(np.float32))


# bench/reward.py:15-24 defaults
R_REACH, R_OOB, C1, C2, C3 = 50.0, -100.0, 2.0, 0.5, 1.0


def reward_batch(d, off_walk, coll, reached, oob):
    """bench/reward.py:29-53."""
    track = (1.0 - np.tanh(d / 1.0)) + 0.2 * (1.0 - np.tanh(d / 0.2))
    term = np.where(reached, R_REACH, 0.0) + np.where(oob, R_OOB, 0.0)
    return term + C1 * track + C2 * np.where(off_walk, -1.0, 0.0) + C3 * np.where(coll, -1.0, 0.0)


N_RAYS, FAN, CAP = 128, np.pi / 4.0, 10.0
HX_N, HY_N, HL, HW = 16, 10, 1.6, 1.0


def ray_offsets():
    """np.linspace(-pi/4, pi/4, 128) (observe.py:23)."""
    step = (2 * FAN) / (N_RAYS - 1)
    o = np.arange(N_RAYS, dtype=np.float64) * step + (-FAN)
    o[-1] = FAN
    return o


def observe(x, y, yaw, goal, vel, elev_r, labels, elev, res, rise):
    """observe.py:39-129 for K robots, one scene per robot (labels/elev (K, ny, nx)):
    float32 ray march in res steps to 10 m stopping at obstacles or rises above
    `rise`; goal vector in the ego frame; velocity projected on the goal
    direction; 16 x 10 ego-aligned relative height patch."""
    K = x.shape[0]
    _, gny, gnx = labels.shape
    ang = (yaw[:, None] + ray_offsets()[None, :]).astype(np.float32)
    dx, dy = np.cos(ang), np.sin(ang)
    ox = x.astype(np.float32)[:, None]
    oy = y.astype(np.float32)[:, None]
    prev = np.broadcast_to(elev_r.astype(np.float32)[:, None], (K, N_RAYS)).copy()
    alive = np.ones((K, N_RAYS), bool)
    depth = np.full((K, N_RAYS), np.float32(CAP), np.float32)
    sem = np.zeros((K, N_RAYS), np.uint8)   # observe.py:49, 84-85: hit cell's label, else 0
    inv = np.float32(1.0 / res)
    lim = np.float32(rise)
    el32 = elev.astype(np.float32)
    ki = np.arange(K)[:, None]
    for k in range(1, int(CAP / res) + 1):
        if not alive.any():
            break
        t = np.float32(k * res)
        px = ox + dx * t
        py = oy + dy * t
        cc = (px * inv).astype(np.int64)
        rr = (py * inv).astype(np.int64)
        inside = (cc >= 0) & (cc < gnx) & (rr >= 0) & (rr < gny)
        r0, c0 = np.where(inside, rr, 0), np.where(inside, cc, 0)
        lab = labels[ki, r0, c0]
        el = el32[ki, r0, c0]
        wall = alive & inside & ((lab == L_OBSTACLE) | (el - prev > lim))
        depth[wall] = t
        sem[wall] = lab[wall]
        alive &= inside & ~wall
        prev = np.where(alive, el, prev)
    gvx, gvy = goal[:, 0] - x, goal[:, 1] - y
    c, s = np.cos(yaw), np.sin(yaw)
    gvec = np.stack([c * gvx + s * gvy, -s * gvx + c * gvy], axis=-1)
    pvel = (vel[:, 0] * gvx + vel[:, 1] * gvy) / np.maximum(np.hypot(gvx, gvy), 1e-12)
    hx = ((np.arange(HX_N) + 0.5) / HX_N * HL)
    hy = ((np.arange(HY_N) + 0.5) / HY_N * HW - HW / 2.0)
    HX, HY = np.meshgrid(hx, hy, indexing="ij")
    hx, hy = HX.ravel()[None, :], HY.ravel()[None, :]
    wx = x[:, None] + c[:, None] * hx - s[:, None] * hy
    wy = y[:, None] + s[:, None] * hx + c[:, None] * hy
    hc = np.clip((wx / res).astype(np.int64), 0, gnx - 1)
    hr = np.clip((wy / res).astype(np.int64), 0, gny - 1)
    hin = (wx >= 0) & (wx < gnx * res) & (wy >= 0) & (wy < gny * res)
    hm = np.where(hin, elev[ki, hr, hc] - elev_r[:, None], 0.0)
    return dict(depth=depth, goal_vector=gvec, proj_vel=pvel,
                height_map=hm.reshape(K, HX_N, HY_N).astype(np.float32), semantics=sem)


class RobotBatch:
    """Robot state of K envs + the robot part of BatchedEnv.step_batch."""

    def __init__(self, labels, elev, res, model, horizon=200, dt=0.05, reach=0.5):
        self.labels, self.elev, self.res = labels, elev, res
        self.m = MODELS[model] if isinstance(model, str) else model
        maps = [traversability_maps(labels[i], elev[i], res, self.m) for i in range(labels.shape[0])]
        self.passable = np.stack([q["passable"] for q in maps])
        self.obstacle = np.stack([q["obstacle"] for q in maps])
        self.horizon, self.dt, self.reach = horizon, dt, reach
        K = labels.shape[0]
        z = lambda: np.zeros(K)
        self.x, self.y, self.yaw, self.vx, self.vy, self.el = z(), z(), z(), z(), z(), z()
        self.goal = np.zeros((K, 2))
        self.tick = np.zeros(K, np.int64)
        self.terminated = np.zeros(K, bool)
        self.truncated = np.zeros(K, bool)

    def step(self, actions, crowd_pos=None, crowd_radius=None, crowd_active=None):
        """batch.py:223-302 after the crowd step; crowd_* are the post-step crowd."""
        a = np.clip(np.asarray(actions, np.float64), -1.0, 1.0)
        live = ~(self.terminated | self.truncated)
        nx, ny, nyaw, nvx, nvy = integrate_motion(self.x, self.y, self.yaw, a[:, 0], a[:, 1],
                                                  self.m, self.dt)
        K, gny, gnx = self.labels.shape
        res = self.res
        w_m, l_m = gnx * res, gny * res
        inside = (nx >= 0) & (nx < w_m) & (ny >= 0) & (ny < l_m)
        rr = np.clip((ny / res).astype(np.int64), 0, gny - 1)
        cc = np.clip((nx / res).astype(np.int64), 0, gnx - 1)
        ki = np.arange(K)
        blocked = inside & ~self.passable[ki, rr, cc]
        coll_static = blocked & self.obstacle[ki, rr, cc]
        hit = np.zeros(K, bool)
        if crowd_pos is not None and crowd_pos.shape[1] > 0:
            d2 = ((crowd_pos - np.stack([nx, ny], -1)[:, None, :]) ** 2).sum(-1)
            rsum = crowd_radius + self.m.body_radius
            hit = ((d2 < rsum ** 2) & crowd_active).any(axis=1)
            blocked = blocked | hit
        coll = coll_static | hit
        move = live & inside & ~blocked
        frozen = live & blocked
        go = move | (live & ~inside)
        self.x = np.where(go, nx, self.x)
        self.y = np.where(go, ny, self.y)
        self.yaw = np.where(live, nyaw, self.yaw)
        self.vx = np.where(move, nvx, np.where(frozen, 0.0, self.vx))
        self.vy = np.where(move, nvy, np.where(frozen, 0.0, self.vy))
        self.vx = np.where(live, self.vx, 0.0)
        self.vy = np.where(live, self.vy, 0.0)
        r2 = np.clip((self.y / res).astype(np.int64), 0, gny - 1)
        c2 = np.clip((self.x / res).astype(np.int64), 0, gnx - 1)
        in_now = (self.x >= 0) & (self.x < w_m) & (self.y >= 0) & (self.y < l_m)
        self.el = np.where(in_now, self.elev[ki, r2, c2], self.el)
        on_walk = in_now & (self.labels[ki, r2, c2] == L_WALKABLE)
        dist = np.hypot(self.goal[:, 0] - self.x, self.goal[:, 1] - self.y)
        pinc = np.where(live, np.hypot(self.vx * self.dt, self.vy * self.dt), 0.0)
        reached = live & (dist <= self.reach)
        oob = live & ~in_now
        rew = np.where(live, reward_batch(dist, live & ~on_walk, live & coll, reached, oob), 0.0)
        self.tick = np.where(live, self.tick + 1, self.tick)
        self.terminated = self.terminated | reached | oob
        self.truncated = self.truncated | (live & (self.tick >= self.horizon) & ~oob)
        ev = dict(collision=live & coll, collision_static=live & coll_static,
                  collision_dynamic=live & hit, on_walkable=on_walk, reached=reached,
                  out_of_bounds=oob, distance=dist, path_inc=pinc)
        obs = observe(self.x, self.y, self.yaw, self.goal, np.stack([self.vx, self.vy], -1), self.el,
                      self.labels, self.elev, res, self.m.max_step_rise)
        return rew, ev, obs
