"""Robot embodiments, the robot part of BatchedEnv.step_batch, and observations
on the device (reference envcore/robot.py, envcore/batch.py:205-302,
envcore/observe.py, bench/reward.py) -- SURVEY §8(f) row 1.

``RobotBatch`` owns the per-env robot state as device tensors (batch.py:98-110)
and the per-model passable map (robot.py:127-179, ``cw_traversability``); its
``step`` runs ``cw_robot_step`` (integrate_motion, gating, crowd contact,
reward, termination, observe_batch) after the caller has stepped the crowd.
There is no host fallback: the ops raise if the library is missing.
"""

from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib


class Embodiment(str, Enum):
    WHEELED = "Wheeled"
    QUADRUPED = "Quadruped"
    WHEELED_LEGGED = "WheeledLegged"
    HUMANOID = "Humanoid"


class KinematicsKind(str, Enum):
    ACKERMANN = "Ackermann"
    HOLONOMIC = "Holonomic"


@dataclass(frozen=True)
class RobotModel:
    """robot.py:31-53 (same fields and validation)."""
    name: str
    embodiment: Embodiment
    body_radius: float
    max_speed: float
    kinematics: KinematicsKind
    wheelbase: float = 0.0
    max_steer: float = 0.0
    max_step_rise: float = 0.25
    max_grade: float = 0.60
    max_roughness: float = 0.15

    def __post_init__(self):
        if self.embodiment == Embodiment.WHEELED and self.kinematics != KinematicsKind.ACKERMANN:
            raise ValueError("wheeled robots use the Ackermann model")
        if self.embodiment != Embodiment.WHEELED and self.kinematics != KinematicsKind.HOLONOMIC:
            raise ValueError("non-wheeled robots are holonomic")
        for f in ("body_radius", "max_speed", "max_step_rise", "max_grade", "max_roughness"):
            if getattr(self, f) <= 0:
                raise ValueError(f"{f} must be > 0")
        if self.kinematics == KinematicsKind.ACKERMANN and (self.wheelbase <= 0 or self.max_steer <= 0):
            raise ValueError("Ackermann needs positive wheelbase and max_steer")

    def to_c(self):
        m = _lib.RobotModel()
        m.body_radius, m.max_speed = self.body_radius, self.max_speed
        m.holonomic = int(self.kinematics == KinematicsKind.HOLONOMIC)
        m.wheelbase, m.max_steer = self.wheelbase, self.max_steer
        m.max_step_rise, m.max_grade, m.max_roughness = self.max_step_rise, self.max_grade, self.max_roughness
        return m


# robot.py:56-80
ROBOT_MODELS = {
    "wheeled": RobotModel("wheeled", Embodiment.WHEELED, 0.35, 2.0, KinematicsKind.ACKERMANN,
                          wheelbase=0.4, max_steer=0.6, max_step_rise=0.05, max_grade=0.15,
                          max_roughness=0.03),
    "quadruped": RobotModel("quadruped", Embodiment.QUADRUPED, 0.35, 2.0, KinematicsKind.HOLONOMIC,
                            max_step_rise=0.25, max_grade=0.60, max_roughness=0.15),
    "wheeled_legged": RobotModel("wheeled_legged", Embodiment.WHEELED_LEGGED, 0.45, 2.0,
                                 KinematicsKind.HOLONOMIC, max_step_rise=0.25, max_grade=0.60,
                                 max_roughness=0.18),
    "humanoid": RobotModel("humanoid", Embodiment.HUMANOID, 0.35, 1.2, KinematicsKind.HOLONOMIC,
                           max_step_rise=0.20, max_grade=0.45, max_roughness=0.12),
}


@dataclass
class RewardConfig:
    """bench/reward.py:15-24."""
    terminal_reach: float = 50.0
    terminal_oob: float = -100.0
    c1: float = 2.0
    c2: float = 0.5
    c3: float = 1.0
    track_scale_far: float = 1.0
    track_scale_near: float = 0.2
    track_near_weight: float = 0.2


EVENT_NAMES = ("collision", "collision_static", "collision_dynamic", "on_walkable", "reached",
               "out_of_bounds")
N_RAYS, HMAP_NX, HMAP_NY = 128, 16, 10


class RobotBatch:
    """Device robot state of E envs over device scene stacks (labels / elevation
    (E, ny, nx)); ``passable`` is computed once per scene (and per resampled row)."""

    def __init__(self, labels, elev, res, model="quadruped", horizon=200, dt=0.05,
                 reach_threshold_m=0.5, reward=None, device=None, semantics=False):
        import torch
        self.labels, self.elev = labels, elev
        self.device = labels.device if device is None else torch.device(device)
        self.E, self.ny, self.nx = (int(v) for v in labels.shape)
        self.res = float(res)
        self.model = ROBOT_MODELS[model] if isinstance(model, str) else model
        self.horizon, self.dt, self.reach = int(horizon), float(dt), float(reach_threshold_m)
        self.reward_cfg = reward or RewardConfig()
        E, d = self.E, self.device
        f64 = dict(dtype=torch.float64, device=d)
        self.x, self.y, self.yaw = (torch.zeros(E, **f64) for _ in range(3))
        self.vx, self.vy, self.el = (torch.zeros(E, **f64) for _ in range(3))
        self.goal = torch.zeros((E, 2), **f64)
        self.tick = torch.zeros(E, dtype=torch.int64, device=d)
        self.terminated = torch.zeros(E, dtype=torch.uint8, device=d)
        self.truncated = torch.zeros(E, dtype=torch.uint8, device=d)
        self.passable = torch.zeros((E, self.ny, self.nx), dtype=torch.uint8, device=d)
        self.reward = torch.zeros(E, **f64)
        self.events = torch.zeros((E, 6), dtype=torch.uint8, device=d)
        self.distance = torch.zeros(E, **f64)
        self.path_inc = torch.zeros(E, **f64)
        self.depth = torch.zeros((E, N_RAYS), dtype=torch.float32, device=d)
        self.goal_vector = torch.zeros((E, 2), **f64)
        self.proj_vel = torch.zeros(E, **f64)
        self.height_map = torch.zeros((E, HMAP_NX, HMAP_NY), dtype=torch.float32, device=d)
        # per-ray hit labels (observe.py:84-85), only when the batch asks for them
        self.semantics = torch.zeros((E, N_RAYS), dtype=torch.uint8, device=d) if semantics else None
        self.refresh_passable()

    # -- traversability (robot.py:127-179) -------------------------------------------
    def _params(self, A=0):
        p = _lib.RobotParams()
        p.E, p.A, p.nx, p.ny = self.E, int(A), self.nx, self.ny
        p.res, p.dt, p.reach_threshold, p.horizon = self.res, self.dt, self.reach, self.horizon
        r = self.reward_cfg
        p.terminal_reach, p.terminal_oob = r.terminal_reach, r.terminal_oob
        p.c1, p.c2, p.c3 = r.c1, r.c2, r.c3
        p.track_far, p.track_near, p.track_near_weight = (r.track_scale_far, r.track_scale_near,
                                                          r.track_near_weight)
        p.model = self.model.to_c()
        return p

    def refresh_passable(self, rows=None):
        """passable map of all rows or of ``rows`` (after a scene resample)."""
        import torch
        sl = None if rows is None else torch.as_tensor(rows, dtype=torch.int32, device=self.device)
        n = self.E if rows is None else int(sl.numel())
        if n == 0:
            return
        L = _lib.lib()
        chunk = min(n, 128)
        scratch = torch.empty(int(L.cw_traversability_scratch_bytes(self.nx, self.ny, chunk)) // 8 + 1,
                              dtype=torch.float64, device=self.device)
        _lib.check(L.cw_traversability(self._params(), n, _lib.ptr(sl), _lib.ptr(self.labels),
                                       _lib.ptr(self.elev), _lib.ptr(self.passable), _lib.ptr(scratch),
                                       chunk, _lib.stream_ptr()), "cw_traversability")

    # -- state ------------------------------------------------------------------------
    def set_state(self, x, y, yaw, goal, vx=0.0, vy=0.0, elev=None, tick=0, terminated=False,
                  truncated=False, rows=None):
        """Install robot poses (host arrays or device tensors) for all rows / ``rows``."""
        import torch
        idx = slice(None) if rows is None else torch.as_tensor(rows, dtype=torch.long, device=self.device)
        t = lambda v, dt=torch.float64: torch.as_tensor(np.asarray(v) if not isinstance(v, torch.Tensor) else v,
                                                          dtype=dt).to(self.device)
        self.x[idx], self.y[idx], self.yaw[idx] = t(x), t(y), t(yaw)
        self.goal[idx] = t(goal).reshape(-1, 2)
        self.vx[idx], self.vy[idx] = t(vx), t(vy)
        if elev is None:   # elevation of the spawn cell (batch.py:194-195)
            rows_all = torch.arange(self.E, device=self.device)[idx]
            r = torch.clamp((self.y[idx] / self.res).long(), 0, self.ny - 1)
            c = torch.clamp((self.x[idx] / self.res).long(), 0, self.nx - 1)
            self.el[idx] = self.elev[rows_all, r, c].double()
        else:
            self.el[idx] = t(elev)
        self.tick[idx] = t(tick, torch.int64)
        self.terminated[idx] = t(terminated, torch.uint8)
        self.truncated[idx] = t(truncated, torch.uint8)
        # distance to the goal at the new pose (batch.py:198 prev_dist): numpy's hypot
        # on the host values (the reference's own call), torch's for device inputs
        if not any(isinstance(v, torch.Tensor) for v in (x, y, goal)):
            g = np.asarray(goal, np.float64).reshape(-1, 2)
            d = np.hypot(g[:, 0] - np.asarray(x, np.float64), g[:, 1] - np.asarray(y, np.float64))
            self.distance[idx] = torch.from_numpy(np.ascontiguousarray(d)).to(self.device)
        else:
            self.distance[idx] = torch.hypot(self.goal[idx, 0] - self.x[idx], self.goal[idx, 1] - self.y[idx])

    def live(self):
        return (self.terminated == 0) & (self.truncated == 0)

    def _state(self, crowd=None):
        s = _lib.RobotState()
        m = dict(x=self.x, y=self.y, yaw=self.yaw, vx=self.vx, vy=self.vy, elev=self.el, goal=self.goal,
                 tick=self.tick, terminated=self.terminated, truncated=self.truncated, labels=self.labels,
                 grid_elev=self.elev, passable=self.passable, reward=self.reward, events=self.events,
                 distance=self.distance, path_inc=self.path_inc, depth=self.depth,
                 goal_vector=self.goal_vector, proj_vel=self.proj_vel, height_map=self.height_map)
        for k, v in m.items():
            setattr(s, k, v.data_ptr())
        if self.semantics is not None:
            s.semantics = self.semantics.data_ptr()
        if crowd is not None:
            pos, radius, active = crowd
            s.crowd_pos, s.crowd_radius, s.crowd_active = pos.data_ptr(), radius.data_ptr(), active.data_ptr()
        return s

    # -- stepping (batch.py:223-302) ---------------------------------------------------
    def step(self, actions, crowd=None):
        """Robot part of a tick after the crowd step.  ``actions`` (E, 2) device or host;
        ``crowd`` = (pos (E, A, 2), radius (E, A), active (E, A) uint8) device tensors
        after the crowd step, or None.  Outputs land in the batch's tensors."""
        import torch
        a = actions if isinstance(actions, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(np.asarray(actions, np.float64)))
        a = a.to(device=self.device, dtype=torch.float64).reshape(self.E, 2).contiguous()
        A = 0 if crowd is None else int(crowd[0].shape[1])
        _lib.check(_lib.lib().cw_robot_step(self._params(A), self._state(crowd if A else None),
                                            _lib.ptr(a), _lib.stream_ptr()), "cw_robot_step")

    def observe(self):
        _lib.check(_lib.lib().cw_robot_observe(self._params(), self._state(), _lib.stream_ptr()),
                   "cw_robot_observe")

    def outputs(self):
        """Device views of the last tick's outputs (no host copies)."""
        return dict(reward=self.reward, events=self.events, distance=self.distance, path_inc=self.path_inc,
                    depth=self.depth, goal_vector=self.goal_vector, proj_vel=self.proj_vel,
                    height_map=self.height_map, terminated=self.terminated, truncated=self.truncated,
                    semantics=self.semantics)
