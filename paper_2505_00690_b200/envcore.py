"""Batched env orchestration for the hot path (envcore/batch.py:62-346, cache.py).

``BatchedEnv`` keeps the reference constructor and seed tree -- per-env seeds
``child_seed(master, "env", i)`` (batch.py:84-96), crowd streams
``child_seed(env_seed, "crowd-run")`` (:165), spawns
``child_seed(env_seed, "crowd", reset_count)`` (:179), resample seeds
``child_seed(env_seed, "resample", n)`` (:332) -- but samples every env on the
device in one batch and steps the crowd with one kernel per tick.
``step_batch`` (batch.py:205-302) runs the crowd tick with the robot lane, then
the robot step, reward and observations on the device (``robot.RobotBatch``);
``step_batch_device`` is the same tick without host copies.

The robot spawns on one of the scene's route anchors (scene.py:102-178, sampled
on the device by ``cw_route_anchors``) exactly as ``batch.py:183-198`` picks it;
``set_robot_state`` installs any other poses.
"""

from dataclasses import dataclass, field, replace
from enum import Enum

import numpy as np

from . import _lib
from .crowd import CrowdConfig, CrowdField, DeviceView
from .errors import BatchShapeMismatch, SlotOutOfRange
from .rng import child_seed, child_seeds_device, seeds_to_tensor
from .robot import EVENT_NAMES, ROBOT_MODELS, RewardConfig, RobotBatch
from .urbangen import SceneSampler, SceneSpec, as_spec


class _SlotSeq:
    """Read-only per-slot sequence whose elements are built on access."""

    def __init__(self, n, get):
        self._n, self._get = int(n), get

    def __len__(self):
        return self._n

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(self._n))]
        i = int(i)
        if i < 0:
            i += self._n
        if not 0 <= i < self._n:
            raise IndexError(i)
        return self._get(i)

    def __iter__(self):
        return (self._get(i) for i in range(self._n))


class Scheme(str, Enum):
    ASYNC = "Async"
    SYNC = "Sync"


@dataclass
class EnvConfig:
    """batch.py:39-49."""
    robot: str = "quadruped"
    horizon: int = 200
    dt: float = 0.05
    auto_reset: bool = False
    resample_on_reset: bool = False
    reach_threshold_m: float = 0.5
    include_semantics: bool = False
    reward: RewardConfig = field(default_factory=RewardConfig)
    crowd: CrowdConfig = field(default_factory=CrowdConfig)


@dataclass
class Observation:
    """observe.py:30-36."""
    depth: np.ndarray
    goal_vector: np.ndarray
    projected_velocity: float
    height_map: np.ndarray
    semantics: np.ndarray = None


@dataclass
class StepResult:
    """batch.py:52-58."""
    observation: Observation
    reward: float
    terminated: bool
    truncated: bool
    events: dict


class BatchedEnv:
    """K env slots: device scenes + device crowd (batch.py:62).

    ``cache`` (an ``AssetCache``, cache.py:15-39) is accepted for API parity: every
    slot is sampled on the device in one batch, and equal specs give bit-identical
    rows (the Sync scheme's shared scene), so nothing is looked up; the scenes'
    identities are ``scene_hashes`` either way."""

    def __init__(self, specs, scheme, master_seed, k=None, cache=None, config=None,
                 env_seeds=None, device="cuda", threads=None, catalog=None, standby=False):
        import torch
        self.config = config or EnvConfig()
        self.scheme = Scheme(scheme)
        if hasattr(specs, "to_dict"):
            k = 1 if k is None else k
            base = as_spec(specs)
        else:
            specs = [as_spec(s) for s in specs]
            k = len(specs)
            base = specs[0]
            if any(replace(s, seed=0) != replace(base, seed=0) for s in specs):
                raise ValueError("a device batch needs one SceneSpec shape (seeds may differ)")
        if k < 1:
            raise ValueError("K must be >= 1")
        self.K = k
        self.master_seed = int(master_seed)
        self.device = torch.device(device)
        if env_seeds is None:
            env_seeds = [child_seed(master_seed, "env", i) for i in range(k)]
        if len(env_seeds) != k:
            raise ValueError("env_seeds must have length K")
        self.env_seeds = [int(s) for s in env_seeds]
        self.cache = cache
        self.env_seeds_t = seeds_to_tensor(self.env_seeds, self.device)
        if self.scheme == Scheme.SYNC:
            if self.config.resample_on_reset:
                raise ValueError("resample_on_reset requires the Async scheme")
            self.scene_seeds_t = self.env_seeds_t[:1].expand(k).contiguous()
        else:
            self.scene_seeds_t = self.env_seeds_t.clone()
        self.spec = replace(base, seed=self.env_seeds[0])
        self.reset_counts = np.zeros(k, dtype=np.int64)
        self.sampler = SceneSampler(self.spec, k, catalog, device)
        self._scene_hashes = [None] * k
        crowd_seeds = child_seeds_device(self.env_seeds_t, "crowd", 0)
        self.batch = self.sampler.sample(self.scene_seeds_t, crowd_seeds)
        run = child_seeds_device(self.env_seeds_t, "crowd-run").cpu().numpy().view(np.uint64)
        self.crowd = CrowdField(self.batch, self.config.crowd, [int(s) for s in run],
                                device=device, threads=threads)
        if self.spec.pedestrian_count > 0:
            self.crowd.set_from_spawn(self.batch)
        self.model = ROBOT_MODELS[self.config.robot]
        self.robot = RobotBatch(self.batch.labels, self.batch.elev, self.resolution, self.model,
                                horizon=self.config.horizon, dt=self.config.dt,
                                reach_threshold_m=self.config.reach_threshold_m,
                                reward=self.config.reward, device=self.device,
                                semantics=self.config.include_semantics)
        self._spawn(np.arange(k))
        # standby: every slot's next scene (and its crowd's first replans) sampled ahead on
        # side streams, so resample() installs instead of sampling (SceneStandby)
        self.standby = None
        if standby and self.scheme == Scheme.ASYNC:
            self.counts_t = torch.zeros(k, dtype=torch.int64, device=self.device)
            self.standby = SceneStandby(self.sampler, self.env_seeds_t, self.counts_t,
                                        field=self.crowd if self.spec.pedestrian_count > 0 else None)

    # -- stacks (batch.py:132-150) ----------------------------------------------------
    @property
    def labels_stack(self):
        return self.batch.labels

    @property
    def elev_stack(self):
        return self.batch.elev

    @property
    def resolution(self):
        return float(self.batch.params.res)

    @property
    def extent(self):
        """batch.py:148-149: (width, length) in metres of the grids."""
        return (int(self.batch.labels.shape[2]) * self.resolution,
                int(self.batch.labels.shape[1]) * self.resolution)

    @property
    def specs(self):
        """batch.py:90-96: each slot's SceneSpec (Sync: the shared one)."""
        if self.scheme == Scheme.SYNC:
            return [replace(self.spec, seed=self.env_seeds[0])] * self.K
        return [replace(self.spec, seed=s) for s in self.env_seeds]

    @property
    def env_index(self):
        """batch.py:137-141: the scene row of each slot (rows are per slot on the device;
        under Sync every row holds the shared scene, so slot i reads row i)."""
        if self.scheme == Scheme.SYNC:
            return np.zeros(self.K, dtype=np.int64)
        return np.arange(self.K, dtype=np.int64)

    @property
    def passable_stack(self):
        """batch.py:145 traversability ``passable`` per slot (device tensor)."""
        return self.robot.passable

    @property
    def obstacle_stack(self):
        """batch.py:146 traversability ``obstacle`` (labels == OBSTACLE) per slot (device)."""
        return self.batch.labels == 0

    # distance to the goal after the last step / at reset (batch.py:114, 198, 280)
    prev_dist = property(lambda self: DeviceView(self.robot.distance))

    @property
    def occs(self):
        """batch.py:99, 129: every slot's OccupancyGrid -- host copies of the slot's device
        raster, taken when an element is read (so they follow re-sampling)."""
        return _SlotSeq(self.K, self.batch.occupancy)

    @property
    def scenes(self):
        """batch.py:98, 128: every slot's SceneDescription (zones, terrain, objects, routes),
        rebuilt from the device batch when an element is read."""
        return _SlotSeq(self.K, lambda i: self.batch.scene(i, self.spec, self.sampler.catalog))

    @property
    def scene_hashes(self):
        """scene_hash of every slot's current scene (batch.py:100, 130): computed
        on first use from the device batch and refreshed for resampled slots."""
        stale = [i for i, h in enumerate(self._scene_hashes) if h is None]
        if stale:
            for i, h in zip(stale, self.sampler.scene_hashes(stale)):
                self._scene_hashes[i] = h
        return list(self._scene_hashes)

    # -- resample / reset (batch.py:326-346) --------------------------------------------
    def resample(self, slots, respawn=True):
        """Re-sample the scenes of ``slots`` (Async) and respawn their crowds; the
        cfg5 driver calls this with the Bernoulli-selected subset each step."""
        import torch
        slots = np.asarray(slots, dtype=np.int64).reshape(-1)
        if slots.size == 0:
            return
        if self.scheme == Scheme.SYNC:
            raise ValueError("resample_on_reset requires the Async scheme")
        if (slots < 0).any() or (slots >= self.K).any():
            raise SlotOutOfRange(f"slots outside [0, {self.K})")
        self.reset_counts[slots] += 1
        sl = torch.from_numpy(slots).to(self.device)
        env = self.env_seeds_t[sl]
        cnt = torch.from_numpy(self.reset_counts[slots]).to(self.device)
        new_scene = child_seeds_device(env, "resample", cnt)
        self.scene_seeds_t[sl] = new_scene
        if self.standby is not None and (respawn or self.spec.pedestrian_count == 0):
            self.counts_t[sl] += 1
            self.standby.take(slots)   # installs the scenes (+ set_from_spawn of their crowds)
            self.batch.check_status(sl)
        else:
            if self.standby is not None:
                self.counts_t[sl] += 1
            crowd_seed = child_seeds_device(env, "crowd", cnt)
            self.sampler.sample(new_scene, crowd_seed, slots=sl)
            if respawn and self.spec.pedestrian_count > 0:
                self.crowd.set_from_spawn(self.batch, rows=sl)
            if self.standby is not None:
                self.standby._launch(slots)   # the rows' standby is now their next-but-one
        for i in slots:
            self._scene_hashes[int(i)] = None
        self.crowd.prepare_step()
        if hasattr(self, "robot"):
            self.robot.refresh_passable(slots)
            if respawn:
                self._spawn(slots)

    def reset(self, slot, resample=None):
        if not (0 <= slot < self.K):
            raise SlotOutOfRange(f"slot {slot} of {self.K}")
        do_resample = self.config.resample_on_reset if resample is None else resample
        if do_resample:
            self.resample([slot])
            return self.observe(slot)
        import torch
        self.reset_counts[slot] += 1
        sl = torch.tensor([slot], device=self.device)
        cseed = child_seeds_device(self.env_seeds_t[sl], "crowd",
                                   torch.tensor([int(self.reset_counts[slot])], device=self.device))
        p = self.sampler.params
        b = self.batch
        err = _lib.lib().cw_spawn_agents(p, 1, _lib.ptr(cseed), _lib.ptr(sl.to(torch.int32)),
                                         _lib.ptr(b.seed_scratch), b.buffers(), _lib.stream_ptr())
        _lib.check(err, "cw_spawn_agents")
        b.check_status(sl)
        self.crowd.set_from_spawn(b, rows=sl)
        self._spawn([slot])
        return self.observe(slot)

    # -- robot spawn / state (batch.py:183-198, 352-361) --------------------------------
    def _spawn(self, rows):
        """batch.py:183-198: route = make_rng(env_seed, "spawn", reset_count).integers(
        len(routes)) of the scene's route anchors (cw_route_anchors); yaw toward the
        goal, elevation of the start cell."""
        rows = np.asarray(rows, dtype=np.int64).reshape(-1)
        if rows.size == 0:
            return
        routes = self.batch.routes[rows].cpu().numpy()
        nr = self.batch.n_routes[rows].cpu().numpy()
        xs, ys, yaws, goals = [], [], [], []
        for i, e in enumerate(rows):
            g = np.random.Generator(np.random.PCG64(
                child_seed(self.env_seeds[e], "spawn", int(self.reset_counts[e]))))
            (sx, sy), (gx, gy) = routes[i, int(g.integers(int(nr[i])))]
            xs.append(float(sx))
            ys.append(float(sy))
            yaws.append(float(np.arctan2(gy - sy, gx - sx)))
            goals.append((float(gx), float(gy)))
        self.robot.set_state(np.array(xs), np.array(ys), np.array(yaws), np.array(goals), rows=rows)

    def set_robot_state(self, x, y, yaw, goal, vx=0.0, vy=0.0, elev=None, tick=0, rows=None):
        """Install robot poses (e.g. the reference's route-anchor spawns)."""
        self.robot.set_state(x, y, yaw, goal, vx=vx, vy=vy, elev=elev, tick=tick, rows=rows)

    # robot state arrays as the reference exposes them (batch.py:98-110): DeviceView
    # windows onto the device tensors (reads copy to the host, item assignment
    # writes through, e.g. ``env.goal[0] = (x, y)``)
    x = property(lambda self: DeviceView(self.robot.x))
    y = property(lambda self: DeviceView(self.robot.y))
    yaw = property(lambda self: DeviceView(self.robot.yaw))
    vx = property(lambda self: DeviceView(self.robot.vx))
    vy = property(lambda self: DeviceView(self.robot.vy))
    elev = property(lambda self: DeviceView(self.robot.el))
    goal = property(lambda self: DeviceView(self.robot.goal))
    tick = property(lambda self: DeviceView(self.robot.tick))
    terminated = property(lambda self: DeviceView(self.robot.terminated, bool))
    truncated = property(lambda self: DeviceView(self.robot.truncated, bool))

    def robot_state(self, i=0):
        r = self.robot
        return {"x": float(r.x[i]), "y": float(r.y[i]), "yaw": float(r.yaw[i]), "vx": float(r.vx[i]),
                "vy": float(r.vy[i]), "elevation": float(r.el[i]),
                "goal": [float(r.goal[i, 0]), float(r.goal[i, 1])], "tick": int(r.tick[i])}

    # -- stepping -------------------------------------------------------------------------
    def step_crowd(self, robot_pos=None, robot_vel=None, robot_radius=0.35, env_mask=None,
                   check=False):
        self.crowd.step(robot_pos=robot_pos, robot_vel=robot_vel, robot_radius=robot_radius,
                        env_mask=env_mask, check=check)

    def step_batch_device(self, actions, check=False):
        """One control step of every live slot on the device (batch.py:205-302) with
        no host synchronisation; returns the RobotBatch output tensors."""
        import torch
        if self.config.auto_reset:
            done = ((self.robot.terminated != 0) | (self.robot.truncated != 0)).nonzero().flatten()
            for i in done.cpu().numpy():
                self._reset_state(int(i))
        live = self.robot.live()
        if self.crowd.A > 0:
            rp = torch.stack([self.robot.x, self.robot.y], -1)
            rv = torch.stack([self.robot.vx, self.robot.vy], -1)
            self.crowd.step(robot_pos=rp, robot_vel=rv, robot_radius=self.model.body_radius,
                            env_mask=live.to(torch.uint8), check=check)
            self.robot.step(actions, (self.crowd.pos_t, self.crowd.radius_t, self.crowd.active_t))
        else:
            self.robot.step(actions)
        return self.robot.outputs()

    def step_batch(self, actions, workers=1):
        """batch.py:205-302: list of StepResult (host copies of the device outputs)."""
        acts = np.asarray(actions, dtype=np.float64)
        if acts.shape != (self.K, 2):
            raise BatchShapeMismatch(f"expected ({self.K}, 2) actions, got {acts.shape}")
        live = self.robot.live().cpu().numpy() if not self.config.auto_reset else None
        out = self.step_batch_device(acts, check=True)
        if live is None:
            live = np.ones(self.K, bool)
        h = {k: v.cpu().numpy() for k, v in out.items() if v is not None}
        sem = h.get("semantics")
        results = []
        for i in range(self.K):
            ev = {n: bool(h["events"][i, j]) for j, n in enumerate(EVENT_NAMES)}
            ev["distance_to_goal"] = float(h["distance"][i])
            ev["path_increment"] = float(h["path_inc"][i])
            obs = Observation(depth=h["depth"][i], goal_vector=h["goal_vector"][i],
                              projected_velocity=float(h["proj_vel"][i]), height_map=h["height_map"][i],
                              semantics=None if sem is None else sem[i])
            results.append(StepResult(observation=obs, reward=float(h["reward"][i]),
                                      terminated=bool(h["terminated"][i]), truncated=bool(h["truncated"][i]),
                                      events=ev))
        return results

    def _reset_state(self, slot, resample=None):
        do_resample = self.config.resample_on_reset if resample is None else resample
        if do_resample:
            self.resample([slot])
        else:
            self.reset(slot, resample=False)

    def observe(self, i=0):
        if not (0 <= i < self.K):
            raise SlotOutOfRange(f"slot {i} of {self.K}")
        self.robot.observe()
        r = self.robot
        return Observation(depth=r.depth[i].cpu().numpy(), goal_vector=r.goal_vector[i].cpu().numpy(),
                           projected_velocity=float(r.proj_vel[i]), height_map=r.height_map[i].cpu().numpy(),
                           semantics=None if r.semantics is None else r.semantics[i].cpu().numpy())


_SCENE_OUT = None


def _scene_out_fields():
    """SceneBatch outputs a re-sampled row consists of (everything but scratch)."""
    global _SCENE_OUT
    if _SCENE_OUT is None:
        _SCENE_OUT = [n for n in _lib.SCENE_BUFFER_FIELDS if not n.startswith("scratch") and n not in ("region", "epoch")] + [
            "routes", "n_routes", "scene_seed"]
    return _SCENE_OUT


class SceneStandby:
    """Asynchronous scene sampling for per-tick re-sampling: every row's *next* scene --
    the one its next reset draws, seeds child_seed(env, "resample", count + 1) and
    child_seed(env, "crowd", count + 1) (batch.py:326-339) -- is sampled ahead into a
    pool batch on a side stream.  A reset then installs the row's standby scene with a
    few row copies and starts sampling the row's following one, which runs beside the
    crowd ticks instead of in front of them.  The scenes are the ones re-sampling at the
    reset would produce (same seeds, same kernels): only the time they are made changes.

    ``sampler``: the main SceneSampler (its batch receives the scenes); ``env_seeds``
    (E,) int64 device tensor; ``counts`` (E,) int64 device tensor of reset counts, read
    when a standby is sampled (the caller increments it at each reset, as BatchedEnv
    does).  With ``field`` (the CrowdField over the main batch, next-tick prefetch on),
    the first tick's replans of every standby crowd are predicted and searched on the
    side stream as well (cw_spec_predict: the first guidance pass after a spawn depends
    only on the spawn and the grid) and installed with the scene (cw_spec_install), so a
    re-sampled env's first tick finds its searches done.  ``take`` then also respawns
    the rows' crowds (``field.set_from_spawn``)."""

    def __init__(self, sampler, env_seeds, counts, field=None):
        import ctypes
        import torch
        b = sampler.batch
        self.main, self.env, self.counts = sampler, env_seeds, counts
        self.device = b.device
        self.pool = SceneSampler(sampler.spec, b.E, catalog=sampler.catalog, device=self.device,
                                 routes=sampler.routes)
        self.side = torch.cuda.Stream(device=self.device)
        self.pred = torch.cuda.Stream(device=self.device)   # first-tick predictions (never waited for)
        self.events = []                               # one per sampling launch
        self.row_launch = np.full(b.E, -1, dtype=np.int64)
        self.field = field
        self._spec = None
        if field is not None and field.prefetch and field.A > 0:
            field.prepare_step()
            pb = self.pool.batch
            E, A = field.E, field.A
            d = self.device
            # the crowd state a spawn leaves (set_from_spawn) over the standby grids
            self._pool_keep = dict(active=torch.ones((E, A), dtype=torch.uint8, device=d),
                                   path_n=torch.zeros((E, A), dtype=torch.int32, device=d),
                                   env_req=torch.zeros((E,), dtype=torch.uint8, device=d))
            st = _lib.CrowdState()
            m = dict(pos=pb.sp_pos, goal=pb.sp_goal, waypoint=pb.sp_goal, vel=pb.sp_goal, active=self._pool_keep["active"],
                     path_cells=field.path_cells_t, path_head=self._pool_keep["path_n"],
                     path_n=self._pool_keep["path_n"], labels=pb.labels, nearest=pb.nearest, has_obs=pb.has_obs,
                     walk=pb.walk, walk_n=pb.walk_n, reach=pb.reach, moves=pb.moves, env_req=self._pool_keep["env_req"],
                     env_epoch=pb.epoch)
            for k, v in m.items():
                setattr(st, k, v.data_ptr())
            self._pool_state = st
            self._params = field._params()
            h = ctypes.c_void_p()
            _lib.check(_lib.lib().cw_spec_create(self._params, ctypes.byref(h)), "cw_spec_create")
            self._spec = h.value
        self._launch(np.arange(b.E))

    def __del__(self):
        try:
            if self._spec:
                _lib.lib().cw_spec_destroy(self._spec)
        except Exception:
            pass

    def _launch(self, rows):
        import torch
        self.side.wait_stream(torch.cuda.current_stream())   # the rows' previous standby is installed
        with torch.cuda.stream(self.side):                  # (every tensor below lives on the side stream)
            sl = torch.as_tensor(rows, dtype=torch.int64, device=self.device)
            env_k = self.env[sl]
            cnt = self.counts[sl] + 1
            self.pool.sample(child_seeds_device(env_k, "resample", cnt), child_seeds_device(env_k, "crowd", cnt),
                             slots=sl, stream=self.side, check=False)
            rows32 = sl.to(torch.int32)
            ev = torch.cuda.Event()
            ev.record(self.side)
        self.row_launch[rows] = len(self.events)
        self.events.append(ev)
        if self._spec:
            # on their own stream: a take waits for the scenes only and installs the
            # predictions finished by then (a later rewrite of a row changes its generation)
            self.pred.wait_event(ev)
            rows32.record_stream(self.pred)
            _lib.check(_lib.lib().cw_spec_predict(self._params, self._pool_state, self._spec, _lib.ptr(rows32),
                                                  len(rows), self.field._step_nt(), _lib.stream_ptr(self.pred)),
                       "cw_spec_predict")

    def take(self, rows):
        """Install the standby scenes of ``rows`` (whose reset count was just incremented)
        into the main batch on the current stream, then sample their next ones."""
        import torch
        rows = np.asarray(rows, dtype=np.int64).reshape(-1)
        if rows.size == 0:
            return
        # the side stream runs its launches in order: the latest one among the rows covers all
        torch.cuda.current_stream().wait_event(self.events[int(self.row_launch[rows].max())])
        sl = torch.as_tensor(rows, dtype=torch.int64, device=self.device)
        dst, src = self.main.batch, self.pool.batch
        for name in _scene_out_fields():
            getattr(dst, name).index_copy_(0, sl, getattr(src, name).index_select(0, sl))
        f = self.field
        if f is not None:
            f.set_from_spawn(dst, rows=sl)
            if self._spec and f._spec_handle():
                rows32 = sl.to(torch.int32)
                _lib.check(_lib.lib().cw_spec_install(f._spec_h, self._spec, _lib.ptr(f.epoch_t),
                                                      _lib.ptr(self.pool.batch.epoch), _lib.ptr(rows32), len(rows),
                                                      _lib.stream_ptr()), "cw_spec_install")
        self._launch(rows)


def run_with_resampling(sampler, field, env_seeds, counts, events, ticks, robot_pos=None, robot_vel=None,
                        robot_radius=0.35, window=5, overlap=False):
    """``ticks`` crowd ticks of every env where env e's scene is re-sampled before
    tick t for every e in ``events[t]`` (the bench's cfg5 driver):
    re-sample seed ``child_seed(env_seed, "resample", n)``, crowd respawn seed
    ``child_seed(env_seed, "crowd", n)`` with n the env's running count (``counts``,
    int64 device tensor, updated in place) -- the same state as re-sampling and
    stepping tick by tick (``batch.py:326-339`` + ``CrowdField.step``).

    Runs in windows of ``window`` ticks (``cw_crowd_run_window`` segments): inside a
    window every env advances without a barrier to the window's end or to its next
    re-sampling tick; at the window boundary the envs stopped at a re-sampling tick
    get their new scene and respawn, and catch up in the next window.  The envs due
    at a boundary are known when its window starts (next re-sampling tick <= window
    end), so with ``overlap`` their scenes are sampled into a pool batch on a side
    stream while the window runs and copied into their rows at the boundary (off by
    default: the sampling kernels compete with the run for the SMs, measured slower).
    Returns the number of re-sampled scenes."""
    import torch
    from .urbangen import SceneSampler
    dev = field.device
    E = field.E
    batch = sampler.batch
    ev_ticks = [[] for _ in range(E)]
    for t in range(ticks):
        for e in np.asarray(events[t], dtype=np.int64).reshape(-1):
            ev_ticks[int(e)].append(t)
    nxt = np.zeros(E, dtype=np.int64)            # index of each env's next event
    cur = np.zeros(E, dtype=np.int64)            # each env's next tick
    env_t = env_seeds if isinstance(env_seeds, torch.Tensor) else seeds_to_tensor(env_seeds, dev)
    first, resampled = True, 0
    windows = rounds = samples = servers = 0
    w_end = 0
    saved = field.run_server_warps
    field.run_server_warps = saved or 4   # respawned envs plan every agent: search bursts
    field.prepare_step()

    def next_ev():
        return np.array([ev_ticks[e][nxt[e]] if nxt[e] < len(ev_ticks[e]) else ticks for e in range(E)],
                        dtype=np.int64)

    def resample_now(rows):
        nonlocal resampled, samples
        sl = torch.as_tensor(rows, dtype=torch.int64, device=dev)
        counts[sl] += 1
        env_k = env_t[sl]
        sampler.sample(child_seeds_device(env_k, "resample", counts[sl]),
                       child_seeds_device(env_k, "crowd", counts[sl]), slots=sl, check=False)
        field.set_from_spawn(batch, rows=sl)
        nxt[rows] += 1
        resampled += len(rows)
        samples += 1

    side = torch.cuda.Stream(device=dev) if overlap else None
    pool = None
    pending = None                               # (env rows, pool stream event) sampled ahead
    while True:
        if pending is not None:                  # boundary: install the scenes sampled ahead
            rows, done = pending
            torch.cuda.current_stream().wait_event(done)
            sl = torch.as_tensor(rows, dtype=torch.int64, device=dev)
            k = len(rows)
            for name in _scene_out_fields():
                getattr(batch, name).index_copy_(0, sl, getattr(pool.batch, name)[:k])
            counts[sl] += 1
            field.set_from_spawn(batch, rows=sl)
            nxt[rows] += 1
            resampled += k
            pending = None
        nev = next_ev()
        due = np.flatnonzero((nev == cur) & (nev < ticks))   # re-sampling tick reached (or tick 0)
        if due.size:
            resample_now(due)
            nev = next_ev()
        if (cur >= ticks).all():
            break
        w_end = min(ticks, max(w_end + window, int(cur.min()) + 1))
        stop = np.maximum(cur, np.minimum(nev, np.maximum(w_end, cur)))
        if overlap:
            ahead = np.flatnonzero((nev > cur) & (nev <= w_end) & (nev < ticks))
            if ahead.size:
                if pool is None or pool.batch.E < ahead.size:
                    cap = max(int(ahead.size * 1.5), 64)
                    pool = SceneSampler(sampler.spec, cap, catalog=sampler.catalog, device=dev,
                                        routes=sampler.routes)
                sl = torch.as_tensor(ahead, dtype=torch.int64, device=dev)
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    env_k = env_t[sl]
                    cnt = counts[sl] + 1
                    pool.sample(child_seeds_device(env_k, "resample", cnt), child_seeds_device(env_k, "crowd", cnt),
                                stream=side, check=False)
                    done = torch.cuda.Event()
                    done.record(side)
                pending = (ahead, done)
                samples += 1
        last = bool((stop >= ticks).all())
        field.run_window(ticks, cur.astype(np.int32), stop.astype(np.int32), first, last, robot_pos, robot_vel,
                         robot_radius, check=False)
        windows += 1
        rounds += int(_lib.lib().cw_crowd_run_rounds())
        servers += int(_lib.lib().cw_crowd_run_servers())
        first = False
        cur = stop
        if last and pending is None:
            break
    field.run_server_warps = saved
    field.prepare_step()
    field.check_flags()
    field.last_run_stats = {"windows": windows, "rounds": rounds, "servers": servers, "sample_calls": samples}
    return resampled
