"""Crowd dynamics on the B200 -- drop-in for the reference's crowd package.

Mirrors /root/reference/pkg/src/citywalk/crowd:
  * ``AgentKind``, ``CrowdAgent``, ``CrowdConfig`` and the kind tables (types.py:9-79)
  * ``CrowdField(occupancies, config, env_seeds, resample_goals=True)`` with
    ``set_agents`` / ``set_env_agents`` / ``replace_env`` / ``step`` / ``agents_of``
    / ``last_gap_by_env`` (field.py:26-430)
  * ``step_crowd`` (step.py:17-34), ``spawn_agents`` (step.py:37-63, with
    ``region_mask``), ``write_trace`` (step.py:66-70)
  * ``sample_routes`` / ``connected_components`` (routes.py:14-87)
  * ``HalfPlane``, ``orca_halfplane``, ``compute_orca_constraints``,
    ``solve_velocity``, ``feasible`` (orca.py:23-246, types.py:83-97) and the
    private pieces the reference tests call: ``_batched_lp`` (field.py:500) and
    ``CrowdField._refresh_guidance`` / ``_preferred_velocities`` /
    ``_build_constraints`` (field.py:165-350)

State lives on the device (float64 SoA, (E, A, 2) / (E, A)); ``step`` is one
``cw_crowd_step`` launch (guidance + A*, neighbours, ORCA, LP, commit, goal
resample for every env).  ``pos`` / ``vel`` / ``goal`` / ... are DeviceView
windows onto the device tensors ``pos_t`` etc.: reads copy to the host, item
assignment writes through (the reference's callers write these arrays).
Every computation here runs in the CUDA library; the host code only moves
arguments and results.
"""

import os
from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from . import _lib
from .errors import STATUS_ERRORS
from .urbangen import OccupancyGrid, SceneBatch, load_catalog


class AgentKind(IntEnum):
    PEDESTRIAN = 0
    CYCLIST = 1
    SCOOTER = 2


MAX_SPEED_OF_KIND = {AgentKind.PEDESTRIAN: 2.0, AgentKind.CYCLIST: 5.0, AgentKind.SCOOTER: 4.0}
PREF_SPEED_RANGE = {AgentKind.PEDESTRIAN: (0.8, 1.4), AgentKind.CYCLIST: (2.0, 4.0),
                    AgentKind.SCOOTER: (1.5, 3.0)}
RADIUS_OF_KIND = {AgentKind.PEDESTRIAN: 0.3, AgentKind.CYCLIST: 0.45, AgentKind.SCOOTER: 0.4}


@dataclass
class CrowdAgent:
    id: int
    position: np.ndarray
    velocity: np.ndarray
    radius: float
    preferred_speed: float
    goal: np.ndarray
    kind: AgentKind = AgentKind.PEDESTRIAN

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=np.float64)
        self.velocity = np.asarray(self.velocity, dtype=np.float64)
        self.goal = np.asarray(self.goal, dtype=np.float64)
        if self.radius <= 0:
            raise ValueError("radius must be > 0")
        if self.preferred_speed <= 0:
            raise ValueError("preferred_speed must be > 0")

    @property
    def max_speed(self):
        return MAX_SPEED_OF_KIND[self.kind]


@dataclass
class CrowdConfig:
    time_horizon: float = 2.0
    obstacle_time_horizon: float = 1.0
    neighbor_distance: float = 5.0
    max_neighbors: int = 10
    dt: float = 0.05
    safety_margin: float = 0.03

    def __post_init__(self):
        for name in ("time_horizon", "obstacle_time_horizon", "neighbor_distance",
                     "max_neighbors", "dt"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be > 0")
        if self.dt > 0.1:
            raise ValueError("dt must be <= 0.1 s")
        if self.safety_margin < 0:
            raise ValueError("safety_margin must be >= 0")


def _u64(seeds, device):
    import torch
    arr = np.array([int(s) & ((1 << 64) - 1) for s in seeds], dtype=np.uint64).view(np.int64)
    return torch.from_numpy(arr).to(device)


class CrowdField:
    """Device CrowdField (field.py:26).  ``occupancies`` is a list of
    OccupancyGrid (host labels, uploaded once) or a device ``SceneBatch``."""

    def __init__(self, occupancies, config, env_seeds, resample_goals=True, device="cuda",
                 threads=None, path_cap=None, heap_cap=None, astar_warps=None, prefetch=None):
        import torch
        self.config = config
        # next-tick search prefetch in step() (cw_spec_create): results are identical with
        # or without it; CW_PREFETCH=0 turns it off for A/B runs
        self.prefetch = (os.environ.get("CW_PREFETCH", "1") != "0") if prefetch is None else bool(prefetch)
        self._spec_h = None
        self._spec_key = None
        self.resample_goals = resample_goals
        self.device = torch.device(device)
        self.threads = threads    # step CTA size per env; None: by crowd size (_step_nt)
        self.run_threads = None   # cw_crowd_run CTA size; None: one lane per agent
        self.run_history_bytes = 256 << 20   # per-call cap of the run's (env, tick) gap history
        self.run_server_warps = None   # search warps per server CTA in cw_crowd_run (None: by round footprint, crowd.cu launch_run)
        self.astar_warps = astar_warps
        if isinstance(occupancies, SceneBatch):
            b = occupancies
            self.E = b.E
            self.ny, self.nx = b.labels.shape[1:]
            self.res = float(b.params.res)
            self.res0 = self.res
            self.labels_t, self.nearest_t, self.has_obs_t = b.labels, b.nearest, b.has_obs
            self.walk_t, self.walk_n_t = b.walk, b.walk_n
            self.reach_t, self.moves_t = b.reach, b.moves
            self.epoch_t = b.epoch   # grid generation, bumped by every sampling call
            self._batch = b
        else:
            occs = list(occupancies)
            self.E = len(occs)
            shapes = {o.labels.shape for o in occs}
            ress = {float(o.resolution) for o in occs}
            if len(shapes) != 1 or len(ress) != 1:
                raise ValueError("the B200 CrowdField needs one grid shape and resolution per batch")
            self.ny, self.nx = occs[0].labels.shape
            self.res = float(occs[0].resolution)
            self.res0 = self.res
            self._batch = None
            self.epoch_t = torch.zeros((self.E,), dtype=torch.int32, device=self.device)
            self._upload_grids(occs)
        check_grid_shape(self.nx, self.ny)
        if len(env_seeds) != self.E:
            raise ValueError("env_seeds must have one seed per env")
        self.rng_t = torch.empty((self.E, 48), dtype=torch.uint8, device=self.device)
        seeds = _u64(env_seeds, self.device)
        _lib.check(_lib.lib().cw_seed_streams(self.E, _lib.ptr(seeds), _lib.ptr(self.rng_t),
                                              _lib.stream_ptr()), "cw_seed_streams")
        N = self.nx * self.ny
        self.path_cap = int(path_cap or 2 * (self.nx + self.ny) + 64)
        self.heap_cap = int(heap_cap or min(max(65536, N), (1 << 19) - 1))
        # persistent A* CTAs: one per SM, cw_astar_warps() search warps sharing its tile pool
        self.astar_ctas = int(torch.cuda.get_device_properties(self.device).multi_processor_count) \
            if self.device.type == "cuda" else 1
        self.last_gap_t = torch.full((self.E,), float("inf"), dtype=torch.float64, device=self.device)
        self.gap_tmp_t = torch.zeros((self.E,), dtype=torch.float64, device=self.device)
        self.flags_t = torch.zeros((8,), dtype=torch.int32, device=self.device)
        self.counters_t = torch.zeros((16,), dtype=torch.int64, device=self.device)
        self.env_req_t = torch.zeros((self.E,), dtype=torch.uint8, device=self.device)
        self._astar_ready = False
        self._alloc(0)

    # -- grids ----------------------------------------------------------------
    def _invalidate(self):
        """Drop the cached launch arguments: they hold raw device pointers of the
        state tensors, which _alloc / grid uploads replace."""
        self.__dict__.pop("_p", None)
        self.__dict__.pop("_s", None)

    def _upload_grids(self, occs):
        import torch
        self._invalidate()
        E, ny, nx = self.E, self.ny, self.nx
        lab = torch.from_numpy(np.stack([o.labels for o in occs]).astype(np.uint8)).to(self.device)
        self.labels_t = lab.contiguous()
        self.nearest_t = torch.empty((E, ny, nx), dtype=torch.int32, device=self.device)
        self.has_obs_t = torch.zeros((E,), dtype=torch.uint8, device=self.device)
        self.walk_t = torch.empty((E, ny * nx), dtype=torch.int32, device=self.device)
        self.walk_n_t = torch.zeros((E,), dtype=torch.int32, device=self.device)
        self.reach_t = torch.empty((E, ny * nx), dtype=torch.int32, device=self.device)
        self.moves_t = torch.zeros((E, ny * nx), dtype=torch.uint8, device=self.device)
        self._prepare(None)
        self.epoch_t += 1

    def _prepare(self, rows):
        """field.py:60-67 (_prepare_env) for all envs or the given rows."""
        import torch
        p = _lib.SceneParams()
        p.nx, p.ny = self.nx, self.ny
        n = self.E if rows is None else len(rows)
        status = torch.zeros((self.E,), dtype=torch.int32, device=self.device)
        scratch = torch.empty((n, 10 * self.nx * self.ny), dtype=torch.int32, device=self.device)
        b = _lib.SceneBuffers()
        b.labels = self.labels_t.data_ptr()
        b.nearest = self.nearest_t.data_ptr()
        b.has_obs = self.has_obs_t.data_ptr()
        b.walk = self.walk_t.data_ptr()
        b.walk_n = self.walk_n_t.data_ptr()
        b.reach = self.reach_t.data_ptr()
        b.moves = self.moves_t.data_ptr()
        b.status = status.data_ptr()
        b.scratch_i32 = scratch.data_ptr()
        sl = None if rows is None else torch.as_tensor(rows, dtype=torch.int32, device=self.device)
        _lib.check(_lib.lib().cw_prepare_envs(p, n, _lib.ptr(sl), b, _lib.stream_ptr()),
                   "cw_prepare_envs")

    # -- population (field.py:71-86, 383-401) ------------------------------------
    def _alloc(self, A):
        import torch
        E, d = self.E, self.device
        self._invalidate()
        self.A = A
        f64 = dict(dtype=torch.float64, device=d)
        self.pos_t = torch.zeros((E, A, 2), **f64)
        self.vel_t = torch.zeros((E, A, 2), **f64)
        self.goal_t = torch.zeros((E, A, 2), **f64)
        self.waypoint_t = torch.zeros((E, A, 2), **f64)
        self.radius_t = torch.full((E, A), 0.3, **f64)
        self.pref_t = torch.full((E, A), 1.0, **f64)
        self.max_speed_t = torch.full((E, A), 2.0, **f64)
        self.kind_t = torch.zeros((E, A), dtype=torch.int8, device=d)
        self.active_t = torch.zeros((E, A), dtype=torch.uint8, device=d)
        self.path_cells_t = torch.zeros((E, A, self.path_cap), dtype=torch.int32, device=d)
        self.path_head_t = torch.zeros((E, A), dtype=torch.int32, device=d)
        self.path_n_t = torch.zeros((E, A), dtype=torch.int32, device=d)
        self.astar_req_t = torch.empty((max(1, E * A), 4), dtype=torch.int32, device=d)

    def _ensure_astar(self):
        import torch
        if self._astar_ready:
            return
        self._invalidate()
        S = self.astar_ctas * int(_lib.lib().cw_astar_warps())   # search warps
        N = self.nx * self.ny
        d = self.device
        slot = int(_lib.lib().cw_astar_slot_bytes(self.nx, self.ny))
        self.astar_rec_t = torch.empty((S * slot // 8,), dtype=torch.int64, device=d)
        self.astar_heap_t = torch.empty((S, self.heap_cap, 2), dtype=torch.int64, device=d)  # far pool
        self._astar_ready = True

    def set_agents(self, agent_lists):
        A = max((len(l) for l in agent_lists), default=0)
        self._alloc(A)
        self._fill([(e, l) for e, l in enumerate(agent_lists)])

    def set_env_agents(self, e, agents):
        if len(agents) > self.A:
            lists = [self.agents_of(k) for k in range(self.E)]
            lists[e] = agents
            self.set_agents(lists)
            return
        self.active_t[e] = 0
        self.path_n_t[e] = 0
        self._fill([(e, agents)])

    def _fill(self, rows):
        import torch
        for e, lst in rows:
            n = len(lst)
            if n == 0:
                continue
            pos = np.array([a.position for a in lst], dtype=np.float64)
            vel = np.array([a.velocity for a in lst], dtype=np.float64)
            goal = np.array([a.goal for a in lst], dtype=np.float64)
            t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(self.device)
            self.pos_t[e, :n] = t(pos)
            self.vel_t[e, :n] = t(vel)
            self.goal_t[e, :n] = t(goal)
            self.waypoint_t[e, :n] = t(goal)
            self.radius_t[e, :n] = t(np.array([a.radius for a in lst], dtype=np.float64))
            self.pref_t[e, :n] = t(np.array([a.preferred_speed for a in lst], dtype=np.float64))
            self.max_speed_t[e, :n] = t(np.array([a.max_speed for a in lst], dtype=np.float64))
            self.kind_t[e, :n] = t(np.array([int(a.kind) for a in lst], dtype=np.int8))
            self.active_t[e, :n] = 1
            self.path_n_t[e, :n] = 0

    def set_from_spawn(self, batch, rows=None):
        """Install the device spawn of a SceneBatch (step.py:37-63 outputs) for all
        rows (re-allocates) or for the given rows (resample path)."""
        import torch
        A = batch.params.peds
        if rows is None:
            self._alloc(A)
            idx = slice(None)
        else:
            idx = torch.as_tensor(rows, dtype=torch.long, device=self.device)
        k = batch.sp_kind[idx].long()
        rad = torch.tensor([0.3, 0.45, 0.4], dtype=torch.float64, device=self.device)
        ms = torch.tensor([2.0, 5.0, 4.0], dtype=torch.float64, device=self.device)
        self.pos_t[idx] = batch.sp_pos[idx]
        self.vel_t[idx] = 0.0
        self.goal_t[idx] = batch.sp_goal[idx]
        self.waypoint_t[idx] = batch.sp_goal[idx]
        self.radius_t[idx] = rad[k]
        self.pref_t[idx] = batch.sp_pref[idx]
        self.max_speed_t[idx] = ms[k]
        self.kind_t[idx] = batch.sp_kind[idx]
        self.active_t[idx] = 1
        self.path_n_t[idx] = 0
        self.epoch_t[idx] += 1   # the rows' grids were (re)sampled

    def replace_env(self, e, occupancy):
        """field.py:403-413 for a host OccupancyGrid."""
        import torch
        if occupancy.labels.shape != (self.ny, self.nx):
            raise ValueError("replacement grid must keep the batch shape")
        self.labels_t[e] = torch.from_numpy(np.ascontiguousarray(occupancy.labels)).to(self.device)
        self._prepare([e])
        self.epoch_t[e] += 1
        self._invalidate()

    # -- stepping (field.py:90-163) -----------------------------------------------
    def _params(self):
        c = self.config
        p = _lib.CrowdParams()
        p.E, p.A, p.nx, p.ny = self.E, self.A, self.nx, self.ny
        p.res, p.res0 = self.res, self.res0
        p.time_horizon = c.time_horizon
        p.obstacle_time_horizon = c.obstacle_time_horizon
        p.neighbor_distance = c.neighbor_distance
        p.nd2 = c.neighbor_distance ** 2
        p.nd2_f32 = float(np.float32(c.neighbor_distance ** 2))
        p.max_neighbors = int(c.max_neighbors)
        p.dt = c.dt
        p.safety_margin = c.safety_margin
        p.goal_reach2 = 0.3 ** 2
        p.stall_c, p.stall_s = float(np.cos(0.6)), float(np.sin(0.6))
        p.resample_goals = int(bool(self.resample_goals))
        # the static lane is gated per env by has_obs (field.py:319-324: envs without
        # obstacles get an invalid lane, which the LP skips), so no global gate
        p.use_static = 1
        p.path_cap, p.heap_cap, p.astar_ctas = self.path_cap, self.heap_cap, self.astar_ctas
        # few replans per tick (small batches): one search warp per SM, whose tick
        # latency is the longest search; large batches: four per SM for throughput
        p.astar_warps = self.astar_warps or (1 if self.E * self.A < 131072 else 4)
        p.run_server_warps = int(self.run_server_warps or 0)
        return p

    def _state(self):
        self._ensure_astar()
        s = _lib.CrowdState()
        m = dict(pos=self.pos_t, vel=self.vel_t, goal=self.goal_t, waypoint=self.waypoint_t,
                 radius=self.radius_t, pref_speed=self.pref_t, max_speed=self.max_speed_t,
                 active=self.active_t, path_cells=self.path_cells_t, path_head=self.path_head_t,
                 path_n=self.path_n_t, labels=self.labels_t, nearest=self.nearest_t,
                 has_obs=self.has_obs_t, walk=self.walk_t, walk_n=self.walk_n_t, reach=self.reach_t,
                 moves=self.moves_t, rng=self.rng_t,
                 last_gap=self.last_gap_t, gap_tmp=self.gap_tmp_t, flags=self.flags_t,
                 astar_rec=self.astar_rec_t, astar_req=self.astar_req_t,
                 astar_heap=self.astar_heap_t, counters=self.counters_t, env_req=self.env_req_t,
                 env_epoch=self.epoch_t)
        for k, v in m.items():
            setattr(s, k, v.data_ptr())
        s.spec = self._spec_handle()
        return s

    def _spec_handle(self):
        """The next-tick prefetch context for the current shapes (None when off)."""
        import ctypes
        if not self.prefetch or self.device.type != "cuda" or self.A == 0:
            return None
        p = self._params()
        key = (p.E, p.A, p.nx, p.ny, p.path_cap, p.heap_cap)
        if key != self._spec_key:
            self._spec_free()
            h = ctypes.c_void_p()
            _lib.check(_lib.lib().cw_spec_create(p, ctypes.byref(h)), "cw_spec_create")
            self._spec_h, self._spec_key = h.value, key
        return self._spec_h

    def _spec_free(self):
        if self._spec_h:
            _lib.lib().cw_spec_destroy(self._spec_h)
        self._spec_h, self._spec_key = None, None

    def __del__(self):
        try:
            self._spec_free()
        except Exception:
            pass

    def prepare_step(self):
        """Build the launch arguments (rebuilt automatically after set_agents /
        set_from_spawn / replace_env, which replace or re-prepare device buffers)."""
        self._s = self._state()
        self._p = self._params()

    def step(self, robot_pos=None, robot_vel=None, robot_radius=0.35, env_mask=None, workers=1,
             stream=None, check=True):
        """Advance every (masked) env one tick.  Array inputs may be numpy (host,
        copied in) or device tensors.  ``workers`` is accepted for API parity."""
        import torch
        if self.A == 0 or self.E == 0:
            return
        if "_p" not in self.__dict__:
            self.prepare_step()
        rp = self._dev(robot_pos, torch.float64, (self.E, 2))
        rv = self._dev(robot_vel, torch.float64, (self.E, 2)) if robot_pos is not None else None
        em = self._dev(env_mask, torch.uint8, (self.E,))
        err = _lib.lib().cw_crowd_step(self._p, self._s, _lib.ptr(rp), _lib.ptr(rv),
                                       float(robot_radius), _lib.ptr(em), self._step_nt(),
                                       _lib.stream_ptr(stream))
        _lib.check(err, "cw_crowd_step")
        if check:
            self.check_flags()

    def run(self, ticks, robot_pos=None, robot_vel=None, robot_radius=0.35, env_mask=None,
            stream=None, check=True, threads=None):
        """``ticks`` calls of ``step`` with the same inputs, without a per-tick
        barrier across envs (``cw_crowd_run``): each env advances on its own and
        the final state is bit-identical.  Blocks until the run is done."""
        import torch
        ticks = int(ticks)
        if self.A == 0 or self.E == 0 or ticks <= 0:
            return
        if key_col_bits(self.nx, self.ny) != 10:
            # the run's search server keeps the default A* key packing (astar.cuh): grids
            # wider or taller than 1024 cells step tick by tick (the same result)
            for _ in range(ticks):
                self.step(robot_pos=robot_pos, robot_vel=robot_vel, robot_radius=robot_radius,
                          env_mask=env_mask, check=check)
            return
        if "_p" not in self.__dict__:
            self.prepare_step()
        rp = self._dev(robot_pos, torch.float64, (self.E, 2))
        rv = self._dev(robot_vel, torch.float64, (self.E, 2)) if robot_pos is not None else None
        em = self._dev(env_mask, torch.uint8, (self.E,))
        # the per-(env, tick) gap history bounds one call's length: long runs go in
        # chunks (a chunk boundary is a barrier across envs; results are unchanged)
        chunk = max(1, min(ticks, self.run_history_bytes // (8 * self.E)))
        nbytes = int(_lib.lib().cw_crowd_run_scratch_bytes(self.E, self.A, chunk))
        if getattr(self, "_run_scratch", None) is None or self._run_scratch.numel() < nbytes:
            self._run_scratch = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        nt = int(threads or self.run_threads or self._run_nt())
        for t0 in range(0, ticks, chunk):
            err = _lib.lib().cw_crowd_run(self._p, self._s, _lib.ptr(rp), _lib.ptr(rv), float(robot_radius),
                                          _lib.ptr(em), nt, min(chunk, ticks - t0), _lib.ptr(self._run_scratch),
                                          _lib.stream_ptr(stream))
            _lib.check(err, "cw_crowd_run")
        if check:
            self.check_flags()

    def run_window(self, ticks, start, stop, first, last, robot_pos=None, robot_vel=None, robot_radius=0.35,
                   env_mask=None, stream=None, check=True, threads=None):
        """One segment of a ``ticks``-long window (``cw_crowd_run_window``): env e runs
        its ticks ``start[e]`` .. ``stop[e] - 1`` without a barrier across envs.
        ``first`` resets the window's per-(env, tick) gap history, ``last`` publishes
        ``last_gap_by_env`` from it.  Between segments the caller may replace env
        state (re-sampled scenes, respawned crowds); per env the result equals the
        same ticks stepped synchronously."""
        import torch
        ticks = int(ticks)
        if self.A == 0 or self.E == 0 or ticks <= 0:
            return
        if key_col_bits(self.nx, self.ny) != 10:
            raise NotImplementedError("run_window on grids wider or taller than 1024 cells "
                                      "(the run's search server keeps the default A* key packing)")
        if "_p" not in self.__dict__:
            self.prepare_step()
        rp = self._dev(robot_pos, torch.float64, (self.E, 2))
        rv = self._dev(robot_vel, torch.float64, (self.E, 2)) if robot_pos is not None else None
        em = self._dev(env_mask, torch.uint8, (self.E,))
        st = torch.as_tensor(start, dtype=torch.int32).to(self.device).contiguous()
        sp = torch.as_tensor(stop, dtype=torch.int32).to(self.device).contiguous()
        nbytes = int(_lib.lib().cw_crowd_run_scratch_bytes(self.E, self.A, ticks))
        if getattr(self, "_win_scratch", None) is None or self._win_scratch.numel() < nbytes:
            if not first:
                raise ValueError("run_window: the window's scratch is gone; start it with first=True")
            self._win_scratch = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        flags = (1 if first else 0) | (2 if last else 0)
        err = _lib.lib().cw_crowd_run_window(self._p, self._s, _lib.ptr(rp), _lib.ptr(rv), float(robot_radius),
                                             _lib.ptr(em), int(threads or self.run_threads or self._run_nt()),
                                             ticks, _lib.ptr(st), _lib.ptr(sp), flags,
                                             _lib.ptr(self._win_scratch), _lib.stream_ptr(stream))
        _lib.check(err, "cw_crowd_run_window")
        if check:
            self.check_flags()

    def _step_nt(self):
        """Step CTA size per env: 64 threads for lane-path crowds (A < 128: one lane per
        agent in the ORCA passes; measured 1-6 % faster ticks than 128 at cfg2 / cfg3 / cfg5),
        256 for the warp-per-agent shape with cell binning (cfg4: an env's commit is the
        tick's tail after its last search -- 8 warps instead of 4 per env, tick 36.0 -> 32.2
        ms; 512 threads: 35.7)."""
        return int(self.threads or (64 if self.A < 128 else 256))

    def _run_nt(self):
        """Round CTA size: one lane per agent (lane ORCA / guide; cell binning from 128
        agents on)."""
        if self.A >= 128:
            # lane path with cell binning (max_neighbors <= 10): 128 threads, so a round CTA
            # (~220 registers per thread) shares an SM with a search-server CTA -- cfg4 run
            # 24.5 -> 23.8 ms/tick (256 threads: 66 ms, one CTA per SM and none beside the
            # server); the warp-per-agent path (more neighbours): 256
            return 128 if self.config.max_neighbors <= 10 else 256
        return 32 if self.A <= 32 else 64 if self.A <= 64 else 128

    def step_phase(self, phase, robot_pos=None, robot_vel=None, robot_radius=0.35, env_mask=None,
                   stream=None):
        """Launch one phase of the tick (1 guide, 2 A*, 4 ORCA+commit); device inputs only."""
        if "_p" not in self.__dict__:
            self.prepare_step()
        err = _lib.lib().cw_crowd_step_phases(self._p, self._s, _lib.ptr(robot_pos), _lib.ptr(robot_vel),
                                              float(robot_radius), _lib.ptr(env_mask), self._step_nt(),
                                              int(phase), _lib.stream_ptr(stream))
        _lib.check(err, "cw_crowd_step_phases")

    def check_flags(self):
        code = int(self.flags_t[1].item())
        if code:
            raise STATUS_ERRORS.get(code, RuntimeError)(
                f"crowd guidance capacity exceeded (code {code}); path_cap={self.path_cap} "
                f"heap_cap={self.heap_cap}")

    def _dev(self, x, dtype, shape):
        import torch
        if x is None:
            return None
        if isinstance(x, torch.Tensor):
            return x.to(device=self.device, dtype=dtype).reshape(shape).contiguous()
        return torch.from_numpy(np.ascontiguousarray(np.asarray(x).astype(
            np.uint8 if dtype == torch.uint8 else np.float64)).reshape(shape)).to(self.device)

    # -- host views (field.py:47-58 ownership) -----------------------------------------
    # The reference exposes its state as numpy arrays that callers read and write
    # (batch.py:240-243, tests/test_acceptance.py:234-249).  Here each attribute is a
    # DeviceView over the device tensor: reads copy to the host, item assignment
    # writes through to the device.
    pos = property(lambda self: DeviceView(self.pos_t), lambda self, v: self._assign("pos_t", v))
    vel = property(lambda self: DeviceView(self.vel_t), lambda self, v: self._assign("vel_t", v))
    goal = property(lambda self: DeviceView(self.goal_t), lambda self, v: self._assign("goal_t", v))
    waypoint = property(lambda self: DeviceView(self.waypoint_t),
                        lambda self, v: self._assign("waypoint_t", v))
    radius = property(lambda self: DeviceView(self.radius_t), lambda self, v: self._assign("radius_t", v))
    pref_speed = property(lambda self: DeviceView(self.pref_t), lambda self, v: self._assign("pref_t", v))
    max_speed = property(lambda self: DeviceView(self.max_speed_t),
                         lambda self, v: self._assign("max_speed_t", v))
    kind = property(lambda self: DeviceView(self.kind_t), lambda self, v: self._assign("kind_t", v))
    active = property(lambda self: DeviceView(self.active_t, bool),
                      lambda self, v: self._assign("active_t", v))

    def _assign(self, name, value):
        """``field.pos = array`` replaces the contents (same shape) on the device."""
        import torch
        t = getattr(self, name)
        src = value.t if isinstance(value, DeviceView) else torch.as_tensor(np.asarray(value))
        if tuple(src.shape) != tuple(t.shape):
            raise ValueError(f"{name[:-2]}: expected shape {tuple(t.shape)}, got {tuple(src.shape)}")
        t.copy_(src.to(device=t.device, dtype=t.dtype))

    @property
    def last_gap_by_env(self):
        return self.last_gap_t.cpu().numpy()

    @property
    def _walk_cells(self):
        """field.py:60-67: per env the walkable cell centres (row-major), the goal
        re-sampling pool."""
        wn = self.walk_n_t.cpu().numpy()
        out = []
        for e in range(self.E):
            flat = self.walk_t[e, :int(wn[e])].cpu().numpy().astype(np.int64)
            r, c = np.divmod(flat, self.nx)
            out.append(np.stack([(c + 0.5) * self.res, (r + 0.5) * self.res], axis=1))
        return out

    @_walk_cells.setter
    def _walk_cells(self, cells):
        """Replace the goal re-sampling pools (tests/test_acceptance.py:234-238 narrows
        them to an interior).  Entries must be cell centres of this grid."""
        import torch
        if len(cells) != self.E:
            raise ValueError("one walk-cell list per env")
        n_max = self.walk_t.shape[1]
        for e, wc in enumerate(cells):
            wc = np.asarray(wc, dtype=np.float64).reshape(-1, 2)
            col = np.floor(wc[:, 0] / self.res).astype(np.int64)
            row = np.floor(wc[:, 1] / self.res).astype(np.int64)
            if wc.shape[0] > n_max or not (np.array_equal((col + 0.5) * self.res, wc[:, 0])
                                           and np.array_equal((row + 0.5) * self.res, wc[:, 1])):
                raise ValueError("walk cells must be cell centres of the env's grid")
            if ((col < 0) | (col >= self.nx) | (row < 0) | (row >= self.ny)).any():
                raise ValueError("walk cells must lie inside the grid")
            flat = torch.from_numpy((row * self.nx + col).astype(np.int32)).to(self.device)
            self.walk_t[e, :flat.numel()] = flat
            self.walk_n_t[e] = int(flat.numel())

    # -- the reference's private stage hooks (tests/test_crowd.py:213-217) ------------
    def _act_tensor(self, e0, e1, act):
        import torch
        a = np.asarray(act, dtype=bool).reshape(e1 - e0, self.A)
        return torch.from_numpy(a.astype(np.uint8)).to(self.device)

    def _refresh_guidance(self, e0, e1, act):
        """field.py:165-212 for envs [e0, e1) and agents ``act``: k_guide + k_astar
        (waypoint pop, stray check, line of sight, A* replans), no ORCA."""
        import torch
        if self.A == 0 or e1 <= e0:
            return
        saved = self.active_t.clone()
        self.active_t[e0:e1] = self._act_tensor(e0, e1, act) & saved[e0:e1]
        mask = torch.zeros(self.E, dtype=torch.uint8, device=self.device)
        mask[e0:e1] = 1
        try:
            self.step_phase(1, env_mask=mask)
            self.step_phase(2, env_mask=mask)
        finally:
            self.active_t.copy_(saved)
            self.flags_t[4:6] = 0      # the A* queue is normally reset by k_orca's last CTA
        self.check_flags()

    def _constraints(self, e0, e1, act, robot_pos=None, robot_vel=None, robot_radius=0.35):
        import torch
        rows = (e1 - e0) * self.A
        kmax = min(int(self.config.max_neighbors), max(self.A - 1, 0))
        use_robot = robot_pos is not None
        use_static = bool(self.has_obs_t.any().item())
        lmax = kmax + int(use_robot) + int(use_static)
        f64 = dict(dtype=torch.float64, device=self.device)
        out = dict(pref=torch.empty((rows, 2), **f64),
                   points=torch.empty((rows, max(lmax, 1), 2), **f64),
                   normals=torch.empty((rows, max(lmax, 1), 2), **f64),
                   valid=torch.empty((rows, max(lmax, 1)), dtype=torch.uint8, device=self.device),
                   inr=torch.empty((rows,), dtype=torch.int32, device=self.device),
                   gap=torch.empty((rows,), **f64))
        if "_p" not in self.__dict__:
            self.prepare_step()
        rp = self._dev(robot_pos, torch.float64, (self.E, 2))
        rv = self._dev(robot_vel, torch.float64, (self.E, 2)) if use_robot else None
        at = self._act_tensor(e0, e1, act)
        _lib.check(_lib.lib().cw_crowd_constraints(
            self._p, self._s, int(e0), int(e1), _lib.ptr(at), _lib.ptr(rp), _lib.ptr(rv), float(robot_radius),
            int(use_static), int(max(lmax, 1)), _lib.ptr(out["pref"]), _lib.ptr(out["points"]),
            _lib.ptr(out["normals"]), _lib.ptr(out["valid"]), _lib.ptr(out["inr"]), _lib.ptr(out["gap"]),
            _lib.stream_ptr()), "cw_crowd_constraints")
        h = {k: v.cpu().numpy() for k, v in out.items()}
        return h, kmax, use_robot, use_static

    def _preferred_velocities(self, e0, e1, act):
        """field.py:214-227: (N, 2) preferred velocities, 0 for inactive rows."""
        if self.A == 0 or e1 <= e0:
            return np.zeros((0, 2))
        return self._constraints(e0, e1, act)[0]["pref"]

    def _build_constraints(self, e0, e1, act, robot_pos, robot_vel, robot_radius):
        """field.py:229-350: (points, normals, valid) with L = K + robot + static
        lanes in the reference layout (K trimmed to the largest in-range count)."""
        h, kmax, use_robot, use_static = self._constraints(e0, e1, act, robot_pos, robot_vel, robot_radius)
        N = (e1 - e0) * self.A
        K = min(kmax, int(h["inr"].max(initial=0))) if kmax > 0 else 0
        L = K + int(use_robot) + int(use_static)
        sel = list(range(K)) + list(range(kmax, kmax + int(use_robot) + int(use_static)))
        points = np.zeros((N, max(L, 1), 2))
        normals = np.zeros((N, max(L, 1), 2))
        normals[..., 0] = 1.0
        valid = np.zeros((N, max(L, 1)), dtype=bool)
        if sel:
            points[:, :L] = h["points"][:, sel]
            normals[:, :L] = h["normals"][:, sel]
            valid[:, :L] = h["valid"][:, sel].astype(bool)
        if K > 0:   # field.py:268-271
            import torch
            gap = h["gap"].reshape(e1 - e0, self.A).min(axis=1)
            self.last_gap_t[e0:e1] = torch.from_numpy(gap).to(self.device)
        return points, normals, valid

    def trace_records(self, tick):
        """field.py:432-443: one {tick, env, id, x, y, vx, vy} record per active agent."""
        act = self.active_t.cpu().numpy()
        pos, vel = self.pos_t.cpu().numpy(), self.vel_t.cpu().numpy()
        return [{"tick": int(tick), "env": int(e), "id": int(a),
                 "x": float(pos[e, a, 0]), "y": float(pos[e, a, 1]),
                 "vx": float(vel[e, a, 0]), "vy": float(vel[e, a, 1])}
                for e in range(self.E) for a in range(self.A) if act[e, a]]

    def agents_of(self, e):
        """field.py:417-430."""
        act = self.active_t[e].cpu().numpy()
        pos, vel, goal = self.pos_t[e].cpu().numpy(), self.vel_t[e].cpu().numpy(), self.goal_t[e].cpu().numpy()
        rad, pref = self.radius_t[e].cpu().numpy(), self.pref_t[e].cpu().numpy()
        kind = self.kind_t[e].cpu().numpy()
        return [CrowdAgent(id=a, position=pos[a].copy(), velocity=vel[a].copy(), radius=float(rad[a]),
                           preferred_speed=float(pref[a]), goal=goal[a].copy(),
                           kind=AgentKind(int(kind[a])))
                for a in range(self.A) if act[a]]

    def stats(self):
        c = self.counters_t.cpu().numpy()
        return {"astar_expansions": int(c[0]), "path_points_scanned": int(c[1]),
                "lp_fallbacks": int(c[2]), "stall_retries": int(c[3]),
                "astar_cycles": int(c[4]), "astar_max_cycles": int(c[5]),
                "cta_cycles": int(c[6]), "cta_max_cycles": int(c[7]),
                "astar_global_retries": int(c[10]), "path_points_read": int(c[12]),
                "los_samples_read": int(c[13]), **self.prefetch_stats()}

    def prefetch_stats(self):
        """Next-tick prefetch: batches launched, cached results used, waits on a
        prediction still running, queued predictions searched in place."""
        import ctypes
        if not self._spec_h:
            return {}
        v = (ctypes.c_longlong * 4)()
        _lib.check(_lib.lib().cw_spec_stats(self._spec_h, v), "cw_spec_stats")
        return {"prefetch_batches": v[0], "prefetch_hits": v[1], "prefetch_waits": v[2],
                "prefetch_claims": v[3]}


def step_crowd(agents, robot_state, occupancy, config, seed=0, resample_goals=True):
    """step.py:17-34 (one env, one tick)."""
    if not agents:
        return []
    f = CrowdField([occupancy], config, [seed], resample_goals=resample_goals)
    f.set_agents([agents])
    if robot_state is None:
        f.step()
    else:
        rp, rv, rr = robot_state
        f.step(robot_pos=np.asarray(rp, np.float64).reshape(1, 2),
               robot_vel=np.asarray(rv, np.float64).reshape(1, 2), robot_radius=rr)
    return f.agents_of(0)


def _grid_batch(occupancy, count, region_mask):
    """1-row SceneBatch holding a host grid (and an optional region mask)."""
    import torch
    from .urbangen import SceneBatch
    ny, nx = occupancy.labels.shape
    p = _lib.SceneParams()
    p.nx, p.ny, p.res = nx, ny, float(occupancy.resolution)
    p.peds = int(count)
    p.obj_max = 1
    b = SceneBatch(p, 1)
    b.labels[0] = torch.from_numpy(np.ascontiguousarray(occupancy.labels)).to(b.device)
    if region_mask is not None:
        m = np.asarray(region_mask, dtype=bool)
        if m.shape != (ny, nx):
            raise ValueError("region_mask must have the grid's shape")
        b.region = torch.from_numpy(m.astype(np.uint8)).to(b.device).reshape(1, ny * nx)
    return p, b


def key_col_bits(nx, ny):
    """Column bits of the A* key's cell field (astar.cuh key_col_bits): 10 up to
    1024 x 1024 cells, else ceil(log2 nx)."""
    b = max(int(nx) - 1, 0).bit_length()
    return 10 if b <= 10 and ny <= 1024 else b


def check_grid_shape(nx, ny):
    """Grids the device crowd accepts: the A* key (astar.cuh make_key2) packs
    row << cb | col in 20 bits and floor(h * 4096) in 23 bits."""
    if (key_col_bits(nx, ny) + max(int(ny) - 1, 0).bit_length() > 20
            or max(nx, ny) + 0.4143 * min(nx, ny) >= 2047.0):
        raise NotImplementedError("grids whose row and column need more than 20 bits together, "
                                  "or whose octile diameter reaches 2047 cells")


def spawn_agents(occupancy, count, seed, region_mask=None):
    """step.py:37-63 through the device sampler's spawn stage."""
    if count == 0:
        return []
    from .rng import seeds_to_tensor
    p, b = _grid_batch(occupancy, count, region_mask)
    seeds = seeds_to_tensor([seed], b.device)
    err = _lib.lib().cw_spawn_agents(p, 1, _lib.ptr(seeds), None, _lib.ptr(b.seed_scratch),
                                     b.buffers(), _lib.stream_ptr())
    _lib.check(err, "cw_spawn_agents")
    b.check_status()
    pos, goal = b.sp_pos[0].cpu().numpy(), b.sp_goal[0].cpu().numpy()
    kind, pref = b.sp_kind[0].cpu().numpy(), b.sp_pref[0].cpu().numpy()
    return [CrowdAgent(id=i, position=pos[i], velocity=np.zeros(2),
                       radius=RADIUS_OF_KIND[AgentKind(int(kind[i]))], preferred_speed=float(pref[i]),
                       goal=goal[i], kind=AgentKind(int(kind[i]))) for i in range(count)]


def sample_routes(occupancy, count, seed, kind=AgentKind.PEDESTRIAN, region_mask=None, max_radius=None):
    """routes.py:35-87 on the device (k_spawn's route stage): ``count`` connected
    (start, goal) pairs, Walkable cells (| Roadway for vehicle kinds), starts at
    least 2 * radius apart, goal in the start's 8-connected component."""
    if count == 0:
        return []
    from .rng import seeds_to_tensor
    p, b = _grid_batch(occupancy, count, region_mask)
    p.route_roadway = 0 if AgentKind(kind) == AgentKind.PEDESTRIAN else 1
    p.route_max_radius = float(max_radius if max_radius is not None else RADIUS_OF_KIND[AgentKind(kind)])
    seeds = seeds_to_tensor([seed], b.device)
    err = _lib.lib().cw_sample_routes(p, 1, _lib.ptr(seeds), None, _lib.ptr(b.seed_scratch), b.buffers(),
                                      _lib.stream_ptr())
    _lib.check(err, "cw_sample_routes")
    b.check_status()
    pos, goal = b.sp_pos[0].cpu().numpy(), b.sp_goal[0].cpu().numpy()
    return [(pos[i].copy(), goal[i].copy()) for i in range(count)]


def connected_components(ok):
    """routes.py:14-32: 8-connected component id per True cell (numbered in
    row-major order of each component's first cell), -1 elsewhere."""
    import torch
    ok = np.asarray(ok, dtype=bool)
    ny, nx = ok.shape
    dev = torch.device("cuda")
    okt = torch.from_numpy(ok.astype(np.uint8)).to(dev).reshape(1, ny * nx)
    comp = torch.empty((1, ny * nx), dtype=torch.int32, device=dev)
    rank = torch.empty_like(comp)
    _lib.check(_lib.lib().cw_connected_components(nx, ny, 1, _lib.ptr(okt), _lib.ptr(comp), _lib.ptr(rank),
                                                  _lib.stream_ptr()), "cw_connected_components")
    return comp.reshape(ny, nx).cpu().numpy()


def write_trace(records, fh):
    """step.py:66-70: newline-delimited JSON {tick, env, id, x, y, vx, vy} records."""
    import json
    for rec in records:
        fh.write(json.dumps(rec, sort_keys=True, separators=(",", ":")))
        fh.write("\n")


# ---------------------------------------------------------------- ORCA (orca.py)
@dataclass
class HalfPlane:
    """types.py:83-97: permitted half of velocity space, (v - point) . normal >= 0."""
    point: np.ndarray
    normal: np.ndarray

    def __post_init__(self):
        self.point = np.asarray(self.point, dtype=np.float64)
        self.normal = np.asarray(self.normal, dtype=np.float64)

    def satisfied(self, v, tol=1e-9):
        v = np.asarray(v, dtype=np.float64)
        return float((v - self.point) @ self.normal) >= -tol


def _halfplanes(rel_pos, rel_vel, rr, horizon, dt, v_self, share):
    """cw_orca_halfplanes over n rows (the device _vo_halfplane)."""
    import torch
    dev = torch.device("cuda")
    n = len(rr)
    if n == 0:
        return np.zeros((0, 2)), np.zeros((0, 2))
    keep = [torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(shape))).to(dev)
            for x, shape in ((rel_pos, (n, 2)), (rel_vel, (n, 2)), (rr, (n,)), (horizon, (n,)),
                             (v_self, (n, 2)), (share, (n,)))]   # alive until the launch is queued
    pt = torch.empty((n, 2), dtype=torch.float64, device=dev)
    nm = torch.empty_like(pt)
    rp, rv, r, h, vs, sh = (_lib.ptr(k) for k in keep)
    _lib.check(_lib.lib().cw_orca_halfplanes(n, rp, rv, r, h, float(dt), vs, sh, _lib.ptr(pt), _lib.ptr(nm),
                                             _lib.stream_ptr()), "cw_orca_halfplanes")
    return pt.cpu().numpy(), nm.cpu().numpy()


def orca_halfplane(rel_pos, rel_vel, combined_radius, horizon, dt, v_self, share):
    """orca.py:23-73: one permitted half-plane (device VO construction)."""
    pt, nm = _halfplanes([rel_pos], [rel_vel], [combined_radius], [horizon], dt, [v_self], [share])
    return HalfPlane(point=pt[0], normal=nm[0])


def compute_orca_constraints(agent, neighbors, static_segments, config, robot=None):
    """orca.py:76-118: half-planes against the nearest ``max_neighbors`` crowd
    neighbours (ordered by (distance^2, id)), the robot (full responsibility) and
    static segments; the half-planes are built on the device in one launch."""
    pos = np.asarray(agent.position, dtype=np.float64)
    vel = np.asarray(agent.velocity, dtype=np.float64)
    in_range = []
    for other in neighbors:
        if other is agent:
            raise ValueError("agent must not be in its own neighbor list")
        d2 = float(((other.position - pos) ** 2).sum())
        if d2 < config.neighbor_distance ** 2:
            in_range.append((d2, other.id, other))
    in_range.sort(key=lambda t: (t[0], t[1]))
    rows = []   # (rel_pos, rel_vel, rr, horizon, share)
    for _, _, o in in_range[: config.max_neighbors]:
        rows.append((o.position - pos, vel - o.velocity, agent.radius + o.radius + config.safety_margin,
                     config.time_horizon, 0.5))
    if robot is not None:
        r_pos, r_vel, r_radius = robot
        r_pos = np.asarray(r_pos, dtype=np.float64)
        if float(((r_pos - pos) ** 2).sum()) < config.neighbor_distance ** 2:
            rows.append((r_pos - pos, vel - np.asarray(r_vel, dtype=np.float64),
                         agent.radius + r_radius + config.safety_margin, config.obstacle_time_horizon, 1.0))
    for seg in static_segments:
        a, b = np.asarray(seg[0], dtype=np.float64), np.asarray(seg[1], dtype=np.float64)
        ab = b - a
        denom = float(ab @ ab)
        closest = a if denom < 1e-12 else a + float(np.clip((pos - a) @ ab / denom, 0.0, 1.0)) * ab
        if float(((closest - pos) ** 2).sum()) < config.neighbor_distance ** 2:
            rows.append((closest - pos, vel.copy(), agent.radius + config.safety_margin,
                         config.obstacle_time_horizon, 1.0))
    if not rows:
        return []
    pt, nm = _halfplanes([r[0] for r in rows], [r[1] for r in rows], [r[2] for r in rows],
                         [r[3] for r in rows], config.dt, [vel] * len(rows), [r[4] for r in rows])
    return [HalfPlane(point=pt[i], normal=nm[i]) for i in range(len(rows))]


def _batched_lp(points, normals, valid, pref, max_speed, lane_active):
    """field.py:500-566 on the device (cw_orca_lp, the LP k_orca runs): closest
    point of the speed disc to ``pref`` in the valid half-planes of each row,
    least-violation fallback for infeasible rows."""
    import torch
    dev = torch.device("cuda")
    points = np.asarray(points, dtype=np.float64)
    N, L = np.asarray(valid).shape
    if N == 0:
        return np.zeros((0, 2))
    keep = [torch.from_numpy(np.ascontiguousarray(np.asarray(x).astype(dt))).to(dev)
            for x, dt in ((points, np.float64), (normals, np.float64), (valid, np.uint8), (pref, np.float64),
                          (max_speed, np.float64), (lane_active, np.uint8))]   # alive until queued
    out = torch.empty((N, 2), dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().cw_orca_lp(N, L, *(_lib.ptr(k) for k in keep), _lib.ptr(out), None, _lib.stream_ptr()),
               "cw_orca_lp")
    return out.cpu().numpy()


def solve_velocity(preferred, constraints, max_speed):
    """orca.py:130-152: one row of the device LP over the given half-planes."""
    if max_speed <= 0:
        raise ValueError("max_speed must be > 0")
    n = len(constraints)
    pts = np.array([hp.point for hp in constraints], dtype=np.float64).reshape(1, n, 2)
    nms = np.array([hp.normal for hp in constraints], dtype=np.float64).reshape(1, n, 2)
    return _batched_lp(pts, nms, np.ones((1, n), dtype=bool), np.asarray(preferred, np.float64).reshape(1, 2),
                       np.array([float(max_speed)]), np.ones(1, dtype=bool))[0]


def feasible(constraints, v, tol=1e-9):
    """orca.py:245-246."""
    return all(hp.satisfied(v, tol) for hp in constraints)


class DeviceView:
    """numpy-like window onto a device tensor (the reference's state arrays).

    Reading (``np.asarray``, arithmetic, ``.copy()``, ``.shape`` ...) works on a host
    copy; ``view[idx] = value`` writes through to the device.  Basic indexing
    returns a DeviceView of the tensor view, so ``field.pos[e][a] = p`` also writes
    through; advanced indexing returns copies, as in numpy."""

    __slots__ = ("t", "_np_dtype")

    def __init__(self, t, np_dtype=None):
        self.t = t
        self._np_dtype = np_dtype

    def __array__(self, dtype=None, copy=None):
        a = self.t.detach().cpu().numpy()
        if self._np_dtype is not None:
            a = a.astype(self._np_dtype)
        return a if dtype is None else a.astype(dtype)

    def numpy(self):
        return self.__array__()

    def _index(self, idx):
        import torch
        conv = lambda i: torch.from_numpy(np.asarray(i)).to(self.t.device) if isinstance(i, (np.ndarray, list)) else i
        return tuple(conv(i) for i in idx) if isinstance(idx, tuple) else conv(idx)

    def __getitem__(self, idx):
        r = self.t[self._index(idx)]
        if r.dim() == 0:
            v = r.item()
            return np.bool_(v) if self._np_dtype is bool else np.asarray(r.cpu().numpy())[()]
        return DeviceView(r, self._np_dtype)

    def __setitem__(self, idx, value):
        import torch
        if isinstance(value, DeviceView):
            value = value.t
        v = torch.as_tensor(np.asarray(value) if not isinstance(value, torch.Tensor) else value)
        self.t[self._index(idx)] = v.to(device=self.t.device, dtype=self.t.dtype)

    def __len__(self):
        return int(self.t.shape[0])

    def __iter__(self):
        return iter(self.__array__())

    def __repr__(self):
        return f"DeviceView({self.__array__()!r})"

    def __getattr__(self, name):          # shape, dtype, copy, sum, reshape, tolist, ...
        if name.startswith("__"):
            # never hand out a temporary array's buffer protocol (__array_interface__,
            # __array_struct__ ...): numpy must go through __array__ and own its copy
            raise AttributeError(name)
        return getattr(self.__array__(), name)

    def __array_ufunc__(self, ufunc, method, *inputs, **kw):
        inputs = tuple(np.asarray(x) if isinstance(x, DeviceView) else x for x in inputs)
        return getattr(ufunc, method)(*inputs, **kw)

    def __array_function__(self, func, types, args, kwargs):
        conv = lambda x: np.asarray(x) if isinstance(x, DeviceView) else (
            type(x)(conv(y) for y in x) if isinstance(x, (list, tuple)) else x)
        return func(*conv(args), **{k: conv(v) for k, v in kwargs.items()})


def _binop(name):
    def f(self, other):
        other = np.asarray(other) if isinstance(other, DeviceView) else other
        return getattr(self.__array__(), name)(other)
    f.__name__ = name
    return f


for _n in ("__add__", "__radd__", "__sub__", "__rsub__", "__mul__", "__rmul__", "__truediv__",
           "__rtruediv__", "__floordiv__", "__pow__", "__mod__", "__neg__", "__pos__", "__abs__",
           "__eq__", "__ne__", "__lt__", "__le__", "__gt__", "__ge__", "__and__", "__or__",
           "__xor__", "__invert__", "__matmul__", "__rmatmul__"):
    if _n in ("__neg__", "__pos__", "__abs__", "__invert__"):
        setattr(DeviceView, _n, (lambda n: lambda self: getattr(self.__array__(), n)())(_n))
    else:
        setattr(DeviceView, _n, _binop(_n))
DeviceView.__hash__ = None
