"""Batched env orchestration for the hot path (envcore/batch.py:62-346, cache.py).

``BatchedEnv`` keeps the reference constructor and seed tree -- per-env seeds
``child_seed(master, "env", i)`` (batch.py:84-96), crowd streams
``child_seed(env_seed, "crowd-run")`` (:165), spawns
``child_seed(env_seed, "crowd", reset_count)`` (:179), resample seeds
``child_seed(env_seed, "resample", n)`` (:332) -- but samples every env on the
device in one batch and steps the crowd with one kernel per tick.  The robot
step / observations / reward (batch.py:223-302) are SURVEY §8f "next" and not
part of this path: ``step_crowd`` advances the crowd with the caller's robot
pos/vel, as ``crowd.step`` does inside ``step_batch`` (batch.py:216-221).
"""

from dataclasses import dataclass, field, replace
from enum import Enum

import numpy as np

from . import _lib
from .crowd import CrowdConfig, CrowdField
from .errors import SlotOutOfRange
from .rng import child_seed, child_seeds_device, seeds_to_tensor
from .urbangen import SceneSampler, SceneSpec


class Scheme(str, Enum):
    ASYNC = "Async"
    SYNC = "Sync"


@dataclass
class EnvConfig:
    resample_on_reset: bool = False
    crowd: CrowdConfig = field(default_factory=CrowdConfig)


class BatchedEnv:
    """K env slots: device scenes + device crowd (batch.py:62)."""

    def __init__(self, specs, scheme, master_seed, k=None, cache=None, config=None,
                 env_seeds=None, device="cuda", threads=128, catalog=None):
        import torch
        self.config = config or EnvConfig()
        self.scheme = Scheme(scheme)
        if isinstance(specs, SceneSpec):
            k = 1 if k is None else k
            base = specs
        else:
            specs = list(specs)
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
        crowd_seeds = child_seeds_device(self.env_seeds_t, "crowd", 0)
        self.batch = self.sampler.sample(self.scene_seeds_t, crowd_seeds)
        run = child_seeds_device(self.env_seeds_t, "crowd-run").cpu().numpy().view(np.uint64)
        self.crowd = CrowdField(self.batch, self.config.crowd, [int(s) for s in run],
                                device=device, threads=threads)
        if self.spec.pedestrian_count > 0:
            self.crowd.set_from_spawn(self.batch)

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
        crowd_seed = child_seeds_device(env, "crowd", cnt)
        self.scene_seeds_t[sl] = new_scene
        self.sampler.sample(new_scene, crowd_seed, slots=sl)
        if respawn and self.spec.pedestrian_count > 0:
            self.crowd.set_from_spawn(self.batch, rows=sl)
        self.crowd.prepare_step()

    def reset(self, slot, resample=None):
        if not (0 <= slot < self.K):
            raise SlotOutOfRange(f"slot {slot} of {self.K}")
        do_resample = self.config.resample_on_reset if resample is None else resample
        if do_resample:
            self.resample([slot])
            return
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

    # -- stepping -------------------------------------------------------------------------
    def step_crowd(self, robot_pos=None, robot_vel=None, robot_radius=0.35, env_mask=None,
                   check=False):
        self.crowd.step(robot_pos=robot_pos, robot_vel=robot_vel, robot_radius=robot_radius,
                        env_mask=env_mask, check=check)

    def step_batch(self, actions, workers=1):
        raise NotImplementedError(
            "robot kinematics / observations / reward are SURVEY §8f 'next'; use step_crowd")
