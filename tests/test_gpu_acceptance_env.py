"""The reference's batch acceptance tests on the device (reference
tests/test_acceptance.py:258-325): batch trajectories bit-equal a sequential replay of
single envs, are invariant to the worker count, and Async == Sync at K = 1."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _act(seed, t):
    from paper_2505_00690_b200.rng import child_seed
    return np.random.Generator(np.random.PCG64(child_seed(seed, "acc-act", t))).uniform(-1, 1, 2)


def test_batch_determinism_replay_and_workers(torch_cuda):
    from paper_2505_00690_b200.envcore import BatchedEnv, Scheme
    from paper_2505_00690_b200.urbangen import SceneSpec, TaskKind
    spec = SceneSpec(seed=0, extent_m=(10.0, 10.0), task_kind=TaskKind.NAV_DYNAMIC, pedestrian_count=2)
    T = 200
    for K in (1, 8, 64):
        batch = BatchedEnv(spec, Scheme.ASYNC, master_seed=31, k=K)
        traj = np.zeros((T, K, 4))
        for t in range(T):
            batch.step_batch(np.stack([_act(batch.env_seeds[i], t) for i in range(K)]))
            traj[t] = np.stack([batch.x, batch.y, batch.vx, batch.vy], axis=-1)
        check = range(K) if K <= 8 else [0, 13, 31, 47, 63]
        for i in check:
            solo = BatchedEnv(spec, Scheme.ASYNC, master_seed=31, k=1, env_seeds=[batch.env_seeds[i]])
            for t in range(T):
                solo.step_batch(_act(batch.env_seeds[i], t)[None])
                row = np.array([solo.x[0], solo.y[0], solo.vx[0], solo.vy[0]])
                assert np.array_equal(row, traj[t, i]), (K, i, t)
        env = BatchedEnv(spec, Scheme.ASYNC, master_seed=31, k=K)
        for t in range(T):
            env.step_batch(np.stack([_act(env.env_seeds[i], t) for i in range(K)]), workers=4)
        assert np.array_equal(np.stack([env.x, env.y, env.vx, env.vy], axis=-1), traj[-1]), K


def test_scheme_semantics_async_equals_sync_at_k1(torch_cuda):
    from paper_2505_00690_b200.envcore import BatchedEnv, Scheme
    from paper_2505_00690_b200.urbangen import SceneSpec, TaskKind
    spec = SceneSpec(seed=0, extent_m=(10.0, 10.0), task_kind=TaskKind.NAV_STATIC)
    trajs = {}
    for scheme in (Scheme.ASYNC, Scheme.SYNC):
        env = BatchedEnv(spec, scheme, master_seed=5, k=1)
        rng = np.random.default_rng(9)
        rows = []
        for _ in range(200):
            env.step_batch(rng.uniform(-1, 1, (1, 2)))
            rows.append((env.x[0], env.y[0], env.yaw[0], env.vx[0], env.vy[0]))
        trajs[scheme] = rows
    assert trajs[Scheme.ASYNC] == trajs[Scheme.SYNC]
    a8 = BatchedEnv(spec, Scheme.ASYNC, master_seed=5, k=8)
    s8 = BatchedEnv(spec, Scheme.SYNC, master_seed=5, k=8)
    assert len(set(a8.scene_hashes)) == 8
    assert len(set(s8.scene_hashes)) == 1
