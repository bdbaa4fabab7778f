"""Generate tests/golden/dropin.npz from the REAL reference (build container only).

Run:  PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_dropin.py

Known answers for the drop-in entry points beyond the batched tick:
  * crowd/routes.py:35 sample_routes (kinds, region masks, max_radius) and
    routes.py:14 connected_components, step.py:37 spawn_agents(region_mask=)
  * urbangen/occupancy.py:28 rasterize_occupancy(scene, resolution) at resolutions
    other than the spec's (the scene travels as its canonical JSON)
  * crowd/field.py:448 _vo_halfplane, :500 _batched_lp and :214/:229
    _preferred_velocities/_build_constraints on seeded crowds
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
MIX = {"Flat": 0.25, "Slope": 0.25, "Stair": 0.25, "Rough": 0.25}


def main():
    sys.path.insert(0, REF)
    from citywalk.crowd import AgentKind, CrowdAgent, CrowdConfig, CrowdField
    from citywalk.crowd import connected_components, sample_routes, spawn_agents
    from citywalk.crowd.field import _batched_lp, _vo_halfplane
    from citywalk.rng import child_seed
    from citywalk.urbangen import SceneSpec, TaskKind, generate_scene, rasterize_occupancy
    from citywalk.urbangen.scene import scene_to_json
    out = {}

    # ---- scenes (as JSON) + rasters at other resolutions
    scenes = [(child_seed(0, "env", 0), 32.0, 0.25, "NavDynamic", 20 / 41, [0.2, 0.5, 0.125, 0.3]),
              (child_seed(0, "env", 1), 32.0, 0.125, "NavDynamic", 64 / 41, [0.25, 0.1]),
              (3, 48.0, 0.25, "NavStatic", 0.5, [0.4, 0.15])]
    occs = []
    for n, (seed, ext, res, task, dens, rlist) in enumerate(scenes):
        spec = SceneSpec(seed=seed, extent_m=(ext, ext), task_kind=TaskKind(task), object_density=dens,
                         pedestrian_count=0, terrain_mix=MIX, grid_resolution_m=res)
        sc = generate_scene(spec)
        out[f"s{n}_json"] = np.array(scene_to_json(sc))
        out[f"s{n}_res"] = np.array(rlist, np.float64)
        for k, r in enumerate(rlist):
            o = rasterize_occupancy(sc, r)
            out[f"s{n}_r{k}_labels"] = o.labels
            out[f"s{n}_r{k}_elev"] = o.elevation
        occs.append(rasterize_occupancy(sc))
        out[f"s{n}_labels"] = occs[-1].labels
        print("scene", n, len(sc.objects))
    out["n_scenes"] = np.int64(len(scenes))

    # ---- routes / components / spawn with region masks
    cases = []
    for n, occ in enumerate(occs):
        ny, nx = occ.labels.shape
        rng = np.random.default_rng(100 + n)
        cols = np.arange(nx)
        band = np.broadcast_to((cols > nx // 5) & (cols < 4 * nx // 5), (ny, nx)).copy()
        rnd = rng.random((ny, nx)) < 0.7
        for k, (count, seed, kind, mask, mr) in enumerate([
                (8, 11 + n, AgentKind.PEDESTRIAN, None, None),
                (12, 12 + n, AgentKind.CYCLIST, None, None),
                (6, 13 + n, AgentKind.PEDESTRIAN, band, 0.45),
                (5, 14 + n, AgentKind.SCOOTER, rnd, None)]):
            routes = sample_routes(occ, count, seed, kind=kind, region_mask=mask, max_radius=mr)
            key = f"rt{n}_{k}"
            out[key + "_args"] = np.array(json.dumps(dict(count=count, seed=seed, kind=int(kind),
                                                          max_radius=mr, scene=n)))
            out[key + "_mask"] = np.zeros((0, 0), bool) if mask is None else mask
            out[key + "_routes"] = np.array([[s, g] for s, g in routes], np.float64)
            cases.append(key)
        walk = occ.labels == 2
        out[f"cc{n}_walk"] = connected_components(walk)
        out[f"cc{n}_rnd"] = connected_components(rnd & (occ.labels != 0))
        sp = spawn_agents(occ, 10, child_seed(7, "crowd", n), region_mask=band)
        out[f"sp{n}"] = np.array([[a.position[0], a.position[1], a.goal[0], a.goal[1], a.preferred_speed,
                                   int(a.kind)] for a in sp], np.float64)
    out["route_cases"] = np.array(cases)

    # ---- half-planes, batched LP, constraints on seeded crowds
    rng = np.random.default_rng(7)
    n = 4000
    rel_pos = rng.uniform(-3, 3, (n, 2))
    rel_pos[:200] *= 0.05                       # colliding rows
    rel_vel = rng.uniform(-2, 2, (n, 2))
    rr = rng.uniform(0.5, 1.0, n)
    v_self = rng.uniform(-1.5, 1.5, (n, 2))
    pt1, nm1 = _vo_halfplane(rel_pos, rel_vel, rr, 2.0, 0.05, v_self, 0.5)
    pt2, nm2 = _vo_halfplane(rel_pos, rel_vel, rr, 1.0, 0.05, v_self, 1.0)
    out.update(hp_rel_pos=rel_pos, hp_rel_vel=rel_vel, hp_rr=rr, hp_v_self=v_self,
               hp_pt_h2=pt1, hp_nm_h2=nm1, hp_pt_h1=pt2, hp_nm_h1=nm2)
    N, L = 3000, 12
    points = rng.uniform(-1.5, 1.5, (N, L, 2))
    ang = rng.uniform(0, 2 * np.pi, (N, L))
    normals = np.stack([np.cos(ang), np.sin(ang)], -1)
    valid = rng.random((N, L)) < 0.6
    pref = rng.uniform(-3, 3, (N, 2))
    ms = rng.uniform(0.5, 2.5, N)
    act = rng.random(N) < 0.9
    v = _batched_lp(points, normals, valid, pref, ms, act)
    out.update(lp_points=points, lp_normals=normals, lp_valid=valid, lp_pref=pref, lp_ms=ms, lp_act=act,
               lp_out=v)

    for m, (A, side, robot) in enumerate([(10, 15.0, False), (24, 12.0, True), (40, 14.0, True)]):
        from citywalk.urbangen.types import OccupancyGrid
        res = 0.1
        nc = int(side / res)
        labels = np.full((nc, nc), 2, np.uint8)
        if m == 2:
            labels[60:80, 30:90] = 0          # a wall: static lane
        occ = OccupancyGrid(resolution=res, labels=labels, elevation=np.zeros((nc, nc), np.float32))
        E = 3
        lists = []
        for e in range(E):
            r = np.random.default_rng(1000 * m + e)
            lst = []
            while len(lst) < A - e:
                p = r.uniform(1, side - 1, 2)
                if labels[int(p[1] / res), int(p[0] / res)] == 0:
                    continue
                if all(np.hypot(*(p - o.position)) > 0.65 for o in lst):
                    lst.append(CrowdAgent(id=len(lst), position=p, velocity=r.uniform(-1, 1, 2), radius=0.3,
                                          preferred_speed=float(r.uniform(0.8, 1.4)),
                                          goal=r.uniform(1, side - 1, 2)))
            lists.append(lst)
        f = CrowdField([occ] * E, CrowdConfig(), env_seeds=list(range(E)), resample_goals=False)
        f.set_agents(lists)
        f.waypoint[:] = f.goal + 0.25        # waypoints apart from goals (pref scaling)
        act = f.active.copy()
        act[1, 3] = False
        rp = np.array([[5.0, 5.0], [6.0, 4.0], [7.0, 7.0]]) if robot else None
        rv = np.array([[0.3, -0.2], [0.0, 0.5], [-0.4, 0.1]]) if robot else None
        pref = f._preferred_velocities(0, E, act)
        pts, nms, val = f._build_constraints(0, E, act, rp, rv, 0.35)
        key = f"bc{m}"
        out[key + "_pos"] = f.pos.copy()
        out[key + "_vel"] = f.vel.copy()
        out[key + "_goal"] = f.goal.copy()
        out[key + "_waypoint"] = f.waypoint.copy()
        out[key + "_radius"] = f.radius.copy()
        out[key + "_pref_speed"] = f.pref_speed.copy()
        out[key + "_active"] = f.active.copy()
        out[key + "_labels"] = labels
        out[key + "_act"] = act
        out[key + "_robot"] = np.zeros((0, 2)) if rp is None else np.concatenate([rp, rv], 1)
        out[key + "_pref"] = pref
        out[key + "_points"] = pts
        out[key + "_normals"] = nms
        out[key + "_valid"] = val
        print("constraints", m, pts.shape)
    np.savez_compressed(os.path.join(OUT, "dropin.npz"), **out)


if __name__ == "__main__":
    main()
