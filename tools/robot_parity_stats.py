"""Max deviations of the device robot step from the reference goldens (GPU)."""
import sys, os
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_golden
from paper_2505_00690_b200.robot import RobotBatch
for run in ["quadruped", "wheeled", "small"]:
    g = load_golden(f"robot_{run}.npz")
    K, T, peds, horizon, auto = (int(v) for v in g["meta"])
    rb = RobotBatch(torch.from_numpy(g["labels"]).cuda(), torch.from_numpy(g["grid_elev"]).cuda(), float(g["res"]), str(g["robot"]), horizon=horizon)
    tick = g["tick"][:, 0]; drop = np.flatnonzero(np.diff(tick) < 0); n = int(drop[0]) + 1 if (auto and drop.size) else T
    cr = torch.from_numpy(g["crowd_radius"]).cuda(); ca = torch.from_numpy(g["crowd_active"].astype(np.uint8)).cuda()
    mx = {}; deq = heq = nd = nh = 0
    for t in range(n):
        pre = {k: (g[f"init_{k}"] if t == 0 else g[k][t - 1]) for k in ("x","y","yaw","vx","vy","elev","tick","terminated","truncated")}
        rb.set_state(pre["x"], pre["y"], pre["yaw"], g["goal"][t], vx=pre["vx"], vy=pre["vy"], elev=pre["elev"], tick=pre["tick"], terminated=pre["terminated"], truncated=pre["truncated"])
        rb.step(g["actions"][t], (torch.from_numpy(g["crowd_pos"][t]).cuda(), cr, ca))
        for k, a in (("x", rb.x), ("y", rb.y), ("yaw", rb.yaw), ("reward", rb.reward), ("goal_vector", rb.goal_vector)):
            mx[k] = max(mx.get(k, 0.0), float(np.abs(a.cpu().numpy() - g[k][t]).max()))
        d = rb.depth.cpu().numpy(); h = rb.height_map.cpu().numpy()
        deq += (d == g["depth"][t]).sum(); nd += d.size; heq += (h == g["height_map"][t]).sum(); nh += h.size
    print(run, {k: f"{v:.2e}" for k, v in mx.items()}, f"depth exact {deq}/{nd}", f"hmap exact {heq}/{nh}")
