"""ctypes binding of libcitywalk_b200.so (the C ABI in include/citywalk_b200.h).

The library is built in-tree (``build()``) for sm_100a.  There is no CPU
fallback: importing the product API without the library raises.
"""

import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.path.join(HERE, "libcitywalk_b200.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("sample.cu", "crowd.cu", "robot.cu", "routes.cu", "sceneio.cu")]
HEADERS = sorted(os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))
                 if f.endswith(".cuh")) + [os.path.join(ROOT, "include", "citywalk_b200.h")]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false",
              "-std=c++17", "-Xcompiler", "-fPIC", "-shared"]

MAX_TILES = 44
MAX_CAT = 32
MAX_BLOCKS = 64
ZONE_PARAMS = 8

c_i32, c_u32, c_f64, c_f32, c_i64 = ctypes.c_int32, ctypes.c_uint32, ctypes.c_double, ctypes.c_float, ctypes.c_int64
P = ctypes.c_void_p


class SceneParams(ctypes.Structure):
    _fields_ = [
        ("nx", c_i32), ("ny", c_i32), ("res", c_f64), ("w", c_f64), ("l", c_f64),
        ("task", c_i32), ("split", c_i32), ("mix", c_f64 * 4), ("layout", c_i32),
        ("brows", c_i32), ("bcols", c_i32), ("quad_cdf", c_f64 * 3),
        ("trows", c_i32), ("tcols", c_i32), ("cpt", c_i32), ("nonflat_split_col", c_i32),
        ("n_cat", c_i32), ("cat_w", c_f64 * MAX_CAT), ("cat_l", c_f64 * MAX_CAT),
        ("cat_reach", c_f64 * MAX_CAT), ("cat_zones", c_u32 * MAX_CAT),
        ("small_first", c_i32 * MAX_CAT), ("obj_count", c_i32), ("obj_max", c_i32),
        ("attempts", c_i32), ("region", c_i32), ("peds", c_i32), ("spawn_region", c_i32),
        ("route_roadway", c_i32), ("route_max_radius", c_f64),
    ]


SCENE_BUFFER_FIELDS = [
    "zones", "labels", "elev", "assign", "n_tiles", "tile_code", "tile_kind", "tile_param",
    "tile_p", "tile_w", "allowed", "noise_seed", "wfc_attempts", "obj_cat", "obj_pose", "obj_n",
    "overflow", "nearest", "has_obs", "walk", "walk_n", "reach", "moves", "sp_pos", "sp_goal", "sp_kind", "sp_pref",
    "status", "scratch_i32", "scratch_f64", "zone_params", "block_var", "region", "epoch",
]


class SceneBuffers(ctypes.Structure):
    _fields_ = [(n, P) for n in SCENE_BUFFER_FIELDS]


class CrowdParams(ctypes.Structure):
    _fields_ = [
        ("E", c_i32), ("A", c_i32), ("nx", c_i32), ("ny", c_i32), ("res", c_f64), ("res0", c_f64),
        ("time_horizon", c_f64), ("obstacle_time_horizon", c_f64), ("neighbor_distance", c_f64),
        ("nd2", c_f64), ("nd2_f32", c_f32), ("max_neighbors", c_i32), ("dt", c_f64),
        ("safety_margin", c_f64), ("goal_reach2", c_f64), ("stall_c", c_f64), ("stall_s", c_f64),
        ("resample_goals", c_i32), ("use_static", c_i32), ("path_cap", c_i32), ("heap_cap", c_i32),
        ("astar_ctas", c_i32), ("astar_warps", c_i32), ("run_server_warps", c_i32),
    ]


CROWD_STATE_FIELDS = [
    "pos", "vel", "goal", "waypoint", "radius", "pref_speed", "max_speed", "active", "path_cells",
    "path_head", "path_n", "labels", "nearest", "has_obs", "walk", "walk_n", "reach", "moves",
    "rng", "last_gap", "gap_tmp", "flags", "astar_rec", "astar_heap", "astar_req",
    "counters", "env_req", "spec", "env_epoch",
]


class CrowdState(ctypes.Structure):
    _fields_ = [(n, P) for n in CROWD_STATE_FIELDS]


class RobotModel(ctypes.Structure):
    _fields_ = [("body_radius", c_f64), ("max_speed", c_f64), ("holonomic", c_i32),
                ("wheelbase", c_f64), ("max_steer", c_f64), ("max_step_rise", c_f64),
                ("max_grade", c_f64), ("max_roughness", c_f64)]


class RobotParams(ctypes.Structure):
    _fields_ = [("E", c_i32), ("A", c_i32), ("nx", c_i32), ("ny", c_i32), ("res", c_f64),
                ("dt", c_f64), ("reach_threshold", c_f64), ("horizon", c_i32),
                ("terminal_reach", c_f64), ("terminal_oob", c_f64), ("c1", c_f64), ("c2", c_f64),
                ("c3", c_f64), ("track_far", c_f64), ("track_near", c_f64),
                ("track_near_weight", c_f64), ("model", RobotModel)]


ROBOT_STATE_FIELDS = [
    "x", "y", "yaw", "vx", "vy", "elev", "goal", "tick", "terminated", "truncated", "labels",
    "grid_elev", "passable", "crowd_pos", "crowd_radius", "crowd_active", "reward", "events",
    "distance", "path_inc", "depth", "goal_vector", "proj_vel", "height_map", "semantics",
]


class RobotState(ctypes.Structure):
    _fields_ = [(n, P) for n in ROBOT_STATE_FIELDS]


EXPORTS = ["cw_scene_seed_scratch_bytes", "cw_sample_scenes", "cw_sample_scenes_routes", "cw_spawn_agents", "cw_prepare_envs",
           "cw_crowd_step_smem_bytes",
           "cw_crowd_step", "cw_crowd_step_phases", "cw_astar_slot_bytes", "cw_astar_warps",
           "cw_traversability_scratch_bytes", "cw_traversability", "cw_robot_step", "cw_robot_observe",
           "cw_route_scratch_bytes", "cw_route_anchors", "cw_seed_streams", "cw_child_seeds", "cw_abi_sizes",
           "cw_scene_rle", "cw_crowd_run_scratch_bytes", "cw_crowd_run",
           "cw_crowd_run_rounds", "cw_crowd_run_servers", "cw_crowd_run_window", "cw_sample_routes", "cw_connected_components",
           "cw_rasterize", "cw_orca_lp", "cw_orca_halfplanes", "cw_crowd_constraints", "cw_trig_probe",
           "cw_spec_bytes", "cw_spec_create", "cw_spec_destroy", "cw_spec_stats", "cw_spec_predict",
           "cw_spec_install"]

_lib = None


def build(force=False, verbose=False):
    """Compile the CUDA library in-tree for sm_100a (nvcc cross-compiles without a GPU).
    One nvcc per translation unit in parallel, then one link."""
    from concurrent.futures import ThreadPoolExecutor
    newest = max(os.path.getmtime(p) for p in SOURCES + HEADERS)
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= newest:
        return LIB_PATH
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in NVCC_FLAGS if f != "-shared"]
    inc = ["-I", os.path.join(ROOT, "include")]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = ["nvcc"] + cflags + inc + ["-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as pool:
        objs = list(pool.map(compile_one, SOURCES))
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           "-o", LIB_PATH] + objs
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return LIB_PATH


def lib():
    """Load the library (raises if it was not built; no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("CW_LIB_PATH", LIB_PATH)   # A/B builds of the same ABI (tools/)
    if not os.path.exists(path):
        raise RuntimeError(f"libcitywalk_b200.so not built ({path}); run __graft_entry__.build()")
    L = ctypes.CDLL(path)
    L.cw_scene_seed_scratch_bytes.restype = ctypes.c_size_t
    L.cw_scene_seed_scratch_bytes.argtypes = [ctypes.c_int]
    L.cw_scene_rle.restype = ctypes.c_int
    L.cw_scene_rle.argtypes = [ctypes.POINTER(SceneParams), ctypes.c_int, P,
                               ctypes.POINTER(SceneBuffers), P, P, P, P]
    L.cw_sample_scenes.restype = ctypes.c_int
    L.cw_sample_scenes.argtypes = [ctypes.POINTER(SceneParams), ctypes.c_int, P, P, P, P,
                                   ctypes.POINTER(SceneBuffers), P]
    L.cw_sample_scenes_routes.restype = ctypes.c_int
    L.cw_sample_scenes_routes.argtypes = [ctypes.POINTER(SceneParams), ctypes.c_int, P, P, P, P,
                                          ctypes.POINTER(SceneBuffers), P, P, P, ctypes.c_int, P]
    L.cw_spawn_agents.restype = ctypes.c_int
    L.cw_spawn_agents.argtypes = [ctypes.POINTER(SceneParams), ctypes.c_int, P, P, P,
                                  ctypes.POINTER(SceneBuffers), P]
    L.cw_prepare_envs.restype = ctypes.c_int
    L.cw_prepare_envs.argtypes = [ctypes.POINTER(SceneParams), ctypes.c_int, P,
                                  ctypes.POINTER(SceneBuffers), P]
    L.cw_crowd_step_smem_bytes.restype = ctypes.c_size_t
    L.cw_crowd_step_smem_bytes.argtypes = [ctypes.c_int, ctypes.c_int]
    L.cw_crowd_step.restype = ctypes.c_int
    L.cw_crowd_step.argtypes = [ctypes.POINTER(CrowdParams), ctypes.POINTER(CrowdState), P, P,
                                ctypes.c_double, P, ctypes.c_int, P]
    L.cw_crowd_step_phases.restype = ctypes.c_int
    L.cw_crowd_step_phases.argtypes = [ctypes.POINTER(CrowdParams), ctypes.POINTER(CrowdState), P,
                                       P, ctypes.c_double, P, ctypes.c_int, ctypes.c_int, P]
    L.cw_crowd_run_scratch_bytes.restype = ctypes.c_size_t
    L.cw_crowd_run_scratch_bytes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
    L.cw_crowd_run_window.restype = ctypes.c_int
    L.cw_crowd_run_window.argtypes = [ctypes.POINTER(CrowdParams), ctypes.POINTER(CrowdState), P, P,
                                      ctypes.c_double, P, ctypes.c_int, ctypes.c_int, P, P, ctypes.c_int, P, P]
    L.cw_crowd_run_rounds.restype = ctypes.c_longlong
    L.cw_crowd_run_rounds.argtypes = []
    L.cw_crowd_run_servers.restype = ctypes.c_longlong
    L.cw_crowd_run_servers.argtypes = []
    L.cw_spec_bytes.restype = ctypes.c_size_t
    L.cw_spec_bytes.argtypes = [ctypes.POINTER(CrowdParams)]
    L.cw_spec_create.restype = ctypes.c_int
    L.cw_spec_create.argtypes = [ctypes.POINTER(CrowdParams), ctypes.POINTER(ctypes.c_void_p)]
    L.cw_spec_destroy.restype = ctypes.c_int
    L.cw_spec_destroy.argtypes = [ctypes.c_void_p]
    L.cw_spec_predict.restype = ctypes.c_int
    L.cw_spec_predict.argtypes = [ctypes.POINTER(CrowdParams), ctypes.POINTER(CrowdState), ctypes.c_void_p, P,
                                  ctypes.c_int, ctypes.c_int, P]
    L.cw_spec_install.restype = ctypes.c_int
    L.cw_spec_install.argtypes = [ctypes.c_void_p, ctypes.c_void_p, P, P, P, ctypes.c_int, P]
    L.cw_spec_stats.restype = ctypes.c_int
    L.cw_spec_stats.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong)]
    L.cw_crowd_run.restype = ctypes.c_int
    L.cw_crowd_run.argtypes = [ctypes.POINTER(CrowdParams), ctypes.POINTER(CrowdState), P, P,
                               ctypes.c_double, P, ctypes.c_int, ctypes.c_int, P, P]
    L.cw_astar_warps.restype = ctypes.c_int
    L.cw_astar_warps.argtypes = []
    L.cw_astar_slot_bytes.restype = ctypes.c_size_t
    L.cw_astar_slot_bytes.argtypes = [ctypes.c_int, ctypes.c_int]
    L.cw_seed_streams.restype = ctypes.c_int
    L.cw_seed_streams.argtypes = [ctypes.c_int, P, P, P]
    L.cw_child_seeds.restype = ctypes.c_int
    L.cw_child_seeds.argtypes = [ctypes.c_int, P, ctypes.c_int, P, P, P]
    L.cw_traversability_scratch_bytes.restype = ctypes.c_size_t
    L.cw_traversability_scratch_bytes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
    L.cw_traversability.restype = ctypes.c_int
    L.cw_traversability.argtypes = [ctypes.POINTER(RobotParams), ctypes.c_int, P, P, P, P, P,
                                    ctypes.c_int, P]
    L.cw_robot_step.restype = ctypes.c_int
    L.cw_robot_step.argtypes = [ctypes.POINTER(RobotParams), ctypes.POINTER(RobotState), P, P]
    L.cw_robot_observe.restype = ctypes.c_int
    L.cw_robot_observe.argtypes = [ctypes.POINTER(RobotParams), ctypes.POINTER(RobotState), P]
    L.cw_route_scratch_bytes.restype = ctypes.c_size_t
    L.cw_route_scratch_bytes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
    L.cw_route_anchors.restype = ctypes.c_int
    L.cw_route_anchors.argtypes = [ctypes.POINTER(SceneParams), ctypes.c_int, P, P,
                                   ctypes.POINTER(SceneBuffers), P, P, P, ctypes.c_int, P]
    L.cw_sample_routes.restype = ctypes.c_int
    L.cw_sample_routes.argtypes = [ctypes.POINTER(SceneParams), ctypes.c_int, P, P, P,
                                   ctypes.POINTER(SceneBuffers), P]
    L.cw_connected_components.restype = ctypes.c_int
    L.cw_connected_components.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P, P]
    L.cw_rasterize.restype = ctypes.c_int
    L.cw_rasterize.argtypes = [ctypes.POINTER(SceneParams), ctypes.c_int, P, ctypes.c_int, ctypes.c_int,
                               ctypes.c_double, ctypes.POINTER(SceneBuffers), P]
    L.cw_orca_lp.restype = ctypes.c_int
    L.cw_orca_lp.argtypes = [ctypes.c_int, ctypes.c_int, P, P, P, P, P, P, P, P, P]
    L.cw_orca_halfplanes.restype = ctypes.c_int
    L.cw_orca_halfplanes.argtypes = [ctypes.c_int, P, P, P, P, ctypes.c_double, P, P, P, P, P]
    L.cw_crowd_constraints.restype = ctypes.c_int
    L.cw_crowd_constraints.argtypes = [ctypes.POINTER(CrowdParams), ctypes.POINTER(CrowdState), ctypes.c_int,
                                       ctypes.c_int, P, P, P, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                       P, P, P, P, P, P, P]
    L.cw_trig_probe.restype = ctypes.c_int
    L.cw_trig_probe.argtypes = [ctypes.c_int, P, P, P, ctypes.c_int, P]
    L.cw_abi_sizes.restype = ctypes.c_int
    L.cw_abi_sizes.argtypes = [ctypes.POINTER(ctypes.c_size_t), ctypes.c_int]
    sizes = (ctypes.c_size_t * 6)()
    L.cw_abi_sizes(sizes, 6)
    mine = [ctypes.sizeof(SceneParams), ctypes.sizeof(SceneBuffers), ctypes.sizeof(CrowdParams),
            ctypes.sizeof(CrowdState), ctypes.sizeof(RobotParams), ctypes.sizeof(RobotState)]
    if list(sizes) != mine:
        raise RuntimeError(f"ABI mismatch: library {list(sizes)} vs ctypes {mine}")
    _lib = L
    return L


def check(err, what):
    if err != 0:
        raise RuntimeError(f"{what} failed with CUDA error {err}")


def ptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
