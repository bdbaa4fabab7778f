"""Scene sampling on the B200 -- the reference's urbangen entry points, batched.

Mirrors /root/reference/pkg/src/citywalk/urbangen:
  * ``SceneSpec`` / ``TaskKind`` / ``Split`` / ``Zone`` / ``CellLabel`` (types.py:11-143)
  * ``generate_scene(spec, catalog=None)`` (scene.py:38) and
    ``rasterize_occupancy(scene, resolution=None)`` (occupancy.py:28)
  * ``load_catalog(path=None)`` (catalog.py:14-24)
plus the batch form the north star asks for: ``SceneSampler.sample(seeds)``
runs zones -> terrain WFC -> placement -> raster -> nearest-obstacle BFS ->
walk list -> spawn for every env on the device in one stream-ordered call
(``cw_sample_scenes``), then the route anchors (``cw_route_anchors``,
scene.py:87, 102-178).  Scene JSON / hashes (scene.py:163-238) are in
``sceneio`` (``SceneSampler.scene_dicts`` / ``scene_hashes``).
"""

import json
import math
import os
from dataclasses import dataclass, field
from enum import Enum, IntEnum

import numpy as np

from . import _lib
from .errors import STATUS_ERRORS


class TaskKind(str, Enum):
    NAV_CLEAR = "NavClear"
    NAV_STATIC = "NavStatic"
    NAV_DYNAMIC = "NavDynamic"
    TRAVERSE = "Traverse"


class Split(str, Enum):
    TRAIN = "Train"
    TEST = "Test"


class Zone(IntEnum):
    SIDEWALK = 0
    CROSSWALK = 1
    PLAZA = 2
    BUILDING = 3
    VEGETATION = 4
    ROADWAY = 5


class CellLabel(IntEnum):
    OBSTACLE = 0
    ROADWAY = 1
    WALKABLE = 2
    NON_WALKABLE_GROUND = 3


TERRAIN_FAMILIES = ("Flat", "Slope", "Stair", "Rough")
TERRAIN_KINDS = ("Flat", "SlopeUp", "SlopeDown", "StairUp", "StairDown", "Rough")
BLOCK_SIZE_M = 20.0
TILE_SIZE_M = 2.0
ATTEMPTS_PER_OBJECT = 100
_TASK_CODE = {TaskKind.NAV_CLEAR: 0, TaskKind.NAV_STATIC: 1, TaskKind.NAV_DYNAMIC: 2,
              TaskKind.TRAVERSE: 3}


@dataclass(frozen=True)
class SceneSpec:
    """urbangen/types.py:88-115 (same fields, defaults and validation)."""

    seed: int
    extent_m: tuple = (10.0, 10.0)
    task_kind: TaskKind = TaskKind.NAV_STATIC
    split: Split = Split.TRAIN
    object_density: float = 1.0
    pedestrian_count: int = 0
    terrain_mix: dict = field(
        default_factory=lambda: {"Flat": 0.7, "Slope": 0.1, "Stair": 0.0, "Rough": 0.2})
    grid_resolution_m: float = 0.1

    def __post_init__(self):
        w, l = self.extent_m
        if not (5.0 <= w <= 1200.0 and 5.0 <= l <= 1200.0):
            raise ValueError("extent_m components must lie in [5.0, 1200.0]")
        if self.object_density < 0:
            raise ValueError("object_density must be >= 0")
        if self.grid_resolution_m <= 0:
            raise ValueError("grid_resolution_m must be > 0")
        total = sum(self.terrain_mix.get(k, 0.0) for k in TERRAIN_FAMILIES)
        if abs(total - 1.0) > 1e-9:
            raise ValueError("terrain_mix weights must sum to 1")
        for k in self.terrain_mix:
            if k not in TERRAIN_FAMILIES:
                raise ValueError(f"unknown terrain family {k!r}")

    def to_dict(self):
        """types.py:117-127."""
        return {"seed": int(self.seed), "extent_m": [float(self.extent_m[0]), float(self.extent_m[1])],
                "task_kind": TaskKind(self.task_kind).value, "split": Split(self.split).value,
                "object_density": float(self.object_density), "pedestrian_count": int(self.pedestrian_count),
                "terrain_mix": {k: float(self.terrain_mix.get(k, 0.0)) for k in TERRAIN_FAMILIES},
                "grid_resolution_m": float(self.grid_resolution_m)}

    @staticmethod
    def from_dict(d):
        """types.py:129-140."""
        return SceneSpec(seed=int(d["seed"]), extent_m=(float(d["extent_m"][0]), float(d["extent_m"][1])),
                         task_kind=TaskKind(d["task_kind"]), split=Split(d["split"]),
                         object_density=float(d["object_density"]),
                         pedestrian_count=int(d["pedestrian_count"]), terrain_mix=dict(d["terrain_mix"]),
                         grid_resolution_m=float(d["grid_resolution_m"]))


@dataclass(frozen=True)
class CatalogEntry:
    category: str
    footprint: tuple
    height: float
    allowed_zones: tuple


def load_catalog(path=None):
    """catalog.py:14-24; the bundled default is data/catalog.json."""
    if path is None:
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "catalog.json")
    with open(path, "r", encoding="utf-8") as fh:
        entries = [CatalogEntry(d["category"], (float(d["footprint"][0]), float(d["footprint"][1])),
                                float(d["height"]), tuple(Zone[z] for z in d["allowed_zones"]))
                   for d in json.load(fh)]
    if not entries:
        raise ValueError("catalog is empty")
    return entries


@dataclass
class OccupancyGrid:
    """types.py:364-379."""

    resolution: float
    labels: np.ndarray
    elevation: np.ndarray

    @property
    def shape(self):
        return self.labels.shape

    def cell_of(self, x, y):
        return int(y / self.resolution), int(x / self.resolution)

    def in_bounds_cell(self, row, col):
        """types.py:377-379."""
        ny, nx = self.labels.shape
        return 0 <= row < ny and 0 <= col < nx


BLOCK_KINDS = ("Straight", "Curve", "Roundabout", "Diverging", "Merging", "Intersection",
               "TIntersection")
BLOCK_SOCKETS = ((1, 0, 1, 0), (1, 1, 0, 0), (1, 1, 1, 1), (1, 1, 0, 1), (1, 1, 0, 1),
                 (1, 1, 1, 1), (1, 1, 0, 1))   # types.py:148-156 (N, E, S, W)
DIR_N, DIR_E, DIR_S, DIR_W = 0, 1, 2, 3
SCHEMA_VERSION = 1


def rotated_sockets(kind, orientation):
    """types.py:159-163."""
    base = BLOCK_SOCKETS[BLOCK_KINDS.index(kind)]
    o = orientation % 4
    return tuple(base[(i - o) % 4] for i in range(4))


@dataclass
class BlockNode:
    """types.py:166-179."""
    kind: str
    cell: tuple
    orientation: int
    sockets: tuple

    def to_dict(self):
        return {"kind": self.kind, "cell": [int(self.cell[0]), int(self.cell[1])],
                "orientation": int(self.orientation), "sockets": [int(v) for v in self.sockets]}


@dataclass
class BlockGraph:
    """types.py:182-215; ``from_variants`` rebuilds edges / capped exactly as
    blocks.py:80-100 (_assemble) from the device's per-block variants."""
    rows: int
    cols: int
    nodes: list
    edges: list
    capped: list

    def node_at(self, row, col):
        return self.nodes[row * self.cols + col]

    @staticmethod
    def from_variants(rows, cols, variants):
        nodes = []
        for i in range(rows * cols):
            k, o = int(variants[i]) >> 2, int(variants[i]) & 3
            nodes.append(BlockNode(BLOCK_KINDS[k], (i // cols, i % cols), o,
                                   rotated_sockets(BLOCK_KINDS[k], o)))
        edges, capped = [], []
        for r in range(rows):
            for c in range(cols):
                so = nodes[r * cols + c].sockets
                if so[DIR_E]:
                    (edges.append(((r, c), (r, c + 1))) if c + 1 < cols else capped.append(((r, c), DIR_E)))
                if so[DIR_S]:
                    (edges.append(((r, c), (r + 1, c))) if r + 1 < rows else capped.append(((r, c), DIR_S)))
                if so[DIR_N] and r == 0:
                    capped.append(((r, c), DIR_N))
                if so[DIR_W] and c == 0:
                    capped.append(((r, c), DIR_W))
        return BlockGraph(rows, cols, nodes, edges, capped)

    def to_dict(self):
        return {"rows": int(self.rows), "cols": int(self.cols), "nodes": [n.to_dict() for n in self.nodes],
                "edges": [[[int(a[0]), int(a[1])], [int(b[0]), int(b[1])]] for a, b in self.edges],
                "capped": [[[int(c[0]), int(c[1])], int(d)] for c, d in self.capped]}

    @staticmethod
    def from_dict(d):
        nodes = [BlockNode(n["kind"], (n["cell"][0], n["cell"][1]), n["orientation"], tuple(n["sockets"]))
                 for n in d["nodes"]]
        return BlockGraph(d["rows"], d["cols"], nodes, [((a[0], a[1]), (b[0], b[1])) for a, b in d["edges"]],
                          [((c[0], c[1]), dd) for c, dd in d["capped"]])


@dataclass
class ZoneMap:
    """types.py:218-229.  ``rle`` carries the device run-length code of ``grid``
    (cw_scene_rle) when the map came from a device batch."""
    resolution: float
    grid: np.ndarray
    params: dict
    rle: list = None

    @property
    def shape(self):
        return self.grid.shape

    def counts(self):
        return {z.name: int(np.count_nonzero(self.grid == int(z))) for z in Zone}


@dataclass
class TerrainTile:
    """types.py:237-259."""
    kind: str
    param: float
    base: float
    shape: dict

    def to_dict(self):
        return {"kind": self.kind, "param": float(self.param), "base": float(self.base), "shape": self.shape}

    @staticmethod
    def from_dict(d):
        return TerrainTile(d["kind"], float(d["param"]), float(d["base"]), d["shape"])


@dataclass
class TerrainGrid:
    """types.py:262-300 (``assignment_rle`` as for ZoneMap.rle)."""
    tile_size: float
    rows: int
    cols: int
    tiles: list
    assignment: np.ndarray
    noise_seed: int
    assignment_rle: list = None

    def kind_at(self, row, col):
        return self.tiles[int(self.assignment[row, col])].kind

    def to_dict(self):
        """types.py:274-285."""
        from .sceneio import rle_encode
        rle = self.assignment_rle if self.assignment_rle is not None else rle_encode(
            np.asarray(self.assignment).astype(np.int64))
        return {"tile_size": float(self.tile_size), "rows": int(self.rows), "cols": int(self.cols),
                "tiles": [t.to_dict() for t in self.tiles], "assignment_rle": rle,
                "noise_seed": int(self.noise_seed)}

    @staticmethod
    def from_dict(d):
        from .sceneio import rle_decode
        a = rle_decode(d["assignment_rle"], dtype=np.int64).reshape(d["rows"], d["cols"]).astype(np.int32)
        return TerrainGrid(float(d["tile_size"]), int(d["rows"]), int(d["cols"]),
                           [TerrainTile.from_dict(t) for t in d["tiles"]], a, int(d["noise_seed"]),
                           assignment_rle=list(d["assignment_rle"]))


@dataclass
class AssetInstance:
    """types.py:328-361."""
    category: str
    x: float
    y: float
    yaw: float
    footprint: tuple
    height: float

    def to_dict(self):
        return {"category": self.category, "x": float(self.x), "y": float(self.y), "yaw": float(self.yaw),
                "footprint": [float(self.footprint[0]), float(self.footprint[1])],
                "height": float(self.height)}

    @staticmethod
    def from_dict(d):
        return AssetInstance(d["category"], float(d["x"]), float(d["y"]), float(d["yaw"]),
                             (float(d["footprint"][0]), float(d["footprint"][1])), float(d["height"]))

    def corners(self):
        """types.py:355-361: world-space corners of the oriented footprint, (4, 2)
        (a host convenience for callers; placement itself runs in k_place)."""
        hw, hl = self.footprint[0] / 2.0, self.footprint[1] / 2.0
        local = np.array([[-hw, -hl], [hw, -hl], [hw, hl], [-hw, hl]])
        c, s = np.cos(self.yaw), np.sin(self.yaw)
        return local @ np.array([[c, -s], [s, c]]).T + np.array([self.x, self.y])


@dataclass
class SceneDescription:
    """types.py:385-394; ``occupancy`` is the device raster of the same scene
    (None for scenes loaded from JSON)."""
    spec: "SceneSpec"
    blocks: BlockGraph
    zones: ZoneMap
    terrain: TerrainGrid
    objects: list
    routes: list
    schema_version: int = SCHEMA_VERSION
    placement_overflow: bool = False
    occupancy: "OccupancyGrid" = None


def scene_params(spec, catalog=None, obj_max=None):
    """Host-side shape derivation shared by every env of a batch (exactly as the
    reference computes it in Python: zones.py:46-49, terrain.py:227-238,
    placement.py:87-97, scene.py:40-79)."""
    catalog = catalog or load_catalog()
    if len(catalog) > _lib.MAX_CAT:
        raise ValueError(f"catalog larger than {_lib.MAX_CAT} entries")
    w, l = spec.extent_m
    res = spec.grid_resolution_m
    p = _lib.SceneParams()
    p.nx = int(np.ceil(w / res))
    p.ny = int(np.ceil(l / res))
    if p.nx < 4 or p.ny < 4:
        from .errors import ExtentTooSmall
        raise ExtentTooSmall(f"extent {spec.extent_m} too small at resolution {res}")
    p.res, p.w, p.l = res, w, l
    task = TaskKind(spec.task_kind)
    p.task = _TASK_CODE[task]
    p.split = 0 if Split(spec.split) == Split.TRAIN else 1
    for i, k in enumerate(TERRAIN_FAMILIES):
        p.mix[i] = float(spec.terrain_mix.get(k, 0.0))
    if min(w, l) >= 2 * BLOCK_SIZE_M and task != TaskKind.TRAVERSE:
        p.layout, p.brows, p.bcols = 1, int(l // BLOCK_SIZE_M), int(w // BLOCK_SIZE_M)
        if p.brows * p.bcols > 64 or p.nx > 1024:
            raise NotImplementedError("block layouts above 64 blocks / 1024 columns")
    elif task == TaskKind.TRAVERSE:
        p.layout = 2
    else:
        p.layout = 0
    probs = np.array([0.4, 0.3, 0.3], dtype=float)
    probs /= probs.sum()
    cdf = probs.cumsum()
    cdf /= cdf[-1]
    for i in range(3):
        p.quad_cdf[i] = float(cdf[i])
    p.trows = max(1, int(np.ceil(p.ny * res / TILE_SIZE_M)))
    p.tcols = max(1, int(np.ceil(p.nx * res / TILE_SIZE_M)))
    if p.trows * p.tcols > 10000:
        raise NotImplementedError("terrain lattices above 100x100 tiles (one WFC warp's shared memory)")
    p.cpt = int(round(TILE_SIZE_M / res))
    p.nonflat_split_col = int(p.nx * 0.5) if task == TaskKind.TRAVERSE else -1
    p.n_cat = len(catalog)
    for i, e in enumerate(catalog):
        p.cat_w[i], p.cat_l[i] = e.footprint
        p.cat_reach[i] = float(np.hypot(*e.footprint)) / 2.0
        p.cat_zones[i] = sum(1 << int(z) for z in e.allowed_zones)
    order = sorted(range(len(catalog)), key=lambda i: catalog[i].footprint[0] * catalog[i].footprint[1])
    for i, k in enumerate(order):
        p.small_first[i] = k
    area = p.ny * p.nx * res * res
    base = 0 if task == TaskKind.NAV_CLEAR else int(np.floor(4.0 * area / 100.0 + 0.5))
    density = spec.object_density * (4.0 / 6.0 if task == TaskKind.TRAVERSE else 1.0)
    p.obj_count = int(np.floor(density * base + 0.5))
    p.obj_max = max(1, p.obj_count if obj_max is None else obj_max)
    p.attempts = ATTEMPTS_PER_OBJECT
    p.region = {TaskKind.NAV_STATIC: 1, TaskKind.NAV_DYNAMIC: 1, TaskKind.TRAVERSE: 2}.get(task, 0)
    p.peds = int(spec.pedestrian_count)
    p.spawn_region = 1 if task == TaskKind.TRAVERSE else 0
    return p


class SceneBatch:
    """Device-resident outputs of one sampling batch (E rows)."""

    def __init__(self, params, E, device="cuda"):
        import torch
        self.params = params
        self.E = E
        self.device = torch.device(device)
        p = params
        N = p.nx * p.ny
        T = _lib.MAX_TILES
        d = dict(device=self.device)
        z = torch.zeros
        self.zones = z((E, p.ny, p.nx), dtype=torch.uint8, **d)
        self.labels = z((E, p.ny, p.nx), dtype=torch.uint8, **d)
        self.elev = z((E, p.ny, p.nx), dtype=torch.float32, **d)
        self.assign = z((E, p.trows, p.tcols), dtype=torch.int32, **d)
        self.n_tiles = z((E,), dtype=torch.int32, **d)
        self.tile_code = z((E, T), dtype=torch.int8, **d)
        self.tile_kind = z((E, T), dtype=torch.int8, **d)
        self.tile_param = z((E, T), dtype=torch.float64, **d)
        self.tile_p = z((E, T, 4), dtype=torch.float64, **d)
        self.tile_w = z((E, T), dtype=torch.float64, **d)
        self.allowed = z((E, 4, T), dtype=torch.int64, **d)
        self.noise_seed = z((E,), dtype=torch.int64, **d)
        self.wfc_attempts = z((E,), dtype=torch.int32, **d)
        self.obj_cat = z((E, p.obj_max), dtype=torch.int32, **d)
        self.obj_pose = z((E, p.obj_max, 3), dtype=torch.float64, **d)
        self.obj_n = z((E,), dtype=torch.int32, **d)
        self.overflow = z((E,), dtype=torch.uint8, **d)
        self.nearest = z((E, p.ny, p.nx), dtype=torch.int32, **d)
        self.has_obs = z((E,), dtype=torch.uint8, **d)
        self.walk = z((E, N), dtype=torch.int32, **d)
        self.walk_n = z((E,), dtype=torch.int32, **d)
        self.reach = z((E, N), dtype=torch.int32, **d)
        self.moves = z((E, N), dtype=torch.uint8, **d)
        A = max(p.peds, 1)
        self.sp_pos = z((E, A, 2), dtype=torch.float64, **d)
        self.sp_goal = z((E, A, 2), dtype=torch.float64, **d)
        self.sp_kind = z((E, A), dtype=torch.int8, **d)
        self.sp_pref = z((E, A), dtype=torch.float64, **d)
        self.status = z((E,), dtype=torch.int32, **d)
        self.routes = z((E, 8, 2, 2), dtype=torch.float64, **d)   # scene.routes (scene.py:87)
        self.n_routes = z((E,), dtype=torch.int32, **d)
        self.scene_seed = z((E,), dtype=torch.int64, **d)
        self.zone_params = z((E, _lib.ZONE_PARAMS), dtype=torch.float64, **d)   # ZoneMap.params
        self.block_var = z((E, _lib.MAX_BLOCKS), dtype=torch.uint8, **d)        # connect_blocks
        self.region = None   # optional (E, N) u8 route region mask (spawn_agents(region_mask=))
        self.epoch = z((E,), dtype=torch.int32, **d)   # grid generation (+1 per row sampled)
        self._scratch_rows = 0
        self._ensure_scratch(min(E, SceneSampler.max_rows))

    def _ensure_scratch(self, rows):
        import torch
        if rows <= self._scratch_rows:
            return
        p = self.params
        N = p.nx * p.ny
        self.scratch_i32 = torch.empty((rows, 10 * N), dtype=torch.int32, device=self.device)
        self.scratch_f64 = torch.empty((rows, max(p.obj_max * 8, N)), dtype=torch.float64,
                                       device=self.device)
        nbytes = _lib.lib().cw_scene_seed_scratch_bytes(rows)
        self.seed_scratch = torch.empty((nbytes,), dtype=torch.uint8, device=self.device)
        self._scratch_rows = rows

    def buffers(self):
        b = _lib.SceneBuffers()
        for name in _lib.SCENE_BUFFER_FIELDS:
            t = getattr(self, name)
            setattr(b, name, None if t is None else t.data_ptr())
        return b

    def check_status(self, rows=None):
        st = self.status.cpu().numpy() if rows is None else self.status[rows].cpu().numpy()
        bad = np.flatnonzero(st)
        if bad.size:
            code = int(st[bad[0]])
            raise STATUS_ERRORS.get(code, RuntimeError)(
                f"scene sampling failed for {bad.size} env(s); first row {int(bad[0])} code {code}")

    # -- host views (reference-shaped) ---------------------------------------------
    def occupancy(self, i):
        return OccupancyGrid(resolution=float(self.params.res), labels=self.labels[i].cpu().numpy(),
                             elevation=self.elev[i].cpu().numpy())

    def objects(self, i, catalog=None):
        catalog = catalog or load_catalog()
        n = int(self.obj_n[i])
        cats = self.obj_cat[i, :n].cpu().numpy()
        pose = self.obj_pose[i, :n].cpu().numpy()
        return [AssetInstance(catalog[int(k)].category, float(x), float(y), float(yaw),
                              catalog[int(k)].footprint, catalog[int(k)].height)
                for k, (x, y, yaw) in zip(cats, pose)]

    def scene(self, i, spec, catalog=None):
        """SceneDescription of row i (types.py:385-394) with its device raster;
        ``spec`` is the batch spec (the row's seed is its scene seed)."""
        from .sceneio import batch_scene_dicts, scene_from_dict
        sc = scene_from_dict(batch_scene_dicts(self, spec, [i], catalog)[0])
        sc.occupancy = self.occupancy(i)
        return sc


class SceneSampler:
    """Samples batches of scenes that share a SceneSpec shape (async scheme:
    every env has its own seed, batch.py:84-96)."""

    def __init__(self, spec, capacity, catalog=None, device="cuda", routes=True):
        self.spec = spec
        self.routes = routes   # also sample scene.routes (scene.py:87, cw_route_anchors)
        self.catalog = catalog or load_catalog()
        self.params = scene_params(spec, self.catalog)
        self.batch = SceneBatch(self.params, capacity, device)

    max_rows = 2048   # envs per cw_sample_scenes call (bounds the scratch footprint)
    route_chunk = int(os.environ.get("CW_ROUTE_CHUNK", 296))  # envs in flight in the route-anchor kernel (CTAs, 2 per SM; 184 B/cell/env scratch)

    def sample(self, scene_seeds, crowd_seeds=None, slots=None, stream=None, check=True):
        """Sample len(scene_seeds) scenes into rows ``slots`` (default 0..E-1).

        scene_seeds / crowd_seeds / slots: device int64 tensors (or sequences)."""
        import torch
        dev = self.batch.device
        seeds = _as_u64_tensor(scene_seeds, dev)
        E = seeds.numel()
        if E == 0:
            return self.batch
        if E > self.max_rows:
            if crowd_seeds is None and self.params.peds > 0:
                from .rng import child_seeds_device
                crowd_seeds = child_seeds_device(seeds, "crowd", 0)
            cs = None if crowd_seeds is None else _as_u64_tensor(crowd_seeds, dev)
            sl = (torch.arange(E, device=dev) if slots is None
                  else torch.as_tensor(slots, dtype=torch.int64, device=dev))
            for k in range(0, E, self.max_rows):
                part = slice(k, min(E, k + self.max_rows))
                self.sample(seeds[part], None if cs is None else cs[part], sl[part], stream, check=False)
            if check:
                self.batch.check_status(sl)
            return self.batch
        if crowd_seeds is None and self.params.peds > 0:
            # first spawn of an env whose env seed is its scene seed (batch.py:179)
            from .rng import child_seeds_device
            crowd_seeds = child_seeds_device(seeds, "crowd", 0)
        cseeds = None if crowd_seeds is None else _as_u64_tensor(crowd_seeds, dev)
        sl = None
        if slots is not None:
            sl = torch.as_tensor(slots, dtype=torch.int32, device=dev).contiguous()
            self.batch.status.index_fill_(0, sl.long(), 0)
            self.batch.scene_seed.index_copy_(0, sl.long(), seeds)
        else:
            if E > self.batch.E:
                raise ValueError("more seeds than batch capacity")
            self.batch.status[:E].zero_()
            self.batch.scene_seed[:E] = seeds
        self.batch._ensure_scratch(E)
        b = self.batch.buffers()
        if self.routes:
            # route anchors (scene.py:87, 102-178) forked off the labels inside the
            # pipeline (cw_sample_scenes_routes), chunked through their own scratch
            p = self.params
            chunk = min(E, self.route_chunk)
            nbytes = int(_lib.lib().cw_route_scratch_bytes(p.nx, p.ny, chunk))
            if getattr(self.batch, "route_scratch", None) is None or self.batch.route_scratch.numel() * 8 < nbytes:
                self.batch.route_scratch = torch.empty(nbytes // 8 + 1, dtype=torch.int64, device=dev)
            err = _lib.lib().cw_sample_scenes_routes(
                self.params, E, _lib.ptr(seeds), _lib.ptr(cseeds), _lib.ptr(sl),
                _lib.ptr(self.batch.seed_scratch), b, _lib.ptr(self.batch.routes), _lib.ptr(self.batch.n_routes),
                _lib.ptr(self.batch.route_scratch), chunk, _lib.stream_ptr(stream))
            _lib.check(err, "cw_sample_scenes_routes")
        else:
            err = _lib.lib().cw_sample_scenes(
                self.params, E, _lib.ptr(seeds), _lib.ptr(cseeds), _lib.ptr(sl),
                _lib.ptr(self.batch.seed_scratch), b, _lib.stream_ptr(stream))
            _lib.check(err, "cw_sample_scenes")
        if check:
            self.batch.check_status(None if sl is None else sl.long())
        return self.batch


    def scene_dicts(self, rows=None):
        """scene_to_dict (scene.py:163-178) of sampled rows (device run-length code)."""
        from .sceneio import batch_scene_dicts
        return batch_scene_dicts(self.batch, self.spec, rows, self.catalog)

    def scene_hashes(self, rows=None):
        """scene_hash (scene.py:229-230) of sampled rows."""
        from .sceneio import batch_scene_hashes
        return batch_scene_hashes(self.batch, self.spec, rows, self.catalog)


def _as_u64_tensor(seeds, device):
    import torch
    if isinstance(seeds, torch.Tensor):
        return seeds.to(device=device, dtype=torch.int64).contiguous()
    arr = np.array([int(s) & ((1 << 64) - 1) for s in seeds], dtype=np.uint64).view(np.int64)
    return torch.from_numpy(arr).to(device)


def as_spec(spec):
    """A SceneSpec from any spec object with the reference's ``to_dict`` (e.g. the
    reference's own SceneSpec passed to the drop-in)."""
    return spec if isinstance(spec, SceneSpec) else SceneSpec.from_dict(spec.to_dict())


def generate_scene(spec, catalog=None, device="cuda"):
    """scene.py:38 generate_scene on the device (including the route anchors).
    The returned scene already carries its occupancy raster."""
    spec = as_spec(spec)
    s = SceneSampler(spec, 1, catalog, device)
    b = s.sample([spec.seed])
    return b.scene(0, spec, s.catalog)


def rasterize_occupancy(scene, resolution=None):
    """occupancy.py:28-57.  At the spec resolution a sampled scene already carries
    its device raster; any other resolution (or a scene without one, e.g. loaded
    from JSON) is rasterised on the device by ``cw_rasterize`` from the scene's zone
    grid, terrain tiles and objects."""
    import torch
    if resolution is None:
        resolution = scene.spec.grid_resolution_m
    if resolution <= 0:
        raise ValueError("resolution must be > 0")
    if resolution == scene.spec.grid_resolution_m and getattr(scene, "occupancy", None) is not None:
        return scene.occupancy
    from .sceneio import _T_CORNER, _T_ROUGH, _T_STAIR_U, _T_STAIR_V
    w, l = scene.spec.extent_m
    nx, ny = int(np.ceil(w / resolution)), int(np.ceil(l / resolution))
    zg = np.ascontiguousarray(np.asarray(scene.zones.grid, dtype=np.uint8))
    zy, zx = zg.shape
    terr = scene.terrain
    tiles = list(terr.tiles)
    if len(tiles) > _lib.MAX_TILES:
        raise ValueError(f"more than {_lib.MAX_TILES} terrain tiles")
    code = np.zeros(_lib.MAX_TILES, dtype=np.int8)
    tp = np.zeros((_lib.MAX_TILES, 4), dtype=np.float64)
    for i, t in enumerate(tiles):
        sh = t.shape
        if sh["type"] == "corner":
            code[i], tp[i] = _T_CORNER, sh["h"]
        elif sh["type"] == "stair":
            code[i] = _T_STAIR_U if sh["axis"] == "u" else _T_STAIR_V
            tp[i, :2] = sh["a"], sh["b"]
        else:
            code[i] = _T_ROUGH
            tp[i, :2] = sh["base"], sh["amp"]
    objs = list(scene.objects)
    foot = sorted({(float(o.footprint[0]), float(o.footprint[1])) for o in objs})
    if len(foot) > _lib.MAX_CAT:
        raise ValueError(f"more than {_lib.MAX_CAT} distinct object footprints")
    p = _lib.SceneParams()
    p.nx, p.ny, p.res = nx, ny, float(resolution)
    p.trows, p.tcols = int(terr.rows), int(terr.cols)
    p.n_cat = len(foot)
    for k, (fw, fl) in enumerate(foot):
        p.cat_w[k], p.cat_l[k] = fw, fl
    p.obj_max = max(1, len(objs))
    b = SceneBatch(p, 1)
    dev = b.device
    b.zones = torch.from_numpy(zg.reshape(1, zy * zx)).to(dev)
    b.assign[0] = torch.from_numpy(np.asarray(terr.assignment, dtype=np.int32)).to(dev)
    b.tile_code[0] = torch.from_numpy(code).to(dev)
    b.tile_p[0] = torch.from_numpy(tp).to(dev)
    b.noise_seed[0] = int(np.uint64(int(terr.noise_seed) & ((1 << 64) - 1)).view(np.int64))
    if objs:
        b.obj_cat[0, :len(objs)] = torch.tensor([foot.index((float(o.footprint[0]), float(o.footprint[1])))
                                                 for o in objs], dtype=torch.int32, device=dev)
        b.obj_pose[0, :len(objs)] = torch.tensor([[o.x, o.y, o.yaw] for o in objs], dtype=torch.float64,
                                                 device=dev)
    b.obj_n[0] = len(objs)
    _lib.check(_lib.lib().cw_rasterize(p, 1, None, zx, zy, float(scene.zones.resolution), b.buffers(),
                                       _lib.stream_ptr()), "cw_rasterize")
    return OccupancyGrid(resolution=float(resolution), labels=b.labels[0].cpu().numpy(),
                         elevation=b.elev[0].cpu().numpy())
