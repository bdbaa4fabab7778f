"""Scene identity and wire format.

Mirrors the reference's serialization surface:
  * ``canonical_dumps`` / ``canonical_bytes`` / ``content_hash`` /
    ``rle_encode`` / ``rle_decode``                (citywalk/jsonio.py:14-60)
  * ``scene_to_dict`` / ``scene_from_dict`` / ``scene_to_json`` /
    ``scene_from_json`` / ``scene_hash`` / ``save_scene`` / ``load_scene``
                                                   (urbangen/scene.py:163-238)
  * ``export_occupancy`` / ``load_occupancy``      (urbangen/occupancy.py:60-100)
  * ``AssetCache``                                  (envcore/cache.py:15-39)

and adds the batch form the device sampler needs: ``batch_scene_dicts`` /
``batch_scene_hashes`` build the reference's scene dict for many rows of a
``SceneBatch`` at once.  The two grids in the dict (zone map, terrain
assignment) are run-length coded on the device (``cw_scene_rle``), so only the
compact run lists, the tile tables, objects and route anchors cross PCIe; the
canonical JSON and SHA-256 are host work (hashlib), as in the reference.
``rle_encode`` here is the host codec for host arrays (scenes loaded from
JSON); scenes that come from a device batch always carry the device code.
"""

import hashlib
import json
import os
import threading

import numpy as np

from . import _lib

_U64 = (1 << 64) - 1
_T_CORNER, _T_STAIR_U, _T_STAIR_V, _T_ROUGH = 0, 1, 2, 3
PGM_ENCODING = {0: 0, 3: 85, 1: 170, 2: 255}   # occupancy.py:19-24 (CellLabel -> grey level)


# -- jsonio.py ----------------------------------------------------------------------
def _plain(obj):
    """jsonio.py:14-26."""
    if isinstance(obj, np.ndarray):
        return [_plain(v) for v in obj.tolist()]
    if isinstance(obj, np.integer):
        return int(obj)
    if isinstance(obj, np.floating):
        return float(obj)
    if isinstance(obj, dict):
        return {str(k): _plain(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [_plain(v) for v in obj]
    return obj


def canonical_dumps(obj):
    """jsonio.py:29-30: sorted keys, compact separators, no NaN, shortest float repr."""
    return json.dumps(_plain(obj), sort_keys=True, separators=(",", ":"), allow_nan=False)


def canonical_bytes(obj):
    return canonical_dumps(obj).encode("utf-8")


def content_hash(obj):
    """jsonio.py:37-39: SHA-256 hex digest of the canonical serialization."""
    return hashlib.sha256(canonical_bytes(obj)).hexdigest()


def rle_encode(values):
    """jsonio.py:42-54 for a host array: [value, run, value, run, ...]."""
    arr = np.asarray(values).ravel()
    if arr.size == 0:
        return []
    starts = np.concatenate(([0], np.flatnonzero(arr[1:] != arr[:-1]) + 1))
    runs = np.diff(np.concatenate((starts, [arr.size])))
    out = np.empty(2 * starts.size, dtype=np.int64)
    out[0::2] = arr[starts]
    out[1::2] = runs
    return out.tolist()


def rle_decode(pairs, dtype=np.uint8):
    """jsonio.py:57-60."""
    vals = np.asarray(pairs[0::2], dtype=dtype)
    runs = np.asarray(pairs[1::2], dtype=np.int64)
    return np.repeat(vals, runs)


# -- device run-length code ------------------------------------------------------------
def device_rle(batch, rows=None, stream=None):
    """cw_scene_rle over rows of a SceneBatch: list of (zones_rle, assignment_rle)
    Python int lists, one pair per row (one count pass, one fill pass, one copy)."""
    import torch
    dev = batch.device
    if rows is None:
        rows_t = torch.arange(batch.E, dtype=torch.int32, device=dev)
    else:
        rows_t = torch.as_tensor(rows, dtype=torch.int32).to(dev).reshape(-1).contiguous()
    n = int(rows_t.numel())
    if n == 0:
        return []
    L = _lib.lib()
    p, b = batch.params, batch.buffers()
    runs = torch.zeros((n, 2), dtype=torch.int32, device=dev)
    _lib.check(L.cw_scene_rle(p, n, _lib.ptr(rows_t), b, _lib.ptr(runs), None, None,
                              _lib.stream_ptr(stream)), "cw_scene_rle")
    sizes = 2 * runs.cpu().numpy().astype(np.int64).reshape(-1)
    offs = np.zeros_like(sizes)
    offs[1:] = np.cumsum(sizes)[:-1]
    pairs = torch.empty(int(sizes.sum()), dtype=torch.int32, device=dev)
    offs_t = torch.from_numpy(offs).to(dev)
    _lib.check(L.cw_scene_rle(p, n, _lib.ptr(rows_t), b, _lib.ptr(runs), _lib.ptr(offs_t),
                              _lib.ptr(pairs), _lib.stream_ptr(stream)), "cw_scene_rle")
    flat = pairs.cpu().numpy().tolist()
    return [(flat[offs[2 * i]:offs[2 * i] + sizes[2 * i]],
             flat[offs[2 * i + 1]:offs[2 * i + 1] + sizes[2 * i + 1]]) for i in range(n)]


# -- dict pieces from the device tables ------------------------------------------------
def _tile_dict(code, kind, param, p):
    """build_tile_set tile records (terrain.py:78-110) from the device tile table."""
    from .urbangen import TERRAIN_KINDS
    if code == _T_CORNER:
        h = [float(v) for v in p]
        base, shape = min(h), {"type": "corner", "h": h}
    elif code in (_T_STAIR_U, _T_STAIR_V):
        a, b = float(p[0]), float(p[1])
        base, shape = min(a, b), {"type": "stair", "axis": "u" if code == _T_STAIR_U else "v", "a": a, "b": b}
    else:
        base, amp = float(p[0]), float(p[1])
        shape = {"type": "rough", "base": base, "amp": amp}
    return {"kind": TERRAIN_KINDS[kind], "param": float(param), "base": base, "shape": shape}


def _zone_params(layout, zp):
    """ZoneMap.params (zones.py:69-122) from the device's per-env record."""
    if layout == 0:
        return {"layout": "courtyard", "blob_half": [float(zp[0]), float(zp[1])],
                "extra_rects": int(zp[2]), "trail": bool(zp[3]), "buildings": int(zp[4])}
    if layout == 1:
        return {"layout": "blocks", "sidewalk_width": float(zp[0]), "road_width": float(zp[1])}
    return {"layout": "strip", "border_m": float(zp[0])}


def _host_tables(batch, rows_t):
    """One bulk device->host copy of every small per-env table the dict needs."""
    names = ("scene_seed", "zone_params", "block_var", "n_tiles", "tile_code", "tile_kind", "tile_param",
             "tile_p", "noise_seed", "obj_cat", "obj_pose", "obj_n", "overflow", "routes", "n_routes")
    idx = rows_t.long()
    return {k: getattr(batch, k).index_select(0, idx).cpu().numpy() for k in names}


def batch_scene_dicts(batch, spec, rows=None, catalog=None, stream=None):
    """scene_to_dict (scene.py:163-178) for rows of a device SceneBatch sampled
    with ``spec`` (each row's spec seed = its scene seed)."""
    import torch
    from dataclasses import replace

    from .urbangen import BlockGraph, load_catalog
    catalog = catalog or load_catalog()
    dev = batch.device
    rows_t = (torch.arange(batch.E, dtype=torch.int32, device=dev) if rows is None
              else torch.as_tensor(rows, dtype=torch.int32).to(dev).reshape(-1))
    rles = device_rle(batch, rows_t, stream)
    h = _host_tables(batch, rows_t)
    p = batch.params
    base = replace(spec, seed=0).to_dict()
    empty_blocks = BlockGraph(0, 0, [], [], []).to_dict()
    out = []
    for i, (zrle, arle) in enumerate(rles):
        sd = dict(base)
        sd["seed"] = int(h["scene_seed"][i]) & _U64
        blocks = (BlockGraph.from_variants(p.brows, p.bcols, h["block_var"][i]).to_dict()
                  if p.layout == 1 else empty_blocks)
        nt = int(h["n_tiles"][i])
        tiles = [_tile_dict(int(h["tile_code"][i, t]), int(h["tile_kind"][i, t]), h["tile_param"][i, t],
                            h["tile_p"][i, t]) for t in range(nt)]
        n_obj = int(h["obj_n"][i])
        objects = []
        for k in range(n_obj):
            e = catalog[int(h["obj_cat"][i, k])]
            x, y, yaw = (float(v) for v in h["obj_pose"][i, k])
            objects.append({"category": e.category, "x": x, "y": y, "yaw": yaw,
                            "footprint": [float(e.footprint[0]), float(e.footprint[1])],
                            "height": float(e.height)})
        routes = [[[float(v) for v in pt] for pt in h["routes"][i, r]] for r in range(int(h["n_routes"][i]))]
        out.append({
            "schema_version": 1,
            "spec": sd,
            "blocks": blocks,
            "zones": {"resolution": float(spec.grid_resolution_m), "shape": [int(p.ny), int(p.nx)],
                      "rle": zrle, "params": _zone_params(p.layout, h["zone_params"][i])},
            "terrain": {"tile_size": 2.0, "rows": int(p.trows), "cols": int(p.tcols), "tiles": tiles,
                        "assignment_rle": arle, "noise_seed": int(h["noise_seed"][i]) & _U64},
            "objects": objects,
            "routes": routes,
            "placement_overflow": bool(h["overflow"][i]),
        })
    return out


def batch_scene_hashes(batch, spec, rows=None, catalog=None, stream=None):
    """scene_hash (scene.py:229-230) of rows of a device SceneBatch."""
    return [content_hash(d) for d in batch_scene_dicts(batch, spec, rows, catalog, stream)]


# -- single scenes (scene.py:163-238) -----------------------------------------------------
def scene_to_dict(scene):
    """scene.py:163-178."""
    z, t = scene.zones, scene.terrain
    return {
        "schema_version": scene.schema_version,
        "spec": scene.spec.to_dict(),
        "blocks": scene.blocks.to_dict(),
        "zones": {"resolution": float(z.resolution), "shape": [int(s) for s in z.grid.shape],
                  "rle": z.rle if z.rle is not None else rle_encode(z.grid), "params": z.params},
        "terrain": {"tile_size": float(t.tile_size), "rows": int(t.rows), "cols": int(t.cols),
                    "tiles": [x.to_dict() for x in t.tiles],
                    "assignment_rle": (t.assignment_rle if t.assignment_rle is not None
                                       else rle_encode(np.asarray(t.assignment).astype(np.int64))),
                    "noise_seed": int(t.noise_seed)},
        "objects": [o.to_dict() for o in scene.objects],
        "routes": scene.routes,
        "placement_overflow": bool(scene.placement_overflow),
    }


def scene_from_dict(d):
    """scene.py:181-199."""
    from .urbangen import (AssetInstance, BlockGraph, SceneDescription, SceneSpec, TerrainGrid,
                           TerrainTile, ZoneMap)
    zs = d["zones"]["shape"]
    zones = ZoneMap(float(d["zones"]["resolution"]), rle_decode(d["zones"]["rle"]).reshape(zs[0], zs[1]),
                    d["zones"]["params"], rle=list(d["zones"]["rle"]))
    td = d["terrain"]
    assignment = rle_decode(td["assignment_rle"], dtype=np.int64).reshape(td["rows"], td["cols"]).astype(np.int32)
    terrain = TerrainGrid(float(td["tile_size"]), int(td["rows"]), int(td["cols"]),
                          [TerrainTile.from_dict(x) for x in td["tiles"]], assignment, int(td["noise_seed"]),
                          assignment_rle=list(td["assignment_rle"]))
    return SceneDescription(spec=SceneSpec.from_dict(d["spec"]), blocks=BlockGraph.from_dict(d["blocks"]),
                            zones=zones, terrain=terrain,
                            objects=[AssetInstance.from_dict(o) for o in d["objects"]], routes=d["routes"],
                            schema_version=int(d["schema_version"]),
                            placement_overflow=bool(d.get("placement_overflow", False)))


def scene_to_json(scene):
    return canonical_dumps(scene_to_dict(scene))


def scene_from_json(text):
    """scene.py:210-221 (SceneLoadError on a malformed or foreign-schema file)."""
    from .errors import SceneLoadError
    try:
        d = json.loads(text)
        if int(d.get("schema_version", -1)) != 1:
            raise ValueError(f"unsupported schema_version {d.get('schema_version')}")
        return scene_from_dict(d)
    except (KeyError, ValueError, TypeError) as exc:
        raise SceneLoadError(str(exc)) from exc


def scene_hash(scene):
    return content_hash(scene_to_dict(scene))


def save_scene(scene, path):
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(scene_to_json(scene))
        fh.write("\n")


def load_scene(path):
    with open(path, "r", encoding="utf-8") as fh:
        return scene_from_json(fh.read())


# -- occupancy export (occupancy.py:60-100) -----------------------------------------------
def export_occupancy(grid, path_prefix):
    """Write <prefix>.pgm, <prefix>.elev.f32 and the <prefix>.json sidecar."""
    labels = np.asarray(grid.labels)
    ny, nx = labels.shape
    lut = np.zeros(256, dtype=np.uint8)
    for label, pix in PGM_ENCODING.items():
        lut[label] = pix
    pgm_path = path_prefix + ".pgm"
    with open(pgm_path, "wb") as fh:
        fh.write(f"P5\n{nx} {ny}\n255\n".encode("ascii"))
        fh.write(lut[labels].tobytes())
    elev_path = path_prefix + ".elev.f32"
    with open(elev_path, "wb") as fh:
        fh.write(np.asarray(grid.elevation).astype("<f4").tobytes())
    sidecar = {"resolution": grid.resolution, "origin": [0.0, 0.0],
               "elevation_file": os.path.basename(elev_path), "width": nx, "height": ny}
    with open(path_prefix + ".json", "w", encoding="utf-8") as fh:
        fh.write(canonical_dumps(sidecar))
        fh.write("\n")
    return pgm_path


def load_occupancy(path_prefix):
    """occupancy.py:88-107."""
    from .urbangen import OccupancyGrid
    with open(path_prefix + ".json", "r", encoding="utf-8") as fh:
        sidecar = json.load(fh)
    with open(path_prefix + ".pgm", "rb") as fh:
        if fh.readline().strip() != b"P5":
            raise ValueError("not a binary PGM")
        dims = fh.readline().split()
        nx, ny = int(dims[0]), int(dims[1])
        fh.readline()
        pixels = np.frombuffer(fh.read(nx * ny), dtype=np.uint8).reshape(ny, nx)
    labels = np.zeros((ny, nx), dtype=np.uint8)
    for label, pix in PGM_ENCODING.items():
        labels[pixels == pix] = label
    elev_file = os.path.join(os.path.dirname(path_prefix) or ".", sidecar["elevation_file"])
    with open(elev_file, "rb") as fh:
        elevation = np.frombuffer(fh.read(), dtype="<f4").reshape(ny, nx).copy()
    return OccupancyGrid(resolution=float(sidecar["resolution"]), labels=labels, elevation=elevation)


# -- AssetCache (envcore/cache.py:15-39) --------------------------------------------------
class AssetCache:
    """Scenes keyed by content_hash(spec.to_dict()) (cache.py:27-36); misses are
    sampled on the device."""

    def __init__(self, catalog=None, catalog_path=None, device="cuda"):
        from .urbangen import load_catalog
        self._catalog = tuple(catalog if catalog is not None else load_catalog(catalog_path))
        self._scenes = {}
        self._lock = threading.Lock()
        self.device = device

    @property
    def catalog(self):
        return self._catalog

    def scene(self, spec):
        from .urbangen import generate_scene
        key = content_hash(spec.to_dict())
        with self._lock:
            hit = self._scenes.get(key)
        if hit is not None:
            return hit
        scene = generate_scene(spec, catalog=list(self._catalog), device=self.device)
        with self._lock:
            self._scenes.setdefault(key, scene)
            return self._scenes[key]

    def __len__(self):
        return len(self._scenes)
