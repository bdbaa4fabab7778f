"""Scene-sampling oracle: zones, terrain tiles + WFC, heightfield, placement,
occupancy raster (test infrastructure only -- see oracle/__init__.py).

Each function restates one reference routine; the citation is in its
docstring (paths relative to /root/reference/pkg/src/citywalk).  Outputs are
plain numpy arrays / tuples so tests can compare them with the device path
bit-for-bit.  Route anchors (scene.py:102-158) are out of scope.
"""

import math
from fractions import Fraction

import numpy as np

from .rng import child_seed, make_rng, pairwise_sum

# Zone / label codes (urbangen/types.py:33-79)
SIDEWALK, CROSSWALK, PLAZA, BUILDING, VEGETATION, ROADWAY = range(6)
OBSTACLE, ROADWAY_L, WALKABLE, NONWALK = range(4)
ZONE_TO_LABEL = np.array([WALKABLE, WALKABLE, WALKABLE, OBSTACLE, NONWALK, ROADWAY_L], np.uint8)
WALKABLE_ZONES = (SIDEWALK, CROSSWALK, PLAZA)
TASKS = ("NavClear", "NavStatic", "NavDynamic", "Traverse")
FAMILIES = ("Flat", "Slope", "Stair", "Rough")
BLOCK_M = 20.0
TILE_M = 2.0
TWO_PI = 2 * np.pi


def fma(a, b, c):
    """Exactly rounded a*b+c (the OpenBLAS kernels the reference hits use FMA)."""
    return float(Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c)))


# -- raster helpers (gridmath.py:42-69) ---------------------------------------

def rect_bounds(shape, x0, y0, x1, y1, res):
    """Cell-centre rectangle [x0,x1)x[y0,y1) -> (r0, r1, c0, c1); gridmath.py:59-69."""
    ny, nx = shape
    c0 = max(0, int(np.ceil(x0 / res - 0.5)))
    c1 = min(nx, int(np.ceil(x1 / res - 0.5)))
    r0 = max(0, int(np.ceil(y0 / res - 0.5)))
    r1 = min(ny, int(np.ceil(y1 / res - 0.5)))
    return r0, r1, c0, c1


def rect_mask(shape, x0, y0, x1, y1, res):
    r0, r1, c0, c1 = rect_bounds(shape, x0, y0, x1, y1, res)
    m = np.zeros(shape, bool)
    if c1 > c0 and r1 > r0:
        m[r0:r1, c0:c1] = True
    return m


def chamfer(mask, res):
    """Two-pass (1, sqrt2) chamfer distance; gridmath.py:8-39."""
    ny, nx = mask.shape
    big = 1e9
    s2 = float(np.sqrt(2.0))
    d = np.where(mask, 0.0, big)
    ar = np.arange(nx)

    def relax(row):
        lft = np.minimum.accumulate(row - ar) + ar
        rgt = (np.minimum.accumulate((row + ar)[::-1]) - ar[::-1])[::-1]
        return np.minimum(lft, rgt)

    def pull(dst, src):
        dg = np.full(nx, big)
        dg[1:] = src[:-1] + s2
        dg[:-1] = np.minimum(dg[:-1], src[1:] + s2)
        return np.minimum(dst, np.minimum(src + 1.0, dg))

    for r in range(ny):
        if r:
            d[r] = pull(d[r], d[r - 1])
        d[r] = relax(d[r])
    for r in range(ny - 2, -1, -1):
        d[r] = pull(d[r], d[r + 1])
        d[r] = relax(d[r])
    return d * res


# -- block graph (urbangen/blocks.py:34-113) -----------------------------------

_BASE_SOCKETS = [(1, 0, 1, 0), (1, 1, 0, 0), (1, 1, 1, 1), (1, 1, 0, 1),
                 (1, 1, 0, 1), (1, 1, 1, 1), (1, 1, 0, 1)]  # types.py:148-156 (N,E,S,W)
VARIANTS = [tuple(b[(i - o) % 4] for i in range(4)) for b in _BASE_SOCKETS for o in range(4)]
VARIANT_KIND = [k for k in range(7) for _ in range(4)]


def connect_blocks(seed, rows, cols):
    """Row-major socket sampling with <=16 restarts, comb fallback; blocks.py:34-46.

    Returns a list of (kind, orientation, sockets) per block, row-major."""
    for attempt in range(16):
        rng = make_rng(seed, "blocks", attempt)
        nodes = []
        for r in range(rows):
            for c in range(cols):
                need_n = nodes[(r - 1) * cols + c][2][2] if r else None
                need_w = nodes[r * cols + c - 1][2][1] if c else None
                opts = [v for v in range(28)
                        if (need_n is None or VARIANTS[v][0] == need_n)
                        and (need_w is None or VARIANTS[v][3] == need_w)]
                v = opts[int(rng.integers(len(opts)))]
                nodes.append((VARIANT_KIND[v], v % 4, VARIANTS[v]))
        if _blocks_connected(nodes, rows, cols):
            return nodes
    comb = []
    for r in range(rows):
        for c in range(cols):
            k = 5 if (r == 0 and cols > 1) else 0
            comb.append((k, 0, VARIANTS[k * 4]))
    return comb


def _blocks_connected(nodes, rows, cols):
    """blocks.py:103-118 -- matched E/S sockets link every block."""
    if rows * cols == 1:
        return True
    adj = [[] for _ in range(rows * cols)]
    for r in range(rows):
        for c in range(cols):
            s = nodes[r * cols + c][2]
            if s[1] and c + 1 < cols:
                adj[r * cols + c].append(r * cols + c + 1)
                adj[r * cols + c + 1].append(r * cols + c)
            if s[2] and r + 1 < rows:
                adj[r * cols + c].append((r + 1) * cols + c)
                adj[(r + 1) * cols + c].append(r * cols + c)
    seen = {0}
    stack = [0]
    while stack:
        for nb in adj[stack.pop()]:
            if nb not in seen:
                seen.add(nb)
                stack.append(nb)
    return len(seen) == rows * cols


# -- ground planning (urbangen/zones.py:44-190) ----------------------------------

def plan_ground(seed, extent, res, task, blocks=None, block_dims=(0, 0)):
    """Zone grid (ny, nx) uint8; zones.py:44-68."""
    w, l = extent
    nx = int(np.ceil(w / res))
    ny = int(np.ceil(l / res))
    rng = make_rng(seed, "zones")
    grid = np.full((ny, nx), VEGETATION, np.uint8)
    if blocks and min(w, l) >= BLOCK_M:
        _block_layout(grid, blocks, block_dims, rng, w, l, res)
    elif task == "Traverse":
        b = min(1.0, 0.2 * min(w, l))
        r0, r1, c0, c1 = rect_bounds(grid.shape, b, b, w - b, l - b, res)
        if r1 > r0 and c1 > c0:
            grid[r0:r1, c0:c1] = PLAZA
    else:
        _courtyard(grid, rng, w, l, res)
    if not np.isin(grid, WALKABLE_ZONES).any():
        raise ValueError("ExtentTooSmall: no walkable zone")
    return grid


def _courtyard(grid, rng, w, l, res):
    """zones.py:79-129."""
    sh = grid.shape
    fx = float(rng.uniform(0.30, 0.42))
    fy = float(rng.uniform(0.30, 0.42))
    cx, cy = w / 2.0, l / 2.0
    walk = rect_mask(sh, cx - fx * w, cy - fy * l, cx + fx * w, cy + fy * l, res)
    for _ in range(int(rng.integers(2, 5))):
        ex = float(rng.uniform(cx - fx * w, cx + fx * w))
        ey = float(rng.uniform(cy - fy * l, cy + fy * l))
        hw = float(rng.uniform(0.10, 0.25)) * w
        hl = float(rng.uniform(0.10, 0.25)) * l
        walk |= rect_mask(sh, ex - hw, ey - hl, ex + hw, ey + hl, res)
    grid[walk] = PLAZA
    if rng.random() < 0.5:
        tw = float(rng.uniform(1.2, 2.2))
        if rng.random() < 0.5:
            tx = float(rng.uniform(cx - 0.2 * w, cx + 0.2 * w))
            band = rect_mask(sh, tx - tw / 2, 0, tx + tw / 2, l, res)
        else:
            ty = float(rng.uniform(cy - 0.2 * l, cy + 0.2 * l))
            band = rect_mask(sh, 0, ty - tw / 2, w, ty + tw / 2, res)
        grid[band & walk] = SIDEWALK
    n_build = int(rng.integers(0, 3))
    corners = [(0.0, 0.0), (w, 0.0), (0.0, l), (w, l)]
    placed = 0
    for idx in rng.permutation(4):
        if placed >= n_build:
            break
        kx, ky = corners[int(idx)]
        bw = float(rng.uniform(0.12, 0.22)) * w
        bl = float(rng.uniform(0.12, 0.22)) * l
        x0 = 0.0 if kx == 0.0 else w - bw
        y0 = 0.0 if ky == 0.0 else l - bl
        m = rect_mask(sh, x0, y0, x0 + bw, y0 + bl, res)
        if not (m & walk).any():
            grid[m] = BUILDING
            placed += 1


def _block_layout(grid, nodes, dims, rng, w, l, res):
    """zones.py:132-190 plus crosswalk painting zones.py:193-234."""
    rows, cols = dims
    sh = grid.shape
    ox = (w - cols * BLOCK_M) / 2.0
    oy = (l - rows * BLOCK_M) / 2.0
    rw = 6.0
    sw = float(rng.uniform(1.5, 3.0))
    road = np.zeros(sh, bool)
    for i, (_, _, s) in enumerate(nodes):
        r, c = divmod(i, cols)
        x0, y0 = ox + c * BLOCK_M, oy + r * BLOCK_M
        cx, cy = x0 + BLOCK_M / 2.0, y0 + BLOCK_M / 2.0
        if s[0]:
            road |= rect_mask(sh, cx - rw / 2, y0, cx + rw / 2, cy, res)
        if s[2]:
            road |= rect_mask(sh, cx - rw / 2, cy, cx + rw / 2, y0 + BLOCK_M, res)
        if s[3]:
            road |= rect_mask(sh, x0, cy - rw / 2, cx, cy + rw / 2, res)
        if s[1]:
            road |= rect_mask(sh, cx, cy - rw / 2, x0 + BLOCK_M, cy + rw / 2, res)
    dist = chamfer(road, res)
    side = (dist > 0) & (dist <= sw)
    grid[side] = SIDEWALK
    grid[road] = ROADWAY
    probs = np.array([0.4, 0.3, 0.3])
    probs /= probs.sum()
    pick_zone = (BUILDING, VEGETATION, PLAZA)
    free = ~(road | side)
    for i in range(len(nodes)):
        r, c = divmod(i, cols)
        x0, y0 = ox + c * BLOCK_M, oy + r * BLOCK_M
        for qx in (0, 1):
            for qy in (0, 1):
                z = pick_zone[int(rng.choice(3, p=probs))]
                m = rect_mask(sh, x0 + qx * BLOCK_M / 2 + 1.0, y0 + qy * BLOCK_M / 2 + 1.0,
                              x0 + (qx + 1) * BLOCK_M / 2 - 1.0, y0 + (qy + 1) * BLOCK_M / 2 - 1.0,
                              res)
                grid[m & free] = z
    ny, nx = sh
    cw = 1.2
    for i, (_, _, s) in enumerate(nodes):
        if sum(s) < 3:
            continue
        r, c = divmod(i, cols)
        x0, y0 = ox + c * BLOCK_M, oy + r * BLOCK_M
        cx, cy = x0 + BLOCK_M / 2.0, y0 + BLOCK_M / 2.0
        spans = []
        if s[0]:
            spans.append((cx - rw / 2, y0 + 1.0, cx + rw / 2, y0 + 1.0 + cw, 0))
        if s[2]:
            spans.append((cx - rw / 2, y0 + BLOCK_M - 1.0 - cw, cx + rw / 2, y0 + BLOCK_M - 1.0, 0))
        if s[3]:
            spans.append((x0 + 1.0, cy - rw / 2, x0 + 1.0 + cw, cy + rw / 2, 1))
        if s[1]:
            spans.append((x0 + BLOCK_M - 1.0 - cw, cy - rw / 2, x0 + BLOCK_M - 1.0, cy + rw / 2, 1))
        for (a0, b0, a1, b1, ax) in spans:
            m = rect_mask(sh, a0, b0, a1, b1, res) & (grid == ROADWAY)
            rr, cc = np.nonzero(m)
            if ax == 0:
                sel = (rr % 2 == 1) & (rr > 0) & (rr < ny - 1)
            else:
                sel = (cc % 2 == 1) & (cc > 0) & (cc < nx - 1)
            grid[rr[sel], cc[sel]] = CROSSWALK


# -- terrain tiles (urbangen/terrain.py:30-212) -----------------------------------

_RANGES = {("Stair", "Train"): (0.05, 0.23), ("Stair", "Test"): (0.10, 0.30),
           ("Slope", "Train"): (0.00, 0.40), ("Slope", "Test"): (0.05, 0.80),
           ("Rough", "Train"): (0.02, 0.10), ("Rough", "Test"): (0.05, 0.20)}
# tile type codes for the elevation table (terrain.py:441-452)
T_CORNER, T_STAIR_U, T_STAIR_V, T_ROUGH = 0, 1, 2, 3
# kind codes (types.py:42-48 order)
K_FLAT, K_SUP, K_SDOWN, K_STUP, K_STDOWN, K_ROUGH = range(6)
FAMILY_OF = {K_FLAT: "Flat", K_SUP: "Slope", K_SDOWN: "Slope", K_STUP: "Stair",
             K_STDOWN: "Stair", K_ROUGH: "Rough"}


def build_tiles(mix, split, seed):
    """Tile palette, adjacency, weights; terrain.py:160-212.

    Returns (tiles, allowed(4,n,n) bool, weights(n,)); each tile is
    (kind, param, type_code, (p0, p1, p2, p3))."""
    rng = make_rng(seed, "tileset")
    tiles = [(K_FLAT, 0.0, T_CORNER, (0.0, 0.0, 0.0, 0.0))]
    mix = {k: float(mix.get(k, 0.0)) for k in FAMILIES}

    def corner(h00, h10, h01, h11, grade):
        hs = (h00, h10, h01, h11)
        if len(set(hs)) == 1:
            return (K_FLAT, 0.0, T_CORNER, hs)
        up = (h10 + h11 - h00 - h01) + (h01 + h11 - h00 - h10)
        return (K_SUP if up > 0 else K_SDOWN, grade, T_CORNER, hs)

    if mix["Slope"] > 0:
        lo, hi = _RANGES[("Slope", split)]
        for g in sorted({float(rng.uniform(lo, hi)) for _ in range(2)}):
            h = g * TILE_M
            if h <= 0:
                continue
            for a in (0.0, h):
                for b in (0.0, h):
                    for c in (0.0, h):
                        for d in (0.0, h):
                            if a == b == c == d == 0.0:
                                continue
                            if a == d and b == c and a != b:
                                continue
                            tiles.append(corner(a, b, c, d, g))
    if mix["Stair"] > 0:
        lo, hi = _RANGES[("Stair", split)]
        rise = float(rng.uniform(lo, hi))
        for code in (T_STAIR_U, T_STAIR_V):
            for low_first in (True, False):
                for lev in range(3):
                    hl, hh = lev * rise, (lev + 1) * rise
                    ab = (hl, hh) if low_first else (hh, hl)
                    tiles.append((K_STUP if low_first else K_STDOWN, rise, code, (ab[0], ab[1], 0.0, 0.0)))
        for lev in range(1, 4):
            h = lev * rise
            tiles.append(corner(h, h, h, h, 0.0))
    if mix["Rough"] > 0:
        lo, hi = _RANGES[("Rough", split)]
        for a in sorted({float(rng.uniform(lo, hi)) for _ in range(2)}):
            tiles.append((K_ROUGH, a, T_ROUGH, (0.0, a, 0.0, 0.0)))

    n = len(tiles)
    allowed = np.zeros((4, n, n), bool)
    for i in range(n):
        for j in range(n):
            allowed[1, i, j] = _compatible(tiles[i], tiles[j], 1)
            allowed[2, i, j] = _compatible(tiles[i], tiles[j], 2)
    allowed[3] = allowed[1].T
    allowed[0] = allowed[2].T
    fam_n = {}
    for t in tiles:
        fam_n[FAMILY_OF[t[0]]] = fam_n.get(FAMILY_OF[t[0]], 0) + 1
    weights = np.array([mix[FAMILY_OF[t[0]]] / fam_n[FAMILY_OF[t[0]]] for t in tiles])
    return tiles, allowed, weights


def _edge_profile(tile, d):
    """(is_step, a, b) of edge d (0=N,1=E,2=S,3=W); terrain.py:248-276."""
    _, _, code, p = tile
    if code == T_CORNER:
        h00, h10, h01, h11 = p
        return {0: (False, h00, h10), 2: (False, h01, h11),
                3: (False, h00, h01), 1: (False, h10, h11)}[d]
    if code == T_STAIR_U:
        a, b = p[0], p[1]
        return {0: (True, a, b), 2: (True, a, b), 3: (False, a, a), 1: (False, b, b)}[d]
    if code == T_STAIR_V:
        a, b = p[0], p[1]
        return {0: (False, a, a), 2: (False, b, b), 3: (True, a, b), 1: (True, a, b)}[d]
    return (False, 0.0, 0.0)   # rough tiles sit at base 0


def _prof_eval(pr, t):
    step, a, b = pr
    if not step:
        return a + (b - a) * t
    return a if t < 0.5 else b


def _compatible(t1, t2, d):
    """terrain.py:194-205, 283-292."""
    p1 = _edge_profile(t1, d)
    p2 = _edge_profile(t2, (d + 2) % 4)
    gap = max(abs(_prof_eval(p1, t) - _prof_eval(p2, t)) for t in (0.0, 0.499999, 0.500001, 1.0))
    tol = 1e-9
    if t1[0] in (K_STUP, K_STDOWN):
        tol = max(tol, t1[1])
    if t2[0] in (K_STUP, K_STDOWN):
        tol = max(tol, t2[1])
    return gap <= tol + 1e-12


# -- WFC (urbangen/wfc.py:24-115) --------------------------------------------------

def _arc_consistent(allowed, dom):
    """Greatest arc-consistent sub-domain (the fixpoint wfc._propagate_from
    reaches in any order); False if a domain empties.  wfc.py:89-115."""
    A = [allowed[d].astype(np.uint8) for d in range(4)]
    while True:
        before = dom.copy()
        f = dom.astype(np.uint8)
        sup = [(f @ A[d]) > 0 for d in range(4)]   # tiles allowed in direction d of each cell
        dom[1:, :] &= sup[2][:-1, :]
        dom[:-1, :] &= sup[0][1:, :]
        dom[:, 1:] &= sup[1][:, :-1]
        dom[:, :-1] &= sup[3][:, 1:]
        if not dom.any(axis=2).all():
            return False
        if np.array_equal(before, dom):
            return True


def wfc_collapse(allowed, weights, domains, seed, max_restarts=16):
    """wfc.py:24-81.  Returns (assignment int32 (rows, cols), attempts_used)."""
    rows, cols, n = domains.shape
    for attempt in range(max_restarts):
        rng = make_rng(seed, "wfc", attempt)
        dom = domains.copy()
        ok = _arc_consistent(allowed, dom)
        while ok:
            cnt = dom.sum(axis=2)
            if not (cnt > 1).any():
                return dom.argmax(axis=2).astype(np.int32), attempt
            flat = int(np.where(cnt > 1, cnt, n + 1).argmin())
            r, c = divmod(flat, cols)
            opts = np.flatnonzero(dom[r, c])
            w = weights[opts]
            tot = pairwise_sum(w)
            if tot <= 0:
                w = np.ones(len(opts))
                tot = float(len(opts))
            pick = opts[int(rng.choice(len(opts), p=w / tot))]
            dom[r, c, :] = False
            dom[r, c, pick] = True
            ok = _arc_consistent(allowed, dom)
    raise RuntimeError("ContradictionAfterRetries")


def terrain_domains(zones, res, n_tiles, nonflat_mask=None):
    """Forced-flat tiles outside the walkable area; terrain.py:215-250."""
    ny, nx = zones.shape
    rows = max(1, int(np.ceil(ny * res / TILE_M)))
    cols = max(1, int(np.ceil(nx * res / TILE_M)))
    walk = np.isin(zones, WALKABLE_ZONES)
    if nonflat_mask is not None:
        walk &= nonflat_mask
    cpt = int(round(TILE_M / res))
    dom = np.ones((rows, cols, n_tiles), bool)
    for r in range(rows):
        for c in range(cols):
            blk = walk[r * cpt:(r + 1) * cpt, c * cpt:(c + 1) * cpt]
            if not (blk.size == cpt * cpt and bool(blk.all())):
                dom[r, c, :] = False
                dom[r, c, 0] = True
    return dom


# -- elevation (terrain.py:264-335) -----------------------------------------------

def _hash_noise(ix, iy, seed):
    h = (ix.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)
         ^ iy.astype(np.uint64) * np.uint64(0xC2B2AE3D27D4EB4F)
         ^ np.uint64(seed & 0xFFFFFFFFFFFFFFFF))
    h ^= h >> np.uint64(33)
    h *= np.uint64(0xFF51AFD7ED558CCD)
    h ^= h >> np.uint64(33)
    return (h >> np.uint64(11)).astype(np.float64) / float(1 << 53) * 2.0 - 1.0


def elevation(tiles, assign, noise_seed, x, y):
    """Elevation (float64) at world points; terrain.py:294-335."""
    rows, cols = assign.shape
    tc = np.clip((x / TILE_M).astype(np.int64), 0, cols - 1)
    tr = np.clip((y / TILE_M).astype(np.int64), 0, rows - 1)
    u = np.clip(x / TILE_M - tc, 0.0, 1.0)
    v = np.clip(y / TILE_M - tr, 0.0, 1.0)
    ids = assign[tr, tc]
    code = np.array([t[2] for t in tiles], np.int8)[ids]
    pp = np.array([t[3] for t in tiles], np.float64)[ids]
    e = ((1 - u) * (1 - v) * pp[..., 0] + u * (1 - v) * pp[..., 1]
         + (1 - u) * v * pp[..., 2] + u * v * pp[..., 3])
    e = np.where(code == T_STAIR_U, np.where(u < 0.5, pp[..., 0], pp[..., 1]), e)
    e = np.where(code == T_STAIR_V, np.where(v < 0.5, pp[..., 0], pp[..., 1]), e)
    rough = code == T_ROUGH
    if rough.any():
        taper = (np.clip(np.minimum(u, 1.0 - u) / 0.125, 0.0, 1.0)
                 * np.clip(np.minimum(v, 1.0 - v) / 0.125, 0.0, 1.0))
        gx, gy = x / 0.5, y / 0.5
        ix, iy = np.floor(gx).astype(np.int64), np.floor(gy).astype(np.int64)
        fx, fy = gx - ix, gy - iy
        sx = fx * fx * (3.0 - 2.0 * fx)
        sy = fy * fy * (3.0 - 2.0 * fy)
        n00 = _hash_noise(ix, iy, noise_seed)
        n10 = _hash_noise(ix + 1, iy, noise_seed)
        n01 = _hash_noise(ix, iy + 1, noise_seed)
        n11 = _hash_noise(ix + 1, iy + 1, noise_seed)
        top = n00 + (n10 - n00) * sx
        bot = n01 + (n11 - n01) * sx
        bump = top + (bot - top) * sy
        e = np.where(rough, pp[..., 0] + pp[..., 1] * taper * bump, e)
    return e


# -- placement (urbangen/placement.py:16-132) -----------------------------------------

def corners(fw, fl, x, y, yaw):
    """AssetInstance.corners (types.py:355-361); the 4x2 @ 2x2 product is
    OpenBLAS dgemm = fma(l1, r1, l0*r0) per entry."""
    hw, hl = fw / 2.0, fl / 2.0
    c, s = float(np.cos(yaw)), float(np.sin(yaw))
    out = []
    for lx, ly in ((-hw, -hl), (hw, -hl), (hw, hl), (-hw, hl)):
        out.append((fma(ly, -s, lx * c) + x, fma(ly, c, lx * s) + y))
    return out


def footprint_cells(fw, fl, x, y, yaw, res, shape):
    """placement.py:33-59."""
    ny, nx = shape
    cs = corners(fw, fl, x, y, yaw)
    x0 = min(p[0] for p in cs)
    x1 = max(p[0] for p in cs)
    y0 = min(p[1] for p in cs)
    y1 = max(p[1] for p in cs)
    c0 = max(0, int(x0 / res) - 1)
    c1 = min(nx - 1, int(x1 / res) + 1)
    r0 = max(0, int(y0 / res) - 1)
    r1 = min(ny - 1, int(y1 / res) + 1)
    if c1 < c0 or r1 < r0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    rr, cc = np.meshgrid(np.arange(r0, r1 + 1), np.arange(c0, c1 + 1), indexing="ij")
    px = (cc + 0.5) * res - x
    py = (rr + 0.5) * res - y
    c, s = np.cos(yaw), np.sin(yaw)
    lx = c * px + s * py
    ly = -s * px + c * py
    inside = (np.abs(lx) <= fw / 2.0) & (np.abs(ly) <= fl / 2.0)
    rows, cols = rr[inside].ravel(), cc[inside].ravel()
    if rows.size == 0:
        rc, cc2 = int(y / res), int(x / res)
        if 0 <= rc < ny and 0 <= cc2 < nx:
            return np.array([rc]), np.array([cc2])
    return rows, cols


def overlap(a, b):
    """SAT test, placement.py:62-78; a/b = (fw, fl, x, y, yaw, reach).
    ``corners @ axis`` is OpenBLAS dgemv = fma(c0, a0, c1*a1)."""
    if (a[2] - b[2]) ** 2 + (a[3] - b[3]) ** 2 > (a[5] + b[5]) ** 2:
        return False
    ca = corners(*a[:5])
    cb = corners(*b[:5])
    for rect in (ca, cb):
        for i in range(2):
            ex = rect[(i + 1) % 4][0] - rect[i][0]
            ey = rect[(i + 1) % 4][1] - rect[i][1]
            ax, ay = -ey, ex
            pa = [fma(p[0], ax, p[1] * ay) for p in ca]
            pb = [fma(p[0], ax, p[1] * ay) for p in cb]
            if max(pa) < min(pb) or max(pb) < min(pa):
                return False
    return True


def place_objects(zones, tiles, assign, catalog, density, seed, task, region_mask, res,
                  attempts=100):
    """placement.py:81-132.  catalog = list of (w, l, allowed_zone_tuple).
    Returns (objects [(cat, x, y, yaw)], overflow, requested)."""
    ny, nx = zones.shape
    area = ny * nx * res * res
    base = 0 if task == "NavClear" else int(np.floor(4.0 * area / 100.0 + 0.5))
    count = int(np.floor(density * base + 0.5))
    if count == 0:
        return [], False, 0
    rng = make_rng(seed, "objects")
    order = sorted(range(len(catalog)), key=lambda i: catalog[i][0] * catalog[i][1])
    reach = [float(np.hypot(e[0], e[1])) / 2.0 for e in catalog]
    placed = []
    trows, tcols = assign.shape
    for _ in range(count):
        ok = False
        for att in range(attempts):
            if att < attempts // 2:
                k = int(rng.integers(len(catalog)))
            else:
                k = order[int(rng.integers(min(5, len(catalog))))]
            x = float(rng.uniform(0, nx * res))
            y = float(rng.uniform(0, ny * res))
            yaw = float(rng.uniform(0, TWO_PI))
            fw, fl, zs = catalog[k]
            rows, cols = footprint_cells(fw, fl, x, y, yaw, res, (ny, nx))
            if rows.size == 0:
                continue
            if not np.isin(zones[rows, cols], list(zs)).all():
                continue
            if region_mask is not None and not region_mask[rows, cols].all():
                continue
            if tiles is not None:
                tr = min(trows - 1, int(y / TILE_M))
                tc = min(tcols - 1, int(x / TILE_M))
                if tiles[int(assign[tr, tc])][0] in (K_STUP, K_STDOWN):
                    continue
            me = (fw, fl, x, y, yaw, reach[k])
            if any(overlap(me, (catalog[o[0]][0], catalog[o[0]][1], o[1], o[2], o[3], reach[o[0]]))
                   for o in placed):
                continue
            placed.append((k, x, y, yaw))
            ok = True
            break
        if not ok:
            return placed, True, count
    return placed, False, count


# -- occupancy raster (urbangen/occupancy.py:28-57) -----------------------------------

def rasterize(zones, zone_res, objects, catalog, tiles, assign, noise_seed, extent, res):
    """labels uint8 (ny, nx), elevation float32 (ny, nx)."""
    w, l = extent
    nx = int(np.ceil(w / res))
    ny = int(np.ceil(l / res))
    zy, zx = zones.shape
    rr = np.minimum((np.arange(ny) + 0.5) * res / zone_res, zy - 1).astype(np.int64)
    cc = np.minimum((np.arange(nx) + 0.5) * res / zone_res, zx - 1).astype(np.int64)
    labels = ZONE_TO_LABEL[zones[rr[:, None], cc[None, :]]]
    for (k, x, y, yaw) in objects:
        orow, ocol = footprint_cells(catalog[k][0], catalog[k][1], x, y, yaw, res, (ny, nx))
        labels[orow, ocol] = OBSTACLE
    xs = (np.arange(nx) + 0.5) * res
    ys = (np.arange(ny) + 0.5) * res
    gx, gy = np.meshgrid(xs, ys)
    elev = elevation(tiles, assign, noise_seed, gx, gy).astype(np.float32)
    return labels, elev


# -- the pipeline (urbangen/scene.py:38-88) ------------------------------------------

def load_catalog_tuples(entries):
    """catalog.json entries -> (w, l, allowed zone codes)."""
    names = ("SIDEWALK", "CROSSWALK", "PLAZA", "BUILDING", "VEGETATION", "ROADWAY")
    return [(float(e["footprint"][0]), float(e["footprint"][1]),
             tuple(names.index(z) for z in e["allowed_zones"])) for e in entries]


def generate_scene(spec, catalog):
    """generate_scene minus route anchors.  spec: dict with seed, extent,
    task, split, density, mix, res.  Returns a dict of arrays."""
    seed = spec["seed"]
    w, l = spec["extent"]
    res = spec["res"]
    task = spec["task"]
    nodes, dims = None, (0, 0)
    if min(w, l) >= 2 * BLOCK_M and task != "Traverse":
        dims = (int(l // BLOCK_M), int(w // BLOCK_M))
        nodes = connect_blocks(child_seed(seed, "blocks"), *dims)
    zones = plan_ground(child_seed(seed, "ground"), (w, l), res, task, nodes, dims)
    nonflat = None
    if task == "Traverse":
        nonflat = np.zeros(zones.shape, bool)
        nonflat[:, int(zones.shape[1] * 0.5):] = True
    tseed = child_seed(seed, "terrain-stage")
    tiles, allowed, weights = build_tiles(spec["mix"], spec["split"], tseed)
    dom = terrain_domains(zones, res, len(tiles), nonflat)
    assign, attempts = wfc_collapse(allowed, weights, dom, child_seed(tseed, "terrain"))
    noise_seed = child_seed(tseed, "terrain-noise")
    density = spec["density"]
    region = None
    if task == "Traverse":
        ny, nx = zones.shape
        region = np.zeros(zones.shape, bool)
        for i in (1, 2, 4, 5):
            region[:, int(nx * i / 6):int(nx * (i + 1) / 6)] = True
        density *= 4.0 / 6.0
    elif task in ("NavStatic", "NavDynamic"):
        region = np.isin(zones, (0, 1, 2))
    objects, overflow, requested = place_objects(
        zones, tiles, assign, catalog, density, child_seed(seed, "placement"), task, region, res)
    labels, elev = rasterize(zones, res, objects, catalog, tiles, assign, noise_seed, (w, l), res)
    return {
        "zones": zones, "tiles": tiles, "allowed": allowed, "weights": weights,
        "assign": assign, "wfc_attempts": attempts, "noise_seed": noise_seed,
        "objects": objects, "overflow": overflow, "requested": requested,
        "labels": labels, "elev": elev, "blocks": nodes,
    }
