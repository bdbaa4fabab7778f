// Scene sampling on B200: every env samples its own layout.
//
//   k_seeds      per-env stream derivation          rng.py:15-26 (+ seed tree)
//   k_zones      courtyard / strip ground planning  zones.py:44-129
//   k_zones_blk  block layout (roads, chamfer       zones.py:132-234, blocks.py:34-118,
//                sidewalks, quadrants, crosswalks)  gridmath.py:8-39
//   k_terrain    tile palette + WFC collapse        terrain.py:160-259, wfc.py:24-115
//   k_place      rejection-sampled objects          placement.py:33-132
//   k_raster     labels + heightfield               occupancy.py:28-57, terrain.py:264-335
//   k_footprint  object footprints -> OBSTACLE      occupancy.py:49-51
//   k_nearest    FIFO-exact multi-source BFS        field.py:571-593
//   k_walk       WALKABLE cell compaction           field.py:60-65
//   k_spawn      kinds, routes, speeds              step.py:37-63, routes.py:14-87
//
// One CTA (or warp) owns one env; results do not depend on launch shape.
#include <algorithm>
#include <cstdio>
#include "common.cuh"
#include "rng.cuh"
#include "citywalk_b200.h"

namespace cw {

// Per-env derived stream seeds / states (scratch, filled by k_seeds).
constexpr int SCRATCH_I32_PER_CELL = 10;  // ints of scratch_i32 per grid cell and env

struct EnvSeeds {
  Pcg64Raw zones;      // make_rng(child_seed(s,"ground"), "zones")
  Pcg64Raw tileset;    // make_rng(child_seed(s,"terrain-stage"), "tileset")
  Pcg64Raw objects;    // make_rng(child_seed(s,"placement"), "objects")
  Pcg64Raw spawn;      // make_rng(crowd_seed, "crowd-spawn")
  uint64_t wfc_seed;   // child_seed(tstage, "terrain")
  uint64_t noise;      // child_seed(tstage, "terrain-noise")
  uint64_t blocks;     // child_seed(s, "blocks")
  uint64_t pad;
};

struct Rect { int r0, r1, c0, c1; };

CW_DEV Rect rect_bounds(const cw_scene_params& P, double x0, double y0, double x1, double y1) {
  // gridmath.py:59-69
  Rect R;
  R.c0 = (int)max(0LL, (long long)ceil(div_h(x0, P.res) - 0.5));
  R.c1 = (int)min((long long)P.nx, (long long)ceil(div_h(x1, P.res) - 0.5));
  R.r0 = (int)max(0LL, (long long)ceil(div_h(y0, P.res) - 0.5));
  R.r1 = (int)min((long long)P.ny, (long long)ceil(div_h(y1, P.res) - 0.5));
  return R;
}
CW_DEV bool rect_nonempty(const Rect& a) { return a.c1 > a.c0 && a.r1 > a.r0; }
CW_DEV bool rect_has(const Rect& a, int r, int c) {
  return r >= a.r0 && r < a.r1 && c >= a.c0 && c < a.c1;
}
CW_DEV bool rect_meet(const Rect& a, const Rect& b) {
  return rect_nonempty(a) && rect_nonempty(b) && a.r0 < b.r1 && b.r0 < a.r1 && a.c0 < b.c1 &&
         b.c0 < a.c1;
}

CW_DEV int env_slot(const int32_t* slots, int e) { return slots ? slots[e] : e; }

// ----------------------------------------------------------------- block scans
template <int NT>
CW_DEV int block_excl_scan(int v, int* sh, int& total) {
  // sh: >= NT/32 + 1 ints
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = lane < NT / 32 ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NT / 32) sh[lane] = s;
  }
  __syncthreads();
  int base = wid ? sh[wid - 1] : 0;
  total = sh[NT / 32 - 1];
  __syncthreads();
  return base + x - v;
}

template <int NT>
CW_DEV unsigned long long block_min_u64(unsigned long long v, unsigned long long* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    unsigned long long y = __shfl_xor_sync(0xffffffffu, v, o);
    v = y < v ? y : v;
  }
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  unsigned long long r = sh[0];
  for (int i = 1; i < NT / 32; ++i) r = sh[i] < r ? sh[i] : r;
  __syncthreads();
  return r;
}

// ----------------------------------------------------------------- union-find
// Lock-free union-find over a CTA's grid (ECL-CC style): parents always point to
// smaller indices, so stale reads are still ancestors.  Labels are only ever
// compared for equality (routes.py:62/74 components, A* reachability).
CW_DEV int uf_find(volatile int32_t* par, int x) {
  int cur = par[x];
  if (cur != x) {
    int prev = x, next;
    while (cur > (next = par[cur])) {
      par[prev] = next;
      prev = cur;
      cur = next;
    }
  }
  return cur;
}

// read-only root lookup for the final labelling pass (no compression writes,
// so a finished label is never overwritten by another thread's path halving)
CW_DEV int uf_root(volatile int32_t* par, int x) {
  int next;
  while (x > (next = par[x])) x = next;
  return x;
}

CW_DEV void uf_union(volatile int32_t* par, int a, int b) {
  a = uf_find(par, a);
  b = uf_find(par, b);
  while (a != b) {
    if (a < b) { int t = a; a = b; b = t; }
    int old = atomicCAS((int32_t*)&par[a], a, b);
    if (old == a) return;
    a = uf_find(par, old);
    b = uf_find(par, b);
  }
}

// Connected components of the cells with ok(f) on an nx*ny grid: each row's
// runs become stars first (no atomics), then only runs of adjacent rows are
// united (once per overlap segment), then a read-only root pass labels cells.
// par[f] ends as the smallest cell index of f's component (-1 where !ok).
template <int NT, bool CONN8, typename OkF>
CW_DEV void grid_components(volatile int32_t* par, int nx, int ny, OkF ok) {
  const int N = nx * ny;
  for (int r = threadIdx.x; r < ny; r += NT) {
    int start = -1;
    for (int c = 0; c < nx; ++c) {
      int f = r * nx + c;
      if (ok(f)) {
        if (start < 0) start = f;
        par[f] = start;
      } else {
        start = -1;
        par[f] = -1;
      }
    }
  }
  __syncthreads();
  for (int f = threadIdx.x; f < N - nx; f += NT) {
    if (!ok(f)) continue;
    const int c = f % nx;
    const bool left = c > 0 && ok(f - 1);
    if (!CONN8) {
      const int g = f + nx;
      if (ok(g) && !(left && ok(g - 1))) uf_union(par, f, g);
    } else {
      for (int d = -1; d <= 1; ++d) {
        const int cc = c + d;
        if (cc < 0 || cc >= nx) continue;
        const int g = f + nx + d;
        if (!ok(g)) continue;
        if (left && cc - 1 >= 0 && ok(g - 1)) continue;  // united at (f-1, g-1)
        uf_union(par, f, g);
      }
    }
  }
  __syncthreads();
  // root pass, four cells' pointer chains in flight per thread (dependent global loads)
  for (int f0 = threadIdx.x; f0 < N; f0 += 4 * NT) {
    int x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = f0 + u * NT < N ? par[f0 + u * NT] : -1;
    bool more = true;
    while (more) {
      more = false;
      int nx_[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) nx_[u] = x[u] >= 0 ? par[x[u]] : x[u];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (nx_[u] < x[u]) { x[u] = nx_[u]; more = true; }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (x[u] >= 0) par[f0 + u * NT] = x[u];
  }
  __syncthreads();
}

// Connected components by flood fill on row-aligned bitmaps in shared memory
// (WPR = ceil(nx / 32) words per row; U = ok cells not yet labelled, C = the component
// being grown).  Components are taken in increasing order of their smallest cell (the
// first set bit of U), grown from it by dilation within U to the fixpoint -- a pass
// re-evaluates the 3 x 3 word neighbourhoods of the words that grew in the previous
// pass (a worklist; a word's runs fill at once) -- and labelled with that cell's
// index: the same output as grid_components (par[f] = smallest flat index of f's
// component, -1 where !ok) without global-memory pointer chasing.  A word is claimed
// by one thread per pass, so C only grows; a word can only grow after a neighbour
// did, so an empty worklist is the fixpoint.
CW_HD int bm_words(int nx, int ny) { return ((nx + 31) >> 5) * ny; }
constexpr size_t kBmCompMax = 100 * 1024;
// dynamic shared memory of bitmap_components (U, C, the claim bitmap Q, two u16 word
// lists), 0 when it exceeds kBmCompMax or the word ids need more than 16 bits (the
// union-find path runs then)
CW_HD size_t bmcomp_smem_bytes(int nx, int ny) {
  const size_t n = (size_t)bm_words(nx, ny);
  const size_t b = n * 8 + ((n + 31) / 32) * 4 + ((n * 2 * 2 + 15) & ~(size_t)15);
  return (b <= kBmCompMax && n <= 65536) ? b : 0;
}

template <int NT, bool CONN8, typename OkF>
CW_DEV void bitmap_components(int32_t* par, int nx, int ny, OkF ok, uint32_t* U) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int WPR = (nx + 31) >> 5, NWR = WPR * ny;
  uint32_t* C = U + NWR;
  uint32_t* Q = C + NWR;                                       // words claimed this pass
  uint16_t* L = reinterpret_cast<uint16_t*>(Q + (NWR + 31) / 32);   // two lists of NWR
  for (int i = threadIdx.x; i < (NWR + 31) / 32; i += NT) Q[i] = 0u;
  __shared__ int s_w0, s_lo, s_hi, s_n[2];
  for (int w = wid; w < NWR; w += NW) {   // warp per word, coalesced
    const int r = w / WPR, c = (w - r * WPR) * 32 + lane;
    const bool o = c < nx && ok(r * nx + c);
    const unsigned b = __ballot_sync(0xffffffffu, o);
    if (c < nx && !o) par[r * nx + c] = -1;
    if (lane == 0) { U[w] = b; C[w] = 0u; }
  }
  if (threadIdx.x == 0) s_w0 = NWR;
  __syncthreads();
  // one word of row r: dilate C around it (rows r-1..r+1, neighbour words' edge bits),
  // keep the ok bits, fill along the word's runs; true if C grew
  auto step = [&](int r, int cw) -> bool {
    const int w = r * WPR + cw;
    const unsigned u = U[w];
    if (!u) return false;
    auto hd = [&](int ww) -> unsigned {
      const unsigned x = C[ww];
      const unsigned l = cw > 0 ? C[ww - 1] : 0u, rt = cw + 1 < WPR ? C[ww + 1] : 0u;
      return x | (x << 1) | (l >> 31) | (x >> 1) | (rt << 31);
    };
    const unsigned cur = C[w];
    unsigned d = hd(w);
    if (CONN8) {
      if (r > 0) d |= hd(w - WPR);
      if (r + 1 < ny) d |= hd(w + WPR);
    } else {
      if (r > 0) d |= C[w - WPR];
      if (r + 1 < ny) d |= C[w + WPR];
    }
    const unsigned x = (d & u) | cur;
    if (x == cur) return false;
    unsigned g = u, y = x;   // parallel-prefix fill, both directions
    y |= (y << 1) & g; g &= g << 1;
    y |= (y << 2) & g; g &= g << 2;
    y |= (y << 4) & g; g &= g << 4;
    y |= (y << 8) & g; g &= g << 8;
    y |= (y << 16) & g;
    unsigned h = u, z = x;
    z |= (z >> 1) & h; h &= h >> 1;
    z |= (z >> 2) & h; h &= h >> 2;
    z |= (z >> 4) & h; h &= h >> 4;
    z |= (z >> 8) & h; h &= h >> 8;
    z |= (z >> 16) & h;
    C[w] = y | z;
    return true;
  };
  int cursor = 0;   // every word before it is empty in U
  while (true) {
    for (int w = cursor + (int)threadIdx.x; w < NWR; w += NT)
      if (U[w]) { atomicMin(&s_w0, w); break; }
    __syncthreads();
    const int w0 = s_w0;
    if (w0 >= NWR) break;
    const int r0 = w0 / WPR;
    const unsigned bit0 = (unsigned)__ffs(U[w0]) - 1u;
    const int id = r0 * nx + (w0 - r0 * WPR) * 32 + (int)bit0;
    cursor = w0;
    __syncthreads();
    if (threadIdx.x == 0) {
      C[w0] = 1u << bit0;
      L[0] = (uint16_t)w0;
      s_n[0] = 1;
      s_n[1] = 0;
      s_lo = s_hi = r0;
      s_w0 = NWR;
    }
    __syncthreads();
    // grow to the fixpoint: a pass evaluates the 3 x 3 word neighbourhoods of the words
    // that grew in the previous pass, each word once (claimed in Q)
    for (int p = 0;; p ^= 1) {
      const int n_in = s_n[p];
      const uint16_t* Lin = L + (size_t)p * NWR;
      uint16_t* Lout = L + (size_t)(p ^ 1) * NWR;
      int rmin = ny, rmax = -1;
      for (int i = threadIdx.x; i < n_in * 9; i += NT) {
        const int e = Lin[i / 9], k = i % 9;
        const int er = e / WPR;
        const int r = er + k / 3 - 1, cw = e - er * WPR + k % 3 - 1;
        if (r < 0 || r >= ny || cw < 0 || cw >= WPR) continue;
        const int wn = r * WPR + cw;
        const unsigned bit = 1u << (wn & 31);
        if (atomicOr(&Q[wn >> 5], bit) & bit) continue;
        if (step(r, cw)) {
          Lout[atomicAdd(&s_n[p ^ 1], 1)] = (uint16_t)wn;
          rmin = min(rmin, r);
          rmax = max(rmax, r);
          // chase the growth up and down the word column in this pass (rows are the
          // slow direction: a word boundary within a row is one pass, a row is one)
          for (int dir = -1; dir <= 1; dir += 2) {
            for (int rr = r + dir; rr >= 0 && rr < ny; rr += dir) {
              const int wc = rr * WPR + cw;
              const unsigned bc = 1u << (wc & 31);
              if (atomicOr(&Q[wc >> 5], bc) & bc) break;
              if (!step(rr, cw)) break;
              Lout[atomicAdd(&s_n[p ^ 1], 1)] = (uint16_t)wc;
              rmin = min(rmin, rr);
              rmax = max(rmax, rr);
            }
          }
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        rmin = min(rmin, __shfl_xor_sync(0xffffffffu, rmin, o));
        rmax = max(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
      }
      if (lane == 0 && rmax >= 0) { atomicMin(&s_lo, rmin); atomicMax(&s_hi, rmax); }
      __syncthreads();
      const int n_out = s_n[p ^ 1];
      for (int i = threadIdx.x; i < (NWR + 31) / 32; i += NT) Q[i] = 0u;   // release the claims
      if (threadIdx.x == 0) s_n[p] = 0;
      __syncthreads();
      if (n_out == 0) break;
    }
    const int lo = s_lo, hi = s_hi;
    for (int w = lo * WPR + wid; w < (hi + 1) * WPR; w += NW) {
      const unsigned b = C[w];
      if (!b) continue;
      const int r = w / WPR, c = (w - r * WPR) * 32 + lane;
      if ((b >> lane) & 1u) par[r * nx + c] = id;
      __syncwarp();
      if (lane == 0) { U[w] &= ~b; C[w] = 0u; }
    }
    __syncthreads();
  }
  __syncthreads();
}

// bitmap_components when the caller has the shared bitmaps (bm != nullptr), else the
// global-memory union-find
template <int NT, bool CONN8, typename OkF>
CW_DEV void components(int32_t* par, int nx, int ny, OkF ok, uint32_t* bm) {
  if (bm) bitmap_components<NT, CONN8>(par, nx, ny, ok, bm);
  else grid_components<NT, CONN8>((volatile int32_t*)par, nx, ny, ok);
}

// ================================================================= k_seeds
__global__ void k_seeds(int E, const uint64_t* __restrict__ scene_seed,
                        const uint64_t* __restrict__ crowd_seed, EnvSeeds* __restrict__ out) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  uint64_t s = scene_seed[e];
  EnvSeeds o;
  pcg_store(o.zones, make_rng(child_seed(s, "ground"), "zones"));
  uint64_t ts = child_seed(s, "terrain-stage");
  pcg_store(o.tileset, make_rng(ts, "tileset"));
  o.wfc_seed = child_seed(ts, "terrain");
  o.noise = child_seed(ts, "terrain-noise");
  pcg_store(o.objects, make_rng(child_seed(s, "placement"), "objects"));
  pcg_store(o.spawn, make_rng(crowd_seed ? crowd_seed[e] : 0ull, "crowd-spawn"));
  o.blocks = child_seed(s, "blocks");
  o.pad = 0;
  out[e] = o;
}

// ================================================================= zones
struct Courtyard {
  double fx, fy;
  int n_extra;
  Rect walk[5];
  int n_walk;
  int trail;
  Rect band;
  Rect build[2];
  int n_build;
};

CW_DEV void courtyard_draw(const cw_scene_params& P, Pcg64& rng, Courtyard& C) {
  // zones.py:79-129
  const double w = P.w, l = P.l;
  double fx = uniform(rng, 0.30, 0.42);
  double fy = uniform(rng, 0.30, 0.42);
  double cx = w / 2.0, cy = l / 2.0;
  C.walk[0] = rect_bounds(P, cx - fx * w, cy - fy * l, cx + fx * w, cy + fy * l);
  int n_extra = 2 + (int)integers32(rng, 3);
  C.fx = fx;
  C.fy = fy;
  C.n_extra = n_extra;
  for (int k = 0; k < n_extra; ++k) {
    double ex = uniform(rng, cx - fx * w, cx + fx * w);
    double ey = uniform(rng, cy - fy * l, cy + fy * l);
    double hw = uniform(rng, 0.10, 0.25) * w;
    double hl = uniform(rng, 0.10, 0.25) * l;
    C.walk[1 + k] = rect_bounds(P, ex - hw, ey - hl, ex + hw, ey + hl);
  }
  C.n_walk = 1 + n_extra;
  C.trail = next_double(rng) < 0.5;
  if (C.trail) {
    double tw = uniform(rng, 1.2, 2.2);
    if (next_double(rng) < 0.5) {
      double tx = uniform(rng, cx - 0.2 * w, cx + 0.2 * w);
      C.band = rect_bounds(P, tx - tw / 2, 0.0, tx + tw / 2, l);
    } else {
      double ty = uniform(rng, cy - 0.2 * l, cy + 0.2 * l);
      C.band = rect_bounds(P, 0.0, ty - tw / 2, w, ty + tw / 2);
    }
  }
  int n_build = (int)integers32(rng, 3);
  int order[4] = {0, 1, 2, 3};
  for (int i = 3; i > 0; --i) {
    int j = (int)interval32(rng, (uint32_t)i);
    int t = order[i]; order[i] = order[j]; order[j] = t;
  }
  const double kx[4] = {0.0, w, 0.0, w}, ky[4] = {0.0, 0.0, l, l};
  C.n_build = 0;
  for (int q = 0; q < 4; ++q) {
    if (C.n_build >= n_build) break;
    int idx = order[q];
    double bw = uniform(rng, 0.12, 0.22) * w;
    double bl = uniform(rng, 0.12, 0.22) * l;
    double x0 = kx[idx] == 0.0 ? 0.0 : w - bw;
    double y0 = ky[idx] == 0.0 ? 0.0 : l - bl;
    Rect m = rect_bounds(P, x0, y0, x0 + bw, y0 + bl);
    bool meet = false;
    for (int k = 0; k < C.n_walk; ++k) meet |= rect_meet(m, C.walk[k]);
    if (!meet) C.build[C.n_build++] = m;
  }
}

__global__ void __launch_bounds__(256) k_zones(cw_scene_params P, int E, const int32_t* slots,
                                               const EnvSeeds* __restrict__ seeds,
                                               cw_scene_buffers B) {
  const int e = blockIdx.x;
  const int slot = env_slot(slots, e);
  __shared__ Courtyard C;
  __shared__ Rect strip;
  if (threadIdx.x == 0) {
    double* zp = B.zone_params + (size_t)slot * CW_ZONE_PARAMS;
    for (int k = 0; k < CW_ZONE_PARAMS; ++k) zp[k] = 0.0;
    if (P.layout == 0) {
      Pcg64 rng = pcg_load(seeds[e].zones);
      courtyard_draw(P, rng, C);
      zp[0] = C.fx;
      zp[1] = C.fy;
      zp[2] = C.n_extra;
      zp[3] = C.trail;
      zp[4] = C.n_build;
    } else {
      double b = fmin(1.0, 0.2 * fmin(P.w, P.l));  // zones.py:71-76
      strip = rect_bounds(P, b, b, P.w - b, P.l - b);
      zp[0] = b;
    }
  }
  __syncthreads();
  uint8_t* Z = B.zones + (size_t)slot * P.ny * P.nx;
  const int N = P.nx * P.ny;
  int mine = 0;
  for (int f = threadIdx.x; f < N; f += blockDim.x) {
    int r = f / P.nx, c = f - r * P.nx;
    uint8_t z = Z_VEGETATION;
    if (P.layout == 0) {
      bool walk = false;
      for (int k = 0; k < C.n_walk; ++k) walk |= rect_has(C.walk[k], r, c);
      if (walk) {
        z = (C.trail && rect_has(C.band, r, c)) ? Z_SIDEWALK : Z_PLAZA;
      } else {
        for (int k = 0; k < C.n_build; ++k)
          if (rect_has(C.build[k], r, c)) z = Z_BUILDING;
      }
    } else if (rect_has(strip, r, c)) {
      z = Z_PLAZA;
    }
    mine |= z <= Z_PLAZA;
    Z[f] = z;
  }
  mine = __syncthreads_or(mine);
  if (threadIdx.x == 0 && !mine) B.status[slot] = CW_E_EXTENT;
}

// ---------------------------------------------------------------- block layout
struct BlockLayout {
  uint8_t sock[CW_MAX_BLOCKS][4];  // N, E, S, W
  uint8_t var[CW_MAX_BLOCKS];      // kind * 4 + orientation
  int n;
  double sw;
  uint8_t quad[CW_MAX_BLOCKS][4];  // zone per (qx, qy) quadrant, index qx*2+qy
};

// blocks.py:24-31 variants: kind-major, orientation-minor; sockets (N,E,S,W)
CW_DEV void variant_sockets(int v, uint8_t s[4]) {
  const uint8_t base[7][4] = {{1, 0, 1, 0}, {1, 1, 0, 0}, {1, 1, 1, 1}, {1, 1, 0, 1},
                              {1, 1, 0, 1}, {1, 1, 1, 1}, {1, 1, 0, 1}};
  int k = v >> 2, o = v & 3;
  for (int i = 0; i < 4; ++i) s[i] = base[k][(i - o + 4) & 3];
}

CW_DEV bool blocks_connected(const BlockLayout& L, int rows, int cols) {
  if (rows * cols == 1) return true;
  uint64_t seen = 1, frontier = 1;
  while (frontier) {
    uint64_t nxt = 0;
    for (int i = 0; i < rows * cols; ++i) {
      if (!((frontier >> i) & 1)) continue;
      int r = i / cols, c = i % cols;
      if (L.sock[i][1] && c + 1 < cols) nxt |= 1ull << (i + 1);
      if (L.sock[i][2] && r + 1 < rows) nxt |= 1ull << (i + cols);
      if (c > 0 && L.sock[i - 1][1]) nxt |= 1ull << (i - 1);
      if (r > 0 && L.sock[i - cols][2]) nxt |= 1ull << (i - cols);
    }
    frontier = nxt & ~seen;
    seen |= nxt;
  }
  return __popcll(seen) == rows * cols;
}

CW_DEV void connect_blocks(uint64_t seed, int rows, int cols, BlockLayout& L) {
  // blocks.py:34-77
  for (int attempt = 0; attempt < 16; ++attempt) {
    Pcg64 rng = pcg_seed(child_seed(seed, "blocks", (uint64_t)attempt));
    for (int r = 0; r < rows; ++r)
      for (int c = 0; c < cols; ++c) {
        int need_n = r ? L.sock[(r - 1) * cols + c][2] : -1;
        int need_w = c ? L.sock[r * cols + c - 1][1] : -1;
        int opts[28], n = 0;
        for (int v = 0; v < 28; ++v) {
          uint8_t s[4];
          variant_sockets(v, s);
          if ((need_n < 0 || s[0] == need_n) && (need_w < 0 || s[3] == need_w)) opts[n++] = v;
        }
        int v = opts[integers32(rng, (uint64_t)n)];
        L.var[r * cols + c] = (uint8_t)v;
        variant_sockets(v, L.sock[r * cols + c]);
      }
    if (blocks_connected(L, rows, cols)) return;
  }
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) {
      L.var[r * cols + c] = (r == 0 && cols > 1) ? 5 * 4 : 0;
      variant_sockets(L.var[r * cols + c], L.sock[r * cols + c]);
    }
}

CW_DEV bool in_road(const cw_scene_params& P, const BlockLayout& L, double ox, double oy, int r,
                    int c) {
  const double bs = 20.0, rw = 6.0;
  for (int i = 0; i < L.n; ++i) {
    int br = i / P.bcols, bc = i % P.bcols;
    double x0 = ox + bc * bs, y0 = oy + br * bs;
    double cx = x0 + bs / 2.0, cy = y0 + bs / 2.0;
    if (L.sock[i][0] && rect_has(rect_bounds(P, cx - rw / 2, y0, cx + rw / 2, cy), r, c)) return true;
    if (L.sock[i][2] && rect_has(rect_bounds(P, cx - rw / 2, cy, cx + rw / 2, y0 + bs), r, c)) return true;
    if (L.sock[i][3] && rect_has(rect_bounds(P, x0, cy - rw / 2, cx, cy + rw / 2), r, c)) return true;
    if (L.sock[i][1] && rect_has(rect_bounds(P, cx, cy - rw / 2, x0 + bs, cy + rw / 2), r, c)) return true;
  }
  return false;
}

// CTA per env.  Chamfer distance (gridmath.py:8-39) kept in float64 scratch.
__global__ void __launch_bounds__(512) k_zones_blk(cw_scene_params P, int E, const int32_t* slots,
                                                   const EnvSeeds* __restrict__ seeds,
                                                   cw_scene_buffers B) {
  constexpr int NT = 512;
  const int e = blockIdx.x;
  const int slot = env_slot(slots, e);
  const int nx = P.nx, ny = P.ny, N = nx * ny;
  __shared__ BlockLayout L;
  __shared__ double rowbuf[2][1024 + 1];
  double* D = B.scratch_f64 + (size_t)e * (size_t)max(P.obj_max * 8, N);
  uint8_t* Z = B.zones + (size_t)slot * N;
  const double bs = 20.0, rw = 6.0;
  const double ox = (P.w - P.bcols * bs) / 2.0, oy = (P.l - P.brows * bs) / 2.0;
  if (threadIdx.x == 0) {
    L.n = P.brows * P.bcols;
    connect_blocks(seeds[e].blocks, P.brows, P.bcols, L);
    Pcg64 rng = pcg_load(seeds[e].zones);
    L.sw = uniform(rng, 1.5, 3.0);
    double* zp = B.zone_params + (size_t)slot * CW_ZONE_PARAMS;
    for (int k = 0; k < CW_ZONE_PARAMS; ++k) zp[k] = 0.0;
    zp[0] = L.sw;
    zp[1] = rw;
    for (int i = 0; i < CW_MAX_BLOCKS; ++i) B.block_var[(size_t)slot * CW_MAX_BLOCKS + i] = i < L.n ? L.var[i] : 0;
    for (int i = 0; i < L.n; ++i)
      for (int qx = 0; qx < 2; ++qx)
        for (int qy = 0; qy < 2; ++qy) {
          double u = next_double(rng);
          int k = 0;
          while (k < 2 && !(P.quad_cdf[k] > u)) ++k;
          const uint8_t zs[3] = {Z_BUILDING, Z_VEGETATION, Z_PLAZA};
          L.quad[i][qx * 2 + qy] = zs[k];
        }
  }
  __syncthreads();
  // road mask -> D (0 on road, 1e9 elsewhere)
  for (int f = threadIdx.x; f < N; f += NT) {
    int r = f / nx, c = f - r * nx;
    D[f] = in_road(P, L, ox, oy, r, c) ? 0.0 : 1e9;
  }
  __syncthreads();
  const double s2 = kSqrt2;
  // horizontal relax of one row in place (prefix/suffix running minima)
  auto relax = [&](double* row) {
    // left: min.accumulate(row - j) + j ; right: reversed analogue
    // block-wide scan over nx <= 1024 using NT threads, two elements each
    double* a = rowbuf[0];
    double* b = rowbuf[1];
    for (int j = threadIdx.x; j < nx; j += NT) {
      a[j] = row[j] - (double)j;
      b[j] = row[nx - 1 - j] + (double)(nx - 1 - j);
    }
    __syncthreads();
    for (int o = 1; o < nx; o <<= 1) {
      double va[2], vb[2];
      int cnt = 0;
      for (int j = threadIdx.x; j < nx; j += NT, ++cnt) {
        va[cnt] = j >= o ? fmin(a[j], a[j - o]) : a[j];
        vb[cnt] = j >= o ? fmin(b[j], b[j - o]) : b[j];
      }
      __syncthreads();
      cnt = 0;
      for (int j = threadIdx.x; j < nx; j += NT, ++cnt) {
        a[j] = va[cnt];
        b[j] = vb[cnt];
      }
      __syncthreads();
    }
    for (int j = threadIdx.x; j < nx; j += NT) {
      double lft = a[j] + (double)j;
      int jr = nx - 1 - j;  // b index of column j
      double rgt = b[jr] - (double)j;
      row[j] = fmin(lft, rgt);
    }
    __syncthreads();
  };
  auto pull = [&](double* dst, const double* src) {
    for (int j = threadIdx.x; j < nx; j += NT) {
      double dg = 1e9;
      if (j >= 1) dg = src[j - 1] + s2;
      if (j + 1 < nx) dg = fmin(dg, src[j + 1] + s2);
      dst[j] = fmin(dst[j], fmin(src[j] + 1.0, dg));
    }
    __syncthreads();
  };
  for (int r = 0; r < ny; ++r) {
    if (r) pull(D + (size_t)r * nx, D + (size_t)(r - 1) * nx);
    relax(D + (size_t)r * nx);
  }
  for (int r = ny - 2; r >= 0; --r) {
    pull(D + (size_t)r * nx, D + (size_t)(r + 1) * nx);
    relax(D + (size_t)r * nx);
  }
  // compose zones
  const double cw_len = 1.2;
  int mine = 0;
  for (int f = threadIdx.x; f < N; f += NT) {
    int r = f / nx, c = f - r * nx;
    double dist = D[f] * P.res;
    bool road = D[f] == 0.0 && in_road(P, L, ox, oy, r, c);
    bool side = dist > 0 && dist <= L.sw;
    uint8_t z = Z_VEGETATION;
    if (side) z = Z_SIDEWALK;
    if (road) z = Z_ROADWAY;
    if (!road && !side) {
      for (int i = 0; i < L.n; ++i) {
        int br = i / P.bcols, bc = i % P.bcols;
        double x0 = ox + bc * bs, y0 = oy + br * bs;
        for (int qx = 0; qx < 2; ++qx)
          for (int qy = 0; qy < 2; ++qy) {
            Rect m = rect_bounds(P, x0 + qx * bs / 2 + 1.0, y0 + qy * bs / 2 + 1.0,
                                 x0 + (qx + 1) * bs / 2 - 1.0, y0 + (qy + 1) * bs / 2 - 1.0);
            if (rect_has(m, r, c)) z = L.quad[i][qx * 2 + qy];
          }
      }
    }
    if (road) {
      for (int i = 0; i < L.n; ++i) {
        const uint8_t* s = L.sock[i];
        if (s[0] + s[1] + s[2] + s[3] < 3) continue;
        int br = i / P.bcols, bc = i % P.bcols;
        double x0 = ox + bc * bs, y0 = oy + br * bs;
        double cx = x0 + bs / 2.0, cy = y0 + bs / 2.0;
        Rect sp[4];
        int ax[4], n = 0;
        if (s[0]) { sp[n] = rect_bounds(P, cx - rw / 2, y0 + 1.0, cx + rw / 2, y0 + 1.0 + cw_len); ax[n++] = 0; }
        if (s[2]) { sp[n] = rect_bounds(P, cx - rw / 2, y0 + bs - 1.0 - cw_len, cx + rw / 2, y0 + bs - 1.0); ax[n++] = 0; }
        if (s[3]) { sp[n] = rect_bounds(P, x0 + 1.0, cy - rw / 2, x0 + 1.0 + cw_len, cy + rw / 2); ax[n++] = 1; }
        if (s[1]) { sp[n] = rect_bounds(P, x0 + bs - 1.0 - cw_len, cy - rw / 2, x0 + bs - 1.0, cy + rw / 2); ax[n++] = 1; }
        for (int k = 0; k < n; ++k) {
          if (!rect_has(sp[k], r, c)) continue;
          bool sel = ax[k] == 0 ? ((r & 1) && r > 0 && r < ny - 1) : ((c & 1) && c > 0 && c < nx - 1);
          if (sel) z = Z_CROSSWALK;
        }
      }
    }
    mine |= z <= Z_PLAZA;
    Z[f] = z;
  }
  mine = __syncthreads_or(mine);
  if (threadIdx.x == 0 && !mine) B.status[slot] = CW_E_EXTENT;
}

// ================================================================= terrain
enum { K_FLAT = 0, K_SUP = 1, K_SDOWN = 2, K_STUP = 3, K_STDOWN = 4, K_ROUGH = 5 };
enum { T_CORNER = 0, T_STAIR_U = 1, T_STAIR_V = 2, T_ROUGH = 3 };

struct TileSet {
  int n;
  int8_t code[CW_MAX_TILES];
  int8_t kind[CW_MAX_TILES];
  double param[CW_MAX_TILES];
  double p[CW_MAX_TILES][4];
  double w[CW_MAX_TILES];
  unsigned long long allowed[4][CW_MAX_TILES];  // N, E, S, W
};

CW_DEV int family_of(int kind) {
  return kind == K_FLAT ? 0 : (kind <= K_SDOWN ? 1 : (kind <= K_STDOWN ? 2 : 3));
}

CW_DEV void ts_corner(TileSet& T, double h00, double h10, double h01, double h11, double grade) {
  // terrain.py:216-227
  int i = T.n++;
  T.code[i] = T_CORNER;
  T.p[i][0] = h00; T.p[i][1] = h10; T.p[i][2] = h01; T.p[i][3] = h11;
  if (h00 == h10 && h10 == h01 && h01 == h11) {
    T.kind[i] = K_FLAT;
    T.param[i] = 0.0;
  } else {
    double up = (h10 + h11 - h00 - h01) + (h01 + h11 - h00 - h10);
    T.kind[i] = up > 0 ? K_SUP : K_SDOWN;
    T.param[i] = grade;
  }
}

CW_DEV void sort2_unique(double* v, int& n) {
  // sorted({a, b})
  if (v[0] == v[1]) { n = 1; return; }
  if (v[1] < v[0]) { double t = v[0]; v[0] = v[1]; v[1] = t; }
  n = 2;
}

CW_DEV void build_tileset_serial(const cw_scene_params& P, Pcg64& rng, TileSet& T) {
  // terrain.py:160-212 (palette + weights; adjacency filled in parallel)
  const double TS = 2.0;
  T.n = 0;
  ts_corner(T, 0, 0, 0, 0, 0);
  const double rs_lo = P.split ? 0.10 : 0.05, rs_hi = P.split ? 0.30 : 0.23;
  const double sl_lo = P.split ? 0.05 : 0.00, sl_hi = P.split ? 0.80 : 0.40;
  const double ro_lo = P.split ? 0.05 : 0.02, ro_hi = P.split ? 0.20 : 0.10;
  if (P.mix[1] > 0) {
    double g[2] = {uniform(rng, sl_lo, sl_hi), uniform(rng, sl_lo, sl_hi)};
    int ng;
    sort2_unique(g, ng);
    for (int k = 0; k < ng; ++k) {
      double h = g[k] * TS;
      if (h <= 0) continue;
      double hv[2] = {0.0, h};
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
          for (int c = 0; c < 2; ++c)
            for (int d = 0; d < 2; ++d) {
              double h00 = hv[a], h10 = hv[b], h01 = hv[c], h11 = hv[d];
              if (h00 == 0.0 && h10 == 0.0 && h01 == 0.0 && h11 == 0.0) continue;
              if (h00 == h11 && h10 == h01 && h00 != h10) continue;
              ts_corner(T, h00, h10, h01, h11, g[k]);
            }
    }
  }
  if (P.mix[2] > 0) {
    double rise = uniform(rng, rs_lo, rs_hi);
    for (int ax = 0; ax < 2; ++ax)
      for (int low = 1; low >= 0; --low)
        for (int lev = 0; lev < 3; ++lev) {
          int i = T.n++;
          double hl = lev * rise, hh = (lev + 1) * rise;
          T.code[i] = ax == 0 ? T_STAIR_U : T_STAIR_V;
          T.kind[i] = low ? K_STUP : K_STDOWN;
          T.param[i] = rise;
          T.p[i][0] = low ? hl : hh;
          T.p[i][1] = low ? hh : hl;
          T.p[i][2] = 0.0;
          T.p[i][3] = 0.0;
        }
    for (int lev = 1; lev <= 3; ++lev) {
      double h = lev * rise;
      ts_corner(T, h, h, h, h, 0.0);
    }
  }
  if (P.mix[3] > 0) {
    double a[2] = {uniform(rng, ro_lo, ro_hi), uniform(rng, ro_lo, ro_hi)};
    int na;
    sort2_unique(a, na);
    for (int k = 0; k < na; ++k) {
      int i = T.n++;
      T.code[i] = T_ROUGH;
      T.kind[i] = K_ROUGH;
      T.param[i] = a[k];
      T.p[i][0] = 0.0; T.p[i][1] = a[k]; T.p[i][2] = 0.0; T.p[i][3] = 0.0;
    }
  }
  int fam_n[4] = {0, 0, 0, 0};
  for (int i = 0; i < T.n; ++i) fam_n[family_of(T.kind[i])]++;
  for (int i = 0; i < T.n; ++i) {
    int f = family_of(T.kind[i]);
    T.w[i] = P.mix[f] / (double)fam_n[f];
  }
}

// edge profile of tile i on edge d (0 N, 1 E, 2 S, 3 W): terrain.py:248-276
CW_DEV void edge_profile(const TileSet& T, int i, int d, int& step, double& a, double& b) {
  const double* p = T.p[i];
  step = 0;
  if (T.code[i] == T_CORNER) {
    if (d == 0) { a = p[0]; b = p[1]; }
    else if (d == 2) { a = p[2]; b = p[3]; }
    else if (d == 3) { a = p[0]; b = p[2]; }
    else { a = p[1]; b = p[3]; }
  } else if (T.code[i] == T_STAIR_U) {
    if (d == 0 || d == 2) { step = 1; a = p[0]; b = p[1]; }
    else if (d == 3) { a = p[0]; b = p[0]; }
    else { a = p[1]; b = p[1]; }
  } else if (T.code[i] == T_STAIR_V) {
    if (d == 0) { a = p[0]; b = p[0]; }
    else if (d == 2) { a = p[1]; b = p[1]; }
    else { step = 1; a = p[0]; b = p[1]; }
  } else {
    a = 0.0; b = 0.0;
  }
}

CW_DEV double prof_eval(int step, double a, double b, double t) {
  if (!step) return a + (b - a) * t;
  return t < 0.5 ? a : b;
}

CW_DEV bool tiles_compatible(const TileSet& T, int i, int j, int d) {
  // terrain.py:283-292
  int s1, s2;
  double a1, b1, a2, b2;
  edge_profile(T, i, d, s1, a1, b1);
  edge_profile(T, j, (d + 2) & 3, s2, a2, b2);
  const double probes[4] = {0.0, 0.499999, 0.500001, 1.0};
  double gap = 0.0;
  for (int k = 0; k < 4; ++k) {
    double g = fabs(prof_eval(s1, a1, b1, probes[k]) - prof_eval(s2, a2, b2, probes[k]));
    gap = k == 0 ? g : fmax(gap, g);
  }
  double tol = 1e-9;
  if (T.kind[i] == K_STUP || T.kind[i] == K_STDOWN) tol = fmax(tol, T.param[i]);
  if (T.kind[j] == K_STUP || T.kind[j] == K_STDOWN) tol = fmax(tol, T.param[j]);
  return gap <= tol + 1e-12;
}

// numpy pairwise sum (n <= 44 < 128): oracle/rng.py:pairwise_sum
CW_DEV double np_pairwise_sum(const double* a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res += a[i];
    return res;
  }
  double r[8];
  for (int k = 0; k < 8; ++k) r[k] = a[k];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int k = 0; k < 8; ++k) r[k] += a[i + k];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += a[i];
  return res;
}

// WFC runs one warp per env (terrain.py:215-259, wfc.py:24-115).  Arc
// consistency has a unique greatest fixpoint, so the initial full propagation
// is a Jacobi sweep over the lattice and the per-collapse propagation is a LIFO
// worklist from the collapsed cell (the reference's order; any order reaches
// the same fixpoint and detects the same wipe-outs).
constexpr int TER_WARPS = 4;

struct WarpWfc {
  TileSet T;
  unsigned long long nib[4][11][16];  // support tables: OR of allowed[d][t] over a nibble of tiles
  double pw[CW_MAX_TILES];            // choice(): the options' weights / probabilities / cdf
};

// tiles allowed next to a cell with domain `dom` in direction d: the OR of the nibble
// tables, all 11 lookups independent (nib[..][0] = 0)
CW_DEV unsigned long long support(const WarpWfc& W, int d, unsigned long long dom) {
  unsigned long long s = 0;
#pragma unroll
  for (int k = 0; k < 11; ++k) s |= W.nib[d][k][(unsigned)(dom >> (4 * k)) & 15u];
  return s;
}

// neighbour (dir d of x): 0 N, 1 E, 2 S, 3 W; tiles allowed there given dom[x]
CW_DEV int wfc_nbr(int x, int d, int rows, int cols) {
  const int r = x / cols, c = x - r * cols;
  if (d == 0) return r > 0 ? x - cols : -1;
  if (d == 1) return c + 1 < cols ? x + 1 : -1;
  if (d == 2) return r + 1 < rows ? x + cols : -1;
  return c > 0 ? x - 1 : -1;
}

// full Jacobi sweep to the fixpoint; false on a wipe-out
CW_DEV bool wfc_propagate_all(const WarpWfc& W, unsigned long long* dom, int rows, int cols, int lane) {
  const int L = rows * cols;
  while (true) {
    bool changed = false, empty = false;
    for (int x0 = 0; x0 < L; x0 += 32) {
      const int x = x0 + lane;
      unsigned long long nd = 0;
      if (x < L) {
        nd = dom[x];
        const int r = x / cols, c = x - r * cols;
        if (r > 0) nd &= support(W, 2, dom[x - cols]);
        if (r + 1 < rows) nd &= support(W, 0, dom[x + cols]);
        if (c > 0) nd &= support(W, 1, dom[x - 1]);
        if (c + 1 < cols) nd &= support(W, 3, dom[x + 1]);
      }
      __syncwarp();
      if (x < L) {
        changed |= nd != dom[x];
        empty |= nd == 0ull;
        dom[x] = nd;
      }
      __syncwarp();
    }
    if (__any_sync(0xffffffffu, empty)) return false;
    if (!__any_sync(0xffffffffu, changed)) return true;
  }
}

// lane-0 LIFO worklist from cell x0 (wfc.py:89-115); false on a wipe-out
CW_DEV bool wfc_propagate_from(const WarpWfc& W, unsigned long long* dom, int* stack,
                               unsigned char* inq, int x0, int rows, int cols) {
  int top = 0;
  stack[top++] = x0;
  inq[x0] = 1;
  bool ok = true;
  while (top > 0) {
    const int x = stack[--top];
    inq[x] = 0;
    const unsigned long long here = dom[x];
    if (here == 0ull) { ok = false; break; }
    for (int d = 0; d < 4; ++d) {
      const int y = wfc_nbr(x, d, rows, cols);
      if (y < 0) continue;
      const unsigned long long before = dom[y];
      const unsigned long long after = before & support(W, d, here);
      if (after == 0ull) { ok = false; break; }
      if (after != before) {
        dom[y] = after;
        if (!inq[y]) { inq[y] = 1; stack[top++] = y; }
      }
    }
    if (!ok) break;
  }
  if (!ok) while (top > 0) inq[stack[--top]] = 0;
  return ok;
}

CW_HD size_t terrain_warp_smem(int L) {
  size_t per = sizeof(WarpWfc) + (size_t)L * 8 * 2 + (size_t)L * 4 + (size_t)L;
  per = (per + 15) & ~(size_t)15;
  return per;
}

__global__ void __launch_bounds__(TER_WARPS * 32) k_terrain(cw_scene_params P, int E,
                                                            const int32_t* slots,
                                                            const EnvSeeds* __restrict__ seeds,
                                                            cw_scene_buffers B) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int e = blockIdx.x * (blockDim.x >> 5) + wid;   // warps per CTA: as many lattices as fit
  if (e >= E) return;
  const int slot = env_slot(slots, e);
  if (B.status[slot] != CW_OK) return;
  const int rows = P.trows, cols = P.tcols, L = rows * cols;
  unsigned char* base = smem_raw + (size_t)wid * terrain_warp_smem(L);
  WarpWfc& W = *reinterpret_cast<WarpWfc*>(base);
  unsigned long long* dom = reinterpret_cast<unsigned long long*>(base + sizeof(WarpWfc));
  unsigned long long* init = dom + L;
  int* stack = reinterpret_cast<int*>(init + L);
  unsigned char* inq = reinterpret_cast<unsigned char*>(stack + L);
  TileSet& T = W.T;
  if (lane == 0) {
    Pcg64 rng = pcg_load(seeds[e].tileset);
    build_tileset_serial(P, rng, T);
  }
  for (int k = lane; k < 4 * CW_MAX_TILES; k += 32) (&T.allowed[0][0])[k] = 0ull;
  __syncwarp();
  const int n = T.n;
  for (int q = lane; q < n * n; q += 32) {
    const int i = q / n, j = q - i * n;
    if (tiles_compatible(T, i, j, 1)) {  // E, and W = E^T
      atomicOr(&T.allowed[1][i], 1ull << j);
      atomicOr(&T.allowed[3][j], 1ull << i);
    }
    if (tiles_compatible(T, i, j, 2)) {  // S, and N = S^T
      atomicOr(&T.allowed[2][i], 1ull << j);
      atomicOr(&T.allowed[0][j], 1ull << i);
    }
  }
  __syncwarp();
  for (int q = lane; q < 4 * 11 * 16; q += 32) {
    const int d = q / 176, k = (q / 16) % 11, v = q & 15;
    unsigned long long sp = 0;
    for (int b = 0; b < 4; ++b) {
      const int t = 4 * k + b;
      if (((v >> b) & 1) && t < n) sp |= T.allowed[d][t];
    }
    W.nib[d][k][v] = sp;
  }
  // forced-flat tiles outside the walkable area (terrain.py:236-250)
  const uint8_t* Z = B.zones + (size_t)slot * P.nx * P.ny;
  const unsigned long long full = (1ull << n) - 1ull;
  const int cpt = P.cpt;
  for (int x = 0; x < L; ++x) {
    const int r = x / cols, c = x - r * cols;
    const int r0 = r * cpt, c0 = c * cpt;
    bool inside = (r0 + cpt <= P.ny) && (c0 + cpt <= P.nx);
    if (inside) {
      bool bad = false;
      for (int k = lane; k < cpt * cpt; k += 32) {
        const int rr = r0 + k / cpt, cc = c0 + k % cpt;
        const uint8_t z = Z[(size_t)rr * P.nx + cc];
        bad |= !(z <= Z_PLAZA && (P.nonflat_split_col < 0 || cc >= P.nonflat_split_col));
      }
      inside = !__any_sync(0xffffffffu, bad);
    }
    if (lane == 0) init[x] = inside ? full : 1ull;
  }
  for (int x = lane; x < L; x += 32) inq[x] = 0;
  __syncwarp();
  int attempt_ok = -1;
  for (int attempt = 0; attempt < 16 && attempt_ok < 0; ++attempt) {
    for (int x = lane; x < L; x += 32) dom[x] = init[x];
    __syncwarp();
    Pcg64 rng;
    if (lane == 0) rng = pcg_seed(child_seed(seeds[e].wfc_seed, "wfc", (uint64_t)attempt));
    bool ok = wfc_propagate_all(W, dom, rows, cols, lane);
    while (ok) {
      // minimum-entropy open cell, ties by lowest flat index (wfc.py:61-70)
      unsigned long long best = ~0ull;
      for (int x = lane; x < L; x += 32) {
        const int cnt = __popcll(dom[x]);
        if (cnt > 1) {
          const unsigned long long key = ((unsigned long long)cnt << 32) | (unsigned)x;
          best = key < best ? key : best;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
        best = y < best ? y : best;
      }
      if (best == ~0ull) break;  // fully collapsed
      // Generator.choice(no, p=w/tot) (wfc.py:71-77): the divisions and the
      // searchsorted tests run one option per lane (each an independent IEEE op, so the
      // same bits); the pairwise total and the cumsum stay sequential in lane 0
      const int x = (int)(best & 0xffffffffu);
      const unsigned long long d = dom[x];
      const int no = __popcll(d);
      const unsigned lo32 = (unsigned)d, hi32 = (unsigned)(d >> 32);
      const int nlo = __popc(lo32);
      auto opt_of = [&](int k) {   // the k-th set bit of d
        return k < nlo ? (int)__fns(lo32, 0, k + 1) : 32 + (int)__fns(hi32, 0, k - nlo + 1);
      };
      for (int k = lane; k < no; k += 32) W.pw[k] = T.w[opt_of(k)];
      __syncwarp();
      double tot = 0.0;
      if (lane == 0) tot = np_pairwise_sum(W.pw, no);
      tot = __shfl_sync(0xffffffffu, tot, 0);
      const bool uniform_w = !(tot > 0);
      if (uniform_w) tot = (double)no;
      double pk[2] = {0.0, 0.0};
      for (int i = 0; i < 2; ++i) {
        const int k = lane + 32 * i;
        if (k < no) pk[i] = (uniform_w ? 1.0 : W.pw[k]) / tot;
      }
      __syncwarp();
      for (int i = 0; i < 2; ++i) if (lane + 32 * i < no) W.pw[lane + 32 * i] = pk[i];
      __syncwarp();
      double u = 0.0;
      if (lane == 0) {   // cdf = cumsum(p) in order
        double acc = W.pw[0];
        for (int k = 1; k < no; ++k) { acc = acc + W.pw[k]; W.pw[k] = acc; }
        u = next_double(rng);
      }
      __syncwarp();
      u = __shfl_sync(0xffffffffu, u, 0);
      const double last = W.pw[no - 1];
      // searchsorted(cdf / last, u, 'right') = the first k with cdf[k] / last > u
      unsigned hit0 = __ballot_sync(0xffffffffu, lane < no && W.pw[lane] / last > u);
      unsigned hit1 = __ballot_sync(0xffffffffu, lane + 32 < no && W.pw[lane + 32] / last > u);
      const int idx = hit0 ? __ffs(hit0) - 1 : (hit1 ? 32 + __ffs(hit1) - 1 : no);
      __syncwarp();
      int okl = 1;
      if (lane == 0) {
        dom[x] = 1ull << opt_of(idx);
        okl = wfc_propagate_from(W, dom, stack, inq, x, rows, cols);
      }
      ok = __shfl_sync(0xffffffffu, okl, 0) != 0;
      __syncwarp();
    }
    if (ok) attempt_ok = attempt;
    __syncwarp();
  }
  int32_t* A = B.assign + (size_t)slot * L;
  if (attempt_ok < 0) {
    if (lane == 0) B.status[slot] = CW_E_CONTRADICTION;
    return;
  }
  for (int x = lane; x < L; x += 32) A[x] = __ffsll((long long)dom[x]) - 1;
  if (lane == 0) {
    B.wfc_attempts[slot] = attempt_ok;
    B.n_tiles[slot] = n;
    B.noise_seed[slot] = seeds[e].noise;
  }
  for (int i = lane; i < CW_MAX_TILES; i += 32) {
    const size_t o = (size_t)slot * CW_MAX_TILES + i;
    const bool v = i < n;
    B.tile_code[o] = v ? T.code[i] : -1;
    B.tile_kind[o] = v ? T.kind[i] : -1;
    B.tile_param[o] = v ? T.param[i] : 0.0;
    B.tile_w[o] = v ? T.w[i] : 0.0;
    for (int k = 0; k < 4; ++k) B.tile_p[o * 4 + k] = v ? T.p[i][k] : 0.0;
    for (int d = 0; d < 4; ++d)
      B.allowed[((size_t)slot * 4 + d) * CW_MAX_TILES + i] = v ? T.allowed[d][i] : 0ull;
  }
}

// ================================================================= placement
// Corners of an oriented footprint: types.py:355-361; the (4,2)@(2,2) product is
// OpenBLAS dgemm = fma(l1, r1, l0*r0) with rot rows (c, -s), (s, c).
CW_DEV void footprint_corners(double fw, double fl, double x, double y, double c, double s,
                              double* cx, double* cy) {
  const double hw = fw / 2.0, hl = fl / 2.0;
  const double lx[4] = {-hw, hw, hw, -hw}, ly[4] = {-hl, -hl, hl, hl};
  for (int i = 0; i < 4; ++i) {
    cx[i] = __fma_rn(ly[i], -s, lx[i] * c) + x;
    cy[i] = __fma_rn(ly[i], c, lx[i] * s) + y;
  }
}

struct FootBox { int r0, r1, c0, c1; bool empty; };

CW_DEV FootBox footprint_box(const cw_scene_params& P, const double* cx, const double* cy) {
  // placement.py:36-44
  double x0 = cx[0], x1 = cx[0], y0 = cy[0], y1 = cy[0];
  for (int i = 1; i < 4; ++i) {
    x0 = fmin(x0, cx[i]); x1 = fmax(x1, cx[i]);
    y0 = fmin(y0, cy[i]); y1 = fmax(y1, cy[i]);
  }
  FootBox b;
  b.c0 = (int)max(0LL, trunc_ll(div_h(x0, P.res)) - 1);
  b.c1 = (int)min((long long)P.nx - 1, trunc_ll(div_h(x1, P.res)) + 1);
  b.r0 = (int)max(0LL, trunc_ll(div_h(y0, P.res)) - 1);
  b.r1 = (int)min((long long)P.ny - 1, trunc_ll(div_h(y1, P.res)) + 1);
  b.empty = b.c1 < b.c0 || b.r1 < b.r0;
  return b;
}

CW_DEV bool cell_inside(const cw_scene_params& P, int r, int c, double x, double y, double cs,
                        double sn, double fw, double fl) {
  // placement.py:45-51
  double px = ((double)c + 0.5) * P.res - x;
  double py = ((double)r + 0.5) * P.res - y;
  double lx = cs * px + sn * py;
  double ly = -sn * px + cs * py;
  return fabs(lx) <= fw / 2.0 && fabs(ly) <= fl / 2.0;
}

// SAT overlap (placement.py:62-78); corners @ axis is OpenBLAS dgemv = fma(c0, a0, c1*a1).
CW_DEV bool sat_overlap(const double* ax_, const double* ay_, const double* bx_, const double* by_) {
  for (int rect = 0; rect < 2; ++rect) {
    const double* rx = rect ? bx_ : ax_;
    const double* ry = rect ? by_ : ay_;
    for (int i = 0; i < 2; ++i) {
      double ex = rx[i + 1] - rx[i], ey = ry[i + 1] - ry[i];
      double axx = -ey, axy = ex;
      double pamin = 0, pamax = 0, pbmin = 0, pbmax = 0;
      for (int k = 0; k < 4; ++k) {
        double pa = __fma_rn(ax_[k], axx, ay_[k] * axy);
        double pb = __fma_rn(bx_[k], axx, by_[k] * axy);
        pamin = k ? fmin(pamin, pa) : pa; pamax = k ? fmax(pamax, pa) : pa;
        pbmin = k ? fmin(pbmin, pb) : pb; pbmax = k ? fmax(pbmax, pb) : pb;
      }
      if (pamax < pbmin || pbmax < pamin) return false;
    }
  }
  return true;
}

CW_DEV bool region_ok(const cw_scene_params& P, uint8_t zone, int c) {
  if (P.region == 1) return zone <= Z_PLAZA;
  if (P.region == 2) {
    for (int i = 1; i <= 5; ++i) {
      if (i == 3) continue;
      int c0 = (int)((long long)P.nx * i / 6), c1 = (int)((long long)P.nx * (i + 1) / 6);
      if (c >= c0 && c < c1) return true;
    }
    return false;
  }
  return true;
}

// Warp per env.  kStage: the env's zone grid (4 bits per cell, 32 KB at 256^2) lives in
// shared memory for the whole rejection loop (one env per CTA, all 1024 cfg2 envs
// resident at once), so every footprint zone / region test reads shared memory; the
// placed objects' SAT data stay in the L1-cached global scratch.  Without kStage
// (grids whose packed tile does not fit) the zones are read from global memory.
template <bool kStage>
__global__ void __launch_bounds__(kStage ? 32 : 128) k_place(cw_scene_params P, int E, const int32_t* slots,
                                                           const EnvSeeds* __restrict__ seeds,
                                                           cw_scene_buffers B) {
  extern __shared__ __align__(16) unsigned char place_sm[];
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (e >= E) return;
  const int slot = env_slot(slots, e);
  if (B.status[slot] != CW_OK) return;
  const size_t N = (size_t)P.nx * P.ny;
  const uint8_t* Z = B.zones + slot * N;
  const int32_t* A = B.assign + (size_t)slot * P.trows * P.tcols;
  const int8_t* TK = B.tile_kind + (size_t)slot * CW_MAX_TILES;
  double* cache = B.scratch_f64 + (size_t)e * (size_t)max(P.obj_max * 8, (int)N);  // corners
  int32_t* ocat = B.obj_cat + (size_t)slot * P.obj_max;
  double* opose = B.obj_pose + (size_t)slot * P.obj_max * 3;
  uint8_t* zs = place_sm;   // staged zones, 2 cells per byte
  if (kStage) {
    const uint4* Z16 = reinterpret_cast<const uint4*>(Z);   // N % 32 == 0 (checked by the launch)
    for (size_t q = lane; q < N / 16; q += 32) {
      const uint4 v = Z16[q];
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
      uint32_t out[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t o = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) o |= ((w[2 * h + b / 4] >> (8 * (b % 4))) & 15u) << (4 * b);
        out[h] = o;
      }
      reinterpret_cast<uint2*>(zs)[q] = make_uint2(out[0], out[1]);
    }
    __syncwarp();
  }
  auto zone_at = [&](size_t f) -> uint8_t {
    if (kStage) return (uint8_t)((zs[f >> 1] >> ((f & 1) * 4)) & 15u);
    return Z[f];
  };
  Pcg64 rng;
  if (lane == 0) rng = pcg_load(seeds[e].objects);
  int placed = 0;
  bool overflow = false;
  const int count = P.obj_count;
  // One try = (category, x, y, yaw) drawn by lane 0 (placement.py:95-105), then the
  // warp tests it.  Tries are drawn in batches of up to 32 ahead and lane t computes
  // try t's correctly rounded sin/cos (the bulk of a try's latency) for all of them at
  // once.  A try's draws depend on the history only through the category rule (first
  // or second half of the object's attempts); a batch is drawn assuming every try of
  // it fails and stops at the half, so an accepted try (attempts restart at 0) leaves
  // the later tries of the batch drawn exactly as they would have been.  Second-half
  // tries are drawn one at a time.
  const int half = P.attempts / 2;
  int obj = 0, att = 0;
  while (obj < count && !overflow) {
    const int nb = att < half ? min(32, half - att) : 1;
    int my_k = 0;
    double my_x = 0.0, my_y = 0.0, my_yaw = 0.0;
    for (int t = 0; t < nb; ++t) {
      int k = 0;
      double x = 0, y = 0, yaw = 0;
      if (lane == 0) {
        if (att + t < half) k = (int)integers32(rng, (uint64_t)P.n_cat);
        else k = P.small_first[integers32(rng, (uint64_t)min(5, P.n_cat))];
        x = uniform(rng, 0.0, P.nx * P.res);
        y = uniform(rng, 0.0, P.ny * P.res);
        yaw = uniform(rng, 0.0, kTwoPi);
      }
      k = __shfl_sync(0xffffffffu, k, 0);
      x = __shfl_sync(0xffffffffu, x, 0);
      y = __shfl_sync(0xffffffffu, y, 0);
      yaw = __shfl_sync(0xffffffffu, yaw, 0);
      if (lane == t) { my_k = k; my_x = x; my_y = y; my_yaw = yaw; }
    }
    double my_cs, my_sn;
    cr_sincos(my_yaw, &my_sn, &my_cs);   // correctly rounded: matches glibc (np.cos / np.sin) but in its rare misroundings
    for (int j = 0; j < nb && obj < count; ++j) {
      const int k = __shfl_sync(0xffffffffu, my_k, j);
      const double x = __shfl_sync(0xffffffffu, my_x, j), y = __shfl_sync(0xffffffffu, my_y, j);
      const double yaw = __shfl_sync(0xffffffffu, my_yaw, j);
      const double cs = __shfl_sync(0xffffffffu, my_cs, j), sn = __shfl_sync(0xffffffffu, my_sn, j);
      const double fw = P.cat_w[k], fl = P.cat_l[k];
      double cx[4], cy[4];
      bool ok = false;
      do {   // one try (break = rejected)
        footprint_corners(fw, fl, x, y, cs, sn, cx, cy);
        FootBox bb = footprint_box(P, cx, cy);
        if (bb.empty) break;
        const int bw = bb.c1 - bb.c0 + 1, nbx = bw * (bb.r1 - bb.r0 + 1);
        bool bad = false, any = false;
        for (int q = lane; q < nbx; q += 32) {
          int r = bb.r0 + q / bw, c = bb.c0 + q % bw;
          if (!cell_inside(P, r, c, x, y, cs, sn, fw, fl)) continue;
          any = true;
          uint8_t z = zone_at((size_t)r * P.nx + c);
          if (!((P.cat_zones[k] >> z) & 1u) || !region_ok(P, z, c)) bad = true;
        }
        any = __any_sync(0xffffffffu, any);
        bad = __any_sync(0xffffffffu, bad);
        if (!any) {
          // degenerate small footprint: the centre cell (placement.py:54-58)
          long long rc = trunc_ll(y / P.res), cc = trunc_ll(x / P.res);
          if (!(rc >= 0 && rc < P.ny && cc >= 0 && cc < P.nx)) break;
          uint8_t z = zone_at((size_t)rc * P.nx + cc);
          if (!((P.cat_zones[k] >> z) & 1u) || !region_ok(P, z, (int)cc)) break;
        } else if (bad) {
          break;
        }
        {  // stair tile under the pose (placement.py:120-124)
          int tr = min(P.trows - 1, (int)trunc_ll(y / 2.0));
          int tc = min(P.tcols - 1, (int)trunc_ll(x / 2.0));
          int kind = TK[A[tr * P.tcols + tc]];
          if (kind == K_STUP || kind == K_STDOWN) break;
        }
        bool hit = false;
        const double reach = P.cat_reach[k];
        for (int jj = lane; jj < placed; jj += 32) {
          const double* o = cache + (size_t)jj * 8;
          const double ox = opose[jj * 3 + 0], oy = opose[jj * 3 + 1];
          double rr = reach + P.cat_reach[ocat[jj]];
          double dx = x - ox, dy = y - oy;
          if (dx * dx + dy * dy > rr * rr) continue;
          if (sat_overlap(cx, cy, o, o + 4)) hit = true;
        }
        if (__any_sync(0xffffffffu, hit)) break;
        ok = true;
      } while (false);
      if (ok) {
        if (lane == 0) {
          ocat[placed] = k;
          opose[placed * 3 + 0] = x;
          opose[placed * 3 + 1] = y;
          opose[placed * 3 + 2] = yaw;
          double* o = cache + (size_t)placed * 8;
          for (int i = 0; i < 4; ++i) { o[i] = cx[i]; o[4 + i] = cy[i]; }
        }
        __syncwarp();
        ++placed;
        ++obj;
        att = 0;
      } else if (++att >= P.attempts) {
        overflow = true;
        break;
      }
    }
  }
  if (lane == 0) {
    B.obj_n[slot] = placed;
    B.overflow[slot] = overflow;
  }
}

// shared memory of the staged k_place: the packed zones
CW_HD size_t place_stage_bytes(const cw_scene_params& p) {
  const size_t N = (size_t)p.nx * p.ny;
  return (N / 2 + 1 + 15) & ~(size_t)15;
}

// ================================================================= raster
CW_DEV double hash_noise(long long ix, long long iy, uint64_t seed) {
  // terrain.py:264-272
  uint64_t h = ((uint64_t)ix * 0x9E3779B97F4A7C15ull) ^ ((uint64_t)iy * 0xC2B2AE3D27D4EB4Full) ^ seed;
  h ^= h >> 33;
  h *= 0xFF51AFD7ED558CCDull;
  h ^= h >> 33;
  return (double)(h >> 11) / 9007199254740992.0 * 2.0 - 1.0;
}

CW_DEV double elevation_at(double x, double y, int rows, int cols, const int32_t* A,
                           const int8_t* code, const double* tp, uint64_t noise) {
  // terrain.py:294-335
  const double T = 2.0;
  long long tc = clampll(trunc_ll(x / T), 0, cols - 1);
  long long tr = clampll(trunc_ll(y / T), 0, rows - 1);
  double u = fmin(fmax(x / T - (double)tc, 0.0), 1.0);
  double v = fmin(fmax(y / T - (double)tr, 0.0), 1.0);
  int id = A[tr * cols + tc];
  const double* p = tp + id * 4;
  int cd = code[id];
  double e = (1 - u) * (1 - v) * p[0] + u * (1 - v) * p[1] + (1 - u) * v * p[2] + u * v * p[3];
  if (cd == T_STAIR_U) e = u < 0.5 ? p[0] : p[1];
  else if (cd == T_STAIR_V) e = v < 0.5 ? p[0] : p[1];
  else if (cd == T_ROUGH) {
    double taper = fmin(fmax(fmin(u, 1.0 - u) / 0.125, 0.0), 1.0) *
                   fmin(fmax(fmin(v, 1.0 - v) / 0.125, 0.0), 1.0);
    double gx = x / 0.5, gy = y / 0.5;
    long long ix = (long long)floor(gx), iy = (long long)floor(gy);
    double fx = gx - (double)ix, fy = gy - (double)iy;
    double sx = fx * fx * (3.0 - 2.0 * fx);
    double sy = fy * fy * (3.0 - 2.0 * fy);
    double n00 = hash_noise(ix, iy, noise), n10 = hash_noise(ix + 1, iy, noise);
    double n01 = hash_noise(ix, iy + 1, noise), n11 = hash_noise(ix + 1, iy + 1, noise);
    double top = n00 + (n10 - n00) * sx;
    double bot = n01 + (n11 - n01) * sx;
    double bump = top + (bot - top) * sy;
    e = p[0] + p[1] * taper * bump;
  }
  return e;
}

// 4 cells per thread: uchar4 label stores + float4 elevation stores (nx % 4 == 0).
__global__ void __launch_bounds__(256) k_raster(cw_scene_params P, int E, const int32_t* slots,
                                                cw_scene_buffers B) {
  const int e = blockIdx.y;
  const int slot = env_slot(slots, e);
  if (B.status[slot] != CW_OK) return;
  const size_t N = (size_t)P.nx * P.ny;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;  // quad index
  if ((size_t)q * 4 >= N) return;
  const int f0 = q * 4;
  const uint8_t* Z = B.zones + slot * N;
  const int32_t* A = B.assign + (size_t)slot * P.trows * P.tcols;
  const int8_t* cd = B.tile_code + (size_t)slot * CW_MAX_TILES;
  const double* p = B.tile_p + (size_t)slot * CW_MAX_TILES * 4;
  const uint64_t noise = B.noise_seed[slot];
  // zone lookup at the same resolution: rr = min((r+0.5)*res/zone_res, zy-1) == r
  if ((P.nx & 3) == 0 && (N & 3) == 0) {
    // fast path: the 4 cells share a row -> uchar4 label + float4 elevation stores
    const int r = f0 / P.nx, c0 = f0 - r * P.nx;
    const uchar4 zz = *reinterpret_cast<const uchar4*>(Z + f0);
    const uchar4 lb = make_uchar4(zone_to_label(zz.x), zone_to_label(zz.y), zone_to_label(zz.z),
                                  zone_to_label(zz.w));
    *reinterpret_cast<uchar4*>(B.labels + slot * N + f0) = lb;
    const double y = ((double)r + 0.5) * P.res;
    float ev[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double x = ((double)(c0 + k) + 0.5) * P.res;
      ev[k] = (float)elevation_at(x, y, P.trows, P.tcols, A, cd, p, noise);
    }
    *reinterpret_cast<float4*>(B.elev + slot * N + f0) = make_float4(ev[0], ev[1], ev[2], ev[3]);
  } else {
    for (int k = 0; k < 4; ++k) {
      const int f = f0 + k;
      if ((size_t)f >= N) break;
      const int r = f / P.nx, c = f - r * P.nx;
      B.labels[slot * N + f] = zone_to_label(Z[f]);
      const double x = ((double)c + 0.5) * P.res, y = ((double)r + 0.5) * P.res;
      B.elev[slot * N + f] = (float)elevation_at(x, y, P.trows, P.tcols, A, cd, p, noise);
    }
  }
}

// warp per (env, object): footprint cells -> OBSTACLE (occupancy.py:49-51)
__global__ void __launch_bounds__(128) k_footprint(cw_scene_params P, int E, const int32_t* slots,
                                                   cw_scene_buffers B) {
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.y;
  const int slot = env_slot(slots, e);
  if (B.status[slot] != CW_OK) return;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= B.obj_n[slot]) return;
  const size_t N = (size_t)P.nx * P.ny;
  uint8_t* Lb = B.labels + slot * N;
  const int k = B.obj_cat[(size_t)slot * P.obj_max + j];
  const double* pose = B.obj_pose + ((size_t)slot * P.obj_max + j) * 3;
  const double x = pose[0], y = pose[1], yaw = pose[2];
  const double fw = P.cat_w[k], fl = P.cat_l[k];
  double cs, sn;
  cr_sincos(yaw, &sn, &cs);
  double cx[4], cy[4];
  footprint_corners(fw, fl, x, y, cs, sn, cx, cy);
  FootBox bb = footprint_box(P, cx, cy);
  if (bb.empty) return;
  const int bw = bb.c1 - bb.c0 + 1, nb = bw * (bb.r1 - bb.r0 + 1);
  bool any = false;
  for (int q = lane; q < nb; q += 32) {
    int r = bb.r0 + q / bw, c = bb.c0 + q % bw;
    if (cell_inside(P, r, c, x, y, cs, sn, fw, fl)) {
      any = true;
      Lb[(size_t)r * P.nx + c] = L_OBSTACLE;
    }
  }
  any = __any_sync(0xffffffffu, any);
  if (!any && lane == 0) {
    long long rc = trunc_ll(y / P.res), cc = trunc_ll(x / P.res);
    if (rc >= 0 && rc < P.ny && cc >= 0 && cc < P.nx) Lb[rc * P.nx + cc] = L_OBSTACLE;
  }
}

// ================================================================= nearest obstacle (BFS)
constexpr int BFS_NT = 1024;

// Level-synchronous BFS that reproduces the FIFO deque of field.py:579-592:
// a level-(k+1) cell belongs to the earliest-ranked level-k parent that
// reaches it, and the next level is ordered by (parent rank, direction).
// Visited cells (obstacles and every cell already claimed) are a bitmap in shared
// memory: the claim pass issues its atomicMin only towards unvisited neighbours, as
// fire-and-forget reductions, and the winner pass loads the owner word only for them
// (all of a cell's candidates at once).  The FIFO order is unchanged: the owner word is
// still the smallest (frontier position, move) key of the level.
CW_HD size_t nearest_smem_bytes(int nx, int ny) { return (((size_t)nx * ny + 31) / 32) * 4; }

__global__ void __launch_bounds__(BFS_NT) k_nearest(cw_scene_params P, int E, const int32_t* slots,
                                                    cw_scene_buffers B) {
  const int e = blockIdx.x;
  const int slot = env_slot(slots, e);
  if (B.status[slot] != CW_OK) return;
  const int nx = P.nx, ny = P.ny, N = nx * ny;
  const uint8_t* Lb = B.labels + (size_t)slot * N;
  int32_t* near = B.nearest + (size_t)slot * N;
  int32_t* owner = B.scratch_i32 + (size_t)e * SCRATCH_I32_PER_CELL * N + 8 * (size_t)N;
  int32_t* Q = owner + N;
  extern __shared__ uint32_t s_vis[];
  __shared__ int sh[BFS_NT / 32 + 1];
  const int UNSEEN = 0x7fffffff;
  const int lane = threadIdx.x & 31;
  // seed: obstacles in row-major order
  int base = 0;
  for (int f0 = 0; f0 < N; f0 += BFS_NT) {
    int f = f0 + threadIdx.x;
    int ob = f < N && Lb[f] == L_OBSTACLE;
    if (f < N) {
      owner[f] = ob ? -1 : UNSEEN;
      near[f] = ob ? f : -1;
    }
    const unsigned vb = __ballot_sync(0xffffffffu, ob);
    if (lane == 0 && f < N) s_vis[f >> 5] = vb;
    int tot;
    int off = block_excl_scan<BFS_NT>(ob, sh, tot);
    if (ob) Q[base + off] = f;
    base += tot;
  }
  if (threadIdx.x == 0) B.has_obs[slot] = base > 0;
  __syncthreads();
  const int dr[8] = {1, -1, 0, 0, 1, 1, -1, -1};
  const int dc[8] = {0, 0, 1, -1, 1, -1, 1, -1};
  auto vis = [&](int x) { return (s_vis[x >> 5] >> (x & 31)) & 1u; };
  int lo = 0, hi = base;
  while (lo < hi) {
    for (int q = lo + threadIdx.x; q < hi; q += BFS_NT) {
      const int p = Q[q], r = p / nx, c = p - r * nx;
      const int key0 = (q - lo) * 8;
#pragma unroll
      for (int d = 0; d < 8; ++d) {
        const int rr = r + dr[d], cc = c + dc[d];
        if (rr < 0 || rr >= ny || cc < 0 || cc >= nx) continue;
        const int x = rr * nx + cc;
        if (!vis(x)) atomicMin(&owner[x], key0 + d);   // result unused: a reduction
      }
    }
    __syncthreads();
    int out = hi;
    for (int q0 = lo; q0 < hi; q0 += BFS_NT) {
      const int q = q0 + threadIdx.x;
      unsigned win = 0;
      int p = 0, r = 0, c = 0;
      if (q < hi) {
        p = Q[q]; r = p / nx; c = p - r * nx;
        const int key0 = (q - lo) * 8;
        int ow[8];
#pragma unroll
        for (int d = 0; d < 8; ++d) {   // the candidates' owner words, loaded together
          const int rr = r + dr[d], cc = c + dc[d];
          const bool in = rr >= 0 && rr < ny && cc >= 0 && cc < nx && !vis(rr * nx + cc);
          ow[d] = in ? ((volatile int32_t*)owner)[rr * nx + cc] : -1;
        }
#pragma unroll
        for (int d = 0; d < 8; ++d)
          if (ow[d] == key0 + d) win |= 1u << d;
      }
      int tot;
      int off = block_excl_scan<BFS_NT>(__popc(win), sh, tot);   // (barrier: every read above is done)
      if (win) {
        int src = near[p];
        int k = 0;
        for (int d = 0; d < 8; ++d) {
          if (!((win >> d) & 1u)) continue;
          int x = (r + dr[d]) * nx + (c + dc[d]);
          Q[out + off + k++] = x;
          near[x] = src;
          owner[x] = -1;
          atomicOr(&s_vis[x >> 5], 1u << (x & 31));
        }
      }
      out += tot;
    }
    __syncthreads();
    lo = hi;
    hi = out;
  }
}

// ================================================================= walkable list + A* move table
// moves[f] bit d: move d of paths.py:75 (N S W E, NW NE SW SE) is legal from cell
// f -- target in bounds and passable, diagonals also need both orthogonal cells
// passable (paths.py:70-72).  One byte load replaces the per-neighbour tests.
__global__ void __launch_bounds__(1024) k_walk(cw_scene_params P, int E, const int32_t* slots,
                                               cw_scene_buffers B) {
  const int e = blockIdx.x;
  const int slot = env_slot(slots, e);
  if (B.status[slot] != CW_OK) return;
  const int nx = P.nx, ny = P.ny, N = nx * ny;
  const uint8_t* Lb = B.labels + (size_t)slot * N;
  int32_t* W = B.walk + (size_t)slot * N;
  uint8_t* MV = B.moves + (size_t)slot * N;
  __shared__ int sh[1024 / 32 + 1];
  int base = 0;
  for (int f0 = 0; f0 < N; f0 += 1024) {
    int f = f0 + threadIdx.x;
    uint8_t lb = f < N ? Lb[f] : L_OBSTACLE;
    int wk = f < N && lb == L_WALKABLE;
    if (f < N) {
      const int r = f / nx, c = f - r * nx;
      auto ps = [&](int rr, int cc) {
        return rr >= 0 && rr < ny && cc >= 0 && cc < nx && Lb[rr * nx + cc] != L_OBSTACLE;
      };
      const bool n = ps(r - 1, c), s = ps(r + 1, c), w = ps(r, c - 1), ea = ps(r, c + 1);
      const unsigned mv = (unsigned)n | ((unsigned)s << 1) | ((unsigned)w << 2) | ((unsigned)ea << 3) |
                          ((unsigned)(n && w && ps(r - 1, c - 1)) << 4) |
                          ((unsigned)(n && ea && ps(r - 1, c + 1)) << 5) |
                          ((unsigned)(s && w && ps(r + 1, c - 1)) << 6) |
                          ((unsigned)(s && ea && ps(r + 1, c + 1)) << 7);
      MV[f] = (uint8_t)mv;
    }
    int tot;
    int off = block_excl_scan<1024>(wk, sh, tot);
    if (wk) W[base + off] = f;
    base += tot;
  }
  if (threadIdx.x == 0) B.walk_n[slot] = base;
}

// 4-connected components of passable cells.  The A* move set (paths.py:14-19,
// 70-72: diagonals only when both orthogonal cells are passable) connects
// exactly the 4-connected components, so reach[start] != reach[goal] <=> the
// search returns None.
__global__ void __launch_bounds__(1024) k_reach(cw_scene_params P, int E, const int32_t* slots,
                                                cw_scene_buffers B) {
  const int e = blockIdx.x;
  const int slot = env_slot(slots, e);
  if (B.status[slot] != CW_OK) return;
  const int nx = P.nx, N = nx * P.ny;
  const uint8_t* Lb = B.labels + (size_t)slot * N;
  int32_t* R = B.reach + (size_t)slot * N;
  extern __shared__ uint32_t reach_bm[];   // bmcomp_smem_bytes(nx, ny) (0: union-find)
  components<1024, false>(R, nx, P.ny, [&](int f) { return Lb[f] != L_OBSTACLE; },
                          bmcomp_smem_bytes(nx, P.ny) ? reach_bm : nullptr);
}

static void launch_reach(const cw_scene_params& p, int E, const int32_t* slots, const cw_scene_buffers& b,
                         cudaStream_t st) {
  const size_t bm = bmcomp_smem_bytes(p.nx, p.ny);
  if (bm > 48 * 1024) cudaFuncSetAttribute(k_reach, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bm);
  k_reach<<<E, 1024, bm, st>>>(p, E, slots, b);
}

// ================================================================= spawn + routes
constexpr int SP_NT = 256;
__device__ __constant__ double kMaxSpeed[3] = {2.0, 5.0, 4.0};     // crowd/types.py:15-19
__device__ __constant__ double kPrefLo[3] = {0.8, 2.0, 1.5};       // types.py:22-26
__device__ __constant__ double kPrefHi[3] = {1.4, 4.0, 3.0};
__device__ __constant__ double kRadius[3] = {0.3, 0.45, 0.4};      // types.py:28-32

CW_DEV bool spawn_region_ok(const cw_scene_params& P, int c) {
  if (P.spawn_region != 1) return true;
  for (int i = 2; i <= 5; i += 3) {
    int c0 = (int)((long long)P.nx * i / 6), c1 = (int)((long long)P.nx * (i + 1) / 6);
    if (c >= c0 && c < c1) return true;
  }
  return false;
}

// candidate cell of sample_routes (routes.py:50-56): Walkable (| Roadway for vehicle
// kinds), the Traverse strip mask (batch.py:174-177) and a caller region mask
CW_DEV bool route_ok(const cw_scene_params& P, const cw_scene_buffers& B, int slot, const uint8_t* Lb, int f,
                     int N) {
  const uint8_t l = Lb[f];
  if (!(l == L_WALKABLE || (P.route_roadway && l == L_ROADWAY))) return false;
  if (P.spawn_region == 1 && !spawn_region_ok(P, f % P.nx)) return false;
  return !B.region || B.region[(size_t)slot * N + f] != 0;
}

// numpy Generator.permutation(n) = Fisher-Yates from the top over a pure next32
// stream (random_interval, masked rejection).  Only the first few entries of the
// final order are consumed (routes.py:69-83), so the kernel (1) generates the
// 32-bit stream with PCG64 jump-ahead across warp 0 while lane 0 runs the serial
// accept/reject scan, recording the swap partner j_i of every step i; (2) links
// the steps by partner (lists of i with j_i == p); (3) resolves final[k] for a
// batch of k in parallel by walking the swap history backwards:
//   final[k] = V(j_k, k+1) (k >= 1), final[0] = V(0, 1), and for p < t
//   V(p, t) = p if no step i >= t has j_i == p, else V(i*, i*+1) with i* the
//   smallest such step (the value at i* just before step i* swaps into p).
constexpr int ORD_BATCH = SP_NT;

// k_spawn dynamic shared memory: accepted starts (2 x A doubles) + the candidate bitmap
CW_HD size_t spawn_smem_bytes(int A, int nx, int ny) {
  return (size_t)A * 2 * sizeof(double) + (((size_t)nx * ny + 31) / 32) * 4 + bmcomp_smem_bytes(nx, ny);
}

CW_DEV int resolve_final(int k, const int32_t* jj, const int32_t* head, const int32_t* nxt) {
  int p, t;
  if (k >= 1) { p = jj[k]; t = k + 1; }
  else { p = 0; t = 1; }
  while (true) {
    int best = 0x7fffffff;
    for (int i = head[p]; i >= 0; i = nxt[i])
      if (i >= t && i < best) best = i;
    if (best == 0x7fffffff) return p;
    p = best;
    t = best + 1;
  }
}

// route_seeds == nullptr: spawn_agents (step.py:37-63: kinds, routes seed, speeds);
// else sample_routes(occ, peds, route_seeds[e], ..., max_radius) alone (routes.py:35).
__global__ void __launch_bounds__(SP_NT) k_spawn(cw_scene_params P, int E, const int32_t* slots,
                                                 const EnvSeeds* __restrict__ seeds,
                                                 cw_scene_buffers B, const uint64_t* __restrict__ route_seeds) {
  const int e = blockIdx.x;
  const int slot = env_slot(slots, e);
  const int A = P.peds;
  if (A == 0 || B.status[slot] != CW_OK) return;
  const int nx = P.nx, ny = P.ny, N = nx * ny;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint8_t* Lb = B.labels + (size_t)slot * N;
  int32_t* comp = B.scratch_i32 + (size_t)e * SCRATCH_I32_PER_CELL * N;
  int32_t* cand = comp + N;       // candidate flat indices (row-major)
  int32_t* jj = cand + N;         // swap partner of Fisher-Yates step i
  int32_t* head = jj + N;         // per position: list of steps i with jj[i] == position
  int32_t* nxt = head + N;
  int32_t* csize = nxt + N;       // per component root: number of candidates
  const int NW32 = (N + 31) / 32;
  uint32_t* cbits = reinterpret_cast<uint32_t*>(csize + N);   // bitmap of one component
  int32_t* cpre = reinterpret_cast<int32_t*>(cbits + NW32);    // exclusive popcount prefix
  int32_t* disk = csize + 2 * (size_t)N;                       // row-major disk cells (<= N)
  __shared__ int sh[SP_NT / 32 + 1];
  __shared__ int s_n, s_idx, s_rank, s_j, s_acc, s_k, s_ordn;
  __shared__ unsigned long long s_seed;
  __shared__ double s_maxr;
  __shared__ uint32_t s_buf[64];
  __shared__ int s_ord[ORD_BATCH];
  __shared__ Pcg64Raw s_rng;
  extern __shared__ __align__(16) unsigned char sp_smem[];
  double* stx = reinterpret_cast<double*>(sp_smem);  // accepted starts (A)
  double* sty = stx + A;
  uint32_t* s_ok = reinterpret_cast<uint32_t*>(sty + A);   // route_ok bitmap (NW32 words)
  int8_t* kind_out = B.sp_kind + (size_t)slot * A;
  double* pref_out = B.sp_pref + (size_t)slot * A;
  if (threadIdx.x == 0 && route_seeds) {
    s_seed = route_seeds[e];
    s_maxr = P.route_max_radius;
  } else if (threadIdx.x == 0) {
    // step.py:41-61 (the spawn stream is independent of the routes stream)
    Pcg64 rng = pcg_load(seeds[e].spawn);
    double maxr = 0.0;
    for (int a = 0; a < A; ++a) {
      double u = next_double(rng);
      int k = u < 0.7 ? 0 : (u < 0.9 ? 1 : 2);
      kind_out[a] = (int8_t)k;
      maxr = a ? fmax(maxr, kRadius[k]) : kRadius[k];
    }
    s_seed = integers_2p63(rng);
    for (int a = 0; a < A; ++a) {
      int k = kind_out[a];
      pref_out[a] = uniform(rng, kPrefLo[k], kPrefHi[k]);
    }
    s_maxr = maxr;
  }
  // candidates: WALKABLE (& region) cells, row-major (routes.py:46-56)
  int base = 0;
  for (int f0 = 0; f0 < N; f0 += SP_NT) {
    int f = f0 + threadIdx.x;
    int ok = f < N && route_ok(P, B, slot, Lb, f, N);
    if (f < N) { comp[f] = ok ? f : -1; head[f] = -1; csize[f] = 0; }
    const unsigned okb = __ballot_sync(0xffffffffu, ok);
    if (lane == 0 && f < N) s_ok[f >> 5] = okb;
    int tot;
    int off = block_excl_scan<SP_NT>(ok, sh, tot);
    if (ok) cand[base + off] = f;
    base += tot;
  }
  if (threadIdx.x == 0) s_n = base;
  __syncthreads();
  const int n = s_n;
  if (n < A) {
    if (threadIdx.x == 0) B.status[slot] = CW_E_NOROUTE;
    return;
  }
  // 8-connected components (routes.py:14-32); only label equality is used
  // downstream (routes.py:62, 74), so any labelling works.
  components<SP_NT, true>(comp, nx, ny, [&](int f) { return ((s_ok[f >> 5] >> (f & 31)) & 1u) != 0u; },
                          bmcomp_smem_bytes(nx, ny) ? s_ok + NW32 : nullptr);
  // component sizes: one atomic per (warp, component) -- nearly every candidate is
  // in the same component, so per-candidate atomics serialise on one address
  for (int q0 = 0; q0 < n; q0 += SP_NT) {
    const int q = q0 + threadIdx.x;
    const int cq = q < n ? comp[cand[q]] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, cq);
    if (cq >= 0 && lane == __ffs(peers) - 1) atomicAdd(&csize[cq], __popc(peers));
  }
  __syncthreads();
  // ---- permutation draws (warp 0): stream generation + warp-speculative
  // accept/reject.  Within a window where i stays above mask>>1 the mask is
  // fixed, so value t (counting from the window start) is accepted iff
  // (v & mask) <= i - t provided all earlier ones were; a ballot finds the
  // first rejection, everything before it is accepted.
  if (wid == 0) {
    const Pcg64 base_rng = pcg_seed(s_seed);
    u128 m1, p1, m32, p32;
    pcg_jump_coeffs((u128)(lane + 1), m1, p1, base_rng.inc);
    pcg_jump_coeffs((u128)32, m32, p32, base_rng.inc);
    u128 st = m1 * base_rng.state + p1;   // S_{lane+1}: produces output #lane
    long long consumed = 0;               // 32-bit values consumed before this round
    int i = n - 1;
    auto mask_of = [](int v) {
      uint32_t m = (uint32_t)v;
      m |= m >> 1; m |= m >> 2; m |= m >> 4; m |= m >> 8; m |= m >> 16;
      return m;
    };
    uint32_t mask = i > 0 ? mask_of(i) : 0u;
    int used_last = 0;
    while (i > 0) {
      uint64_t out = xsl_rr(st);
      st = m32 * st + p32;
      s_buf[2 * lane] = (uint32_t)out;
      s_buf[2 * lane + 1] = (uint32_t)(out >> 32);
      __syncwarp();
      int used = 0;
      for (int half = 0; half < 2 && i > 0; ++half) {
        const uint32_t v = s_buf[32 * half + lane];
        int pos = 0;
        while (pos < 32 && i > 0) {
          // classify against every possible acceptance count a_t in [0, t]:
          // sure accept if (v&mask) <= i - t, sure reject if (v&mask) > i;
          // the first undecided value is then resolved exactly.
          const int t = lane - pos;
          const bool in = lane >= pos;
          const uint32_t vm = v & mask;
          const bool bound = in && (i - t > (int)(mask >> 1)) && (i - t >= 1);
          const bool sure_acc = bound && vm <= (uint32_t)(i - t);
          const bool sure_rej = bound && vm > (uint32_t)i;
          const unsigned qm = __ballot_sync(0xffffffffu, in && !(sure_acc || sure_rej));
          const int f = qm ? __ffs(qm) - 1 : 32;
          const unsigned am = __ballot_sync(0xffffffffu, sure_acc);
          const unsigned range = (f >= 32 ? 0xffffffffu : ((1u << f) - 1u)) & ~((1u << pos) - 1u);
          const unsigned acc_in = am & range;
          if (in && lane < f && sure_acc) {
            const int a_t = __popc(acc_in & ((1u << lane) - 1u));
            jj[i - a_t] = (int32_t)vm;
          }
          i -= __popc(acc_in);
          pos = f;
          if (i > 0 && (uint32_t)i <= (mask >> 1)) mask = mask_of(i);
          if (f < 32 && i > 0) {
            const uint32_t vf = __shfl_sync(0xffffffffu, v, f);
            if ((vf & mask) <= (uint32_t)i) {
              if (lane == 0) jj[i] = (int32_t)(vf & mask);
              --i;
              if (i > 0 && (uint32_t)i <= (mask >> 1)) mask = mask_of(i);
            }
            pos = f + 1;
          }
        }
        used = 32 * half + pos;
      }
      used_last = used;
      if (i > 0) consumed += 64;
      __syncwarp();
    }
    if (lane == 0) {
      // routes stream position right after the shuffle
      const long long q = (n > 1) ? consumed + used_last : 0;
      Pcg64 r;
      r.inc = base_rng.inc;
      u128 mm, pp;
      const long long u = q >> 1;
      if ((q & 1) == 0) {
        pcg_jump_coeffs((u128)u, mm, pp, base_rng.inc);
        r.state = mm * base_rng.state + pp;
        r.has32 = 0;
        r.buf32 = 0;
      } else {
        pcg_jump_coeffs((u128)(u + 1), mm, pp, base_rng.inc);
        r.state = mm * base_rng.state + pp;
        r.has32 = 1;
        r.buf32 = (uint32_t)(xsl_rr(r.state) >> 32);
      }
      pcg_store(s_rng, r);
    }
  }
  __syncthreads();
  // ---- link steps by partner position
  for (int i0 = 1 + threadIdx.x; i0 < n; i0 += 4 * SP_NT) {   // four atomics in flight
    int jv[4], rv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) jv[u] = i0 + u * SP_NT < n ? jj[i0 + u * SP_NT] : -1;
#pragma unroll
    for (int u = 0; u < 4; ++u) rv[u] = jv[u] >= 0 ? atomicExch(&head[jv[u]], i0 + u * SP_NT) : 0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (jv[u] >= 0) nxt[i0 + u * SP_NT] = rv[u];
  }
  if (threadIdx.x == 0) {
    s_acc = 0;
    s_k = 0;
    s_ordn = 0;
  }
  __syncthreads();
  const double res = P.res;
  const double sep = 2.0 * s_maxr;
  const double sep2 = sep * sep;
  double* out_pos = B.sp_pos + (size_t)slot * A * 2;
  double* out_goal = B.sp_goal + (size_t)slot * A * 2;
  // goal candidates of a start = cells of its component minus the disk of cells
  // closer than sep (routes.py:74-76); the rank-th one in row-major order is found
  // through a bitmap of the component with popcount prefixes and the (row-major)
  // list of disk cells -- O(disk + log N) per route instead of a pass over N.
  const int R = (int)ceil(sep / res) + 1;
  const int bw = 2 * R + 1;
  __shared__ int s_ndisk, s_bmc;
  if (threadIdx.x == 0) s_bmc = -1;
  while (true) {
    __syncthreads();
    if (s_acc >= A || s_k >= n) break;
    if (s_k >= s_ordn) {  // resolve the next batch of the final permutation
      const int k = s_ordn + threadIdx.x;
      if (k < n) s_ord[threadIdx.x] = resolve_final(k, jj, head, nxt);
      __syncthreads();
      if (threadIdx.x == 0) s_ordn += ORD_BATCH;
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      s_idx = s_ord[s_k - (s_ordn - ORD_BATCH)];
      s_k += 1;
    }
    __syncthreads();
    const int fs = cand[s_idx];
    const int sr = fs / nx, sc = fs - sr * nx;
    const double sx = ((double)sc + 0.5) * res, sy = ((double)sr + 0.5) * res;
    int close = 0;
    for (int a = threadIdx.x; a < s_acc; a += SP_NT) {
      double dx = sx - stx[a], dy = sy - sty[a];
      if (dx * dx + dy * dy < sep2) close = 1;
    }
    if (__syncthreads_or(close)) continue;
    const int cs = comp[fs];
    // disk cells of the component (not "far"), row-major
    int nd = 0;
    for (int b0 = 0; b0 < bw * bw; b0 += SP_NT) {
      const int b = b0 + threadIdx.x;
      int in = 0, f = -1;
      if (b < bw * bw) {
        const int r = sr - R + b / bw, c = sc - R + b % bw;
        if (r >= 0 && r < ny && c >= 0 && c < nx) {
          f = r * nx + c;
          if (comp[f] == cs) {
            double dx = ((double)c + 0.5) * res - sx, dy = ((double)r + 0.5) * res - sy;
            in = !(dx * dx + dy * dy >= sep2);
          }
        }
      }
      int tot;
      const int off = block_excl_scan<SP_NT>(in, sh, tot);
      if (in) disk[nd + off] = f;
      nd += tot;
    }
    __syncthreads();
    const int total = csize[cs] - nd;
    if (total == 0) continue;
    if (threadIdx.x == 0) {
      Pcg64 rr = pcg_load(s_rng);
      s_rank = (int)integers32(rr, (uint64_t)total);
      pcg_store(s_rng, rr);
      s_ndisk = nd;
    }
    if (s_bmc != cs) {  // bitmap + prefix of component cs
      for (int f0 = 0; f0 < NW32 * 32; f0 += SP_NT) {
        const int f = f0 + threadIdx.x;
        const unsigned bits = __ballot_sync(0xffffffffu, f < N && comp[f] == cs);
        if (lane == 0 && (f >> 5) < NW32) cbits[f >> 5] = bits;
      }
      __syncthreads();
      int base_w = 0;
      for (int w0 = 0; w0 < NW32; w0 += SP_NT) {
        const int w = w0 + threadIdx.x;
        const int c = w < NW32 ? __popc(cbits[w]) : 0;
        int tot;
        const int off = block_excl_scan<SP_NT>(c, sh, tot);
        if (w < NW32) cpre[w] = base_w + off;
        base_w += tot;
      }
      if (threadIdx.x == 0) { cpre[NW32] = base_w; s_bmc = cs; }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int rank = s_rank;
      const int ndisk = s_ndisk;
      int m = 0, cell = -1;
      for (int it = 0; it <= ndisk + 1; ++it) {
        // cell = (rank + m)-th set bit of the component bitmap
        const int k = rank + m;
        int lo = 0, hi = NW32 - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (cpre[mid] <= k) lo = mid; else hi = mid - 1;
        }
        uint32_t w = cbits[lo];
        int kk = k - cpre[lo];
        while (kk-- > 0) w &= w - 1;
        cell = lo * 32 + (__ffs(w) - 1);
        int m2 = 0;
        for (int d = 0; d < ndisk; ++d) m2 += disk[d] <= cell;
        if (m2 == m) break;
        m = m2;
      }
      s_j = cell;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int a = s_acc;
      int fj = s_j;
      stx[a] = sx;
      sty[a] = sy;
      out_pos[a * 2] = sx;
      out_pos[a * 2 + 1] = sy;
      out_goal[a * 2] = ((double)(fj % nx) + 0.5) * res;
      out_goal[a * 2 + 1] = ((double)(fj / nx) + 0.5) * res;
      s_acc = a + 1;
    }
  }
  if (threadIdx.x == 0 && s_acc < A) B.status[slot] = CW_E_NOROUTE;
}


// connected_components (routes.py:14-32): the reference numbers components in the
// order of their first cell in row-major order; the union-find root is the
// component's smallest flat index, so id = rank of the root among the roots.
__global__ void __launch_bounds__(1024) k_components(int nx, int ny, const uint8_t* __restrict__ ok,
                                                     int32_t* __restrict__ comp, int32_t* __restrict__ rank) {
  const int e = blockIdx.x;
  const int N = nx * ny;
  const uint8_t* okb = ok + (size_t)e * N;
  int32_t* par = comp + (size_t)e * N;
  int32_t* rk = rank + (size_t)e * N;
  extern __shared__ uint32_t comp_bm[];   // bmcomp_smem_bytes(nx, ny) (0: union-find)
  components<1024, true>(par, nx, ny, [&](int f) { return okb[f] != 0; },
                         bmcomp_smem_bytes(nx, ny) ? comp_bm : nullptr);
  __shared__ int sh[1024 / 32 + 1];
  int base = 0;
  for (int f0 = 0; f0 < N; f0 += 1024) {
    const int f = f0 + threadIdx.x;
    const int root = f < N && par[f] == f;
    int tot;
    const int off = block_excl_scan<1024>(root, sh, tot);
    if (root) rk[f] = base + off;
    base += tot;
  }
  __syncthreads();
  for (int f = threadIdx.x; f < N; f += 1024) {
    const int r = par[f];
    par[f] = r >= 0 ? rk[r] : -1;
  }
}

// rasterize_occupancy at any resolution (occupancy.py:28-57): labels from the zone
// grid at (row, col) = min(((i + 0.5) res) / zone_res, zone_n - 1) (truncated),
// elevation at cell centres; k_footprint then marks the objects.
__global__ void __launch_bounds__(256) k_raster_res(cw_scene_params P, int E, const int32_t* slots, int zx, int zy,
                                                    double zone_res, cw_scene_buffers B) {
  const int e = blockIdx.y;
  const int slot = env_slot(slots, e);
  if (B.status[slot] != CW_OK) return;
  const size_t N = (size_t)P.nx * P.ny;
  const size_t f = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= N) return;
  const int r = (int)(f / P.nx), c = (int)(f - (size_t)r * P.nx);
  const long long zr = (long long)fmin(((double)r + 0.5) * P.res / zone_res, (double)(zy - 1));
  const long long zc = (long long)fmin(((double)c + 0.5) * P.res / zone_res, (double)(zx - 1));
  B.labels[(size_t)slot * N + f] = zone_to_label(B.zones[(size_t)slot * zx * zy + zr * zx + zc]);
  const int32_t* A = B.assign + (size_t)slot * P.trows * P.tcols;
  const int8_t* cd = B.tile_code + (size_t)slot * CW_MAX_TILES;
  const double* tp = B.tile_p + (size_t)slot * CW_MAX_TILES * 4;
  const double x = ((double)c + 0.5) * P.res, y = ((double)r + 0.5) * P.res;
  B.elev[(size_t)slot * N + f] = (float)elevation_at(x, y, P.trows, P.tcols, A, cd, tp, B.noise_seed[slot]);
}


// trig probe (parity tooling): the device sin/cos the sampling kernels can use
__global__ void k_trig_probe(int n, const double* __restrict__ x, double* __restrict__ s, double* __restrict__ c,
                             int mode) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (mode == 1) cr_sincos(x[i], s + i, c + i);
  else sincos(x[i], s + i, c + i);
}

struct SideStreams {
  int dev = -1;
  cudaStream_t s[3];
  cudaEvent_t fork, join[3];
};

static SideStreams& side_streams() {
  static SideStreams g[16];
  int d = 0;
  cudaGetDevice(&d);
  SideStreams& S = g[d & 15];
  if (S.dev != d) {
    for (int k = 0; k < 3; ++k) {
      cudaStreamCreateWithFlags(&S.s[k], cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&S.join[k], cudaEventDisableTiming);
    }
    cudaEventCreateWithFlags(&S.fork, cudaEventDisableTiming);
    S.dev = d;
  }
  return S;
}

struct RouteJob {   // cw_sample_scenes_routes: the route anchors, forked off the labels
  double* routes;
  int32_t* n_routes;
  void* scratch;
  int chunk;
};

}  // namespace cw

// ================================================================= C ABI
extern "C" {

size_t cw_scene_seed_scratch_bytes(int E) { return (size_t)E * sizeof(cw::EnvSeeds); }

// Sample E scenes (one per scene_seed) end to end on `stream`:
// zones -> terrain -> placement -> raster -> nearest-obstacle BFS -> walk list -> spawn.
// Rows are written at slots[e] (slots may be NULL = identity).  Returns 0 or a
// cudaError_t; per-env failures are reported in B->status.
// grid generation of the rows just written (cw_scene_buffers.epoch)
__global__ void k_bump_epoch(int E, const int32_t* slots, int32_t* epoch) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < E) epoch[slots ? slots[e] : e] += 1;
}

static int sample_impl(const cw_scene_params* P, int E, const uint64_t* scene_seeds, const uint64_t* crowd_seeds,
                       const int32_t* slots, void* seed_scratch, const cw_scene_buffers* B, const cw::RouteJob* rj,
                       void* stream) {
  using namespace cw;
  if (E <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  EnvSeeds* S = (EnvSeeds*)seed_scratch;
  const cw_scene_params p = *P;
  const cw_scene_buffers b = *B;
  k_seeds<<<(E + 127) / 128, 128, 0, st>>>(E, scene_seeds, crowd_seeds, S);
  if (p.layout == 1) k_zones_blk<<<E, 512, 0, st>>>(p, E, slots, S, b);
  else k_zones<<<E, 256, 0, st>>>(p, E, slots, S, b);
  // one warp per env; up to TER_WARPS lattices per CTA (large lattices: fewer, <= 227 KB)
  const size_t per = terrain_warp_smem(p.trows * p.tcols);
  const int wpc = (int)std::max<size_t>(1, std::min<size_t>(TER_WARPS, (227u * 1024u) / per));
  if (per > 227u * 1024u) return (int)cudaErrorInvalidValue;
  const size_t tsm = per * wpc;
  cudaFuncSetAttribute(k_terrain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);
  k_terrain<<<(E + wpc - 1) / wpc, wpc * 32, tsm, st>>>(p, E, slots, S, b);
  {
    const size_t psm = place_stage_bytes(p);
    const size_t N = (size_t)p.nx * p.ny;
    if (psm <= 200u * 1024u && N % 32 == 0) {
      cudaFuncSetAttribute(k_place<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm);
      k_place<true><<<E, 32, psm, st>>>(p, E, slots, S, b);
    } else {
      k_place<false><<<(E + 3) / 4, 128, 0, st>>>(p, E, slots, S, b);
    }
  }
  const int quads = (p.nx * p.ny + 3) / 4;
  k_raster<<<dim3((quads + 255) / 256, E), 256, 0, st>>>(p, E, slots, b);
  if (p.obj_max > 0) k_footprint<<<dim3((p.obj_max + 3) / 4, E), 128, 0, st>>>(p, E, slots, b);
  // the label consumers are independent: BFS, components / walk list and the route
  // anchors run on side streams joined back before returning (fork/join keeps
  // stream order)
  SideStreams& ss = side_streams();
  const int nside = rj ? 3 : 2;
  cudaEventRecord(ss.fork, st);
  for (int k = 0; k < nside; ++k) cudaStreamWaitEvent(ss.s[k], ss.fork, 0);
  if (rj) cw_route_anchors(P, E, scene_seeds, slots, B, rj->routes, rj->n_routes, rj->scratch, rj->chunk, ss.s[2]);
  {
    const size_t nsm = nearest_smem_bytes(p.nx, p.ny);
    if (nsm > 32 * 1024) cudaFuncSetAttribute(k_nearest, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)nsm);
    k_nearest<<<E, BFS_NT, nsm, ss.s[0]>>>(p, E, slots, b);
  }
  k_walk<<<E, 1024, 0, ss.s[1]>>>(p, E, slots, b);
  launch_reach(p, E, slots, b, ss.s[1]);
  if (p.peds > 0) {
    size_t sm = spawn_smem_bytes(p.peds, p.nx, p.ny);
    if (sm > 32 * 1024) cudaFuncSetAttribute(k_spawn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_spawn<<<E, SP_NT, sm, st>>>(p, E, slots, S, b, nullptr);
  }
  for (int k = 0; k < nside; ++k) {
    cudaEventRecord(ss.join[k], ss.s[k]);
    cudaStreamWaitEvent(st, ss.join[k], 0);
  }
  if (b.epoch) k_bump_epoch<<<(E + 255) / 256, 256, 0, st>>>(E, slots, b.epoch);   // after every grid write
  return (int)cudaGetLastError();
}

// Sample E scenes (one per scene_seed) end to end on `stream`:
// zones -> terrain -> placement -> raster -> nearest-obstacle BFS -> walk list -> spawn.
// Rows are written at slots[e] (slots may be NULL = identity).  Returns 0 or a
// cudaError_t; per-env failures are reported in B->status.
int cw_sample_scenes(const cw_scene_params* P, int E, const uint64_t* scene_seeds,
                     const uint64_t* crowd_seeds, const int32_t* slots, void* seed_scratch,
                     const cw_scene_buffers* B, void* stream) {
  return sample_impl(P, E, scene_seeds, crowd_seeds, slots, seed_scratch, B, nullptr, stream);
}

// cw_sample_scenes + cw_route_anchors in one pipeline: the route anchors only read the
// labels, so they run on a side stream beside the BFS, walk list and spawn.
int cw_sample_scenes_routes(const cw_scene_params* P, int E, const uint64_t* scene_seeds,
                            const uint64_t* crowd_seeds, const int32_t* slots, void* seed_scratch,
                            const cw_scene_buffers* B, double* routes, int32_t* n_routes, void* route_scratch,
                            int chunk, void* stream) {
  const cw::RouteJob rj{routes, n_routes, route_scratch, chunk};
  return sample_impl(P, E, scene_seeds, crowd_seeds, slots, seed_scratch, B, &rj, stream);
}

// spawn_agents(occupancy, count, seed) for caller-supplied labels (step.py:37-63).
int cw_spawn_agents(const cw_scene_params* P, int E, const uint64_t* crowd_seeds,
                    const int32_t* slots, void* seed_scratch, const cw_scene_buffers* B,
                    void* stream) {
  using namespace cw;
  if (E <= 0 || P->peds <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  EnvSeeds* S = (EnvSeeds*)seed_scratch;
  k_seeds<<<(E + 127) / 128, 128, 0, st>>>(E, crowd_seeds, crowd_seeds, S);
  size_t sm = spawn_smem_bytes(P->peds, P->nx, P->ny);
  if (sm > 32 * 1024) cudaFuncSetAttribute(k_spawn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_spawn<<<E, SP_NT, sm, st>>>(*P, E, slots, S, *B, nullptr);
  return (int)cudaGetLastError();
}


// sample_routes(occupancy, count, seed, kind, region_mask, max_radius) (routes.py:35-87)
// for rows slots[e] of buffers->labels: params->peds routes, route_roadway for
// vehicle kinds, route_max_radius the separation radius, buffers->region an optional
// (E, ny*nx) u8 mask; starts / goals in sp_pos / sp_goal, NoRouteAvailable in status.
int cw_sample_routes(const cw_scene_params* P, int E, const uint64_t* route_seeds, const int32_t* slots,
                     void* seed_scratch, const cw_scene_buffers* B, void* stream) {
  using namespace cw;
  if (E <= 0 || P->peds <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  EnvSeeds* S = (EnvSeeds*)seed_scratch;
  size_t sm = spawn_smem_bytes(P->peds, P->nx, P->ny);
  if (sm > 32 * 1024) cudaFuncSetAttribute(k_spawn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_spawn<<<E, SP_NT, sm, st>>>(*P, E, slots, S, *B, route_seeds);
  return (int)cudaGetLastError();
}

// connected_components(ok) (routes.py:14-32) for E grids ok (E, ny*nx) u8 -> comp
// (E, ny*nx) int32 (-1 where not ok); rank_scratch (E, ny*nx) int32.
int cw_connected_components(int nx, int ny, int E, const uint8_t* ok, int32_t* comp, int32_t* rank_scratch,
                            void* stream) {
  if (E <= 0 || nx <= 0 || ny <= 0) return 0;
  const size_t bm = cw::bmcomp_smem_bytes(nx, ny);
  if (bm > 48 * 1024) cudaFuncSetAttribute(cw::k_components, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bm);
  cw::k_components<<<E, 1024, bm, (cudaStream_t)stream>>>(nx, ny, ok, comp, rank_scratch);
  return (int)cudaGetLastError();
}

// rasterize_occupancy(scene, resolution) (occupancy.py:28-57) at params->res /
// nx / ny for rows slots[e]: buffers->zones holds the (zone_ny, zone_nx) zone grid
// at zone_res, assign / tile_code / tile_p / noise_seed the terrain, obj_* the
// objects; writes labels and elev (ny*nx) of the row; status must be zero.
int cw_rasterize(const cw_scene_params* P, int E, const int32_t* slots, int zone_nx, int zone_ny,
                 double zone_res, const cw_scene_buffers* B, void* stream) {
  using namespace cw;
  if (E <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t N = (size_t)P->nx * P->ny;
  k_raster_res<<<dim3((unsigned)((N + 255) / 256), E), 256, 0, st>>>(*P, E, slots, zone_nx, zone_ny, zone_res, *B);
  if (P->obj_max > 0) k_footprint<<<dim3((P->obj_max + 3) / 4, E), 128, 0, st>>>(*P, E, slots, *B);
  return (int)cudaGetLastError();
}


// sin / cos of n doubles on the device: mode 0 CUDA sincos, 1 cr_sincos (common.cuh).
int cw_trig_probe(int n, const double* x, double* s, double* c, int mode, void* stream) {
  if (n <= 0) return 0;
  cw::k_trig_probe<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(n, x, s, c, mode);
  return (int)cudaGetLastError();
}

// _prepare_env for caller-supplied label grids (field.py:60-67, 403-413):
// nearest-obstacle map + walkable list for rows slots[e] of B->labels.
int cw_prepare_envs(const cw_scene_params* P, int E, const int32_t* slots,
                    const cw_scene_buffers* B, void* stream) {
  using namespace cw;
  if (E <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t nsm = nearest_smem_bytes(P->nx, P->ny);
  if (nsm > 32 * 1024) cudaFuncSetAttribute(k_nearest, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)nsm);
  k_nearest<<<E, BFS_NT, nsm, st>>>(*P, E, slots, *B);
  k_walk<<<E, 1024, 0, st>>>(*P, E, slots, *B);
  launch_reach(*P, E, slots, *B, st);
  return (int)cudaGetLastError();
}

}  // extern "C"
