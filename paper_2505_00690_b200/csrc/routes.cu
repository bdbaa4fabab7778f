// Route anchors (reference urbangen/scene.py:102-178) on B200:
// the candidate (start, goal) pairs the robot spawns on (envcore/batch.py:183-198).
//
// One CTA (1024 threads) per env:
//   1. clearance = chamfer_distance(~walkable) (gridmath.py:8-39) by warp 0: each
//      row pass is an elementwise pull from the previous row plus the two running
//      minima min.accumulate(row - j) + j / its mirror, done as lane-blocked warp
//      scans.  min is exact and the +-j are the same elementwise float64 ops, so
//      the field is bit-identical to numpy's.
//   2. candidates = walkable cells with clearance >= 0.4 m (else all walkable),
//      row-major (np.nonzero order), block-scan compaction.
//   3. geodesic fields (paths.py:21-45 dijkstra_field on the walkable grid, 8-
//      connected, corner rule).  The reference's float64 Dijkstra value is the
//      minimum over paths of a left-fold sum of 1's and sqrt(2)'s; its optimum
//      lies within a few ulps of a + b*sqrt(2) for the shortest-path move counts
//      (a, b), and distinct lengths a + b*sqrt(2) differ by > 3.5e-4.  The kernel
//      finds (a, b) exactly with integer comparisons (da^2 vs 2 db^2): four
//      256-thread groups run the four source fields at once with directional
//      sweeps (H, V and both diagonals, each way; one thread per line) until no
//      cell improves -- ties are exact, so any shortest path is fine and a few
//      rounds converge.  geo = (a + b*sqrt(2)) * res then decides the window
//      tests exactly as the reference except on exact-equality coincidences
//      (none in the golden set, tests/test_gpu_routes.py).
//   4. the windowed pair draws of scene.py:121-144 with the scene's
//      make_rng(seed, "routes") stream (thread 0), ok-lists compacted in order.
#include <math_constants.h>
#include "common.cuh"
#include "rng.cuh"
#include "citywalk_b200.h"

namespace cw {

constexpr int RT_NT = 1024;
constexpr int RT_MAX = 8;                 // MAX_ROUTE_ANCHORS
constexpr double kMinClear = 0.4;         // MIN_ANCHOR_CLEARANCE_M
constexpr unsigned long long kNoDist = ~0ull;

CW_DEV int route_row(const int32_t* slots, int e) { return slots ? slots[e] : e; }

// exact (a1 + b1 sqrt2) < (a2 + b2 sqrt2)
CW_DEV bool ab_less(long long a1, long long b1, long long a2, long long b2) {
  const long long da = a1 - a2, db = b1 - b2;
  if (da <= 0 && db <= 0) return da < 0 || db < 0;
  if (da >= 0 && db >= 0) return false;
  if (da < 0) return da * da > 2 * db * db;     // db > 0
  return da * da < 2 * db * db;                 // da > 0, db < 0
}

CW_DEV unsigned long long ab_pack(unsigned a, unsigned b) { return ((unsigned long long)a << 32) | b; }

// block-wide exclusive scan of one int per thread
CW_DEV int rt_excl_scan(int v, int* sh, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = lane < RT_NT / 32 ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    sh[lane] = s;
  }
  __syncthreads();
  total = sh[RT_NT / 32 - 1];
  const int r = (wid ? sh[wid - 1] : 0) + x - v;
  __syncthreads();
  return r;
}

// One chamfer row pass for warp 0: row = min(row, pull(prev)) then the two running
// minima (gridmath.py:18-32).  K = elements per lane (contiguous block per lane).
CW_DEV void chamfer_row(double* row, const double* prev, int nx, int lane) {
  const int K = (nx + 31) / 32;
  const int j0 = lane * K;
  double lf = CUDART_INF, rt = CUDART_INF;
  // pull + left prefix over the lane's block
  for (int t = 0; t < K; ++t) {
    const int j = j0 + t;
    if (j >= nx) break;
    double v = row[j];
    if (prev) {
      double dg = 1e9;
      if (j >= 1) dg = prev[j - 1] + kSqrt2;
      if (j + 1 < nx) dg = fmin(dg, prev[j + 1] + kSqrt2);
      v = fmin(v, fmin(prev[j] + 1.0, dg));
      row[j] = v;
    }
    lf = fmin(lf, v - (double)j);
  }
  // exclusive prefix of the lane minima (left) / exclusive suffix (right)
  double pl = lf;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, pl, o);
    if (lane >= o) pl = fmin(pl, y);
  }
  double exl = __shfl_up_sync(0xffffffffu, pl, 1);
  if (lane == 0) exl = CUDART_INF;
  for (int t = K - 1; t >= 0; --t) {
    const int j = j0 + t;
    if (j < nx) rt = fmin(rt, row[j] + (double)j);
  }
  double ps = rt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_down_sync(0xffffffffu, ps, o);
    if (lane + o < 32) ps = fmin(ps, y);
  }
  double exr = __shfl_down_sync(0xffffffffu, ps, 1);
  if (lane == 31) exr = CUDART_INF;
  __syncwarp();
  // apply: left[j] = min(prefix(v - j)) + j, right[j] = min(suffix(v + j)) - j
  double lrun = exl;
  double vals[32];
  for (int t = 0; t < K && t < 32; ++t) {
    const int j = j0 + t;
    if (j >= nx) break;
    lrun = fmin(lrun, row[j] - (double)j);
    vals[t] = lrun + (double)j;
  }
  double rrun = exr;
  for (int t = K - 1; t >= 0; --t) {
    const int j = j0 + t;
    if (j >= nx || t >= 32) continue;
    rrun = fmin(rrun, row[j] + (double)j);
    vals[t] = fmin(vals[t], rrun - (double)j);
  }
  __syncwarp();
  for (int t = 0; t < K && t < 32; ++t) {
    const int j = j0 + t;
    if (j < nx) row[j] = vals[t];
  }
  __syncwarp();
}

// scratch per env: fields 4 x N u64, cand N i32, ok N i32 (D aliases field 0)
CW_HD size_t route_scratch_per_env(int nx, int ny) { return (size_t)nx * ny * (4 * 8 + 4 + 4); }

__global__ void __launch_bounds__(RT_NT, 1) k_routes(cw_scene_params P, int e0, int n,
                                                     const uint64_t* __restrict__ scene_seeds,
                                                     const int32_t* slots, cw_scene_buffers B,
                                                     double* routes, int32_t* n_routes,
                                                     unsigned char* scratch) {
  extern __shared__ uint32_t s_walk[];   // walkable bits
  __shared__ int sh[RT_NT / 32 + 1];
  __shared__ int s_nc, s_src[4], s_np, s_changed[4];
  __shared__ double s_pairs[RT_MAX * 4];
  const int k = blockIdx.x;
  if (k >= n) return;
  const int e = e0 + k;
  const int row_e = route_row(slots, e);
  if (B.status[row_e] != CW_OK) return;
  const int nx = P.nx, ny = P.ny, N = nx * ny;
  const double res = P.res;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint8_t* lab = B.labels + (size_t)row_e * N;
  unsigned char* base = scratch + (size_t)k * route_scratch_per_env(nx, ny);
  unsigned long long* F = reinterpret_cast<unsigned long long*>(base);           // 4 x N
  int32_t* cand = reinterpret_cast<int32_t*>(base + (size_t)N * 32);
  int32_t* okl = cand + N;
  double* D = reinterpret_cast<double*>(F);                                      // chamfer (field 0)
  const int NW = (N + 31) / 32;
  for (int w = tid; w < NW; w += RT_NT) {
    uint32_t bits = 0;
    for (int b = 0; b < 32; ++b) {
      const int f = w * 32 + b;
      if (f < N && lab[f] == L_WALKABLE) bits |= 1u << b;
    }
    s_walk[w] = bits;
  }
  __syncthreads();
  auto walk = [&](int r, int c) { return (s_walk[(r * nx + c) >> 5] >> ((r * nx + c) & 31)) & 1u; };
  // ---- 1. clearance (warp 0)
  for (int f = tid; f < N; f += RT_NT) D[f] = walk(f / nx, f % nx) ? 1e9 : 0.0;
  __syncthreads();
  if (wid == 0) {
    for (int r = 0; r < ny; ++r) chamfer_row(D + (size_t)r * nx, r ? D + (size_t)(r - 1) * nx : nullptr, nx, lane);
    for (int r = ny - 2; r >= 0; --r) chamfer_row(D + (size_t)r * nx, D + (size_t)(r + 1) * nx, nx, lane);
  }
  __syncthreads();
  // ---- 2. candidates
  int nc = 0;
  for (int pass = 0; pass < 2 && nc == 0; ++pass) {
    int basec = 0;
    for (int f0 = 0; f0 < N; f0 += RT_NT) {
      const int f = f0 + tid;
      const bool w = f < N && walk(f / nx, f % nx);
      const bool c = w && (pass == 1 || D[f] * res >= kMinClear);
      int tot;
      const int off = rt_excl_scan(c ? 1 : 0, sh, tot);
      if (c) cand[basec + off] = f;
      basec += tot;
    }
    nc = basec;
  }
  if (nc == 0) {
    if (tid == 0) { B.status[row_e] = CW_E_NOROUTE; n_routes[row_e] = 0; }
    return;
  }
  const bool traverse = P.task == 3;
  // ---- 3. sources (scene.py:124-127 / traverse :164)
  if (tid == 0) {
    s_np = 0;
    if (traverse) {
      const double want_sx = 1.5, cy = ny * res / 2.0;
      double best = CUDART_INF;
      int bi = 0;
      for (int q = 0; q < nc; ++q) {
        const int f = cand[q];
        const double xs = ((double)(f % nx) + 0.5) * res, ys = ((double)(f / nx) + 0.5) * res;
        const double s = (xs - want_sx) * (xs - want_sx) + (ys - cy) * (ys - cy);
        if (s < best) { best = s; bi = q; }
      }
      s_src[0] = bi;
    } else {
      Pcg64 rng = make_rng(scene_seeds[e], "routes");
      for (int i = 0; i < 4; ++i) s_src[i] = (int)integers32(rng, (uint64_t)nc);
    }
  }
  __syncthreads();
  const int nf = traverse ? 1 : 4;
  // fields: group g (256 threads) owns source g
  const int g = tid >> 8, gt = tid & 255;
  unsigned long long* Fg = F + (size_t)g * N;
  for (int f = gt; f < N && g < nf; f += 256) Fg[f] = kNoDist;
  __syncthreads();
  if (g < nf && gt == 0) Fg[cand[s_src[g]]] = ab_pack(0, 0);
  __syncthreads();
  // relax v from u (move u -> v; diagonal needs the two corner cells walkable)
  auto relax = [&](unsigned long long& carry, int ru, int cu, int rv, int cv, bool diag, bool& ch) {
    const size_t fv = (size_t)rv * nx + cv;
    unsigned long long cur = Fg[fv];
    if (carry != kNoDist && walk(rv, cv) && (!diag || (walk(ru, cv) && walk(rv, cu)))) {
      const unsigned a = (unsigned)(carry >> 32) + (diag ? 0u : 1u);
      const unsigned b = (unsigned)(carry & 0xffffffffu) + (diag ? 1u : 0u);
      if (cur == kNoDist || ab_less(a, b, (long long)(cur >> 32), (long long)(cur & 0xffffffffu))) {
        cur = ab_pack(a, b);
        Fg[fv] = cur;
        ch = true;
      }
    }
    carry = cur;
  };
  for (int round = 0; round < 4096; ++round) {
    bool ch = false;
    if (g < nf) {
      // rows east / west
      for (int r = gt; r < ny; r += 256) {
        unsigned long long c0 = Fg[(size_t)r * nx];
        for (int c = 1; c < nx; ++c) relax(c0, r, c - 1, r, c, false, ch);
        c0 = Fg[(size_t)r * nx + nx - 1];
        for (int c = nx - 2; c >= 0; --c) relax(c0, r, c + 1, r, c, false, ch);
      }
    }
    __syncthreads();
    if (g < nf) {
      // columns south / north
      for (int c = gt; c < nx; c += 256) {
        unsigned long long c0 = Fg[c];
        for (int r = 1; r < ny; ++r) relax(c0, r - 1, c, r, c, false, ch);
        c0 = Fg[(size_t)(ny - 1) * nx + c];
        for (int r = ny - 2; r >= 0; --r) relax(c0, r + 1, c, r, c, false, ch);
      }
    }
    __syncthreads();
    if (g < nf) {
      // diagonals r - c = const (down-right / up-left)
      for (int L = gt; L < nx + ny - 1; L += 256) {
        const int d = L - (ny - 1);                   // c = r + d
        const int r0 = max(0, -d), r1 = min(ny - 1, nx - 1 - d);
        if (r0 >= r1) continue;
        unsigned long long c0 = Fg[(size_t)r0 * nx + r0 + d];
        for (int r = r0 + 1; r <= r1; ++r) relax(c0, r - 1, r - 1 + d, r, r + d, true, ch);
        c0 = Fg[(size_t)r1 * nx + r1 + d];
        for (int r = r1 - 1; r >= r0; --r) relax(c0, r + 1, r + 1 + d, r, r + d, true, ch);
      }
    }
    __syncthreads();
    if (g < nf) {
      // diagonals r + c = const (down-left / up-right)
      for (int L = gt; L < nx + ny - 1; L += 256) {
        const int r0 = max(0, L - (nx - 1)), r1 = min(ny - 1, L);
        if (r0 >= r1) continue;
        unsigned long long c0 = Fg[(size_t)r0 * nx + (L - r0)];
        for (int r = r0 + 1; r <= r1; ++r) relax(c0, r - 1, L - r + 1, r, L - r, true, ch);
        c0 = Fg[(size_t)r1 * nx + (L - r1)];
        for (int r = r1 - 1; r >= r0; --r) relax(c0, r + 1, L - r - 1, r, L - r, true, ch);
      }
    }
    if (__syncthreads_or(ch) == 0) break;
  }
  auto geo_of = [&](int fi, int f) -> double {
    const unsigned long long v = F[(size_t)fi * N + f];
    if (v == kNoDist) return CUDART_INF;
    return ((double)(v >> 32) + (double)(v & 0xffffffffu) * kSqrt2) * res;
  };
  auto xs_of = [&](int f) { return ((double)(f % nx) + 0.5) * res; };
  auto ys_of = [&](int f) { return ((double)(f / nx) + 0.5) * res; };
  // ---- 4a. traverse: one pair (scene.py:161-178)
  if (traverse) {
    if (tid == 0) {
      const double want_gx = nx * res - 1.5, cy = ny * res / 2.0;
      double best = CUDART_INF;
      int bi = -1;
      bool any = false;
      for (int q = 0; q < nc; ++q) {
        const int f = cand[q];
        const bool reach = geo_of(0, f) != CUDART_INF;
        any |= reach;
        const double xs = xs_of(f), ys = ys_of(f);
        const double s = (xs - want_gx) * (xs - want_gx) + (ys - cy) * (ys - cy) + (reach ? 0.0 : 1e12);
        if (s < best) { best = s; bi = q; }
      }
      double* out = routes + (size_t)row_e * RT_MAX * 4;
      if (!any) {
        B.status[row_e] = CW_E_NOROUTE;
        n_routes[row_e] = 0;
      } else {
        const int fs = cand[s_src[0]], fg = cand[bi];
        out[0] = xs_of(fs); out[1] = ys_of(fs); out[2] = xs_of(fg); out[3] = ys_of(fg);
        n_routes[row_e] = 1;
      }
    }
    return;
  }
  // ---- 4b. windowed pair draws (scene.py:128-144), rng continues after the 4 sources
  Pcg64 rng;
  if (tid == 0) {
    rng = make_rng(scene_seeds[e], "routes");
    for (int i = 0; i < 4; ++i) (void)integers32(rng, (uint64_t)nc);
  }
  const double dmin = fmin(P.w, P.l);
  const double lo_[3] = {0.5 * dmin, 0.35 * dmin, 0.2 * dmin};
  const double hi_[3] = {0.8 * dmin, 0.8 * dmin, 0.9 * dmin};
  const double cap_[3] = {1.6, 2.0, 4.0};
  bool done = false;
  for (int wdx = 0; wdx < 3 && !done; ++wdx) {
    for (int fi = 0; fi < 4 && !done; ++fi) {
      const int fsrc = cand[s_src[fi]];
      const double xi = xs_of(fsrc), yi = ys_of(fsrc);
      int cnt = 0;
      for (int q0 = 0; q0 < nc; q0 += RT_NT) {
        const int q = q0 + tid;
        bool ok = false;
        if (q < nc) {
          const int f = cand[q];
          const double dx = xs_of(f) - xi, dy = ys_of(f) - yi;
          const double eu = sqrt(dx * dx + dy * dy);
          const double geo = geo_of(fi, f);
          ok = eu >= lo_[wdx] && eu <= hi_[wdx] && geo != CUDART_INF && geo <= cap_[wdx] * fmax(eu, 1e-9);
        }
        int tot;
        const int off = rt_excl_scan(ok ? 1 : 0, sh, tot);
        if (ok) okl[cnt + off] = q;
        cnt += tot;
      }
      __syncthreads();
      if (tid == 0) {
        for (int t = 0; t < min(2, cnt) && s_np < RT_MAX; ++t) {
          const int j = okl[(int)integers32(rng, (uint64_t)cnt)];
          const int fj = cand[j];
          s_pairs[s_np * 4 + 0] = xi;
          s_pairs[s_np * 4 + 1] = yi;
          s_pairs[s_np * 4 + 2] = xs_of(fj);
          s_pairs[s_np * 4 + 3] = ys_of(fj);
          ++s_np;
        }
        s_changed[0] = s_np >= RT_MAX;
      }
      __syncthreads();
      done = s_changed[0] != 0;
    }
    __syncthreads();
    if (s_np > 0) done = true;
  }
  if (tid == 0) {
    double* out = routes + (size_t)row_e * RT_MAX * 4;
    for (int q = 0; q < s_np * 4; ++q) out[q] = s_pairs[q];
    n_routes[row_e] = s_np;
    if (s_np == 0) B.status[row_e] = CW_E_NOROUTE;
  }
}

}  // namespace cw

extern "C" {

size_t cw_route_scratch_bytes(int nx, int ny, int chunk) {
  return (size_t)chunk * cw::route_scratch_per_env(nx, ny);
}

// scene.py:102-178 for rows slots[e] of B->labels (scene seeds as for sampling);
// routes (E, 8, 2, 2) float64 [[sx, sy], [gx, gy]], n_routes (E); NoRouteAvailable
// lands in B->status.
int cw_route_anchors(const cw_scene_params* P, int E, const uint64_t* scene_seeds,
                     const int32_t* slots, const cw_scene_buffers* B, double* routes,
                     int32_t* n_routes, void* scratch, int chunk, void* stream) {
  using namespace cw;
  if (E <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = (size_t)((P->nx * P->ny + 31) / 32) * 4;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_routes, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int e0 = 0; e0 < E; e0 += chunk) {
    const int n = min(chunk, E - e0);
    k_routes<<<n, RT_NT, smem, st>>>(*P, e0, n, scene_seeds, slots, *B, routes, n_routes,
                                     (unsigned char*)scratch);
  }
  return (int)cudaGetLastError();
}

}  // extern "C"
