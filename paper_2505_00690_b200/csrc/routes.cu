// Route anchors (reference urbangen/scene.py:102-178) on B200:
// the candidate (start, goal) pairs the robot spawns on (envcore/batch.py:183-198).
//
// One CTA (512 threads) per env, two per SM:
//   1. clearance test chamfer_distance(~walkable) * res >= 0.4 (gridmath.py:8-39).
//      The two-pass (1, sqrt2) chamfer with full-row relaxation is the octile
//      distance to the nearest non-walkable cell (shortest octile paths can be
//      taken row-monotone), so the test is evaluated by a stencil over the
//      cells within ceil(0.4 / res) of each cell, reading the walkable bitmap in
//      shared memory; a borderline distance is an integer (exact in any order),
//      irrational ones sit >= 3.5e-4 from the threshold.  Above a 6-cell radius
//      the exact two-pass transform runs instead (warp 0: each row pass is the
//      elementwise pull plus the two running minima min.accumulate(row - j) + j
//      as lane-blocked warp scans -- min is exact and the +-j are numpy's
//      elementwise float64 ops).
//   2. candidates = walkable cells with clearance >= 0.4 m (else all walkable),
//      row-major (np.nonzero order), block-scan compaction.
//   3. geodesic fields (paths.py:21-45 dijkstra_field on the walkable grid, 8-
//      connected, corner rule).  The reference's float64 Dijkstra value is the
//      minimum over paths of a left-fold sum of 1's and sqrt(2)'s; its optimum
//      lies within a few ulps of a + b*sqrt(2) for the shortest-path move counts
//      (a, b), and distinct lengths a + b*sqrt(2) differ by > 3.5e-4.  The kernel
//      finds (a, b) exactly: a cell's distance is the 64-bit key
//      (round((a + b sqrt2) 2^24) << 28) | b, whose integer order is the order of
//      the exact lengths (the rounding error < b / 2 units is far below the
//      3.5e-4 * 2^24 gap), so relaxations are atomicMin's.  Four 128-thread
//      groups run the four source fields at once as Dial's algorithm with unit
//      buckets on the exact length: bucket = floor(a + b sqrt2) = key >> 52
//      (exact for b < 3400).  Every move costs >= 1, so a bucket's keys are final
//      when it is expanded and pushes land in the next two buckets (three rotating
//      lists).  A list entry carries the key it was pushed with, and an entry whose
//      cell has since improved is expanded anyway with its old key -- its moves
//      then improve nothing -- so a level costs two dependent memory round trips
//      (list entry, atomicMin) instead of five (no key reload, no pre-filter read,
//      no de-duplication stamp); every cell is still expanded with its final key
//      in its final bucket, so the fields are exact.  geo = (a + b*sqrt(2)) * res then decides
//      the window tests as the reference except on exact-equality coincidences
//      (none in the golden set, tests/test_gpu_routes.py).
//   4. the windowed pair draws of scene.py:121-144 with the scene's
//      make_rng(seed, "routes") stream (thread 0), ok-lists compacted in order.
#include <math_constants.h>
#include "common.cuh"
#include "rng.cuh"
#include "citywalk_b200.h"

namespace cw {

constexpr int RT_NT = 512;    // 64 registers: two CTAs (two envs) per SM
constexpr int RT_GT = RT_NT / 4;   // threads per geodesic field
constexpr int RT_MAX = 8;                 // MAX_ROUTE_ANCHORS
constexpr double kMinClear = 0.4;         // MIN_ANCHOR_CLEARANCE_M
constexpr unsigned long long kNoDist = ~0ull;

CW_DEV int route_row(const int32_t* slots, int e) { return slots ? slots[e] : e; }

// distance key: (round((a + b sqrt2) 2^24) << 28) | b  (a, b < 2^28)
constexpr unsigned long long kKeyS = 1ull << 24;
constexpr unsigned long long kKeyR = 23726566ull;          // round(sqrt(2) * 2^24)
CW_DEV unsigned long long ab_key(unsigned long long a, unsigned long long b) {
  return ((a * kKeyS + b * kKeyR) << 28) | b;
}
CW_DEV void ab_decode(unsigned long long key, unsigned long long& a, unsigned long long& b) {
  b = key & ((1ull << 28) - 1);
  a = ((key >> 28) - b * kKeyR) / kKeyS;
}
// floor(a + b sqrt2) = top bits of the key: b sqrt2 (b > 0) is >= 1 / (2.83 b)
// from every integer, far above the key's rounding b / 2 * 2^-24 for b < 3400
CW_DEV long long ab_bucket(unsigned long long key) { return (long long)(key >> 52); }
// the key one move further: a + 1 (orthogonal) or b + 1 (diagonal), no decode
constexpr unsigned long long kStepOrth = kKeyS << 28;
constexpr unsigned long long kStepDiag = (kKeyR << 28) + 1ull;

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
    if (lane < RT_NT / 32) sh[lane] = s;
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

// scratch per env: 4 fields x (key u64 + three bucket lists of N entries {key u64,
// cell i32}), cand N i32, ok N i32 (the chamfer's D aliases field 0's keys)
CW_HD size_t route_scratch_per_env(int nx, int ny) { return (size_t)nx * ny * (4 * (8 + 3 * 12) + 4 + 4); }

// Shared memory of k_routes: the walkable bitmap, plus (kMv) one byte per cell whose
// bit d says move d of paths.py:35-40 is legal from it (in bounds, walkable, diagonals
// need both orthogonal cells walkable).
CW_HD size_t route_smem_bytes(int nx, int ny, bool mv) {
  const size_t N = (size_t)nx * ny;
  return ((N + 31) / 32) * 4 + (mv ? ((N + 15) & ~(size_t)15) : 0);
}
// above: bitmap only, (entry, move) per thread.  Measured (B200, round 2): at 256^2 the
// bitmap-only path is faster (k_routes 13.3 -> 12.2 ms per 1024 cfg2 envs: 8 KB instead of
// 72 KB of shared memory leaves the L1 to the list / key traffic); at 128^2 the move
// table is 2 % faster.
constexpr size_t kRouteMvSmem = 32 * 1024;

// One env on the whole CTA (scratch `base` is the CTA's slot).
template <bool kMv>
__device__ void route_env(const cw_scene_params& P, int e, const uint64_t* __restrict__ scene_seeds,
                          const int32_t* slots, const cw_scene_buffers& B, double* routes, int32_t* n_routes,
                          unsigned char* base) {
  extern __shared__ uint32_t s_walk[];   // walkable bits (then the move bytes, kMv)
  __shared__ int sh[RT_NT / 32 + 1];
  __shared__ int s_src[4], s_np, s_changed[4];
  __shared__ double s_pairs[RT_MAX * 4];
  const int row_e = route_row(slots, e);
  if (B.status[row_e] != CW_OK) return;
  const int nx = P.nx, ny = P.ny, N = nx * ny;
  const double res = P.res;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint8_t* lab = B.labels + (size_t)row_e * N;
  unsigned long long* F = reinterpret_cast<unsigned long long*>(base);           // 4 x N
  unsigned long long* LKs = F + (size_t)N * 4;                                   // 4 x 3 x N list keys
  int32_t* LCs = reinterpret_cast<int32_t*>(LKs + (size_t)N * 12);               // 4 x 3 x N list cells
  int32_t* cand = LCs + (size_t)N * 12;
  int32_t* okl = cand + N;
  double* D = reinterpret_cast<double*>(F);                                      // chamfer (field 0)
  const int NW = (N + 31) / 32;
  for (int w = wid; w < NW; w += RT_NT / 32) {   // warp per word: coalesced label reads
    const int f = w * 32 + lane;
    const unsigned bits = __ballot_sync(0xffffffffu, f < N && lab[f] == L_WALKABLE);
    if (lane == 0) s_walk[w] = bits;
  }
  uint8_t* s_mv = reinterpret_cast<uint8_t*>(s_walk + NW);
  __syncthreads();
  auto walk = [&](int r, int c) { return (s_walk[(r * nx + c) >> 5] >> ((r * nx + c) & 31)) & 1u; };
  if (kMv) {
    for (int f = tid; f < N; f += RT_NT) {
      const int r = f / nx, c = f - r * nx;
      unsigned m = 0;
      if (walk(r, c)) {
#pragma unroll
        for (int d = 0; d < 8; ++d) {
          const int rr = r + (int)((0x22001120u >> (4 * d)) & 0xF) - 1;
          const int cc = c + (int)((0x20202011u >> (4 * d)) & 0xF) - 1;
          if (rr < 0 || rr >= ny || cc < 0 || cc >= nx || !walk(rr, cc)) continue;
          if (d >= 4 && !(walk(r, cc) && walk(rr, c))) continue;
          m |= 1u << d;
        }
      }
      s_mv[f] = (uint8_t)m;
    }
    __syncthreads();
  }
  // ---- 1. clearance
  const int rad = (int)ceil(kMinClear / res);
  const bool stencil = rad <= 6;
  auto win_bits = [&](int rr, int c0, int w) -> unsigned long long {   // w <= 13 bits from column c0
    const int f = rr * nx + c0, wd = f >> 5, sh = f & 31;
    unsigned long long x = s_walk[wd];
    if (sh + w > 32) x |= (unsigned long long)s_walk[wd + 1] << 32;
    return (x >> sh) & ((1ull << w) - 1ull);
  };
  // The clearance ball: offsets (dr, dc) with octile(|dr|, |dc|) * res < 0.4.  For a
  // fixed |dr| the octile distance grows with |dc|, so the ball's row |dr| is the
  // column range |dc| <= s_half[|dr|] (-1: empty) -- one bit-window test per row.
  __shared__ int s_half[8];
  if (stencil && tid <= rad) {
    int m = -1;
    for (int ac = 0; ac <= rad; ++ac) {
      const double o = kSqrt2 * (double)min(tid, ac) + (double)abs(tid - ac);
      if (o * res < kMinClear) m = ac;
    }
    s_half[tid] = m;
  }
  __syncthreads();
  auto clear_at = [&](int f) -> bool {   // chamfer(~walkable) * res >= 0.4 for a walkable cell
    if (!stencil) return D[f] * res >= kMinClear;
    const int r = f / nx, c = f - r * nx;
    for (int dr = -rad; dr <= rad; ++dr) {
      const int rr = r + dr, m = s_half[abs(dr)];
      if (rr < 0 || rr >= ny || m < 0) continue;
      const int lo = max(c - m, 0), hi = min(c + m, nx - 1), w = hi - lo + 1;
      if (win_bits(rr, lo, w) != ((1ull << w) - 1ull)) return false;   // a non-walkable cell in the ball
    }
    return true;
  };
  if (!stencil) {
    for (int f = tid; f < N; f += RT_NT) D[f] = walk(f / nx, f % nx) ? 1e9 : 0.0;
    __syncthreads();
    if (wid == 0) {
      for (int r = 0; r < ny; ++r) chamfer_row(D + (size_t)r * nx, r ? D + (size_t)(r - 1) * nx : nullptr, nx, lane);
      for (int r = ny - 2; r >= 0; --r) chamfer_row(D + (size_t)r * nx, D + (size_t)(r + 1) * nx, nx, lane);
    }
    __syncthreads();
  }
  // ---- 2. candidates
  int nc = 0;
  for (int pass = 0; pass < 2 && nc == 0; ++pass) {
    int basec = 0;
    for (int f0 = 0; f0 < N; f0 += RT_NT) {
      const int f = f0 + tid;
      const bool w = f < N && walk(f / nx, f % nx);
      const bool c = w && (pass == 1 || clear_at(f));
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
  // fields: group g (RT_GT threads) owns source g; Dial's buckets with atomicMin
  // keys, one named barrier (id 1 + g) per group; three rotating bucket lists of
  // N entries each (an entry per improving relaxation; overflow is reported)
  const int g = tid / RT_GT, gt = tid % RT_GT;
  __shared__ int s_fn[4][3];   // bucket list sizes
  __shared__ int s_ovf;
  if (tid == 0) s_ovf = 0;
  __syncthreads();
  if (g < nf) {
    unsigned long long* Fg = F + (size_t)g * N;
    const int cap = N;
    unsigned long long* LK = LKs + (size_t)g * 3 * N;
    int32_t* LC = LCs + (size_t)g * 3 * N;
    for (int f = gt; f < N; f += RT_GT) Fg[f] = kNoDist;
    auto gsync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(RT_GT) : "memory"); };
    gsync();
    if (gt == 0) {
      const int f0 = cand[s_src[g]];
      Fg[f0] = ab_key(0, 0);
      LK[0] = ab_key(0, 0);
      LC[0] = kMv ? f0 : ((f0 / nx) << 16) | (f0 % nx);
      s_fn[g][0] = 1;
      s_fn[g][1] = 0;
      s_fn[g][2] = 0;
    }
    gsync();
    for (long long k = 0;; ++k) {
      const int cur = (int)(k % 3);
      const int n_cur = s_fn[g][cur];
      if (n_cur == 0 && s_fn[g][(cur + 1) % 3] == 0 && s_fn[g][(cur + 2) % 3] == 0) break;
      const unsigned long long* Kc = LK + (size_t)cur * cap;
      const int32_t* Cc = LC + (size_t)cur * cap;
      if (kMv) {
        // one entry per thread, its legal moves (one shared byte) in two halves of four
        // atomics in flight; pushes aggregated per warp and target list (an orthogonal
        // move from bucket k lands in bucket k + 1, a diagonal one in k + 1 or k + 2)
        const int s1 = cur == 2 ? 0 : cur + 1, s2 = s1 == 2 ? 0 : s1 + 1;
        const unsigned lt = (1u << lane) - 1u;
        for (int q0 = gt - lane; q0 < n_cur; q0 += RT_GT) {
          const int q = q0 + lane;
          const bool live = q < n_cur;
          const int u = live ? Cc[q] : 0;
          const unsigned long long ku = live ? Kc[q] : 0ull;
          const unsigned m = live ? s_mv[u] : 0u;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            unsigned long long kn[4], old[4];
            int vv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int d = 4 * h + j;
              const int dr = (int)((0x22001120u >> (4 * d)) & 0xF) - 1;
              const int dc = (int)((0x20202011u >> (4 * d)) & 0xF) - 1;
              vv[j] = u + dr * nx + dc;
              kn[j] = ku + (h ? kStepDiag : kStepOrth);
              old[j] = ((m >> d) & 1u) ? atomicMin(&Fg[vv[j]], kn[j]) : 0ull;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const bool push = (((m >> (4 * h + j)) & 1u) != 0u) && kn[j] < old[j];
              const bool far = push && h && ab_bucket(kn[j]) != k + 1;
              const unsigned b1 = __ballot_sync(0xffffffffu, push && !far);
              const unsigned b2 = __ballot_sync(0xffffffffu, far);
              int at1 = 0, at2 = 0;
              if (lane == 0 && b1) at1 = atomicAdd(&s_fn[g][s1], __popc(b1));
              if (lane == 0 && b2) at2 = atomicAdd(&s_fn[g][s2], __popc(b2));
              if (b1 | b2) {
                at1 = __shfl_sync(0xffffffffu, at1, 0) + __popc(b1 & lt);
                at2 = __shfl_sync(0xffffffffu, at2, 0) + __popc(b2 & lt);
                if (push) {
                  const int sl = far ? s2 : s1, at = far ? at2 : at1;
                  if (at < cap) {
                    LK[(size_t)sl * cap + at] = kn[j];
                    LC[(size_t)sl * cap + at] = vv[j];
                  } else {
                    s_ovf = 1;
                  }
                }
              }
            }
          }
        }
      } else
      // items (entry, move) in batches of 4 per thread: the loads and atomics of a
      // batch are issued back to back; cells are packed (row << 16 | col)
      for (int q0 = gt; q0 < n_cur * 8; q0 += RT_GT * 4) {
        constexpr int BT = 4;
        int pu[BT], rv[BT], cv[BT], v[BT];
        unsigned long long kk[BT];
        bool ok[BT];
#pragma unroll
        for (int i = 0; i < BT; ++i) {
          const int q = q0 + i * RT_GT;
          pu[i] = q < n_cur * 8 ? Cc[q >> 3] : -1;
          kk[i] = q < n_cur * 8 ? Kc[q >> 3] : ~0ull;
        }
#pragma unroll
        for (int i = 0; i < BT; ++i) {
          const int d = (q0 + i * RT_GT) & 7;
          ok[i] = false;
          v[i] = 0;
          rv[i] = cv[i] = 0;
          if (pu[i] < 0) continue;
          const int ru = pu[i] >> 16, cu = pu[i] & 0xFFFF;
          const int dr = (int)((0x22001120u >> (4 * d)) & 0xF) - 1;
          const int dc = (int)((0x20202011u >> (4 * d)) & 0xF) - 1;
          rv[i] = ru + dr;
          cv[i] = cu + dc;
          if (rv[i] < 0 || rv[i] >= ny || cv[i] < 0 || cv[i] >= nx || !walk(rv[i], cv[i])) continue;
          const bool diag = d >= 4;
          if (diag && !(walk(ru, cv[i]) && walk(rv[i], cu))) continue;
          kk[i] += diag ? kStepDiag : kStepOrth;
          v[i] = rv[i] * nx + cv[i];
          ok[i] = true;
        }
        unsigned long long old[BT];
#ifdef CW_ROUTES_PREFILTER   // A/B: a plain read filters relaxations that cannot improve
#pragma unroll
        for (int i = 0; i < BT; ++i) old[i] = ok[i] ? (unsigned long long)((volatile unsigned long long*)Fg)[v[i]] : 0ull;
#pragma unroll
        for (int i = 0; i < BT; ++i) {
          ok[i] = ok[i] && kk[i] < old[i];
          if (ok[i]) old[i] = atomicMin(&Fg[v[i]], kk[i]);
        }
#else
#pragma unroll
        for (int i = 0; i < BT; ++i) old[i] = ok[i] ? atomicMin(&Fg[v[i]], kk[i]) : 0ull;
#endif
#pragma unroll
        for (int i = 0; i < BT; ++i) {
          if (ok[i] && kk[i] < old[i]) {
            const int slot = (int)(ab_bucket(kk[i]) % 3);   // k + 1 or k + 2
            const int at = atomicAdd(&s_fn[g][slot], 1);
            if (at < cap) {
              LK[(size_t)slot * cap + at] = kk[i];
              LC[(size_t)slot * cap + at] = (rv[i] << 16) | cv[i];
            } else {
              s_ovf = 1;
            }
          }
        }
      }
      gsync();
      if (gt == 0) {
        s_fn[g][cur] = 0;
        for (int b = 0; b < 3; ++b) s_fn[g][b] = min(s_fn[g][b], cap);
      }
      gsync();
    }
  }
  __syncthreads();
  if (s_ovf) {   // a bucket list overflowed: the field may be incomplete -- report, never guess
    if (tid == 0) { B.status[row_e] = CW_E_HEAPCAP; n_routes[row_e] = 0; }
    return;
  }
  __syncthreads();
  auto geo_of = [&](int fi, int f) -> double {
    const unsigned long long v = F[(size_t)fi * N + f];
    if (v == kNoDist) return CUDART_INF;
    unsigned long long a, b;
    ab_decode(v, a, b);
    return ((double)a + (double)b * kSqrt2) * res;
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

// Persistent CTAs (one scratch slot each) take envs from a counter until all are
// done: no launch-to-launch tails between env chunks.
template <bool kMv>
__global__ void __launch_bounds__(RT_NT, 2) k_routes(cw_scene_params P, int E, const uint64_t* __restrict__ scene_seeds,
                                                     const int32_t* slots, cw_scene_buffers B, double* routes,
                                                     int32_t* n_routes, unsigned char* scratch, int* counter) {
  __shared__ int s_e;
  unsigned char* base = scratch + (size_t)blockIdx.x * route_scratch_per_env(P.nx, P.ny);
  while (true) {
    if (threadIdx.x == 0) s_e = atomicAdd(counter, 1);
    __syncthreads();
    const int e = s_e;
    __syncthreads();
    if (e >= E) return;
    route_env<kMv>(P, e, scene_seeds, slots, B, routes, n_routes, base);
    __syncthreads();
  }
}

}  // namespace cw

extern "C" {

size_t cw_route_scratch_bytes(int nx, int ny, int chunk) {
  return (size_t)chunk * cw::route_scratch_per_env(nx, ny) + 256;   // + the env counter
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
  const bool mv = route_smem_bytes(P->nx, P->ny, true) <= kRouteMvSmem;
  const size_t smem = route_smem_bytes(P->nx, P->ny, mv);
  if (smem > 32 * 1024) {
    if (mv) cudaFuncSetAttribute(k_routes<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    else cudaFuncSetAttribute(k_routes<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  int* counter = reinterpret_cast<int*>(static_cast<unsigned char*>(scratch) +
                                        (size_t)chunk * route_scratch_per_env(P->nx, P->ny));
  cudaMemsetAsync(counter, 0, sizeof(int), st);
  if (mv)
    k_routes<true><<<min(chunk, E), RT_NT, smem, st>>>(*P, E, scene_seeds, slots, *B, routes, n_routes,
                                                     (unsigned char*)scratch, counter);
  else
    k_routes<false><<<min(chunk, E), RT_NT, smem, st>>>(*P, E, scene_seeds, slots, *B, routes, n_routes,
                                                      (unsigned char*)scratch, counter);
  return (int)cudaGetLastError();
}

}  // extern "C"
