// A* replanning search (paths.astar_path, reference crowd/paths.py:48-87) on B200.
//
// One warp runs one search; persistent warps pull requests queued by k_guide.
// The open set is the reference's lazy heapq, reproduced entry for entry:
// every push of paths.py:80-84 becomes one entry keyed (f, h, row, col), a
// popped entry whose f exceeds g + h + 1e-12 is skipped (paths.py:70-71), and
// the goal test precedes the stale test (paths.py:66-69).  Only the container
// differs -- the pop order of a min-priority queue with unique keys is the
// sorted order of its contents, whatever the data structure:
//
//   head  the (up to) 32 smallest keys, sorted, one per lane in registers.
//         pop = lane 0 + one shuffle-down; insert = ballot rank + shuffle-up.
//   near  unsorted entries with key < F2, in shared memory (NC entries).
//   far   unsorted entries with key >= F2, in the warp's global slot.
//   Invariant: every head key < T <= every near/far key.
//   refill (head empty): band extraction -- near entries with
//         f < fmin + delta are bitonic-sorted into the head (32 at a time,
//         merged; the rest go back), near is compacted in the same pass and,
//         when large, its part above fmin + delta2 is demoted to far.  When
//         near is empty, far entries below a split key move to near.
//   A decrease-key also drops the cell's stale entry from the head when it
//   is there (a stale pop is a no-op in the reference).
//
// Key = (f bits, k2) compared as one unsigned 128-bit integer.  f, h >= 0, so
// their IEEE bit patterns order like their values; distinct octile h values
// differ by > 3e-4, so k2 keeps h's top 44 bits and puts (row << 10 | col)
// in the low 20 bits, which orders like (row, col).
//
// Search-local cell state (g, the move byte) lives in 8x8-cell tiles in
// shared memory, handed out on first write and released when the search ends
// (see make_key2 below); the tile slot rides in every key, so a pop reads
// g(x) and moves(x) with one shared load each.
#pragma once

namespace cw {

using u64 = unsigned long long;

struct Key {
  u64 f, k;
};

constexpr u64 kInf64 = ~0ull;

CW_DEV Key key_inf() { return {kInf64, kInf64}; }

// cell of a key2 (row << cb | col in bits [40:21], cb = column bits; see make_key2)
CW_DEV int key_col(u64 k, int cb) { return (int)(k >> 21) & ((1 << cb) - 1); }
CW_DEV int key_row(u64 k, int cb) { return (int)(k >> (21 + cb)) & ((1 << (20 - cb)) - 1); }
// column bits of an nx x ny grid
CW_HD int key_col_bits(int nx, int ny) {
  int b = 0;
  while ((1 << b) < nx) ++b;
  return b <= 10 && ny <= 1024 ? 10 : b;
}

// branch-free lexicographic compare (bitwise predicate logic: no short-circuit
// control flow for the compiler to turn into divergent branches)
CW_DEV bool klt(const Key& a, const Key& b) {
  return (a.f < b.f) | ((a.f == b.f) & (a.k < b.k));
}

CW_DEV Key shfl_key(const Key& v, int src) {
  return {__shfl_sync(0xffffffffu, v.f, src), __shfl_sync(0xffffffffu, v.k, src)};
}
CW_DEV Key shfl_key_xor(const Key& v, int m) {
  return {__shfl_xor_sync(0xffffffffu, v.f, m), __shfl_xor_sync(0xffffffffu, v.k, m)};
}
CW_DEV Key shfl_key_down(const Key& v, int d) {
  return {__shfl_down_sync(0xffffffffu, v.f, d), __shfl_down_sync(0xffffffffu, v.k, d)};
}
CW_DEV Key shfl_key_up(const Key& v, int d) {
  return {__shfl_up_sync(0xffffffffu, v.f, d), __shfl_up_sync(0xffffffffu, v.k, d)};
}

// ascending bitonic sort of one key per lane (empty lanes hold +inf)
CW_DEV void warp_sort(Key& v, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const Key p = shfl_key_xor(v, j);
      const bool keep_min = ((lane & j) == 0) == ((lane & k) == 0);
      if (klt(p, v) == keep_min) v = p;
    }
  }
}

// finish a bitonic sequence into ascending order
CW_DEV void warp_bitonic_clean(Key& v, int lane) {
#pragma unroll
  for (int j = 16; j > 0; j >>= 1) {
    const Key p = shfl_key_xor(v, j);
    if (klt(p, v) == ((lane & j) == 0)) v = p;
  }
}

// Open set of one search (warp-uniform except hd).
struct OpenSet {
  Key hd;              // this lane's head entry (+inf beyond h)
  Key T;               // every near/far key >= T
  Key F2;              // near < F2 <= far
  double delta, delta2;
  int h, nn, nf;
  int err;
};

struct Pools {
  OpenEnt* near;       // shared memory, NC entries
  OpenEnt* stg;        // shared memory, 64-entry staging area
  OpenEnt* far;        // global, far_cap entries
  int NC, far_cap;
  const double* gt;    // g tiles of the running search (shared or global)
  short gr, gc;        // goal row / col of the running search (< 2048, crowd.py)
  int cb;              // column bits of the key2 cell field
};

CW_DEV double octile(int r, int c, int gr, int gc);

template <class T>
CW_DEV T ld_grid(const T* p, bool cg) { return cg ? __ldcg(p) : *p; }

// An entry whose cell has since been improved is stale for good (g only
// decreases); the reference pops it and skips it (paths.py:70-71), so it can
// be dropped whenever the pools are scanned.  Key layout: see make_key2.
CW_DEV bool stale_entry(const OpenEnt& v, const Pools& pl) {
  const int r = key_row(v.k, pl.cb), c = key_col(v.k, pl.cb);
  const int sl = (int)(v.k >> 5) & 0xFFFF;
  const double g = pl.gt[(size_t)sl * 64 + (r & 7) * 8 + (c & 7)];
  return __longlong_as_double((long long)v.f) > g + octile(r, c, pl.gr, pl.gc) + 1e-12;
}

CW_DEV u64 f_plus(u64 fb, double d) {
  const u64 t = (u64)__double_as_longlong(__longlong_as_double((long long)fb) + d);
  return t <= fb ? fb + 1ull : t;
}

CW_DEV u64 warp_min_u64(u64 v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

CW_DEV int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// min f over A[0, n) (loads issued four at a time)
CW_DEV u64 fmin_of(const OpenEnt* A, int n, int lane) {
  u64 fm = kInf64;
  for (int i = lane; i < n; i += 128) {
    const u64 a = A[i].f;
    const u64 b = i + 32 < n ? A[i + 32].f : kInf64;
    const u64 c = i + 64 < n ? A[i + 64].f : kInf64;
    const u64 d = i + 96 < n ? A[i + 96].f : kInf64;
    fm = min(fm, min(min(a, b), min(c, d)));
  }
  return warp_min_u64(fm);
}

CW_DEV int count_lt(const OpenEnt* A, int n, const Key& K, int lane) {
  int c = 0;
  for (int i = lane; i < n; i += 32) {
    const OpenEnt e = A[i];
    c += klt(Key{e.f, e.k}, K);
  }
  return warp_sum(c);
}

// A split key K with 1 <= |{A < K}| <= target (n > 0, fm = min f of A): first
// by f (K = (fm + delta, 0), shrinking delta), then, for an equal-f plateau
// larger than target, by bisection on k within f == fm.
CW_DEV Key choose_split(const OpenEnt* A, int n, u64 fm, int target, double& delta, int lane) {
  Key K = {f_plus(fm, delta), 0ull};
  int c = count_lt(A, n, K, lane);
  while (c > target && K.f > fm + 1ull) {
    delta *= 0.25;
    K = {f_plus(fm, delta), 0ull};
    c = count_lt(A, n, K, lane);
  }
  if (c > target) {
    u64 kmin = kInf64, kmax = 0ull;
    for (int i = lane; i < n; i += 32) {
      const OpenEnt e = A[i];
      if (e.f == fm) { kmin = min(kmin, e.k); kmax = max(kmax, e.k); }
    }
    kmin = warp_min_u64(kmin);
    kmax = ~warp_min_u64(~kmax);
    u64 lo = kmin, hi = kmax + 1ull;   // |< (fm, lo)| <= target < |< (fm, hi)|
    while (hi - lo > 1ull) {
      const u64 mid = lo + (hi - lo) / 2ull;
      if (count_lt(A, n, Key{fm, mid}, lane) > target) hi = mid;
      else lo = mid;
    }
    K = {fm, lo > kmin ? lo : kmin + 1ull};
  }
  return K;
}

// Near is about to overflow: demote its entries >= a split key to far.
__device__ __noinline__ OpenSet split_near(OpenSet st, const Pools pl, int lane) {
  const unsigned lt_mask = (1u << lane) - 1u;
  const u64 fm = fmin_of(pl.near, st.nn, lane);
  const Key K = choose_split(pl.near, st.nn, fm, pl.NC / 2, st.delta2, lane);
  int w = 0;
  for (int base = 0; base < st.nn; base += 32) {
    const int i = base + lane;
    OpenEnt v = {kInf64, kInf64};
    if (i < st.nn) v = pl.near[i];
    const bool live = i < st.nn && !stale_entry(v, pl);
    const bool dem = live && !klt(Key{v.f, v.k}, K);
    const bool keep = live && !dem;
    const unsigned dm = __ballot_sync(0xffffffffu, dem);
    const unsigned km = __ballot_sync(0xffffffffu, keep);
    if (dem && st.nf + __popc(dm) <= pl.far_cap) pl.far[st.nf + __popc(dm & lt_mask)] = v;
    st.nf += __popc(dm);
    __syncwarp();
    if (keep) pl.near[w + __popc(km & lt_mask)] = v;
    w += __popc(km);
  }
  st.nn = w;
  st.F2 = K;
  if (st.nf > pl.far_cap) st.err = 1;
  __syncwarp();
  return st;
}

// Head is empty: (far -> near if near is empty), then near -> head.
__device__ __noinline__ OpenSet refill(OpenSet st, const Pools pl, int lane) {
  const unsigned lt_mask = (1u << lane) - 1u;
  if (st.nn == 0) {
    // ---------------- far -> near: entries below a split key (<= 3/4 of near)
    const u64 fm = fmin_of(pl.far, st.nf, lane);
    const Key K = choose_split(pl.far, st.nf, fm, (3 * pl.NC) / 4, st.delta2, lane);
    int w = 0;
    OpenEnt v = {kInf64, kInf64};
    if (lane < st.nf) v = pl.far[lane];
    for (int base = 0; base < st.nf; base += 32) {
      const int i = base + lane;
      OpenEnt vn = {kInf64, kInf64};
      if (i + 32 < st.nf) vn = pl.far[i + 32];          // prefetch the next chunk
      const bool live = i < st.nf && !stale_entry(v, pl);
      const bool in = live && klt(Key{v.f, v.k}, K);
      const bool keep = live && !in;
      const unsigned bm = __ballot_sync(0xffffffffu, in);
      const unsigned km = __ballot_sync(0xffffffffu, keep);
      if (in) pl.near[st.nn + __popc(bm & lt_mask)] = v;
      st.nn += __popc(bm);
      __syncwarp();
      if (keep) pl.far[w + __popc(km & lt_mask)] = v;
      w += __popc(km);
      v = vn;
    }
    st.nf = w;
    st.F2 = K;
    if (st.nn < pl.NC / 16 && st.delta2 < 1024.0) st.delta2 *= 2.0;
    __syncwarp();
  }
  // ---------------- near -> head: f < fmin(near) + delta, sorted; a large
  // near also demotes its part at or above fmin + delta2 to far
  const u64 fm = fmin_of(pl.near, st.nn, lane);
  Key B = {f_plus(fm, st.delta), 0ull};
  if (klt(st.F2, B)) B = st.F2;
  if (st.nn > pl.NC / 4) {
    Key sp = {f_plus(fm, st.delta2), 0ull};
    if (klt(sp, B)) sp = B;
    if (klt(sp, st.F2)) st.F2 = sp;
  }
  Key acc = key_inf();
  bool rejected = false;
  int ns = 0, w = 0, nband = 0;
  // merge `take` staged keys into the sorted accumulator; the larger half of
  // the pairing returns to near (compacted behind the reads)
  auto merge = [&](int take) {
    Key cv = key_inf();
    if (lane < take) { const OpenEnt s = pl.stg[lane]; cv = {s.f, s.k}; }
    __syncwarp();
    if (lane < ns - take) pl.stg[lane] = pl.stg[lane + take];
    __syncwarp();
    ns -= take;
    warp_sort(cv, lane);
    const Key rv = shfl_key(cv, 31 - lane);
    const bool rl = klt(rv, acc);
    const Key hi = rl ? acc : rv;
    if (rl) acc = rv;
    warp_bitonic_clean(acc, lane);
    const bool back = hi.f != kInf64;
    const unsigned rm = __ballot_sync(0xffffffffu, back);
    if (rm) rejected = true;
    if (back) { OpenEnt o = {hi.f, hi.k}; pl.near[w + __popc(rm & lt_mask)] = o; }
    w += __popc(rm);
  };
  OpenEnt v = {kInf64, kInf64};
  if (lane < st.nn) v = pl.near[lane];
  for (int base = 0; base < st.nn; base += 32) {
    const int i = base + lane;
    OpenEnt vn = {kInf64, kInf64};
    if (i + 32 < st.nn) vn = pl.near[i + 32];           // prefetch the next chunk
    const Key kv = {v.f, v.k};
    const bool live = i < st.nn && !stale_entry(v, pl);
    const bool in = live && klt(kv, B);
    const bool dem = live && !in && !klt(kv, st.F2);
    const bool keep = live && !in && !dem;
    const unsigned bm = __ballot_sync(0xffffffffu, in);
    const unsigned km = __ballot_sync(0xffffffffu, keep);
    const unsigned dm = __ballot_sync(0xffffffffu, dem);
    nband += __popc(bm);
    if (in) pl.stg[ns + __popc(bm & lt_mask)] = v;
    ns += __popc(bm);
    if (dem && st.nf + __popc(dm) <= pl.far_cap) pl.far[st.nf + __popc(dm & lt_mask)] = v;
    st.nf += __popc(dm);
    __syncwarp();
    if (keep) pl.near[w + __popc(km & lt_mask)] = v;    // compaction never passes the reads
    w += __popc(km);
    while (ns >= 32) merge(32);
    v = vn;
  }
  if (ns > 0) merge(ns);
  st.nn = w;
  st.h = __popc(__ballot_sync(0xffffffffu, acc.f != kInf64));
  st.hd = acc;
  if (rejected) {
    // T = successor of the largest head key
    const Key mx = shfl_key(acc, 31);
    st.T.k = mx.k + 1ull;
    st.T.f = mx.f + (st.T.k == 0ull ? 1ull : 0ull);
  } else {
    st.T = B;
  }
  if (nband > 48) st.delta *= 0.5;
  else if (nband < 16 && st.delta < 64.0) st.delta *= 2.0;
  if (st.nn > pl.NC / 2) st.delta2 = fmax(st.delta2 * 0.5, st.delta);
  if (st.nf > pl.far_cap) st.err = 1;
  __syncwarp();
  return st;
}

// Search-local cell state lives in 8x8-cell tiles: g (f64, +inf when unset)
// and the move byte.  A tile gets a slot the first time the search writes one
// of its cells; slots [0, S) are in shared memory, the rest in the warp's
// global backing store.  The slot is part of every key, so a pop addresses
// g(x) and moves(x) directly.  Key k2 layout (ordering = (h, row, col)):
//   [63:41] floor(h * 4096)   distinct octile h differ by > 3.5e-4, so this is
//                             injective and monotone on the values that occur
//   [40:21] row << cb | col   [20:5] tile slot  [4:0] 0
// cb = column bits: 10 for grids up to 1024 x 1024 (row and col 10 bits each); a wider
// grid (Traverse strips: 120 m x 10 m at 0.1 m = 1200 x 100) takes cb = ceil(log2 nx) and
// leaves 20 - cb bits to the row -- (row << cb | col) orders like (row, col) either way.
// The host admits grids with ceil(log2 nx) + ceil(log2 ny) <= 20 and octile h < 2048
// (23 bits of floor(h * 4096)); crowd.py checks both.
constexpr u64 kCellMask2 = ((1ull << 20) - 1ull) << 21;
constexpr unsigned kNoSlot = 0xFFFFu;

CW_DEV u64 make_key2(double h, int r, int c, int slot, int cb) {
  return ((u64)(h * 4096.0) << 41) | ((u64)((r << cb) | c) << 21) | ((u64)slot << 5);
}

// bytes of the per-warp global scratch for an nx x ny grid with S shared
// slots: overflow tiles (g f64 + move byte), parent i32 per cell, slot->tile map
CW_HD size_t astar_slot_bytes(int nx, int ny, int S) {
  const size_t nt = (size_t)((nx + 7) / 8) * ((ny + 7) / 8);
  // global tiles: every tile at slot >= S plus the shared pool's S slot ids (a
  // search whose pool runs dry continues here under the same ids)
  const size_t b = (nt + (size_t)S) * 64 * 9 + (size_t)nx * ny * 4 + (nt + (size_t)S) * 4;
  return (b + 255) & ~(size_t)255;
}

// Launch shape of k_astar: one CTA per SM with W search warps (one per SM
// sub-partition).  Each warp owns a near pool (NC x 16 B), a 64-entry staging
// area and a tile map (2 B per tile); the NS tile slots of 576 B (64 x f64 g +
// 64 move bytes) form one pool shared by the CTA's warps (a locked stack of
// free slot ids), so a lone long search can use nearly all of it.  W = 1 is
// the latency shape (few searches per tick: the tick waits on the longest
// one), W = 4 the throughput shape (many searches per tick).
#ifndef CW_ASTAR_WARPS
#define CW_ASTAR_WARPS 4
#endif
constexpr int kAstarWarps = CW_ASTAR_WARPS;   // scratch is sized for the larger shape

struct AstarShape {
  int NC, NS, W;
  size_t per_warp;   // bytes of one warp's private block
  size_t smem;
};

CW_HD AstarShape astar_shape(int nx, int ny, int W, int budget_kb = 0) {
  const int nt = ((nx + 7) / 8) * ((ny + 7) / 8);
  const int NC = W == 1 ? 1024 : 512;
  const size_t per_warp = (size_t)(NC + 64) * 16 + (((size_t)nt * 2 + 15) & ~(size_t)15);
  // W = 1 leaves ~30 KB of the SM's 228 KB for k_orca CTAs running beside it
  if (budget_kb <= 0) budget_kb = W == 1 ? 196 : 220;
  const size_t budget = (size_t)budget_kb * 1024, head = 16;   // lock + stack top
  const size_t fixed = W * per_warp + head;
  int NS = budget > fixed ? (int)((budget - fixed) / (576 + 2)) : 0;
  NS = NS > W * nt ? W * nt : NS;
  NS = NS > 65535 ? 65535 : NS;
  const size_t stack = ((size_t)NS * 2 + 15) & ~(size_t)15;
  return {NC, NS, W, per_warp, fixed + stack + (size_t)NS * 576};
}

// Largest shared pool (slot ids) of the search shapes in use (1, 2 or 4 warps per CTA);
// launches clamp NS to it.
CW_HD int astar_ns_cap(int nx, int ny) {
  const int a = astar_shape(nx, ny, 1).NS, b = astar_shape(nx, ny, 2).NS;
  const int c = astar_shape(nx, ny, kAstarWarps).NS;
  return a > b ? (a > c ? a : c) : (b > c ? b : c);
}

// Per-warp global scratch stride: sized for the largest pool of the shapes.
CW_HD size_t astar_slot_stride(int nx, int ny) { return astar_slot_bytes(nx, ny, astar_ns_cap(nx, ny)); }

// Per-CTA layout shared by the two search instantiations.
struct SearchEnv {
  int nx, ny, N, TW, NT, NS;
  uint16_t* tmap;        // shared, this warp: tile -> slot (kNoSlot when unused)
  double* gts;           // shared, CTA pool: NS x 64 g
  uint8_t* mts;          // shared, CTA pool: NS x 64 move bytes
  uint16_t* free_ids;    // shared, CTA pool: stack of free slot ids
  int* pool_lock;        // shared: [0] lock, [1] stack top
  uint16_t* wbuf;        // shared, this warp: 8 freshly taken slot ids
  double* gtg;           // global, this warp: NT x 64 g (all-global instantiation)
  uint8_t* mtg;          // global, this warp: NT x 64 move bytes
  int32_t* parent;       // global, this warp: N
  int32_t* s2t;          // global, this warp: allocation k -> slot << 16 | tile
  long long* trace;      // debug (counters[15]): expanded cell + f bits of one search
#ifdef CW_ASTAR_PHASES
  long long* ph;         // debug: [head inserts, insert cycles, held pops, refill cycles]
#endif
};

// Take n slots from the CTA pool (lane 0; false if it holds fewer).
CW_DEV bool pool_take(const SearchEnv& E, int n, uint16_t* out) {
  while (atomicCAS(&E.pool_lock[0], 0, 1) != 0) {}
  __threadfence_block();
  volatile int* top_p = &E.pool_lock[1];
  volatile uint16_t* ids = E.free_ids;
  const int top = *top_p;
  const bool ok = top >= n;
  if (ok) {
    for (int i = 0; i < n; ++i) out[i] = ids[top - 1 - i];
    *top_p = top - n;
  }
  __threadfence_block();
  atomicExch(&E.pool_lock[0], 0);
  return ok;
}

// One search, paths.astar_path (paths.py:48-87).  kGlob = false keeps every
// tile in the CTA's shared pool and returns -2 when the pool runs dry (the
// caller releases and retries with kGlob = true, all tiles in the warp's global
// backing store).  Returns 1 found, 0 no path, -1 open-set overflow; `used` =
// tiles handed out (recorded in s2t).
// Resumable search state: a shared-memory search whose tile pool runs dry hands
// its open set over (the popped, not yet expanded cell back in the head) and
// continues all-global on the same open set and the same slot ids -- the used
// tiles are copied to the global store at their slot index first -- instead of
// starting over.  New global tiles then take slots slot_base + k.
struct Resume {
  OpenSet st;
  int active;      // st holds a search in progress
  int slot_base;   // first slot id of new global tiles
  int gcount;      // global tiles handed out so far
};

// kWide: the grid's key2 cell field is not the default 10 / 10 split (pl.cb != 10); the
// default instantiation decodes with constant shifts (the per-expansion critical path)
template <bool kGlob, bool kWide = false>
CW_DEV int run_search(const SearchEnv& E, Pools& pl, const uint8_t* mvt, int start, int goal,
                      double& delta, double& delta2, unsigned& s_exp, int& used, int lane, Resume& rs,
                      bool cg) {
  const int cb = kWide ? (int)pl.cb : 10;
  double* const gt = kGlob ? E.gtg : E.gts;
  uint8_t* const mt = kGlob ? E.mtg : E.mts;
  const int nx = E.nx, ny = E.ny, TW = E.TW, NT = E.NT, NC = pl.NC;
  const unsigned lt_mask = (1u << lane) - 1u;
  // paths.py:75 move order: N S W E, then the diagonals (nibble per lane, +1)
  const int dr_ = lane < 8 ? (int)((0x22001120u >> (4 * lane)) & 0xF) - 1 : 0;
  const int dc_ = lane < 8 ? (int)((0x20202011u >> (4 * lane)) & 0xF) - 1 : 0;
  const unsigned lanebit = lane < 8 ? 1u << lane : 0u;
  const double w_ = lane < 4 ? 1.0 : kSqrt2;
  const int sr = start / nx, sc = start - sr * nx;
  const int gr = goal / nx, gc = goal - gr * nx;
  pl.gt = gt;
  pl.gr = gr;
  pl.gc = gc;
  // tile t gets slot s: g = +inf, move bytes copied from the env table
  auto new_tile = [&](int t, int s) {
    if (lane == 0) E.s2t[used] = (s << 16) | t;
    ++used;
    double* gp = gt + (size_t)s * 64;
    uint8_t* mp = mt + (size_t)s * 64;
    const int r0 = (t / TW) * 8, c0 = (t % TW) * 8;
    gp[lane] = CUDART_INF;
    gp[lane + 32] = CUDART_INF;
    for (int j = lane; j < 64; j += 32) {
      const int rr = r0 + (j >> 3), cc = c0 + (j & 7);
      mp[j] = (rr < ny && cc < nx) ? ld_grid(mvt + rr * nx + cc, cg) : (uint8_t)0;
    }
    if (lane == 0) E.tmap[t] = (uint16_t)s;
    return s;
  };
  // n slot ids for this warp: sequential (all-global) or from the CTA pool
  auto take = [&](int n) -> bool {
    if (kGlob) return true;   // slots rs.slot_base + rs.gcount ... (see new_tile calls)
    bool ok = false;
    if (lane == 0) ok = pool_take(E, n, E.wbuf);
    ok = __shfl_sync(0xffffffffu, ok, 0);
    __syncwarp();
    return ok;
  };
  OpenSet st;
  if (kGlob && rs.active) {
    st = rs.st;                 // continue the handed-over search
    rs.active = 0;
  } else {
    const double h0 = octile(sr, sc, gr, gc);
    if (!take(1)) return -2;
    const int s0 = new_tile((sr >> 3) * TW + (sc >> 3), kGlob ? rs.slot_base + rs.gcount++ : (int)E.wbuf[0]);
    __syncwarp();
    if (lane == 0) {
      gt[(size_t)s0 * 64 + (sr & 7) * 8 + (sc & 7)] = 0.0;
      E.parent[start] = -1;
    }
    st.hd = key_inf();
    if (lane == 0) st.hd = {(u64)__double_as_longlong(h0), make_key2(h0, sr, sc, s0, cb)};
    st.T = key_inf();
    st.F2 = {f_plus((u64)__double_as_longlong(h0), delta2), 0ull};
    st.delta = delta;
    st.delta2 = delta2;
    st.h = 1;
    st.nn = 0;
    st.nf = 0;
    st.err = 0;
  }
  int found = 0;
  // Held pop: in ~70 % of expansions exactly one new key is below the head's minimum
  // (the plateau descent toward the goal; tools/astar_faststat.py) -- that key is the
  // next pop (every head key > it, every pool key >= T > it), so it is kept aside
  // instead of being inserted into the head and popped again.
  bool held = false;
  Key hk = key_inf();
  __syncwarp();
  while (true) {
    if (!held && st.h == 0) {
      if (st.nn == 0 && st.nf == 0) break;
#ifdef CW_ASTAR_PHASES
      const long long tr0 = clock64();
      st = refill(st, pl, lane);
      E.ph[3] += clock64() - tr0;
#else
      st = refill(st, pl, lane);
#endif
      if (st.err) { found = -1; break; }
      continue;
    }
    // ---------------- pop the minimum: the held key, else the head's first
    const bool from_held = held;
    Key popped, h0;   // h0: the head's minimum after the pop (+inf if empty)
    if (from_held) {
      popped = hk;
      h0 = shfl_key(st.hd, 0);
      held = false;
    } else {
      popped = shfl_key(st.hd, 0);
      h0 = shfl_key(st.hd, 1);
      const Key nxt = shfl_key_down(st.hd, 1);
      st.hd = lane < 31 ? nxt : key_inf();
      st.h -= 1;
    }
    const u64 topk = popped.k;
    const int r = key_row(topk, cb), c = key_col(topk, cb);
    const int sx = (int)(topk >> 5) & 0xFFFF;
    const int x = r * nx + c;
    const int ix = sx * 64 + (r & 7) * 8 + (c & 7);
    // g(x), moves(x) and the neighbours' tile slots are read together
    const double gx = gt[ix];
    const unsigned mv = mt[ix];
    const int rr = r + dr_, cc = c + dc_;
    const bool legal = (mv & lanebit) != 0u;
    // the tile-map read does not wait for the move byte (index clamped)
    const int ty = min(max((rr >> 3) * TW + (cc >> 3), 0), NT - 1);
    const int iy = (rr & 7) * 8 + (cc & 7);
    const int sy0 = (int)E.tmap[ty];
    int sy = legal ? sy0 : (int)kNoSlot;
    const double hh = octile(rr, cc, gr, gc);
#ifdef CW_ASTAR_TRACE   // expansion-order trace for tools/astar_trace.py (debug builds only)
    if (E.trace && lane == 0 && s_exp < (1u << 20)) {
      E.trace[2 * s_exp] = x;
      E.trace[2 * s_exp + 1] = __double_as_longlong(gx);
    }
#endif
    if (x == goal) { found = 1; break; }
    // No stale test (paths.py:70-71) is needed here: the head never holds a
    // stale entry (refills drop them, decrease-keys evict the old head copy),
    // and re-expanding a cell with its current g would relax nothing anyway.
    ++s_exp;
    const double gy = sy != (int)kNoSlot ? gt[(size_t)sy * 64 + iy] : CUDART_INF;
    const double ng = gx + w_;
    const bool push = legal & (ng < gy - 1e-12);
    const bool fresh = gy == CUDART_INF;
    // routing never looks at the tile slot ((h, row, col) is unique per
    // cell), so it is decided together with the first-write test
    const Key ne0 = {(u64)__double_as_longlong(ng + hh), make_key2(hh, rr, cc, 0, cb)};
    if (st.nn + 16 > NC) {
      st = split_near(st, pl, lane);
      if (st.err) { found = -1; break; }
    }
    const bool ltT = klt(ne0, st.T), ltF2 = klt(ne0, st.F2);
    const bool need = push & (sy == (int)kNoSlot);
    const bool toH = push & ltT;
    const bool toN = push & !ltT & ltF2;
    const bool toF = push & !ltT & !ltF2;
    const unsigned nm = __ballot_sync(0xffffffffu, need);
    unsigned mh = __ballot_sync(0xffffffffu, toH);
    const unsigned nmk = __ballot_sync(0xffffffffu, toN);
    const unsigned fmk = __ballot_sync(0xffffffffu, toF);
    const unsigned decm = __ballot_sync(0xffffffffu, push & !fresh);
    // first write into a tile: hand out slots (one per distinct tile)
    if (nm) {
      const unsigned peers = __match_any_sync(0xffffffffu, need ? ty : -1 - lane);
      const int leader = __ffs(peers) - 1;
      const unsigned lm = __ballot_sync(0xffffffffu, need && leader == lane);
      if (!take(__popc(lm))) {   // only when !kGlob: hand the search over (see Resume)
        if (from_held && st.h == 32) {   // the popped key goes back into a full head
          const Key ev = shfl_key(st.hd, 31);
          const bool evn = klt(ev, st.F2);
          if (lane == 0) {
            OpenEnt o = {ev.f, ev.k};
            if (evn) pl.near[st.nn] = o;
            else pl.far[st.nf] = o;
          }
          st.nn += evn;
          st.nf += !evn;
          st.T = ev;
          st.h = 31;
        }
        const Key up = shfl_key_up(st.hd, 1);
        st.hd = lane == 0 ? popped : up;
        st.h += 1;
        --s_exp;
        rs.st = st;
        rs.active = 1;
        found = -2;
        break;
      }
      unsigned L = lm;
      int mine = 0, k = 0;
      while (L) {
        const int ld = __ffs(L) - 1;
        L &= L - 1;
        const int s = new_tile(__shfl_sync(0xffffffffu, ty, ld), kGlob ? rs.slot_base + rs.gcount++ : (int)E.wbuf[k]);
        ++k;
        if (lane == ld) mine = s;
      }
      const int got = __shfl_sync(0xffffffffu, mine, leader);
      if (need) sy = got;
      __syncwarp();
    }
    if (push) {
      gt[(size_t)sy * 64 + iy] = ng;
      E.parent[rr * nx + cc] = x;
    }
    const Key ne = {ne0.f, ne0.k | ((u64)sy << 5)};
    if (st.nf + 16 > pl.far_cap) { found = -1; break; }
    if (toN) { OpenEnt o = {ne.f, ne.k}; pl.near[st.nn + __popc(nmk & lt_mask)] = o; }
    if (toF) { OpenEnt o = {ne.f, ne.k}; pl.far[st.nf + __popc(fmk & lt_mask)] = o; }
    st.nn += __popc(nmk);
    st.nf += __popc(fmk);
#ifndef CW_ASTAR_NO_HOLD
    {
      const unsigned lo = __ballot_sync(0xffffffffu, toH & klt(ne0, h0));
      if (__popc(lo) == 1) {
        const int s = __ffs(lo) - 1;
        mh &= ~(1u << s);
        hk = shfl_key(ne, s);
        if ((decm >> s) & 1u) {   // its stale entry leaves the head (see below)
          const unsigned om = __ballot_sync(0xffffffffu, ((st.hd.k ^ hk.k) & kCellMask2) == 0ull);
          if (om) {
            const int L = __ffs(om) - 1;
            const Key dn = shfl_key_down(st.hd, 1);
            if (lane >= L) st.hd = lane < st.h - 1 ? dn : key_inf();
            st.h -= 1;
          }
        }
        held = true;
      }
    }
#endif
#ifdef CW_ASTAR_PHASES
    E.ph[0] += __popc(mh);
    E.ph[2] += held;
    const long long ti0 = clock64();
#endif
    while (mh) {
      const int s = __ffs(mh) - 1;
      mh &= mh - 1;
      const Key v = shfl_key(ne, s);
      if ((decm >> s) & 1u) {
        // decrease-key: the cell's previous (now stale) entry leaves the head
        // if it is there -- a stale pop is a no-op (paths.py:70-71)
        const unsigned om = __ballot_sync(0xffffffffu, ((st.hd.k ^ v.k) & kCellMask2) == 0ull);
        if (om) {
          const int L = __ffs(om) - 1;
          const Key dn = shfl_key_down(st.hd, 1);
          if (lane >= L) st.hd = lane < st.h - 1 ? dn : key_inf();
          st.h -= 1;
        }
      }
      if (!klt(v, st.T)) {
        // an eviction earlier in this loop lowered T to or below v: v now
        // belongs to the pools (the head must stay below every pool key)
        const bool vn = klt(v, st.F2);
        if (lane == 0) {
          OpenEnt o = {v.f, v.k};
          if (vn) pl.near[st.nn] = o;
          else pl.far[st.nf] = o;
        }
        st.nn += vn;
        st.nf += !vn;
        continue;
      }
      const Key up = shfl_key_up(st.hd, 1);
      const int p = __popc(__ballot_sync(0xffffffffu, klt(st.hd, v)));   // +inf beyond h
      if (st.h == 32) {
        // full head: its largest key (or v itself) moves to the pool and bounds it
        const Key ev = p == 32 ? v : shfl_key(st.hd, 31);
        const bool evn = klt(ev, st.F2);
        if (lane == 0) {
          OpenEnt o = {ev.f, ev.k};
          if (evn) pl.near[st.nn] = o;
          else pl.far[st.nf] = o;
        }
        st.nn += evn;
        st.nf += !evn;
        st.T = ev;
        if (p == 32) continue;
        st.h = 31;
      }
      if (lane > p && lane <= st.h) st.hd = up;
      if (lane == p) st.hd = v;
      st.h += 1;
    }
#ifdef CW_ASTAR_PHASES
    E.ph[1] += clock64() - ti0;
#endif
    __syncwarp();
  }
  delta = st.delta;
  delta2 = st.delta2;
  return found;
}

// k_astar: persistent warps pull requests queued by k_guide and run
// paths.astar_path exactly; results go to the agent's path (field.py:204-212).
// Unreachable goals (different 4-connected component, see k_reach) return None
// without searching -- the reference exhausts the component and returns None.
// kRing: persistent search server of cw_crowd_run -- requests come from the
// run ring (runq.cuh) until q->shutdown, and each finished search decrements
// its env's pending count.
// sp.mode (SpecArgs, crowd.cu): 0 plain; 1 the tick's searches, each looked up in the
// next-tick prefetch cache first; 2 a speculative batch (requests from the dry guidance
// pass, results into the cache, its own scratch, no state or error-flag writes).
template <int W, bool kRing>
__global__ void __launch_bounds__(32 * W, 1) k_astar(cw_crowd_params P, cw_crowd_state S, int NC, int NS,
                                                     RunArgs ra, SpecArgs sp) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gw = blockIdx.x * kAstarWarps + w;       // global search-warp id (scratch slot)
  SearchEnv E;
  E.nx = P.nx;
  E.ny = P.ny;
  E.N = P.nx * P.ny;
  E.TW = (P.nx + 7) >> 3;
  E.NT = E.TW * ((P.ny + 7) >> 3);
  E.NS = NS;
  const int nx = E.nx, N = E.N, NT = E.NT;
  const AstarReq* reqs = reinterpret_cast<const AstarReq*>(S.astar_req);
  const AstarShape shp = astar_shape(P.nx, P.ny, W);
  unsigned char* const wblk = sm + (size_t)w * shp.per_warp;
  Pools pl;
  pl.near = reinterpret_cast<OpenEnt*>(wblk);
  pl.stg = pl.near + NC;
  const bool spec = !kRing && sp.mode == 2;
  const size_t slot = spec ? (size_t)sm_id() * kAstarWarps + w : (size_t)gw;
  pl.far = (spec ? sp.heap : reinterpret_cast<OpenEnt*>(S.astar_heap)) + slot * P.heap_cap;
  pl.NC = NC;
  pl.far_cap = P.heap_cap;
  pl.cb = key_col_bits(P.nx, P.ny);

  E.tmap = reinterpret_cast<uint16_t*>(pl.stg + 64);
  unsigned char* const pool = sm + (size_t)W * shp.per_warp;
  E.pool_lock = reinterpret_cast<int*>(pool);
  E.free_ids = reinterpret_cast<uint16_t*>(pool + 16);
  E.gts = reinterpret_cast<double*>(pool + 16 + (((size_t)NS * 2 + 15) & ~(size_t)15));
  E.mts = reinterpret_cast<uint8_t*>(E.gts + (size_t)NS * 64);
  E.wbuf = reinterpret_cast<uint16_t*>(pl.stg) + 0;   // staging area doubles as the slot buffer
  unsigned char* const gbase = (spec ? sp.rec : reinterpret_cast<unsigned char*>(S.astar_rec)) +
                               slot * astar_slot_stride(nx, E.ny);
  const int NTG = NT + astar_ns_cap(nx, E.ny);   // global store: every tile + the pool's slot ids
  E.gtg = reinterpret_cast<double*>(gbase);
  E.mtg = gbase + (size_t)NTG * 64 * 8;
  E.parent = reinterpret_cast<int32_t*>(E.mtg + (size_t)NTG * 64);
  E.s2t = E.parent + N;
  for (int t = lane; t < NT; t += 32) E.tmap[t] = kNoSlot;
  for (int i = threadIdx.x; i < NS; i += blockDim.x) E.free_ids[i] = (uint16_t)i;
  if (threadIdx.x == 0) { E.pool_lock[0] = 0; E.pool_lock[1] = NS; }
  __syncthreads();
  // early commit: the commit pass (k_orca_ec) may start once every search CTA is here
  if (!kRing && sp.mode == 1 && sp.pend) asm volatile("griddepcontrol.launch_dependents;");
  long long* const dbg = (!kRing && !spec && S.counters && S.counters[14])
                             ? reinterpret_cast<long long*>(S.counters[14]) : nullptr;
  long long* const trace = (!kRing && !spec && S.counters && S.counters[15])
                               ? reinterpret_cast<long long*>(S.counters[15]) : nullptr;
  long long t_max = 0, t_sum = 0;
  unsigned long long n_exp = 0, n_glob = 0;
  double delta = 1.0, delta2 = 4.0;   // adaptive band widths, carried across searches
  while (true) {
    int q = 0;
    AstarReq R;
    if (kRing) {
      int ok = 0;
      if (lane == 0) ok = ring_pop(ra, R);
      if (!__shfl_sync(0xffffffffu, ok, 0)) break;
      R.env = __shfl_sync(0xffffffffu, R.env, 0);
      R.agent = __shfl_sync(0xffffffffu, R.agent, 0);
      R.start = __shfl_sync(0xffffffffu, R.start, 0);
      R.goal = __shfl_sync(0xffffffffu, R.goal, 0);
    } else if (spec) {
      // take the next queued item (the late committers may still be adding some: poll
      // until they are all done, bounded by kSpecIdle); a prediction is this warp's
      // once its entry moves queued -> running
      int ok = 0;
      if (lane == 0) {
        const long long idle0 = clock64();
        q = -1;
        while (true) {
          const int taken = *(volatile int*)&sp.qn[1];
          if (taken < ld_acquire_i32(&sp.qn[0])) {
            if (atomicCAS(&sp.qn[1], taken, taken + 1) == taken) { q = taken; break; }
            continue;
          }
          if (ld_acquire_i32(&sp.qn[3]) >= *(volatile int*)&sp.qn[2] &&
              *(volatile int*)&sp.qn[1] >= ld_acquire_i32(&sp.qn[0]))
            break;   // every producer is done and the queue is drained
          if (clock64() - idle0 > kSpecIdle) break;
          __nanosleep(512);
        }
        if (q >= 0) {
          while (ld_acquire_i32(&sp.qr[q]) != (int)sp.tag) __nanosleep(64);   // item written
          R = sp.q[q];
          const unsigned long long t = sp.tag << 8;
          ok = atomicCAS(&sp.ent[(size_t)R.env * P.A + R.agent].word, t | kSpQueued, t | kSpRunning) ==
               (t | kSpQueued) ? 1 : 2;
        }
      }
      ok = __shfl_sync(0xffffffffu, ok, 0);
      if (ok == 0) break;
      if (ok == 2) continue;
      R.env = __shfl_sync(0xffffffffu, R.env, 0);
      R.agent = __shfl_sync(0xffffffffu, R.agent, 0);
      R.start = __shfl_sync(0xffffffffu, R.start, 0);
      R.goal = __shfl_sync(0xffffffffu, R.goal, 0);
    } else {
      if (lane == 0) q = atomicAdd(&S.flags[5], 1);
      q = __shfl_sync(0xffffffffu, q, 0);
      if (q >= *(volatile int*)&S.flags[4]) break;
      R = reqs[q];
    }
    const long long t0 = clock64();
    E.trace = (trace && q == 0) ? trace : nullptr;
#ifdef CW_ASTAR_PHASES
    long long phv[4] = {0, 0, 0, 0};
    E.ph = phv;
#endif

    const int e = R.env;
    const uint8_t* mvt = S.moves + (size_t)e * N;
    const uint8_t* lab = S.labels + (size_t)e * N;
    const int32_t* reach = S.reach + (size_t)e * N;
    const int start = R.start, goal = R.goal;
    int found = 0;  // 1 found, 0 none, -1 open-set overflow
    int used = 0;   // tile slots handed out
    unsigned s_exp = 0;
    bool pooled = true;   // tiles came from the CTA pool (false after an all-global retry)
    auto release = [&]() {
      __syncwarp();
      if (lane == 0 && pooled && used) {
        while (atomicCAS(&E.pool_lock[0], 0, 1) != 0) {}
        __threadfence_block();
      }
      __syncwarp();
      const int top = pooled ? *(volatile int*)&E.pool_lock[1] : 0;
      for (int k = lane; k < used; k += 32) {
        const int v = E.s2t[k];
        E.tmap[v & 0xFFFF] = kNoSlot;
        if (pooled) ((volatile uint16_t*)E.free_ids)[top + k] = (uint16_t)(v >> 16);
      }
      __syncwarp();
      if (lane == 0 && pooled && used) {
        *(volatile int*)&E.pool_lock[1] = top + used;
        __threadfence_block();
        atomicExch(&E.pool_lock[0], 0);
      }
      __syncwarp();
      used = 0;
    };
    const size_t ia = (size_t)e * P.A + R.agent;
    int32_t* cells = (spec ? sp.cells : S.path_cells) + ia * P.path_cap;
    // 1: the cache entry holds this search's result (cells copied below)
    int hit = 0, h_count = 0, h_found = 0, h_over = 0, ep = 0;
    if (spec) {
      if (lane == 0) ep = ld_acquire_i32(&sp.epoch[e]);   // before any read of the env's grid
      __syncwarp();
    } else if (!kRing && sp.mode == 1 && lane == 0) {
      SpecEnt* en = sp.ent + ia;
      const int cur = *(volatile const int*)&sp.epoch[e];
      bool waited = false;
      while (true) {
        const unsigned long long wd = *(volatile unsigned long long*)&en->word;
        const int st = (int)(wd & 0xFFull);
        const bool same = *(volatile int*)&en->start == start && *(volatile int*)&en->goal == goal;
        const unsigned long long claimed = (wd & ~0xFFull) | kSpClaimed;
        if (st == kSpQueued) {   // not started: search it here (a stale prediction is dropped)
          if (atomicCAS(&en->word, wd, claimed) != wd) continue;
          if (same) atomicAdd(&sp.stats[3], 1ull);
          break;
        }
        if (!same) break;
        if (st == kSpRunning) {
          if (!waited) atomicAdd(&sp.stats[2], 1ull);
          waited = true;
          __nanosleep(256);
          continue;
        }
        if (st == kSpDone) {
          __threadfence();
          if (*(volatile int*)&en->epoch == cur) {
            atomicAdd(&sp.stats[1], 1ull);
            hit = 1;
            h_count = *(volatile int*)&en->count;
            h_found = *(volatile int*)&en->found;
            h_over = *(volatile int*)&en->over;
          }
        }
        break;
      }
    }
    if (!kRing && sp.mode == 1) {
      hit = __shfl_sync(0xffffffffu, hit, 0);
      if (hit) {
        h_count = __shfl_sync(0xffffffffu, h_count, 0);
        h_found = __shfl_sync(0xffffffffu, h_found, 0);
        h_over = __shfl_sync(0xffffffffu, h_over, 0);
        if (h_found == 1 && !h_over) {
          const int32_t* src = sp.cells + ia * P.path_cap;
          for (int k = P.path_cap - h_count + lane; k < P.path_cap; k += 32) cells[k] = src[k];
        }
        found = h_found;
      }
    }
    // a speculative batch may outlive a grid rewrite of its env (a later generation):
    // its grid reads bypass L1, which may still hold the earlier generation's lines
    if (!hit && ld_grid(lab + start, spec) != L_OBSTACLE && ld_grid(lab + goal, spec) != L_OBSTACLE &&
        ld_grid(reach + start, spec) == ld_grid(reach + goal, spec)) {
      Resume rs;
      rs.active = 0;
      rs.slot_base = 0;
      rs.gcount = 0;
      found = (kRing || pl.cb == 10)   // the run's server: default packing only (crowd.py)
                  ? run_search<false>(E, pl, mvt, start, goal, delta, delta2, s_exp, used, lane, rs, spec)
                  : run_search<false, true>(E, pl, mvt, start, goal, delta, delta2, s_exp, used, lane, rs, spec);
      if (found == -2 && rs.active) {
        // the shared tile pool ran dry mid-search: move the used tiles to the
        // global store at their slot ids, give the slots back to the CTA pool
        // and continue all-global on the same open set
        for (int k = 0; k < used; ++k) {
          const int sl = E.s2t[k] >> 16;
          E.gtg[(size_t)sl * 64 + lane] = E.gts[(size_t)sl * 64 + lane];
          E.gtg[(size_t)sl * 64 + lane + 32] = E.gts[(size_t)sl * 64 + lane + 32];
          E.mtg[(size_t)sl * 64 + lane] = E.mts[(size_t)sl * 64 + lane];
          E.mtg[(size_t)sl * 64 + lane + 32] = E.mts[(size_t)sl * 64 + lane + 32];
        }
        __syncwarp();
        if (lane == 0) {
          while (atomicCAS(&E.pool_lock[0], 0, 1) != 0) {}
          __threadfence_block();
        }
        __syncwarp();
        const int top = *(volatile int*)&E.pool_lock[1];
        for (int k = lane; k < used; k += 32)
          ((volatile uint16_t*)E.free_ids)[top + k] = (uint16_t)(E.s2t[k] >> 16);
        __syncwarp();
        if (lane == 0) {
          *(volatile int*)&E.pool_lock[1] = top + used;
          __threadfence_block();
          atomicExch(&E.pool_lock[0], 0);
        }
        __syncwarp();
        pooled = false;   // the final release only clears the tile map
        rs.slot_base = NS;
        rs.gcount = 0;
        ++n_glob;
        found = (kRing || pl.cb == 10)
                    ? run_search<true>(E, pl, mvt, start, goal, delta, delta2, s_exp, used, lane, rs, spec)
                    : run_search<true, true>(E, pl, mvt, start, goal, delta, delta2, s_exp, used, lane, rs, spec);
      } else if (found == -2) {   // no tile even for the start cell: all-global from scratch
        release();
        pooled = false;
        s_exp = 0;
        ++n_glob;
        rs.active = 0;
        rs.slot_base = 0;
        rs.gcount = 0;
        found = (kRing || pl.cb == 10)
                    ? run_search<true>(E, pl, mvt, start, goal, delta, delta2, s_exp, used, lane, rs, spec)
                    : run_search<true, true>(E, pl, mvt, start, goal, delta, delta2, s_exp, used, lane, rs, spec);
      }
    }
    // ---- write the guidance result (field.py:204-212)
    int pn = 1, head = 0;
    double wx = 0.0, wy = 0.0;
    if (!spec) {
      wx = S.goal[ia * 2];
      wy = S.goal[ia * 2 + 1];
    }
    if (found == -1 && lane == 0 && !spec) atomicCAS(&S.flags[1], 0, (int)CW_E_HEAPCAP);
    if (found == 1) {
      // one walk of the parent chain (goal -> start, L2 pointer chasing), writing the
      // cells back to front: the path is cells[head .. path_cap - 1] in forward order
      int count = h_count, over = h_over;
      if (lane == 0 && !hit) {
        for (int v = goal; v != start; v = E.parent[v]) {
          if (count == P.path_cap) { over = 1; break; }
          cells[P.path_cap - 1 - count] = v;
          ++count;
        }
      }
      count = __shfl_sync(0xffffffffu, count, 0);
      over = __shfl_sync(0xffffffffu, over, 0);
      __syncwarp();
      if (spec) {
        h_count = count;
        h_over = over;
      } else if (over) {
        if (lane == 0) atomicCAS(&S.flags[1], 0, (int)CW_E_PATHCAP);
      } else if (count >= 1) {
        pn = count + 1;
        head = P.path_cap - count;
        const int f0 = cells[head];
        wx = ((double)(f0 % nx) + 0.5) * P.res;
        wy = ((double)(f0 / nx) + 0.5) * P.res;
      }
    }
    if (spec) {   // publish the prediction (the cells are written above)
      if (lane == 0) {
        SpecEnt* en = sp.ent + ia;
        en->epoch = ep;
        en->count = h_count;
        en->found = found;
        en->over = h_over;
        __threadfence();
        atomicExch(&en->word, (sp.tag << 8) | (found == -1 ? kSpFailed : kSpDone));
      }
    } else if (lane == 0) {
      S.path_head[ia] = head;
      S.path_n[ia] = pn;
      S.waypoint[ia * 2] = wx;
      S.waypoint[ia * 2 + 1] = wy;
    }
    if (!kRing && !spec && sp.mode == 1 && sp.pend) {   // early commit: one search of env e less
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        atomicSub(&sp.pend[e], 1);
      }
    }
    const int used_final = used;
    release();
    if (kRing) {   // publish the result, then count the env's search as done
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        if (atomicSub(&ra.pending[e], 1) == 1) {   // the env's last search
          if (ra.trace) {
            long long* tr = ra.trace + (size_t)e * 8;
            const long long now = global_ns();
            tr[kTrSearchWait] += now - tr[kTrMark];
            tr[kTrMark] = now;
          }
          urgent_push(ra, e);
        }
      }
    }
    const long long dt = clock64() - t0;
    if (dbg && lane == 0) {
      long long* d = dbg + (size_t)q * 8;
      d[0] = dt; d[1] = s_exp; d[2] = e; d[3] = used_final;
#ifdef CW_ASTAR_PHASES
      d[4] = phv[0]; d[5] = phv[1]; d[6] = phv[2]; d[7] = phv[3];
#endif
    }
    n_exp += s_exp;
    t_sum += dt;
    t_max = max(t_max, dt);
  }
  if (lane == 0 && S.counters && !spec) {
    if (n_exp) atomicAdd((unsigned long long*)&S.counters[0], n_exp);
    if (t_sum) atomicAdd((unsigned long long*)&S.counters[4], (unsigned long long)t_sum);
    if (t_max) atomicMax((unsigned long long*)&S.counters[5], (unsigned long long)t_max);
    if (n_glob) atomicAdd((unsigned long long*)&S.counters[10], n_glob);
  }
}

}  // namespace cw
