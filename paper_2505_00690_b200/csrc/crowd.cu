// Crowd dynamics step on B200: one CTA per env, one warp per agent.
//
//   k_guide    field.py:165-212 (waypoint pop, _distance_to_polyline :613,
//              _line_of_sight :601); queues replans for k_astar
//   k_astar    paths.astar_path paths.py:48-87, persistent warps over the queue
//   k_orca     everything below, one CTA per env, one warp per agent
//   pref       field.py:214-227
//   neighbours field.py:246-262  fp32 Gram key fma(y_i,y_j,x_i*x_j), stable top-K
//   half-plane field.py:448-495  (+ robot lane :303-317, static lane :319-348)
//   LP         field.py:500-566  lane-parallel 1-D solve, warp max/min reductions
//   fallback   orca.py:155-242   _solve_least_violation / _lp2_toward / _solve_on_line
//   stall      field.py:135-150; commit + blocked field.py:152-160, 352-366
//   resample   field.py:368-381; last_gap_by_env field.py:268-271
//
// Two-phase: every CTA snapshots its env's pre-step state in shared memory,
// so results are independent of scheduling (field.py:1-9).  Compiled with
// -fmad=false: float64 arithmetic rounds exactly like the numpy reference.
#include <algorithm>
#include <cfloat>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <math_constants.h>
#include "common.cuh"
#include "citywalk_b200.h"
#include "rng.cuh"

namespace cw {

constexpr int MAXC = 12;   // neighbour lanes (<= 10) + robot + static
constexpr double kWaypointReach = 0.5, kStrayLimit = 1.0;

template <int C>
struct ConsT {
  double px[C], py[C], nx[C], ny[C];
};
using WarpCons = ConsT<MAXC>;

// ---------------------------------------------------------------- VO half-plane
// field.py:448-495 for one lane (the selected branch of the vectorised where()).
CW_DEV void vo_halfplane(double rp0, double rp1, double rv0, double rv1, double rr, double horizon,
                         double dt, double vs0, double vs1, double share, double& pt0, double& pt1,
                         double& n0, double& n1) {
  double dsq = rp0 * rp0 + rp1 * rp1;
  double rsq = rr * rr;
  double u0, u1;
  if (dsq <= rsq) {
    double wc0 = rv0 - rp0 / dt, wc1 = rv1 - rp1 / dt;
    double wcl = sqrt(wc0 * wc0 + wc1 * wc1);
    double dist = sqrt(dsq);
    double uc0, uc1;
    if (wcl > kEps) {
      double s = fmax(wcl, kEps);
      uc0 = wc0 / s; uc1 = wc1 / s;
    } else {
      double s = fmax(dist, kEps);
      uc0 = -rp0 / s; uc1 = -rp1 / s;
    }
    if (wcl <= kEps && dist <= kEps) { uc0 = 1.0; uc1 = 0.0; }
    double k = rr / dt - wcl;
    u0 = k * uc0; u1 = k * uc1;
    n0 = uc0; n1 = uc1;
  } else {
    double w0 = rv0 - div_h(rp0, horizon), w1 = rv1 - div_h(rp1, horizon);
    double wlsq = w0 * w0 + w1 * w1;
    double d1 = w0 * rp0 + w1 * rp1;
    if (d1 < 0.0 && d1 * d1 > rsq * wlsq) {
      double wl = sqrt(wlsq);
      double s = fmax(wl, kEps);
      double uw0 = w0 / s, uw1 = w1 / s;
      double k = div_h(rr, horizon) - wl;
      u0 = k * uw0; u1 = k * uw1;
      n0 = uw0; n1 = uw1;
    } else {
      double leg = sqrt(fmax(dsq - rsq, 0.0));
      double det = rp0 * w1 - rp1 * w0;
      double sg = det > 0.0 ? 1.0 : -1.0;
      double sd2 = fmax(dsq, kEps);
      double ld0 = (rp0 * leg - sg * rp1 * rr) / sd2;
      double ld1 = (sg * rp0 * rr + rp1 * leg) / sd2;
      n0 = -sg * ld1; n1 = sg * ld0;
      double d2v = rv0 * ld0 + rv1 * ld1;
      u0 = d2v * ld0 - rv0; u1 = d2v * ld1 - rv1;
    }
  }
  pt0 = vs0 + share * u0;
  pt1 = vs1 + share * u1;
}

// one out-of-line copy for the lane path (three call sites per agent)
struct HalfPlane { double p0, p1, n0, n1; };
__device__ __noinline__ HalfPlane vo_halfplane_ool(double rp0, double rp1, double rv0, double rv1, double rr,
                                                   double horizon, double dt, double vs0, double vs1,
                                                   double share) {
  HalfPlane h;
  vo_halfplane(rp0, rp1, rv0, rv1, rr, horizon, dt, vs0, vs1, share, h.p0, h.p1, h.n0, h.n1);
  return h;
}

// ---------------------------------------------------------------- scalar fallback
// orca.py:155-189, dir_opt=True (only mode the fallback uses)
CW_DEV bool solve_on_line_dir(const double* cpx, const double* cpy, const double* cnx,
                              const double* cny, int i, double ms, double o0, double o1,
                              double& r0, double& r1) {
  double px = cpx[i], py = cpy[i];
  double dx = -cny[i], dy = cnx[i];
  double dpd = dot2_blas(px, py, dx, dy);
  double disc = dpd * dpd + ms * ms - dot2_blas(px, py, px, py);
  if (disc < 0.0) return false;
  double sq = sqrt(disc);
  double tl = -dpd - sq, tr = -dpd + sq;
  for (int j = 0; j < i; ++j) {
    double den = dot2_blas(dx, dy, cnx[j], cny[j]);
    double num = dot2_blas(cpx[j] - px, cpy[j] - py, cnx[j], cny[j]);
    if (fabs(den) < kEps) {
      if (num > kEps) return false;
      continue;
    }
    double t = num / den;
    if (den > 0.0) tl = fmax(tl, t);
    else tr = fmin(tr, t);
    if (tl > tr) return false;
  }
  double tb = dot2_blas(o0, o1, dx, dy) > 0.0 ? tr : tl;
  r0 = px + tb * dx;
  r1 = py + tb * dy;
  return true;
}

template <int CAP>
CW_DEV void least_violation(const ConsT<CAP>& C, int nc, int begin, double ms, double& r0,
                            double& r1) {
  // orca.py:196-212
  double dist = 0.0;
  double qpx[CAP], qpy[CAP], qnx[CAP], qny[CAP];
  for (int i = begin; i < nc; ++i) {
    double pix = C.px[i], piy = C.py[i], nix = C.nx[i], niy = C.ny[i];
    double viol = -dot2_blas(r0 - pix, r1 - piy, nix, niy);
    if (viol <= dist + kEps) continue;
    int np = 0;
    for (int j = 0; j < i; ++j) {
      double pjx = C.px[j], pjy = C.py[j], njx = C.nx[j], njy = C.ny[j];
      double det = nix * njy - niy * njx;
      double dfx = njx - nix, dfy = njy - niy;
      double mx, my;
      if (fabs(det) < kEps) {
        if (dot2_blas(nix, niy, njx, njy) > 0.0) continue;
        mx = 0.5 * (pix + pjx);
        my = 0.5 * (piy + pjy);
      } else {
        double dix = -niy, diy = nix;
        double t = dot2_blas(pjx - pix, pjy - piy, njx, njy) / dot2_blas(dix, diy, njx, njy);
        mx = pix + t * dix;
        my = piy + t * diy;
      }
      double nrm = glibc_hypot(dfx, dfy);
      if (nrm < kEps) continue;
      qpx[np] = mx; qpy[np] = my; qnx[np] = dfx / nrm; qny[np] = dfy / nrm;
      ++np;
    }
    // _lp2_toward(proj, ms, n_i)
    double s = ms / fmax(glibc_hypot(nix, niy), kEps);
    double t0 = nix * s, t1 = niy * s;
    bool ok = true;
    for (int k = 0; k < np && ok; ++k) {
      if (dot2_blas(t0 - qpx[k], t1 - qpy[k], qnx[k], qny[k]) < -kEps)
        ok = solve_on_line_dir(qpx, qpy, qnx, qny, k, ms, nix, niy, t0, t1);
    }
    if (ok) { r0 = t0; r1 = t1; }
    dist = -dot2_blas(r0 - pix, r1 - piy, nix, niy);
  }
}

// out-of-line copy for the lane path (rare; keeps the round kernel's hot code small)
template <int CAP>
__device__ __noinline__ void least_violation_ool(const ConsT<CAP>& C, int nc, int begin, double ms, double& r0,
                                                 double& r1) {
  least_violation(C, nc, begin, ms, r0, r1);
}

// ---------------------------------------------------------------- warp fallback
// orca.py:155-242 (_solve_least_violation / _lp2_toward / _solve_on_line, dir_opt)
// with the whole warp for the warp path (C and Q in shared memory, warp-uniform
// control flow); the lane path keeps the scalar copy above (measured: deferring its
// rare fallbacks to the whole warp costs more in the common case than it saves).  The projected constraints of row i (orca.py:196-207) are built
// one per lane j < i and compacted in j order by a ballot; each line solve
// (orca.py:155-189) reduces over j < k in parallel: it fails iff some j is
// degenerate with num > eps or the running bounds cross -- the bounds only
// tighten, so they cross at some prefix iff the full max(tl) > min(tr) -- and
// otherwise ends at the full max / min.  Same float operations, exact reductions.
CW_DEV bool warp_solve_on_line_dir(const WarpCons& Q, int k, double ms, double o0, double o1, double& r0,
                                   double& r1, int lane) {
  const double px = Q.px[k], py = Q.py[k];
  const double dx = -Q.ny[k], dy = Q.nx[k];
  const double dpd = dot2_blas(px, py, dx, dy);
  const double disc = dpd * dpd + ms * ms - dot2_blas(px, py, px, py);
  if (disc < 0.0) return false;
  const double sq = sqrt(disc);
  double tl = -dpd - sq, tr = -dpd + sq;
  double tlj = -DBL_MAX, trj = DBL_MAX;
  bool bad = false;
  if (lane < k) {
    const double den = dot2_blas(dx, dy, Q.nx[lane], Q.ny[lane]);
    const double num = dot2_blas(Q.px[lane] - px, Q.py[lane] - py, Q.nx[lane], Q.ny[lane]);
    if (fabs(den) < kEps) {
      bad = num > kEps;
    } else {
      const double t = num / den;
      if (den > 0.0) tlj = t;
      else trj = t;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    tlj = fmax(tlj, __shfl_xor_sync(0xffffffffu, tlj, o));
    trj = fmin(trj, __shfl_xor_sync(0xffffffffu, trj, o));
  }
  tl = fmax(tl, tlj);
  tr = fmin(tr, trj);
  if (__any_sync(0xffffffffu, bad) || tl > tr) return false;
  const double tb = dot2_blas(o0, o1, dx, dy) > 0.0 ? tr : tl;
  r0 = px + tb * dx;
  r1 = py + tb * dy;
  return true;
}

CW_DEV void warp_least_violation(const WarpCons& C, WarpCons& Q, int nc, int begin, double ms, double& r0,
                                 double& r1, int lane) {
  double dist = 0.0;
  for (int i = begin; i < nc; ++i) {
    const double pix = C.px[i], piy = C.py[i], nix = C.nx[i], niy = C.ny[i];
    const double viol = -dot2_blas(r0 - pix, r1 - piy, nix, niy);
    if (viol <= dist + kEps) continue;
    bool valid = false;
    double mx = 0.0, my = 0.0, qx = 0.0, qy = 0.0;
    if (lane < i) {
      const double pjx = C.px[lane], pjy = C.py[lane], njx = C.nx[lane], njy = C.ny[lane];
      const double det = nix * njy - niy * njx;
      const double dfx = njx - nix, dfy = njy - niy;
      bool keep = true;
      if (fabs(det) < kEps) {
        if (dot2_blas(nix, niy, njx, njy) > 0.0) keep = false;
        mx = 0.5 * (pix + pjx);
        my = 0.5 * (piy + pjy);
      } else {
        const double dix = -niy, diy = nix;
        const double t = dot2_blas(pjx - pix, pjy - piy, njx, njy) / dot2_blas(dix, diy, njx, njy);
        mx = pix + t * dix;
        my = piy + t * diy;
      }
      if (keep) {
        const double nrm = glibc_hypot(dfx, dfy);
        if (!(nrm < kEps)) {
          valid = true;
          qx = dfx / nrm;
          qy = dfy / nrm;
        }
      }
    }
    const unsigned vm = __ballot_sync(0xffffffffu, valid);
    const int np = __popc(vm);
    __syncwarp();
    if (valid) {
      const int k = __popc(vm & ((1u << lane) - 1u));
      Q.px[k] = mx; Q.py[k] = my; Q.nx[k] = qx; Q.ny[k] = qy;
    }
    __syncwarp();
    // _lp2_toward(proj, ms, n_i)
    const double sc = ms / fmax(glibc_hypot(nix, niy), kEps);
    double t0 = nix * sc, t1 = niy * sc;
    bool ok = true;
    for (int k = 0; k < np && ok; ++k) {
      if (dot2_blas(t0 - Q.px[k], t1 - Q.py[k], Q.nx[k], Q.ny[k]) < -kEps)
        ok = warp_solve_on_line_dir(Q, k, ms, nix, niy, t0, t1, lane);
    }
    if (ok) { r0 = t0; r1 = t1; }
    dist = -dot2_blas(r0 - pix, r1 - piy, nix, niy);
  }
  __syncwarp();
}

// ---------------------------------------------------------------- warp LP
// field.py:500-566 for one agent.  Lane k holds constraint k; all lanes keep
// the running result.  Returns true when the fallback ran.
CW_DEV bool warp_lp(const WarpCons& C, WarpCons& Q, int nc, double pf0, double pf1, double ms, double& r0,
                    double& r1, int lane) {
  double pn = sqrt(pf0 * pf0 + pf1 * pf1);
  double sc = pn > ms ? ms / fmax(pn, kEps) : 1.0;
  r0 = pf0 * sc;
  r1 = pf1 * sc;
  const bool mine = lane < nc;
  const double mpx = mine ? C.px[lane] : 0.0, mpy = mine ? C.py[lane] : 0.0;
  const double mnx = mine ? C.nx[lane] : 1.0, mny = mine ? C.ny[lane] : 0.0;
  for (int i = 0; i < nc; ++i) {
    const double pi0 = C.px[i], pi1 = C.py[i], ni0 = C.nx[i], ni1 = C.ny[i];
    if (!((r0 - pi0) * ni0 + (r1 - pi1) * ni1 < -kEps)) continue;
    const double d0 = -ni1, d1 = ni0;
    const double dpd = pi0 * d0 + pi1 * d1;
    const double disc = dpd * dpd + ms * ms - (pi0 * pi0 + pi1 * pi1);
    bool bad = disc < 0.0;
    const double sq = sqrt(fmax(disc, 0.0));
    double tl = -dpd - sq, tr = -dpd + sq;
    double tlj = -DBL_MAX, trj = DBL_MAX;
    bool badj = false;
    if (lane < i) {
      double den = d0 * mnx + d1 * mny;
      double num = (mpx - pi0) * mnx + (mpy - pi1) * mny;
      if (fabs(den) < kEps) {
        badj = num > kEps;
      } else {
        double t = num / den;
        if (den > 0.0) tlj = t;
        else trj = t;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      tlj = fmax(tlj, __shfl_xor_sync(0xffffffffu, tlj, o));
      trj = fmin(trj, __shfl_xor_sync(0xffffffffu, trj, o));
    }
    bad |= __any_sync(0xffffffffu, badj);
    tl = fmax(tl, tlj);
    tr = fmin(tr, trj);
    bad |= tl > tr;
    if (bad) {
      warp_least_violation(C, Q, nc, i, ms, r0, r1, lane);
      return true;
    }
    double tb = (pf0 - pi0) * d0 + (pf1 - pi1) * d1;
    tb = fmin(fmax(tb, tl), tr);
    r0 = pi0 + tb * d0;
    r1 = pi1 + tb * d1;
  }
  return false;
}

// ---------------------------------------------------------------- lane LP
// warp_lp for one agent held by one lane (constraints in registers, lane
// order).  Identical arithmetic: the lane-parallel max / min over j < i of
// warp_lp is an exact reduction, taken here in j order.
constexpr int MAXK = MAXC - 2;   // neighbour lanes

// slot read with a run-time index (thread-local array, see put_slot)
template <int CAP>
CW_DEV double get_slot(const double (&a)[CAP], int k) {
  return a[k];
}

template <int CAP>
CW_DEV bool lane_lp(const double (&cpx)[CAP], const double (&cpy)[CAP], const double (&cnx)[CAP],
                    const double (&cny)[CAP], int nc, double pf0, double pf1, double ms, double& r0,
                    double& r1) {
  double pn = sqrt(pf0 * pf0 + pf1 * pf1);
  double sc = pn > ms ? ms / fmax(pn, kEps) : 1.0;
  r0 = pf0 * sc;
  r1 = pf1 * sc;
  // the constraint loop stays rolled (one copy of the body: instruction-cache
  // footprint); the inner j loop is unrolled over the register arrays
#pragma unroll 1
  for (int i = 0; i < nc; ++i) {
    const double pi0 = get_slot(cpx, i), pi1 = get_slot(cpy, i);
    const double ni0 = get_slot(cnx, i), ni1 = get_slot(cny, i);
    if (!((r0 - pi0) * ni0 + (r1 - pi1) * ni1 < -kEps)) continue;
    const double d0 = -ni1, d1 = ni0;
    const double dpd = pi0 * d0 + pi1 * d1;
    const double disc = dpd * dpd + ms * ms - (pi0 * pi0 + pi1 * pi1);
    bool bad = disc < 0.0;
    const double sq = sqrt(fmax(disc, 0.0));
    double tl = -dpd - sq, tr = -dpd + sq;
    double tlj = -DBL_MAX, trj = DBL_MAX;
#pragma unroll 1
    for (int j = 0; j < i; ++j) {
      const double den = d0 * cnx[j] + d1 * cny[j];
      const double num = (cpx[j] - pi0) * cnx[j] + (cpy[j] - pi1) * cny[j];
      if (fabs(den) < kEps) {
        bad |= num > kEps;
      } else {
        const double t = num / den;
        if (den > 0.0) tlj = fmax(tlj, t);
        else trj = fmin(trj, t);
      }
    }
    tl = fmax(tl, tlj);
    tr = fmin(tr, trj);
    bad |= tl > tr;
    if (bad) {
      ConsT<CAP> C;
#pragma unroll
      for (int k = 0; k < CAP; ++k) { C.px[k] = cpx[k]; C.py[k] = cpy[k]; C.nx[k] = cnx[k]; C.ny[k] = cny[k]; }
      least_violation_ool(C, nc, i, ms, r0, r1);
      return true;
    }
    double tb = (pf0 - pi0) * d0 + (pf1 - pi1) * d1;
    tb = fmin(fmax(tb, tl), tr);
    r0 = pi0 + tb * d0;
    r1 = pi1 + tb * d1;
  }
  return false;
}

// slot write / read with a run-time index: the arrays live in thread-local memory
// (measured faster than a select chain over register arrays: run 0.342 -> 0.308 ms/tick)
template <int CAP>
CW_DEV void put_slot(double (&a)[CAP], int k, double v) {
  a[k] = v;
}

// ---------------------------------------------------------------- A*
CW_DEV double octile(int r, int c, int gr, int gc) {
  int dr = abs(r - gr), dc = abs(c - gc);
  return kSqrt2 * (double)min(dr, dc) + (double)abs(dr - dc);
}

struct AstarReq { int32_t env, agent, start, goal; };
struct __align__(16) OpenEnt { unsigned long long f, k; };

// ---- next-tick search prefetch (cw_spec_create; see launch_step)
// An A* result is a pure function of (env grid, start cell, goal cell).  While a tick's
// longest searches run, the envs that have already committed (no replan this tick)
// predict their next tick's replans with a read-only copy of the guidance pass and
// search them ahead on a side stream into a per-agent cache entry.  The next tick's
// k_astar looks each request up: an entry with the same (start, goal) and the env's
// current grid generation is the search's result (copied), one still running is
// waited for, one still queued is claimed and searched in place; anything else is
// searched as usual.  Nothing the tick computes depends on whether an entry was used.
enum : int { kSpEmpty = 0, kSpWriting, kSpQueued, kSpRunning, kSpDone, kSpClaimed, kSpFailed };
struct __align__(16) SpecEnt {
  unsigned long long word;   // batch tag << 8 | state (CAS-owned transitions)
  int32_t start, goal;       // the predicted request
  int32_t epoch;             // grid generation read before the search read the grid
  int32_t count, found, over;   // result: cells in cells[path_cap - count, path_cap)
};
struct SpecArgs {
  int mode;                  // 0: plain, 1: tick search with cache lookup, 2: speculative batch
  SpecEnt* ent;              // (E * A)
  int32_t* cells;            // (E * A, path_cap)
  const int32_t* epoch;      // (E) grid generation of each env (bumped by every grid write)
  AstarReq* q;               // mode 2 (and the dry guide): the batch's requests
  int* qn;                   // [0] count, [1] next
  unsigned char* rec;        // mode 2: search scratch per (SM, warp) -- at most one search
  OpenEnt* heap;             //   CTA is resident per SM (shared memory), so %smid indexes it
  size_t rec_stride;
  unsigned long long tag;    // mode 2 / dry guide: this batch's tag
  unsigned long long* stats; // [1] hits, [2] waits on a running prediction, [3] claims
  int* qr;                   // (E * A) per queue item: the tag once the item is written
  int* pend;                 // mode 1 with early commit: (E) the tick's searches still running per env
};
// qn layout: [0] items queued, [1] items taken, [2] envs committing after their searches
// (their dry guidance pass adds items later), [3] of those done; a batch's search warps
// keep polling until [3] == [2] and the queue is drained (or kSpecIdle cycles pass).
constexpr long long kSpecIdle = 1ll << 23;

CW_DEV unsigned sm_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

}  // namespace cw
#include "runq.cuh"
#include "astar.cuh"
namespace cw {

// ---------------------------------------------------------------- guidance pass
CW_DEV void path_point(const int32_t* cells, int head, int n, int k, double gx, double gy,
                       double res, int nx, double& x, double& y) {
  if (k == n - 1) { x = gx; y = gy; return; }
  int f = cells[head + k];
  int r = f / nx, c = f - r * nx;
  x = ((double)c + 0.5) * res;
  y = ((double)r + 0.5) * res;
}

// Queue one predicted request (lane 0 of the guiding warp).  An entry still queued or
// running belongs to an earlier batch and is left alone; an entry already holding this
// (start, goal) for the current grid is kept as it is.
CW_DEV void spec_request(const SpecArgs& sp, const AstarReq& R, size_t ia) {
  SpecEnt* en = sp.ent + ia;
  const unsigned long long w = *(volatile unsigned long long*)&en->word;
  const int st = (int)(w & 0xFFull);
  if (st == kSpWriting || st == kSpQueued || st == kSpRunning) return;
  if (st == kSpDone && *(volatile int*)&en->start == R.start && *(volatile int*)&en->goal == R.goal &&
      *(volatile int*)&en->epoch == *(volatile const int*)&sp.epoch[R.env])
    return;
  if (atomicCAS(&en->word, w, (sp.tag << 8) | kSpWriting) != w) return;
  en->start = R.start;
  en->goal = R.goal;
  const int q = atomicAdd(&sp.qn[0], 1);
  sp.q[q] = R;
  __threadfence();
  atomicExch(&sp.qr[q], (int)sp.tag);
  atomicExch(&en->word, (sp.tag << 8) | kSpQueued);
}

// k_guide: field.py:165-212 minus the A* itself (queued for k_astar).
// Body shared by k_guide (requests appended to astar_req) and k_round (requests
// pushed to the run ring).  Returns the env's request count (CTA-uniform).
// kDry (next-tick search prefetch): the same decisions on the committed state, no
// state writes; each replan it would queue becomes a speculative cache request.  The
// state it reads may be rewritten concurrently by the host (a prediction only), so
// every index it derives is clamped.
template <int NT, bool kRing, bool kDry = false>
__device__ int guide_env(const cw_crowd_params& P, const cw_crowd_state& S, int e,
                         const uint8_t* __restrict__ env_mask, const RunArgs* ra,
                         const SpecArgs* sp = nullptr, bool force = false) {
  const int lane = threadIdx.x & 31;
  const int A = P.A;
  const size_t eA = (size_t)e * A;
  __shared__ int s_req;   // replans this env queued
  if (kDry && !force && S.env_req[e]) return 0;   // still searching this tick: predicted by its commit
  if (!kDry && env_mask && !env_mask[e]) {
    if (threadIdx.x == 0) S.env_req[e] = 0;
    return 0;
  }
  if (threadIdx.x == 0) s_req = 0;
  __syncthreads();
  int my_req = 0;
  const bool has_obs = S.has_obs[e] != 0;
  const int nx = P.nx, ny = P.ny;
  const size_t N = (size_t)nx * ny;
  const uint8_t* lab = S.labels + e * N;
  const double res = P.res;
  long long scanned = 0;   // remaining path points the reference's stray check scans
  long long pts_read = 0;  // path points this kernel reads (scans stop at the first hit)
  long long los_read = 0;  // line-of-sight samples (label bytes) read
  AstarReq* reqs = reinterpret_cast<AstarReq*>(S.astar_req);
  // Every decision below is a boolean (near the path: min distance <= 1 m,
  // field.py:190; line of sight clear), so scans stop at the first hit.
  // Phase A, one lane per agent: waypoint pop + the first kLaneSegs segments.
  // Phase B, the whole warp per deferred agent: the rest of the polyline and
  // the line-of-sight samples, 32 at a time (the original warp-parallel scans).
  constexpr int kLaneSegs = 8;
  const int A_pad = (A + 31) & ~31;   // whole warps iterate together (ballots below)
  for (int a0 = threadIdx.x - lane; a0 < A_pad; a0 += NT) {
    const int a = a0 + lane;
    const size_t ia = eA + a;
    int need = 0;            // 1: continue the polyline scan at segment kLaneSegs + 1; 2: line of sight
    int head = 0, n = 0;
    double px = 0.0, py = 0.0, gx = 0.0, gy = 0.0;
    if (a < A && S.active[ia]) {
      gx = S.goal[ia * 2];
      gy = S.goal[ia * 2 + 1];
      if (!has_obs) {
        if (!kDry) {
          S.waypoint[ia * 2] = gx;
          S.waypoint[ia * 2 + 1] = gy;
        }
      } else {
        px = S.pos[ia * 2];
        py = S.pos[ia * 2 + 1];
        const int32_t* cells = S.path_cells + ia * P.path_cap;
        head = S.path_head[ia];
        n = S.path_n[ia];
        if (kDry) {
          head = min(max(head, 0), P.path_cap);
          n = min(max(n, 0), P.path_cap - head + 1);
        }
        need = 2;
        if (n > 0) {
          double qx, qy;
          path_point(cells, head, n, 0, gx, gy, res, nx, qx, qy);
          if (glibc_hypot(qx - px, qy - py) < kWaypointReach && n > 1) { ++head; --n; }
          path_point(cells, head, n, 0, gx, gy, res, nx, qx, qy);
          bool near = glibc_hypot(qx - px, qy - py) <= kStrayLimit;
          double bx = qx, by = qy;
          const int kend = min(n, kLaneSegs + 1);
          ++pts_read;
          for (int k = 1; k < kend && !near; ++k) {
            ++pts_read;
            const double ax = bx, ay = by;
            path_point(cells, head, n, k, gx, gy, res, nx, bx, by);
            double abx = bx - ax, aby = by - ay;
            double den = dot2_blas(abx, aby, abx, aby);
            double t = 0.0;
            if (!(den < kEps)) t = fmin(fmax(dot2_blas(px - ax, py - ay, abx, aby) / den, 0.0), 1.0);
            near = glibc_hypot(ax + t * abx - px, ay + t * aby - py) <= kStrayLimit;
          }
          scanned += n;   // the reference scans every remaining point (traffic model)
          if (near) {
            if (!kDry) {
              S.path_head[ia] = head;
              S.path_n[ia] = n;
              S.waypoint[ia * 2] = qx;
              S.waypoint[ia * 2 + 1] = qy;
            }
            need = 0;
          } else if (n > kLaneSegs + 1) {
            need = 1;
          }
        }
      }
    }
    unsigned todo = __ballot_sync(0xffffffffu, need != 0);
    while (todo) {
      const int s = __ffs(todo) - 1;
      todo &= todo - 1;
      const int sa = a0 + s;
      const size_t sia = eA + sa;
      const int sneed = __shfl_sync(0xffffffffu, need, s);
      const int shead = __shfl_sync(0xffffffffu, head, s), sn = __shfl_sync(0xffffffffu, n, s);
      const double spx = __shfl_sync(0xffffffffu, px, s), spy = __shfl_sync(0xffffffffu, py, s);
      const double sgx = __shfl_sync(0xffffffffu, gx, s), sgy = __shfl_sync(0xffffffffu, gy, s);
      if (sneed == 1) {   // segments kLaneSegs + 1 .. n - 1, 32 per step
        const int32_t* cells = S.path_cells + sia * P.path_cap;
        bool near = false;
        for (int k0 = kLaneSegs + 1; k0 < sn && !near; k0 += 32) {
          const int k = k0 + lane;
          bool mine = false;
          if (k < sn) {
            ++pts_read;
            double ax, ay, bx, by;
            path_point(cells, shead, sn, k - 1, sgx, sgy, res, nx, ax, ay);
            path_point(cells, shead, sn, k, sgx, sgy, res, nx, bx, by);
            double abx = bx - ax, aby = by - ay;
            double den = dot2_blas(abx, aby, abx, aby);
            double t = 0.0;
            if (!(den < kEps)) t = fmin(fmax(dot2_blas(spx - ax, spy - ay, abx, aby) / den, 0.0), 1.0);
            mine = glibc_hypot(ax + t * abx - spx, ay + t * aby - spy) <= kStrayLimit;
          }
          near = __any_sync(0xffffffffu, mine);
        }
        if (near) {
          if (!kDry && lane == 0) {
            double wx, wy;
            path_point(cells, shead, sn, 0, sgx, sgy, res, nx, wx, wy);
            S.path_head[sia] = shead;
            S.path_n[sia] = sn;
            S.waypoint[sia * 2] = wx;
            S.waypoint[sia * 2 + 1] = wy;
          }
          continue;
        }
      }
      // _line_of_sight (field.py:601-610), 32 samples per step
      double d = glibc_hypot(sgx - spx, sgy - spy);
      long long ns = max(2LL, trunc_ll(div_h(2.0 * d, res)) + 2);
      if (kDry) ns = min(ns, 4LL * (nx + ny) + 2);   // torn reads must not run away
      double step = 1.0 / (double)(ns - 1);
      bool clear = true;
      for (long long k0 = 0; k0 < ns && clear; k0 += 32) {
        const long long k = k0 + lane;
        bool blocked = false;
        if (k < ns) {
          ++los_read;
          double t = k == ns - 1 ? 1.0 : (double)k * step + 0.0;
          double xs = spx + (sgx - spx) * t, ys = spy + (sgy - spy) * t;
          long long rr = clampll(trunc_ll(div_h(ys, res)), 0, ny - 1);
          long long cc = clampll(trunc_ll(div_h(xs, res)), 0, nx - 1);
          blocked = lab[rr * nx + cc] == L_OBSTACLE;
        }
        clear = !__any_sync(0xffffffffu, blocked);
      }
      if (lane == 0) {
        if (clear) {
          if (!kDry) {
            S.path_head[sia] = 0;
            S.path_n[sia] = 1;
            S.waypoint[sia * 2] = sgx;
            S.waypoint[sia * 2 + 1] = sgy;
          }
        } else {
          int sr = (int)fmin(fmax(div_h(spy, res), 0.0), (double)(ny - 1));
          int sc = (int)fmin(fmax(div_h(spx, res), 0.0), (double)(nx - 1));
          int gr = (int)fmin(fmax(div_h(sgy, res), 0.0), (double)(ny - 1));
          int gc = (int)fmin(fmax(div_h(sgx, res), 0.0), (double)(nx - 1));
          AstarReq R = {e, sa, sr * nx + sc, gr * nx + gc};
          if (kDry) {
            spec_request(*sp, R, sia);
          } else if (kRing) {
            ring_push(*ra, R);
          } else {
            int q = atomicAdd(&S.flags[4], 1);
            reqs[q] = R;
          }
          ++my_req;
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    scanned += __shfl_xor_sync(0xffffffffu, scanned, o);
    pts_read += __shfl_xor_sync(0xffffffffu, pts_read, o);
    los_read += __shfl_xor_sync(0xffffffffu, los_read, o);
    my_req += __shfl_xor_sync(0xffffffffu, my_req, o);
  }
  if (kDry) return 0;
  if (lane == 0 && scanned && S.counters)
    atomicAdd((unsigned long long*)&S.counters[1], (unsigned long long)scanned);
  if (lane == 0 && pts_read && S.counters)
    atomicAdd((unsigned long long*)&S.counters[12], (unsigned long long)pts_read);
  if (lane == 0 && los_read && S.counters)
    atomicAdd((unsigned long long*)&S.counters[13], (unsigned long long)los_read);
  if (lane == 0 && my_req) atomicAdd(&s_req, my_req);
  __syncthreads();
  const int n_req = s_req;
  if (threadIdx.x == 0) S.env_req[e] = (uint8_t)(n_req > 0);
  return n_req;
}

// The dry guidance pass over the envs that committed without a replan this tick.
template <int NT>
__global__ void __launch_bounds__(NT) k_guide_dry(cw_crowd_params P, cw_crowd_state S, SpecArgs sp,
                                                  const int32_t* rows = nullptr) {
  if (rows) guide_env<NT, false, true>(P, S, rows[blockIdx.x], nullptr, nullptr, &sp, true);
  else guide_env<NT, false, true>(P, S, blockIdx.x, nullptr, nullptr, &sp);
}

// Install the predictions of context `src` for rows (all agents) into context `dst`:
// an entry of src that is done for the row's current src generation is copied with
// dst's generation of the row (the caller has just installed the same grid there);
// a dst entry a prediction is still running into is left alone (the tick searches it).
__global__ void k_spec_install(int A, int path_cap, SpecEnt* __restrict__ dent, int32_t* __restrict__ dcells,
                               const SpecEnt* __restrict__ sent, const int32_t* __restrict__ scells,
                               const int32_t* __restrict__ depoch, const int32_t* __restrict__ sepoch,
                               const int32_t* __restrict__ rows, unsigned long long tag) {
  const int e = rows[blockIdx.x];
  const int lane = threadIdx.x & 31;
  for (int a = threadIdx.x >> 5; a < A; a += blockDim.x >> 5) {
    const size_t ia = (size_t)e * A + a;
    const SpecEnt* se = sent + ia;
    SpecEnt* de = dent + ia;
    int ok = 0, cnt = 0;
    if (lane == 0) {
      const unsigned long long sw = *(volatile const unsigned long long*)&se->word;
      ok = (int)(sw & 0xFFull) == kSpDone && *(volatile const int*)&se->epoch == sepoch[e];
      if (ok) {
        const unsigned long long dw = *(volatile unsigned long long*)&de->word;
        const int ds = (int)(dw & 0xFFull);
        ok = ds != kSpRunning && ds != kSpWriting && atomicCAS(&de->word, dw, (tag << 8) | kSpWriting) == dw;
      }
      if (ok) cnt = se->found == 1 && !se->over ? se->count : 0;
    }
    ok = __shfl_sync(0xffffffffu, ok, 0);
    cnt = __shfl_sync(0xffffffffu, cnt, 0);
    if (!ok) continue;
    for (int k = path_cap - cnt + lane; k < path_cap; k += 32) dcells[ia * path_cap + k] = scells[ia * path_cap + k];
    __syncwarp();
    if (lane == 0) {
      de->start = se->start;
      de->goal = se->goal;
      de->count = se->count;
      de->found = se->found;
      de->over = se->over;
      de->epoch = depoch[e];
      __threadfence();
      atomicExch(&de->word, (tag << 8) | kSpDone);
    }
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) k_guide(cw_crowd_params P, cw_crowd_state S,
                                              const uint8_t* __restrict__ env_mask, int* pend = nullptr,
                                              int* n_late = nullptr) {
  const int n = guide_env<NT, false>(P, S, blockIdx.x, env_mask, nullptr);
  if (pend && threadIdx.x == 0) {   // early commit: the env's searches, and one more late committer
    pend[blockIdx.x] = n;
    if (n) atomicAdd(n_late, 1);
  }
}

// ---------------------------------------------------------------- ORCA + commit
// Agent binning for the neighbour search (used when A is large).
struct Bins {
  int ncx, ncy;     // 0 = no binning
  double inv_cs;
};

CW_HD Bins make_bins(const cw_crowd_params& P) {
  Bins b = {0, 0, 0.0};
  if (P.A < 128) return b;
  const double cs = P.neighbor_distance + 0.5;
  b.ncx = (int)ceil(P.nx * P.res / cs);
  b.ncy = (int)ceil(P.ny * P.res / cs);
  b.inv_cs = 1.0 / cs;
  return b;
}

CW_HD size_t bins_smem_bytes(const Bins& b, int A) {
  return b.ncx > 0 ? (size_t)(b.ncx * b.ncy + 1 + 2 * A) * 4 : 0;
}

// ORCA + commit + goal resample of env e (body of k_orca and k_round).  With
// ra != nullptr the env's gap goes to the run history at ``tick`` instead of
// gap_tmp / flags[0].
template <int NT, int kLanes>   // 0 warp per agent, 1 lane per agent, 2 lanes + cell binning
__device__ void orca_env(const cw_crowd_params& P, const cw_crowd_state& S, int e,
                         const double* __restrict__ robot_pos, const double* __restrict__ robot_vel,
                         double robot_radius, const uint8_t* __restrict__ env_mask, const Bins& bins,
                         unsigned char* sm, const RunArgs* ra, int tick) {
  constexpr int NW = NT / 32;
  const int A = P.A;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* s_px = reinterpret_cast<double*>(sm);
  double* s_py = s_px + A;
  double* s_vx = s_py + A;
  double* s_vy = s_vx + A;
  double* s_r = s_vy + A;
  double* s_nx = s_r + A;   // post-commit positions (resample)
  double* s_ny = s_nx + A;
  WarpCons* s_cons = reinterpret_cast<WarpCons*>(s_ny + A);
  uint8_t* s_act = reinterpret_cast<uint8_t*>(s_cons + (kLanes ? 0 : 2 * NW));   // warp path: C, then Q (fallback); lanes: none
  // agent binning (large A): cell ends after the scatter, sorted agent ids, agent cell
  int* s_cend = reinterpret_cast<int*>(s_act + ((A + 15) & ~15));
  int* s_sorted = s_cend + bins.ncx * bins.ncy + 1;
  int* s_cell = s_sorted + A;
  __shared__ double s_gap[NW];
  __shared__ int s_anynb[NW];
  {
  const long long t_cta0 = clock64();
    const size_t eA = (size_t)e * A;
    const bool emask = env_mask ? env_mask[e] != 0 : true;
    for (int a = threadIdx.x; a < A; a += NT) {
      s_px[a] = S.pos[(eA + a) * 2];
      s_py[a] = S.pos[(eA + a) * 2 + 1];
      s_vx[a] = S.vel[(eA + a) * 2];
      s_vy[a] = S.vel[(eA + a) * 2 + 1];
      s_r[a] = S.radius[eA + a];
      s_nx[a] = s_px[a];
      s_ny[a] = s_py[a];
      s_act[a] = (S.active[eA + a] && emask) ? 1 : 0;
    }
    __syncthreads();
    if (bins.ncx > 0) {
      // counting sort of the active agents into square cells of side >= nd + 0.5 m:
      // every j with fp32 key(i, j) < nd^2 (key error < 0.03 m^2 on <= 128 m grids)
      // lies in the 3 x 3 cells around i; selection below still uses (key, index)
      const int nc = bins.ncx * bins.ncy;
      for (int c = threadIdx.x; c <= nc; c += NT) s_cend[c] = 0;
      __syncthreads();
      for (int a = threadIdx.x; a < A; a += NT) {
        int cell = -1;
        if (s_act[a]) {
          const int cx = min(max((int)(s_px[a] * bins.inv_cs), 0), bins.ncx - 1);
          const int cy = min(max((int)(s_py[a] * bins.inv_cs), 0), bins.ncy - 1);
          cell = cy * bins.ncx + cx;
          atomicAdd(&s_cend[cell + 1], 1);
        }
        s_cell[a] = cell;
      }
      __syncthreads();
      if (threadIdx.x < 32) {   // exclusive scan of the counts (one warp)
        int carry = 0;
        for (int c0 = 0; c0 <= nc; c0 += 32) {
          const int c = c0 + lane;
          int v = c <= nc ? s_cend[c] : 0;
  #pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
          }
          if (c <= nc) s_cend[c] = v + carry;
          carry += __shfl_sync(0xffffffffu, v, 31);
        }
      }
      __syncthreads();
      for (int a = threadIdx.x; a < A; a += NT)   // afterwards s_cend[c] = end of cell c
        if (s_cell[a] >= 0) s_sorted[atomicAdd(&s_cend[s_cell[a]], 1)] = a;
      __syncthreads();
    }
    const int nx = P.nx, ny = P.ny;
    const size_t N = (size_t)nx * ny;
    const uint8_t* lab = S.labels + e * N;
    const bool has_obs = S.has_obs[e] != 0;
    const double res = P.res;
    const bool use_robot = robot_pos != nullptr;
    double rpx = 0, rpy = 0, rvx = 0, rvy = 0;
    if (use_robot) {
      rpx = robot_pos[e * 2]; rpy = robot_pos[e * 2 + 1];
      if (robot_vel) { rvx = robot_vel[e * 2]; rvy = robot_vel[e * 2 + 1]; }
    }
    WarpCons& C = s_cons[wid];
    WarpCons& Q = s_cons[NW + wid];   // warp path only (lane path: no WarpCons)
    double my_gap = CUDART_INF;
    int my_anynb = 0;
    long long fallbacks = 0, stalls = 0;
    // kLanes: the caller guarantees max_neighbors <= MAXK, so each instantiation holds
    // one of the two paths (code size, registers)
    constexpr bool lanes = kLanes != 0;
    if (lanes) {
      // ---------------- lane per agent: same operations as the warp path
      const int kmax = min(P.max_neighbors, max(A - 1, 0));
      // the fp32 Gram operands of every agent, once (field.py:246-253: p32, |p32|^2); without
      // binning they alias the unused bins region, with it they follow the agent cells
      float* s_fx = reinterpret_cast<float*>(kLanes == 2 ? s_cell + A : s_cend);
      float* s_fy = s_fx + A;
      float* s_fsq = s_fy + A;
      for (int a = threadIdx.x; a < A; a += NT) {
        const float xj = (float)s_px[a], yj = (float)s_py[a];
        s_fx[a] = xj;
        s_fy[a] = yj;
        s_fsq[a] = __fadd_rn(__fmul_rn(xj, xj), __fmul_rn(yj, yj));
      }
      __syncthreads();
      // A <= NT: thread (wid, lane) takes agent lane * NW + wid, so the CTA's warps
      // share the env's agents instead of warp 0 taking all of them
      const bool spread = A <= NT;
      for (int t = threadIdx.x; t < (spread ? NT : A); t += NT) {
        const int a = spread ? lane * NW + wid : t;
        if (a >= A || !s_act[a]) continue;
        const double px = s_px[a], py = s_py[a];
        const size_t ia = eA + a;
        // the static lane's nearest-obstacle cell, loaded first (a dependent random read
        // that the neighbour selection below hides)
        int flat_pre = -1;
        if (P.use_static && has_obs) {
          const long long ri = clampll(trunc_ll(div_h(py, res)), 0, ny - 1);
          const long long ci = clampll(trunc_ll(div_h(px, res)), 0, nx - 1);
          flat_pre = S.nearest[e * N + ri * nx + ci];
        }
        const double gx = S.goal[ia * 2], gy = S.goal[ia * 2 + 1];
        const double wx = S.waypoint[ia * 2], wy = S.waypoint[ia * 2 + 1];
        const double sp = S.pref_speed[ia];
        double tw0 = wx - px, tw1 = wy - py;
        double dist = sqrt(tw0 * tw0 + tw1 * tw1);
        double safe = fmax(dist, kEps);
        double pf0 = tw0 / safe * sp, pf1 = tw1 / safe * sp;
        double tg0 = gx - px, tg1 = gy - py;
        double dg = sqrt(tg0 * tg0 + tg1 * tg1);
        double scl = fmin(1.0, dg / fmax(sp * P.dt * 4, kEps));
        pf0 = pf0 * scl;
        pf1 = pf1 * scl;
        // stable top-K by (fp32 key, index): the scan visits j in increasing order,
        // so a new entry goes after every kept entry with key <= its key
        const float xi = (float)px, yi = (float)py;
        const float sqi = __fadd_rn(__fmul_rn(xi, xi), __fmul_rn(yi, yi));
        const double vxa = s_vx[a], vya = s_vy[a], ra = s_r[a];
        float tk[MAXK];
        int tj[MAXK];
#pragma unroll
        for (int k = 0; k < MAXK; ++k) { tk[k] = CUDART_INF_F; tj[k] = 0; }
        int nb = 0;
        // per 32-candidate chunk: the range test for every j without divergence
        // (a bitmask), then each lane inserts only its own in-range j.  The insertion
        // orders by (key, index), so the visiting order does not matter (binned
        // candidates come in cell order)
        auto insert = [&](float key, int j) {
          int pos = 0;
#pragma unroll
          for (int k = 0; k < MAXK; ++k) pos += (k < nb && (tk[k] < key || (tk[k] == key && tj[k] < j)));
          if (pos >= kmax) return;
#pragma unroll
          for (int k = MAXK - 1; k > 0; --k)
            if (k > pos) { tk[k] = tk[k - 1]; tj[k] = tj[k - 1]; }
#pragma unroll
          for (int k = 0; k < MAXK; ++k)
            if (k == pos) { tk[k] = key; tj[k] = j; }
          nb = min(nb + 1, kmax);
        };
        if constexpr (kLanes == 2) {
          // every j with key < nd^2 lies in the 3 x 3 cells around a's cell (see above)
          const int cx = s_cell[a] % bins.ncx, cy = s_cell[a] / bins.ncx;
          const int x0 = max(cx - 1, 0), x1 = min(cx + 1, bins.ncx - 1);
          for (int d = 0; d < 3; ++d) {
            const int row = cy - 1 + d;
            if (row < 0 || row >= bins.ncy) continue;
            const int c0 = row * bins.ncx + x0, c1 = row * bins.ncx + x1;
            const int t1 = s_cend[c1];
            for (int tt = c0 > 0 ? s_cend[c0 - 1] : 0; tt < t1; ++tt) {
              const int j = s_sorted[tt];   // active agents only
              if (j == a) continue;
              const float xj = s_fx[j], yj = s_fy[j], sqj = s_fsq[j];
              float dot = __fmaf_rn(yi, yj, __fmul_rn(xi, xj));
              float key = __fsub_rn(__fadd_rn(sqi, sqj), __fmul_rn(2.0f, dot));
              if (key < P.nd2_f32) insert(key, j);
            }
          }
        } else {
        for (int j0 = 0; j0 < A; j0 += 32) {
         unsigned inr = 0u;
         const int jn = min(32, A - j0);
         for (int u = 0; u < jn; ++u) {
          const int j = j0 + u;
          const float xj = s_fx[j], yj = s_fy[j], sqj = s_fsq[j];
          float dot = __fmaf_rn(yi, yj, __fmul_rn(xi, xj));
          float key = __fsub_rn(__fadd_rn(sqi, sqj), __fmul_rn(2.0f, dot));
          inr |= (unsigned)((key < P.nd2_f32) & (j != a) & (s_act[j] != 0)) << u;
         }
         while (inr) {
          const int j = j0 + __ffs(inr) - 1;
          inr &= inr - 1u;
          const float xj = s_fx[j], yj = s_fy[j], sqj = s_fsq[j];
          float dot = __fmaf_rn(yi, yj, __fmul_rn(xi, xj));
          float key = __fsub_rn(__fadd_rn(sqi, sqj), __fmul_rn(2.0f, dot));
          // j increases, so every kept entry has a smaller index: (key, index) order is
          // "after every kept entry with key <= this key"
          int pos = 0;
#pragma unroll
          for (int k = 0; k < MAXK; ++k) pos += (k < nb && tk[k] <= key);
          if (pos >= kmax) continue;
#pragma unroll
          for (int k = MAXK - 1; k > 0; --k)
            if (k > pos) { tk[k] = tk[k - 1]; tj[k] = tj[k - 1]; }
#pragma unroll
          for (int k = 0; k < MAXK; ++k)
            if (k == pos) { tk[k] = key; tj[k] = j; }
          nb = min(nb + 1, kmax);
         }
        }
        }
        // thread-local arrays indexed at run time (local memory, L1-resident): slots
        // >= nc are never read
        double cpx[MAXC], cpy[MAXC], cnx[MAXC], cny[MAXC];
        if (nb > 0) {   // field.py:268-271: gap to the nearest neighbour
          const int j = tj[0];
          double rp0 = s_px[j] - px, rp1 = s_py[j] - py;
          double d_near = sqrt(rp0 * rp0 + rp1 * rp1);
          my_gap = fmin(my_gap, d_near - (ra + s_r[j]));
          my_anynb = 1;
        }
        int tjk = tj[0];
#pragma unroll 1
        for (int k = 0; k < nb; ++k) {   // rolled: one copy of vo_halfplane
#pragma unroll
          for (int r = 0; r < MAXK; ++r) tjk = r == k ? tj[r] : tjk;
          const int j = tjk;
          double rp0 = s_px[j] - px, rp1 = s_py[j] - py;
          double rv0 = vxa - s_vx[j], rv1 = vya - s_vy[j];
          double rr = ra + s_r[j] + P.safety_margin;
          const HalfPlane h = vo_halfplane_ool(rp0, rp1, rv0, rv1, rr, P.time_horizon, P.dt, vxa, vya, 0.5);
          put_slot(cpx, k, h.p0); put_slot(cpy, k, h.p1); put_slot(cnx, k, h.n0); put_slot(cny, k, h.n1);
        }
        int nc = nb;
        if (use_robot) {
          double rp0 = rpx - px, rp1 = rpy - py;
          double d2 = rp0 * rp0 + rp1 * rp1;
          if (d2 < P.nd2) {
            double rr = ra + robot_radius + P.safety_margin;
            const HalfPlane h = vo_halfplane_ool(rp0, rp1, vxa - rvx, vya - rvy, rr, P.obstacle_time_horizon,
                                                 P.dt, vxa, vya, 1.0);
            put_slot(cpx, nc, h.p0); put_slot(cpy, nc, h.p1); put_slot(cnx, nc, h.n0); put_slot(cny, nc, h.n1);
            ++nc;
          }
        }
        if (P.use_static && has_obs) {
          const int flat = flat_pre;
          if (flat >= 0) {
            int orow = flat / nx, ocol = flat - orow * nx;
            double rp0 = ((double)ocol + 0.5) * res - px, rp1 = ((double)orow + 0.5) * res - py;
            double d2 = rp0 * rp0 + rp1 * rp1;
            if (d2 < P.nd2) {
              double margin = 0.5 * kSqrt2 * P.res0;
              double rr = ra + margin + P.safety_margin;
              const HalfPlane h = vo_halfplane_ool(rp0, rp1, vxa, vya, rr, P.obstacle_time_horizon, P.dt, vxa,
                                                   vya, 1.0);
              put_slot(cpx, nc, h.p0); put_slot(cpy, nc, h.p1); put_slot(cnx, nc, h.n0); put_slot(cny, nc, h.n1);
              ++nc;
            }
          }
        }
        const double ms = S.max_speed[ia];
        double v0, v1;
        const double want = sqrt(pf0 * pf0 + pf1 * pf1);
        double q0 = pf0, q1 = pf1;
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {   // second pass = stall retry (one LP copy)
          fallbacks += lane_lp(cpx, cpy, cnx, cny, nc, q0, q1, ms, v0, v1);
          if (pass == 1) break;
          const double spd = sqrt(v0 * v0 + v1 * v1);
          if (!(spd < 0.2 * want && want > 1e-6)) break;
          ++stalls;
          q0 = P.stall_c * pf0 + P.stall_s * pf1;
          q1 = -P.stall_s * pf0 + P.stall_c * pf1;
        }
        double npx = px + v0 * P.dt, npy = py + v1 * P.dt;
        bool out = npx < 0 || npy < 0 || npx >= nx * res || npy >= ny * res;
        long long rr = clampll(trunc_ll(div_h(npy, res)), 0, ny - 1);
        long long cc = clampll(trunc_ll(div_h(npx, res)), 0, nx - 1);
        bool blocked = out || lab[rr * nx + cc] == L_OBSTACLE;
        if (!blocked) {
          S.pos[ia * 2] = npx;
          S.pos[ia * 2 + 1] = npy;
          s_nx[a] = npx;
          s_ny[a] = npy;
        }
        S.vel[ia * 2] = blocked ? 0.0 : v0;
        S.vel[ia * 2 + 1] = blocked ? 0.0 : v1;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        my_gap = fmin(my_gap, __shfl_xor_sync(0xffffffffu, my_gap, o));
        my_anynb |= __shfl_xor_sync(0xffffffffu, my_anynb, o);
        fallbacks += __shfl_xor_sync(0xffffffffu, fallbacks, o);
        stalls += __shfl_xor_sync(0xffffffffu, stalls, o);
      }
    }
    for (int a = wid; a < A && !lanes; a += NW) {
      if (!s_act[a]) continue;
      const double px = s_px[a], py = s_py[a];
      const size_t ia = eA + a;
      const double gx = S.goal[ia * 2], gy = S.goal[ia * 2 + 1];
      const double wx = S.waypoint[ia * 2], wy = S.waypoint[ia * 2 + 1];
      // ---------------- preferred velocity (field.py:214-227)
      const double sp = S.pref_speed[ia];
      double tw0 = wx - px, tw1 = wy - py;
      double dist = sqrt(tw0 * tw0 + tw1 * tw1);
      double safe = fmax(dist, kEps);
      double pf0 = tw0 / safe * sp, pf1 = tw1 / safe * sp;
      double tg0 = gx - px, tg1 = gy - py;
      double dg = sqrt(tg0 * tg0 + tg1 * tg1);
      double scl = fmin(1.0, dg / fmax(sp * P.dt * 4, kEps));
      pf0 = pf0 * scl;
      pf1 = pf1 * scl;
      // ---------------- neighbours: fp32 Gram key, stable top-K (field.py:246-262)
      const float xi = (float)px, yi = (float)py;
      const float sqi = __fadd_rn(__fmul_rn(xi, xi), __fmul_rn(yi, yi));
      const double vxa = s_vx[a], vya = s_vy[a], ra = s_r[a];
      float last_k = -CUDART_INF_F;
      int last_j = -1;
      int nb = 0;
      int my_nb = -1;
      const int kmax = min(P.max_neighbors, max(A - 1, 0));
      // candidate ranges: all agents, or the three cell-row runs around a's cell
      int rs[3] = {0, 0, 0}, re[3] = {A, 0, 0};
      if (bins.ncx > 0) {
        const int cx = s_cell[a] % bins.ncx, cy = s_cell[a] / bins.ncx;
        const int x0 = max(cx - 1, 0), x1 = min(cx + 1, bins.ncx - 1);
  #pragma unroll
        for (int d = 0; d < 3; ++d) {
          const int row = cy - 1 + d;
          const bool ok = row >= 0 && row < bins.ncy;
          const int c0 = row * bins.ncx + x0, c1 = row * bins.ncx + x1;
          rs[d] = ok ? (c0 > 0 ? s_cend[c0 - 1] : 0) : 0;
          re[d] = ok ? s_cend[c1] : 0;
        }
      }
      for (int round = 0; round < kmax; ++round) {
        float bk = CUDART_INF_F;
        int bj = 0x7fffffff;
  #pragma unroll
        for (int d = 0; d < 3; ++d) {
          for (int t = rs[d] + lane; t < re[d]; t += 32) {
            const int j = bins.ncx > 0 ? s_sorted[t] : t;
            if (j == a || !s_act[j]) continue;
            float xj = (float)s_px[j], yj = (float)s_py[j];
            float sqj = __fadd_rn(__fmul_rn(xj, xj), __fmul_rn(yj, yj));
            float dot = __fmaf_rn(yi, yj, __fmul_rn(xi, xj));
            float key = __fsub_rn(__fadd_rn(sqi, sqj), __fmul_rn(2.0f, dot));
            if (!(key < P.nd2_f32)) continue;
            bool after = key > last_k || (key == last_k && j > last_j);
            bool better = key < bk || (key == bk && j < bj);
            if (after && better) { bk = key; bj = j; }
          }
        }
  #pragma unroll
        for (int o = 16; o; o >>= 1) {
          float ok_ = __shfl_xor_sync(0xffffffffu, bk, o);
          int oj = __shfl_xor_sync(0xffffffffu, bj, o);
          if (ok_ < bk || (ok_ == bk && oj < bj)) { bk = ok_; bj = oj; }
        }
        if (bj == 0x7fffffff) break;
        if (lane == round) my_nb = bj;
        last_k = bk;
        last_j = bj;
        ++nb;
      }
      // ---------------- constraints (compact list of valid lanes)
      if (lane < nb) {
        const int j = my_nb;
        double rp0 = s_px[j] - px, rp1 = s_py[j] - py;
        double rv0 = vxa - s_vx[j], rv1 = vya - s_vy[j];
        double rr = ra + s_r[j] + P.safety_margin;
        vo_halfplane(rp0, rp1, rv0, rv1, rr, P.time_horizon, P.dt, vxa, vya, 0.5, C.px[lane],
                     C.py[lane], C.nx[lane], C.ny[lane]);
        if (lane == 0) {
          double d_near = sqrt(rp0 * rp0 + rp1 * rp1);   // field.py:268-271
          my_gap = fmin(my_gap, d_near - (ra + s_r[j]));
          my_anynb = 1;
        }
      }
      int nc = nb;
      if (use_robot) {
        double rp0 = rpx - px, rp1 = rpy - py;
        double d2 = rp0 * rp0 + rp1 * rp1;
        if (d2 < P.nd2) {
          if (lane == nc) {
            double rr = ra + robot_radius + P.safety_margin;
            vo_halfplane(rp0, rp1, vxa - rvx, vya - rvy, rr, P.obstacle_time_horizon, P.dt, vxa, vya,
                         1.0, C.px[lane], C.py[lane], C.nx[lane], C.ny[lane]);
          }
          ++nc;
        }
      }
      if (P.use_static && has_obs) {
        long long ri = clampll(trunc_ll(div_h(py, res)), 0, ny - 1);
        long long ci = clampll(trunc_ll(div_h(px, res)), 0, nx - 1);
        int flat = S.nearest[e * N + ri * nx + ci];
        if (flat >= 0) {
          int orow = flat / nx, ocol = flat - orow * nx;
          double rp0 = ((double)ocol + 0.5) * res - px, rp1 = ((double)orow + 0.5) * res - py;
          double d2 = rp0 * rp0 + rp1 * rp1;
          if (d2 < P.nd2) {
            if (lane == nc) {
              double margin = 0.5 * kSqrt2 * P.res0;
              double rr = ra + margin + P.safety_margin;
              vo_halfplane(rp0, rp1, vxa, vya, rr, P.obstacle_time_horizon, P.dt, vxa, vya, 1.0,
                           C.px[lane], C.py[lane], C.nx[lane], C.ny[lane]);
            }
            ++nc;
          }
        }
      }
      __syncwarp();
      // ---------------- LP + stall retry (field.py:133-150)
      const double ms = S.max_speed[ia];
      double v0, v1;
      fallbacks += warp_lp(C, Q, nc, pf0, pf1, ms, v0, v1, lane);
      double spd = sqrt(v0 * v0 + v1 * v1);
      double want = sqrt(pf0 * pf0 + pf1 * pf1);
      if (spd < 0.2 * want && want > 1e-6) {
        ++stalls;
        double q0 = P.stall_c * pf0 + P.stall_s * pf1;
        double q1 = -P.stall_s * pf0 + P.stall_c * pf1;
        fallbacks += warp_lp(C, Q, nc, q0, q1, ms, v0, v1, lane);
      }
      // ---------------- commit (field.py:152-160, 352-366)
      double npx = px + v0 * P.dt, npy = py + v1 * P.dt;
      bool out = npx < 0 || npy < 0 || npx >= nx * res || npy >= ny * res;
      long long rr = clampll(trunc_ll(div_h(npy, res)), 0, ny - 1);
      long long cc = clampll(trunc_ll(div_h(npx, res)), 0, nx - 1);
      bool blocked = out || lab[rr * nx + cc] == L_OBSTACLE;
      if (lane == 0) {
        if (!blocked) {
          S.pos[ia * 2] = npx;
          S.pos[ia * 2 + 1] = npy;
          s_nx[a] = npx;
          s_ny[a] = npy;
        }
        S.vel[ia * 2] = blocked ? 0.0 : v0;
        S.vel[ia * 2 + 1] = blocked ? 0.0 : v1;
      }
      __syncwarp();
    }
    if (lane == 0) {
      s_gap[wid] = my_gap;
      s_anynb[wid] = my_anynb;
    }
    __syncthreads();
    // ---------------- goal resample, agent order (field.py:368-381)
    // warp 0: lanes test 32 agents' goal reach at once (independent loads), lane 0
    // then draws for the reached ones in agent order (rare: the rng stream order is
    // the reference's)
    if (wid == 0) {
      if (lane == 0) {
        double g = CUDART_INF;
        int anynb = 0;
        for (int w = 0; w < NW; ++w) { g = fmin(g, s_gap[w]); anynb |= s_anynb[w]; }
        if (ra) {
          ra->gap_hist[(size_t)e * ra->T + tick] = g;
          if (anynb) ra->anynb[tick] = 1;
        } else {
          S.gap_tmp[e] = g;
          if (anynb) atomicOr(&S.flags[0], 1);
        }
      }
      if (P.resample_goals) {
        Pcg64Raw* raw = reinterpret_cast<Pcg64Raw*>(S.rng) + e;
        bool loaded = false;
        Pcg64 rng;
        const int wn = S.walk_n[e];
        for (int a0 = 0; a0 < A; a0 += 32) {
          bool hit = false;
          if (a0 + lane < A && s_act[a0 + lane]) {
            const size_t ia = eA + a0 + lane;
            double dx = S.goal[ia * 2] - s_nx[a0 + lane], dy = S.goal[ia * 2 + 1] - s_ny[a0 + lane];
            hit = dx * dx + dy * dy < P.goal_reach2;
          }
          unsigned m = __ballot_sync(0xffffffffu, hit);
          if (lane != 0) continue;
          while (m) {
            const int a = a0 + __ffs(m) - 1;
            m &= m - 1u;
            const size_t ia = eA + a;
            if (!loaded) { rng = pcg_load(*raw); loaded = true; }
            int k = (int)integers32(rng, (uint64_t)wn);
            int f = S.walk[e * N + k];
            int r = f / nx, c = f - r * nx;
            S.goal[ia * 2] = ((double)c + 0.5) * res;
            S.goal[ia * 2 + 1] = ((double)r + 0.5) * res;
            S.path_n[ia] = 0;
          }
        }
        if (lane == 0 && loaded) pcg_store(*raw, rng);
      }
    }
    if (lane == 0 && S.counters) {
      if (fallbacks) atomicAdd((unsigned long long*)&S.counters[2], (unsigned long long)fallbacks);
      if (stalls) atomicAdd((unsigned long long*)&S.counters[3], (unsigned long long)stalls);
    }
    if (threadIdx.x == 0 && S.counters) {
      long long tc = clock64() - t_cta0;
      atomicAdd((unsigned long long*)&S.counters[6], (unsigned long long)tc);
      atomicMax((unsigned long long*)&S.counters[7], (unsigned long long)tc);
    }
  }
}

CW_DEV void orca_tail(const cw_crowd_params& P, const cw_crowd_state& S, int pass, bool pdl = false);

template <int NT, int kLanes = 0>
__global__ void __launch_bounds__(NT) k_orca(cw_crowd_params P, cw_crowd_state S,
                                             const double* __restrict__ robot_pos,
                                             const double* __restrict__ robot_vel,
                                             double robot_radius,
                                             const uint8_t* __restrict__ env_mask, Bins bins,
                                             int pass) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int e = blockIdx.x;
  // pass 0: every env; pass 1: envs without A* requests (runs beside k_astar);
  // pass 2: envs with requests (after k_astar).  The body is per env.
  const bool skip = (pass == 1 && S.env_req[e]) || (pass == 2 && !S.env_req[e]);
  if (!skip) orca_env<NT, kLanes>(P, S, e, robot_pos, robot_vel, robot_radius, env_mask, bins, sm, nullptr, 0);
  orca_tail(P, S, pass);
}

// Early commit (next-tick prefetch): pass 2 launched beside k_astar (programmatic
// dependent launch: its CTAs start once every search CTA is resident, so waiting here
// can never keep a search from running).  The CTA of an env with replans waits for
// the env's own searches only, commits it, and at once predicts its next replans
// (dry guidance pass) into the prefetch batch, whose search warps are still polling.
template <int NT, int kLanes>
__global__ void __launch_bounds__(NT) k_orca_ec(cw_crowd_params P, cw_crowd_state S,
                                                const double* __restrict__ robot_pos,
                                                const double* __restrict__ robot_vel, double robot_radius,
                                                const uint8_t* __restrict__ env_mask, Bins bins, SpecArgs sa) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int e = blockIdx.x;
  if (S.env_req[e]) {
    if (threadIdx.x == 0) {
      while (ld_acquire_i32(&sa.pend[e]) > 0) __nanosleep(256);
      __threadfence();
    }
    __syncthreads();
    orca_env<NT, kLanes>(P, S, e, robot_pos, robot_vel, robot_radius, env_mask, bins, sm, nullptr, 0);
    __syncthreads();
    guide_env<NT, false, true>(P, S, e, nullptr, nullptr, &sa, true);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&sa.qn[3], 1);
    }
  }
  orca_tail(P, S, 2, true);
  // block 0 waits for the search grid: this grid (and so the stream) completes after
  // it, and its request queue is reset only when no search warp can still touch it
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    S.flags[4] = 0;
    S.flags[5] = 0;
  }
}

// ---------------- last CTA: publish last_gap_by_env (only when some row had K > 0),
// reset the per-step flags and the A* queue
CW_DEV void orca_tail(const cw_crowd_params& P, const cw_crowd_state& S, int pass, bool pdl) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const int ticket = atomicAdd(&S.flags[2], 1);
    s_last = 0;
    if (ticket == (pass == 0 ? 1 : 2) * (int)gridDim.x - 1) {   // last CTA over all passes
      __threadfence();
      s_last = atomicAdd(&S.flags[0], 0) ? 2 : 1;
    }
  }
  __syncthreads();
  if (s_last) {
    if (s_last == 2)   // the whole CTA copies (one thread's serial copy cost ~0.3 ms at E = 1024)
      for (int k = threadIdx.x; k < P.E; k += blockDim.x) S.last_gap[k] = ((volatile double*)S.gap_tmp)[k];
    __syncthreads();
    if (threadIdx.x == 0) {
      S.flags[0] = 0;
      S.flags[2] = 0;
      if (!pdl) {   // beside k_astar (k_orca_ec) its block 0 resets the queue instead
        S.flags[4] = 0;
        S.flags[5] = 0;
      }
    }
  }
}

// ---------------------------------------------------------------- multi-tick run
// Round CTAs pop ready envs (ring of env ids) and advance each one tick after
// tick until it has to wait for its own searches (the server re-queues it when
// the last one finishes), has run `burst` ticks (re-queued at the back), or
// reaches T; a CTA exits when no env is ready, and the host keeps launching
// rounds until every env is done.  An env is in the ring at most once, so no
// two CTAs ever work on the same env.
template <int NT, int kLanes>
__global__ void __launch_bounds__(NT) k_round(cw_crowd_params P, cw_crowd_state S,
                                              const double* __restrict__ robot_pos,
                                              const double* __restrict__ robot_vel, double robot_radius,
                                              const uint8_t* __restrict__ env_mask, Bins bins,
                                              RunArgs ra) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ int s_e, s_st, s_go;
  if (threadIdx.x == 0) atomicAdd(&ra.q->active_rounds, 1);   // seen by the server's exit test
  while (true) {
    if (threadIdx.x == 0) {
      const int e = ready_pop(ra);
      s_e = e;
      if (e >= 0) {
        __threadfence();   // the server's results (acquire through the ring) before reading state
        s_st = ra.env_state[e];
        if (ra.trace) {
          long long* tr = ra.trace + (size_t)e * 8;
          const long long now = global_ns();
          tr[kTrQueueWait] += now - tr[kTrMark];
          tr[kTrMark] = now;
        }
      }
    }
    __syncthreads();
    const int e = s_e;
    if (e < 0) {
      if (threadIdx.x == 0) atomicSub(&ra.q->active_rounds, 1);
      return;
    }
    int t = s_st >> 2;
    const int stop = ra.stop ? ra.stop[e] : ra.T;
    if (t >= stop) {   // nothing to run in this call (cw_crowd_run_window)
      if (threadIdx.x == 0) {
        ra.env_state[e] = (t << 2) | kRunDone;
        __threadfence();
        if (atomicAdd(&ra.q->n_done, 1) + 1 == ra.E) atomicExch(&ra.q->shutdown, 1);
      }
      __syncthreads();
      continue;
    }
    bool guide = (s_st & 3) == kRunGuide;
    for (int burst = 0;; ++burst) {
      if (burst == ra.burst) {   // yield to the envs queued behind this one
        if (threadIdx.x == 0) {
          if (ra.trace) {
            long long* tr = ra.trace + (size_t)e * 8;
            const long long now = global_ns();
            tr[kTrBusy] += now - tr[kTrMark];
            tr[kTrMark] = now;
          }
          ra.env_state[e] = (t << 2) | kRunGuide;
          __threadfence();
          ready_push(ra, e);
        }
        break;
      }
      if (guide) {
        if (threadIdx.x == 0) {
          ra.pending[e] = kPendingGuard;   // searches may finish before the count is known
          ra.env_state[e] = (t << 2) | kRunWait;
          __threadfence();
        }
        const long long tg0 = clock64();
        const int n = guide_env<NT, true>(P, S, e, env_mask, &ra);
        if (threadIdx.x == 0 && S.counters)
          atomicAdd((unsigned long long*)&S.counters[8], (unsigned long long)(clock64() - tg0));
        if (threadIdx.x == 0) {
          if (ra.trace && n) {   // busy until here; a search wait starts (the server may be done)
            long long* tr = ra.trace + (size_t)e * 8;
            const long long now = global_ns();
            tr[kTrBusy] += now - tr[kTrMark];
            tr[kTrMark] = now;
            tr[kTrWaits] += 1;
          }
          const int left = atomicSub(&ra.pending[e], kPendingGuard - n) - (kPendingGuard - n);
          __threadfence();
          s_go = left == 0;   // else the server queues the env after its last search
        }
        __syncthreads();
        if (!s_go) break;
      }
      orca_env<NT, kLanes>(P, S, e, robot_pos, robot_vel, robot_radius, env_mask, bins, sm, &ra, t);
      __syncthreads();
      if (threadIdx.x == 0) atomicAdd(&ra.q->progress, 1);
      if (++t == stop) {
        if (threadIdx.x == 0) {
          if (ra.trace) {
            long long* tr = ra.trace + (size_t)e * 8;
            const long long now = global_ns();
            tr[kTrBusy] += now - tr[kTrMark];
            tr[kTrDone] = now;
          }
          ra.env_state[e] = (t << 2) | kRunDone;
          __threadfence();
          if (atomicAdd(&ra.q->n_done, 1) + 1 == ra.E) atomicExch(&ra.q->shutdown, 1);
        }
        break;
      }
      guide = true;
    }
    __syncthreads();
  }
}

__global__ void k_run_init(RunArgs ra) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ra.trace && i < (size_t)ra.E) ra.trace[i * 8 + kTrMark] = global_ns();
  // every env starts in the ready ring (positions 0..E-1)
  if (i == 0) *ra.q = RunQueue{0ull, 0ull, 0, 0, 0, 0, 0, 0, 0ull, (unsigned long long)ra.E, 0ull, 0ull};
  if (i < (size_t)ra.E) {
    ra.env_state[i] = (ra.start ? ra.start[i] : 0) << 2;   // kRunGuide at the env's first tick
    ra.pending[i] = 0;
    ra.ritems[i] = (int)i;
  }
  if (i <= ra.rmask) {
    ra.rseq[i] = i < (size_t)ra.E ? i + 1 : i;
    ra.useq[i] = i;
  }
  if (ra.init_hist && i < (size_t)ra.T) ra.anynb[i] = 0;
  if (i <= ra.mask) ra.seq[i] = i;
}

// last_gap_by_env as T synchronous ticks leave it: the gaps of the last tick on
// which some env had a neighbour (k_orca's last-CTA publication).
__global__ void k_run_finish(cw_crowd_state S, RunArgs ra) {
  __shared__ int s_t;
  if (threadIdx.x == 0) {
    int t = ra.T - 1;
    while (t >= 0 && !ra.anynb[t]) --t;
    s_t = t;
  }
  __syncthreads();
  if (s_t < 0) return;
  for (int e = threadIdx.x; e < ra.E; e += blockDim.x)
    S.last_gap[e] = ra.gap_hist[(size_t)e * ra.T + s_t];
}

__global__ void k_seed_streams(int n, const uint64_t* __restrict__ seeds, Pcg64Raw* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) pcg_store(out[i], pcg_seed(seeds[i]));
}

__global__ void k_child_seeds(int n, const uint64_t* __restrict__ parent, int label_id,
                              const uint64_t* __restrict__ k, uint64_t* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const char* labels[4] = {"env", "crowd-run", "crowd", "resample"};
  if (k) out[i] = child_seed(parent[i], labels[label_id], k[i]);
  else out[i] = child_seed(parent[i], labels[label_id]);
}

// Internal streams for the overlapped tick: k_astar (+ the requesting envs' k_orca)
// on a high-priority stream, the other envs' k_orca on a low-priority one, both
// joined back into the caller's stream.  Created once per process.
struct TickStreams {
  cudaStream_t hi = nullptr, lo = nullptr;
  cudaEvent_t guided, hi_done, lo_done;
};

static TickStreams& tick_streams() {
  static TickStreams t;
  if (!t.hi) {
    int least, greatest;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    cudaStreamCreateWithPriority(&t.hi, cudaStreamNonBlocking, greatest);
    cudaStreamCreateWithPriority(&t.lo, cudaStreamNonBlocking, least);
    cudaEventCreateWithFlags(&t.guided, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&t.hi_done, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&t.lo_done, cudaEventDisableTiming);
  }
  return t;
}

static void launch_astar(const cw_crowd_params& P, const cw_crowd_state& S, cudaStream_t st,
                         const SpecArgs& sp = SpecArgs{}) {
  const int W = P.astar_warps == 1 ? 1 : kAstarWarps;
  const AstarShape A = astar_shape(P.nx, P.ny, W);
  const RunArgs none = {};
  if (W == 1) k_astar<1, false><<<P.astar_ctas, 32, A.smem, st>>>(P, S, A.NC, A.NS, none, sp);
  else k_astar<kAstarWarps, false><<<P.astar_ctas, 32 * kAstarWarps, A.smem, st>>>(P, S, A.NC, A.NS, none, sp);
}

// ---- next-tick search prefetch context (cw_spec_create)
// Batches rotate over kSpecBatches low-priority streams: a batch may still be
// finishing a search the next tick waits for while the following batch starts.
// Scratch is indexed by (SM, warp): a search CTA needs more than half of an SM's
// shared memory, so no two are ever resident on one SM.
constexpr int kSpecBatches = 8;
struct SpecCtx {
  int E = 0, A = 0, path_cap = 0, heap_cap = 0, nx = 0, ny = 0, nsm = 0;
  SpecEnt* ent = nullptr;
  int32_t* cells = nullptr;
  AstarReq* q[kSpecBatches] = {};
  int* qr[kSpecBatches] = {};              // per item: batch tag once written
  int* pend = nullptr;                     // (E) early commit: searches left per env
  cudaEvent_t bdone[kSpecBatches] = {};    // the batch's search kernel is done
  int* qn = nullptr;                       // kSpecBatches x 4
  unsigned long long* stats = nullptr;     // 4
  unsigned char* rec = nullptr;
  OpenEnt* heap = nullptr;
  size_t stride = 0;
  cudaEvent_t guided = nullptr;            // the last dry guidance pass is done
  int next = 0;
  unsigned long long tag = 0;
  long long batches = 0;
};

static cudaStream_t spec_stream(int b) {
  static cudaStream_t s[kSpecBatches] = {};
  if (!s[0]) {
    int least, greatest;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    for (int k = 0; k < kSpecBatches; ++k) cudaStreamCreateWithPriority(&s[k], cudaStreamNonBlocking, least);
  }
  return s[b];
}

__global__ void k_nsmid(int* out) {
  unsigned r;
  asm volatile("mov.u32 %0, %%nsmid;" : "=r"(r));
  *out = (int)r;
}

static size_t spec_layout(const cw_crowd_params& P, int nsm, size_t* parts) {
  const size_t EA = (size_t)P.E * P.A;
  auto up = [](size_t v) { return (v + 255) & ~(size_t)255; };
  const size_t warps = (size_t)nsm * kAstarWarps;
  parts[0] = up(EA * sizeof(SpecEnt));
  parts[1] = up(EA * (size_t)P.path_cap * 4);
  parts[2] = up(EA * sizeof(AstarReq)) * kSpecBatches;
  parts[3] = up((size_t)kSpecBatches * 4 * 4 + 4 * 8);
  parts[4] = warps * astar_slot_stride(P.nx, P.ny);
  parts[5] = up(warps * (size_t)P.heap_cap * sizeof(OpenEnt));
  parts[6] = up(EA * 4) * kSpecBatches + up((size_t)P.E * 4);   // item flags, pending counts
  size_t t = 0;
  for (int k = 0; k < 7; ++k) t += parts[k];
  return t;
}

static SpecArgs spec_args(const SpecCtx* X, int mode, const int32_t* epoch, int b) {
  SpecArgs a{};
  a.mode = mode;
  a.ent = X->ent;
  a.cells = X->cells;
  a.epoch = epoch;
  a.q = X->q[b];
  a.qn = X->qn + 4 * b;
  a.rec = X->rec;
  a.heap = X->heap;
  a.rec_stride = X->stride;
  a.tag = X->tag;
  a.stats = X->stats;
  a.qr = X->qr[b];
  a.pend = nullptr;
  return a;
}

// ---- cw_crowd_run scratch layout
struct RunLayout {
  unsigned long long cap, rcap;
  size_t q, env_state, pending, seq, items, rseq, ritems, useq, uitems, gap_hist, anynb, total;
};

static RunLayout run_layout(int E, int A, int T) {
  RunLayout L;
  unsigned long long need = 2ull * (unsigned long long)E * (unsigned long long)A, cap = 1024;
  while (cap < need) cap <<= 1;
  L.cap = cap;
  auto up = [](size_t v) { return (v + 255) & ~(size_t)255; };
  L.q = 0;
  L.env_state = up(sizeof(RunQueue));
  L.pending = L.env_state + up((size_t)E * 4);
  L.seq = L.pending + up((size_t)E * 4);
  L.items = L.seq + up((size_t)cap * 8);
  unsigned long long rcap = 1024;
  while (rcap < (unsigned long long)E) rcap <<= 1;
  L.rcap = rcap;
  L.rseq = L.items + up((size_t)cap * sizeof(AstarReq));
  L.ritems = L.rseq + up((size_t)rcap * 8);
  L.useq = L.ritems + up((size_t)rcap * 4);
  L.uitems = L.useq + up((size_t)rcap * 8);
  L.gap_hist = L.uitems + up((size_t)rcap * 4);
  L.anynb = L.gap_hist + up((size_t)E * T * 8);
  L.total = L.anynb + up((size_t)T * 4);
  return L;
}

constexpr int kRoundStreams = 8;
static long long g_last_rounds = 0;   // rounds launched by the last cw_crowd_run
static long long g_last_servers = 0;  // search-server launches of the last cw_crowd_run

template <int NT>
static int launch_run(const cw_crowd_params& P, const cw_crowd_state& S, const double* rp,
                      const double* rv, double rr, const uint8_t* em, int ticks, const int32_t* start,
                      const int32_t* stop, int flags, void* scratch, cudaStream_t st) {
  const Bins bins = make_bins(P);
  static const bool warp_orca = getenv("CW_RUN_WARP_ORCA") != nullptr;   // A/B
  const bool lanes_ok = P.max_neighbors <= MAXK && !warp_orca;
  // the lane path needs no per-warp constraint block: a smaller footprint lets two
  // round CTAs share an SM with a search-server CTA
  const size_t sm = lanes_ok ? (size_t)P.A * 7 * sizeof(double) + (size_t)((P.A + 15) & ~15) + 16 +
                                   (size_t)P.A * 3 * sizeof(float) + bins_smem_bytes(bins, P.A)
                             : cw_crowd_step_smem_bytes(P.A, NT) + bins_smem_bytes(bins, P.A);
  static bool attrs = false;
  if (!attrs) {
    cudaFuncSetAttribute(k_astar<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    // the server and the rounds share SMs only under one L1 / shared split
    cudaFuncSetAttribute(k_astar<1, true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(k_astar<kAstarWarps, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    cudaFuncSetAttribute(k_astar<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_astar<2, true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(k_astar<kAstarWarps, true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(k_round<NT, 2>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(k_round<NT, 1>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(k_round<NT, 0>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    // Reserve the per-thread local memory (stack) of every kernel of the run now, while
    // nothing is running: a launch that outgrows the reservation makes the driver grow
    // it, which waits for the device to drain -- and the persistent server only drains
    // after the rounds that launch is holding back.
    size_t need = 0;
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, k_round<NT, 2>) == cudaSuccess) need = std::max(need, fa.localSizeBytes);
    if (cudaFuncGetAttributes(&fa, k_round<NT, 1>) == cudaSuccess) need = std::max(need, fa.localSizeBytes);
    if (cudaFuncGetAttributes(&fa, k_round<NT, 0>) == cudaSuccess) need = std::max(need, fa.localSizeBytes);
    if (cudaFuncGetAttributes(&fa, k_astar<1, true>) == cudaSuccess) need = std::max(need, fa.localSizeBytes);
    if (cudaFuncGetAttributes(&fa, k_astar<2, true>) == cudaSuccess) need = std::max(need, fa.localSizeBytes);
    if (cudaFuncGetAttributes(&fa, k_astar<kAstarWarps, true>) == cudaSuccess)
      need = std::max(need, fa.localSizeBytes);
    size_t cur = 0;
    cudaDeviceGetLimit(&cur, cudaLimitStackSize);
    if (need > cur) cudaDeviceSetLimit(cudaLimitStackSize, (need + 255) & ~(size_t)255);
    cudaGetLastError();
    attrs = true;
  }
  // lane-per-agent ORCA (cell-binned candidates from 128 agents on); the warp path only
  // for more than MAXK neighbours (CW_RUN_WARP_ORCA forces it for A/B runs)
  const bool lanes = lanes_ok;
  if (sm > 48 * 1024) {
    cudaFuncSetAttribute(k_round<NT, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_round<NT, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_round<NT, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  }
  const RunLayout L = run_layout(P.E, P.A, ticks);
  unsigned char* base = static_cast<unsigned char*>(scratch);
  RunArgs ra;
  ra.q = reinterpret_cast<RunQueue*>(base + L.q);
  ra.env_state = reinterpret_cast<int*>(base + L.env_state);
  ra.pending = reinterpret_cast<int*>(base + L.pending);
  ra.seq = reinterpret_cast<unsigned long long*>(base + L.seq);
  ra.items = reinterpret_cast<AstarReq*>(base + L.items);
  ra.rseq = reinterpret_cast<unsigned long long*>(base + L.rseq);
  ra.ritems = reinterpret_cast<int*>(base + L.ritems);
  ra.useq = reinterpret_cast<unsigned long long*>(base + L.useq);
  ra.uitems = reinterpret_cast<int*>(base + L.uitems);
  ra.rmask = L.rcap - 1;
  ra.gap_hist = reinterpret_cast<double*>(base + L.gap_hist);
  ra.anynb = reinterpret_cast<int*>(base + L.anynb);
  ra.T = ticks;
  ra.E = P.E;
  ra.start = start;
  ra.stop = stop;
  ra.init_hist = flags & 1;
  ra.mask = L.cap - 1;
  static const int burst = getenv("CW_RUN_BURST") ? atoi(getenv("CW_RUN_BURST")) : 8;
  ra.burst = std::max(1, burst);
  static long long* trace = nullptr;
  static int trace_e = 0;
  static const bool want_trace = getenv("CW_RUN_TRACE") != nullptr;
  ra.trace = nullptr;
  if (want_trace) {
    if (trace_e < P.E) { if (trace) cudaFree(trace); cudaMalloc(&trace, (size_t)P.E * 64); trace_e = P.E; }
    cudaMemsetAsync(trace, 0, (size_t)P.E * 64, st);
    ra.trace = trace;
  }
  const size_t n_init = std::max<size_t>(std::max<size_t>(std::max<size_t>(P.E, ticks), L.cap), L.rcap);
  k_run_init<<<(unsigned)((n_init + 255) / 256), 256, 0, st>>>(ra);

  struct Host {
    int* poll = nullptr;       // pinned: 8 x {n_done, shutdown, error, pad}
    int* one = nullptr;
    cudaEvent_t ev[8], start, srv_done, rounds_done[kRoundStreams];
    cudaStream_t copy, rs[kRoundStreams];
  };
  static Host H;
  if (!H.poll) {
    cudaHostAlloc(&H.poll, 8 * 32, cudaHostAllocDefault);
    cudaHostAlloc(&H.one, 16, cudaHostAllocDefault);
    H.one[0] = 1;
    for (auto& ev : H.ev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&H.start, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&H.srv_done, cudaEventDisableTiming);
    int least, greatest;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    for (int k = 0; k < kRoundStreams; ++k) {
      cudaEventCreateWithFlags(&H.rounds_done[k], cudaEventDisableTiming);
      cudaStreamCreateWithPriority(&H.rs[k], cudaStreamNonBlocking, least);
    }
    cudaStreamCreateWithFlags(&H.copy, cudaStreamNonBlocking);
  }
  TickStreams& TS = tick_streams();
  cudaEventRecord(H.start, st);
  cudaStreamWaitEvent(TS.hi, H.start, 0);
  for (int k = 0; k < kRoundStreams; ++k) cudaStreamWaitEvent(H.rs[k], H.start, 0);
  // The server leaves some SMs without a search CTA, so round CTAs always have
  // somewhere to run whatever their register / shared-memory footprint (the
  // server's warps wait on the rounds' requests: they must never starve them).
  // two search warps per CTA: twice the concurrent searches of the latency shape
  // at nearly its per-expansion cost (the run is bound by each env's own chain)
  // Default server shape by round footprint (bench.py steady state, B200, round 2):
  //  * 32-thread lane-path rounds (A <= 32): 2 warps, 220 KB (cfg2: 0.29 ms/tick; 4 warps 0.32)
  //  * wider lane-path rounds (A <= 128): 4 warps, 200 KB -- three round CTAs fit beside
  //    the server (cfg3: 2.45 -> 1.90 ms/tick; 4 warps at 220 KB 2.52, 2 warps at 180 KB 2.53)
  //  * warp-path rounds (A >= 128, binned neighbours; cfg4 ~86 KB per round CTA): 4 warps and
  //    a pool small enough that one round CTA fits beside the server, 8 SMs left without a
  //    server -- at 220 KB the rounds had only the margin SMs (cfg4: 42.2 -> 24.2 ms/tick;
  //    pools of 80 / 120 / 139 KB within 3 %)
  //  An explicit run_server_warps (the re-sampling windows: 4, search-heavy catch-up) keeps
  //  220 KB and the 1/8 margin.
  int w_def = 2, kb_def = 0, margin_auto = 0;
  if (!P.run_server_warps) {
    if (sm > 16 * 1024) {   // large rounds (binned crowds)
      w_def = 4;
      kb_def = std::min(100, 227 - (int)((sm + 1023) / 1024) - 3);
      margin_auto = 8;
    } else if (NT >= 64) {
      w_def = 4;
      kb_def = 200;
    }
  }
  static const int srv_w_env = getenv("CW_RUN_SERVER_W") ? atoi(getenv("CW_RUN_SERVER_W")) : 0;
  const int srv_w = srv_w_env ? srv_w_env : (P.run_server_warps ? P.run_server_warps : w_def);
  static const int srv_kb_env = getenv("CW_RUN_SERVER_KB") ? atoi(getenv("CW_RUN_SERVER_KB")) : 0;
  const int srv_kb = srv_kb_env ? srv_kb_env : kb_def;
  AstarShape shp = astar_shape(P.nx, P.ny, srv_w == 4 ? kAstarWarps : srv_w == 2 ? 2 : 1, srv_kb);
  shp.NS = std::min(shp.NS, astar_ns_cap(P.nx, P.ny));   // the global store holds NS slot ids
  static const int margin = getenv("CW_RUN_MARGIN") ? atoi(getenv("CW_RUN_MARGIN")) : 0;
  // SMs left without a server CTA: 1/8 of them, except for 32-thread lane-path rounds
  // (A <= 32), which are light enough to run beside the server everywhere -- measured
  // at cfg2: margin 4 / 8 / 18 = 0.289 / 0.296 / 0.309 ms/tick; at cfg3 (64-thread
  // rounds) and cfg4 (256-thread warp-path rounds) a margin of 8 was 14 % / 2x slower
  const int margin_def = margin_auto ? margin_auto : (lanes_ok && NT == 32) ? 4 : P.astar_ctas / 8;
  int srv_ctas = P.astar_ctas - std::max(4, margin > 0 ? margin : margin_def);
  if (const char* v = getenv("CW_RUN_SERVER_CTAS")) srv_ctas = std::min(srv_ctas, atoi(v));
  srv_ctas = std::max(srv_ctas, 1);
  // the search server exits when the run goes quiet (runq.cuh ring_pop) and is
  // relaunched whenever requests are queued and no server launch is pending
  long long n_servers = 0;
  auto launch_server = [&]() {
    if (srv_w == 4)
      k_astar<kAstarWarps, true><<<srv_ctas, 32 * kAstarWarps, shp.smem, TS.hi>>>(P, S, shp.NC, shp.NS, ra, SpecArgs{});
    else if (srv_w == 2)
      k_astar<2, true><<<srv_ctas, 64, shp.smem, TS.hi>>>(P, S, shp.NC, shp.NS, ra, SpecArgs{});
    else
      k_astar<1, true><<<srv_ctas, 32, shp.smem, TS.hi>>>(P, S, shp.NC, shp.NS, ra, SpecArgs{});
    cudaEventRecord(H.srv_done, TS.hi);
    ++n_servers;
  };
  launch_server();
  int err = (int)cudaGetLastError();
  auto t_progress = std::chrono::steady_clock::now();
  int last_progress = -1;
  static const int n_rs = std::min(kRoundStreams, std::max(1, getenv("CW_RUN_STREAMS") ? atoi(getenv("CW_RUN_STREAMS")) : 4));
  static const int kInFlight = std::min(7, std::max(1, getenv("CW_RUN_INFLIGHT") ? atoi(getenv("CW_RUN_INFLIGHT")) : 6));
  static const bool debug = getenv("CW_RUN_DEBUG") != nullptr;
  int status = 0;
  long long n_rounds = 0;
  static const int rpm = getenv("CW_RUN_ROUND_CTAS_PER_SM") ? atoi(getenv("CW_RUN_ROUND_CTAS_PER_SM")) : 4;
  const int round_ctas = std::max(1, std::min(P.E, P.astar_ctas * rpm));
  for (long long i = 0;; ++i) {
    n_rounds = i + 1;
    cudaStream_t rs = H.rs[i % n_rs];
    if (lanes && bins.ncx > 0) k_round<NT, 2><<<round_ctas, NT, sm, rs>>>(P, S, rp, rv, rr, em, bins, ra);
    else if (lanes) k_round<NT, 1><<<round_ctas, NT, sm, rs>>>(P, S, rp, rv, rr, em, bins, ra);
    else k_round<NT, 0><<<round_ctas, NT, sm, rs>>>(P, S, rp, rv, rr, em, bins, ra);
    cudaMemcpyAsync(H.poll + (i & 7) * 8, ra.q, 32, cudaMemcpyDeviceToHost, rs);   // head..progress
    cudaEventRecord(H.ev[i & 7], rs);
    if (i >= kInFlight) {
      const long long j = i - kInFlight;
      cudaEventSynchronize(H.ev[j & 7]);
      const int* pv = H.poll + (j & 7) * 8 + 4;   // n_done, shutdown, error
      if (debug && (j % 2000 == 0 || pv[2])) {
        if (j == 0) fprintf(stderr, "server smem %zu NC %d NS %d ctas %d round smem %zu\n", shp.smem,
                            shp.NC, shp.NS, srv_ctas, sm);
        const unsigned long long* hq = reinterpret_cast<const unsigned long long*>(pv - 4);
        fprintf(stderr, "cw_crowd_run round %lld: head %llu tail %llu done %d/%d shutdown %d error %d\n",
                j, hq[0], hq[1], pv[0], P.E, pv[1], pv[2]);
      }
      if (pv[0] >= P.E) break;
      if (pv[2]) { status = 9001; break; }
      // searches queued and the last server launch has finished: start another
      const unsigned long long* hq = reinterpret_cast<const unsigned long long*>(pv - 4);
      if (hq[1] > hq[0] && cudaEventQuery(H.srv_done) == cudaSuccess) launch_server();
      // watchdog: a run may take long, but it must keep completing env-ticks
      const auto now = std::chrono::steady_clock::now();
      if (pv[3] != last_progress) {
        last_progress = pv[3];
        t_progress = now;
      }
      const double stalled = std::chrono::duration<double>(now - t_progress).count();
      if (stalled > 120.0 || (err = (int)cudaGetLastError()) != 0) { status = err ? err : 9002; break; }
    }
  }
  g_last_rounds = n_rounds;
  g_last_servers = n_servers;
  if (ra.trace) {
    cudaDeviceSynchronize();
    std::vector<long long> tr((size_t)P.E * 8);
    cudaMemcpy(tr.data(), ra.trace, tr.size() * 8, cudaMemcpyDeviceToHost);
    std::vector<int> order(P.E);
    for (int e = 0; e < P.E; ++e) order[e] = e;
    long long t_first = tr[kTrDone], t_last = tr[kTrDone];
    for (int e = 0; e < P.E; ++e) {
      t_first = std::min(t_first, tr[(size_t)e * 8 + kTrDone]);
      t_last = std::max(t_last, tr[(size_t)e * 8 + kTrDone]);
    }
    std::sort(order.begin(), order.end(),
              [&](int a, int b) { return tr[(size_t)a * 8 + kTrDone] > tr[(size_t)b * 8 + kTrDone]; });
    double sb = 0, ss = 0, sq = 0;
    for (int e = 0; e < P.E; ++e) {
      sb += tr[(size_t)e * 8 + kTrBusy];
      ss += tr[(size_t)e * 8 + kTrSearchWait];
      sq += tr[(size_t)e * 8 + kTrQueueWait];
    }
    fprintf(stderr, "cw_crowd_run trace: done spread %.2f ms; mean per env: busy %.2f ms, search wait %.2f ms, "
            "queue wait %.2f ms\n", (t_last - t_first) * 1e-6, sb / P.E * 1e-6, ss / P.E * 1e-6, sq / P.E * 1e-6);
    for (int k = 0; k < 6; ++k) {
      const long long* r = &tr[(size_t)order[k] * 8];
      fprintf(stderr, "  env %5d: busy %.2f ms, search wait %.2f ms (%lld waits), queue wait %.2f ms\n", order[k],
              r[kTrBusy] * 1e-6, r[kTrSearchWait] * 1e-6, r[kTrWaits], r[kTrQueueWait] * 1e-6);
    }
  }
  if (status) {   // end the server through the copy engine (no SM needed)
    cudaMemcpyAsync(&ra.q->shutdown, H.one, 4, cudaMemcpyHostToDevice, H.copy);
    cudaStreamSynchronize(H.copy);
  }
  for (int k = 1; k < kRoundStreams; ++k) {
    cudaEventRecord(H.rounds_done[k], H.rs[k]);
    cudaStreamWaitEvent(H.rs[0], H.rounds_done[k], 0);
  }
  cudaStreamWaitEvent(H.rs[0], H.srv_done, 0);
  if (flags & 2) k_run_finish<<<1, 256, 0, H.rs[0]>>>(S, ra);
  cudaEventRecord(H.rounds_done[0], H.rs[0]);
  cudaStreamWaitEvent(st, H.rounds_done[0], 0);
  if (status) return status;
  return (int)cudaGetLastError();
}

// The overlapped tick's two ORCA passes (pass 1 beside the searches; pass 2 after them,
// or early commit).  kLanes: 1 lane per agent, 2 the same with cell binning -- the same
// operations as the warp path (the run uses it; run == step is asserted bit for bit),
// 4.3x fewer instructions.
template <int NT, int kLanes>
static void launch_orca_passes(const cw_crowd_params& P, const cw_crowd_state& S, const double* rp,
                               const double* rv, double rr, const uint8_t* em, const Bins& bins, size_t sm,
                               cudaStream_t lo, cudaStream_t hi, bool ec, const SpecArgs& sa) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_orca<NT, kLanes>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(k_orca_ec<NT, kLanes>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    attr = true;
  }
  if (sm > 48 * 1024) {
    cudaFuncSetAttribute(k_orca<NT, kLanes>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_orca_ec<NT, kLanes>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  }
  k_orca<NT, kLanes><<<P.E, NT, sm, lo>>>(P, S, rp, rv, rr, em, bins, 1);
  if (ec) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P.E);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = hi;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_orca_ec<NT, kLanes>, P, S, rp, rv, rr, em, bins, sa);
  } else {
    k_orca<NT, kLanes><<<P.E, NT, sm, hi>>>(P, S, rp, rv, rr, em, bins, 2);
  }
}

template <int NT>
static int launch_step(const cw_crowd_params& P, const cw_crowd_state& S, const double* rp,
                       const double* rv, double rr, const uint8_t* em, int phases,
                       cudaStream_t st) {
  const Bins bins = make_bins(P);
  size_t sm = cw_crowd_step_smem_bytes(P.A, NT) + bins_smem_bytes(bins, P.A);
  if ((phases & 4) && sm > 48 * 1024)
    cudaFuncSetAttribute(k_orca<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  SpecCtx* X = (S.spec && S.env_epoch) ? static_cast<SpecCtx*>(S.spec) : nullptr;
  // the previous tick's dry guidance pass reads the state this tick rewrites
  if (X) cudaStreamWaitEvent(st, X->guided, 0);
  if (phases == 7) {
    // overlapped tick: envs without replans commit beside the A* searches.  An SM
    // runs one L1 / shared-memory split at a time, so k_orca asks for the same
    // max-shared carveout as k_astar to be co-resident with it.
    TickStreams& T = tick_streams();
    // a new prefetch batch every tick (its slot's previous batch, eight ticks back, is
    // waited for on the device: normally long done); the envs with replans commit as soon
    // as their own searches finish and predict their next tick at once (early commit)
    const int b = X ? X->next : 0;
    const bool batch = X != nullptr;
    static const bool no_ec = getenv("CW_PREFETCH_NO_EC") != nullptr;
    const bool ec = batch && !no_ec;
    SpecArgs sa{};
    if (batch) {
      X->next = (b + 1) % kSpecBatches;
      ++X->tag;
      ++X->batches;
      sa = spec_args(X, 2, S.env_epoch, b);
      sa.pend = X->pend;   // read by k_orca_ec (the batch's search kernel ignores it)
      cudaStreamWaitEvent(st, X->bdone[b], 0);
      cudaMemsetAsync(sa.qn, 0, 4 * sizeof(int), st);
    }
    k_guide<NT><<<P.E, NT, 0, st>>>(P, S, em, ec ? X->pend : nullptr, ec ? sa.qn + 2 : nullptr);
    cudaEventRecord(T.guided, st);
    cudaStreamWaitEvent(T.hi, T.guided, 0);
    cudaStreamWaitEvent(T.lo, T.guided, 0);
    SpecArgs look = X ? spec_args(X, 1, S.env_epoch, b) : SpecArgs{};
    if (ec) look.pend = X->pend;
    launch_astar(P, S, T.hi, look);
    static const bool warp_orca = getenv("CW_SYNC_WARP_ORCA") != nullptr;   // A/B
    if (!warp_orca && P.max_neighbors <= MAXK)
      (bins.ncx > 0 ? launch_orca_passes<NT, 2> : launch_orca_passes<NT, 1>)(P, S, rp, rv, rr, em, bins, sm,
                                                                             T.lo, T.hi, ec, sa);
    else
      launch_orca_passes<NT, 0>(P, S, rp, rv, rr, em, bins, sm, T.lo, T.hi, ec, sa);
    cudaEventRecord(T.hi_done, T.hi);
    cudaEventRecord(T.lo_done, T.lo);
    if (batch) {
      // the committed envs' next tick: dry guidance, then the batch's searches (polling
      // for the late committers' predictions), on a side stream the caller's does not join
      cudaStream_t ss = spec_stream(b);
      cudaStreamWaitEvent(ss, T.lo_done, 0);
      k_guide_dry<NT><<<P.E, NT, 0, ss>>>(P, S, sa);
      cudaEventRecord(X->guided, ss);
      const AstarShape A = astar_shape(P.nx, P.ny, kAstarWarps);
      const RunArgs none = {};
      static const double share = getenv("CW_SPEC_SHARE") ? atof(getenv("CW_SPEC_SHARE")) : 1.0;
      const int ctas = std::max(1, std::min(P.astar_ctas, (int)(P.astar_ctas * share)));
      k_astar<kAstarWarps, false><<<ctas, 32 * kAstarWarps, A.smem, ss>>>(P, S, A.NC, A.NS, none, sa);
      cudaEventRecord(X->bdone[b], ss);
    }
    cudaStreamWaitEvent(st, T.hi_done, 0);
    cudaStreamWaitEvent(st, T.lo_done, 0);
    return (int)cudaGetLastError();
  }
  if (phases & 1) k_guide<NT><<<P.E, NT, 0, st>>>(P, S, em);
  if (phases & 2) launch_astar(P, S, st);
  static const bool lanes_dbg = getenv("CW_ORCA_LANES") != nullptr;   // profiling the lane path
  if ((phases & 4) && lanes_dbg) {
    if (bins.ncx > 0) {
      if (sm > 48 * 1024) cudaFuncSetAttribute(k_orca<NT, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k_orca<NT, 2><<<P.E, NT, sm, st>>>(P, S, rp, rv, rr, em, bins, 0);
    } else {
      if (sm > 48 * 1024) cudaFuncSetAttribute(k_orca<NT, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k_orca<NT, 1><<<P.E, NT, sm, st>>>(P, S, rp, rv, rr, em, bins, 0);
    }
  } else if (phases & 4) {
    k_orca<NT><<<P.E, NT, sm, st>>>(P, S, rp, rv, rr, em, bins, 0);
  }
  return (int)cudaGetLastError();
}


// ---------------------------------------------------------------- ORCA building blocks
// The pieces of the tick as standalone batched calls, for the reference's
// module-level / private entry points (crowd/orca.py, field.py:229-566).  They
// run the same device functions as k_orca.
constexpr int kApiCap = 64;   // constraints per row accepted by cw_orca_lp

// _batched_lp (field.py:500-566): thread per row; the valid lanes of a row are
// compacted in lane order (the fallback's `begin` is then the compacted index,
// as searchsorted(lanes, fail) in the reference).
__global__ void k_orca_lp(int N, int L, const double* __restrict__ points, const double* __restrict__ normals,
                          const uint8_t* __restrict__ valid, const double* __restrict__ pref,
                          const double* __restrict__ max_speed, const uint8_t* __restrict__ lane_active,
                          double* __restrict__ out, int32_t* __restrict__ fell_back) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double cpx[kApiCap], cpy[kApiCap], cnx[kApiCap], cny[kApiCap];
  int nc = 0;
  if (!lane_active || lane_active[i]) {
    for (int l = 0; l < L; ++l) {
      if (!valid[(size_t)i * L + l]) continue;
      const size_t q = ((size_t)i * L + l) * 2;
      put_slot(cpx, nc, points[q]); put_slot(cpy, nc, points[q + 1]);
      put_slot(cnx, nc, normals[q]); put_slot(cny, nc, normals[q + 1]);
      ++nc;
    }
  }
  double v0, v1;
  const bool fb = lane_lp(cpx, cpy, cnx, cny, nc, pref[2 * i], pref[2 * i + 1], max_speed[i], v0, v1);
  out[2 * i] = v0;
  out[2 * i + 1] = v1;
  if (fell_back) fell_back[i] = fb ? 1 : 0;
}

// _vo_halfplane / orca_halfplane (field.py:448-495, orca.py:23-73): thread per row.
__global__ void k_orca_halfplanes(int n, const double* __restrict__ rel_pos, const double* __restrict__ rel_vel,
                                  const double* __restrict__ rr, const double* __restrict__ horizon, double dt,
                                  const double* __restrict__ v_self, const double* __restrict__ share,
                                  double* __restrict__ pt, double* __restrict__ nm) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  vo_halfplane(rel_pos[2 * i], rel_pos[2 * i + 1], rel_vel[2 * i], rel_vel[2 * i + 1], rr[i], horizon[i], dt,
               v_self[2 * i], v_self[2 * i + 1], share[i], pt[2 * i], pt[2 * i + 1], nm[2 * i], nm[2 * i + 1]);
}

// _preferred_velocities + _build_constraints (field.py:214-350) for envs [e0, e1),
// thread per agent, every lane in the reference layout: lanes [0, kmax) the stable
// top-K neighbours by (fp32 Gram key, index) (invalid: point 0, normal (1, 0)),
// lane kmax the robot (computed for every row, valid iff act and in range), lane
// kmax + use_robot the static obstacle (every row; obstacle point 0 where none).
// inr[row] = in-range neighbour count (the reference trims K to its maximum),
// gap[row] = nearest-neighbour gap or +inf (last_gap_by_env, field.py:268-271).
__global__ void k_crowd_constraints(cw_crowd_params P, cw_crowd_state S, int e0, int e1,
                                    const uint8_t* __restrict__ act, const double* __restrict__ robot_pos,
                                    const double* __restrict__ robot_vel, double robot_radius, int use_static,
                                    int Lmax, double* __restrict__ pref, double* __restrict__ points,
                                    double* __restrict__ normals, uint8_t* __restrict__ valid,
                                    int32_t* __restrict__ inr, double* __restrict__ gap) {
  const int A = P.A;
  const int row = blockIdx.x * blockDim.x + threadIdx.x;   // (e - e0) * A + a
  if (row >= (e1 - e0) * A) return;
  const int e = e0 + row / A, a = row % A;
  const size_t eA = (size_t)e * A, ia = eA + a;
  const uint8_t* ae = act + (size_t)(e - e0) * A;
  const bool me = ae[a] != 0;
  const double px = S.pos[ia * 2], py = S.pos[ia * 2 + 1];
  const double vxa = S.vel[ia * 2], vya = S.vel[ia * 2 + 1], ra = S.radius[ia];
  // preferred velocity (field.py:214-227); 0 for inactive rows
  {
    const double sp = S.pref_speed[ia];
    const double tw0 = S.waypoint[ia * 2] - px, tw1 = S.waypoint[ia * 2 + 1] - py;
    const double dist = sqrt(tw0 * tw0 + tw1 * tw1);
    const double safe = fmax(dist, kEps);
    double pf0 = tw0 / safe * sp, pf1 = tw1 / safe * sp;
    const double tg0 = S.goal[ia * 2] - px, tg1 = S.goal[ia * 2 + 1] - py;
    const double dg = sqrt(tg0 * tg0 + tg1 * tg1);
    const double scl = fmin(1.0, dg / fmax(sp * P.dt * 4, kEps));
    pref[(size_t)row * 2] = me ? pf0 * scl : 0.0;
    pref[(size_t)row * 2 + 1] = me ? pf1 * scl : 0.0;
  }
  const int kmax = min(P.max_neighbors, max(A - 1, 0));
  double* prow = points + (size_t)row * Lmax * 2;
  double* nrow = normals + (size_t)row * Lmax * 2;
  uint8_t* vrow = valid + (size_t)row * Lmax;
  for (int l = 0; l < Lmax; ++l) { prow[2 * l] = 0.0; prow[2 * l + 1] = 0.0; nrow[2 * l] = 1.0; nrow[2 * l + 1] = 0.0; vrow[l] = 0; }
  // neighbours: fp32 key (sq_i + sq_j) - 2 fma(y_i, y_j, x_i x_j), stable by index
  const float xi = (float)px, yi = (float)py;
  const float sqi = __fadd_rn(__fmul_rn(xi, xi), __fmul_rn(yi, yi));
  int cnt = 0, nb = 0;
  float lk = -CUDART_INF_F;
  int lj = -1;
  if (me) {
    for (int round = 0; round <= kmax; ++round) {
      float bk = CUDART_INF_F;
      int bj = -1;
      for (int j = 0; j < A; ++j) {
        if (j == a || !ae[j]) continue;
        const float xj = (float)S.pos[(eA + j) * 2], yj = (float)S.pos[(eA + j) * 2 + 1];
        const float sqj = __fadd_rn(__fmul_rn(xj, xj), __fmul_rn(yj, yj));
        const float dot = __fmaf_rn(yi, yj, __fmul_rn(xi, xj));
        const float key = __fsub_rn(__fadd_rn(sqi, sqj), __fmul_rn(2.0f, dot));
        if (!(key < P.nd2_f32)) continue;
        if (round == 0) ++cnt;
        const bool after = key > lk || (key == lk && j > lj);
        const bool better = bj < 0 || key < bk || (key == bk && j < bj);
        if (after && better) { bk = key; bj = j; }
      }
      if (bj < 0 || round == kmax) break;
      lk = bk;
      lj = bj;
      const size_t ij = eA + bj;
      const double rp0 = S.pos[ij * 2] - px, rp1 = S.pos[ij * 2 + 1] - py;
      const double rv0 = vxa - S.vel[ij * 2], rv1 = vya - S.vel[ij * 2 + 1];
      const double rr = ra + S.radius[ij] + P.safety_margin;
      vo_halfplane(rp0, rp1, rv0, rv1, rr, P.time_horizon, P.dt, vxa, vya, 0.5, prow[2 * nb], prow[2 * nb + 1],
                   nrow[2 * nb], nrow[2 * nb + 1]);
      vrow[nb] = 1;
      if (nb == 0) gap[row] = sqrt(rp0 * rp0 + rp1 * rp1) - (ra + S.radius[ij]);
      ++nb;
    }
  }
  if (nb == 0) gap[row] = CUDART_INF;
  inr[row] = cnt;
  int lane = kmax;
  if (robot_pos) {
    const double rpx = robot_pos[e * 2], rpy = robot_pos[e * 2 + 1];
    const double rvx = robot_vel ? robot_vel[e * 2] : 0.0, rvy = robot_vel ? robot_vel[e * 2 + 1] : 0.0;
    const double rp0 = rpx - px, rp1 = rpy - py;
    const double d2 = rp0 * rp0 + rp1 * rp1;
    const double rr = ra + robot_radius + P.safety_margin;
    vo_halfplane(rp0, rp1, vxa - rvx, vya - rvy, rr, P.obstacle_time_horizon, P.dt, vxa, vya, 1.0,
                 prow[2 * lane], prow[2 * lane + 1], nrow[2 * lane], nrow[2 * lane + 1]);
    vrow[lane] = me && d2 < P.nd2;
    ++lane;
  }
  if (use_static) {
    const int nx = P.nx, ny = P.ny;
    const size_t N = (size_t)nx * ny;
    const double res = P.res;
    double ox = 0.0, oy = 0.0;
    bool has = false;
    if (S.has_obs[e]) {
      const long long ri = clampll(trunc_ll(div_h(py, res)), 0, ny - 1);
      const long long ci = clampll(trunc_ll(div_h(px, res)), 0, nx - 1);
      const int flat = S.nearest[e * N + ri * nx + ci];
      has = flat >= 0;
      const int f = max(flat, 0);
      const int orow = f / nx, ocol = f - orow * nx;
      ox = ((double)ocol + 0.5) * res;
      oy = ((double)orow + 0.5) * res;
    }
    const double rp0 = ox - px, rp1 = oy - py;
    const double d2 = rp0 * rp0 + rp1 * rp1;
    const double margin = 0.5 * kSqrt2 * P.res0;
    const double rr = ra + margin + P.safety_margin;
    vo_halfplane(rp0, rp1, vxa, vya, rr, P.obstacle_time_horizon, P.dt, vxa, vya, 1.0, prow[2 * lane],
                 prow[2 * lane + 1], nrow[2 * lane], nrow[2 * lane + 1]);
    vrow[lane] = has && me && d2 < P.nd2;
  }
}
}  // namespace cw

extern "C" {

size_t cw_crowd_step_smem_bytes(int A, int nt) {
  // + fp32 (x, y, x^2 + y^2) per agent for the lane path (aliases the unused bins region)
  return (size_t)A * 7 * sizeof(double) + (size_t)(nt / 32) * 2 * sizeof(cw::WarpCons) +
         (size_t)((A + 15) & ~15) + 16 + (size_t)A * 3 * sizeof(float);
}

// Search warps per k_astar CTA (astar_rec / astar_heap hold one slot per warp).
int cw_astar_warps(void) { return cw::kAstarWarps; }

static int spec_nsm() {
  static int n = 0;
  if (!n) {
    int* d = nullptr;
    if (cudaMalloc(&d, sizeof(int)) != cudaSuccess) return 0;
    cw::k_nsmid<<<1, 1>>>(d);
    cudaMemcpy(&n, d, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(d);
  }
  return n;
}

size_t cw_spec_bytes(const cw_crowd_params* P) {
  size_t parts[7];
  const int nsm = spec_nsm();
  return nsm ? cw::spec_layout(*P, nsm, parts) : 0;
}

int cw_spec_create(const cw_crowd_params* P, void** handle) {
  using namespace cw;
  *handle = nullptr;
  const int nsm = spec_nsm();
  if (!nsm || P->E <= 0 || P->A <= 0) return (int)cudaErrorInvalidValue;
  size_t parts[7];
  const size_t total = spec_layout(*P, nsm, parts);
  unsigned char* base = nullptr;
  cudaError_t err = cudaMalloc(&base, total);
  if (err != cudaSuccess) return (int)err;
  SpecCtx* X = new SpecCtx();
  X->E = P->E; X->A = P->A; X->path_cap = P->path_cap; X->heap_cap = P->heap_cap;
  X->nx = P->nx; X->ny = P->ny; X->nsm = nsm;
  size_t o = 0;
  X->ent = reinterpret_cast<SpecEnt*>(base + o); o += parts[0];
  X->cells = reinterpret_cast<int32_t*>(base + o); o += parts[1];
  const size_t qb = parts[2] / kSpecBatches;
  for (int b = 0; b < kSpecBatches; ++b) X->q[b] = reinterpret_cast<AstarReq*>(base + o + b * qb);
  o += parts[2];
  X->qn = reinterpret_cast<int*>(base + o);
  X->stats = reinterpret_cast<unsigned long long*>(base + o + kSpecBatches * 4 * 4);
  o += parts[3];
  X->rec = base + o; o += parts[4];
  X->heap = reinterpret_cast<OpenEnt*>(base + o); o += parts[5];
  {
    const size_t qrb = ((size_t)P->E * P->A * 4 + 255) & ~(size_t)255;
    for (int b = 0; b < kSpecBatches; ++b) X->qr[b] = reinterpret_cast<int*>(base + o + b * qrb);
    X->pend = reinterpret_cast<int*>(base + o + kSpecBatches * qrb);
    cudaMemset(base + o, 0, parts[6]);
  }
  X->stride = astar_slot_stride(P->nx, P->ny);
  cudaMemset(X->ent, 0, parts[0]);
  cudaMemset(X->qn, 0, parts[3]);
  cudaEventCreateWithFlags(&X->guided, cudaEventDisableTiming);
  for (int b = 0; b < kSpecBatches; ++b) {
    spec_stream(b);
    cudaEventCreateWithFlags(&X->bdone[b], cudaEventDisableTiming);
  }
  err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    cudaFree(base);
    delete X;
    return (int)err;
  }
  *handle = X;
  return 0;
}

int cw_spec_destroy(void* handle) {
  using namespace cw;
  if (!handle) return 0;
  SpecCtx* X = static_cast<SpecCtx*>(handle);
  for (int b = 0; b < kSpecBatches; ++b) cudaStreamSynchronize(spec_stream(b));
  cudaFree(X->ent);   // the base of the one allocation
  cudaEventDestroy(X->guided);
  for (int b = 0; b < kSpecBatches; ++b) cudaEventDestroy(X->bdone[b]);
  delete X;
  return (int)cudaGetLastError();
}

// Predict and search, into context `handle`, the first-tick replans of freshly spawned
// rows (standby scenes; state S as a spawn leaves it: no paths) -- all on `stream`.
int cw_spec_predict(const cw_crowd_params* P, const cw_crowd_state* S, void* handle, const int32_t* rows,
                    int n_rows, int threads, void* stream) {
  using namespace cw;
  if (!handle || !S->env_epoch) return (int)cudaErrorInvalidValue;
  if (n_rows <= 0) return 0;
  SpecCtx* X = static_cast<SpecCtx*>(handle);
  cudaStream_t st = (cudaStream_t)stream;
  const int b = X->next;
  X->next = (b + 1) % kSpecBatches;
  ++X->tag;
  ++X->batches;
  const SpecArgs sa = spec_args(X, 2, S->env_epoch, b);
  cudaStreamWaitEvent(st, X->bdone[b], 0);
  cudaMemsetAsync(sa.qn, 0, 4 * sizeof(int), st);
  if (threads == 256) k_guide_dry<256><<<n_rows, 256, 0, st>>>(*P, *S, sa, rows);
  else if (threads == 64) k_guide_dry<64><<<n_rows, 64, 0, st>>>(*P, *S, sa, rows);
  else k_guide_dry<128><<<n_rows, 128, 0, st>>>(*P, *S, sa, rows);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_astar<kAstarWarps, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_astar<kAstarWarps, false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    attr = true;
  }
  const AstarShape A = astar_shape(P->nx, P->ny, kAstarWarps);
  const RunArgs none = {};
  // background work: a share of the SMs only, so the ticks' own searches always find some
  static const double share = getenv("CW_STANDBY_SHARE") ? atof(getenv("CW_STANDBY_SHARE")) : 0.5;
  const int ctas = std::max(1, std::min(P->astar_ctas, (int)(P->astar_ctas * share)));
  k_astar<kAstarWarps, false><<<ctas, 32 * kAstarWarps, A.smem, st>>>(*P, *S, A.NC, A.NS, none, sa);
  cudaEventRecord(X->bdone[b], st);
  return (int)cudaGetLastError();
}

// Copy context `src`'s finished predictions for `rows` into context `dst` (see
// k_spec_install); dst_epoch / src_epoch: the two contexts' grid generations (E).
int cw_spec_install(void* dst, void* src, const int32_t* dst_epoch, const int32_t* src_epoch, const int32_t* rows,
                    int n_rows, void* stream) {
  using namespace cw;
  if (!dst || !src) return (int)cudaErrorInvalidValue;
  if (n_rows <= 0) return 0;
  SpecCtx* D = static_cast<SpecCtx*>(dst);
  SpecCtx* Sx = static_cast<SpecCtx*>(src);
  if (D->E != Sx->E || D->A != Sx->A || D->path_cap != Sx->path_cap) return (int)cudaErrorInvalidValue;
  k_spec_install<<<n_rows, 256, 0, (cudaStream_t)stream>>>(D->A, D->path_cap, D->ent, D->cells, Sx->ent, Sx->cells,
                                                         dst_epoch, src_epoch, rows, ++D->tag);
  return (int)cudaGetLastError();
}

int cw_spec_stats(void* handle, long long* out) {
  using namespace cw;
  if (!handle) return (int)cudaErrorInvalidValue;
  SpecCtx* X = static_cast<SpecCtx*>(handle);
  unsigned long long v[4] = {0, 0, 0, 0};
  const cudaError_t err = cudaMemcpy(v, X->stats, sizeof(v), cudaMemcpyDeviceToHost);
  out[0] = X->batches;
  for (int k = 1; k < 4; ++k) out[k] = (long long)v[k];
  return (int)err;
}

// Scratch bytes of cw_crowd_run for E envs x A agents over `ticks` ticks.
size_t cw_crowd_run_scratch_bytes(int E, int A, int ticks) {
  return cw::run_layout(E, A, ticks).total;
}

// Round kernels launched by the last cw_crowd_run (host-only query).
long long cw_crowd_run_rounds(void) { return cw::g_last_rounds; }
// Search-server launches by the last cw_crowd_run (host-only query).
long long cw_crowd_run_servers(void) { return cw::g_last_servers; }

// `ticks` synchronous cw_crowd_step calls with the same inputs, run without a
// per-tick barrier (runq.cuh); same final state bit for bit.
int cw_crowd_run_window(const cw_crowd_params* P, const cw_crowd_state* S, const double* robot_pos,
                        const double* robot_vel, double robot_radius, const uint8_t* env_mask, int threads,
                        int ticks, const int32_t* start_tick, const int32_t* stop_tick, int flags,
                        void* scratch, void* stream) {
  using namespace cw;
  if (P->E <= 0 || P->A <= 0 || ticks <= 0) return 0;
  if (!scratch) return (int)cudaErrorInvalidValue;
  cudaStream_t st = (cudaStream_t)stream;
  if (S->spec && S->env_epoch)   // a dry guidance pass may still read the state
    cudaStreamWaitEvent(st, static_cast<SpecCtx*>(S->spec)->guided, 0);
  const double* rp = robot_pos;
  const double* rv = robot_vel;
  if (threads == 32)
    return launch_run<32>(*P, *S, rp, rv, robot_radius, env_mask, ticks, start_tick, stop_tick, flags, scratch, st);
  if (threads == 256)
    return launch_run<256>(*P, *S, rp, rv, robot_radius, env_mask, ticks, start_tick, stop_tick, flags, scratch, st);
  if (threads == 64)
    return launch_run<64>(*P, *S, rp, rv, robot_radius, env_mask, ticks, start_tick, stop_tick, flags, scratch, st);
  return launch_run<128>(*P, *S, rp, rv, robot_radius, env_mask, ticks, start_tick, stop_tick, flags, scratch, st);
}

int cw_crowd_run(const cw_crowd_params* P, const cw_crowd_state* S, const double* robot_pos,
                 const double* robot_vel, double robot_radius, const uint8_t* env_mask, int threads,
                 int ticks, void* scratch, void* stream) {
  return cw_crowd_run_window(P, S, robot_pos, robot_vel, robot_radius, env_mask, threads, ticks, nullptr,
                             nullptr, 3, scratch, stream);
}

// Bytes of A* scratch (astar_rec) per k_astar search warp for an nx x ny grid.
size_t cw_astar_slot_bytes(int nx, int ny) {
  return cw::astar_slot_stride(nx, ny);
}

// One two-phase tick of every env (field.py:90-163): k_guide -> k_astar -> k_orca,
// stream-ordered.  robot_pos/robot_vel (E,2) may be NULL; env_mask (E) may be NULL.
int cw_crowd_step_phases(const cw_crowd_params* P, const cw_crowd_state* S,
                         const double* robot_pos, const double* robot_vel, double robot_radius,
                         const uint8_t* env_mask, int threads, int phases, void* stream) {
  using namespace cw;
  if (P->E <= 0 || P->A <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  static int attr_set = 0;   // opt-in shared memory (<= 227 KB) for both k_astar shapes
  if (!attr_set) {
    cudaFuncSetAttribute(k_astar<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_astar<kAstarWarps, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    cudaFuncSetAttribute(k_astar<1, false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(k_astar<kAstarWarps, false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    attr_set = 1;
  }
  if (threads == 256)
    return launch_step<256>(*P, *S, robot_pos, robot_vel, robot_radius, env_mask, phases, st);
  if (threads == 64)
    return launch_step<64>(*P, *S, robot_pos, robot_vel, robot_radius, env_mask, phases, st);
  return launch_step<128>(*P, *S, robot_pos, robot_vel, robot_radius, env_mask, phases, st);
}

int cw_crowd_step(const cw_crowd_params* P, const cw_crowd_state* S, const double* robot_pos,
                  const double* robot_vel, double robot_radius, const uint8_t* env_mask,
                  int threads, void* stream) {
  return cw_crowd_step_phases(P, S, robot_pos, robot_vel, robot_radius, env_mask, threads, 7,
                              stream);
}

// PCG64 stream states from integer seeds (numpy PCG64(seed) via SeedSequence).
int cw_seed_streams(int n, const uint64_t* seeds, void* out, void* stream) {
  if (n <= 0) return 0;
  cw::k_seed_streams<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(n, seeds,
                                                                       (cw::Pcg64Raw*)out);
  return (int)cudaGetLastError();
}

// child_seed(parent[i], label[, k[i]]) for label ids 0 "env", 1 "crowd-run", 2 "crowd", 3 "resample"
int cw_child_seeds(int n, const uint64_t* parent, int label_id, const uint64_t* k, uint64_t* out,
                   void* stream) {
  if (n <= 0) return 0;
  cw::k_child_seeds<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(n, parent, label_id, k, out);
  return (int)cudaGetLastError();
}


// ---------------------------------------------------------------- ORCA building blocks
int cw_orca_lp(int N, int L, const double* points, const double* normals, const uint8_t* valid,
               const double* pref, const double* max_speed, const uint8_t* lane_active, double* out,
               int32_t* fell_back, void* stream) {
  if (N <= 0) return 0;
  if (L < 0 || L > cw::kApiCap) return (int)cudaErrorInvalidValue;
  cw::k_orca_lp<<<(N + 127) / 128, 128, 0, (cudaStream_t)stream>>>(N, L, points, normals, valid, pref, max_speed,
                                                                   lane_active, out, fell_back);
  return (int)cudaGetLastError();
}

int cw_orca_halfplanes(int n, const double* rel_pos, const double* rel_vel, const double* combined_radius,
                       const double* horizon, double dt, const double* v_self, const double* share,
                       double* point, double* normal, void* stream) {
  if (n <= 0) return 0;
  cw::k_orca_halfplanes<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(n, rel_pos, rel_vel, combined_radius,
                                                                           horizon, dt, v_self, share, point,
                                                                           normal);
  return (int)cudaGetLastError();
}

int cw_crowd_constraints(const cw_crowd_params* P, const cw_crowd_state* S, int e0, int e1, const uint8_t* act,
                         const double* robot_pos, const double* robot_vel, double robot_radius, int use_static,
                         int lmax, double* pref, double* points, double* normals, uint8_t* valid, int32_t* inr,
                         double* gap, void* stream) {
  const int rows = (e1 - e0) * P->A;
  if (rows <= 0) return 0;
  cw::k_crowd_constraints<<<(rows + 127) / 128, 128, 0, (cudaStream_t)stream>>>(
      *P, *S, e0, e1, act, robot_pos, robot_vel, robot_radius, use_static, lmax, pref, points, normals, valid,
      inr, gap);
  return (int)cudaGetLastError();
}

// ABI self-check for the ctypes mirror (host-only; no device work).
int cw_abi_sizes(size_t* out, int n) {
  const size_t v[6] = {sizeof(cw_scene_params), sizeof(cw_scene_buffers), sizeof(cw_crowd_params),
                       sizeof(cw_crowd_state), sizeof(cw_robot_params), sizeof(cw_robot_state)};
  for (int i = 0; i < n && i < 6; ++i) out[i] = v[i];
  return 6;
}

}  // extern "C"
