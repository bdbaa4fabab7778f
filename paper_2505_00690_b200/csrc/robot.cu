// Robot step, traversability gating, reward and observations on B200
// (reference envcore/batch.py:205-302, robot.py:94-179,
// observe.py:39-129, bench/reward.py:29-53).
//
//   k_trav_cols / k_trav_rows / k_trav_cells   traversability_maps: the 5x5 box
//       mean is a float64 cumulative sum over the edge-padded grid, first down
//       the columns then along the rows (np.cumsum axis=0 then axis=1); each
//       column / row is one thread's sequential sum, so every partial sum
//       rounds exactly as in numpy.  Step rise, grade (central differences of
//       the box surface, glibc hypot) and roughness follow per cell.
//   k_robot_step   warp per env: integrate_motion, gating against the passable
//       map, crowd contact (lanes over agents), elevation / walkable lookup,
//       reward_batch, termination and truncation.
//   k_observe      CTA per env, thread per ray: float32 march in res steps to
//       10 m (obstacle or a rise above max_step_rise stops a ray, leaving the
//       grid ends it at the cap), the 16 x 10 ego height patch, goal vector and
//       projected velocity; with include_semantics the label of the cell each
//       ray stopped in (observe.py:84-85).
//
// Compiled with -fmad=false: float64 / float32 expressions round once per op
// like numpy.  sin / cos / atan2 / tan / tanh come from CUDA's libdevice
// (within 1-2 ulp of the host libm / numpy SIMD kernels the reference calls);
// tests/test_gpu_robot.py states the resulting tolerances.
#include <math_constants.h>
#include "common.cuh"
#include "citywalk_b200.h"

namespace cw {

constexpr int kRays = 128;
constexpr double kFan = 0.7853981633974483;      // np.pi / 4.0
constexpr double kCap = 10.0;
constexpr int kHX = 16, kHY = 10;
constexpr double kHL = 1.6, kHW = 1.0;

CW_DEV int env_row(const int32_t* slots, int e) { return slots ? slots[e] : e; }

// ---------------------------------------------------------------- traversability
// cum: (chunk, ny + 5, nx + 5) float64; row 0 / column 0 are the zero pad of
// np.pad(csum, ((1, 0), (1, 0))); entry (i + 1, j + 1) = csum[i][j].
__global__ void k_trav_cols(cw_robot_params P, int e0, int n, const int32_t* slots,
                            const float* __restrict__ elev, double* cum) {
  const int k = blockIdx.y;
  if (k >= n) return;
  const int nx = P.nx, ny = P.ny, W = nx + 5;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;   // padded column
  if (j > nx + 3) return;
  const float* el = elev + (size_t)env_row(slots, e0 + k) * nx * ny;
  double* C = cum + (size_t)k * (ny + 5) * W;
  const int c = min(max(j - 2, 0), nx - 1);              // np.pad mode="edge"
  double run = 0.0;
  if (j == 0) for (int i = 0; i < ny + 5; ++i) C[(size_t)i * W] = 0.0;
  C[j + 1] = 0.0;
  for (int i = 0; i < ny + 4; ++i) {
    const int r = min(max(i - 2, 0), ny - 1);
    run = run + (double)el[(size_t)r * nx + c];
    C[(size_t)(i + 1) * W + j + 1] = run;
  }
}

__global__ void k_trav_rows(cw_robot_params P, int n, double* cum) {
  const int k = blockIdx.y;
  if (k >= n) return;
  const int nx = P.nx, ny = P.ny, W = nx + 5;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;   // padded row
  if (i > ny + 3) return;
  double* row = cum + (size_t)k * (ny + 5) * W + (size_t)(i + 1) * W;
  double run = 0.0;
  for (int j = 1; j <= nx + 4; ++j) {
    run = run + row[j];
    row[j] = run;
  }
}

CW_DEV double box_at(const double* C, int W, int r, int c) {
  // (cum[5:, 5:] - cum[:-5, 5:] - cum[5:, :-5] + cum[:-5, :-5]) / 25
  return (((C[(size_t)(r + 5) * W + c + 5] - C[(size_t)r * W + c + 5]) - C[(size_t)(r + 5) * W + c]) +
          C[(size_t)r * W + c]) / 25.0;
}

__global__ void k_trav_cells(cw_robot_params P, int e0, int n, const int32_t* slots,
                             const uint8_t* __restrict__ labels, const float* __restrict__ elev,
                             const double* __restrict__ cum, uint8_t* passable) {
  const int k = blockIdx.y;
  if (k >= n) return;
  const int nx = P.nx, ny = P.ny, W = nx + 5;
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nx * ny) return;
  const int row = env_row(slots, e0 + k);
  const size_t base = (size_t)row * nx * ny;
  const float* el = elev + base;
  const double* C = cum + (size_t)k * (ny + 5) * W;
  const int r = f / nx, c = f - r * nx;
  const double e = (double)el[f];
  double step = 0.0;   // np.fmax over the existing 4-neighbours
  if (r + 1 < ny) step = fmax(step, fabs(e - (double)el[f + nx]));
  if (r - 1 >= 0) step = fmax(step, fabs(e - (double)el[f - nx]));
  if (c + 1 < nx) step = fmax(step, fabs(e - (double)el[f + 1]));
  if (c - 1 >= 0) step = fmax(step, fabs(e - (double)el[f - 1]));
  const double box = box_at(C, W, r, c);
  const double rough = fabs(e - box);
  const double two_res = 2.0 * P.res;
  const double gx = (c >= 1 && c + 1 < nx) ? (box_at(C, W, r, c + 1) - box_at(C, W, r, c - 1)) / two_res : 0.0;
  const double gy = (r >= 1 && r + 1 < ny) ? (box_at(C, W, r + 1, c) - box_at(C, W, r - 1, c)) / two_res : 0.0;
  const double grade = glibc_hypot(gx, gy);
  const bool blocked = labels[base + f] == L_OBSTACLE || step > P.model.max_step_rise ||
                       grade > P.model.max_grade || rough > P.model.max_roughness;
  passable[base + f] = blocked ? 0 : 1;
}

// ---------------------------------------------------------------- robot step
// robot.py:94-124 for one env.
CW_DEV void integrate_motion(const cw_robot_model& m, double x, double y, double yaw, double a0,
                             double a1, double dt, double& nx, double& ny, double& nyaw,
                             double& vx, double& vy) {
  if (m.holonomic) {
    const double ex = a0 * m.max_speed, ey = a1 * m.max_speed;
    double s, c;
    cr_sincos(yaw, &s, &c);
    vx = c * ex - s * ey;
    vy = s * ex + c * ey;
    nx = x + vx * dt;
    ny = y + vy * dt;
    const double speed = glibc_hypot(vx, vy);
    const double target = speed > 1e-9 ? atan2(vy, vx) : yaw;
    double ds, dc;
    cr_sincos(target - yaw, &ds, &dc);
    double dyaw = atan2(ds, dc);
    const double lim = kTwoPi * dt;
    dyaw = fmin(fmax(dyaw, -lim), lim);
    nyaw = yaw + dyaw;
    return;
  }
  const double v = a0 * m.max_speed;
  const double steer = a1 * m.max_steer;
  const double yaw_rate = v * tan(steer) / m.wheelbase;
  nyaw = yaw + yaw_rate * dt;
  double s, c;
  cr_sincos(yaw, &s, &c);
  vx = v * c;
  vy = v * s;
  nx = x + vx * dt;
  ny = y + vy * dt;
}

// warp per env; batch.py:223-288
__global__ void __launch_bounds__(128) k_robot_step(cw_robot_params P, cw_robot_state S,
                                                    const double* __restrict__ actions) {
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (e >= P.E) return;
  const int gnx = P.nx, gny = P.ny;
  const size_t N = (size_t)gnx * gny;
  const double res = P.res, dt = P.dt;
  const bool live = !S.terminated[e] && !S.truncated[e];
  const double a0 = fmin(fmax(actions[e * 2], -1.0), 1.0);
  const double a1 = fmin(fmax(actions[e * 2 + 1], -1.0), 1.0);
  const double x = S.x[e], y = S.y[e], yaw = S.yaw[e];
  double nx, ny, nyaw, nvx, nvy;
  integrate_motion(P.model, x, y, yaw, a0, a1, dt, nx, ny, nyaw, nvx, nvy);
  const double w_m = gnx * res, l_m = gny * res;
  const bool inside = nx >= 0 && nx < w_m && ny >= 0 && ny < l_m;
  const long long rr = clampll(trunc_ll(ny / res), 0, gny - 1);
  const long long cc = clampll(trunc_ll(nx / res), 0, gnx - 1);
  const size_t cell = (size_t)e * N + rr * gnx + cc;
  bool blocked = inside && !S.passable[cell];
  const bool coll_static = blocked && S.labels[cell] == L_OBSTACLE;
  // crowd contact (batch.py:243-251): d2 = ((pos - cand) ** 2).sum(-1) < (r + R) ** 2
  bool hit = false;
  if (S.crowd_pos && P.A > 0) {
    for (int j = lane; j < P.A; j += 32) {
      const size_t ia = (size_t)e * P.A + j;
      const double dx = S.crowd_pos[ia * 2] - nx, dy = S.crowd_pos[ia * 2 + 1] - ny;
      const double d2 = dx * dx + dy * dy;
      const double rs = S.crowd_radius[ia] + P.model.body_radius;
      hit |= d2 < rs * rs && S.crowd_active[ia];
    }
    hit = __any_sync(0xffffffffu, hit);
    blocked = blocked || hit;
  }
  if (lane != 0) return;
  const bool coll = coll_static || hit;
  const bool move = live && inside && !blocked;
  const bool frozen = live && blocked;
  const bool go = move || (live && !inside);
  const double X = go ? nx : x, Y = go ? ny : y;
  double vx = move ? nvx : (frozen ? 0.0 : S.vx[e]);
  double vy = move ? nvy : (frozen ? 0.0 : S.vy[e]);
  vx = live ? vx : 0.0;
  vy = live ? vy : 0.0;
  S.x[e] = X;
  S.y[e] = Y;
  S.yaw[e] = live ? nyaw : yaw;
  S.vx[e] = vx;
  S.vy[e] = vy;
  const long long r2 = clampll(trunc_ll(Y / res), 0, gny - 1);
  const long long c2 = clampll(trunc_ll(X / res), 0, gnx - 1);
  const bool in_now = X >= 0 && X < w_m && Y >= 0 && Y < l_m;
  const size_t cell2 = (size_t)e * N + r2 * gnx + c2;
  if (in_now) S.elev[e] = (double)S.grid_elev[cell2];
  const bool on_walk = in_now && S.labels[cell2] == L_WALKABLE;
  const double dist = glibc_hypot(S.goal[e * 2] - X, S.goal[e * 2 + 1] - Y);
  const double pinc = live ? glibc_hypot(vx * dt, vy * dt) : 0.0;
  const bool reached = live && dist <= P.reach_threshold;
  const bool oob = live && !in_now;
  // bench/reward.py:29-53
  const double track = (1.0 - tanh(dist / P.track_far)) +
                       P.track_near_weight * (1.0 - tanh(dist / P.track_near));
  const double term = (reached ? P.terminal_reach : 0.0) + (oob ? P.terminal_oob : 0.0);
  const bool off_walk = live && !on_walk;
  const bool colliding = live && coll;
  const double total = ((term + P.c1 * track) + P.c2 * (off_walk ? -1.0 : 0.0)) +
                       P.c3 * (colliding ? -1.0 : 0.0);
  S.reward[e] = live ? total : 0.0;
  const long long tick = live ? S.tick[e] + 1 : S.tick[e];
  S.tick[e] = tick;
  S.terminated[e] = S.terminated[e] || reached || oob;
  S.truncated[e] = S.truncated[e] || (live && tick >= P.horizon && !oob);
  uint8_t* ev = S.events + (size_t)e * 6;
  ev[0] = live && coll;
  ev[1] = live && coll_static;
  ev[2] = live && hit;
  ev[3] = on_walk;
  ev[4] = reached;
  ev[5] = oob;
  S.distance[e] = dist;
  S.path_inc[e] = pinc;
}

// ---------------------------------------------------------------- observations
// CTA per env, thread per ray; observe.py:39-129
__global__ void __launch_bounds__(kRays) k_observe(cw_robot_params P, cw_robot_state S) {
  const int e = blockIdx.x;
  const int k = threadIdx.x;
  const int gnx = P.nx, gny = P.ny;
  const size_t N = (size_t)gnx * gny;
  const double res = P.res;
  const uint8_t* lab = S.labels + (size_t)e * N;
  const float* el = S.grid_elev + (size_t)e * N;
  const double x = S.x[e], y = S.y[e], yaw = S.yaw[e], er = S.elev[e];
  // np.linspace(-pi/4, pi/4, 128) then (yaw + offset).astype(float32)
  const double step_o = (2.0 * kFan) / (double)(kRays - 1);
  const double off = k == kRays - 1 ? kFan : (double)k * step_o + (-kFan);
  const float ang = (float)(yaw + off);
  float dx, dy;
  sincosf(ang, &dy, &dx);
  const float ox = (float)x, oy = (float)y;
  const float inv = (float)(1.0 / res);
  const float lim = (float)P.model.max_step_rise;
  float prev = (float)er;
  float depth = (float)kCap;
  uint8_t sem = 0;   // observe.py:49, 84-85
  const int n_steps = (int)(kCap / res);
  for (int s = 1; s <= n_steps; ++s) {
    const float t = (float)(s * res);
    const float px = __fadd_rn(ox, __fmul_rn(dx, t));
    const float py = __fadd_rn(oy, __fmul_rn(dy, t));
    const long long cc = (long long)__fmul_rn(px, inv);
    const long long rr = (long long)__fmul_rn(py, inv);
    if (!(cc >= 0 && cc < gnx && rr >= 0 && rr < gny)) break;   // left the grid: cap
    const size_t f = (size_t)rr * gnx + cc;
    const float ev = el[f];
    const uint8_t lf = lab[f];
    if (lf == L_OBSTACLE || __fsub_rn(ev, prev) > lim) { depth = t; sem = lf; break; }
    prev = ev;
  }
  S.depth[(size_t)e * kRays + k] = depth;
  if (S.semantics) S.semantics[(size_t)e * kRays + k] = sem;
  // ego-aligned height patch (observe.py:112-121), 160 samples over the CTA
  double s, c;
  cr_sincos(yaw, &s, &c);
  for (int q = k; q < kHX * kHY; q += kRays) {
    const int i = q / kHY, j = q - i * kHY;
    const double hx = ((double)i + 0.5) / kHX * kHL;
    const double hy = ((double)j + 0.5) / kHY * kHW - kHW / 2.0;
    const double wx = (x + c * hx) - s * hy;
    const double wy = (y + s * hx) + c * hy;
    const long long hc = clampll(trunc_ll(wx / res), 0, gnx - 1);
    const long long hr = clampll(trunc_ll(wy / res), 0, gny - 1);
    const bool hin = wx >= 0 && wx < gnx * res && wy >= 0 && wy < gny * res;
    const double hm = hin ? (double)el[hr * gnx + hc] - er : 0.0;
    S.height_map[(size_t)e * kHX * kHY + q] = (float)hm;
  }
  if (k == 0) {
    const double gvx = S.goal[e * 2] - x, gvy = S.goal[e * 2 + 1] - y;
    S.goal_vector[e * 2] = c * gvx + s * gvy;
    S.goal_vector[e * 2 + 1] = -s * gvx + c * gvy;
    const double gn = glibc_hypot(gvx, gvy);
    S.proj_vel[e] = (S.vx[e] * gvx + S.vy[e] * gvy) / fmax(gn, 1e-12);
  }
}

}  // namespace cw

extern "C" {

size_t cw_traversability_scratch_bytes(int nx, int ny, int chunk) {
  return (size_t)chunk * (ny + 5) * (nx + 5) * sizeof(double);
}

int cw_traversability(const cw_robot_params* P, int E, const int32_t* slots, const uint8_t* labels,
                      const float* grid_elev, uint8_t* passable, void* scratch, int chunk,
                      void* stream) {
  using namespace cw;
  if (E <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  double* cum = (double*)scratch;
  const int nx = P->nx, ny = P->ny;
  for (int e0 = 0; e0 < E; e0 += chunk) {
    const int n = min(chunk, E - e0);
    k_trav_cols<<<dim3((nx + 4 + 127) / 128, n), 128, 0, st>>>(*P, e0, n, slots, grid_elev, cum);
    k_trav_rows<<<dim3((ny + 4 + 127) / 128, n), 128, 0, st>>>(*P, n, cum);
    k_trav_cells<<<dim3((nx * ny + 255) / 256, n), 256, 0, st>>>(*P, e0, n, slots, labels, grid_elev,
                                                                cum, passable);
  }
  return (int)cudaGetLastError();
}

int cw_robot_step(const cw_robot_params* P, const cw_robot_state* S, const double* actions,
                  void* stream) {
  using namespace cw;
  if (P->E <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  k_robot_step<<<(P->E + 3) / 4, 128, 0, st>>>(*P, *S, actions);
  k_observe<<<P->E, kRays, 0, st>>>(*P, *S);
  return (int)cudaGetLastError();
}

int cw_robot_observe(const cw_robot_params* P, const cw_robot_state* S, void* stream) {
  using namespace cw;
  if (P->E <= 0) return 0;
  k_observe<<<P->E, kRays, 0, (cudaStream_t)stream>>>(*P, *S);
  return (int)cudaGetLastError();
}

}  // extern "C"
