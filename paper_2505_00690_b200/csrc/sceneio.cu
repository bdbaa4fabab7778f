// Scene identity / wire format on the device.
//
// scene_to_dict (urbangen/scene.py:163-178) run-length codes two grids with
// jsonio.rle_encode (jsonio.py:42-54): the zone map (ny, nx) u8 and the terrain
// assignment (trows, tcols) int32, as [value, run, value, run, ...] over the
// row-major flattening.  This file produces those pair lists for a batch of
// envs straight from the sampled rows in HBM, so the host only serialises the
// compact lists (sceneio.py) instead of copying and scanning whole grids.
//
// One CTA per (env, grid).  A cell p opens a run iff p == 0 or v[p] != v[p-1]
// and closes one iff p == n-1 or v[p] != v[p+1]; run k opens at the k-th
// opening cell and closes at the k-th closing cell.  Each chunk of
// NT * kItems cells is scanned once with a packed (opens | closes << 16)
// block scan: an opening cell writes (value, p) to pair k, a closing cell
// later rewrites the second word to p + 1 - start (opens and closes are
// counted separately across chunks: a run may span chunks).  Both counts within a
// chunk stay below 2^16, so the packed scan cannot carry across halves.
// HBM-bound: one read of each grid per pass (count pass + fill pass).

#include <cstdint>

#include "common.cuh"
#include "citywalk_b200.h"

namespace {

constexpr int kRleThreads = 256;
constexpr int kItems = 4;

CW_DEV uint32_t block_excl_scan(uint32_t v, uint32_t* warp_tot, uint32_t& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < kRleThreads / 32 ? warp_tot[lane] : 0u;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += y;
    }
    if (lane < kRleThreads / 32) warp_tot[lane] = w;
  }
  __syncthreads();
  total = warp_tot[kRleThreads / 32 - 1];
  uint32_t before = wid ? warp_tot[wid - 1] : 0u;
  __syncthreads();  // warp_tot is reused by the next chunk
  return before + x - v;
}

// count (pairs == nullptr): runs[e] = number of runs; fill: pairs + offs[e].
template <typename T>
__global__ void __launch_bounds__(kRleThreads) k_rle(const T* __restrict__ grid, size_t stride, int n,
                                                     const int32_t* __restrict__ rows,
                                                     int32_t* __restrict__ runs, int runs_stride,
                                                     const int64_t* __restrict__ offs,
                                                     int32_t* __restrict__ pairs) {
  __shared__ uint32_t warp_tot[kRleThreads / 32];
  const int e = blockIdx.x;
  const int row = rows ? rows[e] : e;
  const T* v = grid + (size_t)row * stride;
  int32_t* out = pairs ? pairs + offs[(size_t)e * runs_stride] : nullptr;
  uint32_t base = 0, base_c = 0;  // runs opened / closed before this chunk
  for (int c0 = 0; c0 < n; c0 += kRleThreads * kItems) {
    const int p0 = c0 + threadIdx.x * kItems;
    T val[kItems + 2];
#pragma unroll
    for (int i = 0; i < kItems + 2; ++i) {
      int p = p0 - 1 + i;
      val[i] = (p >= 0 && p < n) ? v[p] : T(0);
    }
    uint32_t opens = 0, closes = 0, packed = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      int p = p0 + i;
      if (p >= n) break;
      bool o = p == 0 || val[i + 1] != val[i];
      bool c = p == n - 1 || val[i + 1] != val[i + 2];
      opens |= (uint32_t)o << i;
      closes |= (uint32_t)c << i;
    }
    packed = (uint32_t)__popc(opens) | ((uint32_t)__popc(closes) << 16);
    uint32_t total;
    uint32_t ex = block_excl_scan(packed, warp_tot, total);
    if (out) {
      uint32_t k = base + (ex & 0xffffu);
#pragma unroll
      for (int i = 0; i < kItems; ++i)
        if ((opens >> i) & 1) {
          out[2 * k] = (int32_t)val[i + 1];
          out[2 * k + 1] = p0 + i;
          ++k;
        }
      __syncthreads();
      k = base_c + (ex >> 16);
#pragma unroll
      for (int i = 0; i < kItems; ++i)
        if ((closes >> i) & 1) {
          out[2 * k + 1] = p0 + i + 1 - out[2 * k + 1];
          ++k;
        }
    }
    base += total & 0xffffu;
    base_c += total >> 16;
  }
  if (!out && threadIdx.x == 0) runs[(size_t)e * runs_stride] = (int32_t)base;
}

}  // namespace

extern "C" {

int cw_scene_rle(const cw_scene_params* P, int E, const int32_t* rows, const cw_scene_buffers* B,
                 int32_t* runs, const int64_t* offsets, int32_t* pairs, void* stream) {
  if (!P || !B || !runs || E < 0 || (offsets == nullptr) != (pairs == nullptr))
    return (int)cudaErrorInvalidValue;
  if (E == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int N = P->nx * P->ny, NT = P->trows * P->tcols;
  k_rle<uint8_t><<<E, kRleThreads, 0, st>>>(B->zones, (size_t)N, N, rows, runs, 2, offsets, pairs);
  k_rle<int32_t><<<E, kRleThreads, 0, st>>>(B->assign, (size_t)NT, NT, rows, runs + 1, 2,
                                            offsets ? offsets + 1 : nullptr, pairs);
  return (int)cudaGetLastError();
}

}  // extern "C"
