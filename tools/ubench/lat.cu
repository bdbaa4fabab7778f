// Dependent-chain latency of a few primitives on one warp (cycles per op).
#include <cstdio>
#include <cstdint>
__global__ void k(long long* out, const double* gd, double* sink, int iters) {
  __shared__ double sd[1024];
  __shared__ unsigned long long su[1024];
  int lane = threadIdx.x;
  for (int i = lane; i < 1024; i += 32) { sd[i] = gd[i]; su[i] = (unsigned long long)(i * 7 % 1024); }
  __syncwarp();
  long long t0, t1;
  // 1 SHFL.IDX chain (32-bit)
  unsigned v = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_sync(0xffffffffu, v, (v + 1) & 31);
  t1 = clock64(); if (lane == 0) out[0] = (t1 - t0);
  // 2 VOTE.ballot -> popc chain
  unsigned b = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) b = __popc(__ballot_sync(0xffffffffu, (b & 1) ^ (lane & 1)));
  t1 = clock64(); if (lane == 0) out[1] = (t1 - t0);
  // 3 DADD chain
  double d = gd[lane];
  t0 = clock64();
  for (int i = 0; i < iters; ++i) d = d + 1.0000001;
  t1 = clock64(); if (lane == 0) out[2] = (t1 - t0);
  // 4 I2F.F64 + DMUL chain
  int iv = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { double x = (double)iv * 1.5; iv = (int)x & 1023; }
  t1 = clock64(); if (lane == 0) out[3] = (t1 - t0);
  // 5 LDS.64 pointer chase
  unsigned long long p = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) p = su[p];
  t1 = clock64(); if (lane == 0) out[4] = (t1 - t0);
  // 6 LDG L1-hit pointer chase (global array of 1024 u64 indices, warmed)
  const unsigned long long* gu = reinterpret_cast<const unsigned long long*>(gd + 1024);
  unsigned long long q = lane;
  for (int i = 0; i < 2048; ++i) q = gu[q];
  t0 = clock64();
  for (int i = 0; i < iters; ++i) q = gu[q];
  t1 = clock64(); if (lane == 0) out[5] = (t1 - t0);
  // 7 IADD chain (integer)
  unsigned a = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) a = a * 3u + 1u;
  t1 = clock64(); if (lane == 0) out[6] = (t1 - t0);
  // 8 u128 compare + select chain
  unsigned long long kf = lane, kk = lane * 3;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    unsigned __int128 A = ((unsigned __int128)kf << 64) | kk, B = ((unsigned __int128)kk << 64) | kf;
    bool lt = A < B; kf = lt ? kk + 1 : kf + 2; kk = lt ? kf : kk + 1;
  }
  t1 = clock64(); if (lane == 0) out[7] = (t1 - t0);
  // 9 SHFL 64-bit (2x SHFL) chain
  unsigned long long w = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) w = __shfl_sync(0xffffffffu, w, (int)(w + 1) & 31);
  t1 = clock64(); if (lane == 0) out[8] = (t1 - t0);
  // 10 L2-hit LDG pointer chase over a 64 MB region (stride > L1)
  const unsigned* big = reinterpret_cast<const unsigned*>(gd + 4096);
  unsigned z = lane * 4099;
  t0 = clock64();
  for (int i = 0; i < iters / 8; ++i) z = __ldcg(big + (z & ((16u << 20) - 1)));
  t1 = clock64(); if (lane == 0) out[9] = (t1 - t0) * 8;
  sink[lane] = (double)(v + b + iv + p + q + a + kf + kk + w + z) + d;
}
int main() {
  const size_t big = (size_t)(4096 + (16u << 20) / 2 + 16) * 8;
  double* gd; cudaMalloc(&gd, big);
  double h[4096 + 8];
  for (int i = 0; i < 1024; ++i) h[i] = i;
  unsigned long long* hu = reinterpret_cast<unsigned long long*>(h + 1024);
  for (int i = 0; i < 1024; ++i) hu[i] = (unsigned long long)((i * 389 + 17) % 1024);
  cudaMemcpy(gd, h, 2048 * 8, cudaMemcpyHostToDevice);
  // big chase table: random-ish permutation-ish indices
  unsigned* hb = (unsigned*)malloc((16u << 20) * 4);
  for (unsigned i = 0; i < (16u << 20); ++i) hb[i] = (i * 2654435761u) >> 8;
  cudaMemcpy(gd + 4096, hb, (16u << 20) * 4, cudaMemcpyHostToDevice);
  long long* out; cudaMallocManaged(&out, 16 * 8);
  double* sink; cudaMalloc(&sink, 32 * 8);
  int iters = 4096;
  k<<<1, 32>>>(out, gd, sink, iters);
  k<<<1, 32>>>(out, gd, sink, iters);
  cudaDeviceSynchronize();
  const char* names[] = {"SHFL32", "VOTE+POPC", "DADD", "I2F+DMUL+F2I", "LDS.64 chase", "LDG L1 chase", "IMAD", "u128 cmp+sel", "SHFL64", "LDG L2 chase"};
  for (int i = 0; i < 10; ++i) printf("%-14s %6.1f cycles/op\n", names[i], (double)out[i] / iters);
  return 0;
}
