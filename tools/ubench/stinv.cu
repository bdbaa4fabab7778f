// Does a global store evict/invalidate the L1 line for later loads by the same warp?
#include <cstdio>
__global__ void k(double* g, long long* out) {
  int lane = threadIdx.x;
  volatile double s = 0;
  double acc = 0;
  // warm: load line 0..63 (each 128 B = 16 doubles)
  for (int i = 0; i < 64; ++i) acc += g[i * 16 + 1];
  long long t0, t1;
  // (a) reload hits
  double a = 0;
  t0 = clock64();
  for (int i = 0; i < 64; ++i) { double v; asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(g + i * 16 + 2 + (int)a * 0)); a += v; }
  t1 = clock64(); out[0] = t1 - t0;
  // (b) store to word 3 of each line, then dependent reload of word 4
  t0 = clock64();
  for (int i = 0; i < 64; ++i) {
    if (lane == 0) g[i * 16 + 3] = a;
    double v; asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(g + i * 16 + 4 + (int)a * 0)); a += v;
  }
  t1 = clock64(); out[1] = t1 - t0;
  // (c) reload word 5 after all stores (are lines still in L1?)
  t0 = clock64();
  for (int i = 0; i < 64; ++i) { double v; asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(g + i * 16 + 5 + (int)a * 0)); a += v; }
  t1 = clock64(); out[2] = t1 - t0;
  // (d) cold lines 64..127 for reference (L2)
  t0 = clock64();
  for (int i = 64; i < 128; ++i) { double v; asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(g + i * 16 + 5 + (int)a * 0)); a += v; }
  t1 = clock64(); out[3] = t1 - t0;
  if (lane == 0) g[4096] = a + acc + s;
}
int main() {
  double* g; cudaMalloc(&g, 1 << 20); cudaMemset(g, 0, 1 << 20);
  long long* out; cudaMallocManaged(&out, 64);
  k<<<1, 32>>>(g, out); cudaDeviceSynchronize();
  printf("hit reload %.1f | store+reload same line %.1f | reload after stores %.1f | cold %.1f cycles/load\n",
         out[0] / 64.0, out[1] / 64.0, out[2] / 64.0, out[3] / 64.0);
}
