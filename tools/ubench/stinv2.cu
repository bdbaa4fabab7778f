#include <cstdio>
#define LD(v, p) asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p))
#define LDCG(v, p) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p))
__global__ void k(double* g, long long* out) {
  int lane = threadIdx.x;
  double a = 0;
  for (int i = 0; i < 256; ++i) a += g[i * 16 + 1];
  long long t0, t1;
  // (b) all lanes store word 3, reload word 4 (same line), dependent chain
  t0 = clock64();
  for (int i = 0; i < 64; ++i) { g[i * 16 + 3] = a; double v; LD(v, g + i * 16 + 4 + ((long long)a & 0)); a += v; }
  t1 = clock64(); out[0] = t1 - t0;
  // (c) store line i, load line i+100 (different line)
  t0 = clock64();
  for (int i = 0; i < 64; ++i) { g[i * 16 + 3] = a; double v; LD(v, g + (i + 100) * 16 + 4 + ((long long)a & 0)); a += v; }
  t1 = clock64(); out[1] = t1 - t0;
  // (d) store, then .cg load same line
  t0 = clock64();
  for (int i = 0; i < 64; ++i) { g[i * 16 + 3] = a; double v; LDCG(v, g + i * 16 + 4 + ((long long)a & 0)); a += v; }
  t1 = clock64(); out[2] = t1 - t0;
  // (e) .cg loads without stores (L2 latency)
  t0 = clock64();
  for (int i = 0; i < 64; ++i) { double v; LDCG(v, g + i * 16 + 5 + ((long long)a & 0)); a += v; }
  t1 = clock64(); out[3] = t1 - t0;
  // (f) dependent L1-hit loads, no stores
  t0 = clock64();
  for (int i = 0; i < 64; ++i) { double v; LD(v, g + i * 16 + 6 + ((long long)a & 0)); a += v; }
  t1 = clock64(); out[4] = t1 - t0;
  // (g) store same line, then load the same line only after 8 other dependent L1-hit loads
  t0 = clock64();
  for (int i = 0; i < 64; ++i) {
    g[i * 16 + 3] = a;
    for (int j = 0; j < 8; ++j) { double v; LD(v, g + (200 + j) * 16 + ((long long)a & 0)); a += v * 0.0; }
    double v; LD(v, g + i * 16 + 4 + ((long long)a & 0)); a += v;
  }
  t1 = clock64(); out[5] = t1 - t0;
  // (h) volatile STS/LDS equivalents in shared memory
  __shared__ double sm[4096];
  for (int i = lane; i < 4096; i += 32) sm[i] = i;
  __syncwarp();
  t0 = clock64();
  for (int i = 0; i < 64; ++i) { sm[i * 16 + 3] = a; double v = ((volatile double*)sm)[i * 16 + 4 + ((long long)a & 0)]; a += v; }
  t1 = clock64(); out[6] = t1 - t0;
  if (lane == 0) g[8192] = a;
}
int main() {
  double* g; cudaMalloc(&g, 1 << 20); cudaMemset(g, 0, 1 << 20);
  long long* out; cudaMallocManaged(&out, 128);
  k<<<1, 32>>>(g, out); cudaDeviceSynchronize();
  const char* n[] = {"st+ld same line", "st+ld other line", "st+ld.cg same line", "ld.cg only", "ld L1 hit dep", "st, 8 loads, ld same line", "smem st+ld"};
  for (int i = 0; i < 7; ++i) printf("%-28s %7.1f cycles/iter\n", n[i], out[i] / 64.0);
}
