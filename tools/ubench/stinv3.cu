#include <cstdio>
#define LD(v, p) asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p))
// grid of 256x256 doubles; walk a cell x along a path; each iteration lanes 0..7 load
// the 8 neighbours of x (dependent on the previous iteration), then store to them.
__global__ void k(double* G, double* other, long long* out, int mode) {
  const int lane = threadIdx.x, nx = 256;
  const int dr = lane < 8 ? (int)((0x22001120u >> (4 * lane)) & 0xF) - 1 : 0;
  const int dc = lane < 8 ? (int)((0x20202011u >> (4 * lane)) & 0xF) - 1 : 0;
  int r = 100, c = 100;
  double acc = 0;
  // warm region
  for (int i = lane; i < 256 * 256; i += 32) acc += G[i] * 0.0;
  long long t0 = clock64();
  for (int it = 0; it < 512; ++it) {
    const int y = (r + dr) * nx + (c + dc);
    double v = 0;
    if (lane < 8) LD(v, G + y);
    double s = v;
    for (int o = 4; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);   // depend on all 8 loads
    acc += s;
    if (lane < 8) {
      if (mode == 1) G[y] = acc;                 // store to the loaded (neighbour) cells
      if (mode == 2) other[(it * 8 + lane) * 16] = acc;   // store to unrelated lines
    }
    // random-ish walk, one cell per step (diagonal / straight), stays in [20, 236)
    const int m = (it * 7 + (int)(s * 0.0)) & 7;
    r += (m & 1) ? 1 : ((m & 2) ? -1 : 0);
    c += (m & 4) ? 1 : -((m >> 1) & 1);
    r = min(max(r, 20), 235); c = min(max(c, 20), 235);
  }
  long long t1 = clock64();
  if (lane == 0) { out[mode] = t1 - t0; other[1 << 20] = acc; }
}
int main() {
  double *G, *o; cudaMalloc(&G, 256 * 256 * 8); cudaMalloc(&o, (2 << 20) * 8);
  cudaMemset(G, 0, 256 * 256 * 8);
  long long* out; cudaMallocManaged(&out, 64);
  for (int m = 0; m < 3; ++m) k<<<1, 32>>>(G, o, out, m);
  cudaDeviceSynchronize();
  const char* n[] = {"loads only", "store to loaded cells", "store to other lines"};
  for (int m = 0; m < 3; ++m) printf("%-24s %7.1f cycles/iter\n", n[m], out[m] / 512.0);
}
