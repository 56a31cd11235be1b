// Dependent-chain latency of the fp64 / warp ops the replay kernel chains on.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o latency_probe latency_probe.cu
#include <cstdio>
#include <cstdint>

#define N_IT 4096
__global__ void k(double* out, long long* cyc, double a, double b, int x) {
  double v = a; long long t0, t1; int iv = x; unsigned u = x;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < N_IT; ++i) v = __dadd_rn(v, b);
  t1 = clock64(); cyc[0] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < N_IT; ++i) v = __dmul_rn(v, b);
  t1 = clock64(); cyc[1] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < N_IT; ++i) v = __ddiv_rn(v, b);
  t1 = clock64(); cyc[2] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < N_IT; ++i) { iv = (int)__ll2double_rn((long long)iv + 3) & 0xffff; }
  t1 = clock64(); cyc[3] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < N_IT; ++i) { v = (v > b) ? v + 1.0 : v - 1.0; }
  t1 = clock64(); cyc[4] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < N_IT; ++i) { u = __reduce_max_sync(0xffffffffu, u + threadIdx.x); }
  t1 = clock64(); cyc[5] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < N_IT; ++i) { u = __shfl_sync(0xffffffffu, u, (u + 1) & 31); }
  t1 = clock64(); cyc[6] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < N_IT; ++i) { iv = iv * 3 + 1; }
  t1 = clock64(); cyc[7] = t1 - t0;
  out[threadIdx.x] = v + iv + u;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 256 * 8); cudaMalloc(&c, 64 * 8);
  k<<<1, 32>>>(d, c, 1.0, 1.0000001, 5);
  k<<<1, 32>>>(d, c, 1.0, 1.0000001, 5);
  long long h[8]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const char* n[8] = {"DADD", "DMUL", "DDIV(__ddiv_rn)", "I2F.F64+F2I", "DSETP+select+DADD", "REDUX", "SHFL", "IMAD"};
  for (int i = 0; i < 8; ++i) printf("%-22s %.1f cycles/op\n", n[i], (double)h[i] / N_IT);
  return 0;
}
