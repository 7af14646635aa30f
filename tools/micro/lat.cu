// Dependent-chain latency of a few fp64 / int64 operations on the GPU (one
// thread, clock64 deltas).  Diagnostics only.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b, long long ia) {
  double x = a;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 512; ++i) { x = __dadd_rn(x, b); x = __dadd_rn(x, b); x = __dadd_rn(x, b); x = __dadd_rn(x, b); x = __dadd_rn(x, b); x = __dadd_rn(x, b); x = __dadd_rn(x, b); x = __dadd_rn(x, b); }
  long long t1 = clock64();
  double y = a;
#pragma unroll 1
  for (int i = 0; i < 512; ++i) { y = __dmul_rn(y, b); y = __dmul_rn(y, b); y = __dmul_rn(y, b); y = __dmul_rn(y, b); y = __dmul_rn(y, b); y = __dmul_rn(y, b); y = __dmul_rn(y, b); y = __dmul_rn(y, b); }
  long long t2 = clock64();
  long long z = ia;
#pragma unroll 1
  for (int i = 0; i < 512; ++i) { z = z * 3 + i; z = z * 3 + i; z = z * 3 + i; z = z * 3 + i; z = z * 3 + i; z = z * 3 + i; z = z * 3 + i; z = z * 3 + i; }
  long long t3 = clock64();
  double w = a;
#pragma unroll 1
  for (int i = 0; i < 4096; ++i) w = (double)(long long)w + b;
  long long t4 = clock64();
  double u = a;
#pragma unroll 1
  for (int i = 0; i < 4096; ++i) u = (u <= b) ? __dadd_rn(u, 1.0) : __dadd_rn(u, -1.0);
  long long t5 = clock64();
  out[0] = x + y + (double)z + w + u;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 8); cudaMallocManaged(&c, 64);
  k<<<1, 1>>>(o, c, 1.0, 1e-9, 7);
  cudaDeviceSynchronize();
  k<<<1, 1>>>(o, c, 1.0, 1e-9, 7);
  cudaDeviceSynchronize();
  const char* n[] = {"DADD", "DMUL", "IMAD64", "F2I+I2F+DADD", "DSETP+branch+DADD"};
  for (int i = 0; i < 5; ++i) printf("%-20s %.1f cycles/op\n", n[i], c[i] / 4096.0);
  return 0;
}
