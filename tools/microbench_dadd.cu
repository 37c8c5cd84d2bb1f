// Dependent-chain latency of FP64 add / mul and FP32 add on this GPU
// (one thread, clock64), the floor of a serial activity chain.
#include <cstdio>
__global__ void k(double* out, float* outf, long long* cyc, double x0, float f0) {
  double a = x0, b = x0 * 0.5;
  float f = f0;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 4096; ++i) a = __dadd_rn(a, b);
  long long t1 = clock64();
#pragma unroll 16
  for (int i = 0; i < 4096; ++i) a = __dmul_rn(a, 1.0000001);
  long long t2 = clock64();
#pragma unroll 16
  for (int i = 0; i < 4096; ++i) f = __fadd_rn(f, 0.5f);
  long long t3 = clock64();
  out[0] = a;
  outf[0] = f;
  cyc[0] = t1 - t0;
  cyc[1] = t2 - t1;
  cyc[2] = t3 - t2;
}
int main() {
  double* o; float* of; long long* c;
  cudaMalloc(&o, 8); cudaMalloc(&of, 4); cudaMalloc(&c, 24);
  for (int r = 0; r < 2; ++r) k<<<1, 1>>>(o, of, c, 1.0, 1.0f);
  long long h[3];
  cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("cycles per dependent op: DADD %.2f  DMUL %.2f  FADD %.2f\n", h[0] / 4096.0, h[1] / 4096.0, h[2] / 4096.0);
  return 0;
}
