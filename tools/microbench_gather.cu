// Microbenchmark: the memory floor of one propagation round.
// Streams vals (f64) + cols (i32) and gathers one random per-column record
// per entry, reducing into a per-thread sum (no propagation math).
//   mode 0: stream only (12 B/entry)
//   mode 1: + 16 B gather (LDG.128)
//   mode 2: + 32 B gather (LDG.256)
//   mode 3: + 8 B gather
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_gather tools/microbench_gather.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

struct __align__(32) Rec {
  double a, b, c, d;
};

template <int MODE, int ITEMS>
__global__ void k(const double* __restrict__ vals, const int* __restrict__ cols,
                  const Rec* __restrict__ recs, long long nnz, double* out) {
  double acc = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x * ITEMS;
  for (long long base = (long long)blockIdx.x * blockDim.x * ITEMS + threadIdx.x; base < nnz;
       base += stride) {
    double v[ITEMS];
    int c[ITEMS];
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      const long long e = base + (long long)q * blockDim.x;
      if (e < nnz) {
        v[q] = __ldg(vals + e);
        c[q] = __ldg(cols + e);
      } else {
        v[q] = 0;
        c[q] = 0;
      }
    }
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      double g = 0;
      if (MODE == 1) {
        const double2 r = __ldg(reinterpret_cast<const double2*>(recs + c[q]));
        g = r.x + r.y;
      } else if (MODE == 2) {
        double a, b, cc, d;
        asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
            : "=d"(a), "=d"(b), "=d"(cc), "=d"(d)
            : "l"(recs + c[q]));
        g = a + b + cc + d;
      } else if (MODE == 3) {
        g = __ldg(reinterpret_cast<const double*>(recs + c[q]));
      }
      acc += v[q] * g + v[q];
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

template <int MODE, int ITEMS = 8>
float run(const double* v, const int* c, const Rec* r, long long nnz, double* out, int grid,
          int threads = 256) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k<MODE, ITEMS><<<grid, threads>>>(v, c, r, nnz, out);
  cudaEventRecord(a);
  const int reps = 10;
  for (int i = 0; i < reps; ++i) k<MODE, ITEMS><<<grid, threads>>>(v, c, r, nnz, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main(int argc, char** argv) {
  const long long nnz = argc > 1 ? atoll(argv[1]) : 12000000;
  const int n = argc > 2 ? atoi(argv[2]) : 1000000;
  std::vector<int> hc(nnz);
  unsigned long long s = 88172645463325252ull;
  for (long long i = 0; i < nnz; ++i) {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    hc[i] = (int)(s % n);
  }
  double *v, *out;
  int* c;
  Rec* r;
  cudaMalloc(&v, nnz * 8);
  cudaMalloc(&c, nnz * 4);
  cudaMalloc(&r, (size_t)n * sizeof(Rec));
  cudaMalloc(&out, 8);
  cudaMemset(v, 0, nnz * 8);
  cudaMemset(r, 0, (size_t)n * sizeof(Rec));
  cudaMemcpy(c, hc.data(), nnz * 4, cudaMemcpyHostToDevice);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int occ : {4, 8, 16}) {
    const int grid = sms * occ;
    const float t0 = run<0>(v, c, r, nnz, out, grid);
    const float t1 = run<1>(v, c, r, nnz, out, grid);
    const float t2 = run<2>(v, c, r, nnz, out, grid);
    const float t3 = run<3>(v, c, r, nnz, out, grid);
    printf("grid %d: stream %.1f us (%.0f GB/s) | +16B gather %.1f us | +32B gather %.1f us | +8B gather %.1f us\n",
           grid, t0 * 1e3, 12.0 * nnz / (t0 * 1e-3) / 1e9, t1 * 1e3, t2 * 1e3, t3 * 1e3);
  }
  // memory-level-parallelism sweep for the 16 B gather: warps/SM x items
  printf("MLP sweep (16 B gather, 12M entries): warps/SM items -> us, in-flight/SM\n");
  for (int wps : {4, 8, 12, 16, 24, 32}) {
    const int grid = sms * wps / 4;  // 128-thread CTAs
    const float t1 = run<1, 1>(v, c, r, nnz, out, grid, 128);
    const float t2 = run<1, 2>(v, c, r, nnz, out, grid, 128);
    const float t4 = run<1, 4>(v, c, r, nnz, out, grid, 128);
    const float t8 = run<1, 8>(v, c, r, nnz, out, grid, 128);
    printf("  %2d warps/SM: items1 %.1f | items2 %.1f | items4 %.1f | items8 %.1f us\n", wps,
           t1 * 1e3, t2 * 1e3, t4 * 1e3, t8 * 1e3);
  }
  return 0;
}
