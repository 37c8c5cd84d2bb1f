// Microbenchmark: random 32 B record gathers through the LSU/L1 path versus
// TMA tile::gather4 (four rows of a 2-D tensor per instruction, straight to
// shared memory, no L1 wavefront queue).
//   12M entries, columns uniform over 1M records of 32 B (the C2 shape).
// nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_tma_gather tools/microbench_tma_gather.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));          \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

// ---- LSU path --------------------------------------------------------------------
template <int ITEMS>
__global__ void k_lsu(const double* __restrict__ vals, const int* __restrict__ cols,
                      const double4* __restrict__ rec, long long nnz, double* out) {
  double acc = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x * ITEMS;
  for (long long b = (long long)blockIdx.x * blockDim.x * ITEMS + threadIdx.x; b < nnz; b += stride) {
    double v[ITEMS];
    int c[ITEMS];
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      const long long e = b + (long long)q * blockDim.x;
      v[q] = e < nnz ? __ldg(vals + e) : 0.0;
      c[q] = e < nnz ? __ldg(cols + e) : 0;
    }
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      double x, y, z, w;
      asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(x), "=d"(y), "=d"(z), "=d"(w) : "l"(rec + c[q]));
      acc += v[q] * (x + y) + z * w;
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

// ---- TMA gather4 path --------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* map, int c0, int r0, int r1, int r2,
                                        int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

constexpr int kWarps = 8;
constexpr int kChunk = 128;  // entries per stage per warp (4 per lane, one gather4 per lane)

template <int S>
__global__ void __launch_bounds__(kWarps * 32) k_tma(const double* __restrict__ vals, const int* __restrict__ cols,
                                                     const __grid_constant__ CUtensorMap map, long long nnz,
                                                     double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double4* buf = reinterpret_cast<double4*>(sm) + (size_t)warp * S * kChunk;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)kWarps * S * kChunk * 32) + warp * S;
  if (lane == 0)
    for (int i = 0; i < S; ++i) mbar_init(&bars[i], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const long long nch = (nnz + kChunk - 1) / kChunk;
  const long long gw = (long long)blockIdx.x * kWarps + warp, nw = (long long)gridDim.x * kWarps;
  double acc = 0.0;
  // chunks gw, gw + nw, ...; stage i holds the i-th of this warp's chunks (mod S)
  auto issue = [&](long long ch, int st) {
    const long long e0 = ch * kChunk + 4 * lane;
    int4 c = make_int4(0, 0, 0, 0);
    if (e0 + 3 < nnz) c = __ldg(reinterpret_cast<const int4*>(cols + e0));
    if (lane == 0) mbar_expect_tx(&bars[st], kChunk * 32);
    __syncwarp();
    gather4(buf + st * kChunk + 4 * lane, &map, 0, c.x, c.y, c.z, c.w, &bars[st]);
  };
  long long it = 0;
  for (int i = 0; i < S; ++i)
    if (gw + i * nw < nch) issue(gw + i * nw, i);
  for (long long ch = gw; ch < nch; ch += nw, ++it) {
    const int st = (int)(it % S);
    mbar_wait(&bars[st], (uint32_t)((it / S) & 1));
    const long long e0 = ch * kChunk + 4 * lane;
    double4 v = make_double4(0, 0, 0, 0);
    if (e0 + 3 < nnz) v = *reinterpret_cast<const double4*>(vals + e0);
    const double4* r = buf + st * kChunk + 4 * lane;
    const double4 r0 = r[0], r1 = r[1], r2 = r[2], r3 = r[3];
    acc += v.x * (r0.x + r0.y) + r0.z * r0.w + v.y * (r1.x + r1.y) + r1.z * r1.w + v.z * (r2.x + r2.y) +
           r2.z * r2.w + v.w * (r3.x + r3.y) + r3.z * r3.w;
    __syncwarp();
    const long long nx = ch + (long long)S * nw;
    if (nx < nch) issue(nx, st);
  }
  if (acc == 12345.678) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const long long nnz = 12'000'000;
  const int n = 1'000'000;
  std::vector<int> hc(nnz);
  srand(7);
  for (auto& c : hc) c = (int)(((unsigned long long)rand() * 2654435761ull) % n);
  double *vals, *out;
  int* cols;
  double4* rec;
  CK(cudaMalloc(&vals, nnz * 8));
  CK(cudaMalloc(&cols, nnz * 4));
  CK(cudaMalloc(&rec, (size_t)n * 32));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemcpy(cols, hc.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(vals, 0, nnz * 8));
  CK(cudaMemset(rec, 0, (size_t)n * 32));
  void* flush;
  CK(cudaMalloc(&flush, 256 << 20));

  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap map;
  const cuuint64_t dims[2] = {4, (cuuint64_t)n};
  const cuuint64_t strides[1] = {32};
  const cuuint32_t box[2] = {4, 1};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, rec, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d\n", (int)r);

  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto time = [&](auto launch, const char* name) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemset(flush, rep, 256 << 20);
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) best = ms < best ? ms : best;
    }
    cudaError_t e = cudaGetLastError();
    printf("%-28s %8.1f us  %s\n", name, best * 1e3, e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  for (int per : {8, 16})
    time([&] { k_lsu<4><<<sms * per, 256>>>(vals, cols, rec, nnz, out); },
         per == 8 ? "lsu items4 grid x8" : "lsu items4 grid x16");
  for (int S : {2, 4, 6}) {
    const size_t shm = (size_t)kWarps * S * kChunk * 32 + kWarps * S * 8;
    auto fn = S == 2 ? (void*)k_tma<2> : S == 4 ? (void*)k_tma<4> : (void*)k_tma<6>;
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    for (int per : {1, 2, 3}) {
      if (shm * per > 228 * 1024) continue;
      char nm[64];
      snprintf(nm, sizeof nm, "tma gather4 S=%d blocks/SM=%d", S, per);
      if (S == 2) time([&] { k_tma<2><<<sms * per, kWarps * 32, shm>>>(vals, cols, map, nnz, out); }, nm);
      if (S == 4) time([&] { k_tma<4><<<sms * per, kWarps * 32, shm>>>(vals, cols, map, nnz, out); }, nm);
      if (S == 6) time([&] { k_tma<6><<<sms * per, kWarps * 32, shm>>>(vals, cols, map, nnz, out); }, nm);
    }
  }
  return 0;
}
