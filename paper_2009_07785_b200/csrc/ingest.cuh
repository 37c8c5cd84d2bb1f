// ingest.cuh -- on-device CSR build from triplets.
//
// csr_from_triplets (core/src/model.cpp:37-80): range check (the first bad
// triplet decides the message, rows checked before columns), stable sort by
// (row, col), duplicates summed in input order starting from 0.0, zero sums
// dropped.  On the device: one 64-bit key per triplet (row above col), an
// LSD radix sort of (key, value) pairs -- stable, so equal keys keep their
// input order -- then every run head sums its run sequentially (the
// reference's `sum += value` order; runs are almost always length 1),
// compaction by an exclusive scan of the keep flags, row counts by atomics
// into an exclusive scan.
#pragma once

#include <cstdint>

namespace pgb {

// first triplet index with a bad row or column (atomicMin over indices)
__global__ void k_trip_check(const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                             int64_t count, int32_t m, int32_t n,
                             unsigned long long* __restrict__ first_bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rows[i], c = cols[i];
    if (r < 0 || r >= m || c < 0 || c >= n) atomicMin(first_bad, (unsigned long long)i);
  }
}

__global__ void k_trip_keys(const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                            int64_t count, int colbits, unsigned long long* __restrict__ key) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    key[i] = ((unsigned long long)(uint32_t)rows[i] << colbits) | (uint32_t)cols[i];
}

// run heads: sequential sum of the run, keep flag (sum != 0), row counts
__global__ void k_trip_runs(const unsigned long long* __restrict__ key,
                            const double* __restrict__ val, int64_t count, int colbits,
                            double* __restrict__ sum, int32_t* __restrict__ keep,
                            int32_t* __restrict__ row_cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = key[i];
    int32_t kp = 0;
    if (i == 0 || key[i - 1] != k) {
      double s = 0.0;
      for (int64_t j = i; j < count && key[j] == k; ++j) s = __dadd_rn(s, val[j]);
      sum[i] = s;
      if (s != 0.0) {
        kp = 1;
        atomicAdd(&row_cnt[k >> colbits], 1);
      }
    }
    keep[i] = kp;
  }
}

__global__ void k_trip_emit(const unsigned long long* __restrict__ key,
                            const double* __restrict__ sum, const int32_t* __restrict__ keep,
                            const int32_t* __restrict__ pos, int64_t count, int colbits,
                            int32_t* __restrict__ col_out, double* __restrict__ val_out) {
  const unsigned long long cmask = (1ull << colbits) - 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    if (keep[i]) {
      col_out[pos[i]] = (int32_t)(key[i] & cmask);
      val_out[pos[i]] = sum[i];
    }
}

}  // namespace pgb
