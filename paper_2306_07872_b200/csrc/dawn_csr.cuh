// dawn_csr.cuh — canonical CSR construction on the device.
//
// Replaces build_csr (reference graph.py:303-322): rows by source, columns
// ascending, ties in input order, duplicates and self-loops kept.  The order
// is a STABLE radix sort of the 64-bit key u*n + v (CUB onesweep, LSD, hence
// stable), so equal (u, v) pairs keep their input order exactly as the
// reference's np.lexsort((v, u)) does.  row_ptr comes from the sorted keys
// (row boundaries), not from atomics, so it is deterministic.
#pragma once
#include <cub/device/device_radix_sort.cuh>

namespace dawn {

enum : unsigned { CSR_ERR_NODE = 1u, CSR_ERR_WEIGHT = 2u };

__global__ void k_csr_keys(const int64_t* __restrict__ u, const int64_t* __restrict__ v,
                           const double* __restrict__ w, int64_t n, int64_t m,
                           unsigned long long* __restrict__ keys, unsigned long long* __restrict__ idx,
                           unsigned* flags) {
  unsigned f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = u[i], b = v[i];
    if (a < 0 || a >= n || b < 0 || b >= n) f |= CSR_ERR_NODE;
    if (!isfinite(w[i])) f |= CSR_ERR_WEIGHT;
    keys[i] = (unsigned long long)a * (unsigned long long)n + (unsigned long long)b;
    idx[i] = (unsigned long long)i;
  }
  if (f) atomicOr(flags, f);
}

// col/val gathered in sorted order
__global__ void k_csr_emit(const unsigned long long* __restrict__ keys, const unsigned long long* __restrict__ idx,
                           const double* __restrict__ w, int64_t n, int64_t m, int64_t* __restrict__ col,
                           double* __restrict__ val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    col[i] = (int64_t)(k % (unsigned long long)n);
    val[i] = w[idx[i]];
  }
}

// row_ptr[q] = first sorted position whose row is >= q (a lower bound on the
// sorted keys): parallel over rows, no atomics, empty rows free.
__global__ void k_csr_rowptr(const unsigned long long* __restrict__ keys, int64_t n, int64_t m,
                             int64_t* __restrict__ row_ptr) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q <= n; q += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long t = (unsigned long long)q * (unsigned long long)n;
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < t) lo = mid + 1; else hi = mid;
    }
    row_ptr[q] = lo;
  }
}

__global__ void k_csr_empty(int64_t n, int64_t* row_ptr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
    row_ptr[i] = 0;
}

}  // namespace dawn
