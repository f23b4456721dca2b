// dawn_fw.cuh — dense all-pairs Floyd–Warshall on the device,
// the cross-check oracle floyd_warshall_apsp (oracles.py:141-162) at sizes the
// NumPy loop cannot reach.
//
// Semantics kept exactly (float64):
//   init : D = +inf, D[i][i] = 0, then D[u][v] = min(D[u][v], w) over every
//          edge (parallel edges and self-loops included: np.minimum.at);
//   step k (k = 0..n-1): D = min(D, col_k + row_k) where col_k = D[:, k] and
//          row_k = D[k, :] are the values BEFORE step k (NumPy materialises
//          mat[:, k:k+1] + mat[k:k+1, :] before the minimum), the sum is one
//          IEEE add, and the minimum keeps D unless the sum is strictly
//          smaller;
//   negative_cycle = any D[i][i] < 0.
// Not blocked: a tiled (blocked) Floyd–Warshall relaxes through pivots of the
// same block in a different order, which is exact for integers but can round
// differently for floats.  Each step is one pass over the matrix (L2-resident
// up to n ≈ 3900 for 126 MB of L2); one persistent cooperative launch runs
// all n steps with one grid barrier per step.  The pre-step row/column of
// step k+1 are double-buffered: whoever owns D[i][k+1] / D[k+1][j] writes its
// step-k result there too, so no extra barrier is needed for the snapshot.
#pragma once
#include "dawn_device.cuh"

namespace dawn {

// order-preserving u64 key of a double (for the init's atomic minimum)
__device__ __forceinline__ unsigned long long fw_key(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double fw_unkey(unsigned long long k) {
  const unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)b);
}

// D as keys: +inf everywhere, 0 on the diagonal
__global__ void fw_init(unsigned long long* D, int64_t n) {
  const unsigned long long kinf = fw_key(CUDART_INF), kzero = fw_key(0.0);
  const int64_t nn = n * n;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < nn; x += (int64_t)gridDim.x * blockDim.x)
    D[x] = (x / n == x % n) ? kzero : kinf;
}

// np.minimum.at(mat, (u, col), val): every edge, order-free exact minimum
__global__ void fw_edges(unsigned long long* D, int64_t n, const int64_t* __restrict__ row_ptr,
                         const int64_t* __restrict__ col, const double* __restrict__ val, unsigned* bad) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = row_ptr[u], b = row_ptr[u + 1];
    for (int64_t e = a; e < b; ++e) {
      const int64_t v = col[e];
      if (v < 0 || v >= n) {
        atomicOr(bad, 1u);
        continue;
      }
      atomicMin(D + u * n + v, fw_key(val[e]));
    }
  }
}

// keys -> doubles in place, and the step-0 row/column snapshot
__global__ void fw_decode(unsigned long long* D, int64_t n, double* col0, double* row0) {
  const int64_t nn = n * n;
  double* M = reinterpret_cast<double*>(D);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < nn; x += (int64_t)gridDim.x * blockDim.x) {
    const double d = fw_unkey(D[x]);
    M[x] = d;
    if (x % n == 0) col0[x / n] = d;
    if (x < n) row0[x] = d;
  }
}

// all n steps; thread t owns elements t, t + T, ... of the row-major matrix
__global__ void __launch_bounds__(256) fw_steps(double* __restrict__ M, int64_t n, double* __restrict__ colb,
                                                double* __restrict__ rowb, unsigned* bar) {
  const int64_t nn = n * n;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t Tq = T / n, Tr = T % n, i0 = t0 / n, j0 = t0 % n;  // (row, col) steps of the stride
  for (int64_t k = 0; k < n; ++k) {
    const double* ck = colb + (k & 1) * n;  // D[:, k] before step k
    const double* rk = rowb + (k & 1) * n;  // D[k, :] before step k
    double* cn = colb + ((k + 1) & 1) * n;  // D[:, k+1] after step k
    double* rn = rowb + ((k + 1) & 1) * n;
    const int64_t k1 = k + 1;
    int64_t i = i0, j = j0;
    for (int64_t x = t0; x < nn; x += T) {
      const double s = __dadd_rn(__ldcg(ck + i), __ldcg(rk + j));
      double d = M[x];
      if (s < d) {
        d = s;
        M[x] = d;
      }
      if (j == k1) cn[i] = d;
      if (i == k1) rn[j] = d;
      i += Tq;
      j += Tr;
      if (j >= n) {
        j -= n;
        ++i;
      }
    }
    if (grid_sync(bar, bar + 3)) return;  // [3]: watchdog abort word
  }
}

// any negative diagonal entry
__global__ void fw_negdiag(const double* M, int64_t n, unsigned* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (M[i * n + i] < 0.0) atomicOr(flag, 1u);
}

}  // namespace dawn
