// gather_bench.cu — ceiling of the relax access pattern on this GPU.
//
// Streams m packed (col, w) edges of an RMAT graph (same counter hash as the
// library's generator, so the destination skew is the real one) and gathers
// dist[col] with several load flavours.  No frontier logic: this is the
// hardware bound the X phase is measured against.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/gather_bench tools/gather_bench.cu
//   ./build/gather_bench [scale=22] [edge_factor=16]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t err_ = (x); if (err_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(err_)); exit(1); } } while (0)

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ unsigned long long draw64(unsigned long long seed, unsigned long long i, unsigned lvl) {
  return mix64(seed * 0x9E3779B97F4A7C15ull + i * 64ull + lvl + 0x9E3779B97F4A7C15ull);
}

__global__ void gen(int scale, long long m, uint2* e, int relabel_hot) {
  const uint32_t A = (uint32_t)(0.57 * 16777216.0), AB = (uint32_t)(0.76 * 16777216.0), ABC = (uint32_t)(0.95 * 16777216.0);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
    uint32_t v = 0;
    for (int l = 0; l < scale; ++l) {
      const uint32_t q = (uint32_t)(draw64(1, i, l) >> 40);
      v |= (uint32_t)((q >= A && q < AB) || q >= ABC) << l;
    }
    const unsigned long long h = draw64(2, i, 63);
    e[i] = make_uint2(v, __float_as_uint((float)(h >> 40) * (1.0f / 16777216.0f)));
  }
}

__device__ __forceinline__ uint2 ld_stream(const uint2* p) {
  uint2 r;
  asm("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

template <int MODE>
__global__ void __launch_bounds__(256) relax_like(const uint2* __restrict__ e, long long m, uint32_t* dist,
                                                  unsigned long long* out) {
  // MODE 0: stream only; 1: + ld.cg gather; 2: + ld.ca gather; 3: + ld.cg gather + red.min when better
  unsigned long long acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x * 8;
  for (long long base = (blockIdx.x * (long long)blockDim.x) * 8 + threadIdx.x; base < m; base += stride) {
    uint2 x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const long long i = base + j * blockDim.x;
      x[j] = i < m ? ld_stream(e + i) : make_uint2(0, 0);
    }
    if (MODE == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += x[j].x ^ x[j].y;
    } else {
      uint32_t c[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) c[j] = (MODE == 2 || MODE == 4) ? __ldca(dist + x[j].x) : __ldcg(dist + x[j].x);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t cand = x[j].y + 0x3F000000u;
        if (cand < c[j]) {
          if (MODE == 3 || MODE == 4) atomicMin(dist + x[j].x, cand);
          acc++;
        }
      }
    }
  }
  if (acc == 0xFFFFFFFFFFFFull) *out = acc;
}

int main(int argc, char** argv) {
  const int scale = argc > 1 ? atoi(argv[1]) : 22;
  const long long ef = argc > 2 ? atoll(argv[2]) : 16;
  const long long n = 1ll << scale, m = ef * n;
  uint2* e;
  uint32_t* dist;
  unsigned long long* out;
  CK(cudaMalloc(&e, 8 * m));
  CK(cudaMalloc(&dist, 4 * n));
  CK(cudaMalloc(&out, 8));
  void* flush;
  CK(cudaMalloc(&flush, 256 << 20));
  gen<<<148 * 16, 256>>>(scale, m, e, 0);
  CK(cudaDeviceSynchronize());
  int nsm = 148;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"stream only", "stream + ld.cg gather", "stream + ld.ca gather", "stream + gather + red.min",
                         "ld.ca gather + red.min"};
  for (int mode = 0; mode < 5; ++mode) {
    for (int bps : {4, 8}) {
      float best = 1e9f;
      for (int rep = 0; rep < 5; ++rep) {
        CK(cudaMemset(dist, 0x3F, 4 * n));  // ~0.75: about half the candidates "improve"
        CK(cudaMemset(flush, rep, 256 << 20));
        cudaEventRecord(a);
        switch (mode) {
          case 0: relax_like<0><<<nsm * bps, 256>>>(e, m, dist, out); break;
          case 1: relax_like<1><<<nsm * bps, 256>>>(e, m, dist, out); break;
          case 2: relax_like<2><<<nsm * bps, 256>>>(e, m, dist, out); break;
          case 3: relax_like<3><<<nsm * bps, 256>>>(e, m, dist, out); break;
          default: relax_like<4><<<nsm * bps, 256>>>(e, m, dist, out); break;
        }
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("%-28s ctas/sm=%d  %.3f ms  %.1f G edges/s  stream %.0f GB/s\n", names[mode], bps, best,
             m / best / 1e6, 8.0 * m / best / 1e6);
    }
  }
  // L1 capacity sensitivity: ld.ca gather with the shared-memory carveout forced up
  for (int carve : {0, 25, 50, 75, 100}) {
    CK(cudaFuncSetAttribute(relax_like<2>, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaMemset(dist, 0x3F, 4 * n));
      CK(cudaMemset(flush, rep, 256 << 20));
      cudaEventRecord(a);
      relax_like<2><<<nsm * 8, 256, 1024>>>(e, m, dist, out);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("ld.ca gather, smem carveout %3d%%  %.3f ms  %.1f G edges/s\n", carve, best, m / best / 1e6);
  }
  return 0;
}
