// Grid-barrier cost on one B200 (persistent cooperative launch).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bb tools/barrier_bench.cu && /tmp/bb
// Variants: 0 = dawn_device.cuh grid_sync (flip-bit counter, acquire spin)
//           1 = same with __nanosleep backoff in the spin
//           2 = generation flag: arrivals on a counter, the last arriver bumps a
//               flag in a separate line, waiters poll the flag
//           3 = cooperative_groups grid.sync()
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int VAR>
__device__ __forceinline__ void gsync(unsigned* bar, unsigned* flag, unsigned& gen) {
  if constexpr (VAR == 3) {
    cg::this_grid().sync();
    return;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if constexpr (VAR == 0 || VAR == 1) {
      const unsigned nb = gridDim.x;
      const unsigned inc = (blockIdx.x == 0) ? (0x80000000u - (nb - 1u)) : 1u;
      __threadfence();
      const unsigned old = atomicAdd(bar, inc);
      while (((old ^ ld_acquire(bar)) & 0x80000000u) == 0u) {
        if (VAR == 1) __nanosleep(64);
      }
      __threadfence();
    } else {
      __threadfence();
      const unsigned old = atomicAdd(bar, 1u);
      if (old == gridDim.x - 1) {
        *bar = 0;
        __threadfence();
        atomicAdd(flag, 1u);
      } else {
        while (ld_acquire(flag) == gen) {
        }
      }
      gen++;
      __threadfence();
    }
  }
  __syncthreads();
}

template <int VAR>
__global__ void k(unsigned* bar, unsigned* flag, int iters, unsigned long long* out) {
  unsigned gen = 0;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) gsync<VAR>(bar, flag, gen);
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

template <int VAR>
float run(int grid, int iters) {
  unsigned *bar, *flag;
  unsigned long long* out;
  cudaMalloc(&bar, 256);
  cudaMalloc(&flag, 256);
  cudaMalloc(&out, 8);
  cudaMemset(bar, 0, 256);
  cudaMemset(flag, 0, 256);
  void* args[] = {&bar, &flag, &iters, &out};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaLaunchCooperativeKernel((void*)k<VAR>, grid, 256, args, 0, 0);
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  cudaLaunchCooperativeKernel((void*)k<VAR>, grid, 256, args, 0, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  cudaFree(bar);
  cudaFree(flag);
  cudaFree(out);
  return 1e3f * ms / iters;
}

int main() {
  const int iters = 20000;
  for (int grid : {148, 296, 444, 592}) {
    printf("grid %4d: flip %.2f us  flip+sleep %.2f us  genflag %.2f us  cg %.2f us\n", grid, run<0>(grid, iters),
           run<1>(grid, iters), run<2>(grid, iters), run<3>(grid, iters));
  }
  return 0;
}
