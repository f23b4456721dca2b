// dawn_device.cuh — device-side building blocks for the weighted-DAWN kernels.
//
// Value traits map every supported distance type onto an order-preserving
// unsigned key so one atomicMin(uint32/uint64) implements the reference's
// strict-`>` relax `if alpha[idx] > cand: alpha[idx] = cand`
// (solver.py:298, :373) deterministically on any type.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <type_traits>

namespace dawn {

#ifndef DAWN_MIN_BLOCKS
#define DAWN_MIN_BLOCKS 2   // resident CTAs per SM the register budget is sized for (128 regs, no spills)
#endif

#ifndef DAWN_NT
#define DAWN_NT 256
#endif
constexpr int NT = DAWN_NT;         // threads per CTA
constexpr int ITEMS = 8;            // virtual edges per thread per tile
constexpr int TILE = NT * ITEMS;    // virtual edges per tile (2048)

// ---------------------------------------------------------------------------
// value traits.  Every key array is initialised by memset(0xFF): the all-ones
// key is the "unreachable" sentinel (reference: math.inf, solver.py:276, :343).
// ---------------------------------------------------------------------------
template <class V> struct Val;

template <> struct Val<int32_t> {
  using K = uint32_t;
  using WB = uint32_t;  // weight bits as stored in the edge array
  static constexpr K INF = 0xFFFFFFFFu;  // == enc(INT32_MAX); host bound keeps sums below it
  __device__ __forceinline__ static K enc(int32_t v) { return (uint32_t)v ^ 0x80000000u; }
  __device__ __forceinline__ static int32_t dec(K k) { return (int32_t)(k ^ 0x80000000u); }
  __device__ __forceinline__ static K relax(K ku, WB w) { return enc(dec(ku) + (int32_t)w); }
  __device__ __forceinline__ static bool usable(K c) { return true; }
  __device__ __forceinline__ static double to_f64(K k) {
    return k == INF ? CUDART_INF : (double)dec(k);
  }
};

template <> struct Val<int64_t> {
  using K = unsigned long long;
  using WB = unsigned long long;
  static constexpr K INF = 0xFFFFFFFFFFFFFFFFull;
  __device__ __forceinline__ static K enc(int64_t v) {
    return (unsigned long long)v ^ 0x8000000000000000ull;
  }
  __device__ __forceinline__ static int64_t dec(K k) {
    return (int64_t)(k ^ 0x8000000000000000ull);
  }
  __device__ __forceinline__ static K relax(K ku, WB w) { return enc(dec(ku) + (int64_t)w); }
  __device__ __forceinline__ static bool usable(K c) { return true; }
  __device__ __forceinline__ static double to_f64(K k) {
    return k == INF ? CUDART_INF : (double)dec(k);
  }
};

template <> struct Val<float> {
  using K = uint32_t;
  using WB = uint32_t;
  static constexpr K INF = 0xFFFFFFFFu;       // sentinel (a NaN pattern, never produced)
  static constexpr K FINF = 0xFF800000u;      // enc(+inf): candidates >= this never write
  __device__ __forceinline__ static K enc(float f) {
    uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  }
  __device__ __forceinline__ static float dec(K k) {
    uint32_t b = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
    return __uint_as_float(b);
  }
  __device__ __forceinline__ static K relax(K ku, WB w) {
    float c = __fadd_rn(dec(ku), __uint_as_float(w));
    return enc(__fadd_rn(c, 0.0f));  // -0 -> +0 so key order == numeric order
  }
  // reference: `alpha[idx] > cand` is false for cand == inf (overflow), so never write it
  __device__ __forceinline__ static bool usable(K c) { return c < FINF; }
  __device__ __forceinline__ static double to_f64(K k) {
    return k == INF ? CUDART_INF : (double)dec(k);
  }
};

template <> struct Val<double> {
  using K = unsigned long long;
  using WB = unsigned long long;
  static constexpr K INF = 0xFFFFFFFFFFFFFFFFull;
  static constexpr K FINF = 0xFFF0000000000000ull;  // enc(+inf)
  __device__ __forceinline__ static K enc(double f) {
    unsigned long long b = (unsigned long long)__double_as_longlong(f);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
  }
  __device__ __forceinline__ static double dec(K k) {
    unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    return __longlong_as_double((long long)b);
  }
  __device__ __forceinline__ static K relax(K ku, WB w) {
    double c = __dadd_rn(dec(ku), __longlong_as_double((long long)w));
    return enc(__dadd_rn(c, 0.0));
  }
  __device__ __forceinline__ static bool usable(K c) { return c < FINF; }
  __device__ __forceinline__ static double to_f64(K k) { return k == INF ? CUDART_INF : dec(k); }
};

// ---------------------------------------------------------------------------
// Key codec used by the kernels.  RAW (the graph has no negative weight, so
// every distance is >= +0): a non-negative value's own bit pattern is already
// order-preserving as an unsigned integer, so keys are raw bits and one relax
// is a single add.  Otherwise the sign-flip encoding of Val<V>.  Row values
// are decoded once per frontier row (C), never per edge.
// ---------------------------------------------------------------------------
template <class V> struct Bits;
template <> struct Bits<float> {
  __device__ __forceinline__ static uint32_t to(float x) { return __float_as_uint(x); }
  __device__ __forceinline__ static float from(uint32_t b) { return __uint_as_float(b); }
};
template <> struct Bits<double> {
  __device__ __forceinline__ static unsigned long long to(double x) { return (unsigned long long)__double_as_longlong(x); }
  __device__ __forceinline__ static double from(unsigned long long b) { return __longlong_as_double((long long)b); }
};

template <class V, bool RAW>
struct Codec {
  using B = Val<V>;
  using K = typename B::K;
  using WB = typename B::WB;
  using C = V;  // per-row compute value
  static constexpr K INF = B::INF;
  static constexpr bool FP = std::is_floating_point<V>::value;
  __device__ __forceinline__ static C dec(K k) {
    if constexpr (!RAW) return B::dec(k);
    else if constexpr (FP) return Bits<V>::from(k);
    else return (C)k;
  }
  __device__ __forceinline__ static K enc(C c) {
    if constexpr (!RAW) return B::enc(c);
    else if constexpr (FP) return Bits<V>::to(c);
    else return (K)c;
  }
  __device__ __forceinline__ static K relax(C du, WB w) {
    if constexpr (FP) {
      C sum;
      if constexpr (sizeof(V) == 4) sum = __fadd_rn(du, Bits<V>::from(w));
      else sum = __dadd_rn(du, Bits<V>::from(w));
      if constexpr (!RAW) {  // -0 -> +0 so key order == numeric order
        if constexpr (sizeof(V) == 4) sum = __fadd_rn(sum, 0.0f);
        else sum = __dadd_rn(sum, 0.0);
      }
      return enc(sum);
    } else {
      return enc(du + (C)w);
    }
  }
  // reference: `alpha[idx] > cand` is false for cand == inf (overflow): never write it
  __device__ __forceinline__ static bool usable(K c) {
    if constexpr (!FP) return true;
    else if constexpr (RAW) return c < Bits<V>::to((V)CUDART_INF);
    else return c < B::FINF;
  }
  __device__ __forceinline__ static double to_f64(K k) {
    return k == INF ? CUDART_INF : (double)dec(k);
  }
};

// ---------------------------------------------------------------------------
// memory helpers
// ---------------------------------------------------------------------------
// Data written by other CTAs inside the same persistent launch must bypass the
// (non-coherent) L1: ld.global.cg.
template <class T> __device__ __forceinline__ T ldcg(const T* p) { return __ldcg(p); }

// Edge stream: read exactly once per relax, keep it out of L1 so L1 holds dist.
__device__ __forceinline__ uint2 ld_stream(const uint2* p) {
  uint2 r;
  asm("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) {
  uint32_t r;
  asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ unsigned long long ld_stream(const unsigned long long* p) {
  unsigned long long r;
  asm("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(r) : "l"(p));
  return r;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Grid-wide barrier for a cooperative (co-resident) launch.  One counter; the
// arrivals sum to 0x80000000 so the top bit flips exactly once per barrier and
// the counter never needs a reset.  Watchdog: if the grid makes no progress
// for 30 s (a CTA never arrives), the waiting CTA sets *abort and leaves the
// barrier; every CTA sees the flag at its next barrier (returns true) and the
// kernel winds down cooperatively, so the host gets an error code instead of
// a sticky device trap that would poison the caller's CUDA context
// (DAWN_DEBUG_TRAP restores the trap for debugging).
__device__ __forceinline__ bool grid_sync(unsigned* bar, unsigned* abort) {
  __shared__ unsigned s_aborted;
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned nb = gridDim.x;
    const unsigned inc = (blockIdx.x == 0) ? (0x80000000u - (nb - 1u)) : 1u;
    __threadfence();
    const unsigned old = atomicAdd(bar, inc);
    unsigned long long t0 = 0;
    unsigned spins = 0, ab = 0;
    while (((old ^ ld_acquire(bar)) & 0x80000000u) == 0u) {
      if ((++spins & 4095u) == 0u) {
        if (ld_acquire(abort)) { ab = 1; break; }
        unsigned long long t = globaltimer();
        if (t0 == 0) t0 = t;
        else if (t - t0 > 30ull * 1000000000ull) {
#ifdef DAWN_DEBUG_TRAP
          asm volatile("trap;");
#endif
          atomicExch(abort, 1u);
          ab = 1;
          break;
        }
      }
    }
    __threadfence();
    s_aborted = ab | ld_acquire(abort);
  }
  __syncthreads();
  return s_aborted != 0u;
}

// ---------------------------------------------------------------------------
// block-wide scans (NT threads)
// ---------------------------------------------------------------------------
template <class T>
__device__ __forceinline__ T warp_incl_sum(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += y;
  }
  return v;
}

// inclusive block sum-scan; `scratch` holds NT/32 elements; returns the
// inclusive prefix and writes the block total to *total (all threads).
template <class T>
__device__ __forceinline__ T block_incl_sum(T v, T* scratch, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T incl = warp_incl_sum(v);
  if (lane == 31) scratch[warp] = incl;
  __syncthreads();
  T pre = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) {
    T x = scratch[w];
    if (w < warp) pre += x;
    tot += x;
  }
  __syncthreads();
  *total = tot;
  return pre + incl;
}

// ---------------------------------------------------------------------------
// persistent-solver state shared by all CTAs (device memory)
// ---------------------------------------------------------------------------
struct DevState {
  unsigned long long res[2];     // packed frontier reservation (count << ebits | edges) per queue
  unsigned long long wround[2];  // nodes lowered in the round with this parity
  unsigned tile_ctr[2];          // dynamic tile counters (relax pass)
  unsigned tile_ctr2[2];         // dynamic tile counters (predecessor pass)
  unsigned sctr[2];              // dense S phase: chunks claimed beyond the first two per CTA, by round parity
  unsigned bar;                  // grid barrier word (never reset)
  unsigned round;                // next round to run (1 = seeding round)
  unsigned dense_prev;           // round-1 recorded its writes densely (stamps only)
  unsigned resume_x;             // stepping: the frontier of `round` is built, resume at its X phase
  unsigned done;
  unsigned flag;                 // negative cycle
  unsigned abort;                // watchdog: the solve made no progress for 30 s and wound down
  unsigned early;                // stopped by the predecessor-cycle check
  unsigned cyc;                  // scratch for the cycle check
  unsigned long long steps;
  unsigned long long R, W, FD, multi;
  // worklist tail (async schedule): ticket counters, one 128-byte line each
  alignas(128) unsigned long long wl_head;  // next ring slot a consumer warp claims (low 32 bits used)
  alignas(128) unsigned long long wl_ctr;   // (items pushed and not yet retired << 32) | next ring slot to reserve
  unsigned long long wl_items;              // items taken (statistics)
  unsigned wl_mode;                         // the persistent kernel handed the solve to dawn_worklist
  unsigned long long wl_batches, wl_busy_ns, wl_wait_ns, wl_t0, wl_t1;  // worklist timeline (sums over warps)
  // near-far schedule (dawn_nearfar): per-round counters, triple-buffered by round
  unsigned long long nf_near[3];    // near rows left for the next round (ring overflow)
  unsigned long long nf_farmin[3];  // smallest key among the far rows left pending (all-ones = none)
  unsigned long long nf_buckets;    // threshold advances (statistics)
};

}  // namespace dawn
