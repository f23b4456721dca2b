// dawn_nearfar.cuh — the near-far schedule for high-diameter, low-degree graphs
// (grids, road-like networks) under schedule="async".
//
// On such graphs the snapshot-Jacobi rounds of govm_sssp (solver.py:356-392)
// rewrite every node hundreds of times: a 4096^2 grid with weights 1..100
// takes 8,503 rounds and relaxes each edge ~195 times (mu in the hundreds),
// and every round pays two grid barriers plus a frontier build.  This kernel
// runs the same relaxation (`cand < dist[v]` => atomicMin, strict `>` as in
// solver.py:298, :373) in a work-efficient order instead:
//
//   * pending rows live in a bitmap (one bit per node).  Round r sweeps the
//     bitmap, takes every set bit (atomicExch of the word) and relaxes the
//     rows whose live distance is below the threshold T ("near"); the others
//     ("far") go back to the bitmap.  When a round ends with no near row
//     pending, T advances to (smallest pending far key) + delta.  This is the
//     near-far / delta-stepping bucket order: a row is relaxed when its value
//     is close to final, so each edge is relaxed ~1-3 times instead of ~195.
//   * a node lowered below T is not written back to the bitmap: the lowering
//     warp appends it to its own FIFO ring in shared memory and relaxes it in
//     the same round (a grid wavefront advances many hops per round, one grid
//     barrier per round instead of two per hop).  Ring overflow and far
//     lowerings set the node's bit.
//   * rows are expanded warp-cooperatively (degree prefix over the batch's
//     rows, owner lane found by a 5-step shuffle search), so a long row costs
//     the same per edge as a short one.
//
// Why the result is the reference's: every candidate is fl(d + w) for a value
// d that dist[u] held, values only decrease, and a node is (re)queued every
// time it is lowered — its bit is set after the returning atomicMin proved the
// write, and a consumer clears the bit before it reads the value — so the run
// stops only at the greatest fixpoint of d[v] = min(d[v], fl(d[u] + w)) that
// the snapshot rounds reach (the async argument).  Graphs with a
// negative weight never take this path (no negative cycles can exist here).
// Counters are this run's own: relaxations = edges of every relaxed row,
// writes = successful lowerings, first_discoveries exact (the unique
// atomicMin that returned INF), nodes lowered twice exact (per-node count of
// re-lowerings, summed in one sweep at the end),
// outer_steps = rounds + 1 (the seeding step, as the reference counts it).
#pragma once
#include "dawn_kernels.cuh"

namespace dawn {

constexpr uint32_t NF_RING = 256;  // per-warp FIFO of near rows (power of two)
constexpr int NF_U = 4;            // 32-edge strides in flight per warp

// next threshold: key(dec(fm) + delta), strictly above fm (float rounding,
// integer saturation), so the row holding fm is near in the next round
template <class V>
__device__ __forceinline__ typename Val<V>::K nf_next_threshold(typename Val<V>::K fm, double delta) {
  using CD = Codec<V, true>;
  using K = typename Val<V>::K;
  K t;
  if constexpr (std::is_floating_point<V>::value) {
    const double x = (double)CD::dec(fm) + delta;
    t = CD::enc((V)x);
  } else {
    const double x = (double)CD::dec(fm) + delta;
    const double cap = (double)(std::is_same<V, int32_t>::value ? 2147483646.0 : 9.0e18);
    t = CD::enc((V)(x < cap ? x : cap));
  }
  return t > fm ? t : fm + 1;
}

template <class V, class EI>
__global__ void __launch_bounds__(NT, DAWN_MIN_BLOCKS) dawn_nearfar(KParams<V, EI> P) {
  using CD = Codec<V, true>;  // no negative weights: raw value bits are order-preserving keys
  using K = typename CD::K;
  using WB = typename CD::WB;
  using C = typename CD::C;
  constexpr uint32_t NONE = 0xFFFFFFFFu;
  __shared__ uint32_t ring_s[WPB][NF_RING];
  DevState* st = P.st;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  uint32_t* ring = ring_s[wid];
  const uint32_t n = P.n, nwords = (n + 31u) >> 5;
  const uint32_t gw = blockIdx.x * WPB + wid, nw = gridDim.x * WPB;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long acc_r = 0, acc_w = 0, acc_fd = 0, acc_multi = 0;

  K T = nf_next_threshold<V>(CD::enc((C)0), P.nf_delta);
  uint32_t head = 0, tail = 0;  // warp-uniform FIFO window [head, tail)
  if (gw == 0) {  // round 1 starts from the source row (seeding, solver.py:212-250)
    if (lane == 0) ring[0] = P.src;
    tail = 1;
  }
  __syncwarp();

  K fmin = CD::INF;     // per lane: smallest key this lane left pending as far
  uint32_t nearc = 0;   // per lane: near rows this lane left pending (ring full)

  // set the pending bit of v (after the atomicMin that lowered it returned)
  auto set_pending = [&](uint32_t v) { atomicOr(P.bmap + (v >> 5), 1u << (v & 31u)); };

  // relax NF_U candidates per lane (no read-before-write filter here, unlike
  // the round kernels: in bucket order most candidates lower their target and
  // the returning min is the test anyway — one dependent access less per hop);
  // lowered targets below T continue in this warp's ring
  auto relax_stride = [&](const uint32_t (&col)[NF_U], const K (&cand)[NF_U], const bool (&ok)[NF_U]) {
    bool push[NF_U];
#pragma unroll
    for (int j = 0; j < NF_U; ++j) {
      push[j] = false;
      if (ok[j]) {
        const K old = atomicMin(P.dist + col[j], cand[j]);
        if (old > cand[j]) {  // this relax lowered dist[v] (strict >, solver.py:298)
          acc_w++;
          if (old == CD::INF) acc_fd++;
          else atomicAdd(P.stamp + col[j], 1u);  // re-lowered (counted once per node at the end)
          if (cand[j] < T) {
            push[j] = true;
          } else {
            set_pending(col[j]);
            fmin = cand[j] < fmin ? cand[j] : fmin;
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NF_U; ++j) {
      const unsigned pm = __ballot_sync(0xffffffffu, push[j]);
      if (pm == 0u) continue;
      const uint32_t space = NF_RING - (tail - head);
      const uint32_t rank = __popc(pm & lt_mask);
      if (push[j]) {
        if (rank < space) {
          ring[(tail + rank) & (NF_RING - 1)] = col[j];
        } else {  // ring full: the next round takes it
          set_pending(col[j]);
          nearc++;
        }
      }
      const uint32_t k = __popc(pm);
      tail += k < space ? k : space;
    }
  };

  // relax the rows of the batch (one node per lane or NONE)
  auto relax_batch = [&](uint32_t u) {
    const bool has = u != NONE;
    K ku = CD::INF;
    EI a = 0, b = 0;
    if (has) {
      ku = ldcg(P.dist + u);  // live value (after the bit was cleared / the ring entry was made)
      a = __ldg(P.row_ptr + u);
      b = __ldg(P.row_ptr + u + 1);
    }
    const bool near = has && ku < T;
    if (has && !near) {  // far: back to the bitmap
      set_pending(u);
      fmin = ku < fmin ? ku : fmin;
    }
    const uint32_t deg = near ? (uint32_t)(b - a) : 0u;
    acc_r += deg;
    const C du = CD::dec(ku);
    if (__all_sync(0xffffffffu, deg <= (uint32_t)NF_U)) {
      // short rows (grids, road networks): each lane streams its own row, no shuffles
      uint32_t col[NF_U];
      K cand[NF_U];
      bool ok[NF_U];
#pragma unroll
      for (int j = 0; j < NF_U; ++j) {
        ok[j] = (uint32_t)j < deg;
        WB w = 0;
        col[j] = 0;
        if (ok[j]) EdgeAccess<V>::load(P, a + (EI)j, col[j], w);
        cand[j] = CD::relax(du, w);
        ok[j] = ok[j] && CD::usable(cand[j]);
      }
      relax_stride(col, cand, ok);
    } else {
      // rows of any length: the batch's edges as one list, 32 * NF_U per pass
      uint32_t incl = deg;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= (uint32_t)d) incl += y;
      }
      const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t ex = incl - deg;
      for (uint32_t base = 0; base < tot; base += 32u * NF_U) {
        uint32_t col[NF_U];
        K cand[NF_U];
        bool ok[NF_U];
#pragma unroll
        for (int j = 0; j < NF_U; ++j) {
          const uint32_t i = base + (uint32_t)j * 32u + lane;
          // owner: the first lane whose inclusive degree prefix exceeds i
          uint32_t lo = 0;
#pragma unroll
          for (uint32_t s = 16; s >= 1; s >>= 1) {
            const uint32_t x = __shfl_sync(0xffffffffu, incl, lo + s - 1);
            if (x <= i) lo += s;
          }
          const EI ea = (EI)__shfl_sync(0xffffffffu, (unsigned long long)a, lo);
          const uint32_t eo = __shfl_sync(0xffffffffu, ex, lo);
          const C d = __shfl_sync(0xffffffffu, du, lo);
          ok[j] = i < tot;
          WB w = 0;
          col[j] = 0;
          if (ok[j]) EdgeAccess<V>::load(P, ea + (EI)(i - eo), col[j], w);
          cand[j] = CD::relax(d, w);
          ok[j] = ok[j] && CD::usable(cand[j]);
        }
        relax_stride(col, cand, ok);
      }
    }
    __syncwarp();
  };

  // relax ring entries until fewer than `keep` are left.  Budget per round:
  // the batches the swept rows need plus P.nf_cap continuation batches (a
  // warp must not walk a whole bucket alone while the others idle: what is
  // left goes back to the bitmap at the end of the round)
  uint32_t rb = 0, swept = gw == 0 ? 1u : 0u;  // (the source row of round 1)
  auto drain = [&](uint32_t keep, bool force) {
    while (tail - head > keep && (force || rb < (swept + 31u) / 32u + P.nf_cap)) {
      ++rb;
      const uint32_t cnt = min(32u, tail - head);
      const uint32_t u = lane < cnt ? ring[(head + lane) & (NF_RING - 1)] : NONE;
      head += cnt;
      __syncwarp();
      relax_batch(u);
    }
  };

  const bool prof = P.prof != nullptr;
  uint32_t r = 1;
  for (;;) {
    const int p = r % 3;
    if (prof && leader && r < P.prof_cap) P.prof[4 * r + 0] = globaltimer();
    if (leader) {  // counters of round r+1; last read after round r-2's barrier
      st->nf_near[(r + 1) % 3] = 0ull;
      st->nf_farmin[(r + 1) % 3] = (unsigned long long)CD::INF;
    }
    // ---- sweep: take every pending row.  A warp owns 128 consecutive words
    // (lane l holds words l, 32+l, 64+l, 96+l: a contiguous run of pending
    // rows spreads over the lanes); its set bits are compacted into the ring
    // 32 at a time (popc prefix + shuffle search + __fns), so batches are full
    // however the bits cluster. ----
    for (uint32_t c = gw; c * 128u < nwords; c += nw) {
      uint32_t wd[4];
#pragma unroll
      for (uint32_t q = 0; q < 4; ++q) {
        const uint32_t wi = c * 128u + q * 32u + lane;
        wd[q] = wi < nwords ? ldcg(P.bmap + wi) : 0u;
      }
#pragma unroll
      for (uint32_t q = 0; q < 4; ++q)
        if (wd[q]) wd[q] = atomicExch(P.bmap + c * 128u + q * 32u + lane, 0u);  // cleared before values are read
#pragma unroll
      for (uint32_t q = 0; q < 4; ++q) {
        const uint32_t pc = __popc(wd[q]);
        uint32_t incl = pc;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
          if (lane >= (uint32_t)d) incl += y;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t ex = incl - pc;
        for (uint32_t s0 = 0; s0 < total; s0 += 32) {
          const uint32_t slot = s0 + lane;
          uint32_t lo = 0;
#pragma unroll
          for (uint32_t sh = 16; sh >= 1; sh >>= 1) {
            const uint32_t x = __shfl_sync(0xffffffffu, incl, lo + sh - 1);
            if (x <= slot) lo += sh;
          }
          const uint32_t word = __shfl_sync(0xffffffffu, wd[q], lo & 31u);
          const uint32_t k = slot - __shfl_sync(0xffffffffu, ex, lo & 31u);
          const uint32_t cnt = min(32u, total - s0);
          if (tail - head > NF_RING - 32u) drain(NF_RING - 32u, true);  // room for 32
          if (lane < cnt)
            ring[(tail + lane) & (NF_RING - 1)] =
                ((c * 128u + q * 32u + lo) << 5) + (uint32_t)__fns(word, 0u, (int)k + 1);
          tail += cnt;
          swept += cnt;
          __syncwarp();
          drain(31, false);  // full batches as they accumulate
        }
      }
    }
    drain(0, false);
    if (prof && r < P.prof_cap && lane == 0) {  // [1] batches (sum), [2] max batches of a warp, [3] swept rows
      atomicAdd(&P.prof[4 * r + 1], (unsigned long long)rb);
      atomicMax(&P.prof[4 * r + 2], (unsigned long long)rb);
      atomicAdd(&P.prof[4 * r + 3], (unsigned long long)swept);
    }
    // ring entries beyond the continuation budget: next round (near)
    for (uint32_t i = head + lane; i < tail; i += 32) {
      set_pending(ring[i & (NF_RING - 1)]);
      nearc++;
    }
    head = tail = 0;
    rb = swept = 0;
    __syncwarp();
    // ---- round counters ----
    {
      K m = fmin;
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        const K y = (K)__shfl_xor_sync(0xffffffffu, (unsigned long long)m, d);
        m = y < m ? y : m;
      }
      const uint32_t nc = __reduce_add_sync(0xffffffffu, nearc);
      if (lane == 0) {
        if (m != CD::INF) atomicMin(&st->nf_farmin[p], (unsigned long long)m);
        if (nc) atomicAdd(&st->nf_near[p], (unsigned long long)nc);
      }
      fmin = CD::INF;
      nearc = 0;
    }
    if (grid_sync(&st->bar, &st->abort)) break;  // watchdog: wind down, the host reports it
    const unsigned long long nearp = ldcg(&st->nf_near[p]);
    const K fm = (K)ldcg(&st->nf_farmin[p]);
    if (nearp == 0ull) {
      if (fm == CD::INF) break;  // nothing pending: the fixpoint
      T = nf_next_threshold<V>(fm, P.nf_delta);
      if (leader) st->nf_buckets++;
    }
    ++r;
  }
  // nodes lowered in >= 2 writes (updated_ratio numerator): stamp counts re-lowerings
  for (uint32_t v = blockIdx.x * NT + threadIdx.x; v < n; v += gridDim.x * NT)
    acc_multi += ldcg(P.stamp + v) != 0u;
  if (leader) {
    st->steps = (unsigned long long)r + 1ull;
    st->round = r + 1;
    st->done = 1u;
  }
  acc_r = warp_sum_u64(acc_r);
  acc_w = warp_sum_u64(acc_w);
  acc_fd = warp_sum_u64(acc_fd);
  acc_multi = warp_sum_u64(acc_multi);
  if (lane == 0) {
    if (acc_r) atomicAdd(&st->R, acc_r);
    if (acc_w) atomicAdd(&st->W, acc_w);
    if (acc_fd) atomicAdd(&st->FD, acc_fd);
    if (acc_multi) atomicAdd(&st->multi, acc_multi);
  }
}

// sum of the edge weights (mean weight -> the auto bucket width), float64 accumulation
template <class V>
__global__ void dawn_weight_sum(const uint2* __restrict__ e2, const unsigned long long* __restrict__ ew, uint64_t m,
                                double* out) {
  double acc = 0.0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    if constexpr (std::is_same<V, int32_t>::value) acc += (double)(int32_t)e2[i].y;
    else if constexpr (std::is_same<V, float>::value) acc += (double)__uint_as_float(e2[i].y);
    else if constexpr (std::is_same<V, int64_t>::value) acc += (double)(long long)ew[i];
    else acc += __longlong_as_double((long long)ew[i]);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

}  // namespace dawn
