// dawn_small.cuh — one thread-block cluster solves a small graph (config 1: RMAT-14).
//
// On a 16 K-node graph the persistent kernel's rounds are latency-bound: two
// grid barriers over every SM, a frontier build and a handful of dependent L2
// accesses per round (~15 us) for a few thousand edges.  This kernel runs the
// same snapshot-Jacobi rounds (solver.py:284-285, :356-395: strict `>` relax,
// round 1 = seeding, cap step < n) inside ONE cluster of CL CTAs (up to 16
// SMs), so a round costs two hardware cluster barriers (~0.2 us):
//
//   * node v is owned by CTA (v ^ mix(v >> cls)) & (CL-1) — a bijection that
//     spreads a skewed graph's hubs (RMAT's heavy nodes share their low bits);
//     the owner keeps v's write state, its round-start distance and the
//     frontier entries of its rows in shared memory;
//   * X: a CTA relaxes the edge list of its own frontier rows (1024 threads,
//     contiguous edge ranges, binary search for the first row then a walk):
//     read-before-write filter on dist[v] in L2 (ld.ca: the cluster barrier
//     invalidates L1, so "cand < cur" still proves v is lowered this round),
//     then a fire-and-forget red.min — no return, no flag;
//   * S: each owner compares its nodes' distances with the round-start copy
//     (lowered = smaller now), does the write bookkeeping, keeps the new copy
//     (the snapshot key of round r+1) and lays out its entries (one block
//     scan, node order); the round's write count is summed in CTA 0 over DSMEM.
//
// Distances live in HBM/L2 (the solver's key array, decoded as usual) and are
// initialised here, so the solve needs no separate begin kernel.  Counters are
// exactly the persistent kernel's (relaxations = edges of the frontier rows,
// writes = (node, round) lowerings, first discoveries, nodes lowered in >= 2
// rounds), so the Jacobi oracle pins them.  Graphs without negative weights
// only (raw-bit keys; the negative-cycle machinery stays in the persistent
// kernel).
#pragma once
#include <cooperative_groups.h>

#include "dawn_kernels.cuh"

namespace dawn {

constexpr int SM_NT = 1024;      // threads per CTA
#ifndef DAWN_SM_NS
#define DAWN_SM_NS 4
#endif
constexpr int SM_NS = DAWN_SM_NS;         // edges in flight per thread in the relax
constexpr int SM_RUN = 4;        // S phase: owned nodes per thread whose row bounds stay in registers
constexpr int SM_MAXCL = 16;      // cluster size (non-portable above 8)

// shared-memory bytes per CTA for n nodes over a cluster of cl CTAs
template <class V, class EI>
__host__ __device__ inline size_t small_smem_bytes(uint32_t n, uint32_t cl) {
  using K = typename Val<V>::K;
  auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
  const size_t nl = (n + cl - 1) / cl;
  return al(sizeof(K) * nl) + al(nl) + al(4 * (nl + 1)) + al(sizeof(EI) * nl) + al(sizeof(K) * nl);
}

// inclusive block scan of a u64 over SM_NT threads; *total = the sum
__device__ __forceinline__ unsigned long long small_scan(unsigned long long v, unsigned long long* wsum,
                                                         unsigned long long* total) {
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= (uint32_t)d) v += y;
  }
  if (lane == 31) wsum[w] = v;
  __syncthreads();
  if (w == 0) {
    unsigned long long x = wsum[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= (uint32_t)d) x += y;
    }
    wsum[lane] = x;
  }
  __syncthreads();
  const unsigned long long r = v + (w ? wsum[w - 1] : 0ull);
  *total = wsum[31];
  __syncthreads();
  return r;
}

template <class V, class EI, bool LIVE>
__global__ void __launch_bounds__(SM_NT, 1) dawn_small(KParams<V, EI> P) {
  namespace cg = cooperative_groups;
  using CD = Codec<V, true>;
  using K = typename CD::K;
  using WB = typename CD::WB;
  using C = typename CD::C;
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t CL = cluster.num_blocks(), me = cluster.block_rank();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ unsigned long long wsum[32];
  __shared__ unsigned long long s_E, s_cnt;
  __shared__ unsigned long long s_wr[2];  // CTA 0: the round's writes over the cluster, by round parity
  auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
  const uint32_t n = P.n;
  const uint32_t nl_max = (n + CL - 1) / CL;                     // layout size (same in every CTA)
  const uint32_t nl = nl_max;  // local slots; node_of(l) >= n marks an unused slot (n not a multiple of CL)
  unsigned char* p = smem_raw;
  K* sd = reinterpret_cast<K*>(p);                 p += al(sizeof(K) * nl_max);  // round-start copy of owned keys
  uint8_t* ws = reinterpret_cast<uint8_t*>(p);     p += al((size_t)nl_max);
  uint32_t* qpre = reinterpret_cast<uint32_t*>(p); p += al(4 * ((size_t)nl_max + 1));
  EI* qrs = reinterpret_cast<EI*>(p);              p += al(sizeof(EI) * (size_t)nl_max);
  K* qkey = reinterpret_cast<K*>(p);               // snapshot key (Jacobi) or node id (async)
  // the owners' arrays, through DSMEM.  CL is a power of two; node v lives at
  // index v >> cls of CTA (v ^ mix(v >> cls)) & (CL-1): a bijection that does
  // not send every low-bit pattern to one CTA (RMAT's heavy nodes share their
  // low bits, so owner = v % CL put the hubs' rows in CTA 0)
  const uint32_t cls = (uint32_t)(__ffs((int)CL) - 1), cm = CL - 1;
  auto owner = [&](uint32_t v) { return (v ^ ((v >> cls) * 0x9E3779B1u >> 16)) & cm; };
  auto node_of = [&](uint32_t l) { return (l << cls) | ((me ^ ((l * 0x9E3779B1u) >> 16)) & cm); };
  unsigned long long* wr0 = cluster.map_shared_rank(s_wr, 0);
  const uint32_t tid = threadIdx.x;
  const bool gsvm = P.algo == 1;
  const uint32_t src = P.src;

  for (uint32_t l = tid; l < nl_max; l += SM_NT) {
    const uint32_t v = node_of(l);
    const K k0 = v == src ? CD::enc((C)0) : CD::INF;
    sd[l] = k0;
    ws[l] = 0;
    if (v < n) P.dist[v] = k0;
  }
  if (tid == 0 && me == 0) {  // the solve state (no begin kernel ran)
    DevState* st = P.st;
    st->R = st->W = st->FD = st->multi = st->steps = 0ull;
    st->flag = st->abort = st->early = 0u;
    st->done = 0u;
  }
  if (tid == 0) {  // round 1's frontier: the source row (seed_source, solver.py:212-250), in its owner
    s_E = s_cnt = 0ull;
    qpre[0] = 0u;
    if (owner(src) == me) {
      const EI a = P.row_ptr[src], b = P.row_ptr[src + 1];
      s_E = (unsigned long long)(b - a);
      s_cnt = b > a ? 1ull : 0ull;
      qpre[1] = (uint32_t)(b - a);
      qrs[0] = a;
      qkey[0] = LIVE ? (K)src : CD::enc((C)0);
    }
    s_wr[0] = s_wr[1] = 0ull;
  }
  // owned nodes of this thread: local indices [l0, l1)
  const uint32_t per = (nl + SM_NT - 1) / SM_NT;
  const uint32_t l0 = min(nl, tid * per), l1 = min(nl, l0 + per);
  const bool inreg = per <= (uint32_t)SM_RUN;
  EI ra[SM_RUN], rb[SM_RUN];
  if (inreg) {
#pragma unroll
    for (int j = 0; j < SM_RUN; ++j) {
      const uint32_t v = node_of(l0 + (uint32_t)j);
      ra[j] = (l0 + (uint32_t)j < l1 && v < n) ? __ldg(P.row_ptr + v) : (EI)0;
      rb[j] = (l0 + (uint32_t)j < l1 && v < n) ? __ldg(P.row_ptr + v + 1) : (EI)0;
    }
  }
  cluster.sync();
  unsigned long long R = 0, Wt = 0, FD = 0, MW = 0;
  uint32_t r = 1, steps = 0;
  bool flag = false;
  const bool prof = P.prof != nullptr && me == 0 && tid == 0;
  for (;; ++r) {
    // ---- X: relax this CTA's frontier rows (edges [0, E) of its list) ----
    const uint32_t E = (uint32_t)s_E, F = (uint32_t)s_cnt;
    if (prof && r < P.prof_cap) {  // timeline (CTA 0): [0] X start [1] S start [2] round end [3] CTA 0's list
      P.prof[4 * r + 0] = globaltimer();
      P.prof[4 * r + 3] = ((unsigned long long)F << P.ebits) | E;
    }
    R += E;
    const uint32_t c = (E + SM_NT - 1) / SM_NT;
    uint32_t i = min(E, tid * c);
    const uint32_t iend = min(E, i + c);
    {
      uint32_t k = 0;
      if (i < iend) {
        uint32_t lo = 0, hi = F;  // last entry with qpre <= i
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (qpre[mid] <= i) lo = mid; else hi = mid;
        }
        k = lo;
      }
      while (__any_sync(0xffffffffu, i < iend)) {  // warp-uniform: the relax step folds across lanes
        EI pos[SM_NS];
        C du[SM_NS];
        uint32_t cnt = 0;
#pragma unroll
        for (int q = 0; q < SM_NS; ++q) {
          if (i < iend) {
            while (qpre[k + 1] <= i) ++k;
            pos[q] = qrs[k] + (EI)(i - qpre[k]);
            if (LIVE) {
              du[q] = CD::dec(ldcg(P.dist + (uint32_t)qkey[k]));
            } else {
              du[q] = CD::dec(qkey[k]);
            }
            ++i;
            ++cnt;
          }
        }
        uint32_t col[SM_NS];
        WB w[SM_NS];
#pragma unroll
        for (int q = 0; q < SM_NS; ++q) {
          col[q] = 0;
          w[q] = 0;
          if ((uint32_t)q < cnt) {
            if constexpr (sizeof(K) == 4) {
              const uint2 x = __ldg(P.e2 + pos[q]);
              col[q] = x.x;
              w[q] = (WB)x.y;
            } else {
              col[q] = __ldg(P.ecol + pos[q]);
              w[q] = (WB)__ldg(P.ew + pos[q]);
            }
          }
        }
        K cur[SM_NS];
#pragma unroll
        for (int q = 0; q < SM_NS; ++q) cur[q] = (uint32_t)q < cnt ? __ldca(P.dist + col[q]) : (K)0;
#pragma unroll
        for (int q = 0; q < SM_NS; ++q) {
          const K cand = CD::relax(du[q], w[q]);
          // strict `>` (solver.py:298, :373); no weight is negative, so the source
          // (key 0) is never undercut and its guard (:299-303) never fires
          if ((uint32_t)q < cnt && CD::usable(cand) && cand < cur[q]) atomicMin(P.dist + col[q], cand);
        }
      }
    }
    cluster.sync();
    if (prof && r < P.prof_cap) P.prof[4 * r + 1] = globaltimer();
    // ---- S: this CTA's writes of round r (bookkeeping) and its round r+1 frontier ----
    auto each = [&](auto&& visit) {  // visit(l, a, b) over the thread's used slots (node_of(l) < n)
      if (inreg) {
#pragma unroll
        for (int j = 0; j < SM_RUN; ++j)
          if (l0 + (uint32_t)j < l1 && node_of(l0 + (uint32_t)j) < n) visit(l0 + (uint32_t)j, ra[j], rb[j]);
      } else {
        for (uint32_t l = l0; l < l1; ++l) {
          const uint32_t v = node_of(l);
          if (v < n) visit(l, __ldg(P.row_ptr + v), __ldg(P.row_ptr + v + 1));
        }
      }
    };
    uint32_t nsel = 0, nw_ = 0;
    unsigned long long deg = 0;
    each([&](uint32_t l, EI a, EI b) {
      const K now = ldcg(P.dist + node_of(l));
      const bool lw = now < sd[l];  // lowered in round r
      if (lw) {
        ++nw_;
        sd[l] = now;
        const uint8_t s = ws[l];
        if (s == 0) { ++FD; ws[l] = 1; }
        else if (s == 1) { ++MW; ws[l] = 2; }
      }
      if ((lw || (gsvm && now != CD::INF)) && b > a) {
        ++nsel;
        deg += (unsigned long long)(b - a);
      }
      // the lowered flag for the second pass: ws bit 7 (cleared there)
      if (lw) ws[l] |= 0x80;
    });
    unsigned long long tot;
    const unsigned long long incl = small_scan(((unsigned long long)nsel << 32) | deg, wsum, &tot);
    const unsigned long long at = incl - (((unsigned long long)nsel << 32) | deg);
    uint32_t pos = (uint32_t)(at >> 32), off = (uint32_t)at;
    each([&](uint32_t l, EI a, EI b) {
      const bool lw = (ws[l] & 0x80) != 0;
      ws[l] &= 0x7F;
      if ((lw || (gsvm && sd[l] != CD::INF)) && b > a) {
        qpre[pos] = off;
        qrs[pos] = a;
        qkey[pos] = LIVE ? (K)node_of(l) : sd[l];
        ++pos;
        off += (uint32_t)(b - a);
      }
    });
    // this CTA's writes into CTA 0's round counter (warp-aggregated)
    const uint32_t wsumw = __reduce_add_sync(0xffffffffu, nw_);
    if ((tid & 31) == 0 && wsumw) atomicAdd(wr0 + (r & 1), (unsigned long long)wsumw);
    __syncthreads();
    if (tid == 0) {
      s_cnt = tot >> 32;
      s_E = tot & 0xFFFFFFFFull;
      qpre[tot >> 32] = (uint32_t)(tot & 0xFFFFFFFFull);
      if (me == 0) s_wr[(r + 1) & 1] = 0ull;  // next round's counter (last read before this round's barrier)
    }
    cluster.sync();
    if (prof && r < P.prof_cap) P.prof[4 * r + 2] = globaltimer();
    const unsigned long long wr = wr0[r & 1];
    Wt += wr;
    // termination (solver.py:284-285, :313-317, :356-358, :388-395)
    if (r >= 2 && wr == 0) { steps = r; break; }
    if (r >= n) { steps = r; flag = wr > 0; break; }
  }
  // results: the keys are already in HBM (decoded by the usual kernel); counters to the solve state
  const unsigned long long fd = warp_sum_u64(FD), mw = warp_sum_u64(MW);
  DevState* st = P.st;
  if ((tid & 31) == 0) {
    if (fd) atomicAdd(&st->FD, fd);
    if (mw) atomicAdd(&st->multi, mw);
  }
  if (tid == 0) atomicAdd(&st->R, R);
  if (tid == 0 && me == 0) {
    st->W = Wt;
    st->steps = steps;
    st->flag = flag ? 1u : 0u;
    st->round = steps + 1;
    st->done = 1u;
  }
  cluster.sync();  // no CTA exits while another may still update CTA 0's shared counter
}

}  // namespace dawn
