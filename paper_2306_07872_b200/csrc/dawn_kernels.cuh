// dawn_kernels.cuh — the persistent weighted-DAWN solver (GOVM + GSVM).
//
// One cooperative launch runs the reference's whole round loop
// (`while step < n`, solver.py:284, :356) on the device with no host sync per
// round.  Round r is two grid-synchronised phases:
//
//   S (frontier build): the frontier of round r — the nodes lowered in round
//      r-1 (Alg. 2's "Copy beta to delta") or, for GSVM,
//      every finite node (solver.py:287-289) — is laid out as entries
//      {node, edge offset, row base, snapshot key}.  The snapshot key gives
//      frontier-synchronous (snapshot-Jacobi) semantics: every relax of round
//      r reads its row's distance as of the start of round r.  S also marks,
//      for every TILE-edge tile of the frontier's virtual edge list, the entry
//      owning the tile's first edge.  Two ways to build it:
//        dense  — a coalesced sweep over all nodes selecting stamp == r-1
//                 (after a heavy round; also counts that round's writes);
//        sparse — snapshot of the queue the X phase filled (after a light round).
//   X (expand): persistent CTAs stream the tiles (merge-path load balance:
//      a hub row of 10^5 edges and a 1-edge row cost the same per edge), find
//      each edge's row by a max-scan over row-start marks, stream the packed
//      (col, w) pairs, and relax:
//          cur = dist[v] (ld.cg, coherent at L2)
//          cand < cur  =>  v WILL be lowered this round, so
//          red.min(dist[v], cand) needs no return value, and the write stamp
//          stamp[v] = r is a plain store (dense) or an atomic exchange whose
//          old value elects the one thread that enqueues v (sparse).
//      The reference's strict `>` (solver.py:298, :373) is `cand < cur` on the
//      order-preserving key; the source guard (solver.py:299-303) flags.
//
// Optional passes: predecessors (record_pred) and the predecessor-graph
// cycle check (integer weights with negative edges).
#pragma once
#include "dawn_device.cuh"

namespace dawn {

template <class V, class EI>
struct KParams {
  using K = typename Val<V>::K;
  uint32_t n;
  uint32_t src;
  const EI* row_ptr;
  const uint2* e2;                     // packed {col, wbits} for 4-byte value types
  const uint32_t* ecol;                // SoA columns for 8-byte value types
  const unsigned long long* ew;        // SoA weights for 8-byte value types
  K* dist;
  uint32_t* stamp;                     // last round that lowered the node (0 = never)
  uint32_t* bmap;                      // bitmap-frontier kernels: nodes lowered in a light round, 1 bit each
  uint8_t* wstate;                     // 0 never lowered, 1 lowered in one round, 2 in >= 2
  unsigned long long* pred;            // (round << 32) | ~u, or nullptr
  uint32_t* jmp0;
  uint32_t* jmp1;
  uint32_t* qnode[2];
  EI* qoff[2];
  EI* qbase[2];                        // row_start - off, so edge position = base + e
  K* qkey[2];
  uint32_t* tile_row;
  DevState* st;
  int algo;                            // 0 = GOVM, 1 = GSVM
  int pred_on;
  int negcheck_period;                 // 0 = off
  int logn;                            // ceil(log2(n))
  int ebits;                           // packed reservation split
  unsigned max_rounds;
  unsigned long long dense_edges;      // a round relaxing >= this many edges builds the next frontier densely
  unsigned long long* prof;            // optional per-round timeline (4 words/round) or nullptr
  unsigned prof_cap;                   // rounds the timeline can hold
  unsigned long long* cta_prof;        // debug: per-CTA S/X work end times [round][2][grid], or nullptr
  int live;                            // async schedule: frontier rows relaxed with their live value (no snapshot)
  int skip_if_done;                    // speculative negative-weight solves: return at once if a previous
                                       // launch already finished the solve (see Impl::run)
  // worklist tail (async schedule, non-negative weights, unbounded run): once a
  // round relaxes < wl_edges edges the rest of the solve runs barrier-free
  unsigned long long* wl_ring;         // ring of 16-byte row items (uint4); nullptr = off
  unsigned long long wl_mask;          // ring capacity - 1 (power of two)
  unsigned long long wl_edges;
  // priority window (async GOVM, non-negative 4-byte values, unbounded run): a
  // heavy round relaxes only the frontier rows whose live value lies in the
  // lowest pw_frac of the frontier's edges (degree-weighted histogram built by
  // the dense S phase); the others are deferred to the next round
  int pw;                              // on for this run
  float pw_frac;
  unsigned long long pw_edges;         // rounds relaxing >= this many edges apply the window
  unsigned long long pw_seed_edges;    // a seeding round relaxing >= this many edges records its writes
                                       // densely, so round 2 is histogrammed and windowed too
  uint32_t* phist;                     // [2][PW_BINS] degree-weighted value histograms, by round parity
  double nf_delta;                     // near-far schedule: bucket width in weight units (dawn_nearfar.cuh)
  uint32_t nf_cap;                     // near-far: continuation batches a warp may run per round
};

constexpr int WPB = NT / 32;       // warps per CTA
// Virtual edges per lane of a warp tile in the X phase (template XI): as many
// independent edge loads + dist gathers in flight per lane as the 128-register
// budget holds without spilling.  Two widths are instantiated for 4-byte
// values: XI_WIDE (14, best of 8/10/12/14/16 on C2) for graphs with heavy
// rounds, 8 otherwise (the grid and small graphs prefer more, smaller tiles;
// profiles/r01_experiments.md).  8-byte values always use 8.
#ifndef DAWN_XITEMS_WIDE
#define DAWN_XITEMS_WIDE 14
#endif
constexpr int XI_NARROW = 8;
constexpr unsigned CTA_PROF_ROUNDS = 64;  // rounds of the per-CTA debug timeline
constexpr int XI_WIDE = DAWN_XITEMS_WIDE;
constexpr int WT_MIN = 32 * (XI_NARROW < XI_WIDE ? XI_NARROW : XI_WIDE);

// Per-warp shared memory is only the row-start marks of a short-row tile
// (512 B): everything else stays in registers or is read through L1, so the
// shared-memory carveout stays minimal and L1 keeps ~200 KB for dist[] gathers.
template <int XI>
struct __align__(16) WarpRows {
  uint16_t mark[32 * XI];       // row-start marks -> per-edge row index (max-scan)
};

template <class V, class EI, int XI>
struct __align__(16) Smem {
  WarpRows<XI> w[WPB];
  unsigned long long scr64[WPB];
  unsigned long long basepk;
  uint32_t claim[2];  // dense S phase: the chunk after next (double-buffered by iteration)
  uint32_t pw_tb;     // priority window: last histogram bin relaxed this round
};

// Priority window helpers.  A value's bin is the top 11 bits of its float32
// representation (exponent + 2 mantissa bits: bins ~19 % wide), monotone for
// the non-negative values the window runs on.  A deferred frontier row keeps
// stamp (r | STAMP_DEFER): the next dense S phase selects it again without
// counting it as a write of round r.
constexpr int PW_BINS = 1024;
constexpr uint32_t STAMP_DEFER = 0x80000000u;
template <class C>
__device__ __forceinline__ uint32_t pw_bin(C v) {
  const uint32_t b = __float_as_uint((float)v) >> 21;
  return b < (uint32_t)PW_BINS ? b : (uint32_t)(PW_BINS - 1);
}
template <class V, class K>
__device__ __forceinline__ uint32_t pw_bin_key(K key) {  // raw (non-negative) keys only
  if constexpr (std::is_same<V, float>::value) return pw_bin(__uint_as_float((uint32_t)key));
  else if constexpr (std::is_same<V, double>::value) return pw_bin(__longlong_as_double((long long)key));
  else return pw_bin((V)key);
}

template <class V> struct EdgeAccess;
template <> struct EdgeAccess<int32_t> {  // 4-byte value types: one 8-byte load per edge
  template <class P, class EI> __device__ __forceinline__ static void load(const P& p, EI pos, uint32_t& c, uint32_t& w) {
    uint2 x = ld_stream(p.e2 + pos); c = x.x; w = x.y;
  }
};
template <> struct EdgeAccess<float> {
  template <class P, class EI> __device__ __forceinline__ static void load(const P& p, EI pos, uint32_t& c, uint32_t& w) {
    uint2 x = ld_stream(p.e2 + pos); c = x.x; w = x.y;
  }
};
template <> struct EdgeAccess<int64_t> {
  template <class P, class EI> __device__ __forceinline__ static void load(const P& p, EI pos, uint32_t& c, unsigned long long& w) {
    c = ld_stream(p.ecol + pos); w = ld_stream(p.ew + pos);
  }
};
template <> struct EdgeAccess<double> {
  template <class P, class EI> __device__ __forceinline__ static void load(const P& p, EI pos, uint32_t& c, unsigned long long& w) {
    c = ld_stream(p.ecol + pos); w = ld_stream(p.ew + pos);
  }
};

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

__device__ __forceinline__ unsigned long long pk_count(unsigned long long pk, int ebits) { return pk >> ebits; }
__device__ __forceinline__ unsigned long long pk_edges(unsigned long long pk, int ebits) {
  return pk & ((1ull << ebits) - 1ull);
}

// mark the warp tiles whose first virtual edge falls inside [off, off + deg)
template <int XI, class EI>
__device__ __forceinline__ void mark_tiles(uint32_t* tile_row, EI off, EI deg, uint32_t entry) {
  constexpr int WT = 32 * XI;
  EI t0 = (off + (EI)(WT - 1)) / (EI)WT;
  EI t1 = (off + deg - 1) / (EI)WT;
  for (EI t = t0; t <= t1; ++t) tile_row[t] = entry;
}

// Warp-collective mark_tiles (every lane calls it; `has` = this lane has a row):
// short rows are marked by their lane, rows spanning >= 32 tiles by the whole
// warp.  Used by the batched kernel, whose 32-edge tiles make a hub row
// (10^5 edges = thousands of tiles) hold one thread — and its CTA, and the
// grid barrier behind it — for ~10 us.  (The single-source S phases keep the
// per-lane loop: their tiles are 8-14x wider and the warp vote cost more
// than it saved on config 2.)
template <int WT, class EI>
__device__ __forceinline__ void mark_tiles_warp(uint32_t* tile_row, bool has, EI off, EI deg, uint32_t entry) {
  EI t0 = 0, t1 = 0;
  bool lng = false;
  if (has && deg > 0) {
    t0 = (off + (EI)(WT - 1)) / (EI)WT;
    t1 = (off + deg - 1) / (EI)WT;
    if (t1 >= t0 + (EI)32) lng = true;
    else
      for (EI t = t0; t <= t1; ++t) tile_row[t] = entry;
  }
  unsigned lm = __ballot_sync(0xffffffffu, lng);
  const uint32_t lane = threadIdx.x & 31;
  while (lm) {
    const int L = __ffs(lm) - 1;
    lm &= lm - 1u;
    const EI a = (EI)__shfl_sync(0xffffffffu, (unsigned long long)t0, L);
    const EI b = (EI)__shfl_sync(0xffffffffu, (unsigned long long)t1, L);
    const uint32_t e = __shfl_sync(0xffffffffu, entry, L);
    for (EI t = a + (EI)lane; t <= b; t += (EI)32) tile_row[t] = e;
  }
}

// ---------------------------------------------------------------------------
// S phase, sparse: snapshot the queue the previous X phase built
// ---------------------------------------------------------------------------
template <class V, class EI, int XI>
__device__ void phase_snapshot(const KParams<V, EI>& P, int p) {
  const unsigned long long pk = ldcg(&P.st->res[p]);
  const uint32_t cnt = (uint32_t)pk_count(pk, P.ebits);
  const EI E = (EI)pk_edges(pk, P.ebits);
  const uint32_t* qn = P.qnode[p];
  const EI* qo = P.qoff[p];
  for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < cnt; i += gridDim.x * NT) {
    const uint32_t u = ldcg(qn + i);
    if (!P.live) P.qkey[p][i] = ldcg(P.dist + u);  // the async schedule reads live values instead
    const EI off = ldcg(qo + i);
    const EI nxt = (i + 1 < cnt) ? ldcg(qo + i + 1) : E;
    mark_tiles<XI, EI>(P.tile_row, off, nxt - off, i);
  }
}

// ---------------------------------------------------------------------------
// S phase, dense: one coalesced sweep over all nodes.  Counts round r-1's
// writes (stamp == r-1) and selects GOVM's frontier (those nodes) or GSVM's
// (every finite node, solver.py:287-289).  Each thread owns ITEMS consecutive
// nodes and reads them with 128-bit loads; one packed block scan
// (count << ebits | degree) places the chunk's entries.
// ---------------------------------------------------------------------------
template <class T>
__device__ __forceinline__ void ldcg8(const T* p, T (&o)[ITEMS]) {
  static_assert(ITEMS == 8, "vector loads assume 8 items");
  if constexpr (sizeof(T) == 4) {
    const uint4 a = __ldcg(reinterpret_cast<const uint4*>(p));
    const uint4 b = __ldcg(reinterpret_cast<const uint4*>(p) + 1);
    o[0] = (T)a.x; o[1] = (T)a.y; o[2] = (T)a.z; o[3] = (T)a.w;
    o[4] = (T)b.x; o[5] = (T)b.y; o[6] = (T)b.z; o[7] = (T)b.w;
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const ulonglong2 a = __ldcg(reinterpret_cast<const ulonglong2*>(p) + q);
      o[2 * q] = (T)a.x; o[2 * q + 1] = (T)a.y;
    }
  }
}
template <class T>
__device__ __forceinline__ void ldg8(const T* p, T (&o)[ITEMS]) {
  if constexpr (sizeof(T) == 4) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(p));
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(p) + 1);
    o[0] = (T)a.x; o[1] = (T)a.y; o[2] = (T)a.z; o[3] = (T)a.w;
    o[4] = (T)b.x; o[5] = (T)b.y; o[6] = (T)b.z; o[7] = (T)b.w;
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(p) + q);
      o[2 * q] = (T)a.x; o[2 * q + 1] = (T)a.y;
    }
  }
}

template <class V, class EI, int XI>
__device__ void phase_compact(const KParams<V, EI>& P, int p, uint32_t r, Smem<V, EI, XI>& s,
                              unsigned long long& acc_w, unsigned long long& acc_fd,
                              unsigned long long& acc_multi, uint32_t& prev_w, uint32_t tb = 0xFFFFFFFFu) {
  using VT = Val<V>;
  using K = typename VT::K;
  const uint32_t n = P.n;
  const uint32_t nchunks = (n + TILE - 1) / TILE;
  const bool gsvm = P.algo == 1;
  const int eb = P.ebits;
  // keys: the snapshot values (Jacobi) and GSVM's finite test; the async schedule's GOVM needs neither
  const bool need_keys = gsvm || !P.live || tb != 0xFFFFFFFFu;
  // Everything a chunk needs — stamps, write states, keys, row bounds — is
  // loaded one iteration ahead, unconditionally: a CTA walks ~7 chunks per
  // phase and a per-chunk chain of dependent loads (stamps -> keys/rows/state)
  // cost ~1.5 us each (timeline in profiles/r01_experiments.md).  The extra
  // bytes (keys and row bounds of chunks without writes) are L2 reads of
  // arrays the round touches anyway.
  struct Pre {
    uint32_t st[ITEMS];
    K keys[ITEMS];
    EI rp[ITEMS + 1];
    uint2 ws;
  };
  auto load_chunk = [&](uint32_t c, Pre& o) {
    const uint32_t u = c * TILE + threadIdx.x * ITEMS;
    if (u + ITEMS <= n) {
      ldcg8<uint32_t>(P.stamp + u, o.st);
      if (need_keys) ldcg8<K>(P.dist + u, o.keys);
      else {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) o.keys[j] = (K)0;  // GOVM + live rows: a stamped node is finite
      }
      ldg8<EI>(P.row_ptr + u, *reinterpret_cast<EI(*)[ITEMS]>(o.rp));
      o.rp[ITEMS] = __ldg(P.row_ptr + u + ITEMS);
      o.ws = __ldcg(reinterpret_cast<const uint2*>(P.wstate + u));
    } else {
      uint8_t* b = reinterpret_cast<uint8_t*>(&o.ws);
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        o.st[j] = (u + j < n) ? ldcg(P.stamp + u + j) : 0u;
        o.keys[j] = (u + j < n) ? (need_keys ? ldcg(P.dist + u + j) : (K)0) : VT::INF;
        o.rp[j] = (u + j <= n) ? __ldg(P.row_ptr + u + j) : (EI)0;
        b[j] = (u + j < n) ? ldcg(P.wstate + u + j) : (uint8_t)0;
      }
      o.rp[ITEMS] = (u + ITEMS <= n) ? __ldg(P.row_ptr + u + ITEMS) : (EI)0;
    }
  };
  // Chunks: the first two per CTA are static (blockIdx.x, + gridDim.x), the
  // rest are claimed from a counter one chunk ahead of the prefetch, so CTAs
  // that drew cheap chunks take more (a hub chunk costs ~3x a typical one;
  // static striding left the slowest CTA ~40 % behind the median).
  Pre nx;
  uint32_t c = blockIdx.x, cn = blockIdx.x + gridDim.x;
  if (c < nchunks) load_chunk(c, nx);
  for (uint32_t it = 0; c < nchunks; ++it) {
    const uint32_t u0 = c * TILE + threadIdx.x * ITEMS;
    const Pre cur = nx;
    if (cn < nchunks) load_chunk(cn, nx);
    uint32_t claim = nchunks;  // issued now, consumed (stored) only before the last barrier below
    if (threadIdx.x == 0 && cn < nchunks) claim = 2u * gridDim.x + atomicAdd(&P.st->sctr[p], 1u);
    const K (&keys)[ITEMS] = cur.keys;
    const EI (&rp)[ITEMS + 1] = cur.rp;
    const bool full = u0 + ITEMS <= n;
    unsigned wm = 0, dm = 0;  // lowered in round r-1 / deferred by it (priority window)
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) wm |= (unsigned)(cur.st[j] == r - 1 && u0 + j < n) << j;
    if (P.pw) {
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) dm |= (unsigned)(cur.st[j] == ((r - 1) | STAMP_DEFER) && u0 + j < n) << j;
    }
    const unsigned want = gsvm ? ((u0 < n) ? 0xFFu : 0u) : (wm | dm);
    unsigned sel = 0, dfr = 0;
    uint32_t mycnt = 0;
    EI mydeg = 0;
    if (want) {
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        if (((want >> j) & 1u) && u0 + j < n && keys[j] != VT::INF && rp[j + 1] > rp[j]) {
          if (tb != 0xFFFFFFFFu && pw_bin_key<V>(keys[j]) > tb) {
            dfr |= 1u << j;  // priority window: relaxed in a later round
          } else {
            sel |= 1u << j;
            mycnt++;
            mydeg += rp[j + 1] - rp[j];
          }
        }
      }
      if (dfr) {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j)
          if ((dfr >> j) & 1u) P.stamp[u0 + j] = r | STAMP_DEFER;
      }
    }
    // write bookkeeping for round r-1 (first_discoveries, >= 2-round nodes)
    if (wm) {
      uint2 ws = cur.ws;
      uint8_t* b = reinterpret_cast<uint8_t*>(&ws);
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        if ((wm >> j) & 1u) {
          prev_w++;
          acc_w++;
          if (b[j] == 0) { acc_fd++; b[j] = 1; }
          else if (b[j] == 1) { acc_multi++; b[j] = 2; }
        }
      }
      if (full) *reinterpret_cast<uint2*>(P.wstate + u0) = ws;
      else {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j)
          if (u0 + j < n) P.wstate[u0 + j] = b[j];
      }
    }
    // place the chunk's entries: one packed scan, one reservation
    const unsigned long long mine = ((unsigned long long)mycnt << eb) | (unsigned long long)mydeg;
    unsigned long long tot;
    const unsigned long long incl = block_incl_sum<unsigned long long>(mine, s.scr64, &tot);
    if (threadIdx.x == 0) {
      if (tot != 0ull) s.basepk = atomicAdd(&P.st->res[p], tot);
      s.claim[it & 1] = claim;
    }
    __syncthreads();
    if (sel) {
      const unsigned long long at = s.basepk + incl - mine;
      uint32_t pos = (uint32_t)pk_count(at, eb);
      EI off = (EI)pk_edges(at, eb);
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        if (sel & (1u << j)) {
          const EI deg = rp[j + 1] - rp[j];
          P.qnode[p][pos] = u0 + j;
          P.qoff[p][pos] = off;
          P.qbase[p][pos] = rp[j] - off;
          if (!P.live) P.qkey[p][pos] = keys[j];
          mark_tiles<XI, EI>(P.tile_row, off, deg, pos);
          pos++;
          off += deg;
        }
      }
    }
    c = cn;
    cn = s.claim[it & 1];  // written before this iteration's barriers
  }
}

// Priority window, first pass of a heavy round's S phase: the degree-weighted
// histogram of the frontier's values (rows lowered or deferred in round r-1).
template <class V, class EI, int XI>
__device__ void phase_hist(const KParams<V, EI>& P, int p, uint32_t r, Smem<V, EI, XI>& s) {
  using K = typename Val<V>::K;
  uint32_t* hist = reinterpret_cast<uint32_t*>(&s.w[0]);  // the S phase does not use the warp marks
  static_assert(sizeof(s.w) >= PW_BINS * sizeof(uint32_t), "histogram overlays the warp marks");
  for (int i = threadIdx.x; i < PW_BINS; i += NT) hist[i] = 0u;
  __syncthreads();
  const uint32_t n = P.n;
  const uint32_t nchunks = (n + TILE - 1) / TILE;
  for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint32_t u0 = c * TILE + threadIdx.x * ITEMS;
    if (u0 >= n) continue;
    uint32_t st[ITEMS];
    K keys[ITEMS];
    EI rp[ITEMS + 1];
    if (u0 + ITEMS <= n) {
      ldcg8<uint32_t>(P.stamp + u0, st);
      ldcg8<K>(P.dist + u0, keys);
      ldg8<EI>(P.row_ptr + u0, *reinterpret_cast<EI(*)[ITEMS]>(rp));
      rp[ITEMS] = __ldg(P.row_ptr + u0 + ITEMS);
    } else {
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        st[j] = (u0 + j < n) ? ldcg(P.stamp + u0 + j) : 0u;
        keys[j] = (u0 + j < n) ? ldcg(P.dist + u0 + j) : (K)0;
        rp[j] = (u0 + j <= n) ? __ldg(P.row_ptr + u0 + j) : (EI)0;
      }
      rp[ITEMS] = (u0 + ITEMS <= n) ? __ldg(P.row_ptr + u0 + ITEMS) : (EI)0;
    }
#pragma unroll
    for (int j = 0; j < ITEMS; ++j)
      if ((st[j] & ~STAMP_DEFER) == r - 1 && u0 + j < n && rp[j + 1] > rp[j])
        atomicAdd(hist + pw_bin_key<V>(keys[j]), (uint32_t)(rp[j + 1] - rp[j]));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < PW_BINS; i += NT)
    if (hist[i]) atomicAdd(P.phist + (size_t)p * PW_BINS + i, hist[i]);
}

// Priority window: the last bin of round r's histogram inside the lowest
// pw_frac of its (degree-weighted) mass.  Every thread of the CTA calls it.
template <class V, class EI, int XI>
__device__ uint32_t pw_threshold(const KParams<V, EI>& P, int p, Smem<V, EI, XI>& s) {
  constexpr int BPT = PW_BINS / NT;
  static_assert(PW_BINS % NT == 0, "bins per thread");
  const uint32_t* h = P.phist + (size_t)p * PW_BINS + threadIdx.x * BPT;
  uint32_t b[BPT];
  unsigned long long mine = 0;
#pragma unroll
  for (int i = 0; i < BPT; ++i) { b[i] = ldcg(h + i); mine += b[i]; }
  unsigned long long tot;
  const unsigned long long incl = block_incl_sum<unsigned long long>(mine, s.scr64, &tot);
  const unsigned long long want = (unsigned long long)((double)P.pw_frac * (double)tot);
  unsigned long long run = incl - mine;
  if (threadIdx.x == 0) s.pw_tb = tot >= P.pw_edges ? PW_BINS - 1 : 0xFFFFFFFFu;  // light frontier: no window
  __syncthreads();
  if (tot >= P.pw_edges && run < want && incl >= want) {  // exactly one thread holds the crossing
#pragma unroll
    for (int i = 0; i < BPT; ++i) {
      run += b[i];
      if (run >= want) { s.pw_tb = threadIdx.x * BPT + i; break; }
    }
  }
  __syncthreads();
  return s.pw_tb;
}

// ---------------------------------------------------------------------------
// S phase after a light round, bitmap-frontier kernels (low-degree graphs such
// as the grid, where a light round lowers ~25% of the nodes it touches and the
// enqueue path's election + reservation chain per write dominates).  A warp
// takes 128 bitmap words (4096 nodes), spreads their set bits evenly over its
// lanes (popc prefix + per-lane search + __fns), does the write bookkeeping,
// sizes its entries, reserves them with ONE atomic and writes them (a second
// pass re-derives the same slots; the first two slots per lane are kept).
// ---------------------------------------------------------------------------
#ifndef DAWN_BITMAP_SLOTS
#define DAWN_BITMAP_SLOTS 2
#endif
template <class V, class EI, int XI>
__device__ void phase_bitmap(const KParams<V, EI>& P, int p, uint32_t r, unsigned long long& acc_w,
                             unsigned long long& acc_fd, unsigned long long& acc_multi, uint32_t& prev_w) {
  using K = typename Val<V>::K;
  constexpr int SL = DAWN_BITMAP_SLOTS;  // slots per lane per iteration
  constexpr uint32_t WPL = 4;        // bitmap words per lane (one 16-byte load)
  constexpr uint32_t CW = 32 * WPL;  // words per warp chunk
  const uint32_t n = P.n;
  const uint32_t nwords = (n + 31u) >> 5;
  const uint32_t nchunks = (nwords + CW - 1) / CW;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (NT / 32);
  const int eb = P.ebits;
  auto load_words = [&](uint32_t c, uint4& w4) {
    const uint32_t w0 = c * CW + lane * WPL;
    if (w0 + WPL <= nwords) {
      w4 = __ldcg(reinterpret_cast<const uint4*>(P.bmap + w0));
    } else {
      w4.x = (w0 + 0 < nwords) ? ldcg(P.bmap + w0 + 0) : 0u;
      w4.y = (w0 + 1 < nwords) ? ldcg(P.bmap + w0 + 1) : 0u;
      w4.z = (w0 + 2 < nwords) ? ldcg(P.bmap + w0 + 2) : 0u;
      w4.w = (w0 + 3 < nwords) ? ldcg(P.bmap + w0 + 3) : 0u;
    }
  };
  uint32_t c = blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
  uint4 nxt = make_uint4(0, 0, 0, 0);
  if (c < nchunks) load_words(c, nxt);
  for (; c < nchunks; c += nwarps) {
    const uint4 w4 = nxt;
    if (c + nwarps < nchunks) load_words(c + nwarps, nxt);  // prefetch the next chunk
    const uint32_t any = w4.x | w4.y | w4.z | w4.w;
    if (!__any_sync(0xffffffffu, any != 0u)) continue;
    const uint32_t w0 = c * CW + lane * WPL;
    if (any) {  // consumed: the next light round sets bits again
      if (w0 + WPL <= nwords) *reinterpret_cast<uint4*>(P.bmap + w0) = make_uint4(0, 0, 0, 0);
      else
        for (uint32_t q = 0; q < WPL; ++q)
          if (w0 + q < nwords) P.bmap[w0 + q] = 0u;
    }
    const uint32_t pc = __popc(w4.x) + __popc(w4.y) + __popc(w4.z) + __popc(w4.w);
    uint32_t incl = pc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= (uint32_t)d) incl += y;
    }
    const uint32_t excl = incl - pc;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    auto slot_node = [&](uint32_t sl) -> uint32_t {
      uint32_t lo = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const uint32_t x = __shfl_sync(0xffffffffu, excl, (lo + step) & 31);
        if (lo + step < 32u && x <= sl) lo += step;
      }
      uint32_t k = sl - __shfl_sync(0xffffffffu, excl, lo);
      const uint32_t a0 = __shfl_sync(0xffffffffu, w4.x, lo), a1 = __shfl_sync(0xffffffffu, w4.y, lo);
      const uint32_t a2 = __shfl_sync(0xffffffffu, w4.z, lo), a3 = __shfl_sync(0xffffffffu, w4.w, lo);
      uint32_t wd = a0, q = 0;
      const uint32_t c0 = __popc(a0), c1 = __popc(a1), c2 = __popc(a2);
      if (k >= c0) { k -= c0; wd = a1; q = 1; if (k >= c1) { k -= c1; wd = a2; q = 2; if (k >= c2) { k -= c2; wd = a3; q = 3; } } }
      return ((c * CW + lo * WPL + q) << 5) + (uint32_t)__fns(wd, 0, (int)k + 1);
    };
    // ---- pass A: bookkeeping of round r-1's writes; size this lane's entries.
    // Two slots per lane per iteration (more loads in flight); the first
    // iteration's slots are kept for pass B. ----
    unsigned long long mine = 0;  // (entries << eb) | edges
    uint32_t kv[SL];
    EI ka[SL], kb[SL];
#pragma unroll
    for (int h = 0; h < SL; ++h) { kv[h] = 0; ka[h] = 0; kb[h] = 0; }
    for (uint32_t s0 = 0, it = 0; s0 < total; s0 += 32 * SL, ++it) {
      uint32_t vv[SL];
      EI aa[SL], bb[SL];
      uint8_t ww[SL];
#pragma unroll
      for (int h = 0; h < SL; ++h) {
        const uint32_t sl = s0 + 32 * h + lane;
        vv[h] = slot_node(sl < total ? sl : total - 1);
      }
#pragma unroll
      for (int h = 0; h < SL; ++h) {
        ww[h] = ldcg(P.wstate + vv[h]);
        aa[h] = __ldg(P.row_ptr + vv[h]);
        bb[h] = __ldg(P.row_ptr + vv[h] + 1);
      }
#pragma unroll
      for (int h = 0; h < SL; ++h) {
        const uint32_t sl = s0 + 32 * h + lane;
        if (sl < total) {
          const uint32_t v = vv[h];
          prev_w++;
          acc_w++;
          if (ww[h] == 0) { acc_fd++; P.wstate[v] = 1; }
          else if (ww[h] == 1) { acc_multi++; P.wstate[v] = 2; }
          P.stamp[v] = r - 1;
          if (bb[h] > aa[h]) mine += (1ull << eb) + (unsigned long long)(bb[h] - aa[h]);
          if (it == 0) { kv[h] = v; ka[h] = aa[h]; kb[h] = bb[h]; }
        }
      }
    }
    unsigned long long pre = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, pre, d);
      if (lane >= (uint32_t)d) pre += y;
    }
    const unsigned long long tot = __shfl_sync(0xffffffffu, pre, 31);
    if (tot == 0ull) continue;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&P.st->res[p], tot);
    base = __shfl_sync(0xffffffffu, base, 0);
    const unsigned long long at = base + pre - mine;
    uint32_t pos = (uint32_t)pk_count(at, eb);
    EI off = (EI)pk_edges(at, eb);
    // ---- pass B: write the entries (the same slots in the same order) ----
    for (uint32_t s0 = 0, it = 0; s0 < total; s0 += 32 * SL, ++it) {
      uint32_t vv[SL];
      EI aa[SL], bb[SL];
      K kk[SL];
#pragma unroll
      for (int h = 0; h < SL; ++h) {
        const uint32_t sl = s0 + 32 * h + lane;
        if (it == 0) {
          vv[h] = kv[h];
          aa[h] = ka[h];
          bb[h] = kb[h];
        } else {
          vv[h] = slot_node(sl < total ? sl : total - 1);
          aa[h] = __ldg(P.row_ptr + vv[h]);
          bb[h] = __ldg(P.row_ptr + vv[h] + 1);
        }
        kk[h] = ldcg(P.dist + vv[h]);
      }
#pragma unroll
      for (int h = 0; h < SL; ++h) {
        const uint32_t sl = s0 + 32 * h + lane;
        if (sl < total && bb[h] > aa[h]) {
          P.qnode[p][pos] = vv[h];
          P.qoff[p][pos] = off;
          P.qbase[p][pos] = aa[h] - off;
          if (!P.live) P.qkey[p][pos] = kk[h];
          mark_tiles<XI, EI>(P.tile_row, off, bb[h] - aa[h], pos);
          pos++;
          off += bb[h] - aa[h];
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// X phase: warp tiles of the frontier's virtual edge list.
//   PRED == false : relax (+ enqueue when !dense)
//   PRED == true  : predecessor pass — among this round's frontier edges that
//                   reproduce the final value of a node lowered this round,
//                   keep the smallest source node (deterministic witness).
// Every warp owns whole WT-edge tiles (t = global warp id + k * total warps;
// all tiles have WT edges) and never waits for another warp.
// Row lookup: a tile with <= 32 frontier rows keeps row k in lane k's
// registers; for each 32-edge window one OR-reduction of row-start bits plus a
// popc gives every lane its row, and shuffles fetch the row's base and value
// (no shared memory, no scan).  Tiles with more rows (short rows) use
// row-start marks in shared memory and a warp max-scan.
// Software pipeline: while tile t streams, the first 32 rows of the warp's
// next tile and the row range of the one after are in flight.
// ---------------------------------------------------------------------------
constexpr uint32_t SENT = 0xFFFFFFFFu;

template <class V, class EI, bool PRED, bool RAW, int XI, bool FB = false>
__device__ void phase_expand(const KParams<V, EI>& P, int p, uint32_t r, bool dense, Smem<V, EI, XI>& s,
                             unsigned long long& acc_w, unsigned long long& acc_fd,
                             unsigned long long& acc_multi, uint32_t& round_w) {
  using CD = Codec<V, RAW>;
  using K = typename CD::K;
  using WB = typename CD::WB;
  using C = typename CD::C;
  constexpr int WT = 32 * XI;
  const unsigned long long pk = ldcg(&P.st->res[p]);
  const uint32_t cnt = (uint32_t)pk_count(pk, P.ebits);
  const EI E = (EI)pk_edges(pk, P.ebits);
  if (E == 0) return;
  const EI T = (E + (EI)(WT - 1)) / (EI)WT;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const EI GW = (EI)gridDim.x * WPB;
  EI t = (EI)blockIdx.x * WPB + wid;
  if (t >= T) return;  // warp-uniform; no CTA barrier below
  WarpRows<XI>& w = s.w[wid];
  const int np = p ^ 1;
  const int eb = P.ebits;
  const uint32_t src = P.src;
  const uint32_t* tile_row = P.tile_row;
  const EI* qbase = P.qbase[p];
  const EI* qoff = P.qoff[p];
  const K* qkey = P.qkey[p];
  const uint32_t* qnode = P.qnode[p];
  auto row_bound = [&](EI q, uint32_t which) -> uint32_t {
    const EI x = q + (EI)which;
    return (x < T) ? ldcg(tile_row + x) : cnt - 1;
  };

  // prologue: first 32 rows of tile t into registers, row range of t+GW
  uint32_t i0 = row_bound(t, 0), il = row_bound(t, 1);
  uint32_t tr = (lane < 2 && t + GW < T) ? row_bound(t + GW, lane) : 0u;
  EI pf_base = 0, pf_off = 0;
  K pf_key = 0;
  uint32_t pf_node = 0;
  bool pf_live = false;  // async: pf_key of the next tile still to load from pf_node
  if (lane <= il - i0) {
    pf_base = ldcg(qbase + i0 + lane);
    pf_off = ldcg(qoff + i0 + lane);
    pf_key = (!PRED && P.live) ? ldcg(P.dist + ldcg(qnode + i0 + lane)) : ldcg(qkey + i0 + lane);
    if (PRED) pf_node = ldcg(qnode + i0 + lane);
  }

#ifdef DAWN_XTIMING
  // debug timeline (variant builds only): per round r < 16 and global warp, the
  // last tile's checkpoints [0] tile start [1] filter done [2] elections back
  // [3] row bounds / scan done [4] reservation back [5] tile end
  const uint32_t xt_gw = blockIdx.x * WPB + wid;
#define XT_MARK(k)                                                                                   \
  do {                                                                                               \
    if (P.cta_prof && r < 16 && xt_gw < 2368 && lane == 0)                                           \
      P.cta_prof[((size_t)r * 2368 + xt_gw) * 6 + (k)] = globaltimer();                              \
  } while (0)
#endif
  for (; t < T; t += GW) {
#ifdef DAWN_XTIMING
    XT_MARK(0);
#endif
    const EI e0 = t * (EI)WT;
    const uint32_t len = (E - e0 < (EI)WT) ? (uint32_t)(E - e0) : (uint32_t)WT;
    const uint32_t nrows = il - i0 + 1;
    const bool fast = nrows <= 32;
    const uint32_t ci0 = i0;
    // this tile's rows (lane k = row k) from the prefetch registers
    const EI c_base = pf_base;
    const C c_val = CD::dec(pf_key);
    const uint32_t c_node = pf_node;
    const uint32_t c_rst = (lane < nrows) ? (uint32_t)(pf_off > e0 ? pf_off - e0 : (EI)0) : 0xFFFFFFFFu;
    if (!fast) {
      // ---- short rows: mark row starts (row data is read through L1 below) ----
#pragma unroll
      for (int q = 0; q < XI; ++q) w.mark[lane * XI + q] = 0;
      __syncwarp();
      if (c_rst < len) w.mark[c_rst] = (uint16_t)lane;
      for (uint32_t k = 32 + lane; k < nrows; k += 32) {
        const EI off = __ldca(qoff + ci0 + k);
        const EI rst = off > e0 ? off - e0 : (EI)0;
        if (rst < (EI)len) w.mark[rst] = (uint16_t)k;
      }
    }
    // ---- advance the pipeline: rows of the next tile, range of the one after ----
    {
      const EI tn = t + GW;
      const uint32_t ni0 = __shfl_sync(0xffffffffu, tr, 0), nil = __shfl_sync(0xffffffffu, tr, 1);
      if (tn < T) {
        i0 = ni0;
        il = nil;
        if (lane <= il - i0) {
          pf_base = ldcg(qbase + i0 + lane);
          pf_off = ldcg(qoff + i0 + lane);
          // async: only the node here; its live value is loaded after this tile's
          // edge loads are issued (the dependent load stalled the warp mid-tile)
          if (!PRED && P.live) pf_node = ldcg(qnode + i0 + lane);
          else pf_key = ldcg(qkey + i0 + lane);
          if (PRED) pf_node = ldcg(qnode + i0 + lane);
        }
        pf_live = !PRED && P.live && lane <= il - i0;
        tr = (lane < 2 && tn + GW < T) ? row_bound(tn + GW, lane) : 0u;
      }
    }
    if (!fast) {
      __syncwarp();
      // inclusive max-scan of the marks: each lane owns XI consecutive slots
      uint32_t m8[XI];
#pragma unroll
      for (int j = 0; j < XI; ++j) m8[j] = w.mark[lane * XI + j];
      uint32_t run = 0;
#pragma unroll
      for (int j = 0; j < XI; ++j) { run = max(run, m8[j]); m8[j] = run; }
      uint32_t incl = run;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= (uint32_t)d) incl = max(incl, y);
      }
      uint32_t pre = __shfl_up_sync(0xffffffffu, incl, 1);
      if (lane == 0) pre = 0;
#pragma unroll
      for (int j = 0; j < XI; ++j) w.mark[lane * XI + j] = (uint16_t)max(m8[j], pre);
      __syncwarp();
    }

    // ---- phase 1a: row of every edge (collectives / L1 only, no edge loads yet) ----
    EI pos[XI];
    C rv[XI];          // row value (decoded once per row)
    uint32_t rowk[XI];
    if (fast) {
      uint32_t before = 0;  // rows starting before the current 32-edge window
#pragma unroll
      for (int j = 0; j < XI; ++j) {
        const uint32_t lo = j * 32;
        const uint32_t bit = (c_rst - lo < 32u) ? (1u << (c_rst - lo)) : 0u;
        const uint32_t B = __reduce_or_sync(0xffffffffu, bit);
        const uint32_t k = before + __popc(B & (0xFFFFFFFFu >> (31 - lane))) - 1;
        before += __popc(B);
        rowk[j] = k;
        pos[j] = __shfl_sync(0xffffffffu, c_base, k) + e0 + (EI)(lo + lane);
        rv[j] = __shfl_sync(0xffffffffu, c_val, k);
      }
    } else {
#pragma unroll
      for (int j = 0; j < XI; ++j) {
        // queue entries were written before the last grid barrier, whose fence
        // invalidated L1: L1-cached reads are coherent here
        const uint32_t k = w.mark[j * 32 + lane];
        rowk[j] = k;
        pos[j] = __ldca(qbase + ci0 + k) + e0 + (EI)(j * 32 + lane);
        rv[j] = CD::dec((!PRED && P.live) ? ldcg(P.dist + __ldca(qnode + ci0 + k)) : __ldca(qkey + ci0 + k));
      }
    }
    // ---- phase 1b: all edge loads back to back (nothing consumes them yet) ----
    uint32_t col[XI];
    WB wv[XI];
    unsigned okm = (XI >= 32) ? 0xFFFFFFFFu : ((1u << XI) - 1u);  // items inside the tile
    if (len != (uint32_t)WT) {
      okm = 0;
#pragma unroll
      for (int j = 0; j < XI; ++j) okm |= (unsigned)(j * 32 + lane < len) << j;
    }
    {
      const EI safe0 = __shfl_sync(0xffffffffu, c_base, 0) + e0;  // the tile's first edge
#pragma unroll
      for (int j = 0; j < XI; ++j) EdgeAccess<V>::load(P, ((okm >> j) & 1u) ? pos[j] : safe0, col[j], wv[j]);
    }
    if (!PRED && pf_live) {  // the next tile's live row values (its nodes arrived meanwhile)
      pf_key = ldcg(P.dist + pf_node);
      pf_live = false;
    }
    // ---- phase 2: candidates ----
    K cand[XI];
#pragma unroll
    for (int j = 0; j < XI; ++j) {
      cand[j] = CD::relax(rv[j], wv[j]);
      if (!CD::usable(cand[j])) okm &= ~(1u << j);
    }
    if (!PRED) {
      // ---- phase 3: read-before-write filter, all gathers in flight ----
      // L1-allocating loads (ld.ca): RMAT-like destinations are skewed, so a
      // large share of gathers hit L1 (measured 2.2x over L2-only gathers,
      // tools/gather_bench.cu).  Safe for the "cand < cur => lowered this
      // round" inference: every grid barrier's fence invalidates L1
      // (CCTL.IVALL) and no gather is outstanding at a barrier, so a value
      // seen in L1 during round r was read after round r began and is <= the
      // round-start value.
      K cur[XI];
#pragma unroll
      for (int j = 0; j < XI; ++j) cur[j] = ((okm >> j) & 1u) ? __ldca(P.dist + col[j]) : (K)0;
      unsigned need = 0;
#pragma unroll
      for (int j = 0; j < XI; ++j) {
        if (((okm >> j) & 1u) && cand[j] < cur[j]) {
          if (col[j] == src) P.st->flag = 1u;  // source guard (solver.py:299-303, :374-376, :236-239)
          else need |= 1u << j;
        }
      }
      // ---- phase 4: fire-and-forget min (cand < cur proves v is lowered this round) ----
      if (need) {
#pragma unroll
        for (int j = 0; j < XI; ++j)
          if ((need >> j) & 1u) atomicMin(P.dist + col[j], cand[j]);
      }
      if (dense) {
        if (need) {
#pragma unroll
          for (int j = 0; j < XI; ++j)
            if ((need >> j) & 1u) P.stamp[col[j]] = r;
        }
      } else if constexpr (FB) {
        // ---- light round, bitmap frontier: one bit per lowered node (red.or) ----
        if (need) {
#pragma unroll
          for (int j = 0; j < XI; ++j)
            if ((need >> j) & 1u) atomicOr(P.bmap + (col[j] >> 5), 1u << (col[j] & 31u));
        }
      } else if (__any_sync(0xffffffffu, need != 0u)) {
        // ---- sparse: elect one writer per (node, round), enqueue its row ----
#ifdef DAWN_XTIMING
        XT_MARK(1);
#endif
        unsigned first = 0;
#pragma unroll
        for (int j = 0; j < XI; ++j)
          if (((need >> j) & 1u) && atomicExch(P.stamp + col[j], r) != r) first |= 1u << j;
#ifdef DAWN_XTIMING
        if (__any_sync(0xffffffffu, first != 0u)) XT_MARK(2);
#endif
        unsigned long long mine = 0;  // (entries << eb) | edges of this lane
        EI rs[XI], re[XI];
        uint8_t wsv[XI];
        // every load first (write states, row bounds), all in flight together:
        // a store before the next element's load would serialise the chain
        // (the compiler cannot reorder a load above a possibly-aliasing store)
#pragma unroll
        for (int j = 0; j < XI; ++j) {
          rs[j] = re[j] = 0;
          wsv[j] = 0;
          if ((first >> j) & 1u) {
            wsv[j] = P.wstate[col[j]];
            rs[j] = __ldg(P.row_ptr + col[j]);
            re[j] = __ldg(P.row_ptr + col[j] + 1);
          }
        }
#pragma unroll
        for (int j = 0; j < XI; ++j) {
          if ((first >> j) & 1u) {
            round_w++;
            acc_w++;
            // first-write bookkeeping (runs once per (node, round)): first_discoveries
            // (solver.py:378-379) and nodes lowered in >= 2 rounds (solver.py:258-262)
            if (wsv[j] == 0) { acc_fd++; P.wstate[col[j]] = 1; }
            else if (wsv[j] == 1) { acc_multi++; P.wstate[col[j]] = 2; }
            if (re[j] > rs[j]) {  // rows without edges never need a rescan
              mine += (1ull << eb) + (unsigned long long)(re[j] - rs[j]);
              wv[j] = (WB)(re[j] - rs[j]);  // reuse: degree
            } else {
              first &= ~(1u << j);
            }
          }
        }
        unsigned long long incl = mine;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, d);
          if (lane >= (uint32_t)d) incl += y;
        }
        const unsigned long long tot = __shfl_sync(0xffffffffu, incl, 31);
#ifdef DAWN_XTIMING
        XT_MARK(3);
#endif
        if (tot) {
          unsigned long long base = 0;
          if (lane == 0) base = atomicAdd(&P.st->res[np], tot);
          base = __shfl_sync(0xffffffffu, base, 0);
#ifdef DAWN_XTIMING
          XT_MARK(4);
#endif
          const unsigned long long at = base + incl - mine;
          uint32_t pos = (uint32_t)pk_count(at, eb);
          EI off = (EI)pk_edges(at, eb);
#pragma unroll
          for (int j = 0; j < XI; ++j) {
            if ((first >> j) & 1u) {
              P.qnode[np][pos] = col[j];
              P.qoff[np][pos] = off;
              P.qbase[np][pos] = rs[j] - off;
              pos++;
              off += (EI)wv[j];
            }
          }
        }
      }
    } else {
      unsigned sv[XI];
#pragma unroll
      for (int j = 0; j < XI; ++j)
        sv[j] = (((okm >> j) & 1u) && col[j] != src) ? ldcg(P.stamp + col[j]) : 0u;
      K dv[XI];
#pragma unroll
      for (int j = 0; j < XI; ++j) dv[j] = (sv[j] == r) ? ldcg(P.dist + col[j]) : (K)0;
#pragma unroll
      for (int j = 0; j < XI; ++j) {
        const uint32_t u = fast ? __shfl_sync(0xffffffffu, c_node, rowk[j]) : __ldca(qnode + ci0 + rowk[j]);
        if (sv[j] == r && ((okm >> j) & 1u) && col[j] != src && cand[j] == dv[j])
          atomicMax(P.pred + col[j], ((unsigned long long)r << 32) | (unsigned long long)(~u));
      }
    }
    __syncwarp();  // the warp is done with its rows / marks
#ifdef DAWN_XTIMING
    XT_MARK(5);
#endif
  }
}


// ---------------------------------------------------------------------------
// Worklist tail (async schedule only; graphs without negative weights; a run
// without a round limit).  The last rounds of an RMAT solve relax ~1 % of the
// edges but cost ~15 % of the time: a round is a chain of ~10 dependent global
// accesses plus two grid barriers (~20 us) however few rows it has.  Once a
// round relaxes fewer than wl_edges edges, the rest of the solve runs
// barrier-free (dawn_worklist, launched behind the persistent kernel) off a
// ring of 16-byte row items {node, degree, first edge, value}:
//   * a relax that lowers dist[v] pushes v's row carrying the value it wrote
//     (no re-read of dist[v], no queued flag: the item itself is the message);
//     rows longer than CH = 32*XI edges travel as one split item that the warp
//     taking it turns into one item per CH-edge chunk;
//   * a warp claims up to 32 consecutive ring slots (fewer when the queue is
//     short), takes whichever are filled and relaxes their rows together as
//     one virtual edge list cut into warp tiles (the X phase's <= 32-row tile);
//     an item whose value is no longer dist[v] is dropped (a lower write
//     pushed its own item);
//   * one 64-bit counter carries (pending items << 32 | ring tail): a push
//     adds (k << 32 | k) before its items become visible; a warp retires the
//     items it took with one subtraction after its own pushes, so
//     pending == 0 is final.
// Why the result is the reference's: every candidate is fl(d + w) for a value
// d that dist[u] held, values only decrease, and every lowering pushes an item
// whose relax uses the value written, so the run stops only at the greatest
// fixpoint the snapshot rounds reach (the async argument).
// first_discoveries is exact (the unique atomicMin that returned INF); writes,
// nodes lowered twice and relaxations are this run's own.
// ---------------------------------------------------------------------------
constexpr uint32_t WL_NONE = 0xFFFFFFFFu;   // empty slot (node field)
constexpr uint32_t WL_SPLIT = 0xFFFFFFFFu;  // degree field: the whole long row (split when taken)
constexpr uint32_t WL_CHUNK = 0x80000000u;  // degree field: chunk index of a long row

__device__ __forceinline__ unsigned long long wl_retire(unsigned n) { return 0ull - ((unsigned long long)n << 32); }

__device__ __forceinline__ uint4 ld_relaxed_v4(const uint4* p) {
  uint4 v;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_v4(uint4* p, uint4 v) {
  asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// item layout: x = node, y = degree / WL_SPLIT / WL_CHUNK|chunk, z,w = value key (64-bit)
template <class K>
__device__ __forceinline__ uint4 wl_item(uint32_t node, uint32_t y, K key) {
  const unsigned long long k = (unsigned long long)key;
  return make_uint4(node, y, (uint32_t)k, (uint32_t)(k >> 32));
}

// store an item into a reserved slot; waits only if the slot's previous item
// (one lap back) has not been taken yet.  Watchdog: after 30 s without the
// slot freeing (or once another warp gave up) the solve is aborted
// cooperatively (the host reports DAWN_ECUDA) instead of trapping.
__device__ __forceinline__ void wl_store(uint4* q, uint32_t pre_node, uint4 item, unsigned* abort) {
  unsigned long long t0 = 0;
  while (pre_node != WL_NONE) {
    __nanosleep(64);
    pre_node = ld_relaxed_u32(&q->x);
    if (ld_acquire(abort)) return;
    const unsigned long long t = globaltimer();
    if (t0 == 0) t0 = t;
    else if (t - t0 > 30ull * 1000000000ull) {
#ifdef DAWN_DEBUG_TRAP
      asm volatile("trap;");
#endif
      atomicExch(abort, 1u);
      return;
    }
  }
  st_relaxed_v4(q, item);
}

// push the rows of node[j] (mask msk, degree deg[j]) with the values key[j]
// this lane wrote.  Warp-collective.
template <class V, class EI, int NJ, class K>
__device__ __forceinline__ void wl_push(const KParams<V, EI>& P, const uint32_t (&node)[NJ],
                                        const uint32_t (&deg)[NJ], const K (&key)[NJ], unsigned msk, uint32_t CH) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t mine = __popc(msk);
  const uint32_t incl = warp_incl_sum<uint32_t>(mine);
  const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
  if (tot == 0) return;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(&P.st->wl_ctr, ((unsigned long long)tot << 32) | tot);
  const uint32_t slot0 = (uint32_t)__shfl_sync(0xffffffffu, base, 0) + incl - mine;
  uint4* ring = reinterpret_cast<uint4*>(P.wl_ring);
  // a slot below the ring size has not been used yet in this solve (every slot is empty when a
  // solve starts): the lap check is only needed once the tickets wrap
  const bool wrapped = (unsigned long long)(uint32_t)__shfl_sync(0xffffffffu, base, 0) + tot > P.wl_mask + 1ull;
  uint32_t pre[NJ];
  uint32_t t = 0;
#pragma unroll
  for (int j = 0; j < NJ; ++j)  // all lap checks in flight at once
    if ((msk >> j) & 1u) pre[j] = wrapped ? ld_relaxed_u32(&ring[(slot0 + t++) & P.wl_mask].x) : WL_NONE;
  t = 0;
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    if ((msk >> j) & 1u) {
      uint4* q = ring + ((slot0 + t++) & P.wl_mask);
      wl_store(q, pre[j], wl_item<K>(node[j], deg[j] > CH ? WL_SPLIT : deg[j], key[j]), &P.st->abort);
    }
  }
}

// A warp keeps up to 32 of the rows it lowered as its own next batch (no ring
// round trip on the dependency chain: a hop costs edges -> gathers -> min);
// the rest, and rows longer than one chunk, go to the ring for other warps.
template <class K, class EI>
struct WlLocal {
  uint32_t node[32];
  uint32_t deg[32];
  K key[32];
  EI a[32];
};

// relax edges [e0, e0 + len) (len <= 32*XI) of the rows held in lanes 0..nb-1
// (first virtual edge off_k ascending, first real edge a_k, value val_k, every
// row non-empty; rows flagged `skip` — undercut values — relax nothing) and
// emit the rows they lower: into the warp's local list while it has room,
// else to the ring.  Warp-collective.
template <class V, class EI, int XI>
__device__ __forceinline__ void wl_relax_tile(const KParams<V, EI>& P, uint32_t nb, uint32_t off, EI a,
                                              typename Codec<V, true>::C val, bool skip, uint32_t e0, uint32_t len,
                                              WlLocal<typename Codec<V, true>::K, EI>& L, uint32_t& ln,
                                              unsigned long long& acc_w, unsigned long long& acc_fd,
                                              unsigned long long& acc_multi) {
  using CD = Codec<V, true>;
  using K = typename CD::K;
  using WB = typename CD::WB;
  using C = typename CD::C;
  constexpr uint32_t CH = 32 * XI;
  const uint32_t lane = threadIdx.x & 31;
  // rows starting at or before e0: the last of them holds e0
  const uint32_t i0 = __popc(__ballot_sync(0xffffffffu, lane < nb && off <= e0)) - 1;
  const uint32_t rst = (lane < nb && lane >= i0) ? (off > e0 ? off - e0 : 0u) : 0xFFFFFFFFu;
  uint32_t col[XI];
  WB wv[XI];
  C rv[XI];
  unsigned okm = 0;
  uint32_t before = 0;
#pragma unroll
  for (int j = 0; j < XI; ++j) {
    const uint32_t lo = j * 32;
    const uint32_t bit = (rst - lo < 32u) ? (1u << (rst - lo)) : 0u;
    const uint32_t B = __reduce_or_sync(0xffffffffu, bit);
    const uint32_t k = i0 + before + __popc(B & (0xFFFFFFFFu >> (31 - lane))) - 1;
    before += __popc(B);
    const uint32_t x = e0 + lo + lane;
    const EI pos = __shfl_sync(0xffffffffu, a, k) + (EI)(x - __shfl_sync(0xffffffffu, off, k));
    rv[j] = __shfl_sync(0xffffffffu, val, k);
    const bool live = lo + lane < len;
    const bool sk = __shfl_sync(0xffffffffu, skip, k);  // every lane takes part in the shuffle
    okm |= (unsigned)(live && !sk) << j;
    if (live) EdgeAccess<V>::load(P, pos, col[j], wv[j]);
    else { col[j] = 0; wv[j] = 0; }
  }
  K cand[XI];
#pragma unroll
  for (int j = 0; j < XI; ++j) {
    cand[j] = CD::relax(rv[j], wv[j]);
    if (!CD::usable(cand[j])) okm &= ~(1u << j);
  }
  // gathers and the lowered rows' bounds in flight together
  K cur[XI];
  EI ra[XI], rb[XI];
#pragma unroll
  for (int j = 0; j < XI; ++j) {
    const bool ok = (okm >> j) & 1u;
    cur[j] = ok ? ldcg(P.dist + col[j]) : (K)0;
    ra[j] = ok ? __ldg(P.row_ptr + col[j]) : (EI)0;
    rb[j] = ok ? __ldg(P.row_ptr + col[j] + 1) : (EI)0;
  }
  // lower: a target that was +inf takes a returning min (first discoveries are counted exactly
  // once); the others a fire-and-forget one.  The rows are emitted before any returned value is
  // looked at (an item whose min lost the race is dropped by its taker as undercut).
  unsigned need = 0, infm = 0;
  uint32_t dg[XI];
  K old[XI];
#pragma unroll
  for (int j = 0; j < XI; ++j) {
    dg[j] = (uint32_t)(rb[j] - ra[j]);
    old[j] = 0;
    if (((okm >> j) & 1u) && cand[j] < cur[j]) {
      if (col[j] == P.src) { P.st->flag = 1u; continue; }
      need |= 1u << j;
      if (cur[j] == CD::INF) {
        infm |= 1u << j;
        old[j] = atomicMin(P.dist + col[j], cand[j]);
      } else {
        atomicMin(P.dist + col[j], cand[j]);
      }
    }
  }
  unsigned emit = 0, small = 0;
#pragma unroll
  for (int j = 0; j < XI; ++j) {
    if (((need >> j) & 1u) && dg[j] > 0) {
      emit |= 1u << j;
      if (dg[j] <= CH) small |= 1u << j;
    }
  }
  {  // local list first (rows of at most one chunk), the overflow and long rows to the ring
    const uint32_t c = __popc(small);
    const uint32_t incl = warp_incl_sum<uint32_t>(c);
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t room = 32u - ln;
    uint32_t pos = incl - c;
    unsigned ring_m = emit & ~small;
#pragma unroll
    for (int j = 0; j < XI; ++j) {
      if ((small >> j) & 1u) {
        if (pos < room) {
          const uint32_t at = ln + pos;
          L.node[at] = col[j];
          L.deg[at] = dg[j];
          L.key[at] = cand[j];
          L.a[at] = ra[j];
        } else {
          ring_m |= 1u << j;
        }
        ++pos;
      }
    }
    ln += min(tot, room);
    __syncwarp();
    wl_push<V, EI, XI, K>(P, col, dg, cand, ring_m, CH);
  }
  // bookkeeping from the returned values
#pragma unroll
  for (int j = 0; j < XI; ++j) {
    if ((need >> j) & 1u) {
      const uint32_t v = col[j];
      unsigned* wsw = reinterpret_cast<unsigned*>(P.wstate + (v & ~3u));
      const unsigned sh = 8u * (v & 3u);
      if ((infm >> j) & 1u) {
        if (old[j] == CD::INF) {
          acc_fd++;
          acc_w++;
          atomicOr(wsw, 1u << sh);
        } else if (cand[j] < old[j]) {
          acc_w++;
          if (!(atomicOr(wsw, 2u << sh) & (2u << sh))) acc_multi++;
        }
      } else {
        acc_w++;
        if (!(atomicOr(wsw, 2u << sh) & (2u << sh))) acc_multi++;
      }
    }
  }
}

// round r's frontier (queue p) becomes the first items; the persistent kernel
// then exits and dawn_worklist (launched behind it) takes over
template <class V, class EI>
__device__ void wl_seed(const KParams<V, EI>& P, int p) {
  using K = typename Codec<V, true>::K;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * NT + threadIdx.x) >> 5, nw = gridDim.x * WPB;
  const uint32_t cnt = (uint32_t)pk_count(ldcg(&P.st->res[p]), P.ebits);
  for (uint32_t b0 = gw * 32; b0 < cnt; b0 += nw * 32) {
    const bool ok = b0 + lane < cnt;
    uint32_t v[1] = {ok ? ldcg(P.qnode[p] + b0 + lane) : 0u};
    K key[1] = {ok ? ldcg(P.dist + v[0]) : (K)0};
    uint32_t dg[1] = {ok ? (uint32_t)(__ldg(P.row_ptr + v[0] + 1) - __ldg(P.row_ptr + v[0])) : 0u};
    wl_push<V, EI, 1, K>(P, v, dg, key, (ok && dg[0] > 0) ? 1u : 0u, 32u * XI_NARROW);
  }
}

template <class V, class EI>
__global__ void __launch_bounds__(NT, 2) dawn_worklist(KParams<V, EI> P) {
  constexpr int XI = XI_NARROW;
  using CD = Codec<V, true>;
  using K = typename CD::K;
  using C = typename CD::C;
  constexpr uint32_t CH = 32 * XI;
  DevState* st = P.st;
  if (ldcg(&st->wl_mode) == 0u) return;  // the solve finished in rounds
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nw = gridDim.x * WPB;
  uint4* ring = reinterpret_cast<uint4*>(P.wl_ring);
  unsigned long long acc_w = 0, acc_fd = 0, acc_multi = 0, acc_e = 0, acc_i = 0;
  const unsigned long long t_begin = globaltimer();
  unsigned long long busy = 0, nbatch = 0;
  __shared__ WlLocal<K, EI> locs[WPB];
  WlLocal<K, EI>& L = locs[threadIdx.x >> 5];
  uint32_t ln = 0;    // rows in this warp's local list (warp-uniform)
  uint32_t held = 0;  // ring items taken and not yet retired (they keep pending > 0 for the local chain)
  unsigned own = 0;   // claimed slots h + lane not taken yet
  uint32_t h = 0;
  unsigned ns = 32;
  unsigned long long t0 = 0, seen = 0;
  for (;;) {
    unsigned got;
    uint32_t u = 0, y = 0;
    K key = 0;
    EI a = 0;
    bool have_a = false;
    unsigned long long t_got;
    if (ln > 0) {
      // ---- the rows this warp lowered itself: no ring round trip ----
      got = (ln >= 32) ? 0xFFFFFFFFu : ((1u << ln) - 1u);
      if (lane < ln) {
        u = L.node[lane];
        y = L.deg[lane];
        key = L.key[lane];
        a = L.a[lane];
      }
      have_a = true;
      ln = 0;
      __syncwarp();
      t_got = globaltimer();
    } else {
      if (held) {  // back to the ring: retire what the local chain grew from (its pushes are counted)
        if (lane == 0) atomicAdd(&st->wl_ctr, wl_retire(held));
        held = 0;
      }
      if (own == 0) {
        uint32_t c = 1;
        if (lane == 0) {
          const uint32_t tail = (uint32_t)ld_relaxed(&st->wl_ctr), head = (uint32_t)ld_relaxed(&st->wl_head);
          const uint32_t avail = tail - head;
          c = (avail < 0x80000000u) ? min(32u, max(1u, avail / nw)) : 1u;
          h = (uint32_t)atomicAdd(&st->wl_head, (unsigned long long)c);
        }
        c = __shfl_sync(0xffffffffu, c, 0);
        h = __shfl_sync(0xffffffffu, h, 0);
        own = (c >= 32) ? 0xFFFFFFFFu : ((1u << c) - 1u);
      }
      uint4* q = ring + ((h + lane) & P.wl_mask);
      uint4 it = make_uint4(WL_NONE, WL_NONE, WL_NONE, WL_NONE);
      if ((own >> lane) & 1u) it = ld_relaxed_v4(q);
      // filled = both 8-byte halves written (w, the key's high word, is <= 0x7FFFFFFF in a real item)
      got = __ballot_sync(0xffffffffu, it.x != WL_NONE && it.w != WL_NONE);
      if (got == 0) {
        bool fin = false;
        if (lane == 0) {
          const unsigned long long ctr = ld_relaxed(&st->wl_ctr);
          fin = (ctr >> 32) == 0ull;
          // watchdog: trap only if the whole worklist made no progress (no push, no retire) for 30 s;
          // waiting long while other warps work (a long dependency chain) is legitimate
          const unsigned long long t = globaltimer();
          if (t0 == 0 || ctr != seen) {
            t0 = t;
            seen = ctr;
          } else if (t - t0 > 30ull * 1000000000ull) {
#ifdef DAWN_DEBUG_TRAP
            asm volatile("trap;");
#endif
            atomicExch(&st->abort, 1u);
          }
          fin = fin || ld_acquire(&st->abort) != 0u;
        }
        if (__shfl_sync(0xffffffffu, fin, 0)) break;
        __nanosleep(ns);
        if (ns < 128) ns <<= 1;
        continue;
      }
      ns = 32;
      t0 = 0;
      t_got = globaltimer();
      own &= ~got;
      if ((got >> lane) & 1u) st_relaxed_v4(q, make_uint4(WL_NONE, WL_NONE, WL_NONE, WL_NONE));
      u = it.x;
      y = it.y;
      key = (K)(((unsigned long long)it.w << 32) | it.z);
      held += __popc(got);
    }
    const bool mine = (got >> lane) & 1u;
    // single-chunk rows: first edge; the undercut check runs beside the edge loads
    const bool single = mine && y <= CH;
    K now = key;
    if (single) {
      if (!have_a) a = __ldg(P.row_ptr + u);
      now = ldcg(P.dist + u);
    }
    const unsigned sm = __ballot_sync(0xffffffffu, single);
    if (sm) {
      const uint32_t nb = __popc(sm);
      const uint32_t fl = (lane < nb) ? __fns(sm, 0, lane + 1) : 0u;
      const EI ra = __shfl_sync(0xffffffffu, a, fl);
      const uint32_t rd = __shfl_sync(0xffffffffu, y, fl);
      const K rk = __shfl_sync(0xffffffffu, key, fl);
      // drop (relax nothing for) a row whose value was undercut: a lower write emitted its own row;
      // a value above the row's means the row's own fire-and-forget min has not landed yet
      const bool skip = __shfl_sync(0xffffffffu, now < key, fl);
      const uint32_t rdeg = (lane < nb) ? rd : 0u;
      const uint32_t incl = warp_incl_sum<uint32_t>(rdeg);
      const uint32_t Eb = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t off = incl - rdeg;
      const C val = CD::dec(rk);
      for (uint32_t e0 = 0; e0 < Eb; e0 += CH)
        wl_relax_tile<V, EI, XI>(P, nb, off, ra, val, skip, e0, min(CH, Eb - e0), L, ln, acc_w, acc_fd, acc_multi);
      if (lane == 0) acc_e += Eb;
    }
    // long rows (ring only): split items and chunks, one at a time
    unsigned lm = __ballot_sync(0xffffffffu, mine && y > CH);
    while (lm) {
      const int l = __ffs(lm) - 1;
      lm &= lm - 1;
      const uint32_t lu = __shfl_sync(0xffffffffu, u, l), ly = __shfl_sync(0xffffffffu, y, l);
      const K lk = __shfl_sync(0xffffffffu, key, l);
      const EI la = __ldg(P.row_ptr + lu), lb = __ldg(P.row_ptr + lu + 1);
      if (ldcg(P.dist + lu) < lk) continue;  // undercut: a lower write emitted its own row
      if (ly == WL_SPLIT) {
        const uint32_t nch = (uint32_t)((lb - la + (EI)CH - 1) / (EI)CH);
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&st->wl_ctr, ((unsigned long long)nch << 32) | nch);
        const uint32_t b0 = (uint32_t)__shfl_sync(0xffffffffu, base, 0);
        for (uint32_t c = lane; c < nch; c += 32) {
          uint4* qq = ring + ((b0 + c) & P.wl_mask);
          wl_store(qq, ld_relaxed_u32(&qq->x), wl_item<K>(lu, WL_CHUNK | c, lk), &st->abort);
        }
        __syncwarp();
      } else {
        const EI e0 = la + (EI)(ly & ~WL_CHUNK) * (EI)CH;
        const uint32_t len = (lb - e0 < (EI)CH) ? (uint32_t)(lb - e0) : CH;
        wl_relax_tile<V, EI, XI>(P, 1u, 0u, e0, CD::dec(lk), false, 0u, len, L, ln, acc_w, acc_fd, acc_multi);
        if (lane == 0) acc_e += len;
      }
    }
    __syncwarp();
    if (lane == 0) {
      acc_i += __popc(got);
      busy += globaltimer() - t_got;
      nbatch++;
    }
  }
  const unsigned long long t_end = globaltimer();
  acc_w = warp_sum_u64(acc_w);
  acc_fd = warp_sum_u64(acc_fd);
  acc_multi = warp_sum_u64(acc_multi);
  if (lane == 0) {
    if (acc_e) atomicAdd(&st->R, acc_e);
    if (acc_i) atomicAdd(&st->wl_items, acc_i);
    if (acc_w) atomicAdd(&st->W, acc_w);
    if (acc_fd) atomicAdd(&st->FD, acc_fd);
    if (acc_multi) atomicAdd(&st->multi, acc_multi);
    atomicAdd(&st->wl_batches, nbatch);
    atomicAdd(&st->wl_busy_ns, busy);
    atomicAdd(&st->wl_wait_ns, t_end - t_begin - busy);
    atomicMin(&st->wl_t0, t_begin);
    atomicMax(&st->wl_t1, t_end);
  }
}

// ---------------------------------------------------------------------------
// Negative-cycle early exit: a cycle in the predecessor graph (each finite
// node -> the frontier node that produced its value in its last lowering
// round) implies a reachable negative cycle when arithmetic is exact
// (integers): around such a cycle the weights sum to
//   -sum(snapshot - final) < 0,
// because the rounds cannot all advance by exactly one around a cycle.
// The reference then keeps writing until its n-round cap and flags
// (solver.py:394-395), so stopping early gives the same verdict.
// Pointer doubling: after ceil(log2 n) squarings every finite node points at
// the source iff its chain is acyclic.
// ---------------------------------------------------------------------------
template <class V, class EI>
__device__ bool pred_graph_has_cycle(const KParams<V, EI>& P) {
  using VT = Val<V>;
  const uint32_t n = P.n, src = P.src;
  const uint32_t gtid = blockIdx.x * NT + threadIdx.x, gsz = gridDim.x * NT;
  if (gtid == 0) P.st->cyc = 0u;
  for (uint32_t v = gtid; v < n; v += gsz) {
    uint32_t j = v;
    if (v != src && ldcg(P.dist + v) != VT::INF) j = ~(uint32_t)ldcg(P.pred + v);
    P.jmp0[v] = j;
  }
  if (grid_sync(&P.st->bar, &P.st->abort)) return true;
  uint32_t* a = P.jmp0;
  uint32_t* b = P.jmp1;
  for (int it = 0; it < P.logn; ++it) {
    for (uint32_t v = gtid; v < n; v += gsz) b[v] = ldcg(a + ldcg(a + v));
    if (grid_sync(&P.st->bar, &P.st->abort)) return true;
    uint32_t* t = a; a = b; b = t;
  }
  for (uint32_t v = gtid; v < n; v += gsz) {
    if (v != src && ldcg(P.dist + v) != VT::INF && ldcg(a + v) != src) P.st->cyc = 1u;
  }
  if (grid_sync(&P.st->bar, &P.st->abort)) return true;
  return ldcg(&P.st->cyc) != 0u;
}

// ---------------------------------------------------------------------------
// the persistent kernel
// ---------------------------------------------------------------------------
// WITH_PRED instantiates the predecessor pass and the negative-cycle check;
// the plain instance carries none of their registers.
// FB: light rounds record their writes in a bitmap (low-degree graphs) instead
// of enqueueing them; never combined with WITH_PRED.
template <class V, class EI, bool WITH_PRED, bool RAW, int XI, bool FB = false>
__global__ void __launch_bounds__(NT, DAWN_MIN_BLOCKS) dawn_persistent(KParams<V, EI> P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<V, EI, XI>& s = *reinterpret_cast<Smem<V, EI, XI>*>(smem_raw);
  DevState* st = P.st;
  const bool leader = (blockIdx.x == 0 && threadIdx.x == 0);
  if (P.skip_if_done && ldcg(&st->done)) return;  // uniform: written by an earlier launch

  uint32_t r = ldcg(&st->round);
  bool dense_prev = ldcg(&st->dense_prev) != 0u;  // how round r-1 recorded its writes
  bool skip_s = ldcg(&st->resume_x) != 0u;         // stepping: round r's frontier is already built
  unsigned long long acc_w = 0, acc_fd = 0, acc_multi = 0, acc_r = 0;
  unsigned long long E_prev = 0;  // frontier edges of the previous round (priority window)
  uint32_t tb = 0xFFFFFFFFu;       // priority window of this round's S phase (0xFFFFFFFF = none)
  bool pw_prev = false;            // the previous round was windowed
  unsigned rounds = 0;
  for (;;) {
    const int p = r & 1;
    const bool prof = leader && P.prof != nullptr && r < P.prof_cap;
    tb = 0xFFFFFFFFu;
    if (!skip_s) {
      if (prof) P.prof[4 * r + 0] = globaltimer();
      // ---- S phase: build round r's frontier ----
      if (leader) {
        st->res[p ^ 1] = 0ull;  // queue of round r+1 (filled by X_r or S_{r+1})
        st->wround[p] = 0ull;   // writes of round r (counted in X_r or S_{r+1})
        st->sctr[p ^ 1] = 0u;   // chunk counter of S_{r+1} (S_{r-1} used it and is over)
      }
      if (P.pw && blockIdx.x == 0)  // histogram of round r+1 (X_{r-1} read it before the last barrier)
        for (int i = threadIdx.x; i < PW_BINS; i += NT) P.phist[(size_t)(p ^ 1) * PW_BINS + i] = 0u;
      if (r >= 2 && (dense_prev || P.algo == 1)) {
        uint32_t prev_w = 0;
        if constexpr (RAW && !WITH_PRED && !FB) {
          // priority window: a heavy round's frontier is histogrammed first (one
          // sweep + barrier), then only its lowest pw_frac (by edges) is selected
          // (histogrammed after a heavy or windowed round and in round 2 after a
          // dense seeding round; windowed when the frontier holds >= pw_edges edges)
          if (P.pw && (r == 2 || E_prev >= P.pw_edges || pw_prev)) {
            phase_hist<V, EI, XI>(P, p, r, s);
            if (grid_sync(&st->bar, &st->abort)) break;
            tb = pw_threshold<V, EI, XI>(P, p, s);
          }
        }
        phase_compact<V, EI, XI>(P, p, r, s, acc_w, acc_fd, acc_multi, prev_w, tb);
        prev_w = __reduce_add_sync(0xffffffffu, prev_w);
        if ((threadIdx.x & 31) == 0 && prev_w) atomicAdd(&st->wround[p ^ 1], (unsigned long long)prev_w);
      } else if (FB && r >= 2) {
        uint32_t prev_w = 0;
        phase_bitmap<V, EI, XI>(P, p, r, acc_w, acc_fd, acc_multi, prev_w);
        prev_w = __reduce_add_sync(0xffffffffu, prev_w);
        if ((threadIdx.x & 31) == 0 && prev_w) atomicAdd(&st->wround[p ^ 1], (unsigned long long)prev_w);
      } else {
        phase_snapshot<V, EI, XI>(P, p);
      }
#ifndef DAWN_XTIMING
      if (P.cta_prof != nullptr && r < CTA_PROF_ROUNDS && threadIdx.x == 0)
        P.cta_prof[((size_t)r * 2 + 0) * gridDim.x + blockIdx.x] = globaltimer();
#endif
      if (grid_sync(&st->bar, &st->abort)) break;
      // ---- termination (solver.py:284-285, :313-317, :356-358, :388-395) ----
      if (r >= 2) {
        const unsigned long long wprev = ldcg(&st->wround[p ^ 1]);
        bool stop = false, capflag = false;
        // a loop round wrote nothing (and, under the priority window, deferred nothing)
        if (r - 1 >= 2 && wprev == 0 && (!P.pw || pk_count(ldcg(&st->res[p]), P.ebits) == 0)) stop = true;
        else if (r - 1 >= P.n) { stop = true; capflag = wprev > 0; }  // cap reached still writing
        if (stop) {
          if (leader) {
            st->steps = r - 1;
            if (capflag) st->flag = 1u;
            st->done = 1u;
            st->round = r;
          }
          break;
        }
        if (WITH_PRED && P.negcheck_period > 0 && r > 2 && ((r - 1) % (unsigned)P.negcheck_period) == 0) {
          if (pred_graph_has_cycle(P)) {
            if (leader) {
              st->steps = r - 1;
              st->flag = 1u;
              st->early = 1u;
              st->done = 1u;
              st->round = r;
            }
            break;
          }
        }
      }
      if (rounds == P.max_rounds) {  // stepping: resume at X_r next launch
        if (leader) {
          st->round = r;
          st->resume_x = 1u;
        }
        break;
      }
    }
    skip_s = false;
    // ---- X phase ----
    const unsigned long long E = pk_edges(ldcg(&st->res[p]), P.ebits);
    // a round whose S phase deferred rows records its writes densely (the next
    // dense S phase picks the deferred rows up again) and never hands over to
    // the worklist (its queue would miss them)
    const bool pw_round = tb != 0xFFFFFFFFu;
    const bool dense = P.algo == 1 || E >= P.dense_edges || pw_round || (P.pw && r == 1 && E >= P.pw_seed_edges);
    if (prof) {
      P.prof[4 * r + 1] = globaltimer();
      P.prof[4 * r + 3] = ldcg(&st->res[p]);
    }
    if constexpr (RAW && !WITH_PRED && !FB) {
      if (P.wl_ring != nullptr && P.live && P.algo == 0 && P.max_rounds == 0xFFFFFFFFu && r >= 2 &&
          E < P.wl_edges && !pw_round) {
        wl_seed<V, EI>(P, p);
        if (prof) P.prof[4 * r + 2] = globaltimer();  // the seeding; dawn_worklist runs after
        if (leader) {
          st->wl_mode = 1u;
          st->steps = r;
          st->done = 1u;
          st->round = r + 1;
        }
        break;
      }
    }
    if (leader) acc_r += E;  // relaxations (solver.py:297, :372)
    E_prev = E;
    pw_prev = pw_round;
    uint32_t round_w = 0;
    phase_expand<V, EI, false, RAW, XI, FB>(P, p, r, dense, s, acc_w, acc_fd, acc_multi, round_w);
    round_w = __reduce_add_sync(0xffffffffu, round_w);
    if ((threadIdx.x & 31) == 0 && round_w) atomicAdd(&st->wround[p], (unsigned long long)round_w);
#ifndef DAWN_XTIMING
    if (P.cta_prof != nullptr && r < CTA_PROF_ROUNDS) {
      __syncthreads();
      if (threadIdx.x == 0) P.cta_prof[((size_t)r * 2 + 1) * gridDim.x + blockIdx.x] = globaltimer();
    }
#endif
    if (grid_sync(&st->bar, &st->abort)) break;
    if (leader) st->resume_x = 0u;  // every CTA has read it (first barrier passed)
    if constexpr (WITH_PRED) {
      phase_expand<V, EI, true, RAW, XI>(P, p, r, dense, s, acc_w, acc_fd, acc_multi, round_w);
      if (grid_sync(&st->bar, &st->abort)) break;
    }
    if (prof) P.prof[4 * r + 2] = globaltimer();
    dense_prev = dense;
    ++r;
    ++rounds;
  }
  if (leader) st->dense_prev = dense_prev ? 1u : 0u;
  // flush per-thread counters
  acc_w = warp_sum_u64(acc_w);
  acc_fd = warp_sum_u64(acc_fd);
  acc_multi = warp_sum_u64(acc_multi);
  if ((threadIdx.x & 31) == 0) {
    if (acc_w) atomicAdd(&st->W, acc_w);
    if (acc_fd) atomicAdd(&st->FD, acc_fd);
    if (acc_multi) atomicAdd(&st->multi, acc_multi);
  }
  if (leader && acc_r) atomicAdd(&st->R, acc_r);
}

// ---------------------------------------------------------------------------
// small kernels
// ---------------------------------------------------------------------------
// solve init (solver.py:275-280, :343-350), everything in one launch: dist =
// INF with the source's key 0, stamps / write states / bitmap cleared, and
// (block 0) the seed frontier {source} plus the solve state — instead of four
// memsets and a launch (26 -> 12 us of a config-2 step)
template <class V, class EI, bool RAW>
__global__ void dawn_begin_solve(KParams<V, EI> P) {
  using CD = Codec<V, RAW>;
  using K = typename CD::K;
  if (P.skip_if_done && ldcg(&P.st->done)) return;  // the speculative run converged: keep its result
  const uint32_t n = P.n;
  const size_t T = (size_t)gridDim.x * blockDim.x;
  const size_t t0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const K k0 = CD::enc((V)0);
  for (size_t i = t0; i < n; i += T) {
    P.dist[i] = (i == P.src) ? k0 : CD::INF;
    P.stamp[i] = 0u;
  }
  uint32_t* ws = reinterpret_cast<uint32_t*>(P.wstate);  // allocated n + 4 bytes
  for (size_t i = t0; i < ((size_t)n + 3) / 4; i += T) ws[i] = 0u;
  for (size_t i = t0; i < ((size_t)n + 31) / 32 + 4; i += T) P.bmap[i] = 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    DevState* st = P.st;
    const uint32_t s = P.src;
    const EI a = P.row_ptr[s], b = P.row_ptr[s + 1];
    const unsigned long long deg = (unsigned long long)(b - a);
    st->res[0] = 0ull;
    st->res[1] = deg ? ((1ull << P.ebits) | deg) : 0ull;
    P.qnode[1][0] = s;
    P.qoff[1][0] = 0;
    P.qbase[1][0] = a;
    st->wround[0] = st->wround[1] = 0ull;
    st->sctr[0] = st->sctr[1] = 0u;
    st->round = 1u;
    st->dense_prev = 0u;
    st->resume_x = 0u;
    st->done = 0u;
    st->flag = 0u;
    st->abort = 0u;
    st->early = 0u;
    st->cyc = 0u;
    st->steps = 0ull;
    st->R = st->W = st->FD = st->multi = 0ull;
    st->wl_head = st->wl_ctr = st->wl_items = 0ull;
    st->wl_mode = 0u;
    st->wl_batches = st->wl_busy_ns = st->wl_wait_ns = st->wl_t1 = 0ull;
    st->wl_t0 = ~0ull;
  }
}

template <class V, bool RAW>
__global__ void dawn_decode_dist(const typename Val<V>::K* __restrict__ keys, uint32_t n,
                                 double* __restrict__ out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = Codec<V, RAW>::to_f64(keys[i]);
}

template <class V>
__global__ void dawn_decode_pred(const typename Val<V>::K* __restrict__ keys,
                                 const unsigned long long* __restrict__ pred, uint32_t n,
                                 uint32_t src, int64_t* __restrict__ out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int64_t v = -1;
    if (i != src && keys[i] != Val<V>::INF && pred[i] != 0ull) v = (int64_t)(~(uint32_t)pred[i]);
    out[i] = v;
  }
}

}  // namespace dawn
