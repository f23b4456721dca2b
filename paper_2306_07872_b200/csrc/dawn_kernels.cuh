// dawn_kernels.cuh — the persistent weighted-DAWN solver (GOVM + GSVM).
//
// One cooperative launch runs the whole round loop of the reference's
// `while step < n` (solver.py:284, :356) on the device: no host sync per
// round.  Each round r is two grid-synchronised phases:
//
//   S (snapshot/compact): frontier entries take a snapshot of their node's
//      distance (snapshot-Jacobi semantics: every relax in round r reads the
//      value as of the start of round r) and mark which frontier entry owns
//      the first virtual edge of every TILE-edge tile.  GSVM builds its
//      frontier here by compacting all finite rows (solver.py:287-289).
//   X (expand): persistent CTAs claim TILE-edge tiles of the frontier's
//      virtual edge list (merge-path style load balance, so hub rows of
//      10^5 edges and 1-edge rows cost the same per edge), find each edge's
//      row with a block max-scan over row-start marks, stream the packed
//      (col, w) pairs, and relax with read-before-atomicMin on the ordered
//      key.  The first lowering of a node in a round (write stamp) counts
//      the write, the first discovery and the >=2-round nodes, and enqueues
//      the node into the next frontier through a per-CTA buffer flushed with
//      one packed 64-bit atomicAdd reserving (entries, edge offsets)
//      together — the frontier "Copy beta to delta" of Alg. 2
//       without an O(n) scan.
//
// Optional passes: a predecessor pass (record_pred) and a predecessor-graph
// cycle check by pointer doubling (integer weights with negative edges).
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
  uint32_t* stamp;
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
};

template <class V, class EI>
struct __align__(16) Smem {
  using K = typename Val<V>::K;
  uint16_t mark[TILE];          // row-start marks -> per-edge row index (max-scan)
  K key[TILE + 1];              // snapshot key per tile row
  EI base[TILE + 1];            // row base per tile row
  uint32_t qnode[TILE + 1];     // enqueue buffer nodes; tile row nodes in the pred pass
  EI qrs[TILE];                 // enqueue buffer: row start
  EI qdeg[TILE];                // enqueue buffer: degree, then local offset
  EI scr[NT / 32];
  unsigned long long scr64[NT / 32];
  uint32_t wmark[NT / 32];
  unsigned long long basepk;
  uint32_t tile;
  int qcnt;
};

template <class V> struct EdgeAccess;
// 4-byte value types: one 8-byte load per edge
template <> struct EdgeAccess<int32_t> {
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

// mark the tiles whose first virtual edge falls inside [off, off + deg)
template <class EI>
__device__ __forceinline__ void mark_tiles(uint32_t* tile_row, EI off, EI deg, uint32_t entry) {
  EI t0 = (off + (EI)(TILE - 1)) / (EI)TILE;
  EI t1 = (off + deg - 1) / (EI)TILE;
  for (EI t = t0; t <= t1; ++t) tile_row[t] = entry;
}

// ---------------------------------------------------------------------------
// S phase, GOVM (and round 1 of GSVM): snapshot the frontier keys
// ---------------------------------------------------------------------------
template <class V, class EI>
__device__ void phase_snapshot(const KParams<V, EI>& P, int p) {
  const unsigned long long pk = ldcg(&P.st->res[p]);
  const uint32_t cnt = (uint32_t)pk_count(pk, P.ebits);
  const EI E = (EI)pk_edges(pk, P.ebits);
  const uint32_t* qn = P.qnode[p];
  const EI* qo = P.qoff[p];
  for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < cnt; i += gridDim.x * NT) {
    const uint32_t u = ldcg(qn + i);
    P.qkey[p][i] = ldcg(P.dist + u);
    const EI off = ldcg(qo + i);
    const EI nxt = (i + 1 < cnt) ? ldcg(qo + i + 1) : E;
    mark_tiles<EI>(P.tile_row, off, nxt - off, i);
  }
}

// ---------------------------------------------------------------------------
// S phase, GSVM rounds >= 2: every finite row with edges is rescanned
// (solver.py:287-289); compaction builds the frontier with snapshots.
// ---------------------------------------------------------------------------
template <class V, class EI>
__device__ void phase_compact_all(const KParams<V, EI>& P, int p, Smem<V, EI>& s) {
  using VT = Val<V>;
  using K = typename VT::K;
  const uint32_t n = P.n;
  const uint32_t nchunks = (n + TILE - 1) / TILE;
  for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    uint32_t u0 = c * TILE + threadIdx.x * ITEMS;
    uint32_t selmask = 0;
    EI degs[ITEMS];
    EI rs[ITEMS];
    K keys[ITEMS];
    uint32_t mycnt = 0;
    EI mydeg = 0;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      uint32_t u = u0 + j;
      degs[j] = 0;
      rs[j] = 0;
      keys[j] = VT::INF;
      if (u < n) {
        K k = ldcg(P.dist + u);
        keys[j] = k;
        if (k != VT::INF) {
          EI a = __ldg(P.row_ptr + u), b = __ldg(P.row_ptr + u + 1);
          if (b > a) {
            selmask |= 1u << j;
            degs[j] = b - a;
            rs[j] = a;
            mycnt++;
            mydeg += b - a;
          }
        }
      }
    }
    EI tot_deg;
    EI incl_deg = block_incl_sum<EI>(mydeg, s.scr, &tot_deg);
    unsigned long long tot_cnt;
    unsigned long long incl_cnt = block_incl_sum<unsigned long long>(mycnt, s.scr64, &tot_cnt);
    if (threadIdx.x == 0 && tot_cnt > 0) {
      s.basepk = atomicAdd(&P.st->res[p], (tot_cnt << P.ebits) | (unsigned long long)tot_deg);
    }
    __syncthreads();
    if (tot_cnt > 0) {
      const unsigned long long bp = s.basepk;
      uint32_t pos = (uint32_t)(pk_count(bp, P.ebits) + incl_cnt - mycnt);
      EI off = (EI)pk_edges(bp, P.ebits) + incl_deg - mydeg;
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        if (selmask & (1u << j)) {
          P.qnode[p][pos] = u0 + j;
          P.qoff[p][pos] = off;
          P.qbase[p][pos] = rs[j] - off;
          P.qkey[p][pos] = keys[j];
          mark_tiles<EI>(P.tile_row, off, degs[j], pos);
          pos++;
          off += degs[j];
        }
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// X phase: tiles of the frontier's virtual edge list.
//   PRED == false : relax + count + enqueue (GOVM)
//   PRED == true  : predecessor pass — among this round's frontier edges that
//                   reproduce the final value of a node lowered this round,
//                   keep the smallest source node (deterministic witness).
// ---------------------------------------------------------------------------
template <class V, class EI, bool PRED>
__device__ void phase_expand(const KParams<V, EI>& P, int p, uint32_t r, Smem<V, EI>& s,
                             unsigned long long& acc_w, unsigned long long& acc_fd,
                             unsigned long long& acc_multi, uint32_t& round_w) {
  using VT = Val<V>;
  using K = typename VT::K;
  using WB = typename VT::WB;
  const unsigned long long pk = ldcg(&P.st->res[p]);
  const uint32_t cnt = (uint32_t)pk_count(pk, P.ebits);
  const EI E = (EI)pk_edges(pk, P.ebits);
  if (E == 0) return;
  const EI T = (E + (EI)(TILE - 1)) / (EI)TILE;
  const int np = p ^ 1;
  const bool govm = (P.algo == 0);
  const uint32_t src = P.src;
  unsigned* tctr = PRED ? &P.st->tile_ctr2[p] : &P.st->tile_ctr[p];
  const int tid = threadIdx.x;

  for (;;) {
    if (tid == 0) s.tile = atomicAdd(tctr, 1u);
    __syncthreads();
    const EI t = (EI)s.tile;
    if (t >= T) break;
    const EI e0 = t * (EI)TILE;
    const EI e1 = (E - e0 < (EI)TILE) ? E : e0 + (EI)TILE;
    const uint32_t i0 = ldcg(P.tile_row + t);
    const uint32_t ilast = (t + 1 < T) ? ldcg(P.tile_row + t + 1) : cnt - 1;
    const uint32_t nrows = ilast - i0 + 1;
    const bool multi_row = nrows > 1;
    if (multi_row) reinterpret_cast<uint4*>(s.mark)[tid] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    for (uint32_t k = tid; k < nrows; k += NT) {
      const uint32_t i = i0 + k;
      s.base[k] = ldcg(P.qbase[p] + i);
      s.key[k] = ldcg(P.qkey[p] + i);
      if (PRED) s.qnode[k] = ldcg(P.qnode[p] + i);
      if (multi_row) {
        EI off = ldcg(P.qoff[p] + i);
        EI start = off > e0 ? off : e0;
        if (start < e1) s.mark[start - e0] = (uint16_t)k;
      }
    }
    __syncthreads();
    if (multi_row) {
      // inclusive max-scan of the marks: each thread owns ITEMS consecutive slots
      uint4 mv = reinterpret_cast<uint4*>(s.mark)[tid];
      uint32_t m8[8] = {mv.x & 0xFFFFu, mv.x >> 16, mv.y & 0xFFFFu, mv.y >> 16,
                        mv.z & 0xFFFFu, mv.z >> 16, mv.w & 0xFFFFu, mv.w >> 16};
      uint32_t run = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) { run = max(run, m8[j]); m8[j] = run; }
      const int lane = tid & 31, warp = tid >> 5;
      uint32_t incl = run;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl = max(incl, y);
      }
      uint32_t excl = __shfl_up_sync(0xffffffffu, incl, 1);
      if (lane == 0) excl = 0;
      if (lane == 31) s.wmark[warp] = incl;
      __syncthreads();
      uint32_t pre = excl;
      for (int w = 0; w < warp; ++w) pre = max(pre, s.wmark[w]);
#pragma unroll
      for (int j = 0; j < 8; ++j) m8[j] = max(m8[j], pre);
      reinterpret_cast<uint4*>(s.mark)[tid] =
          make_uint4(m8[0] | (m8[1] << 16), m8[2] | (m8[3] << 16), m8[4] | (m8[5] << 16),
                     m8[6] | (m8[7] << 16));
      __syncthreads();
    }

    // ---- stream the tile's edges: ITEMS independent loads per thread ----
    uint32_t col[ITEMS];
    K cand[ITEMS];
    uint32_t rowk[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const uint32_t idx = j * NT + tid;
      const EI e = e0 + idx;
      col[j] = 0xFFFFFFFFu;
      rowk[j] = 0;
      if (e < e1) {
        const uint32_t k = multi_row ? (uint32_t)s.mark[idx] : 0u;
        rowk[j] = k;
        WB w;
        EdgeAccess<V>::load(P, s.base[k] + e, col[j], w);
        cand[j] = VT::relax(s.key[k], w);
        if (!VT::usable(cand[j])) col[j] = 0xFFFFFFFFu;
      }
    }
    if (!PRED) {
      K cur[ITEMS];
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) cur[j] = (col[j] != 0xFFFFFFFFu) ? P.dist[col[j]] : (K)0;
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        const uint32_t v = col[j];
        if (v == 0xFFFFFFFFu || !(cand[j] < cur[j])) continue;
        if (v == src) {  // source guard (solver.py:299-303, :374-376, seed :236-239)
          P.st->flag = 1u;
          continue;
        }
        const K old = atomicMin(P.dist + v, cand[j]);
        if (!(cand[j] < old)) continue;
        const unsigned os = atomicMax(P.stamp + v, r << 1);
        if ((os >> 1) >= r) continue;  // already lowered earlier in this round
        round_w++;
        acc_w++;
        if (os == 0u) {
          acc_fd++;  // left infinity (first_discoveries, solver.py:378-379)
        } else {
          if (!(os & 1u)) acc_multi++;  // second round that lowers v
          atomicOr(P.stamp + v, 1u);
        }
        if (govm) {
          const EI a = __ldg(P.row_ptr + v), b = __ldg(P.row_ptr + v + 1);
          if (b > a) {  // rows without edges never need a rescan
            const int slot = atomicAdd(&s.qcnt, 1);
            s.qnode[slot] = v;
            s.qrs[slot] = a;
            s.qdeg[slot] = b - a;
          }
        }
      }
      if (govm) {
        // ---- flush the enqueue buffer: one packed reservation per tile ----
        __syncthreads();
        const int q = s.qcnt;
        if (q > 0) {
          EI carry = 0;
          for (int c0 = 0; c0 < q; c0 += NT) {
            const int i = c0 + tid;
            const EI d = (i < q) ? s.qdeg[i] : (EI)0;
            EI tot;
            const EI incl = block_incl_sum<EI>(d, s.scr, &tot);
            if (i < q) s.qdeg[i] = carry + incl - d;
            carry += tot;
          }
          if (tid == 0) {
            s.basepk = atomicAdd(&P.st->res[np],
                                 ((unsigned long long)q << P.ebits) | (unsigned long long)carry);
          }
          __syncthreads();
          const unsigned long long bp = s.basepk;
          const uint32_t bc = (uint32_t)pk_count(bp, P.ebits);
          const EI be = (EI)pk_edges(bp, P.ebits);
          for (int i = tid; i < q; i += NT) {
            const EI off = be + s.qdeg[i];
            P.qnode[np][bc + i] = s.qnode[i];
            P.qoff[np][bc + i] = off;
            P.qbase[np][bc + i] = s.qrs[i] - off;
          }
          __syncthreads();
          if (tid == 0) s.qcnt = 0;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        const uint32_t v = col[j];
        if (v == 0xFFFFFFFFu || v == src) continue;
        const unsigned sv = ldcg(P.stamp + v);
        if ((sv >> 1) != r) continue;
        if (cand[j] == ldcg(P.dist + v)) {
          const uint32_t u = s.qnode[rowk[j]];
          atomicMax(P.pred + v, ((unsigned long long)r << 32) | (unsigned long long)(~u));
        }
      }
    }
    __syncthreads();
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
  grid_sync(&P.st->bar);
  uint32_t* a = P.jmp0;
  uint32_t* b = P.jmp1;
  for (int it = 0; it < P.logn; ++it) {
    for (uint32_t v = gtid; v < n; v += gsz) b[v] = ldcg(a + ldcg(a + v));
    grid_sync(&P.st->bar);
    uint32_t* t = a; a = b; b = t;
  }
  for (uint32_t v = gtid; v < n; v += gsz) {
    if (v != src && ldcg(P.dist + v) != VT::INF && ldcg(a + v) != src) P.st->cyc = 1u;
  }
  grid_sync(&P.st->bar);
  return ldcg(&P.st->cyc) != 0u;
}

// ---------------------------------------------------------------------------
// the persistent kernel
// ---------------------------------------------------------------------------
template <class V, class EI>
__global__ void __launch_bounds__(NT) dawn_persistent(KParams<V, EI> P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<V, EI>& s = *reinterpret_cast<Smem<V, EI>*>(smem_raw);
  DevState* st = P.st;
  const bool leader = (blockIdx.x == 0 && threadIdx.x == 0);
  if (threadIdx.x == 0) s.qcnt = 0;
  __syncthreads();

  uint32_t r = ldcg(&st->round);
  unsigned long long acc_w = 0, acc_fd = 0, acc_multi = 0, acc_r = 0;
  unsigned rounds = 0;
  for (;;) {
    const int p = r & 1;
    // ---- termination (solver.py:284-285, :313-317, :356-358, :388-395) ----
    if (r >= 2) {
      const unsigned long long wprev = ldcg(&st->wround[(r - 1) & 1]);
      bool stop = false, capflag = false;
      if (r - 1 >= 2 && wprev == 0) stop = true;        // a loop round wrote nothing
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
      if (P.negcheck_period > 0 && r > 2 && ((r - 1) % (unsigned)P.negcheck_period) == 0) {
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
    if (rounds == P.max_rounds) {
      if (leader) st->round = r;
      break;
    }
    // ---- S phase ----
    if (leader) {
      st->res[p ^ 1] = 0ull;
      st->wround[p] = 0ull;
      st->tile_ctr[p] = 0u;
      st->tile_ctr2[p] = 0u;
    }
    if (P.algo == 1 && r >= 2) phase_compact_all<V, EI>(P, p, s);
    else phase_snapshot<V, EI>(P, p);
    grid_sync(&st->bar);
    // ---- X phase ----
    if (leader) acc_r += pk_edges(ldcg(&st->res[p]), P.ebits);  // relaxations (solver.py:297, :372)
    uint32_t round_w = 0;
    phase_expand<V, EI, false>(P, p, r, s, acc_w, acc_fd, acc_multi, round_w);
    round_w = __reduce_add_sync(0xffffffffu, round_w);
    if ((threadIdx.x & 31) == 0 && round_w) atomicAdd(&st->wround[p], (unsigned long long)round_w);
    grid_sync(&st->bar);
    if (P.pred_on) {
      phase_expand<V, EI, true>(P, p, r, s, acc_w, acc_fd, acc_multi, round_w);
      grid_sync(&st->bar);
    }
    ++r;
    ++rounds;
  }
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
// solve init: seed frontier {source} with key 0 (solver.py:275-280, :343-350)
template <class V, class EI>
__global__ void dawn_init_solve(KParams<V, EI> P) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    using VT = Val<V>;
    DevState* st = P.st;
    const uint32_t s = P.src;
    P.dist[s] = VT::enc((V)0);
    const EI a = P.row_ptr[s], b = P.row_ptr[s + 1];
    const unsigned long long deg = (unsigned long long)(b - a);
    st->res[0] = 0ull;
    st->res[1] = deg ? ((1ull << P.ebits) | deg) : 0ull;
    P.qnode[1][0] = s;
    P.qoff[1][0] = 0;
    P.qbase[1][0] = a;
    st->wround[0] = st->wround[1] = 0ull;
    st->tile_ctr[0] = st->tile_ctr[1] = 0u;
    st->tile_ctr2[0] = st->tile_ctr2[1] = 0u;
    st->round = 1u;
    st->done = 0u;
    st->flag = 0u;
    st->early = 0u;
    st->cyc = 0u;
    st->steps = 0ull;
    st->R = st->W = st->FD = st->multi = 0ull;
  }
}

template <class V>
__global__ void dawn_decode_dist(const typename Val<V>::K* __restrict__ keys, uint32_t n,
                                 double* __restrict__ out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = Val<V>::to_f64(keys[i]);
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
