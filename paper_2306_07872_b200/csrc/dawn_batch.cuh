// dawn_batch.cuh — batched multi-source weighted DAWN (K9 of SURVEY §7.2).
//
// Replaces the per-source loop of mssp / apsp (solver.py:426-495): up to 32
// sources advance together, one per warp lane.  Distances are stored
// node-major, bd[v][l] (l = source lane), so the 32 lanes of a warp that
// relax one edge (u, v, w) read and update one contiguous 128-byte line
// (4-byte values) — the edge's (col, w) is read once for all sources and
// the dist gather is a single coalesced request instead of 32 random ones.
//
// Round r of the batch (each lane follows exactly the snapshot-Jacobi
// semantics of the single-source kernel, so every per-source distance AND
// counter equals a single-source solve — DESIGN.md §Batched multi-source):
//
//   B (build): a coalesced sweep over nmask[v] = lanes that lowered v in
//      round r-1.  It clears nmask, does the write bookkeeping of round r-1
//      (writes, first discoveries, nodes lowered in >= 2 rounds: per-lane
//      counts via bit-sliced adds + warp bit transposes, no atomics), and lays the frontier of round r
//      out as entries {node, lane mask, edge offset, row base} plus a
//      32-lane snapshot of the row's distances (the value each lane relaxes
//      with, as of the start of the round).  GOVM: lane mask = lanes that
//      lowered the node (Alg. 2); GSVM: lanes where the node
//      is finite and the lane is still running (solver.py:287-289).
//   X (expand): warps stream WT-edge tiles of the frontier's virtual edge
//      list (merge-path balanced, as the single-source kernel).  Per edge,
//      each active lane forms cand = snap + w, reads its bd[v][lane]
//      (one 128 B line for the warp) and, when cand < cur, issues a
//      fire-and-forget red.min and the warp ORs the improved lanes into
//      nmask[v] (red.or): the strict `>` relax of solver.py:298, :373.
//
// Only graphs without negative weights take this path (raw-bit keys, no
// negative-cycle machinery); the host routes everything else to the
// single-source kernel, one source at a time.
#pragma once
#include "dawn_kernels.cuh"

namespace dawn {

#ifndef DAWN_BATCH_MIN_BLOCKS
#define DAWN_BATCH_MIN_BLOCKS 2  // resident CTAs per SM the batched kernel's registers are sized for
#endif

constexpr int BL = 32;    // sources per batch (warp lanes)
constexpr int BWT = 32;   // virtual edges per warp tile (<= 32 rows per tile)

struct BState {
  unsigned long long res[2];   // packed frontier reservation (count << ebits | edges), by round parity
  unsigned long long res_s[2]; // ... of the lane-sparse row list (async schedule), by round parity
  unsigned long long le[2];    // lane-edges (relaxations) of the round with this parity
  unsigned bar;                // grid barrier word (never reset)
  unsigned wrote[2];           // lanes that lowered any node in the round with this parity
  unsigned guard;              // lanes whose source guard fired (solver.py:299-303)
  unsigned abort;              // watchdog: the batch made no progress for 30 s and wound down
  unsigned rounds;             // rounds executed (incl. seeding)
  unsigned lastw[BL];          // per lane: last round that lowered a node (0 = none)
  unsigned long long R[BL], W[BL], FD[BL], MW[BL];
};

template <class V, class EI>
struct BParams {
  using K = typename Val<V>::K;
  uint32_t n;
  uint32_t nlanes;                 // sources in this batch (<= 32)
  const EI* row_ptr;
  const uint2* e2;
  const uint32_t* ecol;
  const unsigned long long* ew;
  K* bd;                           // [n][32] distance keys (raw bits)
  uint32_t* nmask;                 // [n] lanes that lowered the node this round
  uint32_t* w1;                    // [n] lanes that lowered it in >= 1 round
  uint32_t* w2;                    // [n] ... in >= 2 rounds
  uint32_t* smask;                 // [n] lanes whose source is the node (GSVM frontier)
  // frontier row lists: [0] = rows relaxed across the whole distance line,
  // [1] = rows with few active sources, relaxed lane by lane (async schedule)
  uint32_t* qnode[2];
  uint32_t* qmask[2];
  EI* qoff[2];
  EI* qbase[2];
  K* qkey;                         // [cap][32] snapshot of the frontier rows (list 0)
  uint32_t* tile_row[2];
  BState* st;
  uint32_t src[BL];                // lane -> source node (0xFFFFFFFF = unused lane)
  int ebits;
  int algo;                        // 0 = GOVM, 1 = GSVM
  uint32_t sparse_util;            // a round with lane-edges < this * edges relaxes lane-sparse;
                                   // async: rows with fewer active sources go to list 1
  unsigned long long* prof;        // optional per-round timeline, 4 words/round, or nullptr
  unsigned prof_cap;
};

template <class V, class EI>
struct __align__(16) BSmem {
  unsigned long long scr64[NT / 32];
  unsigned long long basepk, basepk_s;
  unsigned rl[BL];            // relaxations per source lane counted by lane-sparse rounds (< 2^32 per CTA)
  uint32_t src[BL];           // lane -> source node (lane-sparse source guard)
};

template <class V> struct BEdge;
template <> struct BEdge<float> {
  template <class P, class EI> __device__ __forceinline__ static void load(const P& p, EI pos, uint32_t& c, uint32_t& w) {
    uint2 x = ld_stream(p.e2 + pos); c = x.x; w = x.y;
  }
};
template <> struct BEdge<int32_t> {
  template <class P, class EI> __device__ __forceinline__ static void load(const P& p, EI pos, uint32_t& c, uint32_t& w) {
    uint2 x = ld_stream(p.e2 + pos); c = x.x; w = x.y;
  }
};
template <> struct BEdge<double> {
  template <class P, class EI> __device__ __forceinline__ static void load(const P& p, EI pos, uint32_t& c, unsigned long long& w) {
    c = ld_stream(p.ecol + pos); w = ld_stream(p.ew + pos);
  }
};
template <> struct BEdge<int64_t> {
  template <class P, class EI> __device__ __forceinline__ static void load(const P& p, EI pos, uint32_t& c, unsigned long long& w) {
    c = ld_stream(p.ecol + pos); w = ld_stream(p.ew + pos);
  }
};

template <class T>
__device__ __forceinline__ T shfl_any(T v, int src) {
  if constexpr (sizeof(T) == 8) {
    const unsigned long long x = (unsigned long long)v;
    unsigned lo = __shfl_sync(0xffffffffu, (unsigned)x, src);
    unsigned hi = __shfl_sync(0xffffffffu, (unsigned)(x >> 32), src);
    return (T)(((unsigned long long)hi << 32) | lo);
  } else {
    return (T)__shfl_sync(0xffffffffu, (unsigned)v, src);
  }
}

#ifndef DAWN_BATCH_CUR_CG
#define DAWN_BATCH_CUR_CG 1  // target lines through L2 only (ld.cg): fresher values, L1 kept for the row lines
#endif

#ifndef DAWN_BATCH_BKSLICE
#define DAWN_BATCH_BKSLICE 1  // per-lane write counts by bit-sliced adds + warp bit transposes
#endif

__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (c & (a ^ b)); }

// per-bit counts (0..8) of eight lane masks as four bit planes (carry-save adder tree)
__device__ __forceinline__ void csa8(const uint32_t (&q)[ITEMS], uint32_t (&p)[4]) {
  static_assert(ITEMS == 8, "csa8 sums eight masks");
  const uint32_t s1 = q[0] ^ q[1] ^ q[2], c1 = maj3(q[0], q[1], q[2]);
  const uint32_t s2 = q[3] ^ q[4] ^ q[5], c2 = maj3(q[3], q[4], q[5]);
  const uint32_t s3 = q[6] ^ q[7], c3 = q[6] & q[7];
  p[0] = s1 ^ s2 ^ s3;
  const uint32_t c4 = maj3(s1, s2, s3);
  const uint32_t s5 = c1 ^ c2 ^ c3, c5 = maj3(c1, c2, c3);
  p[1] = s5 ^ c4;
  const uint32_t c6 = s5 & c4;
  p[2] = c5 ^ c6;
  p[3] = c5 & c6;
}

// 32x32 bit transpose across the warp: lane b returns the word whose bit t is
// bit b of lane t's x
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, uint32_t lane) {
  constexpr uint32_t MK[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const uint32_t j = 16u >> s, m = MK[s];
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
    x = (lane & j) ? ((x & ~m) | ((y & ~m) >> j)) : ((x & m) | ((y & m) << j));
  }
  return x;
}

// lane b: how many of the warp's 32 x 8 masks have bit b set
__device__ __forceinline__ uint32_t warp_bitcount8(const uint32_t (&q)[ITEMS], uint32_t lane) {
  uint32_t p[4];
  csa8(q, p);
  uint32_t c = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) c += (uint32_t)__popc(warp_transpose32(p[i], lane)) << i;
  return c;
}

// ---------------------------------------------------------------------------
// B phase: consume nmask (round r-1's writes), build round r's frontier
// ---------------------------------------------------------------------------
template <class V, class EI, bool LIVE>
__device__ void bphase_build(const BParams<V, EI>& P, uint32_t r, uint32_t active, BSmem<V, EI>& s,
                             unsigned long long& accW, unsigned long long& accFD,
                             unsigned long long& accMW) {
  using K = typename Val<V>::K;
  const uint32_t n = P.n;
  const uint32_t nchunks = (n + TILE - 1) / TILE;
  const uint32_t lane = threadIdx.x & 31;
  const int eb = P.ebits;
  const bool gsvm = P.algo == 1 && r >= 2;
  for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint32_t u0 = c * TILE + threadIdx.x * ITEMS;
    const bool full = u0 + ITEMS <= n;
    // every load of the chunk up front (lane masks, write states, row bounds):
    // conditional loads behind each other — and behind the bookkeeping stores,
    // which the compiler cannot reorder them past — made a serial chain
    uint32_t M[ITEMS], W1[ITEMS], W2[ITEMS];
    EI rp[ITEMS + 1];
    if (full) {
      ldcg8<uint32_t>(P.nmask + u0, M);
      ldcg8<uint32_t>(P.w1 + u0, W1);
      ldcg8<uint32_t>(P.w2 + u0, W2);
      ldg8<EI>(P.row_ptr + u0, *reinterpret_cast<EI(*)[ITEMS]>(rp));
      rp[ITEMS] = __ldg(P.row_ptr + u0 + ITEMS);
    } else {
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        const bool in = u0 + j < n;
        M[j] = in ? ldcg(P.nmask + u0 + j) : 0u;
        W1[j] = in ? ldcg(P.w1 + u0 + j) : 0u;
        W2[j] = in ? ldcg(P.w2 + u0 + j) : 0u;
        rp[j] = (u0 + j <= n) ? __ldg(P.row_ptr + u0 + j) : (EI)0;
      }
      rp[ITEMS] = (u0 + ITEMS <= n) ? __ldg(P.row_ptr + u0 + ITEMS) : (EI)0;
    }
    uint32_t anyM = 0;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) anyM |= M[j];
    if (r >= 2) {
      // ---- write bookkeeping of round r-1 (the seeding round's frontier is not a write) ----
      uint32_t FDm[ITEMS], MWm[ITEMS];
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) { FDm[j] = 0; MWm[j] = 0; }
      if (anyM) {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
          FDm[j] = M[j] & ~W1[j];
          MWm[j] = M[j] & W1[j] & ~W2[j];
          W2[j] |= M[j] & W1[j];
          W1[j] |= M[j];
        }
        if (full) {
          reinterpret_cast<uint4*>(P.w1 + u0)[0] = make_uint4(W1[0], W1[1], W1[2], W1[3]);
          reinterpret_cast<uint4*>(P.w1 + u0)[1] = make_uint4(W1[4], W1[5], W1[6], W1[7]);
          reinterpret_cast<uint4*>(P.w2 + u0)[0] = make_uint4(W2[0], W2[1], W2[2], W2[3]);
          reinterpret_cast<uint4*>(P.w2 + u0)[1] = make_uint4(W2[4], W2[5], W2[6], W2[7]);
          reinterpret_cast<uint4*>(P.nmask + u0)[0] = make_uint4(0, 0, 0, 0);
          reinterpret_cast<uint4*>(P.nmask + u0)[1] = make_uint4(0, 0, 0, 0);
        } else {
#pragma unroll
          for (int j = 0; j < ITEMS; ++j)
            if (u0 + j < n) { P.w1[u0 + j] = W1[j]; P.w2[u0 + j] = W2[j]; P.nmask[u0 + j] = 0u; }
        }
      }
#if DAWN_BATCH_BKSLICE
      // per-lane counts: lane b sums bit b over the warp's 256 nodes — the eight
      // masks of a thread added bit-sliced, the planes transposed across the warp
      if (__any_sync(0xffffffffu, anyM != 0u)) {
        accW += warp_bitcount8(M, lane);
        accFD += warp_bitcount8(FDm, lane);
        accMW += warp_bitcount8(MWm, lane);
      }
#else
      // per-lane counts: lane b sums bit b over the warp's nodes (one REDUX per bit)
#pragma unroll 1
      for (int j = 0; j < ITEMS; ++j) {
        if (__any_sync(0xffffffffu, M[j] != 0u)) {
#pragma unroll 4
          for (int b = 0; b < BL; ++b) {
            const uint32_t x = ((M[j] >> b) & 1u) | (((FDm[j] >> b) & 1u) << 10) | (((MWm[j] >> b) & 1u) << 20);
            const uint32_t t = __reduce_add_sync(0xffffffffu, x);
            if (lane == (uint32_t)b) {
              accW += t & 1023u;
              accFD += (t >> 10) & 1023u;
              accMW += t >> 20;
            }
          }
        }
      }
#endif
    } else if (anyM) {
      if (full) {
        reinterpret_cast<uint4*>(P.nmask + u0)[0] = make_uint4(0, 0, 0, 0);
        reinterpret_cast<uint4*>(P.nmask + u0)[1] = make_uint4(0, 0, 0, 0);
      } else {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j)
          if (u0 + j < n) P.nmask[u0 + j] = 0u;
      }
    }
    // ---- frontier of round r ----
    uint32_t F[ITEMS];
    if (gsvm) {
      uint32_t SM[ITEMS];
      if (full) ldcg8<uint32_t>(P.smask + u0, SM);
      else {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) SM[j] = (u0 + j < n) ? ldcg(P.smask + u0 + j) : 0u;
      }
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) F[j] = (W1[j] | SM[j]) & active;
    } else {
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) F[j] = M[j];
    }
    uint32_t anyF = 0;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) anyF |= F[j];
    unsigned sel = 0, sel_s = 0;  // rows of list 0 / list 1 (few active sources, async)
    uint32_t mycnt = 0, mycnt_s = 0;
    EI mydeg = 0, mydeg_s = 0;
    if (anyF) {
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        if (F[j] && u0 + j < n && rp[j + 1] > rp[j]) {
          if (LIVE && (uint32_t)__popc(F[j]) < P.sparse_util) {
            sel_s |= 1u << j;
            mycnt_s++;
            mydeg_s += rp[j + 1] - rp[j];
          } else {
            sel |= 1u << j;
            mycnt++;
            mydeg += rp[j + 1] - rp[j];
          }
        }
      }
    }
    const unsigned long long mine = ((unsigned long long)mycnt << eb) | (unsigned long long)mydeg;
    unsigned long long tot;
    const unsigned long long incl = block_incl_sum<unsigned long long>(mine, s.scr64, &tot);
    if (threadIdx.x == 0 && tot != 0ull) s.basepk = atomicAdd(&P.st->res[r & 1], tot);
    unsigned long long mine_s = 0, incl_s = 0;
    if (LIVE) {
      __syncthreads();  // scr64 reuse
      mine_s = ((unsigned long long)mycnt_s << eb) | (unsigned long long)mydeg_s;
      unsigned long long tot_s;
      incl_s = block_incl_sum<unsigned long long>(mine_s, s.scr64, &tot_s);
      if (threadIdx.x == 0 && tot_s != 0ull) s.basepk_s = atomicAdd(&P.st->res_s[r & 1], tot_s);
    }
    __syncthreads();
    if (!__any_sync(0xffffffffu, (sel | sel_s) != 0u)) continue;
    {  // lane-edges of round r: chooses the relax mode of the X phase (and the profile)
      unsigned long long le = 0;
#pragma unroll
      for (int j = 0; j < ITEMS; ++j)
        if (((sel | sel_s) >> j) & 1u) le += (unsigned long long)__popc(F[j]) * (unsigned long long)(rp[j + 1] - rp[j]);
      le = warp_sum_u64(le);
      if (lane == 0 && le) {
        atomicAdd(&P.st->le[r & 1], le);
        if (P.prof != nullptr && r < P.prof_cap) atomicAdd(P.prof + 4 * r + 3, le);
      }
    }
    // this thread's entries: metadata, tile marks and the 32-lane snapshot
    // (one full 128/256-byte line per entry, vector loads all in flight)
#pragma unroll 1
    for (int q = 0; q < (LIVE ? 2 : 1); ++q) {
      const unsigned qs = q ? sel_s : sel;
      if (!__any_sync(0xffffffffu, qs != 0u)) continue;  // warp-uniform: the tile marks are warp-collective
      const unsigned long long at = q ? s.basepk_s + incl_s - mine_s : s.basepk + incl - mine;
      uint32_t pos = (uint32_t)pk_count(at, eb);
      EI off = (EI)pk_edges(at, eb);
      constexpr int NV = BL * (int)sizeof(K) / 16;
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        const bool has = (qs >> j) & 1u;
        const EI dg = has ? rp[j + 1] - rp[j] : (EI)0;
        if (has) {
          const uint32_t v = u0 + j;
          const uint4* srcl = reinterpret_cast<const uint4*>(P.bd + (size_t)v * BL);
          uint4* dstl = reinterpret_cast<uint4*>(P.qkey + (size_t)pos * BL);
          uint4 x[8];
          if (!LIVE) {
#pragma unroll
            for (int qq = 0; qq < 8; ++qq) x[qq] = __ldcg(srcl + qq);
          }
          P.qnode[q][pos] = v;
          P.qmask[q][pos] = F[j];
          P.qoff[q][pos] = off;
          P.qbase[q][pos] = rp[j] - off;
          if (!LIVE) {  // the async schedule reads the live line instead
#pragma unroll
            for (int qq = 0; qq < 8; ++qq) dstl[qq] = x[qq];
#pragma unroll
            for (int h = 8; h < NV; h += 8) {  // 8-byte keys: second half of the line
#pragma unroll
              for (int qq = 0; qq < 8; ++qq) x[qq] = __ldcg(srcl + h + qq);
#pragma unroll
              for (int qq = 0; qq < 8; ++qq) dstl[h + qq] = x[qq];
            }
          }
        }
        mark_tiles_warp<BWT, EI>(P.tile_row[q], has, off, dg, pos);
        if (has) {
          pos++;
          off += dg;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// X phase.  A thread owns LPT = 16 / sizeof(key) consecutive source lanes of
// one edge (one 16-byte vector of the node's distance line), so TPE = 32/LPT
// threads cover an edge and a warp relaxes EPW = LPT edges per step; the
// (col, w) pairs and row lookups of 32 edges are loaded cooperatively first.
// ---------------------------------------------------------------------------
template <class V>
struct BLanes {
  using K = typename Val<V>::K;
  static constexpr int LPT = 16 / (int)sizeof(K);
  static constexpr int TPE = BL / LPT;
  static constexpr int EPW = 32 / TPE;
  static constexpr uint32_t LMASK = (1u << LPT) - 1u;
};

template <class K, int LPT>
__device__ __forceinline__ void ld16_ca(const K* p, K (&o)[LPT], bool cg = false) {
  const uint4 x = cg ? __ldcg(reinterpret_cast<const uint4*>(p)) : __ldca(reinterpret_cast<const uint4*>(p));
  if constexpr (LPT == 4) {
    o[0] = (K)x.x; o[1] = (K)x.y; o[2] = (K)x.z; o[3] = (K)x.w;
  } else {
    o[0] = (K)(((unsigned long long)x.y << 32) | x.x);
    o[1] = (K)(((unsigned long long)x.w << 32) | x.z);
  }
}

// One 32-edge tile of the frontier's virtual edge list as a warp sees it:
// lane j holds edge j (column, weight, row index relative to i0) and lane k
// holds row i0+k's lane mask (a tile spans at most 32 rows: its first row
// owns edge 0, every other row starts inside it).
template <class WB>
struct BTile {
  uint32_t i0;     // first entry
  uint32_t len;    // edges in the tile (0 = no tile)
  uint32_t col;    // lane j: column of edge j
  WB w;            // lane j: weight bits of edge j
  uint32_t kr;     // lane j: row of edge j, relative to i0
  uint32_t rmask;  // lane k: lane mask of row i0+k
  uint32_t rnode;  // lane k: node of row i0+k (async schedule)
};

template <class V, class EI>
struct BRows {        // row metadata of a tile in flight
  uint32_t i0, il;
  EI off, base;       // lane k: row i0+k
  uint32_t rmask;
  uint32_t rnode;
};

// the row range [i0, il] of tile t (first stage of a row load)
template <class V, class EI>
__device__ __forceinline__ void brows_bounds(const BParams<V, EI>& P, int q, EI t, EI T, uint32_t cnt,
                                             uint32_t& i0, uint32_t& il) {
  i0 = __ldca(P.tile_row[q] + t);
  il = (t + 1 < T) ? __ldca(P.tile_row[q] + t + 1) : cnt - 1;
}

// the rows' metadata once the range is known (second stage)
template <class V, class EI, bool LIVE>
__device__ __forceinline__ void brows_finish(const BParams<V, EI>& P, int q, uint32_t i0, uint32_t il, uint32_t lane,
                                             BRows<V, EI>& R) {
  R.i0 = i0;
  R.il = il;
  R.off = 0;
  R.base = 0;
  R.rmask = 0;
  R.rnode = 0;
  if (lane <= R.il - R.i0) {
    R.off = __ldca(P.qoff[q] + R.i0 + lane);
    R.base = __ldca(P.qbase[q] + R.i0 + lane);
    R.rmask = __ldca(P.qmask[q] + R.i0 + lane);
    if (LIVE) R.rnode = __ldca(P.qnode[q] + R.i0 + lane);
  }
}

template <class V, class EI, bool LIVE>
__device__ __forceinline__ void brows_load(const BParams<V, EI>& P, int q, EI t, EI T, uint32_t cnt, uint32_t lane,
                                           BRows<V, EI>& R) {
  uint32_t i0, il;
  brows_bounds<V, EI>(P, q, t, T, cnt, i0, il);
  brows_finish<V, EI, LIVE>(P, q, i0, il, lane, R);
}

// row of every edge (row-start bits + popc), then the edge loads
template <class V, class EI>
__device__ __forceinline__ void btile_issue(const BParams<V, EI>& P, EI t, EI E, uint32_t lane,
                                            const BRows<V, EI>& R, BTile<typename Val<V>::K>& X) {
  const EI e0 = t * (EI)BWT;
  X.len = (E - e0 < (EI)BWT) ? (uint32_t)(E - e0) : (uint32_t)BWT;
  X.i0 = R.i0;
  X.rmask = R.rmask;
  X.rnode = R.rnode;
  const uint32_t nrows = R.il - R.i0 + 1;
  const uint32_t rst = (lane < nrows && R.off >= e0 && R.off - e0 < (EI)32) ? (uint32_t)(R.off - e0) : 32u;
  const uint32_t B = __reduce_or_sync(0xffffffffu, rst < 32u ? (1u << rst) : 0u);
  const uint32_t start0 = B & 1u;  // row i0 starts exactly at the tile
  X.kr = (uint32_t)__popc(B & (0xFFFFFFFFu >> (31 - lane))) - start0;
  const EI base = shfl_any<EI>(R.base, (int)X.kr);
  X.col = 0;
  X.w = 0;
  if (lane < X.len) BEdge<V>::load(P, base + e0 + (EI)lane, X.col, X.w);
}

// SPARSE: lane-sparse rounds (few active sources per frontier row, e.g. the
// first rounds, where every source still explores its own neighbourhood): a
// thread owns one edge and walks the row's set lanes one by one (scalar
// gathers), instead of 8 threads covering all 32 lanes of the distance line.
template <class V, class EI, bool SPARSE, bool LIVE>
__device__ void bphase_expand(const BParams<V, EI>& P, int q, uint32_t r, const uint32_t (&msrc)[BLanes<V>::LPT],
                              unsigned& guard, unsigned& wrote, unsigned long long (&accR)[BLanes<V>::LPT],
                              BSmem<V, EI>& sm) {
  using CD = Codec<V, true>;
  using K = typename CD::K;
  using WB = typename CD::WB;
  constexpr int LPT = BLanes<V>::LPT, TPE = BLanes<V>::TPE, EPW = BLanes<V>::EPW;
  constexpr uint32_t LMASK = BLanes<V>::LMASK;
  constexpr int STEPS = 32 / EPW;               // warp steps per tile
#ifndef DAWN_BATCH_U
#define DAWN_BATCH_U 4
#endif
  constexpr int U = sizeof(K) == 4 ? DAWN_BATCH_U : 2;  // steps in flight
  // a candidate is usable iff it is below +inf: clamp the current value there,
  // so `cand < min(cur, +inf)` is the reference's `alpha[idx] > cand` with an
  // infinite candidate never written (solver.py:298, :373)
  constexpr K CAP = std::is_same<V, float>::value ? (K)0x7F800000u
                  : std::is_same<V, double>::value ? (K)0x7FF0000000000000ull : CD::INF;
  const unsigned long long pk = ldcg(q ? &P.st->res_s[r & 1] : &P.st->res[r & 1]);
  const uint32_t cnt = (uint32_t)pk_count(pk, P.ebits);
  const EI E = (EI)pk_edges(pk, P.ebits);
  if (E == 0) return;
  const EI T = (E + (EI)(BWT - 1)) / (EI)BWT;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t sub = lane % TPE, eg = lane / TPE;
  const uint32_t lsh = sub * LPT;  // first source lane of this thread
  const EI GW = (EI)gridDim.x * WPB;
  EI t = (EI)blockIdx.x * WPB + wid;
  if (t >= T) return;  // warp-uniform
  // software pipeline (depth 3): edges of tile t and t+GW in flight, rows of
  // t+2GW in flight and the row range of t+3GW, while tile t's distance lines
  // are gathered and relaxed
  BTile<WB> A, Bt;
  BRows<V, EI> Rn;
  {
    BRows<V, EI> R0;
    brows_load<V, EI, LIVE>(P, q, t, T, cnt, lane, R0);
    btile_issue<V, EI>(P, t, E, lane, R0, A);
  }
  Bt.len = 0;
  if (t + GW < T) {
    BRows<V, EI> R1;
    brows_load<V, EI, LIVE>(P, q, t + GW, T, cnt, lane, R1);
    btile_issue<V, EI>(P, t + GW, E, lane, R1, Bt);
  }
  bool have_rn = t + 2 * GW < T;
  if (have_rn) brows_load<V, EI, LIVE>(P, q, t + 2 * GW, T, cnt, lane, Rn);
  // and the row range of t+3GW (its metadata loads wait on it: one stage ahead)
  uint32_t nb_i0 = 0, nb_il = 0;
  if (t + 3 * GW < T) brows_bounds<V, EI>(P, q, t + 3 * GW, T, cnt, nb_i0, nb_il);
  // relaxations (solver.py:297, :372) of this thread's lanes: LPT 8/16-bit
  // counters packed in one register (a thread sees STEPS <= 16 edges per tile),
  // flushed into accR after every tile
  constexpr uint32_t SPREAD = LPT == 4 ? 0x204081u : 0x8001u;     // bit i -> field i
  constexpr uint32_t FMASK = LPT == 4 ? 0x01010101u : 0x00010001u;
  constexpr int FBITS = LPT == 4 ? 8 : 16;
  for (;;) {
    if constexpr (SPARSE) {
      // ---- relax tile A, lane-sparse: lane j = edge j, loop over the row's lanes ----
      const uint32_t mrow = __shfl_sync(0xffffffffu, A.rmask, A.kr & 31);
      uint32_t lanes = lane < A.len ? mrow : 0u;
      // the row's line: its round-start snapshot, or (async) the live line bd[u]
      const uint32_t rnode = LIVE ? __shfl_sync(0xffffffffu, A.rnode, A.kr & 31) : 0u;
      const K* rowl = LIVE ? P.bd + (size_t)rnode * BL : P.qkey + (size_t)(A.i0 + A.kr) * BL;
      while (lanes) {
        const uint32_t l = __ffs(lanes) - 1;
        lanes &= lanes - 1u;
        atomicAdd(&sm.rl[l], 1u);  // relaxation of source lane l (solver.py:297, :372)
        const K c = CD::relax(CD::dec(__ldca(rowl + l)), A.w);
        const K cur = __ldca(P.bd + (size_t)A.col * BL + l);
        if (c < CAP && c < cur) {
          if (A.col == sm.src[l]) {
            guard |= 1u << l;  // source guard (solver.py:299-303)
          } else {
            atomicMin(P.bd + (size_t)A.col * BL + l, c);
            atomicOr(P.nmask + A.col, 1u << l);
            wrote |= 1u << l;
          }
        }
      }
    } else {
    // ---- relax tile A ----
    uint32_t rcp = 0;
#pragma unroll 1
    for (int q0 = 0; q0 < STEPS; q0 += U) {
      if ((uint32_t)(q0 * EPW) >= A.len) break;  // warp-uniform
      K cand[U][LPT], cur[U][LPT];
      uint32_t vq[U], am[U];
      WB wq[U];
      // every load of the U steps first — the rows' own lines (snapshot, or the
      // live line under async) into cand[], the targets' lines into cur[] —
      // then the candidates: a row line loaded inside the step and consumed at
      // once serialised the steps of short-row tiles
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t j = (uint32_t)((q0 + u) * EPW) + eg;
        vq[u] = __shfl_sync(0xffffffffu, A.col, j & 31);
        const uint32_t kq = __shfl_sync(0xffffffffu, A.kr, j & 31);
        wq[u] = shfl_any<WB>(A.w, j & 31);
        const uint32_t mq = __shfl_sync(0xffffffffu, A.rmask, kq & 31);
        const uint32_t nq = LIVE ? __shfl_sync(0xffffffffu, A.rnode, kq & 31) : 0u;
        const uint32_t a = (j < A.len) ? ((mq >> lsh) & LMASK) : 0u;
        ld16_ca<K, LPT>((LIVE ? P.bd + (size_t)nq * BL : P.qkey + (size_t)(A.i0 + kq) * BL) + lsh, cand[u]);
        rcp += (a * SPREAD) & FMASK;
        am[u] = a;
        // threads without an active lane still read their part of the edge's own
        // target line (unpredicated, one request per line; predicating them off or
        // pointing them at another line was slower)
        ld16_ca<K, LPT>(P.bd + (size_t)vq[u] * BL + lsh, cur[u], DAWN_BATCH_CUR_CG != 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int i = 0; i < LPT; ++i) cand[u][i] = CD::relax(CD::dec(cand[u][i]), wq[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        uint32_t imp = 0;
#pragma unroll
        for (int i = 0; i < LPT; ++i) {
          const K cc = cur[u][i] < CAP ? cur[u][i] : CAP;
          imp |= (((am[u] >> i) & 1u) && cand[u][i] < cc) ? (1u << i) : 0u;
        }
        if (imp) {
#pragma unroll
          for (int i = 0; i < LPT; ++i) {
            if ((imp >> i) & 1u) {
              if (vq[u] == msrc[i]) {  // source guard (solver.py:299-303)
                guard |= 1u << (lsh + i);
                imp &= ~(1u << i);
              } else {
                atomicMin(P.bd + (size_t)vq[u] * BL + lsh + i, cand[u][i]);
              }
            }
          }
          if (imp) atomicOr(P.nmask + vq[u], imp << lsh);
          wrote |= imp << lsh;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < LPT; ++i) accR[i] += (rcp >> (FBITS * i)) & ((1u << FBITS) - 1u);
    }  // dense lanes
    // ---- advance the pipeline ----
    if (Bt.len == 0) break;  // warp-uniform: no next tile
    t += GW;
    A = Bt;
    Bt.len = 0;
    if (have_rn) {
      btile_issue<V, EI>(P, t + GW, E, lane, Rn, Bt);
      have_rn = t + 2 * GW < T;
      if (have_rn) {
        brows_finish<V, EI, LIVE>(P, q, nb_i0, nb_il, lane, Rn);
        if (t + 3 * GW < T) brows_bounds<V, EI>(P, q, t + 3 * GW, T, cnt, nb_i0, nb_il);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// the persistent batched kernel
// ---------------------------------------------------------------------------
template <class V, class EI, bool LIVE>
__global__ void __launch_bounds__(NT, DAWN_BATCH_MIN_BLOCKS) dawn_batch_persistent(BParams<V, EI> P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BSmem<V, EI>& s = *reinterpret_cast<BSmem<V, EI>*>(smem_raw);
  BState* st = P.st;
  const uint32_t lane = threadIdx.x & 31;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  constexpr int LPT = BLanes<V>::LPT;
  uint32_t msrc[LPT];  // sources of this thread's lanes in the X phase
#pragma unroll
  for (int i = 0; i < LPT; ++i) msrc[i] = P.src[(lane % BLanes<V>::TPE) * LPT + i];
  unsigned long long accW = 0, accFD = 0, accMW = 0;
  unsigned long long accR[BLanes<V>::LPT];  // relaxations of this thread's X-phase lanes
#pragma unroll
  for (int i = 0; i < BLanes<V>::LPT; ++i) accR[i] = 0;
  unsigned guard = 0;
  uint32_t lastw = 0;  // this lane's last writing round (identical in every thread of the lane)
  const uint32_t valid = __ballot_sync(0xffffffffu, lane < P.nlanes);
  uint32_t active = valid;
  if (threadIdx.x < BL) {
    s.rl[threadIdx.x] = 0u;
    s.src[threadIdx.x] = P.src[threadIdx.x];
  }
  __syncthreads();
  uint32_t r = 1;
  // Round r = B(r) [builds into res[r&1]] | barrier | X(r) [ORs its writers into
  // wrote[r&1]] | barrier.  Double-buffered by parity, so every reset happens
  // a full barrier after the last read of the slot and before its next write.
  for (;; ++r) {
    if (r >= 2) {
      // ---- round r-1's writers; termination (solver.py:284-285, :356-358, :388-395) ----
      const unsigned wr = ldcg(&st->wrote[(r - 1) & 1]);
      if ((wr >> lane) & 1u) lastw = r - 1;
      if (r >= 3) active &= wr;  // a lane runs round r iff it wrote in r-1 (round 2 always runs)
      if (r >= 3 && wr == 0u) break;
      if (r - 1 >= P.n) break;
    }
    // ---- B phase ----
    const bool prof = leader && P.prof != nullptr && r < P.prof_cap;
    if (prof) P.prof[4 * r + 0] = globaltimer();
    if (leader) {  // last read by X(r-1), next written by B(r+1)
      st->res[(r + 1) & 1] = 0ull;
      st->res_s[(r + 1) & 1] = 0ull;
      st->le[(r + 1) & 1] = 0ull;
    }
    bphase_build<V, EI, LIVE>(P, r, active, s, accW, accFD, accMW);
    if (grid_sync(&st->bar, &st->abort)) break;
    // ---- X phase ----
    if (prof) {
      P.prof[4 * r + 1] = globaltimer();
      P.prof[4 * r + 2] = ldcg(&st->res[r & 1]);
    }
    if (leader) st->wrote[(r + 1) & 1] = 0u;  // last read at the top of round r, next written by X(r+1)
    unsigned wrote = 0;
    {
      // lane-sparse relax when the round's rows carry few active sources on average
      const unsigned long long E = pk_edges(ldcg(&st->res[r & 1]), P.ebits);
      const unsigned long long LE = ldcg(&st->le[r & 1]);
      if (LIVE) {  // rows split by their active sources in the B phase
        bphase_expand<V, EI, false, LIVE>(P, 0, r, msrc, guard, wrote, accR, s);
        bphase_expand<V, EI, true, LIVE>(P, 1, r, msrc, guard, wrote, accR, s);
      } else if (LE < (unsigned long long)P.sparse_util * E) {
        bphase_expand<V, EI, true, LIVE>(P, 0, r, msrc, guard, wrote, accR, s);
      } else {
        bphase_expand<V, EI, false, LIVE>(P, 0, r, msrc, guard, wrote, accR, s);
      }
    }
    wrote = __reduce_or_sync(0xffffffffu, wrote);
    if (lane == 0 && wrote) atomicOr(&st->wrote[r & 1], wrote);
    if (grid_sync(&st->bar, &st->abort)) break;
  }
  // ---- per-lane results ----
  if (leader) st->rounds = r - 1;
  if (leader && P.prof != nullptr && r < P.prof_cap) P.prof[4 * r + 0] = globaltimer();
  guard = __reduce_or_sync(0xffffffffu, guard);
  if (lane == 0 && guard) atomicOr(&st->guard, guard);
  // block-level reduction of the per-lane counters, then one atomic per lane per CTA
  __shared__ unsigned long long red[NT / 32][BL][4];
  const uint32_t wid = threadIdx.x >> 5;
  // R: lanes with the same sub own the same source lanes; fold them, then the
  // eg == 0 thread of each sub writes its LPT lanes
  {
    constexpr int TPE = BLanes<V>::TPE;
#pragma unroll
    for (int i = 0; i < BLanes<V>::LPT; ++i) {
#pragma unroll
      for (int d = TPE; d < 32; d <<= 1) accR[i] += __shfl_xor_sync(0xffffffffu, accR[i], d);
    }
    if (lane < (uint32_t)TPE) {
#pragma unroll
      for (int i = 0; i < BLanes<V>::LPT; ++i) red[wid][lane * BLanes<V>::LPT + i][0] = accR[i];
    }
  }
  red[wid][lane][1] = accW;
  red[wid][lane][2] = accFD;
  red[wid][lane][3] = accMW;
  __syncthreads();
  if (threadIdx.x < BL * 4) {
    const uint32_t l = threadIdx.x >> 2, f = threadIdx.x & 3;
    unsigned long long sum = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) sum += red[w][l][f];
    if (f == 0) sum += (unsigned long long)s.rl[l];  // relaxations counted by lane-sparse rounds
    if (sum) {
      unsigned long long* dst = f == 0 ? st->R : f == 1 ? st->W : f == 2 ? st->FD : st->MW;
      atomicAdd(dst + l, sum);
    }
  }
  if (blockIdx.x == 0 && wid == 0) st->lastw[lane] = lastw;
}

// batch init: sources' own distance 0, their bit in nmask (the seeding
// frontier) and smask; everything else was memset by the host.
template <class V, class EI>
__global__ void dawn_batch_init(BParams<V, EI> P) {
  const uint32_t l = threadIdx.x;
  if (l < P.nlanes) {
    const uint32_t s = P.src[l];
    P.bd[(size_t)s * BL + l] = Codec<V, true>::enc((V)0);
    atomicOr(P.nmask + s, 1u << l);
    atomicOr(P.smask + s, 1u << l);
  }
  if (l == 0) {
    BState* st = P.st;
    st->res[0] = st->res[1] = 0ull;
    st->res_s[0] = st->res_s[1] = 0ull;
    st->le[0] = st->le[1] = 0ull;
    st->wrote[0] = st->wrote[1] = 0u;
    st->guard = 0u;
    st->abort = 0u;
    st->rounds = 0u;
  }
  if (l < BL) {
    P.st->lastw[l] = 0u;
    P.st->R[l] = P.st->W[l] = P.st->FD[l] = P.st->MW[l] = 0ull;
  }
}

// bd[n][32] -> out[l][n] for l < nlanes (row-major source x node), via a
// 32x32 shared-memory transpose.  OUT = double (reference DistanceVector)
// or the value type itself (device-resident tiles).
template <class V, class OUT>
__global__ void dawn_batch_decode(const typename Val<V>::K* __restrict__ bd, uint32_t n, uint32_t nlanes,
                                  OUT* __restrict__ out, size_t ld) {
  __shared__ OUT tile[32][33];
  const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
  for (uint32_t v0 = blockIdx.x * 32; v0 < n; v0 += gridDim.x * 32) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t v = v0 + ty + 8 * k;
      OUT x = 0;
      if (v < n) {
        const typename Val<V>::K key = bd[(size_t)v * BL + tx];
        x = (OUT)Codec<V, true>::to_f64(key);
      }
      tile[ty + 8 * k][tx] = x;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t l = ty + 8 * k;
      const uint32_t v = v0 + tx;
      if (l < nlanes && v < n) out[(size_t)l * ld + v] = tile[tx][l];
    }
    __syncthreads();
  }
}

}  // namespace dawn
