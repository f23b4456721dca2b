/*
 * dawn.h — C ABI of the B200-native weighted-DAWN shortest-path library (libdawn.so).
 *
 * This is the drop-in boundary for the reference package `sparsepath`
 * (/root/reference/pkg/src/sparsepath).  Every entry point below replaces one
 * function of the reference's hot path; the citation next to each one names
 * the reference symbol (file:line) whose behaviour it reproduces.  The
 * reference is pure Python, so the "FFI binding a maintainer would add" is a
 * ctypes stub; INTEGRATION.md shows it.
 *
 * Conventions
 *   - All functions return an int status: DAWN_OK (0) or a DAWN_E* code.
 *     dawn_last_error() returns a thread-local message for the last failure.
 *   - Plain pointers and sizes only.  `stream` is a cudaStream_t passed as
 *     void* (NULL = legacy default stream).
 *   - Host arrays use the reference's CsrGraph layout (graph.py:64-109):
 *     int64 row_ptr[n+1], int64 col[m], float64 val[m].
 *   - Distances come back as float64 with +inf for unreachable nodes, the
 *     reference's DistanceVector.dist contract (solver.py:66-71).
 *   - Negative cycles are not errors: they set dawn_stats_t.negative_cycle,
 *     as the reference does (solver.py:17-24).
 *   - No CPU fallback: every solve runs on the GPU; without a CUDA device the
 *     calls fail with DAWN_ECUDA.
 */
#ifndef DAWN_H_
#define DAWN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DAWN_ABI_VERSION 1

/* status codes */
#define DAWN_OK 0
#define DAWN_EINVAL 1        /* bad argument (maps to ValueError) */
#define DAWN_ESOURCE 2       /* source out of range (ValueError "source s out of range for n=N", solver.py:253-255) */
#define DAWN_ECUDA 3         /* CUDA runtime failure / no device (RuntimeError) */
#define DAWN_ENOMEM 4        /* device allocation failed */
#define DAWN_EUNSUPPORTED 5  /* graph too large for the packed frontier reservation, etc. */

/* value (distance/weight) types on the device */
#define DAWN_I32 0
#define DAWN_I64 1
#define DAWN_F32 2
#define DAWN_F64 3

/* precision policy for dawn_choose_vtype */
#define DAWN_PREC_AUTO 0  /* integral weights -> I32/I64 (bit-exact vs the fp64 reference); else F64 */
#define DAWN_PREC_FP32 1  /* opt-in: F32 weights and accumulation (<= 1e-6 relative, north_star) */
#define DAWN_PREC_FP64 2  /* always F64 (bit-exact vs the reference's Python floats) */

/* algorithms (the reference's SOLVERS registry, solver.py:402) */
#define DAWN_GOVM 0  /* frontier rescans, govm_sssp solver.py:324-399 */
#define DAWN_GSVM 1  /* full rescans,     gsvm_sssp solver.py:265-321 */

/* solve flags */
#define DAWN_F_PRED 1u        /* record predecessors (record_pred=True, solver.py:309-310, :383-384) */
#define DAWN_F_NEGCHECK 2u    /* early negative-cycle exit via predecessor-graph cycle check
                                 (integer types only; same verdict as the n-round cap, solver.py:394-395) */
#define DAWN_F_PROFILE 4u     /* solver flag: record a per-round device timeline (globaltimer) */
#define DAWN_F_ASYNC 8u       /* solve flag: "async" schedule — a frontier row is relaxed with its LIVE
                                 distance (possibly lowered earlier in the same round, as in the
                                 reference's in-place order, solver.py:369-385) instead of the
                                 round-start snapshot.  Same distances and negative-cycle flag (the
                                 same greatest fixpoint); work counters become timing-dependent.
                                 Ignored with DAWN_F_PRED / the negative-cycle check. */

typedef struct dawn_graph_s* dawn_graph_t;
typedef struct dawn_solver_s* dawn_solver_t;

/* Per-solve counters (SolveStats, solver.py:118-149).  Counts follow
 * snapshot-Jacobi round semantics (SURVEY §8(a) conventions 1-7):
 * `writes` counts (node, round) changes, `multi_written` the nodes changed in
 * >= 2 rounds (numerator of updated_ratio, solver.py:258-262). */
typedef struct {
  int64_t outer_steps;
  int64_t relaxations;
  int64_t writes;
  int64_t first_discoveries;
  int64_t multi_written;
  int32_t negative_cycle;
  int32_t early_exit;   /* 1 when DAWN_F_NEGCHECK stopped the solve before the cap */
} dawn_stats_t;

int dawn_abi_version(void);
const char* dawn_last_error(void);
int dawn_device_count(int* count_out);

/* Precision probe: picks the device value type for a float64 weight array
 * (CsrGraph.val, graph.py:85-87).  AUTO chooses I32 when every weight is
 * integral and n*max|w| fits in int32, I64 when it fits in 2^53 (where the
 * reference's float64 sums are still exact), else F64. */
int dawn_choose_vtype(int64_t n, int64_t m, const double* val, int precision, int* vtype_out);

/* Upload an immutable CSR graph (CsrGraph, graph.py:64-109) to `device`.
 * row_ptr/col/val are host pointers unless src_is_device != 0, in which case
 * they are device pointers on `device`.  Page-locked (pinned) host arrays are
 * read in place by the conversion kernels over PCIe (no staging copy);
 * pageable ones are staged through a temporary device buffer.  Weights are converted to `vtype`;
 * for integer vtypes a non-integral or out-of-range weight is DAWN_EINVAL
 * (never silently truncated, SURVEY §8(b) constraint 5). */
int dawn_graph_create(int device, int64_t n, int64_t m, const int64_t* row_ptr,
                      const int64_t* col, const double* val, int vtype, int src_is_device,
                      dawn_graph_t* out);
int dawn_graph_destroy(dawn_graph_t g);
int dawn_graph_info(dawn_graph_t g, int64_t* n, int64_t* m, int* vtype, int64_t* device_bytes);

/* A solver owns the per-solve device workspace for one graph (dist keys,
 * write stamps, two frontier queues, tile map).  One solver per concurrent
 * stream; the graph itself is shareable.  flags: DAWN_F_PRED reserves the
 * predecessor arrays. */
int dawn_solver_create(dawn_graph_t g, unsigned flags, dawn_solver_t* out);
int dawn_solver_destroy(dawn_solver_t s);
/* Tuning knobs (results never depend on them):
 *   "dense_edges_per_node" (default 0.5): a round that relaxes at least
 *   value*n edges records its writes as plain stamps and the next frontier is
 *   rebuilt by a coalesced sweep; lighter rounds enqueue written nodes.
 *   "batch_min_sources" (default 4): dawn_mssp batches k >= value sources.
 *   "batch_sparse_util" (default 4): batched rounds whose rows carry fewer
 *   active sources per edge than this relax lane by lane (0 = never, 33 =
 *   always).
 *   "wide_tiles" (default -1 = auto): 1 / 0 forces wide (14 edges per lane)
 *   or narrow (8) X-phase warp tiles for 4-byte values; auto = wide when
 *   m >= 2^25 and m >= 8n.
 *   "bitmap_frontier" (default -1 = auto): 1 / 0 forces / disables the
 *   bitmap frontier of light rounds (auto: average out-degree < 8 and
 *   n >= 4096, narrow tiles; never with predecessors).
 *   "worklist_edges" (default 2^20; 0 = off): under DAWN_F_ASYNC, on graphs
 *   without negative weights, GOVM, unbounded runs, once a round relaxes
 *   fewer edges than this the rest of the solve runs barrier-free (a ring of
 *   row items taken by all warps).  Distances, negative_cycle and
 *   first_discoveries are unchanged; outer_steps reports the round at which
 *   the worklist took over. */
int dawn_solver_tune(dawn_solver_t s, const char* key, double value);

/* One single-source solve: govm_sssp / gsvm_sssp (solver.py:265-399),
 * including the seeding round seed_source (solver.py:212-250).
 *   dist_out  : float64[n], host or device pointer, or NULL to keep the
 *               result device-resident (read later with dawn_solver_result).
 *   pred_out  : int64[n] (-1 = None), host or device, or NULL.  Requires
 *               DAWN_F_PRED in `flags` and in the solver's flags.
 *   stats_out : if non-NULL the call synchronises `stream` and fills it;
 *               if NULL the call is fully asynchronous.
 * Source range is checked before any device work (DAWN_ESOURCE). */
int dawn_sssp(dawn_solver_t s, int64_t source, int algo, unsigned flags, double* dist_out,
              int64_t* pred_out, dawn_stats_t* stats_out, void* stream);

/* Debug stepping for the reference's `trace` hook (solver.py:328-336,
 * :386-387): begin a solve, then advance at most `max_rounds` rounds per call
 * (each call synchronises).  round_out receives the last completed round
 * (step), done_out 1 once the solve has terminated. */
int dawn_sssp_begin(dawn_solver_t s, int64_t source, int algo, unsigned flags, void* stream);
int dawn_sssp_advance(dawn_solver_t s, int max_rounds, int64_t* round_out, int* done_out,
                      void* stream);
/* Asynchronous advance (no synchronisation, no state read-back): runs at
 * most `max_rounds` rounds (0 = to completion) of the solve begun with
 * dawn_sssp_begin.  Used to time the persistent kernel alone. */
int dawn_sssp_run(dawn_solver_t s, int max_rounds, void* stream);
/* Copy out the current state: dist (float64[n]) and the per-node write stamp
 * (uint32[n]: the last round that lowered the node, 0 = never).  Any pointer
 * may be NULL.  Synchronises `stream`. */
int dawn_solver_state(dawn_solver_t s, double* dist_out, uint32_t* stamp_out, void* stream);
/* Result of the last solve on this solver (after dawn_sssp with NULL
 * outputs, or after stepping finished). Synchronises `stream`. */
int dawn_solver_result(dawn_solver_t s, double* dist_out, int64_t* pred_out,
                       dawn_stats_t* stats_out, void* stream);

/* Per-round timeline of the last solve (solver created with DAWN_F_PROFILE):
 * 4 uint64 per round r (index r = round number, row 0 unused):
 *   [0] S-phase start ns, [1] X-phase start ns, [2] round end ns,
 *   [3] frontier reservation word (entries << ebits | edges).
 * Copies min(cap_rounds, rounds run + 1) rows; *nrounds = rows available. */
int dawn_solver_round_profile(dawn_solver_t s, uint64_t* out, int64_t cap_rounds, int64_t* nrounds,
                              void* stream);

/* Debug (DAWN_F_PROFILE solvers): per-CTA end times (ns, globaltimer) of the
 * S and X work of the first 64 rounds of the last solve, before each phase's
 * grid barrier: out[(round * 2 + phase) * grid + cta], grid in *grid_out. */
int dawn_solver_cta_profile(dawn_solver_t s, uint64_t* out, int64_t cap_rounds, int* grid_out, void* stream);
/* Worklist tail of the last solve (all zero if the solve finished in rounds):
 * out[0] = round handed over, [1] items taken, [2] warp batches, [3] / [4]
 * warp-ns busy / waiting (sums over warps), [5] kernel span in ns.
 * Synchronises `stream`. */
int dawn_solver_worklist_stats(dawn_solver_t s, uint64_t* out, void* stream);

/* Multi-source: independent solves from sources[0..k) (host int64 array) in
 * the given order — mssp (solver.py:426-457).  Uses the batched kernel
 * (dawn_mssp_batch) when eligible and k >= the "batch_min_sources" tuning
 * value (default 4), else one persistent solve per source.  dist_out is a row-major
 * float64 [k][n] tile (host or device) or NULL; stats_out a host array of k
 * entries or NULL.  All sources are validated before any work
 * (solver.py:441-443).  One synchronisation at the end. */
int dawn_mssp(dawn_solver_t s, const int64_t* sources, int64_t k, int algo, unsigned flags,
              double* dist_out, dawn_stats_t* stats_out, void* stream);

/* Batched multi-source solves: up to 32 sources advance
 * together, one per warp lane, over a node-major [n][32] distance layout, so
 * each edge is read once per batch and its 32 distance updates are one
 * coalesced line.  Every per-source distance and counter equals the
 * single-source dawn_sssp result (same snapshot-Jacobi rounds per lane).
 * Replaces the per-source loop of mssp / apsp (solver.py:426-457, :460-495).
 * Eligible when the graph has no negative weight, n >= 2 and DAWN_F_PRED is
 * not requested (dawn_batch_supported); otherwise DAWN_EUNSUPPORTED.
 *   dist_out : row-major [k][ld] tile, host or device, or NULL.  out_vtype
 *              DAWN_F64 (float64 rows, +inf = unreachable, the reference's
 *              DistanceVector) or DAWN_F32 for a float32 graph (device-
 *              resident result tiles at half the bytes).
 *   stats_out: k entries or NULL.  With a device dist_out and NULL stats the
 *              call is fully asynchronous on `stream`. */
int dawn_batch_supported(dawn_solver_t s, int algo, unsigned flags, int* out);
int dawn_mssp_batch(dawn_solver_t s, const int64_t* sources, int64_t k, int algo, unsigned flags,
                    void* dist_out, int out_vtype, int64_t ld, dawn_stats_t* stats_out, void* stream);

/* Canonical CSR construction on the device — build_csr (reference
 * graph.py:303-322): rows by source u, columns ascending, ties in input order,
 * duplicates and self-loops kept, row_ptr[n+1].  Inputs u, v (int64), w
 * (float64) of m edges are host (src_is_device = 0) or device arrays; outputs
 * are host or device arrays of the reference CsrGraph layout (int64 row_ptr,
 * int64 col, float64 val).  An endpoint outside [0, n) or a non-finite weight
 * is DAWN_EINVAL (EdgeList.validate, graph.py:53-60).  Synchronises `stream`. */
int dawn_build_csr(int device, int64_t n, int64_t m, const int64_t* u, const int64_t* v, const double* w,
                   int src_is_device, int64_t* row_ptr_out, int64_t* col_out, double* val_out, void* stream);

/* Synthetic generators on the device (SURVEY §8(f) row F1 inputs).  They
 * write an edge list (u, v, w) of m edges, deterministic in `seed` through a
 * counter-based hash, identical to the host restatement in
 * paper_2306_07872_b200/generators.py.
 *   rmat : Graph500 quadrant probabilities a,b,c (d = 1-a-b-c), 2^scale nodes,
 *          m = edge_factor * 2^scale edges; duplicates and self-loops kept.
 *   wkind: 0 = integer uniform in [wlo, whi] ; 1 = float32 uniform in [0,1). */
int dawn_gen_rmat(int device, int scale, int64_t edge_factor, double a, double b, double c,
                  uint64_t seed, int wkind, int64_t wlo, int64_t whi, uint64_t wseed,
                  int64_t* u_out, int64_t* v_out, double* w_out, void* stream);

/* 4-neighbour grid of rows x cols nodes (id = r*cols + c), both directions,
 * written directly in canonical CSR order (no sort): row_ptr_out[n+1],
 * col_out / val_out [m], m = 4*rows*cols - 2*rows - 2*cols.  Bit-identical
 * to generators.grid_graph (weights drawn per CSR position). */
int dawn_gen_grid(int device, int64_t rows, int64_t cols, int wkind, int64_t wlo, int64_t whi,
                  uint64_t wseed, int64_t* row_ptr_out, int64_t* col_out, double* val_out, void* stream);

/* Dense all-pairs Floyd–Warshall on the device: floyd_warshall_apsp
 * (oracles.py:141-162), the cross-check oracle, float64, same step order and
 * rounding as the NumPy loop (not blocked).  Input: the CsrGraph arrays
 * (int64 row_ptr[n+1], int64 col[m], float64 val[m]; host or device).
 * out: float64[n][n] row-major, host or device.  *negative_cycle_out = any
 * diagonal entry < 0.  The n-size cap (GraphSizeError) is the caller's.
 * Synchronises `stream`. */
int dawn_floyd_warshall(int device, int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                        double* out, int* negative_cycle_out, void* stream);

/* Distance rows as text, host side (format_distance_row, solver.py:498-506):
 * for each of the k rows (row r at rows + r*ld, float64[n], host memory) one
 * line "source,d0,...,d{n-1}\n" with "%.17g" values and the literal "inf"
 * (and "nan" / "-inf" as Python prints them), concatenated into `out`.
 * cap must be >= k * (24 + 26n) (else DAWN_EINVAL and *len_out = the bound);
 * *len_out = bytes written.  threads <= 0: all hardware threads. */
int dawn_format_rows(const double* rows, int64_t k, int64_t n, int64_t ld, const int64_t* sources, char* out,
                     int64_t cap, int64_t* len_out, int threads);

/* Independent cross-check oracles, computed on the HOST by design (they check
 * the device kernels from outside and share no code with them; the solvers
 * above never call them).  Native restatements of the reference's oracles
 * with the same visiting order and float64 arithmetic, so dist, relaxation
 * counts and the negative-cycle verdict equal the reference's exactly.
 * Inputs are the CsrGraph host arrays (int64 row_ptr[n+1], int64 col[m],
 * float64 val[m]); dist_out is float64[n].  The negative-weight check
 * (NegativeWeightError) is the caller's.
 *   dawn_oracle_dijkstra     : dijkstra_sssp     (oracles.py:59-91), binary heap
 *                              over (dist, node) with lazy deletion.
 *   dawn_oracle_bellman_ford : bellman_ford_sssp (oracles.py:94-138), n-1 in-place
 *                              passes in row order + one detection pass; no
 *                              source guard (dist[source] may go below 0). */
int dawn_oracle_dijkstra(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                         int64_t source, double* dist_out, int64_t* relaxations_out);
int dawn_oracle_bellman_ford(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                             int64_t source, double* dist_out, int64_t* relaxations_out, int* negative_cycle_out);

#ifdef __cplusplus
}
#endif
#endif /* DAWN_H_ */
