// Independent cross-check oracles on the host: heap Dijkstra and textbook
// Bellman–Ford (reference sparsepath/oracles.py:59-91, :94-138).
//
// These are deliberately NOT device kernels and share no code with the
// solvers: their only job is to check the device path from outside
// (experiments.py:_cross_check compares solver rows against them at atol
// 1e-9), so computing them with the kernels under test would be circular.
// Native C++ instead of the reference's Python loops: same visiting order,
// same IEEE float64 arithmetic (no fast-math), so distances, relaxation counts
// and negative-cycle verdicts are identical to the reference's, including the
// reference's unguarded behaviour on negative cycles (dist[source] may drop
// below 0).  None of this is on the hot path.

#include <math.h>
#include <stdint.h>

#include <functional>
#include <queue>
#include <utility>
#include <vector>

#include "../../include/dawn.h"

namespace {

bool valid_graph(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val, int64_t source,
                 double* dist_out, int64_t* relax_out) {
  if (n <= 0 || !row_ptr || !dist_out || !relax_out || source < 0 || source >= n) return false;
  return row_ptr[n] == 0 || (col && val);
}

}  // namespace

// Binary heap keyed by (distance, node) — the order of Python's heapq over
// (d, u) tuples — with lazy deletion of stale entries.
extern "C" int dawn_oracle_dijkstra(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                                    int64_t source, double* dist_out, int64_t* relaxations_out) {
  if (!valid_graph(n, row_ptr, col, val, source, dist_out, relaxations_out)) return DAWN_EINVAL;
  using Item = std::pair<double, int64_t>;
  std::priority_queue<Item, std::vector<Item>, std::greater<Item>> heap;
  for (int64_t i = 0; i < n; ++i) dist_out[i] = INFINITY;
  dist_out[source] = 0.0;
  heap.emplace(0.0, source);
  int64_t relax = 0;
  while (!heap.empty()) {
    const auto [d, u] = heap.top();
    heap.pop();
    if (d > dist_out[u]) continue;
    relax += row_ptr[u + 1] - row_ptr[u];
    for (int64_t k = row_ptr[u]; k < row_ptr[u + 1]; ++k) {
      const double nd = d + val[k];
      const int64_t v = col[k];
      if (nd < dist_out[v]) {
        dist_out[v] = nd;
        heap.emplace(nd, v);
      }
    }
  }
  *relaxations_out = relax;
  return DAWN_OK;
}

// n-1 in-place passes over the rows in index order (stopping after a pass
// with no change), then one detection pass that stops at the first edge that
// could still improve a finite tail.
extern "C" int dawn_oracle_bellman_ford(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                                        int64_t source, double* dist_out, int64_t* relaxations_out,
                                        int* negative_cycle_out) {
  if (!valid_graph(n, row_ptr, col, val, source, dist_out, relaxations_out) || !negative_cycle_out)
    return DAWN_EINVAL;
  double* dist = dist_out;
  for (int64_t i = 0; i < n; ++i) dist[i] = INFINITY;
  dist[source] = 0.0;
  int64_t relax = 0;
  for (int64_t pass = 0; pass + 1 < n; ++pass) {
    bool changed = false;
    for (int64_t u = 0; u < n; ++u) {
      if (dist[u] == INFINITY) continue;
      relax += row_ptr[u + 1] - row_ptr[u];
      for (int64_t k = row_ptr[u]; k < row_ptr[u + 1]; ++k) {
        const double nd = dist[u] + val[k];  // live dist[u]: a self-loop may lower it mid-row
        if (nd < dist[col[k]]) {
          dist[col[k]] = nd;
          changed = true;
        }
      }
    }
    if (!changed) break;
  }
  int neg = 0;
  for (int64_t u = 0; u < n && !neg; ++u) {
    if (dist[u] == INFINITY) continue;
    for (int64_t k = row_ptr[u]; k < row_ptr[u + 1]; ++k) {
      ++relax;
      if (dist[u] + val[k] < dist[col[k]]) {
        neg = 1;
        break;
      }
    }
  }
  *relaxations_out = relax;
  *negative_cycle_out = neg;
  return DAWN_OK;
}
