// BDLR skeleton selection on the host: integer work that must be bit-exact
// (src/graph.py:171-228).  Boundary = own-side vertices with a neighbour on
// the other side; multi-source BFS restricted to the own side; selection =
// positions with d <= depth ordered by (d, vertex id).
#include <algorithm>
#include <cstdint>
#include <vector>

#include "hk_graph.h"

namespace hk {

// dist[k] for own[k]: BFS distance to the boundary within own; -1 = unreachable.
// max_depth >= 0: vertices beyond it are left at -1 (enough for a depth
// selection; BFS distances only grow, so the <= max_depth ones are exact).
void side_distance(int64_t nverts, const int64_t* indptr, const int64_t* indices,
                   const int64_t* own, int64_t n_own, const int64_t* other, int64_t n_other,
                   std::vector<int64_t>& dist, int64_t max_depth) {
  // per-thread scratch over the whole vertex range, reset after use
  thread_local std::vector<int8_t> is_other;
  thread_local std::vector<int64_t> where;
  if ((int64_t)is_other.size() < nverts) {
    is_other.assign(nverts, 0);
    where.assign(nverts, -1);
  }
  for (int64_t k = 0; k < n_other; ++k) is_other[other[k]] = 1;
  for (int64_t k = 0; k < n_own; ++k) where[own[k]] = k;
  // boundary vertices sorted by id (graph.py:179-180)
  std::vector<int64_t> bnd;
  for (int64_t k = 0; k < n_own; ++k) {
    const int64_t v = own[k];
    for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e)
      if (is_other[indices[e]]) { bnd.push_back(v); break; }
  }
  std::sort(bnd.begin(), bnd.end());
  dist.assign(n_own, -1);
  std::vector<int64_t> queue;
  queue.reserve(n_own);
  for (int64_t v : bnd) {
    dist[where[v]] = 0;
    queue.push_back(v);
  }
  // FIFO BFS in the reference's visiting order (deque popleft, neighbours in CSR order)
  for (size_t head = 0; head < queue.size(); ++head) {
    const int64_t v = queue[head];
    const int64_t dv = dist[where[v]];
    if (max_depth >= 0 && dv >= max_depth) break;   // FIFO: every later vertex is as far
    for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
      const int64_t u = indices[e];
      const int64_t k = where[u];
      if (k >= 0 && dist[k] < 0) {
        dist[k] = dv + 1;
        queue.push_back(u);
      }
    }
  }
  for (int64_t k = 0; k < n_other; ++k) is_other[other[k]] = 0;
  for (int64_t k = 0; k < n_own; ++k) where[own[k]] = -1;
}

bool select_by_depth(int64_t nverts, const int64_t* indptr, const int64_t* indices,
                     const int64_t* row_verts, int64_t n_rows, const int64_t* col_verts,
                     int64_t n_cols, int depth, std::vector<int64_t>& row_sel,
                     std::vector<int64_t>& col_sel) {
  for (int side = 0; side < 2; ++side) {
    const int64_t* own = side == 0 ? row_verts : col_verts;
    const int64_t n_own = side == 0 ? n_rows : n_cols;
    const int64_t* oth = side == 0 ? col_verts : row_verts;
    const int64_t n_oth = side == 0 ? n_cols : n_rows;
    std::vector<int64_t> dist;
    side_distance(nverts, indptr, indices, own, n_own, oth, n_oth, dist, depth);
    std::vector<int64_t> keep;
    for (int64_t k = 0; k < n_own; ++k)
      if (dist[k] >= 0 && dist[k] <= depth) keep.push_back(k);
    // lexsort((own[keep], d[keep])): primary d, secondary vertex id (ids are unique)
    std::sort(keep.begin(), keep.end(), [&](int64_t a, int64_t b) {
      if (dist[a] != dist[b]) return dist[a] < dist[b];
      return own[a] < own[b];
    });
    (side == 0 ? row_sel : col_sel) = keep;
  }
  return !row_sel.empty() && !col_sel.empty();
}

}  // namespace hk
