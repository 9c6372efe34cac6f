// Host-side graph selection (graph.cpp).
#pragma once
#include <cstdint>
#include <vector>

namespace hk {
void side_distance(int64_t nverts, const int64_t* indptr, const int64_t* indices,
                   const int64_t* own, int64_t n_own, const int64_t* other, int64_t n_other,
                   std::vector<int64_t>& dist, int64_t max_depth = -1);
bool select_by_depth(int64_t nverts, const int64_t* indptr, const int64_t* indices,
                     const int64_t* row_verts, int64_t n_rows, const int64_t* col_verts,
                     int64_t n_cols, int depth, std::vector<int64_t>& row_sel,
                     std::vector<int64_t>& col_sel);
}  // namespace hk
