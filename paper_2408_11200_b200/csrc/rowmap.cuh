// rowmap.cuh — how a spline layer maps (sample b, feature i) to a table row (spline.cu).
//   KAN : T = coeffs viewed as [d_in*(G+k), d_out], row_bi = i*(G+k) + cell_bi
//   UKAN: T = CG output viewed as [n_u*K, d_out] (slot-major), row_bi = base_row[b,i]
// Each feature i owns a contiguous row segment [row0_i, row0_i + R_i) of T.
#pragma once
#include "common.cuh"

namespace ukan {

// How a layer maps (b, i) to a table row and in-cell position.
struct RowMap {
  // KAN
  KanGrid grid;
  int R;  // G + k
  // UKAN
  double inv_dg;
  const int32_t* base_row;   // [B, d_in]
  const int32_t* seg_start;  // [d_in + 1]
  int K;
};

template <bool UKAN>
__device__ __forceinline__ bool locate_row(const RowMap& rm, float xv, int64_t b, int i,
                                           int d_in, int& row, double& u, bool& mask) {
  if constexpr (UKAN) {
    int64_t gid;
    ukan_locate(xv, rm.inv_dg, gid, u);
    row = rm.base_row[(size_t)b * d_in + i];
    mask = true;
    return true;
  } else {
    int cell;
    const bool ok = kan_locate(xv, rm.grid, cell, u, mask);
    row = i * rm.R + cell;
    return ok;
  }
}

template <bool UKAN>
__device__ __forceinline__ void feature_rows(const RowMap& rm, int i, int& row0, int& nrows) {
  if constexpr (UKAN) {
    const int s0 = rm.seg_start[i], s1 = rm.seg_start[i + 1];
    row0 = s0 * rm.K;
    nrows = (s1 - s0) * rm.K;
  } else {
    row0 = i * rm.R;
    nrows = rm.R;
  }
}

}  // namespace ukan
