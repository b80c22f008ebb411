// Shared between the pair-chain sweep kernels (gq_chain.cu, gq_chainm.cu): the order of the
// theta neighbour records of a block and the 8x8 tiling of the factor matrices.
#pragma once

#include "gq_async.cuh"
#include "gq_internal.h"

namespace gq {

// theta neighbour records of a block, relative to (column a = 2v, row 2k): the twelve nodes
// outside the pair that the 13-point Psi diamond of its four nodes reaches
// (kkt_assembly.py:645-662).  Order: the two middle columns a-1, a+2 at rows -1, 0 (records
// 0..3), the same columns at rows +1, +2 (records 4..7), the outer columns a-2, a+3 at rows
// 0, +1 (records 8..11).  Records 4..7 of block k are records 0..3 of block k+1, so a sweep
// that walks the chain fetches eight new records per block and carries four.
__host__ __device__ constexpr int th_dc(int r) {
  return r < 8 ? ((r & 2) ? 2 : -1) : (r < 10 ? -2 : 3);
}
__host__ __device__ constexpr int th_dr(int r) {
  return r < 4 ? (r & 1) - 1 : r < 8 ? (r & 1) + 1 : (r & 1);
}
// omega slot u of a node at row offset dr (0, 1) in the pair's left (dc = 0) / right (dc = 1)
// column -> record index; the u order is that of k_build_rows / k_build_omega
__host__ __device__ constexpr int th_rec(int dc, int u, int dr) {
  // position in the column-major walk (a-2: rows 0,1 | a-1: rows -1..2 | a+2: rows -1..2 |
  // a+3: rows 0,1) ...
  const int o = (dc == 0 ? (u == 0 ? 0 : u == 1 ? 2 : u == 2 ? 3 : u == 3 ? 4 : 7)
                         : (u == 0 ? 3 : u == 1 ? 6 : u == 2 ? 7 : u == 3 ? 8 : 10)) + dr;
  // ... to the record order above
  return o < 2 ? 8 + o : o < 4 ? o - 2 : o < 6 ? o : o < 8 ? o - 4 : o < 10 ? o - 2 : o;
}

// element (r, c) of a Q x kc matrix stored as 8x8 tiles (row-major tiles, row-major inside)
__host__ __device__ __forceinline__ int tile_at(int r, int c, int kc) {
  return ((r >> 3) * (kc >> 3) + (c >> 3)) * 64 + (r & 7) * 8 + (c & 7);
}

// ---- twelve-warp chain sweeps with carried theta fragments, n = 2 (gq_chainm.cu) ----
bool chainm_supported(const Geo& g, int sm_count);
bool chainm_all();   // GQ_CHAINM=2: every sweep form on the twelve-warp kernel (tests)
cudaError_t launch_chainm(const Geo& g, const ChainOps& co, bool inner, const double* rhs,
                          const double* th, double* out, const double* rdot, int sm_count,
                          double* partials, PcgState* st, int dotmode, cudaStream_t s);
cudaError_t launch_chainm_fr(const Geo& g, const ChainOps& co, double* r, const double* y,
                             double* out, int sm_count, double* partials, PcgState* st,
                             cudaStream_t s);

}  // namespace gq
