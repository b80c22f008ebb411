// Host-side launchers shared between the kernel translation units and the C-ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "gq_common.cuh"

namespace gq {

// Per-device one-time kernel configuration (max dynamic shared memory, resident blocks per
// SM).  `cache` is a zero-initialised static int[64] owned by the call site.
template <typename Kern>
inline cudaError_t kernel_occupancy(Kern kernel, int threads, size_t smem, int* cache,
                                    int& per_sm) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 63;
  if (!cache[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem);
    cache[dev] = n > 0 ? n : 1;
  }
  per_sm = cache[dev];
  return cudaSuccess;
}

enum StencilMode { kDelta = 0, kOuter = 1, kInner = 2, kOuterRhs = 3 };

struct SetupErr {
  int code;        // 0 ok, 1 not SPD
  int cls, v, k, j;
  double pivot, tol;
};

// Returns false if n has no compiled instantiation.
bool n_supported(int n);

// ---- setup (gq_setup.cu) ----
cudaError_t launch_spd_inverse(const double* in, double* out, long long count, int dim,
                               SetupErr* err, cudaStream_t s);
cudaError_t launch_brb(const Geo& g, int m, int n_dyn, const double* B, const double* rinv,
                       double* brb, cudaStream_t s);
cudaError_t launch_xi(const Geo& g, int nxc, const int* xi_keys, const double* A,
                      const double* C, const double* qinv, double* xi, double* xit,
                      cudaStream_t s);
cudaError_t launch_psi(const Geo& g, int npc, const int* psi_keys, const double* A,
                       const double* C, const double* qinv, const double* brb, double* psi,
                       cudaStream_t s);
cudaError_t launch_factor(const Geo& g, int npc, const double* psi, double* fac,
                          double* scratch, SetupErr* err, cudaStream_t s);

// primal recovery (which = 0: x, u, objective partials) and KKT residual partials
// (which = 1: per block {max|r_x|, max|r_u|, max|r_dyn|}); vectors in the reference order
int recover_blocks(const Geo& g);
cudaError_t launch_recover(const Geo& g, int m, const double* A, const double* C,
                           const double* qinv, const double* B, const double* R,
                           const double* rinv, const double* Q, const int* dcls,
                           const int* ccls, int which, const double* lam, const double* x,
                           const double* u, const double* off, double* xo, double* uo,
                           double* part, cudaStream_t s);

// ---- stencil (gq_stencil.cu) ----
struct StencilShape {
  int nchunk, nstrip, rows, blocks, threads;
};
StencilShape stencil_shape(const Geo& g, int mode, int sm_count);
cudaError_t launch_stencil(const Geo& g, const Ops& op, int mode, const double* x, double* y,
                           const StencilShape& sh, double* partials, PcgState* st,
                           int dotmode, cudaStream_t s);

// ---- pair sweeps (gq_sweep.cu) ----
struct SweepShape {
  int blocks, threads;
};
SweepShape sweep_shape(const Geo& g, bool outer);
cudaError_t launch_sweep(const Geo& g, const Ops& op, bool inner, bool outer, const double* r,
                         const double* theta, const double* delta, double* out,
                         const SweepShape& sh, double* partials, PcgState* st, int dotmode,
                         cudaStream_t s);

// ---- pipelined fast-path kernels (gq_fast.cu) ----
struct FastOps {
  const double* oprow;   // [npc][N][K][23][n][n]  Psi(13) | Xi_0(5) | Xi_0'(5)
  const double* omega;   // [npc][N][K][5][n][n]   cross-pair Psi blocks, sweep order
  const double* fac3;    // [npc][V][nb][3][q][q]  G_k | L_k^-1 | H_k        (FMA sweep)
  const int* psi_cls;
  const double* fac4;    // [npc][V][nb][4][q][q]  L^-1 | -G | L^-T | -H      (DMMA sweep)
};
cudaError_t launch_build_fast(const Geo& g, int npc, const Ops& op, double* oprow, double* omega,
                              double* fac3, double* fac4, cudaStream_t s);
bool tc_supported(int n);
// stencil modes kDelta (y = Delta x, optional y.x) and kOuterRhs (y = r + Xi~ x)
cudaError_t launch_stencil3(const Geo& g, const FastOps& fo, int mode, const double* x,
                            const double* rin, double* y, const StencilShape& sh,
                            double* partials, PcgState* st, int dotmode, cudaStream_t s);
cudaError_t launch_sweep3(const Geo& g, const FastOps& fo, bool inner, const double* rhs,
                          const double* th, double* out, const double* rdot, int sm_count,
                          double* partials, PcgState* st, int dotmode, cudaStream_t s);
bool fast_supported(int n);
long long fast_max_blocks(const Geo& g, const StencilShape& sh, int sm_count);

// ---- lean DMMA pair-chain sweeps (gq_chain.cu) ----
struct ChainOps {
  const double* ff;    // [npc][V][nb] L^-1 | -G | -L^-1 Omega~   (8x8 tiles)
  const double* fb;    // [npc][V][nb] L^-T | -H                  (8x8 tiles)
  const int4* seg;     // [nseg] (t0, nvalid <= 8, psi class, 0): class-pure stage chunks
  int nseg;
  const int4* seg16;   // [nseg16] the same with chunks of <= 16 stages (two M-tiles per warp)
  int nseg16;
  const double* omega = nullptr;   // [npc][N][K][5][n][n] cross-pair Psi blocks (n = 8 inner)
  const int4* grp = nullptr;       // CTA items (n = 8: all classes; n = 2: class-1 runs)
  int ngrp = 0;
};
// seg[i].w = 1 for the segments of classes whose coupling tiles (G, L^-1 Omega~, H) are all
// zero (n = 2; flags: npc ints of scratch); k_chainm zero-fills those tiles instead of reading
// them (gq_chainm.cu)
cudaError_t launch_chainm_mark(const Geo& g, int npc, const ChainOps& co, int4* seg, int nseg,
                               int* flags, cudaStream_t s);

// n = 8 pair-chain sweeps with CTA-shared factor tiles (gq_chain8c.cu)
bool chain8c_enabled();
cudaError_t launch_chain8c(const Geo& g, const ChainOps& co, bool inner, const double* rhs,
                           const double* th, double* out, const double* rdot, int sm_count,
                           double* partials, PcgState* st, int dotmode, cudaStream_t s);
bool chain_supported(int n);
size_t chain_ff_doubles(const Geo& g, int npc);
size_t chain_fb_doubles(const Geo& g, int npc);
cudaError_t launch_build_chain(const Geo& g, int npc, const double* fac, const double* omega,
                               double* ff, double* fb, cudaStream_t s);
cudaError_t launch_chain(const Geo& g, const ChainOps& co, bool inner, const double* rhs,
                         const double* th, double* out, const double* rdot, int sm_count,
                         double* partials, PcgState* st, int dotmode, cudaStream_t s);
long long chain_max_blocks(const Geo& g, int nseg, int sm_count);
// cross-pair Psi blocks for the chain tiles when the fast-path operator rows are not built (n = 8)
cudaError_t launch_build_omega(const Geo& g, int npc, const double* psi, double* omega,
                               cudaStream_t s);
// outer sweep with the PCG residual update fused in (r -= alpha y, max|r|, history)
cudaError_t launch_chain_fr(const Geo& g, const ChainOps& co, double* r, const double* y,
                            double* out, int sm_count, double* partials, PcgState* st,
                            cudaStream_t s);
long long chain_fr_max_blocks(const Geo& g, int nseg, int sm_count);

// ---- n = 8 block stencils on DMMA (gq_st8.cu) ----
bool st8_supported(const Geo& g, int nxc);
// modes kDelta (y = Delta x, optional curvature) and kOuterRhs (y = rin + Xi~ x); seg = the
// class-pure stage chunks of the chain sweeps
cudaError_t launch_st8(const Geo& g, const Ops& op, const int4* seg, int nseg, int mode,
                       const double* x, const double* rin, double* y, int sm_count,
                       double* partials, PcgState* st, int dotmode, cudaStream_t s);
long long st8_max_blocks(int sm_count);

// ---- t-loop factored Delta apply, n = 2 (gq_dstep.cu) ----
struct DstepOps {
  const double* A;      // [nd][N][K][n][n]
  const double* C;      // [nd][4][N][K][n][n]  couplings (west, east, north, south)
  const double* qinv;   // [nq][N][K][n][n]
  const double* brb;    // [nd][N][K][n][n]     B R^-1 B'
  const int* dcls;      // [T]  dynamics set of stage t -> t+1
  const int* ccls;      // [T1] cost set of stage t
};
bool dstep_supported(const Geo& g);
bool dstep_preferred(const Geo& g, int sm_count);   // large enough grid (or GQ_DSTEP=1)
long long dstep_max_blocks(int sm_count);
// TMA view of a stage-inner vector: 4-stage boxes of a tile with a halo of `halo` nodes (2:
// the Delta input, 0: its output)
bool dstep_make_map(const Geo& g, const double* base, int halo, CUtensorMap* m);
// y = Delta x for the vector behind `dmap` into the vector behind `ymap` (+ y.x curvature,
// alpha, breakdown when dotmode != kDotNone); stage-slab halo rows are written as zeros
cudaError_t launch_dstep(const Geo& g, const CUtensorMap& dmap, const CUtensorMap& ymap,
                         const DstepOps& op, double* y, double* partials, PcgState* st,
                         int dotmode, int sm_count, cudaStream_t s);
// y = r - (Xi_{t-1} x_{t-1} + Xi_t' x_{t+1}) by TMA tiles (n = 2, one Xi class): views of x
// (input = true: one-node halo) and of r / y; needs T >= 2
bool rstep_make_map(const Geo& g, const double* base, bool input, CUtensorMap* m);
cudaError_t launch_rstep(const Geo& g, const CUtensorMap& xmap, const CUtensorMap& rmap,
                         const CUtensorMap& ymap, const double* x, const double* r,
                         double* y, const double* xi, const double* xit, PcgState* st,
                         int sm_count, cudaStream_t s);

// ---- lean n = 2 grid stencils (gq_grid.cu) ----
struct GridShape {
  int nchunk = 0, nstrip = 0, rows = 0, blocks = 0;
};
bool grid_supported(int n);
GridShape grid_shape(const Geo& g, int sm_count);
// modes kDelta (y = Delta x, optional curvature) and kOuterRhs (y = r + Xi~ x)
cudaError_t launch_grid(const Geo& g, const FastOps& fo, int mode, const double* x,
                        const double* rin, double* y, const GridShape& sh, double* partials,
                        PcgState* st, int dotmode, cudaStream_t s);

// ---- vector kernels (gq_vec.cu) ----
int vec_blocks(int sm_count);
cudaError_t launch_update(const Geo& g, double* x, double* r, const double* d, const double* y,
                          int blocks, double* partials, PcgState* st, cudaStream_t s);
cudaError_t launch_nonfinite(const Geo& g, const double* v, int blocks, PcgState* st,
                             cudaStream_t s);
cudaError_t launch_update_r(const Geo& g, double* r, const double* y, int blocks,
                            double* partials, PcgState* st, cudaStream_t s);
cudaError_t launch_update_x(const Geo& g, double* x, const double* d, int blocks, PcgState* st,
                            cudaStream_t s);
cudaError_t launch_dirupdate(const Geo& g, double* d, const double* q, int blocks,
                             PcgState* st, cudaStream_t s);
cudaError_t launch_dirupdate_x(const Geo& g, double* d, const double* q, double* x, int blocks,
                               PcgState* st, cudaStream_t s);
cudaError_t launch_maxdiff(const Geo& g, const double* a, const double* b, int blocks,
                          double* partials, unsigned int* counter, double* out, cudaStream_t s);
cudaError_t launch_add(const Geo& g, double* out, const double* a, const double* b, int blocks,
                       cudaStream_t s);
cudaError_t launch_dot(const Geo& g, const double* a, const double* b, int blocks,
                       double* partials, PcgState* st, int dotmode, cudaStream_t s);
cudaError_t launch_sub(const Geo& g, double* out, const double* a, const double* b, int blocks,
                       cudaStream_t s);
cudaError_t launch_to_internal(const Geo& g, const double* ref, double* dev, cudaStream_t s);
cudaError_t launch_to_reference(const Geo& g, const double* dev, double* ref, cudaStream_t s);

// stage-slab mode (gq_slab.cu): halo-stage zeroing, scalar fix-ups after the host-side
// reductions (which: 0 alpha, 2 save mu, 3 convergence + beta), halo stage pack/unpack
cudaError_t launch_stage_zero(const Geo& g, int t, double* v, int sm_count, cudaStream_t s);
cudaError_t launch_slab_scalar(int which, PcgState* st, cudaStream_t s);
cudaError_t launch_stage_pack(const Geo& g, int t, const double* v, double* buf, int sm_count,
                              cudaStream_t s);
cudaError_t launch_stage_unpack(const Geo& g, int t, const double* buf, double* v, int sm_count,
                                cudaStream_t s);

}  // namespace gq
