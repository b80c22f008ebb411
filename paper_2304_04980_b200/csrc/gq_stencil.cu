// Block-stencil applies over (i, j, t): the reduced operator Delta, the outer (stage)
// coupling Xi~ and the inner (cross-pair) coupling Omega~.
//
// Reference semantics:
//   Delta:  (Delta x)_t = Psi_t x_t + Xi_{t-1} x_{t-1} + Xi_t' x_{t+1}
//           SchurOperator.apply / _stage_row           gridlq/kkt_assembly.py:379-403
//   outer:  (Xi~ x)_t = -(Xi_{t-1} x_{t-1} + Xi_t' x_{t+1})
//           SchurOperator.apply_outer_coupling         gridlq/kkt_assembly.py:414-425
//   inner:  (Omega~ x) = -(cross-pair blocks of Psi_t) x_t
//           PairSplitting.apply_inner_coupling         gridlq/kkt_assembly.py:645-662
//
// Thread mapping: one warp = one grid column j x 30 consecutive stages (+1 halo stage on
// each side) x one strip of rows; each lane walks the rows of its strip keeping a
// register window of the 13-point diamond of x_t around (i, j).  The stage coupling is
// exchanged through the warp instead of memory: lane t computes
//   e_t(a) = sum_u Xi_t(a, a+u) x_t(a+u)      (needed by stage t+1)
//   f_t(a) = sum_u Xi_{t-1}(a+u, a)' x_t(a+u) (needed by stage t-1)
// from its own window and one shuffle each hands them to the neighbouring stages, so
// every x element is loaded from HBM once per launch and the t+-1 terms cost 2n
// shuffles instead of 10 extra loads.  Operator blocks are per (stage class, node):
// warp-uniform broadcast loads that stay L2 resident for time-invariant problems.
#include <algorithm>

#include "gq_internal.h"

namespace gq {

template <int NS, int MODE>
__global__ void __launch_bounds__(256) k_stencil(Geo g, Ops op, const double* __restrict__ x,
                                                 double* __restrict__ y, int nchunk,
                                                 int nstrip, int rows, double* partials,
                                                 PcgState* st, int dotmode) {
  if (st != nullptr) {
    if (dotmode == kDotStep) {
      // first kernel of a PCG step: the step budget is checked here so that the step
      // that reaches max_steps still completes (pcg.py:98-131 runs its whole body)
      const bool stop = st->done || st->step >= st->max_steps;
      if (blockIdx.x == 0 && threadIdx.x == 0) st->skip = stop ? 1 : 0;
      if (stop) return;
    } else if (halted(st)) {
      return;
    }
  }
  constexpr bool HALO = (MODE != kInner);
  constexpr int CH = HALO ? kHaloChunk : 32;
  constexpr int B2 = NS * NS;
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long total = (long long)g.N * nchunk * nstrip;
  const bool active = gw < total;
  int strip = 0, chunk = 0, j = 0;
  if (active) {
    strip = (int)(gw % nstrip);
    const long long rest = gw / nstrip;
    chunk = (int)(rest % nchunk);
    j = (int)(rest / nchunk);
  }
  const int t = chunk * CH + lane - (HALO ? 1 : 0);
  const bool tv = active && t >= 0 && t < g.T1;
  const bool useful = tv && (!HALO || (lane >= 1 && lane <= kHaloChunk)) &&
                      (MODE != kDelta || slab_owned(g, t));
  const int pc = tv ? op.psi_cls[t] : 0;
  const int xce = (tv && t < g.T) ? op.xi_cls[t] : -1;      // e_t uses Xi_t
  const int xcf = (tv && t >= 1) ? op.xi_cls[t - 1] : -1;   // f_t uses Xi_{t-1}
  double dot = 0.0;

  auto LD = [&](int jj, int ii) -> Vec<NS> {
    if (tv && jj >= 0 && jj < g.N && ii >= 0 && ii < g.K) return ldv_nc<NS>(x + vidx(g, jj, ii, t));
    return vzero<NS>();
  };

  if (active) {
    const int i0 = strip * rows;
    const int i1 = min(g.K, i0 + rows);
    Vec<NS> c0[5], cm[3], cp[3], cm2, cp2;
    c0[0] = LD(j, i0 - 2);
    c0[1] = LD(j, i0 - 1);
    c0[2] = LD(j, i0);
    c0[3] = LD(j, i0 + 1);
    cm[0] = LD(j - 1, i0 - 1);
    cm[1] = LD(j - 1, i0);
    cp[0] = LD(j + 1, i0 - 1);
    cp[1] = LD(j + 1, i0);
    for (int i = i0; i < i1; ++i) {
      c0[4] = LD(j, i + 2);
      cm[2] = LD(j - 1, i + 1);
      cp[2] = LD(j + 1, i + 1);
      cm2 = LD(j - 2, i);
      cp2 = LD(j + 2, i);
      const long long node = (long long)j * g.K + i;
      Vec<NS> acc = vzero<NS>();
      if (MODE == kDelta) {
        const double* P = op.psi + ((long long)pc * g.nk + node) * 13 * B2;
        mac<NS>(acc, P + 0 * B2, c0[2]);
        mac<NS>(acc, P + 1 * B2, c0[1]);
        mac<NS>(acc, P + 2 * B2, c0[3]);
        mac<NS>(acc, P + 3 * B2, cm[1]);
        mac<NS>(acc, P + 4 * B2, cp[1]);
        mac<NS>(acc, P + 5 * B2, c0[0]);
        mac<NS>(acc, P + 6 * B2, c0[4]);
        mac<NS>(acc, P + 7 * B2, cm2);
        mac<NS>(acc, P + 8 * B2, cp2);
        mac<NS>(acc, P + 9 * B2, cm[0]);
        mac<NS>(acc, P + 10 * B2, cp[0]);
        mac<NS>(acc, P + 11 * B2, cm[2]);
        mac<NS>(acc, P + 12 * B2, cp[2]);
      } else if (MODE == kInner) {
        const double* P = op.psi + ((long long)pc * g.nk + node) * 13 * B2;
        Vec<NS> s = vzero<NS>();
        if ((j & 1) == 0) {   // even column: pair v-1 on the left, col j+2 of pair v+1
          mac<NS>(s, P + 7 * B2, cm2);
          mac<NS>(s, P + 9 * B2, cm[0]);
          mac<NS>(s, P + 3 * B2, cm[1]);
          mac<NS>(s, P + 11 * B2, cm[2]);
          mac<NS>(s, P + 8 * B2, cp2);
        } else {              // odd column: col j-2 of pair v-1, pair v+1 on the right
          mac<NS>(s, P + 7 * B2, cm2);
          mac<NS>(s, P + 10 * B2, cp[0]);
          mac<NS>(s, P + 4 * B2, cp[1]);
          mac<NS>(s, P + 12 * B2, cp[2]);
          mac<NS>(s, P + 8 * B2, cp2);
        }
#pragma unroll
        for (int k = 0; k < NS; ++k) acc.v[k] = -s.v[k];
      }
      if (MODE != kInner) {
        Vec<NS> e = vzero<NS>(), f = vzero<NS>();
        if (xce >= 0) {
          const double* E = op.xi + ((long long)xce * g.nk + node) * 5 * B2;
          mac<NS>(e, E + 0 * B2, c0[2]);
          mac<NS>(e, E + 1 * B2, c0[1]);
          mac<NS>(e, E + 2 * B2, c0[3]);
          mac<NS>(e, E + 3 * B2, cm[1]);
          mac<NS>(e, E + 4 * B2, cp[1]);
        }
        if (xcf >= 0) {
          const double* F = op.xit + ((long long)xcf * g.nk + node) * 5 * B2;
          mac<NS>(f, F + 0 * B2, c0[2]);
          mac<NS>(f, F + 1 * B2, c0[1]);
          mac<NS>(f, F + 2 * B2, c0[3]);
          mac<NS>(f, F + 3 * B2, cm[1]);
          mac<NS>(f, F + 4 * B2, cp[1]);
        }
        const Vec<NS> eu = shfl_up<NS>(e, 1);    // e_{t-1}
        const Vec<NS> fd = shfl_down<NS>(f, 1);  // f_{t+1}
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          if (MODE == kDelta) {
            if (t >= 1) acc.v[k] += eu.v[k];
            if (t < g.T) acc.v[k] += fd.v[k];
          } else {
            if (t >= 1) acc.v[k] -= eu.v[k];
            if (t < g.T) acc.v[k] -= fd.v[k];
          }
        }
      }
      if (useful) {
        stv<NS>(y + vidx(g, j, i, t), acc);
        if (dotmode != kDotNone) {
#pragma unroll
          for (int k = 0; k < NS; ++k) dot = fma(acc.v[k], c0[2].v[k], dot);
        }
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) c0[r] = c0[r + 1];
      cm[0] = cm[1];
      cm[1] = cm[2];
      cp[0] = cp[1];
      cp[1] = cp[2];
    }
  }
  if (dotmode != kDotNone) {
    double c;
    if (grid_reduce<false>(dot, partials, &st->counter[0], c) && threadIdx.x == 0) {
      // pcg.py:101-108 -- curvature check, then alpha = mu / curvature
      st->curv = c;
      if (c <= 0.0) {
        st->breakdown = 1;
        st->done = 1;
      } else {
        st->alpha = st->mu / c;
      }
    }
  }
}

StencilShape stencil_shape(const Geo& g, int mode, int sm_count) {
  StencilShape sh;
  const int ch = (mode == kInner) ? 32 : kHaloChunk;
  sh.nchunk = (g.T1 + ch - 1) / ch;
  const long long base = (long long)g.N * sh.nchunk;
  const long long target = (long long)sm_count * 40;   // ~40 warps of work per SM
  int nstrip = (int)std::max(1LL, (target + base - 1) / base);
  nstrip = std::min(nstrip, std::max(1, g.K / 8));
  sh.rows = (g.K + nstrip - 1) / nstrip;
  sh.nstrip = (g.K + sh.rows - 1) / sh.rows;
  sh.threads = 256;
  const long long warps = base * sh.nstrip;
  sh.blocks = (int)((warps * 32 + sh.threads - 1) / sh.threads);
  return sh;
}

template <int NS>
static cudaError_t launch_stencil_n(const Geo& g, const Ops& op, int mode, const double* x,
                                    double* y, const StencilShape& sh, double* partials,
                                    PcgState* st, int dotmode, cudaStream_t s) {
  switch (mode) {
    case kDelta:
      k_stencil<NS, kDelta><<<sh.blocks, sh.threads, 0, s>>>(g, op, x, y, sh.nchunk, sh.nstrip,
                                                             sh.rows, partials, st, dotmode);
      break;
    case kOuter:
      k_stencil<NS, kOuter><<<sh.blocks, sh.threads, 0, s>>>(g, op, x, y, sh.nchunk, sh.nstrip,
                                                             sh.rows, partials, st, kDotNone);
      break;
    default:
      k_stencil<NS, kInner><<<sh.blocks, sh.threads, 0, s>>>(g, op, x, y, sh.nchunk, sh.nstrip,
                                                             sh.rows, partials, st, kDotNone);
  }
  return cudaGetLastError();
}

cudaError_t launch_stencil(const Geo& g, const Ops& op, int mode, const double* x, double* y,
                           const StencilShape& sh, double* partials, PcgState* st, int dotmode,
                           cudaStream_t s) {
  switch (g.n) {
    case 1: return launch_stencil_n<1>(g, op, mode, x, y, sh, partials, st, dotmode, s);
    case 2: return launch_stencil_n<2>(g, op, mode, x, y, sh, partials, st, dotmode, s);
    case 3: return launch_stencil_n<3>(g, op, mode, x, y, sh, partials, st, dotmode, s);
    case 4: return launch_stencil_n<4>(g, op, mode, x, y, sh, partials, st, dotmode, s);
    case 8: return launch_stencil_n<8>(g, op, mode, x, y, sh, partials, st, dotmode, s);
    default: return cudaErrorInvalidValue;
  }
}

bool n_supported(int n) { return n == 1 || n == 2 || n == 3 || n == 4 || n == 8; }

}  // namespace gq
