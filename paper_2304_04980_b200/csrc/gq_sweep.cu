// One inner sweep of the nested block Jacobi preconditioner: for every (column pair v,
// stage t) solve the block tri-diagonal system  Phi_{v,t} theta = tau  with
//   tau = r  [+ Xi~ delta  (outer sweeps s >= 1)]  [+ Omega~ theta_prev  (inner l >= 1)]
// using the setup-time block Cholesky factors (explicit L_k^-1 and C_k), i.e.
//   forward  w_k = L_k^-1 (tau_k - C_k w_{k-1})
//   backward x_k = L_k^-T (w_k - C_{k+1}^T x_{k+1})
// Reference: NestedJacobiPreconditioner.inner_sweep / _pair_solves
// (gridlq/nested_jacobi.py:65-103), BlockTridiagCholesky.solve (block_linalg.py:336-358),
// the outer rhs r + apply_outer_coupling(delta) (nested_jacobi.py:117-121) and the inner
// rhs + apply_inner_coupling(theta) (kkt_assembly.py:645-662).
//
// Mapping: one lane = one chain (v, t); a warp holds 30 (outer sweeps: +2 halo lanes for
// the t+-1 exchange) or 32 consecutive stages of one pair, so the factor blocks of the
// chain (same for all stages of a class) are warp-uniform broadcast loads and every
// vector access of the warp is one contiguous segment in the stage-inner layout.  The
// right-hand side, including both coupling terms, is formed on the fly block by block:
// no intermediate vector is materialised.  The forward iterate w is parked in `out`
// (same addresses the backward sweep overwrites, so it stays in L2 between the sweeps).
#include "gq_internal.h"

namespace gq {

template <int Q>
__device__ __forceinline__ void ld_row(double* row, const double* __restrict__ p) {
#pragma unroll
  for (int c = 0; c < Q; c += 2) {
    double2 t = __ldg(reinterpret_cast<const double2*>(p + c));
    row[c] = t.x;
    row[c + 1] = t.y;
  }
}

template <int NS, bool INNER, bool OUTER>
__global__ void __launch_bounds__(128) k_sweep(Geo g, Ops op, const double* __restrict__ r,
                                               const double* __restrict__ th,
                                               const double* __restrict__ dl, double* out,
                                               double* partials, PcgState* st, int dotmode) {
  if (halted(st)) return;
  constexpr int Q = 4 * NS;
  constexpr int B2 = NS * NS;
  constexpr int CH = OUTER ? kHaloChunk : 32;
  const int nchunk = (g.T1 + CH - 1) / CH;
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const bool active = gw < (long long)g.V * nchunk;
  const int chunk = active ? (int)(gw % nchunk) : 0;
  const int v = active ? (int)(gw / nchunk) : 0;
  const int t = chunk * CH + lane - (OUTER ? 1 : 0);
  const bool tv = active && t >= 0 && t < g.T1;
  const bool useful = tv && (!OUTER || (lane >= 1 && lane <= kHaloChunk));
  const int pc = tv ? op.psi_cls[t] : 0;
  const int xce = (tv && t < g.T) ? op.xi_cls[t] : -1;
  const int xcf = (tv && t >= 1) ? op.xi_cls[t - 1] : -1;
  const double* F = op.fac + ((long long)pc * g.V + v) * g.nb * 2 * Q * Q;
  double dot = 0.0;

  auto LDD = [&](int jj, int ii) -> Vec<NS> {
    if (tv && jj >= 0 && jj < g.N && ii >= 0 && ii < g.K) return ldv_nc<NS>(dl + vidx(g, jj, ii, t));
    return vzero<NS>();
  };
  auto LDT = [&](int jj, int ii) -> Vec<NS> {
    if (tv && jj >= 0 && jj < g.N && ii >= 0 && ii < g.K) return ldv_nc<NS>(th + vidx(g, jj, ii, t));
    return vzero<NS>();
  };

  if (active) {
    double wprev[Q];
#pragma unroll
    for (int p = 0; p < Q; ++p) wprev[p] = 0.0;
    // ---------------- forward sweep ----------------
    for (int k = 0; k < g.nb; ++k) {
      double b[Q];
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int i = 2 * k + (s >> 1);
        const int j = 2 * v + (s & 1);
        const bool real = (i < g.K) && (j < g.N);   // warp-uniform
        Vec<NS> rv = (real && tv) ? ldv_nc<NS>(r + vidx(g, j, i, t)) : vzero<NS>();
        if (OUTER) {
          Vec<NS> e = vzero<NS>(), f = vzero<NS>();
          if (real) {
            const Vec<NS> d0 = LDD(j, i), dn = LDD(j, i - 1), ds = LDD(j, i + 1),
                          dw = LDD(j - 1, i), de = LDD(j + 1, i);
            const long long node = (long long)j * g.K + i;
            if (xce >= 0) {
              const double* E = op.xi + ((long long)xce * g.nk + node) * 5 * B2;
              mac<NS>(e, E + 0 * B2, d0);
              mac<NS>(e, E + 1 * B2, dn);
              mac<NS>(e, E + 2 * B2, ds);
              mac<NS>(e, E + 3 * B2, dw);
              mac<NS>(e, E + 4 * B2, de);
            }
            if (xcf >= 0) {
              const double* Fx = op.xit + ((long long)xcf * g.nk + node) * 5 * B2;
              mac<NS>(f, Fx + 0 * B2, d0);
              mac<NS>(f, Fx + 1 * B2, dn);
              mac<NS>(f, Fx + 2 * B2, ds);
              mac<NS>(f, Fx + 3 * B2, dw);
              mac<NS>(f, Fx + 4 * B2, de);
            }
          }
          const Vec<NS> eu = shfl_up<NS>(e, 1);
          const Vec<NS> fd = shfl_down<NS>(f, 1);
#pragma unroll
          for (int kk = 0; kk < NS; ++kk) {
            double o = 0.0;
            if (t >= 1) o -= eu.v[kk];
            if (t < g.T) o -= fd.v[kk];
            rv.v[kk] += o;
          }
        }
        if (INNER && real) {
          const double* P = op.psi + ((long long)pc * g.nk + (long long)j * g.K + i) * 13 * B2;
          Vec<NS> sacc = vzero<NS>();
          if ((s & 1) == 0) {
            mac<NS>(sacc, P + 7 * B2, LDT(j - 2, i));
            mac<NS>(sacc, P + 9 * B2, LDT(j - 1, i - 1));
            mac<NS>(sacc, P + 3 * B2, LDT(j - 1, i));
            mac<NS>(sacc, P + 11 * B2, LDT(j - 1, i + 1));
            mac<NS>(sacc, P + 8 * B2, LDT(j + 2, i));
          } else {
            mac<NS>(sacc, P + 7 * B2, LDT(j - 2, i));
            mac<NS>(sacc, P + 10 * B2, LDT(j + 1, i - 1));
            mac<NS>(sacc, P + 4 * B2, LDT(j + 1, i));
            mac<NS>(sacc, P + 12 * B2, LDT(j + 1, i + 1));
            mac<NS>(sacc, P + 8 * B2, LDT(j + 2, i));
          }
#pragma unroll
          for (int kk = 0; kk < NS; ++kk) rv.v[kk] -= sacc.v[kk];
        }
#pragma unroll
        for (int kk = 0; kk < NS; ++kk) b[s * NS + kk] = rv.v[kk];
      }
      const double* Lk = F + (long long)k * 2 * Q * Q;
      double seg[Q];
      if (k > 0) {
        const double* Ck = Lk + Q * Q;
#pragma unroll
        for (int p = 0; p < Q; ++p) {
          double row[Q];
          ld_row<Q>(row, Ck + p * Q);
          double sacc = 0.0;
#pragma unroll
          for (int c = 0; c < Q; ++c) sacc = fma(row[c], wprev[c], sacc);
          seg[p] = b[p] - sacc;
        }
      } else {
#pragma unroll
        for (int p = 0; p < Q; ++p) seg[p] = b[p];
      }
#pragma unroll
      for (int p = 0; p < Q; ++p) {
        double row[Q];
        ld_row<Q>(row, Lk + p * Q);
        double sacc = 0.0;
#pragma unroll
        for (int c = 0; c <= p; ++c) sacc = fma(row[c], seg[c], sacc);
        wprev[p] = sacc;
      }
      if (useful) {
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const int i = 2 * k + (s >> 1);
          const int j = 2 * v + (s & 1);
          if (i < g.K && j < g.N) {
            Vec<NS> w;
#pragma unroll
            for (int kk = 0; kk < NS; ++kk) w.v[kk] = wprev[s * NS + kk];
            stv<NS>(out + vidx(g, j, i, t), w);
          }
        }
      }
    }
    // ---------------- backward sweep ----------------
    double xn[Q];
#pragma unroll
    for (int p = 0; p < Q; ++p) xn[p] = 0.0;
    for (int k = g.nb - 1; k >= 0; --k) {
      double w[Q];
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int i = 2 * k + (s >> 1);
        const int j = 2 * v + (s & 1);
        Vec<NS> wv = (useful && i < g.K && j < g.N) ? ldv<NS>(out + vidx(g, j, i, t)) : vzero<NS>();
#pragma unroll
        for (int kk = 0; kk < NS; ++kk) w[s * NS + kk] = wv.v[kk];
      }
      double seg[Q];
      if (k + 1 < g.nb) {
        const double* Cn = F + (long long)(k + 1) * 2 * Q * Q + Q * Q;
        double acc[Q];
#pragma unroll
        for (int p = 0; p < Q; ++p) acc[p] = 0.0;
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          double row[Q];
          ld_row<Q>(row, Cn + c * Q);
#pragma unroll
          for (int p = 0; p < Q; ++p) acc[p] = fma(row[p], xn[c], acc[p]);
        }
#pragma unroll
        for (int p = 0; p < Q; ++p) seg[p] = w[p] - acc[p];
      } else {
#pragma unroll
        for (int p = 0; p < Q; ++p) seg[p] = w[p];
      }
      const double* Lk = F + (long long)k * 2 * Q * Q;
#pragma unroll
      for (int p = 0; p < Q; ++p) xn[p] = 0.0;
#pragma unroll
      for (int c = 0; c < Q; ++c) {
        double row[Q];
        ld_row<Q>(row, Lk + c * Q);
#pragma unroll
        for (int p = 0; p <= c; ++p) xn[p] = fma(row[p], seg[c], xn[p]);
      }
      if (useful) {
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const int i = 2 * k + (s >> 1);
          const int j = 2 * v + (s & 1);
          if (i < g.K && j < g.N) {
            Vec<NS> xv;
#pragma unroll
            for (int kk = 0; kk < NS; ++kk) xv.v[kk] = xn[s * NS + kk];
            stv<NS>(out + vidx(g, j, i, t), xv);
            if (dotmode != kDotNone) {
              const Vec<NS> rv = ldv_nc<NS>(r + vidx(g, j, i, t));
#pragma unroll
              for (int kk = 0; kk < NS; ++kk) dot = fma(xv.v[kk], rv.v[kk], dot);
            }
          }
        }
      }
    }
  }
  if (dotmode != kDotNone) {
    double mu;
    if (grid_reduce<false>(dot, partials, &st->counter[2], mu) && threadIdx.x == 0) {
      if (dotmode == kDotInit) {
        st->mu = mu;                       // pcg.py:92
      } else {
        st->beta = mu / st->mu;            // pcg.py:127-131
        st->mu = mu;
      }
    }
  }
}

SweepShape sweep_shape(const Geo& g, bool outer) {
  SweepShape sh;
  const int ch = outer ? kHaloChunk : 32;
  const long long warps = (long long)g.V * ((g.T1 + ch - 1) / ch);
  sh.threads = 128;
  sh.blocks = (int)((warps * 32 + sh.threads - 1) / sh.threads);
  return sh;
}

template <int NS>
static cudaError_t launch_sweep_n(const Geo& g, const Ops& op, bool inner, bool outer,
                                  const double* r, const double* th, const double* dl,
                                  double* out, const SweepShape& sh, double* partials,
                                  PcgState* st, int dotmode, cudaStream_t s) {
#define GQ_SWEEP(I, O) \
  k_sweep<NS, I, O><<<sh.blocks, sh.threads, 0, s>>>(g, op, r, th, dl, out, partials, st, dotmode)
  if (inner && outer) GQ_SWEEP(true, true);
  else if (inner) GQ_SWEEP(true, false);
  else if (outer) GQ_SWEEP(false, true);
  else GQ_SWEEP(false, false);
#undef GQ_SWEEP
  return cudaGetLastError();
}

cudaError_t launch_sweep(const Geo& g, const Ops& op, bool inner, bool outer, const double* r,
                         const double* th, const double* dl, double* out, const SweepShape& sh,
                         double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  switch (g.n) {
    case 1: return launch_sweep_n<1>(g, op, inner, outer, r, th, dl, out, sh, partials, st, dotmode, s);
    case 2: return launch_sweep_n<2>(g, op, inner, outer, r, th, dl, out, sh, partials, st, dotmode, s);
    case 3: return launch_sweep_n<3>(g, op, inner, outer, r, th, dl, out, sh, partials, st, dotmode, s);
    case 4: return launch_sweep_n<4>(g, op, inner, outer, r, th, dl, out, sh, partials, st, dotmode, s);
    case 8: return launch_sweep_n<8>(g, op, inner, outer, r, th, dl, out, sh, partials, st, dotmode, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gq
