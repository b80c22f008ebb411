// C ABI of libgridlq_b200.so: context lifetime, setup, unit applies and the PCG driver.
//
// PCG driver = pcg_solve's loop (gridlq/pcg.py:98-131) as one captured CUDA graph per
// step.  All scalars (mu, alpha, beta, curvature, residual), the step counter, the
// residual history and the done/converged/breakdown flags live in device memory, so a
// step needs no host round trip; the host launches the graph in growing batches and only
// reads the 64-byte state between batches.  Kernels of a step after convergence,
// breakdown or the step budget see `done` and exit immediately, which preserves the
// reference's exact stopping semantics while launching ahead.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <map>
#include <array>
#include <algorithm>
#include <functional>
#include <thread>
#include <tuple>
#include <sys/mman.h>

#include "gq_internal.h"
#include "../../include/gridlq_b200.h"

using namespace gq;

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

namespace gq {
// for the entry points that live in other translation units (gq_rhs.cu)
int api_fail(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace gq

#define CK(call)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      return fail(GQ_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr int kStageChunks = 8;   // pinned-staging pipeline depth (import_vec / export_vec)

struct gq_ctx {
  Geo g{};
  int m = 0, L = 2, S = 2, n_dyn = 0, n_cost = 0, npc = 0, nxc = 0, sm_count = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;          // parallel graph branch (x update)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  double *A = nullptr, *B = nullptr, *R = nullptr, *C = nullptr, *Q = nullptr;
  double *qinv = nullptr, *rinv = nullptr, *brb = nullptr;
  double *psi = nullptr, *xi = nullptr, *xit = nullptr, *fac = nullptr;
  int *psi_cls = nullptr, *xi_cls = nullptr, *psi_keys = nullptr, *xi_keys = nullptr;
  int *dcls = nullptr, *ccls = nullptr;   // per-stage dynamics / cost class (recovery)
  double *x = nullptr, *r = nullptr, *d = nullptr, *y = nullptr, *q = nullptr;
  double *th[2] = {nullptr, nullptr}, *dl[2] = {nullptr, nullptr};
  double *tmp0 = nullptr, *tmp1 = nullptr;
  int t0pad = 0;                    // stages of zero padding in front of every work vector
  std::vector<double*> vec_bases;   // their allocations (the vectors start t0pad stages in)
  double* rs = nullptr;        // r + Xi~ delta of the current outer sweep (fast path)
  double *oprow = nullptr, *omega = nullptr, *fac3 = nullptr, *fac4 = nullptr;
  FastOps fo{};
  double *cff = nullptr, *cfb = nullptr;
  int4* seg = nullptr;
  ChainOps co{};
  bool chain = false;          // lean DMMA chain sweeps (n in {2, 4})
  bool fuse_x = false;         // x update fused into the direction update (L2-resident sizes)
  bool fuse_r = false;         // r update fused into the first outer sweep (chain kernel)
  bool grid = false;           // lean n = 2 grid stencils
  bool dstep = false;          // t-loop factored Delta apply (n = 2)
  DstepOps dso{};
  CUtensorMap map_d{}, map_tmp0{};   // TMA views of the Delta inputs (d, unit-apply scratch)
  CUtensorMap map_y{};               // ... and of its output
  bool rstep = false;          // tiled outer rhs on the same TMA views
  std::vector<std::tuple<const double*, int, CUtensorMap>> maps;   // (vector, halo) -> view
  bool st8 = false;            // n = 8 DMMA block stencils
  GridShape gsh{};
  bool fast = false;           // pipelined v2 kernels eligible (stage classes warp-compatible)
  double* partials = nullptr;
  PcgState* st = nullptr;
  PcgState* h_st = nullptr;   // pinned mirror
  double* h_stage = nullptr;  // pinned staging vector for pageable host buffers
  cudaEvent_t ev_stage[kStageChunks] = {};   // its chunked copies
  double* hist = nullptr;
  long long hist_cap = 0;
  SetupErr* err = nullptr;
  Ops op{};
  StencilShape sh_delta{}, sh_outer{}, sh_inner{};
  SweepShape sw{}, sw_outer{};
  int vblocks = 0;
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  bool started = false;
  int use_precond = 1;
  std::vector<std::string> knames;
  // stage-slab mode: local halo stages (-1: none), a pinned scratch for status reads
  bool slab = false;
  int slab_t0 = -1, slab_t1 = -1;
};

extern "C" const char* gq_last_error(void) { return g_err.c_str(); }
extern "C" const char* gq_version(void) { return "gridlq_b200 0.1.0 (sm_100a, fp64)"; }

static bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

template <typename T>
static cudaError_t dalloc(T** p, size_t count) {
  return cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T));
}

static void release(gq_ctx* c) {
  if (!c) return;
  for (auto& ge : c->gexec)
    if (ge) cudaGraphExecDestroy(ge);
  void* ptrs[] = {c->A, c->B, c->R, c->C, c->Q, c->qinv, c->rinv, c->brb, c->psi, c->xi,
                  c->xit, c->fac, c->psi_cls, c->xi_cls, c->psi_keys, c->xi_keys, c->oprow, c->omega, c->fac3, c->fac4, c->cff, c->cfb, c->seg, c->dcls, c->ccls, c->partials, c->st, c->hist, c->err};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (double* p : c->vec_bases)
    if (p) cudaFree(p);
  if (c->h_st) cudaFreeHost(c->h_st);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  for (cudaEvent_t& e : c->ev_stage)
    if (e) cudaEventDestroy(e);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->side) cudaStreamDestroy(c->side);
  delete c;
}

extern "C" void gq_destroy(gq_ctx* ctx) { release(ctx); }

extern "C" int64_t gq_dim(const gq_ctx* ctx) { return ctx ? ctx->g.dim : -1; }

extern "C" int gq_set_stream(gq_ctx* ctx, void* stream) {
  if (!ctx) return fail(GQ_INVALID_ARG, "null context");
  ctx->stream = static_cast<cudaStream_t>(stream);
  for (auto& ge : ctx->gexec)
    if (ge) {
      cudaGraphExecDestroy(ge);
      ge = nullptr;
    }
  return GQ_OK;
}

extern "C" int gq_set_sweeps(gq_ctx* ctx, int32_t inner_sweeps, int32_t outer_sweeps) {
  if (!ctx) return fail(GQ_INVALID_ARG, "null context");
  if (inner_sweeps < 1 || outer_sweeps < 1)
    return fail(GQ_INVALID_ARG, "sweep budgets must be at least 1");
  if (inner_sweeps == ctx->L && outer_sweeps == ctx->S) return GQ_OK;
  ctx->L = inner_sweeps;
  ctx->S = outer_sweeps;
  for (auto& ge : ctx->gexec)
    if (ge) {
      cudaGraphExecDestroy(ge);
      ge = nullptr;
    }
  return GQ_OK;
}

extern "C" int gq_synchronize(gq_ctx* ctx) {
  if (!ctx) return fail(GQ_INVALID_ARG, "null context");
  CK(cudaStreamSynchronize(ctx->stream));
  return GQ_OK;
}

static int check_setup_err(gq_ctx* c) {
  SetupErr e;
  CK(cudaMemcpy(&e, c->err, sizeof(e), cudaMemcpyDeviceToHost));
  if (e.code == 0) return GQ_OK;
  char buf[256];
  if (e.code == 1)
    snprintf(buf, sizeof(buf),
             "pivot %.3e at index %d (threshold %.3e) in pair block %d of pair %d, stage class %d",
             e.pivot, e.j, e.tol, e.k, e.v, e.cls);
  else
    snprintf(buf, sizeof(buf), "cost weight %d: pivot %.3e at index %d (threshold %.3e)", e.cls,
             e.pivot, e.j, e.tol);
  return fail(GQ_NOT_SPD, buf);
}

extern "C" int gq_create(const gq_problem_desc* desc, int32_t inner_sweeps,
                         int32_t outer_sweeps, gq_ctx** out) {
  if (!desc || !out) return fail(GQ_INVALID_ARG, "null argument");
  *out = nullptr;
  const gq_problem_desc& D = *desc;
  if (D.K < 1 || D.N < 1 || D.T < 1)
    return fail(GQ_INVALID_ARG, "grid dimensions must be positive");
  if (D.n < 1 || D.m < 1 || D.m > 8) return fail(GQ_INVALID_ARG, "bad state/input dimension");
  if (!n_supported(D.n))
    return fail(GQ_UNSUPPORTED, "state dimension n=" + std::to_string(D.n) +
                                    " has no compiled kernel (supported: 1, 2, 3, 4, 8)");
  if (inner_sweeps < 1 || outer_sweeps < 1)
    return fail(GQ_INVALID_ARG, "sweep budgets must be at least 1");
  if (D.n_dyn < 1 || D.n_cost < 1) return fail(GQ_INVALID_ARG, "need at least one data set");
  for (int t = 0; t < D.T; ++t)
    if (D.dyn_class[t] < 0 || D.dyn_class[t] >= D.n_dyn)
      return fail(GQ_INVALID_ARG, "dyn_class out of range");
  for (int t = 0; t <= D.T; ++t)
    if (D.cost_class[t] < 0 || D.cost_class[t] >= D.n_cost)
      return fail(GQ_INVALID_ARG, "cost_class out of range");

  gq_ctx* c = new gq_ctx();
  c->m = D.m;
  c->L = inner_sweeps;
  c->S = outer_sweeps;
  c->n_dyn = D.n_dyn;
  c->n_cost = D.n_cost;
  Geo& g = c->g;
  g.K = D.K;
  g.N = D.N;
  g.T = D.T;
  g.T1 = D.T + 1;
  g.n = D.n;
  g.V = (D.N + 1) / 2;
  g.nb = (D.K + 1) / 2;
  g.nk = (long long)D.K * D.N;
  g.dim = g.nk * D.n * g.T1;
  {
    // x += alpha d rides in the direction update (one pass over d less; the five-stream
    // kernel runs at 6.4 TB/s): headline 710 against 693 steps/s with the x update on its own
    // graph branch, configs 1-3 +3-4% for one kernel less.  GQ_FUSE_X=0 brings the branch back.
    const char* e = getenv("GQ_FUSE_X");
    c->fuse_x = (e && *e) ? *e == '1' : true;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, dev);

  // stage classes (GridArrays.psi_classes / xi_classes)
  std::map<std::array<int, 3>, int> pmap;
  std::vector<int> pcls(g.T1), pkeys;
  for (int t = 0; t < g.T1; ++t) {
    std::array<int, 3> key = t == 0 ? std::array<int, 3>{D.cost_class[0], -1, -1}
                                    : std::array<int, 3>{D.cost_class[t], D.dyn_class[t - 1],
                                                         D.cost_class[t - 1]};
    auto it = pmap.find(key);
    if (it == pmap.end()) {
      it = pmap.emplace(key, (int)pmap.size()).first;
      pkeys.insert(pkeys.end(), key.begin(), key.end());
    }
    pcls[t] = it->second;
  }
  // Stage stride and front padding of the device vectors: the stage where the long class run
  // starts (1 when stage 0 is a class of its own, as for every time-invariant problem) sits
  // on a 128-byte boundary of the allocation and every node spans a multiple of 8 stages, so
  // the 8-stage records the chain sweeps move are whole 128-byte lines (GQ_NO_PAD=1: dense).
  {
    const char* np = getenv("GQ_NO_PAD");
    const int first = (g.T1 > 1 && pcls[0] != pcls[1]) ? 1 : 0;
    // short horizons stay dense: the padding must not cost more than a quarter of the bytes
    const int padded = ((8 - first) % 8 + g.T1 + 7) / 8 * 8;
    const bool dense = (np && *np == '1') || 4 * padded > 5 * g.T1;
    c->t0pad = dense ? 0 : (8 - first) % 8;
    g.TS = dense ? g.T1 : padded;
    g.T0 = c->t0pad;
    g.span = (g.nk - 1) * (long long)g.TS * g.n + (long long)g.T1 * g.n;
  }
  std::map<std::array<int, 2>, int> xmap;
  std::vector<int> xcls(std::max(g.T, 1)), xkeys;
  for (int t = 0; t < g.T; ++t) {
    std::array<int, 2> key{D.dyn_class[t], D.cost_class[t]};
    auto it = xmap.find(key);
    if (it == xmap.end()) {
      it = xmap.emplace(key, (int)xmap.size()).first;
      xkeys.insert(xkeys.end(), key.begin(), key.end());
    }
    xcls[t] = it->second;
  }
  c->npc = (int)pmap.size();
  c->nxc = (int)xmap.size();
  {
    // v2 kernels: one Xi class and at most two Psi classes inside every warp's stage range
    auto ok_chunks = [&](int chunk, int halo) {
      for (int t0 = -halo; t0 < g.T1; t0 += chunk) {
        int ca = -1, cb = -1;
        for (int t = std::max(t0, 0); t < std::min(t0 + 32, g.T1); ++t) {
          const int cl = pcls[t];
          if (ca < 0 || cl == ca) ca = cl;
          else if (cb < 0 || cl == cb) cb = cl;
          else return false;
        }
      }
      return true;
    };
    const char* force = getenv("GQ_FORCE_V1");
    c->fast = fast_supported(g.n) && c->nxc == 1 && ok_chunks(kHaloChunk, 1) &&
              ok_chunks(32, 0) && !(force && *force == '1');
  }

  const int n = D.n, m = D.m, q = 4 * n;
  const size_t nn = (size_t)n * n;
  const size_t nk = (size_t)g.nk;
  auto bail = [&](int code) {
    release(c);
    return code;
  };
#define CKB(call)                                                                          \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return bail(fail(GQ_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_))); \
  } while (0)
  CKB(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  CKB(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  CKB(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  CKB(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  CKB(dalloc(&c->A, D.n_dyn * nk * nn));
  CKB(dalloc(&c->B, D.n_dyn * nk * n * m));
  CKB(dalloc(&c->R, D.n_dyn * nk * m * m));
  CKB(dalloc(&c->C, D.n_dyn * 4 * nk * nn));
  CKB(dalloc(&c->Q, D.n_cost * nk * nn));
  CKB(cudaMemcpy(c->A, D.A, D.n_dyn * nk * nn * 8, cudaMemcpyHostToDevice));
  CKB(cudaMemcpy(c->B, D.B, D.n_dyn * nk * n * m * 8, cudaMemcpyHostToDevice));
  CKB(cudaMemcpy(c->R, D.R, D.n_dyn * nk * m * m * 8, cudaMemcpyHostToDevice));
  CKB(cudaMemcpy(c->C, D.C, D.n_dyn * 4 * nk * nn * 8, cudaMemcpyHostToDevice));
  CKB(cudaMemcpy(c->Q, D.Q, D.n_cost * nk * nn * 8, cudaMemcpyHostToDevice));
  CKB(dalloc(&c->psi_cls, g.T1));
  CKB(dalloc(&c->xi_cls, xcls.size()));
  CKB(dalloc(&c->psi_keys, pkeys.size()));
  CKB(dalloc(&c->xi_keys, std::max<size_t>(xkeys.size(), 1)));
  CKB(cudaMemcpy(c->psi_cls, pcls.data(), pcls.size() * 4, cudaMemcpyHostToDevice));
  CKB(cudaMemcpy(c->xi_cls, xcls.data(), xcls.size() * 4, cudaMemcpyHostToDevice));
  CKB(cudaMemcpy(c->psi_keys, pkeys.data(), pkeys.size() * 4, cudaMemcpyHostToDevice));
  if (!xkeys.empty())
    CKB(cudaMemcpy(c->xi_keys, xkeys.data(), xkeys.size() * 4, cudaMemcpyHostToDevice));
  CKB(dalloc(&c->dcls, std::max(g.T, 1)));
  CKB(dalloc(&c->ccls, g.T1));
  if (g.T > 0)
    CKB(cudaMemcpy(c->dcls, D.dyn_class, (size_t)g.T * 4, cudaMemcpyHostToDevice));
  CKB(cudaMemcpy(c->ccls, D.cost_class, (size_t)g.T1 * 4, cudaMemcpyHostToDevice));
  CKB(dalloc(&c->err, 1));
  CKB(cudaMemset(c->err, 0, sizeof(SetupErr)));

  // cost inverses, B R^-1 B'
  CKB(dalloc(&c->qinv, D.n_cost * nk * nn));
  CKB(dalloc(&c->rinv, D.n_dyn * nk * m * m));
  CKB(dalloc(&c->brb, D.n_dyn * nk * nn));
  CKB(launch_spd_inverse(c->Q, c->qinv, D.n_cost * (long long)nk, n, c->err, c->stream));
  CKB(launch_spd_inverse(c->R, c->rinv, D.n_dyn * (long long)nk, m, c->err, c->stream));
  CKB(cudaStreamSynchronize(c->stream));
  {
    int rc = check_setup_err(c);
    if (rc != GQ_OK) return bail(rc);
  }
  CKB(launch_brb(g, m, D.n_dyn, c->B, c->rinv, c->brb, c->stream));
  // operator blocks per stage class
  CKB(dalloc(&c->psi, (size_t)c->npc * nk * 13 * nn));
  CKB(dalloc(&c->xi, (size_t)std::max(c->nxc, 1) * nk * 5 * nn));
  CKB(dalloc(&c->xit, (size_t)std::max(c->nxc, 1) * nk * 5 * nn));
  CKB(launch_xi(g, c->nxc, c->xi_keys, c->A, c->C, c->qinv, c->xi, c->xit, c->stream));
  CKB(launch_psi(g, c->npc, c->psi_keys, c->A, c->C, c->qinv, c->brb, c->psi, c->stream));
  // pair factors
  double* scratch = nullptr;
  CKB(dalloc(&c->fac, (size_t)c->npc * g.V * g.nb * 2 * q * q));
  CKB(dalloc(&scratch, (size_t)c->npc * g.V * 5 * q * q));
  cudaError_t fe = launch_factor(g, c->npc, c->psi, c->fac, scratch, c->err, c->stream);
  cudaError_t se = cudaStreamSynchronize(c->stream);
  cudaFree(scratch);
  CKB(fe);
  CKB(se);
  {
    int rc = check_setup_err(c);
    if (rc != GQ_OK) return bail(rc);
  }
  c->op = Ops{c->psi, c->xi, c->xit, c->fac, c->psi_cls, c->xi_cls};
  if (c->fast) {
    CKB(dalloc(&c->oprow, (size_t)c->npc * nk * 23 * nn));
    CKB(dalloc(&c->omega, (size_t)c->npc * nk * 5 * nn));
    // per-lane sweep factors: only needed when the chain kernel does not run the sweeps
    if (!chain_supported(g.n)) {
      if (tc_supported(g.n))
        CKB(dalloc(&c->fac4, (size_t)c->npc * g.V * g.nb * 4 * q * q));
      else
        CKB(dalloc(&c->fac3, (size_t)c->npc * g.V * g.nb * 3 * q * q));
    }
    CKB(launch_build_fast(g, c->npc, c->op, c->oprow, c->omega, c->fac3, c->fac4, c->stream));
    CKB(cudaStreamSynchronize(c->stream));
    c->fo = FastOps{c->oprow, c->omega, c->fac3, c->psi_cls, c->fac4};
    if (chain_supported(g.n)) {
      // class-pure chunks of <= w stages: runs of equal Psi class split into w's
      auto chunks = [&](int w) {
        std::vector<int4> segs;
        for (int t = 0; t < g.T1;) {
          int e = t + 1;
          while (e < g.T1 && e - t < w && pcls[e] == pcls[t]) ++e;
          segs.push_back(make_int4(t, e - t, pcls[t], 0));
          t = e;
        }
        return segs;
      };
      const std::vector<int4> s8 = chunks(8), s16 = chunks(16);
      CKB(dalloc(&c->cff, chain_ff_doubles(g, c->npc)));
      CKB(dalloc(&c->cfb, chain_fb_doubles(g, c->npc)));
      CKB(dalloc(&c->seg, s8.size() + s16.size()));
      CKB(cudaMemcpy(c->seg, s8.data(), s8.size() * sizeof(int4), cudaMemcpyHostToDevice));
      CKB(cudaMemcpy(c->seg + s8.size(), s16.data(), s16.size() * sizeof(int4),
                     cudaMemcpyHostToDevice));
      CKB(launch_build_chain(g, c->npc, c->fac, c->omega, c->cff, c->cfb, c->stream));
      CKB(cudaStreamSynchronize(c->stream));
      c->co = ChainOps{c->cff, c->cfb, c->seg, (int)s8.size(), c->seg + s8.size(),
                       (int)s16.size()};
      {
        // classes without coupling tiles (stage 0: Psi_0 = Q_0^-1) read only L^-1 and L^-T
        int* flags = nullptr;
        CKB(dalloc(&flags, (size_t)c->npc));
        cudaError_t me = launch_chainm_mark(g, c->npc, c->co, c->seg, (int)s8.size(), flags,
                                            c->stream);
        if (me == cudaSuccess) me = cudaStreamSynchronize(c->stream);
        cudaFree(flags);
        CKB(me);
      }
      c->chain = true;
      c->st8 = st8_supported(g, c->nxc);   // n = 4: DMMA block stencils (two nodes per warp)
    }
  }

  if (!c->fast && g.n == 8 && chain_supported(g.n)) {
    // n = 8: DMMA pair-chain sweeps without the fast-path stencils (generic v1 stencils for
    // Delta and Xi~); the chain tiles need the cross-pair Psi blocks
    std::vector<int4> s8;
    for (int t = 0; t < g.T1;) {
      int e = t + 1;
      while (e < g.T1 && e - t < 8 && pcls[e] == pcls[t]) ++e;
      s8.push_back(make_int4(t, e - t, pcls[t], 0));
      t = e;
    }
    CKB(dalloc(&c->omega, (size_t)c->npc * nk * 5 * nn));
    CKB(launch_build_omega(g, c->npc, c->psi, c->omega, c->stream));
    CKB(dalloc(&c->cff, chain_ff_doubles(g, c->npc)));
    CKB(dalloc(&c->cfb, chain_fb_doubles(g, c->npc)));
    // CTA items of the n = 8 CTA-shared kernel: runs of one class, <= 8 segments each
    std::vector<int4> grp;
    for (size_t i = 0; i < s8.size();) {
      size_t e = i + 1;
      while (e < s8.size() && e - i < 8 && s8[e].z == s8[i].z) ++e;
      grp.push_back(make_int4((int)i, (int)(e - i), s8[i].z, 0));
      i = e;
    }
    CKB(dalloc(&c->seg, s8.size() + grp.size()));
    CKB(cudaMemcpy(c->seg, s8.data(), s8.size() * sizeof(int4), cudaMemcpyHostToDevice));
    CKB(cudaMemcpy(c->seg + s8.size(), grp.data(), grp.size() * sizeof(int4),
                   cudaMemcpyHostToDevice));
    CKB(launch_build_chain(g, c->npc, c->fac, c->omega, c->cff, c->cfb, c->stream));
    CKB(cudaStreamSynchronize(c->stream));
    c->co = ChainOps{c->cff, c->cfb, c->seg, (int)s8.size(), c->seg, (int)s8.size(), c->omega,
                     c->seg + s8.size(), (int)grp.size()};
    c->chain = true;
    c->st8 = st8_supported(g, c->nxc);
  }
  {
    const char* e = getenv("GQ_NO_FUSE_R");
    // n = 8: the fused outer sweep measured 4.1 ms against 2.4 + 0.5 ms split (config 5)
    c->fuse_r = c->chain && g.n != 8 && !(e && *e == '1');
  }
  // work vectors (stage-inner layout) and the reference-layout staging buffers
  const size_t vlen = (size_t)g.nk * g.TS * g.n + (size_t)(c->t0pad + 8) * g.n;
  double** vecs[] = {&c->x, &c->r, &c->d, &c->y, &c->q, &c->th[0], &c->th[1],
                     &c->dl[0], &c->dl[1], &c->tmp0, &c->tmp1, &c->rs};
  for (double** p : vecs) {
    double* base = nullptr;
    CKB(dalloc(&base, vlen));
    c->vec_bases.push_back(base);
    CKB(cudaMemset(base, 0, vlen * sizeof(double)));   // the padding stages stay zero
    *p = base + (size_t)c->t0pad * g.n;
  }
  c->sh_delta = stencil_shape(g, kDelta, c->sm_count);
  c->grid = c->fast && grid_supported(g.n);
  if (c->grid) c->gsh = grid_shape(g, c->sm_count);
  {
    const char* e = getenv("GQ_NO_DSTEP");
    const char* f = getenv("GQ_FORCE_V1");
    if (dstep_supported(g) && dstep_preferred(g, c->sm_count) && !(e && *e == '1') &&
        !(f && *f == '1') &&
        dstep_make_map(g, c->d, 2, &c->map_d) &&
        dstep_make_map(g, c->tmp0, 2, &c->map_tmp0) &&
        dstep_make_map(g, c->y, 0, &c->map_y)) {
      c->dso = DstepOps{c->A, c->C, c->qinv, c->brb, c->dcls, c->ccls};
      c->dstep = true;
      const char* r = getenv("GQ_NO_RSTEP");
      c->rstep = c->nxc == 1 && !(r && *r == '1');   // tiled outer rhs (one Xi class)
    }
  }
  c->sh_outer = stencil_shape(g, kOuter, c->sm_count);
  c->sh_inner = stencil_shape(g, kInner, c->sm_count);
  c->sw = sweep_shape(g, false);
  c->sw_outer = sweep_shape(g, true);
  c->vblocks = vec_blocks(c->sm_count);
  long long maxb = std::max({(long long)c->sh_delta.blocks, (long long)c->sw.blocks,
                             (long long)c->sw_outer.blocks, (long long)c->vblocks,
                             fast_max_blocks(g, c->sh_delta, c->sm_count),
                             fast_max_blocks(g, c->sh_outer, c->sm_count),
                             c->chain ? chain_max_blocks(g, c->co.nseg, c->sm_count) : 0LL,
                             c->st8 ? st8_max_blocks(c->sm_count) : 0LL,
                             c->chain ? (long long)c->sm_count * 2 : 0LL,
                             c->dstep ? dstep_max_blocks(c->sm_count) : 0LL,
                             c->chain ? chain_fr_max_blocks(g, c->co.nseg, c->sm_count) : 0LL,
                             c->grid ? (long long)c->gsh.blocks : 0LL});
  CKB(dalloc(&c->partials, (size_t)maxb + 32));
  CKB(dalloc(&c->st, 1));
  CKB(cudaMemset(c->st, 0, sizeof(PcgState)));
  CKB(cudaMallocHost(reinterpret_cast<void**>(&c->h_st), sizeof(PcgState)));
  // pinned staging for pageable host vectors (see export_vec); part of setup, not of a solve
  if (g.dim * 8 >= (8LL << 20))
    CKB(cudaMallocHost(reinterpret_cast<void**>(&c->h_stage), (size_t)g.dim * 8));
  memset(c->h_st, 0, sizeof(PcgState));
#undef CKB
  *out = c;
  return GQ_OK;
}

// ---- boundary helpers -----------------------------------------------------------------

// user vector (reference layout, host or device) -> internal vector `dst`
static int ensure_stage(gq_ctx* c);
static size_t stage_chunk_begin(const gq_ctx* c, int k);
static bool is_pageable_host(const void* p);
static void parallel_copy(double* dst, const double* src, size_t n);

static int import_vec(gq_ctx* c, const double* src, double* dst) {
  const double* ref = src;
  if (!is_device_ptr(src)) {
    if (is_pageable_host(src) && c->g.dim * 8 >= (8LL << 20)) {
      int rc = ensure_stage(c);
      if (rc) return rc;
      CK(cudaStreamSynchronize(c->stream));   // the stage may still feed an earlier copy
      // chunked: the host copy of chunk k+1 overlaps the DMA of chunk k
      for (int k = 0; k < kStageChunks; ++k) {
        const size_t b = stage_chunk_begin(c, k), e = stage_chunk_begin(c, k + 1);
        parallel_copy(c->h_stage + b, src + b, e - b);
        CK(cudaMemcpyAsync(c->tmp1 + b, c->h_stage + b, (e - b) * 8, cudaMemcpyHostToDevice,
                           c->stream));
      }
    } else {
      CK(cudaMemcpyAsync(c->tmp1, src, c->g.dim * 8, cudaMemcpyHostToDevice, c->stream));
    }
    ref = c->tmp1;
  }
  if (c->g.TS != c->g.T1 || c->t0pad)
    // padded layout: the transpose writes the real stages only; clear the padding too, so
    // that nothing a previous solve left there (NaN scalars after a breakdown) reaches the
    // flat reductions
    CK(cudaMemsetAsync(dst - (size_t)c->t0pad * c->g.n, 0,
                       ((size_t)c->g.span + (size_t)c->t0pad * c->g.n) * 8, c->stream));
  CK(launch_to_internal(c->g, ref, dst, c->stream));
  return GQ_OK;
}

// internal vector -> user vector (reference layout, host or device); synchronises
// pageable host buffers go through a persistent pinned staging vector and a multi-threaded
// host copy: a direct pageable cudaMemcpy of a 210 MB vector runs at ~5 GB/s (measured)
static bool is_pageable_host(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

static void parallel_copy(double* dst, const double* src, size_t n) {
  const size_t bytes = n * 8;
  unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (bytes < (8u << 20)) nt = 1;
  if (nt == 1) {
    memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  const size_t per = (n + nt - 1) / nt;
  for (unsigned i = 0; i < nt; ++i) {
    const size_t b = i * per, e = std::min(n, b + per);
    if (b >= e) break;
    th.emplace_back([=] { memcpy(dst + b, src + b, (e - b) * 8); });
  }
  for (auto& t : th) t.join();
}

// Fault in the pages of a fresh host buffer from several threads (one write per 4 KiB page):
// the result array of a solve is 211 MB at the headline, and a single thread takes tens of
// milliseconds to touch it on some hosts -- as long as the whole 20-step solve.
extern "C" void* gq_host_alloc(int64_t bytes) {
  void* p = nullptr;
  if (bytes <= 0 || cudaMallocHost(&p, (size_t)bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

extern "C" void gq_host_free(void* p) {
  if (p && cudaFreeHost(p) != cudaSuccess) cudaGetLastError();
}

extern "C" void gq_touch_pages(void* p, int64_t bytes) {
  if (!p || bytes <= 0) return;
  char* base = static_cast<char*>(p);
  const size_t n = (size_t)bytes, page = 4096;
  {
    // ask for transparent huge pages on the 2 MiB-aligned interior (best effort: 100 faults
    // instead of 51k for a 211 MB buffer, and a TLB-friendlier host copy afterwards)
    const uintptr_t lo = (reinterpret_cast<uintptr_t>(base) + (2u << 20) - 1) & ~(uintptr_t)((2u << 20) - 1);
    const uintptr_t hi = (reinterpret_cast<uintptr_t>(base) + n) & ~(uintptr_t)((2u << 20) - 1);
    if (hi > lo) madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);
  }
  unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (n < (8u << 20)) nt = 1;
  const size_t pages = (n + page - 1) / page, per = (pages + nt - 1) / nt;
  std::vector<std::thread> th;
  for (unsigned i = 0; i < nt; ++i) {
    const size_t b = i * per, e = std::min(pages, b + per);
    if (b >= e) break;
    th.emplace_back([=] {
      for (size_t q = b; q < e; ++q) {
        volatile char* c = base + q * page;
        *c = 0;
      }
    });
  }
  for (auto& t : th) t.join();
}

static int ensure_stage(gq_ctx* c) {
  if (!c->h_stage) CK(cudaMallocHost(reinterpret_cast<void**>(&c->h_stage), c->g.dim * 8));
  for (int k = 0; k < kStageChunks; ++k)
    if (!c->ev_stage[k]) CK(cudaEventCreateWithFlags(&c->ev_stage[k], cudaEventDisableTiming));
  return GQ_OK;
}

static size_t stage_chunk_begin(const gq_ctx* c, int k) {
  return (size_t)c->g.dim * (size_t)k / kStageChunks;
}

static int export_vec(gq_ctx* c, const double* src, double* dst) {
  if (is_device_ptr(dst)) {
    CK(launch_to_reference(c->g, src, dst, c->stream));
  } else {
    CK(launch_to_reference(c->g, src, c->tmp1, c->stream));
    if (is_pageable_host(dst) && c->g.dim * 8 >= (8LL << 20)) {
      int rc = ensure_stage(c);
      if (rc) return rc;
      // chunked: the host copy of chunk k overlaps the DMA of the chunks after it
      for (int k = 0; k < kStageChunks; ++k) {
        const size_t b = stage_chunk_begin(c, k), e = stage_chunk_begin(c, k + 1);
        CK(cudaMemcpyAsync(c->h_stage + b, c->tmp1 + b, (e - b) * 8, cudaMemcpyDeviceToHost,
                           c->stream));
        CK(cudaEventRecord(c->ev_stage[k], c->stream));
      }
      for (int k = 0; k < kStageChunks; ++k) {
        const size_t b = stage_chunk_begin(c, k), e = stage_chunk_begin(c, k + 1);
        CK(cudaEventSynchronize(c->ev_stage[k]));
        parallel_copy(dst + b, c->h_stage + b, e - b);
      }
      return GQ_OK;
    }
    CK(cudaMemcpyAsync(dst, c->tmp1, c->g.dim * 8, cudaMemcpyDeviceToHost, c->stream));
  }
  CK(cudaStreamSynchronize(c->stream));
  return GQ_OK;
}

// k_rstep's TMA view of a stage-inner vector (halo = 1: the x input), cached per pointer
static const CUtensorMap* tma_view(gq_ctx* c, const double* v, int halo) {
  for (auto& m : c->maps)
    if (std::get<0>(m) == v && std::get<1>(m) == halo) return &std::get<2>(m);
  CUtensorMap m;
  if (!rstep_make_map(c->g, v, halo != 0, &m)) return nullptr;
  if (c->maps.size() >= 32) c->maps.clear();   // callers' device vectors come and go
  c->maps.emplace_back(v, halo, m);
  return &std::get<2>(c->maps.back());
}

// y = rin + Xi~ x on the tiled kernel; false if a view cannot be built (caller falls back)
static bool outer_rhs_tiled(gq_ctx* c, const double* x, const double* rin, double* y,
                            PcgState* st, cudaError_t* err) {
  if (!c->rstep) return false;
  const CUtensorMap* mx = tma_view(c, x, 1);
  if (!mx) return false;
  const CUtensorMap xm = *mx;   // the cache may move on the next lookup
  const CUtensorMap* mr = tma_view(c, rin, 0);
  if (!mr) return false;
  const CUtensorMap rm = *mr;
  const CUtensorMap* my = tma_view(c, y, 0);
  if (!my) return false;
  *err = launch_rstep(c->g, xm, rm, *my, x, rin, y, c->xi, c->xit, st, c->sm_count, c->stream);
  return true;
}

// Outer sweep s of the preconditioner, inner sweeps [l0, L) (the stage-slab phases run an
// outer sweep in pieces; enqueue_precond runs them all).
static int enqueue_outer(gq_ctx* c, int s, int l0, int l1, const double* rin, double* out,
                         PcgState* st,
                         int dotmode, std::vector<std::string>* names,
                         const std::function<int()>& mark, const double* fuse_y) {
  {
    if ((c->fast || c->chain) && s > 0 && l0 == 0) {
      // rhs_s = r + Xi~ delta_{s-1}, materialised once per outer sweep (nested_jacobi.py:119-121)
      cudaError_t te = cudaSuccess;
      if (outer_rhs_tiled(c, c->dl[(s - 1) % 2], rin, c->rs, st, &te)) {
        CK(te);
      } else if (c->grid) {
        CK(launch_grid(c->g, c->fo, kOuterRhs, c->dl[(s - 1) % 2], rin, c->rs, c->gsh,
                       c->partials, st, kDotNone, c->stream));
      } else if (c->st8) {
        CK(launch_st8(c->g, c->op, c->co.seg, c->co.nseg, kOuterRhs, c->dl[(s - 1) % 2], rin,
                      c->rs, c->sm_count, c->partials, st, kDotNone, c->stream));
      } else if (c->fast) {
        CK(launch_stencil3(c->g, c->fo, kOuterRhs, c->dl[(s - 1) % 2], rin, c->rs, c->sh_outer,
                           c->partials, st, kDotNone, c->stream));
      } else {   // chain sweeps without the fast stencils: generic Xi~ apply + add
        CK(launch_stencil(c->g, c->op, kOuter, c->dl[(s - 1) % 2], c->rs, c->sh_outer,
                          c->partials, st, kDotNone, c->stream));
        CK(launch_add(c->g, c->rs, rin, c->rs, c->vblocks, c->stream));
      }
      if (names) names->push_back("outer_rhs_s" + std::to_string(s));
      if (mark) {
        const int rc = mark();
        if (rc) return rc;
      }
    }
    for (int l = l0; l < l1; ++l) {
      const bool last = (l == c->L - 1);
      double* ob = last ? (s == c->S - 1 ? out : c->dl[s % 2]) : c->th[l % 2];
      const double* tp = l > 0 ? c->th[(l - 1) % 2] : nullptr;
      const double* dp = s > 0 ? c->dl[(s - 1) % 2] : nullptr;
      const int dm = (last && s == c->S - 1) ? dotmode : kDotNone;
      if (fuse_y != nullptr && s == 0 && l == 0) {
        // first sweep of a PCG step: r -= alpha y, max|r| and the convergence test run on
        // the staged right-hand side (the separate r-update kernel is skipped)
        CK(launch_chain_fr(c->g, c->co, const_cast<double*>(rin), fuse_y, ob, c->sm_count,
                           c->partials, st, c->stream));
      } else if (c->chain) {
        CK(launch_chain(c->g, c->co, l > 0, s > 0 ? c->rs : rin, tp, ob, rin, c->sm_count,
                        c->partials, st, dm, c->stream));
      } else if (c->fast) {
        CK(launch_sweep3(c->g, c->fo, l > 0, s > 0 ? c->rs : rin, tp, ob, rin, c->sm_count,
                         c->partials, st, dm, c->stream));
      } else {
        CK(launch_sweep(c->g, c->op, l > 0, s > 0, rin, tp, dp, ob, s > 0 ? c->sw_outer : c->sw,
                        c->partials, st, dm, c->stream));
      }
      if (names)
        names->push_back("sweep_s" + std::to_string(s) + "_l" + std::to_string(l) +
                         (!c->fast && !c->chain && s > 0 ? "_xi" : "") +
                         (fuse_y != nullptr && s == 0 && l == 0 ? "_r" : ""));
      if (mark) {
        const int rc = mark();
        if (rc) return rc;
      }
    }
  }
  return GQ_OK;
}

// S outer x L inner sweeps from zero: out = P r  (nested_jacobi.py:105-122)
static int enqueue_precond(gq_ctx* c, const double* rin, double* out, PcgState* st, int dotmode,
                           std::vector<std::string>* names,
                           const std::function<int()>& mark = nullptr,
                           const double* fuse_y = nullptr) {
  for (int s = 0; s < c->S; ++s) {
    const int rc = enqueue_outer(c, s, 0, c->L, rin, out, st, dotmode, names, mark, fuse_y);
    if (rc) return rc;
  }
  return GQ_OK;
}

// One pair-chain sweep out = Phi~^-1 (rhs + Omega~ th) (th null: out = Phi~^-1 rhs) on whichever
// sweep kernel the context selected; v1 contexts (no materialised outer rhs) take the
// outer-coupling source `xi` and add Xi~ xi to rhs on the fly (nested_jacobi.py:79-103).
static int launch_one_sweep(gq_ctx* c, const double* rhs, const double* th, const double* xi,
                            double* out) {
  const bool inner = th != nullptr;
  if (c->chain) {
    CK(launch_chain(c->g, c->co, inner, rhs, th, out, nullptr, c->sm_count, c->partials,
                    nullptr, kDotNone, c->stream));
  } else if (c->fast) {
    CK(launch_sweep3(c->g, c->fo, inner, rhs, th, out, nullptr, c->sm_count, c->partials,
                     nullptr, kDotNone, c->stream));
  } else {
    CK(launch_sweep(c->g, c->op, inner, xi != nullptr, rhs, th, xi, out,
                    xi != nullptr ? c->sw_outer : c->sw, c->partials, nullptr, kDotNone,
                    c->stream));
  }
  return GQ_OK;
}

// Standalone nested block Jacobi iteration (nested_jacobi.py:124-151, nbjm_solve :155-159).
// Outer sweep s = 0 runs L inner sweeps from zero on the right-hand side; every later outer
// sweep runs L inner sweeps on rhs + Xi~ delta warm-started from delta (so its fixed point
// solves Delta x = rhs), until max |new - prev| < tol.  Any inner budget >= 1 (odd allowed).
// The test is read back once per outer sweep.  GQ_MAX_ITER leaves the last iterate in x_out.
extern "C" int gq_nbjm_solve(gq_ctx* c, const double* rhs, double tol, int64_t max_outer,
                             double* x_out, int64_t* outers) {
  if (!c || !rhs || !x_out || !outers) return fail(GQ_INVALID_ARG, "null argument");
  if (max_outer < 1) return fail(GQ_INVALID_ARG, "need at least one outer sweep");
  c->started = false;   // the PCG work vectors are reused below
  int rc = import_vec(c, rhs, c->r);
  if (rc) return rc;
  double* delta = c->d;
  double* fresh = c->q;
  double* res = reinterpret_cast<double*>(c->st);   // scratch: mu slot of the PCG state
  unsigned int* counter = &c->st->counter[3];
  double h = 0.0;
  for (int64_t s = 0; s < max_outer; ++s) {
    const double* rhs_s = c->r;
    const double* xi = nullptr;
    if (s > 0) {
      cudaError_t te = cudaSuccess;
      if (outer_rhs_tiled(c, delta, c->r, c->rs, nullptr, &te)) {
        CK(te);
        rhs_s = c->rs;
      } else if (c->grid) {
        CK(launch_grid(c->g, c->fo, kOuterRhs, delta, c->r, c->rs, c->gsh, c->partials,
                       nullptr, kDotNone, c->stream));
        rhs_s = c->rs;
      } else if (c->st8) {
        CK(launch_st8(c->g, c->op, c->co.seg, c->co.nseg, kOuterRhs, delta, c->r, c->rs,
                      c->sm_count, c->partials, nullptr, kDotNone, c->stream));
        rhs_s = c->rs;
      } else if (c->fast) {
        CK(launch_stencil3(c->g, c->fo, kOuterRhs, delta, c->r, c->rs, c->sh_outer,
                           c->partials, nullptr, kDotNone, c->stream));
        rhs_s = c->rs;
      } else if (c->chain) {
        CK(launch_stencil(c->g, c->op, kOuter, delta, c->rs, c->sh_outer, c->partials, nullptr,
                          kDotNone, c->stream));
        CK(launch_add(c->g, c->rs, c->r, c->rs, c->vblocks, c->stream));
        rhs_s = c->rs;
      } else {
        xi = delta;   // v1 sweeps add Xi~ delta on the fly
      }
    }
    // theta_0 = delta (warm start) for s > 0; from zero at s = 0
    const double* th = s > 0 ? delta : nullptr;
    for (int l = 0; l < c->L; ++l) {
      double* ob = (l == c->L - 1) ? fresh : c->th[l % 2];
      rc = launch_one_sweep(c, rhs_s, th, xi, ob);
      if (rc) return rc;
      th = ob;
    }
    CK(launch_maxdiff(c->g, fresh, s > 0 ? delta : nullptr, c->vblocks, c->partials, counter,
                      res, c->stream));
    CK(cudaMemcpyAsync(&h, res, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    std::swap(delta, fresh);   // delta = new
    if (h < tol) {              // nested_jacobi.py:145-146 (NaN compares false: keeps going)
      *outers = s + 1;
      return export_vec(c, delta, x_out);
    }
  }
  *outers = max_outer;
  rc = export_vec(c, delta, x_out);
  if (rc) return rc;
  return fail(GQ_MAX_ITER, "nested Jacobi did not converge within " + std::to_string(max_outer) +
                               " outer sweeps");
}

extern "C" int gq_apply_delta(gq_ctx* c, const double* x, double* y) {
  if (!c || !x || !y) return fail(GQ_INVALID_ARG, "null argument");
  int rc = import_vec(c, x, c->tmp0);
  if (rc) return rc;
  if (c->dstep)
    CK(launch_dstep(c->g, c->map_tmp0, c->map_y, c->dso, c->y, c->partials, nullptr, kDotNone,
                    c->sm_count, c->stream));
  else if (c->st8)
    CK(launch_st8(c->g, c->op, c->co.seg, c->co.nseg, kDelta, c->tmp0, nullptr, c->y,
                  c->sm_count, c->partials, nullptr, kDotNone, c->stream));
  else if (c->grid)
    CK(launch_grid(c->g, c->fo, kDelta, c->tmp0, nullptr, c->y, c->gsh, c->partials, nullptr,
                   kDotNone, c->stream));
  else if (c->fast)
    CK(launch_stencil3(c->g, c->fo, kDelta, c->tmp0, nullptr, c->y, c->sh_delta, c->partials,
                       nullptr, kDotNone, c->stream));
  else
    CK(launch_stencil(c->g, c->op, kDelta, c->tmp0, c->y, c->sh_delta, c->partials, nullptr,
                      kDotNone, c->stream));
  return export_vec(c, c->y, y);
}

extern "C" int gq_apply_outer_coupling(gq_ctx* c, const double* x, double* y) {
  if (!c || !x || !y) return fail(GQ_INVALID_ARG, "null argument");
  int rc = import_vec(c, x, c->tmp0);
  if (rc) return rc;
  // the kernel the preconditioner runs (rhs = 0 + Xi~ x) where one is selected
  cudaError_t te = cudaSuccess;
  if (c->rstep || c->grid) CK(cudaMemsetAsync(c->tmp1, 0, c->g.span * 8, c->stream));
  if (outer_rhs_tiled(c, c->tmp0, c->tmp1, c->y, nullptr, &te)) {
    CK(te);
  } else if (c->grid) {
    CK(launch_grid(c->g, c->fo, kOuterRhs, c->tmp0, c->tmp1, c->y, c->gsh, c->partials,
                   nullptr, kDotNone, c->stream));
  } else {
    CK(launch_stencil(c->g, c->op, kOuter, c->tmp0, c->y, c->sh_outer, c->partials, nullptr,
                      kDotNone, c->stream));
  }
  return export_vec(c, c->y, y);
}

extern "C" int gq_apply_inner_coupling(gq_ctx* c, const double* x, double* y) {
  if (!c || !x || !y) return fail(GQ_INVALID_ARG, "null argument");
  int rc = import_vec(c, x, c->tmp0);
  if (rc) return rc;
  CK(launch_stencil(c->g, c->op, kInner, c->tmp0, c->y, c->sh_inner, c->partials, nullptr,
                    kDotNone, c->stream));
  return export_vec(c, c->y, y);
}

extern "C" int gq_pair_solve(gq_ctx* c, const double* rhs, double* out) {
  if (!c || !rhs || !out) return fail(GQ_INVALID_ARG, "null argument");
  int rc = import_vec(c, rhs, c->tmp0);
  if (rc) return rc;
  // the sweep kernel the preconditioner runs (DMMA chains / lane-per-stage / generic)
  rc = launch_one_sweep(c, c->tmp0, nullptr, nullptr, c->y);
  if (rc) return rc;
  return export_vec(c, c->y, out);
}

extern "C" int gq_apply_precond(gq_ctx* c, const double* r, double* q) {
  if (!c || !r || !q) return fail(GQ_INVALID_ARG, "null argument");
  if (c->L % 2)
    return fail(GQ_INVALID_ARG, "preconditioner use requires an even inner budget (got " +
                                    std::to_string(c->L) + "); odd budgets are standalone-only");
  int rc = import_vec(c, r, c->tmp0);
  if (rc) return rc;
  rc = enqueue_precond(c, c->tmp0, c->y, nullptr, kDotNone, nullptr);
  if (rc) return rc;
  return export_vec(c, c->y, q);
}

// ---- PCG ----------------------------------------------------------------------------------

// y = Delta d with the curvature y.d and alpha (first kernel of a PCG step, pcg.py:99-108)
static int enqueue_delta_step(gq_ctx* c) {
  if (c->dstep)
    CK(launch_dstep(c->g, c->map_d, c->map_y, c->dso, c->y, c->partials, c->st, kDotStep, c->sm_count,
                    c->stream));
  else if (c->st8)
    CK(launch_st8(c->g, c->op, c->co.seg, c->co.nseg, kDelta, c->d, nullptr, c->y, c->sm_count,
                  c->partials, c->st, kDotStep, c->stream));
  else if (c->grid)
    CK(launch_grid(c->g, c->fo, kDelta, c->d, nullptr, c->y, c->gsh, c->partials, c->st,
                   kDotStep, c->stream));
  else if (c->fast)
    CK(launch_stencil3(c->g, c->fo, kDelta, c->d, nullptr, c->y, c->sh_delta, c->partials, c->st,
                       kDotStep, c->stream));
  else
    CK(launch_stencil(c->g, c->op, kDelta, c->d, c->y, c->sh_delta, c->partials, c->st,
                      kDotStep, c->stream));
  return GQ_OK;
}

static int enqueue_step(gq_ctx* c, int use_precond, std::vector<std::string>* names,
                        std::vector<cudaEvent_t>* evs) {
  size_t ei = 0;
  auto mark = [&]() -> int {
    if (evs) CK(cudaEventRecord((*evs)[ei++], c->stream));
    return GQ_OK;
  };
  int rc = mark();
  if (rc) return rc;
  if ((rc = enqueue_delta_step(c))) return rc;
  if (names) names->push_back("delta");
  if ((rc = mark())) return rc;
  // x += alpha d only feeds the result.  By default it is a separate kernel on a parallel
  // branch of the step graph (joined before d is overwritten), or in line when GQ_NO_FORK=1
  // or when the step is profiled.  GQ_FUSE_X=1 fuses it into the direction update at the
  // end of the step (one pass over q, d, x).
  static const bool no_fork = [] {
    const char* e = getenv("GQ_NO_FORK");
    return e && *e == '1';
  }();
  const bool fuse_x = c->fuse_x;
  const bool fork = !fuse_x && evs == nullptr && !no_fork;
  if (fuse_x) {
    // nothing here: k_dirupdate_x below
  } else if (fork) {
    CK(cudaEventRecord(c->ev_fork, c->stream));
    CK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    CK(launch_update_x(c->g, c->x, c->d, c->vblocks, c->st, c->side));
    CK(cudaEventRecord(c->ev_join, c->side));
  } else {
    CK(launch_update_x(c->g, c->x, c->d, c->vblocks, c->st, c->stream));
    if (names) names->push_back("update_x");
    if ((rc = mark())) return rc;
  }
  const bool fuse_r = use_precond && c->fuse_r;
  if (!fuse_r) {
    CK(launch_update_r(c->g, c->r, c->y, c->vblocks, c->partials, c->st, c->stream));
    if (names) names->push_back("update");
    if ((rc = mark())) return rc;
  }
  const double* qv = c->q;
  if (use_precond) {
    rc = enqueue_precond(c, c->r, c->q, c->st, kDotStep, names,
                         evs ? std::function<int()>(mark) : std::function<int()>(),
                         fuse_r ? c->y : nullptr);
    if (rc) return rc;
  } else {
    CK(launch_dot(c->g, c->r, c->r, c->vblocks, c->partials, c->st, kDotStep, c->stream));
    if (names) names->push_back("dot");
    if ((rc = mark())) return rc;
    qv = c->r;
  }
  if (fork) CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  if (fuse_x) {
    CK(launch_dirupdate_x(c->g, c->d, qv, c->x, c->vblocks, c->st, c->stream));
    if (names) names->push_back("dirupdate_x");
  } else {
    CK(launch_dirupdate(c->g, c->d, qv, c->vblocks, c->st, c->stream));
    if (names) names->push_back("dirupdate");
  }
  return mark();
}

extern "C" int gq_launches_per_step(gq_ctx* c) {
  if (!c) return -1;
  const int vec = c->fuse_x ? 3 : 4;   // delta, r update, direction update (+ x update)
  if (!c->use_precond) return vec + 1;
  return vec - (c->fuse_r ? 1 : 0) + c->S * c->L + (c->fast || c->chain ? c->S - 1 : 0);
}

extern "C" int gq_pcg_start(gq_ctx* c, const double* rhs, const double* x0, int32_t use_precond) {
  if (!c || !rhs) return fail(GQ_INVALID_ARG, "null argument");
  if (use_precond && (c->L % 2))
    return fail(GQ_INVALID_ARG, "preconditioner use requires an even inner budget (got " +
                                    std::to_string(c->L) + "); odd budgets are standalone-only");
  c->use_precond = use_precond ? 1 : 0;
  c->started = false;
  memset(c->h_st, 0, sizeof(PcgState));
  c->h_st->hist = c->hist;
  c->h_st->max_steps = 1;
  CK(cudaMemcpyAsync(c->st, c->h_st, sizeof(PcgState), cudaMemcpyHostToDevice, c->stream));
  int rc = import_vec(c, rhs, c->r);
  if (rc) return rc;
  // ValueError for a non-finite rhs (pcg.py:65-66), checked on the device
  CK(launch_nonfinite(c->g, c->r, c->vblocks, c->st, c->stream));
  CK(cudaMemcpyAsync(c->h_st, c->st, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (c->h_st->nonfinite)
    return fail(GQ_INVALID_ARG, "right-hand side contains non-finite entries");
  if (x0) {
    // r = rhs - Delta x0  (pcg.py:82-85)
    rc = import_vec(c, x0, c->x);
    if (rc) return rc;
    CK(launch_stencil(c->g, c->op, kDelta, c->x, c->y, c->sh_delta, c->partials, nullptr,
                      kDotNone, c->stream));
    CK(launch_sub(c->g, c->tmp0, c->r, c->y, c->vblocks, c->stream));
    CK(cudaMemcpyAsync(c->r, c->tmp0, c->g.span * 8, cudaMemcpyDeviceToDevice, c->stream));
  } else {
    CK(cudaMemsetAsync(c->x, 0, c->g.span * 8, c->stream));
  }
  if (use_precond) {
    // d = P r ; mu = d.r   (pcg.py:87-93)
    rc = enqueue_precond(c, c->r, c->q, c->st, kDotInit, nullptr);
    if (rc) return rc;
    CK(cudaMemcpyAsync(c->d, c->q, c->g.span * 8, cudaMemcpyDeviceToDevice, c->stream));
  } else {
    CK(cudaMemcpyAsync(c->d, c->r, c->g.span * 8, cudaMemcpyDeviceToDevice, c->stream));
    CK(launch_dot(c->g, c->d, c->r, c->vblocks, c->partials, c->st, kDotInit, c->stream));
  }
  CK(cudaStreamSynchronize(c->stream));
  c->started = true;
  return GQ_OK;
}

static int ensure_hist(gq_ctx* c, long long cap) {
  if (cap <= c->hist_cap) return GQ_OK;
  long long ncap = std::max(cap, std::max(64LL, c->hist_cap * 2));
  double* nh = nullptr;
  CK(dalloc(&nh, (size_t)ncap));
  if (c->hist) {
    CK(cudaMemcpyAsync(nh, c->hist, c->hist_cap * 8, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(c->hist);
  }
  c->hist = nh;
  c->hist_cap = ncap;
  return GQ_OK;
}

static int ensure_graph(gq_ctx* c) {
  const int k = c->use_precond;
  if (c->gexec[k]) return GQ_OK;
  cudaGraph_t graph;
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  int rc = enqueue_step(c, k, nullptr, nullptr);
  cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
  if (rc) return rc;
  if (e != cudaSuccess) return fail(GQ_CUDA_ERROR, std::string("capture: ") + cudaGetErrorString(e));
  e = cudaGraphInstantiate(&c->gexec[k], graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return fail(GQ_CUDA_ERROR, std::string("instantiate: ") + cudaGetErrorString(e));
  return GQ_OK;
}

extern "C" int gq_pcg_run(gq_ctx* c, double tol, int64_t max_steps, int64_t* steps_done,
                          int32_t* converged) {
  if (!c) return fail(GQ_INVALID_ARG, "null context");
  if (!c->started) return fail(GQ_INVALID_ARG, "gq_pcg_start has not been called");
  if (!(tol > 0)) return fail(GQ_INVALID_ARG, "tolerance must be positive");
  if (max_steps < 1) return fail(GQ_INVALID_ARG, "need at least one step");
  CK(cudaMemcpyAsync(c->h_st, c->st, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  PcgState& h = *c->h_st;
  if (!h.converged && !h.breakdown && h.step < max_steps) {
    // the history grows with the steps actually launched (not with max_steps, whose
    // reference default dim + 50 would reserve O(dim) doubles): each chunk of graph launches
    // first makes room for its own steps
    int rc = ensure_hist(c, std::min<long long>(max_steps, h.step + 2));
    if (rc) return rc;
    h.hist = c->hist;
    h.tol = tol;
    h.max_steps = max_steps;
    h.done = 0;
    CK(cudaMemcpyAsync(c->st, c->h_st, sizeof(PcgState), cudaMemcpyHostToDevice, c->stream));
    rc = ensure_graph(c);
    if (rc) return rc;
    long long chunk = 2;
    while (true) {
      const long long todo = std::min<long long>(chunk, max_steps - h.step);
      if (h.step + todo > c->hist_cap) {
        // the state is quiescent here (read back above): move the history, repoint the state
        rc = ensure_hist(c, h.step + todo);
        if (rc) return rc;
        h.hist = c->hist;
        CK(cudaMemcpyAsync(&c->st->hist, &c->hist, sizeof(double*), cudaMemcpyHostToDevice,
                           c->stream));
      }
      for (long long i = 0; i < todo; ++i) CK(cudaGraphLaunch(c->gexec[c->use_precond], c->stream));
      CK(cudaMemcpyAsync(c->h_st, c->st, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      if (h.done || h.step >= max_steps) break;
      chunk = std::min<long long>(chunk * 2, 64);
    }
  }
  if (steps_done) *steps_done = h.step;
  if (converged) *converged = h.converged;
  if (h.breakdown)
    return fail(GQ_BREAKDOWN, "non-positive curvature " + std::to_string(h.curv) +
                                  "; operator or preconditioner is not positive definite");
  if (h.converged) return GQ_OK;
  return fail(GQ_MAX_ITER, "conjugate gradient did not reach the tolerance within " +
                               std::to_string(h.step) + " steps");
}

extern "C" int gq_pcg_read(gq_ctx* c, int32_t which, double* out) {
  if (!c || !out) return fail(GQ_INVALID_ARG, "null argument");
  if (!c->started) return fail(GQ_INVALID_ARG, "gq_pcg_start has not been called");
  const double* src = which == GQ_VEC_R ? c->r : c->x;
  return export_vec(c, src, out);
}

extern "C" int gq_pcg_history(gq_ctx* c, double* out, int64_t count) {
  if (!c || (!out && count > 0)) return fail(GQ_INVALID_ARG, "null argument");
  if (count <= 0) return GQ_OK;
  if (count > c->hist_cap) return fail(GQ_INVALID_ARG, "history request exceeds recorded steps");
  CK(cudaMemcpyAsync(out, c->hist, count * 8, cudaMemcpyDefault, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return GQ_OK;
}

extern "C" int gq_pcg_scalars(gq_ctx* c, double* mu, double* curv, double* alpha, double* beta) {
  if (!c) return fail(GQ_INVALID_ARG, "null context");
  CK(cudaMemcpyAsync(c->h_st, c->st, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (mu) *mu = c->h_st->mu;
  if (curv) *curv = c->h_st->curv;
  if (alpha) *alpha = c->h_st->alpha;
  if (beta) *beta = c->h_st->beta;
  return GQ_OK;
}

// ---- stage-slab mode (driven by slab.py) ------------------------
// The context holds a stage window of the global problem.  A PCG step is split into phases
// at the points where the slabs must agree: the host exchanges halo stages (d before Delta,
// delta^s between outer sweeps) and reduces the partial scalars (curvature, max|r|, q.r)
// between phases; each phase starts with the kernel that turns the reduced value into the
// global decision (gq_slab.cu).  Phases are enqueued on the context stream without a sync.

extern "C" int gq_slab_enable(gq_ctx* c, int32_t own_lo, int32_t own_hi) {
  if (!c) return fail(GQ_INVALID_ARG, "null context");
  const int T1 = c->g.T1;
  if (own_lo < 0 || own_lo > 1 || own_hi <= own_lo || own_hi > T1 || own_hi < T1 - 1)
    return fail(GQ_INVALID_ARG, "slab window: owned stages must be the window minus at most one "
                                "halo stage per side");
  c->slab = true;
  c->slab_t0 = own_lo > 0 ? 0 : -1;
  c->slab_t1 = own_hi < T1 ? T1 - 1 : -1;
  // Delta leaves the halo rows of y unwritten (zero from gq_slab_start on), so y.d, r,
  // max|r| and q.r cover the owned stages only
  c->g.hx0 = c->slab_t0;
  c->g.hx1 = c->slab_t1;
  c->fuse_x = false;
  for (auto& ge : c->gexec)
    if (ge) {
      cudaGraphExecDestroy(ge);
      ge = nullptr;
    }
  c->started = false;
  return GQ_OK;
}

extern "C" int gq_slab_start(gq_ctx* c, const double* r0, const double* x0, int32_t use_precond,
                             double tol, int64_t max_steps) {
  if (!c || !r0) return fail(GQ_INVALID_ARG, "null argument");
  if (!c->slab) return fail(GQ_INVALID_ARG, "gq_slab_enable has not been called");
  if (use_precond && (c->L % 2))
    return fail(GQ_INVALID_ARG, "preconditioner use requires an even inner budget (got " +
                                    std::to_string(c->L) + "); odd budgets are standalone-only");
  if (!(tol > 0)) return fail(GQ_INVALID_ARG, "tolerance must be positive");
  if (max_steps < 1) return fail(GQ_INVALID_ARG, "need at least one step");
  int rc = ensure_hist(c, max_steps);
  if (rc) return rc;
  c->use_precond = use_precond ? 1 : 0;
  memset(c->h_st, 0, sizeof(PcgState));
  c->h_st->hist = c->hist;
  c->h_st->tol = tol;
  c->h_st->max_steps = max_steps;
  c->h_st->defer = 1;   // convergence is decided on the global max|r| (DIRECTION phase)
  CK(cudaMemcpyAsync(c->st, c->h_st, sizeof(PcgState), cudaMemcpyHostToDevice, c->stream));
  // r0 is the slab's initial residual (rhs, or rhs - Delta x0 formed by the caller), zero on
  // the halo stages; x0 only seeds the iterate
  if ((rc = import_vec(c, r0, c->r))) return rc;
  for (int t : {c->slab_t0, c->slab_t1})
    if (t >= 0) CK(launch_stage_zero(c->g, t, c->y, c->sm_count, c->stream));
  if (x0) {
    if ((rc = import_vec(c, x0, c->x))) return rc;
  } else {
    CK(cudaMemsetAsync(c->x, 0, c->g.span * 8, c->stream));
  }
  c->started = true;
  return GQ_OK;
}

extern "C" int gq_slab_phase(gq_ctx* c, int32_t kind, int32_t s) {
  if (!c || !c->slab || !c->started) return fail(GQ_INVALID_ARG, "slab solve not started");
  const bool pc = c->use_precond != 0;
  const bool fr = pc && c->fuse_r;
  const std::function<int()> none;
  int rc = GQ_OK;
  switch (kind) {
    case GQ_SLAB_INIT_OUTER:   // d = P r, mu = d.r (pcg.py:87-93), outer sweep s
      if (pc) {
        if (s < 0 || s >= c->S) return fail(GQ_INVALID_ARG, "outer sweep index out of range");
        rc = enqueue_outer(c, s, 0, c->L, c->r, c->q, c->st, kDotInit, nullptr, none, nullptr);
      } else {
        CK(cudaMemcpyAsync(c->d, c->r, c->g.span * 8, cudaMemcpyDeviceToDevice, c->stream));
        CK(launch_dot(c->g, c->d, c->r, c->vblocks, c->partials, c->st, kDotInit, c->stream));
      }
      break;
    case GQ_SLAB_INIT_FINISH:
      if (pc) CK(cudaMemcpyAsync(c->d, c->q, c->g.span * 8, cudaMemcpyDeviceToDevice, c->stream));
      break;
    case GQ_SLAB_DELTA:        // y = Delta d, partial y.d over the owned stages
      if ((rc = enqueue_delta_step(c))) return rc;
      break;
    case GQ_SLAB_UPDATE:       // alpha; x += alpha d; r -= alpha y with the partial max|r|
      CK(launch_slab_scalar(0, c->st, c->stream));
      // x += alpha d on the side stream, joined before d is overwritten (DIRECTION), as in
      // the one-context step graph
      CK(cudaEventRecord(c->ev_fork, c->stream));
      CK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
      CK(launch_update_x(c->g, c->x, c->d, c->vblocks, c->st, c->side));
      CK(cudaEventRecord(c->ev_join, c->side));
      if (fr)
        rc = enqueue_outer(c, 0, 0, 1, c->r, c->q, c->st, kDotStep, nullptr, none, c->y);
      else
        CK(launch_update_r(c->g, c->r, c->y, c->vblocks, c->partials, c->st, c->stream));
      break;
    case GQ_SLAB_OUTER: {      // outer sweep s of q = P r (+ partial q.r in the last one)
      const int S = pc ? c->S : 1;
      if (s < 0 || s >= S) return fail(GQ_INVALID_ARG, "outer sweep index out of range");
      if (s == S - 1) CK(launch_slab_scalar(2, c->st, c->stream));
      if (pc)
        rc = enqueue_outer(c, s, (s == 0 && fr) ? 1 : 0, c->L, c->r, c->q, c->st, kDotStep,
                           nullptr, none, nullptr);
      else
        CK(launch_dot(c->g, c->r, c->r, c->vblocks, c->partials, c->st, kDotStep, c->stream));
      break;
    }
    case GQ_SLAB_DIRECTION:    // convergence test and beta; d = q + beta d
      CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
      CK(launch_slab_scalar(3, c->st, c->stream));
      CK(launch_dirupdate(c->g, c->d, pc ? c->q : c->r, c->vblocks, c->st, c->stream));
      break;
    default:
      return fail(GQ_INVALID_ARG, "unknown slab phase");
  }
  return rc;
}

static double* slab_vec(gq_ctx* c, int which) {
  return which == GQ_SLAB_VEC_D ? c->d : which == GQ_SLAB_VEC_DL0 ? c->dl[0]
       : which == GQ_SLAB_VEC_DL1 ? c->dl[1] : nullptr;
}

extern "C" int gq_slab_pack(gq_ctx* c, int32_t which, int32_t t, double* buf) {
  if (!c || !buf) return fail(GQ_INVALID_ARG, "null argument");
  double* v = slab_vec(c, which);
  if (!v || t < 0 || t >= c->g.T1) return fail(GQ_INVALID_ARG, "bad halo vector or stage");
  CK(launch_stage_pack(c->g, t, v, buf, c->sm_count, c->stream));
  return GQ_OK;
}

extern "C" int gq_slab_unpack(gq_ctx* c, int32_t which, int32_t t, const double* buf) {
  if (!c || !buf) return fail(GQ_INVALID_ARG, "null argument");
  double* v = slab_vec(c, which);
  if (!v || t < 0 || t >= c->g.T1) return fail(GQ_INVALID_ARG, "bad halo vector or stage");
  CK(launch_stage_unpack(c->g, t, buf, v, c->sm_count, c->stream));
  return GQ_OK;
}

extern "C" void* gq_slab_scalar_ptr(gq_ctx* c, int32_t which) {
  if (!c || !c->st) return nullptr;
  switch (which) {
    case GQ_SLAB_CURV: return &c->st->curv;
    case GQ_SLAB_RES: return &c->st->res;
    case GQ_SLAB_MU: return &c->st->mu;
    default: return nullptr;
  }
}

extern "C" int gq_slab_status(gq_ctx* c, int64_t* step, int32_t* done, int32_t* converged,
                              int32_t* breakdown) {
  if (!c) return fail(GQ_INVALID_ARG, "null context");
  CK(cudaMemcpyAsync(c->h_st, c->st, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (step) *step = c->h_st->step;
  if (done) *done = c->h_st->done;
  if (converged) *converged = c->h_st->converged;
  if (breakdown) *breakdown = c->h_st->breakdown;
  return GQ_OK;
}

extern "C" int gq_pcg(gq_ctx* c, const double* rhs, const double* x0, double tol,
                      int64_t max_steps, int32_t use_precond, double* x_out, double* hist_out,
                      int64_t hist_capacity, int64_t* steps, int32_t* converged) {
  int rc = gq_pcg_start(c, rhs, x0, use_precond);
  if (rc) return rc;
  int64_t s = 0;
  int32_t conv = 0;
  const int status = gq_pcg_run(c, tol, max_steps, &s, &conv);
  if (status != GQ_OK && status != GQ_MAX_ITER && status != GQ_BREAKDOWN) return status;
  const std::string msg = g_err;
  if (x_out && (rc = gq_pcg_read(c, GQ_VEC_X, x_out))) return rc;
  if (hist_out && (rc = gq_pcg_history(c, hist_out, std::min<int64_t>(s, hist_capacity))))
    return rc;
  if (steps) *steps = s;
  if (converged) *converged = conv;
  g_err = msg;
  return status;
}

extern "C" int gq_profile_steps(gq_ctx* c, int32_t steps, float* ms_out, int32_t count) {
  if (!c || !c->started) return fail(GQ_INVALID_ARG, "gq_pcg_start has not been called");
  const int nk = gq_launches_per_step(c);
  // extend the step budget so the profiled steps really run
  CK(cudaMemcpyAsync(c->h_st, c->st, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (c->h_st->converged || c->h_st->breakdown)
    return fail(GQ_INVALID_ARG, "solve already finished; restart with gq_pcg_start");
  c->h_st->max_steps = c->h_st->step + steps;
  c->h_st->done = 0;
  {
    int rc0 = ensure_hist(c, c->h_st->max_steps);
    if (rc0) return rc0;
  }
  c->h_st->hist = c->hist;
  CK(cudaMemcpyAsync(c->st, c->h_st, sizeof(PcgState), cudaMemcpyHostToDevice, c->stream));
  std::vector<cudaEvent_t> ev(nk + 1);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  std::vector<double> acc(nk, 0.0);
  c->knames.clear();
  int rc = GQ_OK;
  for (int s = 0; s < steps && rc == GQ_OK; ++s) {
    std::vector<std::string> names;
    rc = enqueue_step(c, c->use_precond, &names, &ev);
    if (rc) break;
    cudaError_t e = cudaEventSynchronize(ev[nk]);
    if (e != cudaSuccess) {
      rc = fail(GQ_CUDA_ERROR, cudaGetErrorString(e));
      break;
    }
    for (int i = 0; i < nk; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      acc[i] += ms;
    }
    c->knames = names;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  if (rc) return rc;
  for (int i = 0; i < nk && i < count; ++i) ms_out[i] = (float)acc[i];
  return nk;
}

// ---- primal recovery and KKT residuals (recovery.py:50-80) -------------------------------
namespace {
// device view of a user vector (host or device pointer); owns a temporary when needed
struct DevVec {
  double* p = nullptr;
  double* tmp = nullptr;
  ~DevVec() {
    if (tmp) cudaFree(tmp);
  }
};
int dev_in(gq_ctx* c, const double* src, size_t n, DevVec& v) {
  if (is_device_ptr(src)) {
    v.p = const_cast<double*>(src);
    return GQ_OK;
  }
  CK(cudaMalloc(&v.tmp, std::max<size_t>(n, 1) * 8));
  if (n) CK(cudaMemcpyAsync(v.tmp, src, n * 8, cudaMemcpyHostToDevice, c->stream));
  v.p = v.tmp;
  return GQ_OK;
}
int dev_out(gq_ctx* c, double* dst, size_t n, DevVec& v) {
  if (is_device_ptr(dst)) {
    v.p = dst;
    return GQ_OK;
  }
  CK(cudaMalloc(&v.tmp, std::max<size_t>(n, 1) * 8));
  v.p = v.tmp;
  return GQ_OK;
}
int dev_back(gq_ctx* c, double* dst, size_t n, const DevVec& v) {
  if (v.tmp && n) CK(cudaMemcpyAsync(dst, v.tmp, n * 8, cudaMemcpyDeviceToHost, c->stream));
  return GQ_OK;
}
}  // namespace

extern "C" int64_t gq_input_dim(const gq_ctx* c) {
  return c ? (int64_t)c->g.T * c->g.nk * c->m : -1;
}

extern "C" int gq_recover(gq_ctx* c, const double* lam, double* x_out, double* u_out,
                          double* objective) {
  if (!c || !lam || !x_out || !u_out) return fail(GQ_INVALID_ARG, "null argument");
  const size_t nx = (size_t)c->g.dim, nu = (size_t)c->g.T * c->g.nk * c->m;
  DevVec L, X, U;
  int rc;
  if ((rc = dev_in(c, lam, nx, L)) || (rc = dev_out(c, x_out, nx, X)) || (rc = dev_out(c, u_out, nu, U)))
    return rc;
  const int nbk = recover_blocks(c->g);
  double* part = nullptr;
  CK(cudaMalloc(&part, (size_t)nbk * 8));
  cudaError_t e = launch_recover(c->g, c->m, c->A, c->C, c->qinv, c->B, c->R, c->rinv, c->Q,
                                 c->dcls, c->ccls, 0, L.p, nullptr, nullptr, nullptr, X.p, U.p,
                                 part, c->stream);
  std::vector<double> hp(nbk);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(hp.data(), part, (size_t)nbk * 8, cudaMemcpyDeviceToHost, c->stream);
  if ((rc = dev_back(c, x_out, nx, X)) || (rc = dev_back(c, u_out, nu, U))) {
    cudaFree(part);
    return rc;
  }
  cudaError_t e2 = cudaStreamSynchronize(c->stream);
  cudaFree(part);
  if (e != cudaSuccess || e2 != cudaSuccess)
    return fail(GQ_CUDA_ERROR, std::string("gq_recover: ") +
                                   cudaGetErrorString(e != cudaSuccess ? e : e2));
  double obj = 0.0;
  for (double v : hp) obj += v;   // fixed block order: reproducible
  if (objective) *objective = 0.5 * obj;
  return GQ_OK;
}

extern "C" int gq_kkt_residual(gq_ctx* c, const double* lam, const double* x, const double* u,
                               const double* offset, double* res3) {
  if (!c || !lam || !x || !u || !offset || !res3) return fail(GQ_INVALID_ARG, "null argument");
  const size_t nx = (size_t)c->g.dim, nu = (size_t)c->g.T * c->g.nk * c->m;
  DevVec L, X, U, O;
  int rc;
  if ((rc = dev_in(c, lam, nx, L)) || (rc = dev_in(c, x, nx, X)) || (rc = dev_in(c, u, nu, U)) ||
      (rc = dev_in(c, offset, nx, O)))
    return rc;
  const int nbk = recover_blocks(c->g);
  double* part = nullptr;
  CK(cudaMalloc(&part, (size_t)nbk * 3 * 8));
  cudaError_t e = launch_recover(c->g, c->m, c->A, c->C, c->qinv, c->B, c->R, c->rinv, c->Q,
                                 c->dcls, c->ccls, 1, L.p, X.p, U.p, O.p, nullptr, nullptr, part,
                                 c->stream);
  std::vector<double> hp((size_t)nbk * 3);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(hp.data(), part, (size_t)nbk * 3 * 8, cudaMemcpyDeviceToHost, c->stream);
  cudaError_t e2 = cudaStreamSynchronize(c->stream);
  cudaFree(part);
  if (e != cudaSuccess || e2 != cudaSuccess)
    return fail(GQ_CUDA_ERROR, std::string("gq_kkt_residual: ") +
                                   cudaGetErrorString(e != cudaSuccess ? e : e2));
  res3[0] = res3[1] = res3[2] = 0.0;
  for (int b = 0; b < nbk; ++b)
    for (int k = 0; k < 3; ++k) {
      const double v = hp[3 * b + k];
      if (v != v || v > res3[k]) res3[k] = v;   // NaN propagates (np.max semantics)
    }
  return GQ_OK;
}

extern "C" const char* gq_kernel_name(gq_ctx* c, int32_t i) {
  if (!c || i < 0 || i >= (int)c->knames.size()) return "";
  return c->knames[i].c_str();
}
