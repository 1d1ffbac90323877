// C-ABI of libls.so (include/ls_api.h): context setup, fd_apply, ls_matvec,
// ls_rhs, pcg_solve.  All arithmetic of the hot path runs in the kernels of
// fd_kernels.cuh / matvec_kernels.cuh / pcg_kernels.cuh; this file is glue.
#include "ls_api.h"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <vector>

#include "comm.hpp"
#include "plan.hpp"
#include "fd_kernels.cuh"
#include "fd_rd_launch.cuh"
#include "fd_time_kernel.cuh"
#include "ft.hpp"
#include "fd_plane_kernel.cuh"
#include "pl.hpp"
#include "matvec_kernels.cuh"
#include "matvec2_kernels.cuh"
#include "matvec3_kernels.cuh"
#include "mv4_kernels.cuh"
#include "mv5_kernels.cuh"
#include "matvec6_kernels.cuh"
#include "pcg_kernels.cuh"
#include "setup_host.hpp"
#include "geo.hpp"
#include "err.hpp"

using namespace ls;
namespace ls {
extern int g_mv4_ctas;  // mv4.cu
}

int ls::g_ls_pdl = 1;  // programmatic dependent launch of the FD mode kernels (LS_TUNE_PDL)
int ls::g_rd_tail = 0;    // DFMA tail rows in the split FD kernels (LS_TUNE_FD_TAIL = 2, RDCfg::TR; measured slower, off)
int ls::g_rd_staged = 0;  // staged split FD kernel (LS_TUNE_FD_STAGED; measured slower except p = 8, off)

#define LS_CUDA(x)                                                                        \
  do {                                                                                    \
    cudaError_t err_ = (x);                                                               \
    if (err_ != cudaSuccess) {                                                            \
      std::fprintf(stderr, "[libls] CUDA error %s at %s:%d\n", cudaGetErrorString(err_), \
                   __FILE__, __LINE__);                                                   \
      return LS_ECUDA;                                                                    \
    }                                                                                     \
  } while (0)

#define LS_CHECK(x)            \
  do {                         \
    int rc_ = (x);             \
    if (rc_ != LS_OK) return rc_; \
  } while (0)

static constexpr int NMAX_STACK = 256;  // stride of stacked univariate vectors
static constexpr int N_MAX = 136;       // largest supported univariate size (KS <= 34)

struct ls_ctx {
  int d = 0, p = 0;  // p: space degree p_s
  int pt = 0;        // time degree p_t (PAPER.md 179-180: p = (p_s, p_t))
  int64_t n_el[4] = {0, 0, 0, 0};
  int n[3] = {1, 1, 1};  // n_1..n_d
  int nt = 0;
  int64_t Ns = 0, Ntot = 0;  // global sizes
  // distributed layout
  int rank = 0, world = 1;
  int64_t t0 = 0, ntl = 0, Nl = 0;  // local slab [t0, t0+ntl), Nl = ntl * Ns
  std::unique_ptr<Comm> comm;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int64_t launches = 0;
  int fd_variant = 0;  // ls_tune knob LS_TUNE_FD_KERNEL: 0 auto, 1 smem-staged (v2/pp), 2 register-direct
  int fd_tail = 1;     // ls_tune knob LS_TUNE_FD_TAIL: DFMA tail rows in the ping-pong FD kernel
  // centrosymmetric split of the spatial modes (fd_rd_kernel.cuh CS): cs_dir[k] = direction k's
  // eigenbasis was built from the even / odd reduced pencils; fd_cs = ls_tune LS_TUNE_FD_CS
  bool cs_dir[3] = {false, false, false};
  int fd_cs = 1;
  int fd_time = 1;
  int fd_plane = 0;  // ls_tune LS_TUNE_FD_PLANE: spatial modes 1 + 2 in one launch (fd_plane_kernel.cuh;
                     // opt-in: measured slower than the per-direction split kernels)  // ls_tune LS_TUNE_FD_TIME: fused time mode (fd_time_kernel.cuh) where n_t <= 104
  double* Wf_cs[3] = {nullptr, nullptr, nullptr};  // [A_e^T (he x he) | A_o^T (ho x ho)]
  double* Wb_cs[3] = {nullptr, nullptr, nullptr};  // [A_e | A_o]
  int mv_variant = 0;  // ls_tune knob LS_TUNE_MATVEC: 0 auto, 1 four passes (v1), 2 three fused passes (v2)
  int mv6 = 0;         // ls_tune LS_TUNE_MV6: v4's direction-3 and time passes as DFMA stencil passes
                       // (matvec6_kernels.cuh): 0 off (default: measured slower), 1 on
  int mv2_sweep = 1;
  int mv4_sweep = 0;   // ls_tune LS_TUNE_MV4_SWEEP: v4's plane pass as the DFMA register sweep (d = 3, p <= 4;
                       // opt-in: measured 2.2x slower than the DMMA plane pass at config 5 p = 4)   // ls_tune LS_TUNE_MV2_SWEEP: v2's d = 3 plane pass as the register sweep (p = 2)
  int pq_fuse = 1;     // ls_tune LS_TUNE_PQ_FUSE: p.q in the matvec's last-pass epilogue
  int mv5 = 2;         // ls_tune knob LS_TUNE_MV5: v4's direction-3 and time passes fused (mv5_kernels.cuh):
                       // 0 off, 1 on, 2 automatic (p <= 4: measured faster there, slower above)
  // PCG: the next ls_matvec also forms p.q (x.y) into scal[fuse_dot_slot] when its last pass can
  // (v4 time-pass epilogue); fuse_dot_done reports whether it did
  int fuse_dot_slot = -1;
  bool fuse_dot_done = false;
  // matvec v2: Toeplitz stencil + boundary corrections per band matrix (matvec2_kernels.cuh)
  struct Split {
    std::vector<double> s;  // 2p+1
    double* E = nullptr;     // device [nb][2p+1]
  };
  struct DirSplit {
    Split M, K, J, K2;  // space: M, K, J, 2K ; time: M = M_t, K = K_t
    int lo = 0, hi = 0;
  };
  DirSplit dsplit[3], tsplit;
  // matvec v3: band blocks in DMMA A-fragment order per direction (matvec3_kernels.cuh)
  double* frag_dir[3] = {nullptr, nullptr, nullptr};  // mats M, J, K, 2K
  double* frag_time = nullptr;                        // mats K_t, M_t
  int n1p = 0;                 // padded direction-1 row of the v3 intermediates
  double** scatter_tab = nullptr;  // fd_apply_scatter: device copy of the caller's table
  // fd_apply_host pipeline: copy stream + events (H2D / D2H per time-slice chunk)
  cudaStream_t copy_stream = nullptr;
  // fd_apply_host_batch: the second device buffer pair, the H2D / D2H streams and their events
  double* hb_r = nullptr;
  double* hb_z = nullptr;
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  cudaEvent_t bev[7] = {};
  // distributed path: NCCL stream of the pipelined all-to-all / halo exchange and its events
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t cev[12] = {};
  cudaEvent_t hev[17] = {};
  double** scatter_stage = nullptr;  // pinned host staging of that table
  double* xT_pad = nullptr;    // v3: the last time slice of x in the padded layout
  double* tcol = nullptr;      // v5: column bands of K_t, M_t per time slice [nt][32]

  // host copies (introspection)
  std::vector<double> hM[3], hK[3], hJ[3], hMt, hKt, hlam[4], hU[4];

  // device data
  double* Wf[4] = {nullptr, nullptr, nullptr, nullptr};  // U^T, n x n row-major (index 3 = time)
  double* Wb[4] = {nullptr, nullptr, nullptr, nullptr};  // U
  double* lam[4] = {nullptr, nullptr, nullptr, nullptr};
  double* lam_s = nullptr;  // Lambda_s per spatial index (N_s)
  double* bM[3] = {nullptr, nullptr, nullptr};
  double* bK[3] = {nullptr, nullptr, nullptr};
  double* bJ[3] = {nullptr, nullptr, nullptr};
  double* bMt = nullptr;
  double* bKt = nullptr;
  double* tmp[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // matvec / fd workspaces
  double* pr = nullptr;  // pcg vectors
  double* pz = nullptr;
  double* pp = nullptr;
  double* pq = nullptr;
  double* partials = nullptr;
  double* scal = nullptr;
  double* h_scal = nullptr;  // pinned
  double* rhs_buf = nullptr; // stacked univariate load vectors (device)
  // mapped domain (ls_setup_geo): physical stencil factors, P^G scaling
  std::unique_ptr<GeoMap> gmap;
  std::unique_ptr<GeoDev> geo;
  int precond = LS_PRECOND_P;
  double* dm12 = nullptr;    // D^{-1/2} (N) for P^G
  double fit_res = 0.0;
  // graph-resident PCG loop (one GPU): the iteration body captured once under a WHILE node
  int pcg_graph = 1;                 // ls_tune LS_TUNE_PCG_GRAPH
  cudaStream_t cap_stream = nullptr;
  cudaStream_t cap_stream2 = nullptr;
  cudaGraphExec_t pcg_exec = nullptr;
  const double* pcg_key_b = nullptr;
  const double* pcg_key_x = nullptr;
  int64_t pcg_fixed_launches = 0;
  double pcg_key_tol = -1.0;
  int pcg_key_iter = -1;
  int64_t pcg_body_launches = 0;
  std::vector<void*> allocs;
  // profiling of the mode kernel
  bool prof = false;
  struct ProfRec { cudaEvent_t a, b; double flops; };
  std::vector<ProfRec> prof_recs;
  std::vector<cudaEvent_t> ev_pool;
  cudaEvent_t get_event() {
    if (!ev_pool.empty()) { cudaEvent_t e = ev_pool.back(); ev_pool.pop_back(); return e; }
    cudaEvent_t e; cudaEventCreate(&e); return e;
  }

  ~ls_ctx() {
    for (auto& r : prof_recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : ev_pool) cudaEventDestroy(e);
    for (void* a : allocs) cudaFree(a);
    if (h_scal) cudaFreeHost(h_scal);
    if (scatter_stage) cudaFreeHost(scatter_stage);
    for (auto e : hev)
      if (e) cudaEventDestroy(e);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    for (auto e : bev)
      if (e) cudaEventDestroy(e);
    if (h2d_stream) cudaStreamDestroy(h2d_stream);
    if (d2h_stream) cudaStreamDestroy(d2h_stream);
    for (auto e : cev)
      if (e) cudaEventDestroy(e);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    if (pcg_exec) cudaGraphExecDestroy(pcg_exec);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (cap_stream2) cudaStreamDestroy(cap_stream2);
  }
  int alloc(double** ptr, size_t count) {
    void* v = nullptr;
    cudaError_t e = cudaMalloc(&v, std::max<size_t>(count, 1) * sizeof(double));
    if (e != cudaSuccess) return LS_ENOMEM;
    allocs.push_back(v);
    *ptr = static_cast<double*>(v);
    return LS_OK;
  }
};

// ------------------------------------------------------------------------------------------
// mode-product dispatch
// ------------------------------------------------------------------------------------------
template <class C>
static int launch_mode_cfg(ls_ctx* ctx, const ModeArgs& a0) {
  static int occ = -1;
  if (occ < 0) {
    LS_CUDA(cudaFuncSetAttribute(fd_mode_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(C::SMEM)));
    LS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fd_mode_kernel<C>, C::THREADS,
                                                          C::SMEM));
    if (occ < 1) occ = 1;
  }
  ModeArgs a = a0;
  a.ntiles = (a.ncols + C::BN - 1) / C::BN;
  if (a.ntiles == 0) return LS_OK;
  unsigned grid = std::min<unsigned>(a.ntiles, unsigned(ctx->num_sms * occ));
  ls_ctx::ProfRec rec{};
  if (ctx->prof) {
    rec.a = ctx->get_event();
    rec.b = ctx->get_event();
    rec.flops = 2.0 * double(a.n) * double(a.n) * double(a.ncols);
    cudaEventRecord(rec.a, ctx->stream);
  }
  LS_CUDA(launch_pdl(fd_mode_kernel<C>, grid, C::THREADS, C::SMEM, ctx->stream, a));
  ctx->launches++;
  if (ctx->prof) {
    cudaEventRecord(rec.b, ctx->stream);
    ctx->prof_recs.push_back(rec);
  }
  LS_CUDA(cudaGetLastError());
  return LS_OK;
}

template <class C>
static int launch_mode_pp(ls_ctx* ctx, const ModeArgs& a0) {
  static int ready = 0;
  if (!ready) {
    LS_CUDA(cudaFuncSetAttribute(fd_mode_pp_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(C::SMEM)));
    ready = 1;
  }
  ModeArgs a = a0;
  a.ntiles = (a.ncols + C::BN - 1) / C::BN;
  if (a.ntiles == 0) return LS_OK;
  unsigned grid = std::min<unsigned>(a.ntiles, unsigned(ctx->num_sms));
  ls_ctx::ProfRec rec{};
  if (ctx->prof) {
    rec.a = ctx->get_event();
    rec.b = ctx->get_event();
    rec.flops = 2.0 * double(a.n) * double(a.n) * double(a.ncols);
    cudaEventRecord(rec.a, ctx->stream);
  }
  LS_CUDA(launch_pdl(fd_mode_pp_kernel<C>, grid, C::THREADS, C::SMEM, ctx->stream, a));
  ctx->launches++;
  if (ctx->prof) {
    cudaEventRecord(rec.b, ctx->stream);
    ctx->prof_recs.push_back(rec);
  }
  LS_CUDA(cudaGetLastError());
  return LS_OK;
}

// ping-pong kernel: SPS stages per warp set (buckets A-C)
template <int KS, int NT, int SPS, int TAIL>
static int launch_mode_ks_t(ls_ctx* ctx, const ModeArgs& a, bool mode1, bool scale) {
  if (mode1) return launch_mode_pp<PPCfg<KS, NT, true, false, SPS, TAIL>>(ctx, a);
  if (scale) return launch_mode_pp<PPCfg<KS, NT, false, true, SPS, TAIL>>(ctx, a);
  return launch_mode_pp<PPCfg<KS, NT, false, false, SPS, TAIL>>(ctx, a);
}

template <int KS, int NT, int SPS>
static int launch_mode_ks(ls_ctx* ctx, const ModeArgs& a, bool mode1, bool scale) {
  // odd k-step buckets: n = 8 (MTILES - 1) + 1 or + 2 (e.g. 65, 66 in bucket 17) leaves 1-2
  // valid rows in the last m-tile; those rows go to DFMAs (compute_tile_tail)
  if constexpr ((KS & 1) != 0) {
    const int tail = a.n - 8 * ((KS + 1) / 2 - 1);
    if (ctx->fd_tail && tail == 1) return launch_mode_ks_t<KS, NT, SPS, 1>(ctx, a, mode1, scale);
    if (ctx->fd_tail && tail == 2) return launch_mode_ks_t<KS, NT, SPS, 2>(ctx, a, mode1, scale);
  }
  return launch_mode_ks_t<KS, NT, SPS, 0>(ctx, a, mode1, scale);
}

// balanced m-half kernel (bucket D, n <= 136: W fills 148 KB of shared memory, one tile
// in flight per stage; measured faster than ping-pong there)
template <int KS, int NT, int NSTAGE>
static int launch_mode_half(ls_ctx* ctx, const ModeArgs& a, bool mode1, bool scale) {
  if (mode1) return launch_mode_cfg<ModeCfg<KS, NT, true, false, NSTAGE>>(ctx, a);
  if (scale) return launch_mode_cfg<ModeCfg<KS, NT, false, true, NSTAGE>>(ctx, a);
  return launch_mode_cfg<ModeCfg<KS, NT, false, false, NSTAGE>>(ctx, a);
}

// buckets by k-steps (KS = ceil(n/4)): (NT, NSTAGE) sized for <= 227 KB of shared memory
#define KS_A(K) case K: return launch_mode_ks<K, 4, 2>(ctx, a, mode1, scale);
#define KS_B(K) case K: return launch_mode_ks<K, 2, 2>(ctx, a, mode1, scale);
#define KS_C(K) case K: return launch_mode_ks<K, 2, 1>(ctx, a, mode1, scale);
#define KS_D(K) case K: return launch_mode_half<K, 1, 2>(ctx, a, mode1, scale);

static int round_ks(int ks) {
  static const int list[] = {2, 4, 5, 8, 12, 16, 17, 18, 24, 25, 26, 30, 33, 34};
  for (int v : list)
    if (ks <= v) return v;
  return -1;
}

// register-direct kernel (fd_rd_kernel.cuh), one explicit instantiation per k-step bucket
static int round_ks_rd(int ks) {
  static const int list[] = {
#define LS_RD_ITEM(K) K,
      LS_RD_BUCKETS(LS_RD_ITEM)
#undef LS_RD_ITEM
  };
  for (int v : list)
    if (ks <= v) return v;
  return -1;
}

// cs: 0 = n x n product; 1 / 2 = centrosymmetric fold / unfold (two half-size products,
// W = [W_e | W_o]; the k-step bucket is that of the half extent ceil(n/2))
static int launch_mode_rd(ls_ctx* ctx, const ModeArgs& a, bool mode1, bool scale, int cs = 0) {
  if (a.ncols == 0) return LS_OK;
  const int he = (a.n + 1) / 2, ho = a.n / 2;
  ls_ctx::ProfRec rec{};
  if (ctx->prof) {
    rec.a = ctx->get_event();
    rec.b = ctx->get_event();
    // algorithmic flops of the launch: 2 n^2 per column, or 2 (he^2 + ho^2) with the split
    rec.flops = (cs ? 2.0 * (double(he) * he + double(ho) * ho) : 2.0 * double(a.n) * double(a.n)) * double(a.ncols);
    cudaEventRecord(rec.a, ctx->stream);
  }
  cudaError_t e = cudaErrorInvalidValue;
  switch (round_ks_rd(((cs ? he : a.n) + 3) / 4)) {
#define LS_RD_CASE(K) case K: e = rd_launch<K>(a, mode1, scale, cs, ctx->stream, ctx->num_sms); break;
    LS_RD_BUCKETS(LS_RD_CASE)
#undef LS_RD_CASE
    default: return LS_EINVAL;
  }
  ctx->launches++;
  if (ctx->prof) {
    cudaEventRecord(rec.b, ctx->stream);
    ctx->prof_recs.push_back(rec);
  }
  LS_CUDA(e);
  return LS_OK;
}

static int launch_mode(ls_ctx* ctx, const double* X, double* Y, const double* W, int n, uint64_t P,
                       uint64_t Q, bool scale, const double* lam_a = nullptr,
                       const double* lam_c = nullptr, int cs = 0) {
  ModeArgs a{};
  a.y16 = (reinterpret_cast<uintptr_t>(Y) & 15) == 0;
  a.X = X;
  a.Y = Y;
  a.W = W;
  a.lam_a = lam_a;
  a.lam_c = lam_c;
  a.n = n;
  a.P = uint32_t(P);
  a.Q = uint32_t(Q);
  a.ncols = uint32_t(P * Q);
  const bool mode1 = (Q == 1) && !scale;  // the scaled (time) mode always uses the strided variant
  // auto (measured, tools/fd_variants.py): register-direct for n > 116 (config 4: 75% -> 86% of
  // the FP64 peak), smem-staged ping-pong / m-half kernels below (config 3: 56% vs 37%)
  // it also wins at n = 96 / 97 (bucket 24 / 25: the last m-tile of n = 96 is full, n = 97
  // adds one 8-row tile with one valid row; tools/fdk_sel.py, config 5 p = 2: 4.67 -> 4.45 ms;
  // rd for n = 96 only: 4.51 ms).  Only these measured extents: at n = 98 / 99 and 102 / 103
  // (config 5 p = 4 / 8) the smem-staged kernels stay 13 / 9 % faster.
  if (cs) return launch_mode_rd(ctx, a, mode1, false, cs);  // the split exists in the register-direct kernel
  const bool rd_auto = (n + 3) / 4 >= 30 || n == 96 || n == 97;
  if (ctx->fd_variant == 2 || (ctx->fd_variant == 0 && rd_auto)) return launch_mode_rd(ctx, a, mode1, scale);
  switch (round_ks((n + 3) / 4)) {
    KS_A(2) KS_A(4) KS_A(5) KS_A(8)
    KS_B(12) KS_B(16) KS_B(17) KS_B(18)
    KS_C(24) KS_C(25) KS_C(26)
    KS_D(30) KS_D(33) KS_D(34)
    default: return LS_EINVAL;
  }
}

// ------------------------------------------------------------------------------------------
// setup
// ------------------------------------------------------------------------------------------
static int to_band(ls_ctx* ctx, const std::vector<double>& A, int n, int hb, double** out) {
  const int W = 2 * hb + 1;
  std::vector<double> band(size_t(n) * W, 0.0);
  for (int a = 0; a < n; ++a)
    for (int i = std::max(0, a - hb); i <= std::min(n - 1, a + hb); ++i)
      band[size_t(a) * W + (i - a + hb)] = A[size_t(a) * n + i];
  LS_CHECK(ctx->alloc(out, band.size()));
  LS_CUDA(cudaMemcpy(*out, band.data(), band.size() * sizeof(double), cudaMemcpyHostToDevice));
  return LS_OK;
}

// generalized eigendecomposition K U = M U Lambda, U^T M U = I (eq:eig_dec): host,
// extended-precision Cholesky + Jacobi (setup_host.cpp; reading c17 in DESIGN.md)
static int gen_eig(const std::vector<double>& K, const std::vector<double>& M, int n,
                   std::vector<double>& lam, std::vector<double>& U) {
  if (generalized_eig(K, M, n, lam, U) != 0) return LS_ENOTSPD;
  // sanity: U^T M U = I (PAPER.md 945)
  double err = 0;
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b) {
      double s = 0;
      for (int i = 0; i < n; ++i) {
        double mu = 0;
        for (int j = std::max(0, i - 16); j < std::min(n, i + 17); ++j) mu += M[size_t(i) * n + j] * U[size_t(j) * n + b];
        s += U[size_t(i) * n + a] * mu;
      }
      err = std::max(err, std::fabs(s - (a == b ? 1.0 : 0.0)));
    }
  if (!(err < 1e-8)) return LS_ENOTSPD;
  return LS_OK;
}

// R A R = A up to assembly rounding (64 ulps of max|A|; measured asymmetry <= 1 ulp: the
// exact integrals on uniform open knots are centrosymmetric, PAPER.md 144-147, 1111-1112)
static bool centrosymmetric(const std::vector<double>& A, int n) {
  double mx = 0;
  for (double v : A) mx = std::max(mx, std::fabs(v));
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      if (std::fabs(A[size_t(i) * n + j] - A[size_t(n - 1 - i) * n + (n - 1 - j)]) > 64 * 2.220446049250313e-16 * mx)
        return false;
  return true;
}

static int upload(ls_ctx* ctx, const std::vector<double>& v, double** out);

// eq:eig_dec (PAPER.md 939-945) for a centrosymmetric pencil (J, M), by its even and odd
// reductions (fd_rd_kernel.cuh CS): with Q_e = [e_k + e_{n-1-k}] (k < he; e_h alone at the
// middle of an odd n) and Q_o = [e_k - e_{n-1-k}] (k < ho), J_e = Q_e^T J Q_e, M_e = Q_e^T M Q_e
// (the same for o), formed in 80-bit.  J_e a = M_e a lambda with a^T M_e a = 1 gives the
// eigenvector u = Q_e a of (J, M) with u^T M u = 1, so U = [Q_e A_e | Q_o A_o] and
// lambda = [lambda_e | lambda_o] (ascending within each half).  The cross terms Q_e^T J Q_o are
// the assembly's last-ulp asymmetry and are dropped: this is the eigenbasis of (J + RJR)/2,
// (M + RMR)/2 (z moves by <= 4e-14 relative, reading c25).
static int cs_eig(ls_ctx* ctx, int k, const std::vector<double>& J, const std::vector<double>& M, int n) {
  const int he = (n + 1) / 2, ho = n / 2;
  auto reduce = [&](const std::vector<double>& A, int nh, int sg, std::vector<long double>& E) {
    E.assign(size_t(nh) * nh, 0.0L);
    for (int a = 0; a < nh; ++a)
      for (int b = 0; b < nh; ++b) {
        const int ra = n - 1 - a, rb = n - 1 - b;
        long double v = A[size_t(a) * n + b];
        if (rb != b) v += sg * (long double)A[size_t(a) * n + rb];
        if (ra != a) v += sg * (long double)A[size_t(ra) * n + b];
        if (ra != a && rb != b) v += (long double)A[size_t(ra) * n + rb];
        E[size_t(a) * nh + b] = v;
      }
  };
  std::vector<long double> Je, Me, Jo, Mo;
  reduce(J, he, 1, Je);
  reduce(M, he, 1, Me);
  reduce(J, ho, -1, Jo);
  reduce(M, ho, -1, Mo);
  std::vector<double> le, lo, Ae, Ao;
  if (generalized_eig(Je, Me, he, le, Ae) != 0) return LS_ENOTSPD;
  if (ho > 0 && generalized_eig(Jo, Mo, ho, lo, Ao) != 0) return LS_ENOTSPD;
  std::vector<double>& U = ctx->hU[k];
  std::vector<double>& lam = ctx->hlam[k];
  U.assign(size_t(n) * n, 0.0);
  lam.assign(n, 0.0);
  for (int j = 0; j < he; ++j) {
    lam[j] = le[j];
    for (int i = 0; i < n; ++i) U[size_t(i) * n + j] = Ae[size_t(std::min(i, n - 1 - i)) * he + j];
  }
  for (int j = 0; j < ho; ++j) {
    lam[he + j] = lo[j];
    for (int i = 0; i < ho; ++i) {
      U[size_t(i) * n + he + j] = Ao[size_t(i) * ho + j];
      U[size_t(n - 1 - i) * n + he + j] = -Ao[size_t(i) * ho + j];
    }
  }
  // sanity: U^T M U = I, U^T J U = Lambda (PAPER.md 945) on the full matrices
  {
    std::vector<double> MU(size_t(n) * n, 0.0), JU(size_t(n) * n, 0.0);
    for (int i = 0; i < n; ++i)
      for (int l = 0; l < n; ++l) {
        const double m = M[size_t(i) * n + l], jj = J[size_t(i) * n + l];
        if (m == 0.0 && jj == 0.0) continue;
        for (int c = 0; c < n; ++c) {
          MU[size_t(i) * n + c] += m * U[size_t(l) * n + c];
          JU[size_t(i) * n + c] += jj * U[size_t(l) * n + c];
        }
      }
    double em = 0, ej = 0;
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b) {
        double sm = 0, sj = 0;
        for (int i = 0; i < n; ++i) {
          sm += U[size_t(i) * n + a] * MU[size_t(i) * n + b];
          sj += U[size_t(i) * n + a] * JU[size_t(i) * n + b];
        }
        em = std::max(em, std::fabs(sm - (a == b ? 1.0 : 0.0)));
        ej = std::max(ej, std::fabs(sj - (a == b ? lam[a] : 0.0)) / std::max(1.0, std::fabs(lam[b])));
      }
    if (!(em < 1e-8) || !(ej < 1e-8)) return LS_ENOTSPD;
  }
  std::vector<double> wf(size_t(he) * he + size_t(ho) * ho), wb(wf.size());
  for (int a = 0; a < he; ++a)
    for (int i = 0; i < he; ++i) {
      wf[size_t(a) * he + i] = Ae[size_t(i) * he + a];
      wb[size_t(i) * he + a] = Ae[size_t(i) * he + a];
    }
  const size_t o = size_t(he) * he;
  for (int a = 0; a < ho; ++a)
    for (int i = 0; i < ho; ++i) {
      wf[o + size_t(a) * ho + i] = Ao[size_t(i) * ho + a];
      wb[o + size_t(i) * ho + a] = Ao[size_t(i) * ho + a];
    }
  LS_CHECK(upload(ctx, wf, &ctx->Wf_cs[k]));
  LS_CHECK(upload(ctx, wb, &ctx->Wb_cs[k]));
  ctx->cs_dir[k] = true;
  return LS_OK;
}

static int upload(ls_ctx* ctx, const std::vector<double>& v, double** out) {
  LS_CHECK(ctx->alloc(out, v.size()));
  LS_CUDA(cudaMemcpy(*out, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice));
  return LS_OK;
}

// Toeplitz split B = T + E of the band matrices of one direction (matvec2_kernels.cuh):
// stencil s = the middle row; zone [lo, hi) = the maximal run of rows around the middle
// whose band equals s to 64 ulps (relative to max|s|) in every matrix of the set; E =
// B - T on the other rows.  n < 2p + 1: empty zone, s = 0, E = B.
static int make_split(ls_ctx* ctx, const std::vector<double>* const* mats, int nm, int n, int p,
                      ls_ctx::DirSplit& out, bool space) {
  const int W = 2 * p + 1;
  const int c = n / 2;
  const bool has_mid = (n >= W) && (c - p >= 0) && (c + p < n);
  std::vector<std::vector<double>> st(nm, std::vector<double>(W, 0.0));
  if (has_mid)
    for (int m = 0; m < nm; ++m)
      for (int j = 0; j < W; ++j) st[m][j] = (*mats[m])[size_t(c) * n + (c - p + j)];
  auto interior = [&](int i) {
    if (!has_mid || i - p < 0 || i + p >= n) return false;
    for (int m = 0; m < nm; ++m) {
      double mx = 0;
      for (int j = 0; j < W; ++j) mx = std::max(mx, std::fabs(st[m][j]));
      for (int j = 0; j < W; ++j)
        if (std::fabs((*mats[m])[size_t(i) * n + (i - p + j)] - st[m][j]) > 64 * 2.220446049250313e-16 * mx)
          return false;
    }
    return true;
  };
  int lo = n, hi = n;
  if (has_mid && interior(c)) {
    lo = c;
    hi = c + 1;
    while (lo - 1 >= 0 && interior(lo - 1)) --lo;
    while (hi < n && interior(hi)) ++hi;
  }
  out.lo = lo;
  out.hi = hi;
  const int nb = lo + (n - hi);
  auto fill = [&](int m, double scale, ls_ctx::Split& sp) -> int {
    sp.s.assign(W, 0.0);
    for (int j = 0; j < W; ++j) sp.s[j] = scale * st[m][j];
    std::vector<double> E(size_t(std::max(nb, 1)) * W, 0.0);
    for (int i = 0; i < n; ++i) {
      if (i >= lo && i < hi) continue;
      const int e = (i < lo) ? i : lo + (i - hi);
      for (int j = 0; j < W; ++j) {
        const int col = i - p + j;
        E[size_t(e) * W + j] = (col >= 0 && col < n) ? scale * ((*mats[m])[size_t(i) * n + col] - st[m][j]) : 0.0;
      }
    }
    return upload(ctx, E, &sp.E);
  };
  // space: mats = {M, K, J}; time: mats = {M_t, K_t}
  LS_CHECK(fill(0, 1.0, out.M));
  LS_CHECK(fill(1, 1.0, out.K));
  if (space) {
    LS_CHECK(fill(2, 1.0, out.J));
    LS_CHECK(fill(1, 2.0, out.K2));
  }
  return LS_OK;
}

// band blocks of `nm` matrices in m8n8k4 A-fragment order for matvec v3:
// out[((m*MT + mt)*NKB + j)*32 + l] = scale[m] * W_m[8mt + S0 + l/4][4(2mt - OFF + j) + l%4]
static int make_frags(ls_ctx* ctx, const std::vector<double>* const* mats, const double* scale, int nm,
                      int n, int p, double** out) {
  const int MT = mv3_mt(p, n), NKB = mv3_nkb(p), OFF = mv3_off(p), S0 = mv3_s0(p);
  std::vector<double> f(size_t(nm) * MT * NKB * 32, 0.0);
  for (int m = 0; m < nm; ++m)
    for (int mt = 0; mt < MT; ++mt)
      for (int j = 0; j < NKB; ++j)
        for (int l = 0; l < 32; ++l) {
          const int row = 8 * mt + S0 + l / 4, col = 4 * (2 * mt - OFF + j) + l % 4;
          if (row >= 0 && row < n && col >= 0 && col < n && std::abs(row - col) <= p)
            f[((size_t(m) * MT + mt) * NKB + j) * 32 + l] = scale[m] * (*mats[m])[size_t(row) * n + col];
        }
  return upload(ctx, f, out);
}

static int setup_common(ls_ctx* ctx) {
  const int d = ctx->d, p = ctx->p, pt = ctx->pt;
  int dev = 0;
  LS_CUDA(cudaGetDevice(&dev));
  LS_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, dev));
  // sizes (reading c1): n_k = n_el + p - 2, n_t = n_el + p - 1
  ctx->Ns = 1;
  for (int k = 0; k < d; ++k) {
    ctx->n[k] = int(ctx->n_el[k] + p - 2);
    ctx->Ns *= ctx->n[k];
  }
  ctx->nt = int(ctx->n_el[d] + pt - 1);
  for (int k = 0; k < d; ++k)
    if (ctx->n[k] > N_MAX) return LS_EINVAL;
  if (ctx->nt > N_MAX) return LS_EINVAL;
  ctx->Ntot = ctx->Ns * ctx->nt;
  if (ctx->Ns >= (int64_t(1) << 31)) return LS_EINVAL;
  // slab layout: uneven split of n_t over `world` ranks
  split_part(ctx->nt, ctx->world, ctx->rank, &ctx->t0, &ctx->ntl);
  ctx->Nl = ctx->ntl * ctx->Ns;
  // memory estimate: 6 workspaces + 4 pcg vectors (+ 2 all-to-all buffers when distributed)
  {
    size_t fr = 0, tot = 0;
    LS_CUDA(cudaMemGetInfo(&fr, &tot));
    const double need = double(ctx->Nl) * 8.0 * (10 + (ctx->world > 1 ? 2 : 0)) + 64e6;
    if (need > double(fr)) return LS_ENOMEM;
  }

  // host assembly (PAPER.md 686-703, 738-757)
  int rc = LS_OK;
  // P^G (PAPER.md 969-1045): weighted univariate pencils (M^G_k, J^G_k) for the eigen step
  const bool pg = ctx->gmap && ctx->precond == LS_PRECOND_PG;
  std::vector<double> mu[3], om[3], wM[3], wJ[3];
  if (pg) LS_CHECK(pg_weights(*ctx->gmap, ctx->n_el, mu, om, &ctx->fit_res));
  for (int k = 0; k < d && rc == LS_OK; ++k) {
    Factors f = space_factors(int(ctx->n_el[k]), p);
    ctx->hM[k] = f.M;
    ctx->hK[k] = f.K;
    ctx->hJ[k] = f.J;
    if (pg) {
      weighted_space_factors(int(ctx->n_el[k]), p, mu[k], om[k], wM[k], wJ[k]);
      rc = gen_eig(wJ[k], wM[k], f.n, ctx->hlam[k], ctx->hU[k]);
    } else if (centrosymmetric(f.J, f.n) && centrosymmetric(f.M, f.n)) {
      rc = cs_eig(ctx, k, f.J, f.M, f.n);
    } else {
      rc = gen_eig(f.J, f.M, f.n, ctx->hlam[k], ctx->hU[k]);
    }
  }
  Factors ft = time_factors(int(ctx->n_el[d]), pt);
  ctx->hMt = ft.M;
  ctx->hKt = ft.K;
  if (rc == LS_OK) rc = gen_eig(ft.K, ft.M, ft.n, ctx->hlam[3], ctx->hU[3]);
  if (rc != LS_OK) return rc;

  // device copies: W_fwd = U^T, W_bwd = U (row-major), eigenvalues
  for (int k = 0; k < 4; ++k) {
    if (k >= d && k != 3) continue;
    const int n = (k == 3) ? ctx->nt : ctx->n[k];
    std::vector<double> Ut(size_t(n) * n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) Ut[size_t(j) * n + i] = ctx->hU[k][size_t(i) * n + j];
    LS_CHECK(upload(ctx, Ut, &ctx->Wf[k]));
    LS_CHECK(upload(ctx, ctx->hU[k], &ctx->Wb[k]));
    LS_CHECK(upload(ctx, ctx->hlam[k], &ctx->lam[k]));
  }
  LS_CHECK(ctx->alloc(&ctx->lam_s, ctx->Ns));
  lambda_s_kernel<<<1024, 256, 0, ctx->stream>>>(ctx->lam_s, ctx->lam[0], d >= 2 ? ctx->lam[1] : nullptr,
                                                 d >= 3 ? ctx->lam[2] : nullptr, ctx->n[0],
                                                 d >= 2 ? ctx->n[1] : 1, d, uint64_t(ctx->Ns));
  ctx->launches++;
  LS_CUDA(cudaGetLastError());
  // banded factors for A (identity map, T = 1: K_t = K_t^, M_t = M_t^; reading c9)
  for (int k = 0; k < d; ++k) {
    LS_CHECK(to_band(ctx, ctx->hM[k], ctx->n[k], p, &ctx->bM[k]));
    LS_CHECK(to_band(ctx, ctx->hK[k], ctx->n[k], p, &ctx->bK[k]));
    LS_CHECK(to_band(ctx, ctx->hJ[k], ctx->n[k], p, &ctx->bJ[k]));
  }
  LS_CHECK(to_band(ctx, ctx->hMt, ctx->nt, pt, &ctx->bMt));
  LS_CHECK(to_band(ctx, ctx->hKt, ctx->nt, pt, &ctx->bKt));
  // matvec v2 stencil splits (reading c18)
  for (int k = 0; k < d; ++k) {
    const std::vector<double>* mats[3] = {&ctx->hM[k], &ctx->hK[k], &ctx->hJ[k]};
    LS_CHECK(make_split(ctx, mats, 3, ctx->n[k], p, ctx->dsplit[k], true));
  }
  {
    const std::vector<double>* mats[2] = {&ctx->hMt, &ctx->hKt};
    LS_CHECK(make_split(ctx, mats, 2, ctx->nt, pt, ctx->tsplit, false));
  }
  // matvec v3 band fragments
  for (int k = 0; k < d; ++k) {
    const std::vector<double>* mats[4] = {&ctx->hM[k], &ctx->hJ[k], &ctx->hK[k], &ctx->hK[k]};
    const double scale[4] = {1.0, 1.0, 1.0, 2.0};
    LS_CHECK(make_frags(ctx, mats, scale, 4, ctx->n[k], p, &ctx->frag_dir[k]));
  }
  {
    const std::vector<double>* mats[2] = {&ctx->hKt, &ctx->hMt};
    const double scale[2] = {1.0, 1.0};
    LS_CHECK(make_frags(ctx, mats, scale, 2, ctx->nt, pt, &ctx->frag_time));
  }
  if (pt <= 8) {  // v5 time scatter: tcol[t'][k] = K_t[t' - p_t + k][t'], tcol[t'][20 + k] = M_t[..][t']
    const int nt = ctx->nt;
    std::vector<double> tc(size_t(nt) * 40, 0.0);
    for (int t = 0; t < nt; ++t)
      for (int k = 0; k <= 2 * pt; ++k) {
        const int r = t - pt + k;
        if (r < 0 || r >= nt) continue;
        tc[size_t(t) * 40 + k] = ctx->hKt[size_t(r) * nt + t];
        tc[size_t(t) * 40 + 20 + k] = ctx->hMt[size_t(r) * nt + t];
      }
    LS_CHECK(upload(ctx, tc, &ctx->tcol));
  }
  // workspaces (halo rows for the distributed matvec: p slices each side)
  const size_t halo = size_t(2 * pt) * ctx->Ns;  // time halo of the banded time factors
  // v3 matvec intermediates use 64-byte rows along direction 1 (d >= 2, n_1 >= 64):
  // unaligned 132-double rows made the strided and contiguous passes re-read ~50 %
  ctx->n1p = (d >= 2 && ctx->n[0] >= 64) ? (ctx->n[0] + 7) / 8 * 8 : ctx->n[0];
  // buffers sized for the widest padding ls_tune may select (16 doubles = 128-byte rows)
  const size_t nsp = size_t(ctx->Ns / ctx->n[0]) * ((ctx->n[0] + 15) / 16 * 16);
  const size_t tmp_sz = std::max(size_t(ctx->Nl) + halo, size_t(ctx->ntl) * nsp);
  for (int i = 0; i < 6; ++i) LS_CHECK(ctx->alloc(&ctx->tmp[i], tmp_sz));
  LS_CHECK(ctx->alloc(&ctx->xT_pad, nsp));
  LS_CHECK(ctx->alloc(&ctx->pr, ctx->Nl));
  LS_CHECK(ctx->alloc(&ctx->pz, ctx->Nl));
  LS_CHECK(ctx->alloc(&ctx->pp, ctx->Nl + halo));
  LS_CHECK(ctx->alloc(&ctx->pq, ctx->Nl));
  LS_CHECK(ctx->alloc(&ctx->partials, RED_BLOCKS));
  LS_CHECK(ctx->alloc(&ctx->scal, S_NSLOT));
  LS_CHECK(ctx->alloc(&ctx->rhs_buf, 6 * NMAX_STACK));
  LS_CUDA(cudaMallocHost(&ctx->h_scal, S_NSLOT * sizeof(double)));
  if (ctx->gmap) {
    // physical spatial factors on the device (eq:A_kron on Omega, PAPER.md 697-703)
    ctx->geo.reset(new GeoDev());
    ctx->geo->pt = pt;
    LS_CHECK(geo_assemble(*ctx->geo, *ctx->gmap, d, p, ctx->n_el, ctx->stream, &ctx->launches));
    if (pg) {
      // diag(Pbar^G) = diag(K_t) (x) prod_k diag(M^G_k) + diag(M_t) (x) sum_k diag(J^G_k) prod_{j!=k} diag(M^G_j)
      const int nt = ctx->nt;
      std::vector<double> pdt(2 * size_t(nt)), pds(2 * size_t(ctx->Ns));
      for (int t = 0; t < nt; ++t) {
        pdt[t] = ctx->hKt[size_t(t) * nt + t];
        pdt[nt + t] = ctx->hMt[size_t(t) * nt + t];
      }
      for (int64_t i = 0; i < ctx->Ns; ++i) {
        int ik[3] = {0, 0, 0};
        int64_t r = i;
        for (int k = 0; k < d; ++k) {
          ik[k] = int(r % ctx->n[k]);
          r /= ctx->n[k];
        }
        double m = 1, j = 0;
        for (int k = 0; k < d; ++k) {
          const int n = ctx->n[k];
          double jk = wJ[k][size_t(ik[k]) * n + ik[k]];
          for (int l = 0; l < d; ++l)
            if (l != k) jk *= wM[l][size_t(ik[l]) * ctx->n[l] + ik[l]];
          j += jk;
          m *= wM[k][size_t(ik[k]) * n + ik[k]];
        }
        pds[i] = m;
        pds[ctx->Ns + i] = j;
      }
      double *dpdt, *dpds;
      LS_CHECK(upload(ctx, pdt, &dpdt));
      LS_CHECK(upload(ctx, pds, &dpds));
      LS_CHECK(ctx->alloc(&ctx->dm12, ctx->Nl));
      LS_CHECK(pg_scaling(*ctx->geo, ctx->bKt, ctx->bMt, nt, dpdt, dpds, ctx->dm12, int(ctx->t0), int(ctx->ntl),
                          ctx->stream, &ctx->launches));
    }
  }
  LS_CUDA(cudaDeviceSynchronize());
  return LS_OK;
}

static int validate(int d, int p, int pt, const int64_t* n_elems) {
  // p_s >= 2 (Assumption 2, PAPER.md 218-223: C^1 in space); p_t >= 1
  if (d < 1 || d > 3 || p < 2 || pt < 1 || n_elems == nullptr) return LS_EINVAL;
  for (int k = 0; k <= d; ++k)
    if (n_elems[k] < 1 || n_elems[k] > 100000) return LS_EINVAL;
  return LS_OK;
}

extern "C" int ls_setup_deg(int d, int p_s, int p_t, const int64_t* n_elems, ls_ctx** out) {
  if (!out) return LS_EINVAL;
  *out = nullptr;
  LS_CHECK(validate(d, p_s, p_t, n_elems));
  auto* ctx = new ls_ctx();
  ctx->d = d;
  ctx->p = p_s;
  ctx->pt = p_t;
  for (int k = 0; k <= d; ++k) ctx->n_el[k] = n_elems[k];
  int rc = setup_common(ctx);
  if (rc != LS_OK) {
    delete ctx;
    return rc;
  }
  *out = ctx;
  return LS_OK;
}

extern "C" int ls_setup(int d, int p, const int64_t* n_elems, ls_ctx** out) {
  return ls_setup_deg(d, p, p, n_elems, out);
}

extern "C" int ls_setup_geo(int d, int p_s, int p_t, const int64_t* n_elems, const ls_geometry* geo, int precond,
                            ls_ctx** out) {
  return ls_setup_geo_dist(d, p_s, p_t, n_elems, geo, precond, 0, 1, nullptr, out);
}

extern "C" int ls_setup_geo_dist(int d, int p_s, int p_t, const int64_t* n_elems, const ls_geometry* geo,
                                 int precond, int rank, int world, const void* nccl_unique_id, ls_ctx** out) {
  if (!out) return LS_EINVAL;
  *out = nullptr;
  LS_CHECK(validate(d, p_s, p_t, n_elems));
  if (!geo || (precond != LS_PRECOND_P && precond != LS_PRECOND_PG)) return LS_EINVAL;
  if (world < 1 || rank < 0 || rank >= world || (world > 1 && !nccl_unique_id)) return LS_EINVAL;
  if (world > 1 && (n_elems[d] + p_t - 1) / world < p_t) return LS_EINVAL;  // slab thinner than the halo
  int nloc = 1;
  for (int k = 0; k < d; ++k) nloc *= p_s + 1;
  if (nloc > 343) return LS_EINVAL;
  auto* ctx = new ls_ctx();
  ctx->d = d;
  ctx->p = p_s;
  ctx->pt = p_t;
  ctx->precond = precond;
  ctx->rank = rank;
  ctx->world = world;
  for (int k = 0; k <= d; ++k) ctx->n_el[k] = n_elems[k];
  ctx->gmap.reset(new GeoMap());
  int rc = geo_copy(geo, d, *ctx->gmap);
  if (rc == LS_OK) {
    // stencil storage 3 (2p+1)^d N_s on top of the usual estimate
    int64_t Ns = 1, S = 1;
    for (int k = 0; k < d; ++k) {
      Ns *= n_elems[k] + p_s - 2;
      S *= 2 * p_s + 1;
    }
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) rc = LS_ECUDA;
    else if (double(3 * S) * double(Ns) * 8.0 > 0.5 * double(fr)) rc = LS_ENOMEM;  // the three stencil arrays
  }
  if (rc == LS_OK) rc = setup_common(ctx);
  if (rc == LS_OK && world > 1) {
    ctx->comm.reset(new Comm());
    rc = ctx->comm->init(nccl_unique_id, rank, world, ctx->nt, ctx->Ns);
    if (rc == LS_OK && cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking) != cudaSuccess) rc = LS_ECUDA;
    for (auto& e : ctx->cev)
      if (rc == LS_OK && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) rc = LS_ECUDA;
  }
  if (rc != LS_OK) {
    delete ctx;
    return rc;
  }
  *out = ctx;
  return LS_OK;
}

extern "C" int ls_pg_factors(const ls_geometry* geo, int d, int p_s, const int64_t* n_elems, double* mu,
                             double* omega, double* Mw, double* Jw, double* fit_rel_res) {
  if (!geo || d < 1 || d > 3 || p_s < 2 || !n_elems || !mu || !omega || !Mw || !Jw) return LS_EINVAL;
  for (int k = 0; k < d; ++k)
    if (n_elems[k] < 1 || n_elems[k] > 100000) return LS_EINVAL;
  GeoMap g;
  LS_CHECK(geo_copy(geo, d, g));
  std::vector<double> m[3], o[3];
  LS_CHECK(pg_weights(g, n_elems, m, o, fit_rel_res));
  size_t off = 0, moff = 0;
  for (int k = 0; k < d; ++k) {
    std::copy(m[k].begin(), m[k].end(), mu + off);
    std::copy(o[k].begin(), o[k].end(), omega + off);
    off += m[k].size();
    std::vector<double> M, J;
    weighted_space_factors(int(n_elems[k]), p_s, m[k], o[k], M, J);
    std::copy(M.begin(), M.end(), Mw + moff);
    std::copy(J.begin(), J.end(), Jw + moff);
    moff += M.size();
  }
  return LS_OK;
}

extern "C" int ls_geo_info(const ls_ctx* ctx, double* out2) {
  if (!ctx || !out2) return LS_EINVAL;
  if (!ctx->geo) return LS_ENOTSUP;
  out2[0] = ctx->fit_res;
  out2[1] = ctx->geo->S;
  return LS_OK;
}

extern "C" int ls_get_unique_id(void* out128) {
  if (!out128) return LS_EINVAL;
  return comm_unique_id(out128);
}

extern "C" int ls_setup_dist_deg(int d, int p_s, int p_t, const int64_t* n_elems, int rank, int world,
                                 const void* nccl_unique_id, ls_ctx** out) {
  if (!out || world < 1 || rank < 0 || rank >= world || (world > 1 && !nccl_unique_id))
    return LS_EINVAL;
  *out = nullptr;
  LS_CHECK(validate(d, p_s, p_t, n_elems));
  auto* ctx = new ls_ctx();
  ctx->d = d;
  ctx->p = p_s;
  ctx->pt = p_t;
  ctx->rank = rank;
  ctx->world = world;
  for (int k = 0; k <= d; ++k) ctx->n_el[k] = n_elems[k];
  // every slab must be at least p_t time slices thick (halo of the banded time factors)
  if (world > 1 && (n_elems[d] + p_t - 1) / world < p_t) {
    delete ctx;
    return LS_EINVAL;
  }
  int rc = setup_common(ctx);
  if (rc == LS_OK && world > 1) {
    ctx->comm.reset(new Comm());
    rc = ctx->comm->init(nccl_unique_id, rank, world, ctx->nt, ctx->Ns);
    if (rc == LS_OK && cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking) != cudaSuccess) rc = LS_ECUDA;
    for (auto& e : ctx->cev)
      if (rc == LS_OK && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) rc = LS_ECUDA;
  }
  if (rc != LS_OK) {
    delete ctx;
    return rc;
  }
  *out = ctx;
  return LS_OK;
}

extern "C" int ls_setup_dist(int d, int p, const int64_t* n_elems, int rank, int world,
                             const void* nccl_unique_id, ls_ctx** out) {
  return ls_setup_dist_deg(d, p, p, n_elems, rank, world, nccl_unique_id, out);
}

extern "C" int ls_layout(const ls_ctx* ctx, int64_t* n_t, int64_t* n_s, int64_t* t0,
                         int64_t* nt_local) {
  if (!ctx) return LS_EINVAL;
  if (n_t) *n_t = ctx->nt;
  if (n_s)
    for (int k = 0; k < ctx->d; ++k) n_s[k] = ctx->n[k];
  if (t0) *t0 = ctx->t0;
  if (nt_local) *nt_local = ctx->ntl;
  return LS_OK;
}

extern "C" int ls_set_stream(ls_ctx* ctx, void* s) {
  if (!ctx) return LS_EINVAL;
  ctx->stream = static_cast<cudaStream_t>(s);
  if (ctx->comm) ctx->comm->stream = ctx->stream;
  return LS_OK;
}

// ------------------------------------------------------------------------------------------
// fd_apply: Algorithm 1 steps 2-4
// ------------------------------------------------------------------------------------------
static inline bool aligned8(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 7) == 0; }

// direction k runs the centrosymmetric split (half the DMMA work of its mode products)
static inline bool use_cs(const ls_ctx* ctx, int k) { return ctx->fd_cs && ctx->cs_dir[k]; }

// directions 1 and 2 run as one plane launch (fd_plane_kernel.cuh): both split, n_1 = n_2
static bool use_plane(const ls_ctx* ctx) {
  return ctx->fd_plane && ctx->d >= 2 && use_cs(ctx, 0) && use_cs(ctx, 1) && ctx->n[0] == ctx->n[1] &&
         pl_supported(ctx->n[0]);
}

static int launch_plane(ls_ctx* ctx, const double* X, double* Y, uint64_t planes, bool forward) {
  if (planes == 0) return LS_OK;
  PLArgs a{};
  a.X = X;
  a.Y = Y;
  a.W2 = forward ? ctx->Wf_cs[1] : ctx->Wb_cs[1];
  a.W1 = forward ? ctx->Wf_cs[0] : ctx->Wb_cs[0];
  a.n = ctx->n[0];
  a.planes = uint32_t(planes);
  ls_ctx::ProfRec rec{};
  if (ctx->prof) {
    rec.a = ctx->get_event();
    rec.b = ctx->get_event();
    const double he = (a.n + 1) / 2, ho = a.n / 2;
    rec.flops = 2.0 * 2.0 * (he * he + ho * ho) * double(a.n) * double(planes);  // two split products per plane
    cudaEventRecord(rec.a, ctx->stream);
  }
  const cudaError_t e = pl_launch(a, forward, ctx->stream, ctx->num_sms);
  ctx->launches++;
  if (ctx->prof) {
    cudaEventRecord(rec.b, ctx->stream);
    ctx->prof_recs.push_back(rec);
  }
  LS_CUDA(e);
  return LS_OK;
}

// spatial modes on a [rows][n_d]..[n_1] block (rows = local time slices)
static int spatial_modes(ls_ctx* ctx, const double* in, double* out, double* ws0, double* ws1,
                         uint64_t rows, bool forward) {
  const int d = ctx->d;
  // steps: direction k (0-based), or -1 = the plane launch of directions 1 + 2.  forward:
  // 1..d, backward: d..1.  Ping-pong ws0/ws1, the first step reads `in`, the last writes `out`.
  int steps[3], ns = 0;
  const bool plane = use_plane(ctx);
  if (forward) {
    if (plane) steps[ns++] = -1;
    for (int k = plane ? 2 : 0; k < d; ++k) steps[ns++] = k;
  } else {
    for (int k = d - 1; k >= (plane ? 2 : 0); --k) steps[ns++] = k;
    if (plane) steps[ns++] = -1;
  }
  const double* src = in;
  for (int s = 0; s < ns; ++s) {
    double* dst = (s == ns - 1) ? out : ((s % 2 == 0) ? ws0 : ws1);
    const int k = steps[s];
    if (k < 0) {
      uint64_t P = rows;
      for (int j = 2; j < d; ++j) P *= ctx->n[j];
      LS_CHECK(launch_plane(ctx, src, dst, P, forward));
      src = dst;
      continue;
    }
    uint64_t Q = 1, P = rows;
    for (int j = 0; j < k; ++j) Q *= ctx->n[j];
    for (int j = k + 1; j < d; ++j) P *= ctx->n[j];
    if (use_cs(ctx, k))
      LS_CHECK(launch_mode(ctx, src, dst, forward ? ctx->Wf_cs[k] : ctx->Wb_cs[k], ctx->n[k], P, Q, false, nullptr,
                           nullptr, forward ? 1 : 2));
    else
      LS_CHECK(launch_mode(ctx, src, dst, forward ? ctx->Wf[k] : ctx->Wb[k], ctx->n[k], P, Q, false));
    src = dst;
  }
  return LS_OK;
}

// F2: the time mode on columns [n_t][ld] (ncols used; Lambda_s of column 0 at lam_c):
// U_t^T, /(lambda_t + Lambda_s), U_t.  One fused launch (fd_time_kernel.cuh: the intermediate
// stays in registers) where n_t <= 104, else the scaled forward launch into `mid` and the
// backward launch.  X -> Z; Z may equal X on the fused path only.
static int time_modes(ls_ctx* ctx, const double* X, double* mid, double* Z, uint64_t ncols, const double* lam_c) {
  if (ncols == 0) return LS_OK;
  if (ctx->fd_time && ft_bucket(ctx->nt) > 0) {
    FTArgs a{};
    a.X = X;
    a.Z = Z;
    a.U = ctx->Wb[3];
    a.lam_t = ctx->lam[3];
    a.lam_s = lam_c;
    a.nt = ctx->nt;
    a.ncols = uint32_t(ncols);
    a.ld = ncols;
    ls_ctx::ProfRec rec{};
    if (ctx->prof) {
      rec.a = ctx->get_event();
      rec.b = ctx->get_event();
      rec.flops = 4.0 * double(ctx->nt) * double(ctx->nt) * double(ncols);  // two n_t x n_t products
      cudaEventRecord(rec.a, ctx->stream);
    }
    const cudaError_t e = ft_launch(a, ctx->stream, ctx->num_sms);
    ctx->launches++;
    if (ctx->prof) {
      cudaEventRecord(rec.b, ctx->stream);
      ctx->prof_recs.push_back(rec);
    }
    LS_CUDA(e);
    return LS_OK;
  }
  LS_CHECK(launch_mode(ctx, X, mid, ctx->Wf[3], ctx->nt, 1, ncols, true, ctx->lam[3], lam_c));
  return launch_mode(ctx, mid, Z, ctx->Wb[3], ctx->nt, 1, ncols, false);
}

static int fd_core(ls_ctx* ctx, const double* r, double* z);

extern "C" int fd_apply(ls_ctx* ctx, const double* r, double* z) {
  if (!ctx || !r || !z || !aligned8(r) || !aligned8(z)) return LS_EINVAL;
  if (ctx->dm12) {
    // P^G = D^{1/2} Pbar^G D^{1/2}: z = D^{-1/2} Pbar^{-1} D^{-1/2} r (PAPER.md 1040-1045)
    double* rs = ctx->tmp[5];
    LS_CHECK(scale_vec(ctx->dm12, r, rs, ctx->Nl, ctx->stream, &ctx->launches));
    LS_CHECK(fd_core(ctx, rs, z));
    return scale_vec(ctx->dm12, z, z, ctx->Nl, ctx->stream, &ctx->launches);
  }
  return fd_core(ctx, r, z);
}

static int fd_core(ls_ctx* ctx, const double* r, double* z) {
  double* A = ctx->tmp[0];
  double* B = ctx->tmp[1];
  double* C = ctx->tmp[2];
  if (ctx->world == 1) {
    // F1: forward spatial modes r -> A ; F2: time fwd + scale (A -> B), time bwd (B -> C)
    LS_CHECK(spatial_modes(ctx, r, A, B, C, ctx->nt, true));
    LS_CHECK(time_modes(ctx, A, B, C, ctx->Ns, ctx->lam_s));
    // F3: backward spatial modes C -> z
    LS_CHECK(spatial_modes(ctx, C, z, A, B, ctx->nt, false));
    return LS_OK;
  }
  return comm_fd_apply(ctx, r, z);
}

// the three stages of fd_apply on caller-chosen pieces (what each rank of the distributed
// path runs between its all-to-alls; exposed for custom decompositions and for testing)
extern "C" int fd_apply_stage(ls_ctx* ctx, int stage, const double* in, double* out, int64_t a, int64_t b) {
  if (!ctx || !in || !out || in == out || !aligned8(in) || !aligned8(out)) return LS_EINVAL;
  if (ctx->geo) return LS_ENOTSUP;
  switch (stage) {
    case 0:
    case 2: {  // spatial modes (forward / backward) on `a` time slices [a][N_s]
      if (a < 1 || a > ctx->ntl) return LS_EINVAL;
      return spatial_modes(ctx, in, out, ctx->tmp[3], ctx->tmp[4], uint64_t(a), stage == 0);
    }
    case 1: {  // time mode U_t^T, /(lambda_t + Lambda_s), U_t on a chunk [n_t][b] at spatial offset a
      if (a < 0 || b < 1 || a + b > ctx->Ns || int64_t(ctx->nt) * b > (ctx->Nl + 2 * ctx->pt * ctx->Ns)) return LS_EINVAL;
      return time_modes(ctx, in, ctx->tmp[3], out, uint64_t(b), ctx->lam_s + a);
    }
    default: return LS_EINVAL;
  }
}

// ---- fused all-to-all pieces (register-direct kernel with peer-memory epilogues) ----------
// forward spatial modes 1..d-1 on `rows` slab slices, then mode d scattering its output
// straight into the owners' chunk buffers (plan.hpp a2a_fwd_dest).  Workspaces tmp[3], tmp[4].
static int spatial_fwd_scatter(ls_ctx* ctx, const double* in, uint64_t rows, double* const* peer, int world,
                               int me) {
  const int d = ctx->d;
  if (d < 2) return LS_ENOTSUP;
  const double* src = in;
  double* ws[2] = {ctx->tmp[3], ctx->tmp[4]};
  for (int k = 0; k < d - 1; ++k) {
    uint64_t Q = 1, P = rows;
    for (int j = 0; j < k; ++j) Q *= ctx->n[j];
    for (int j = k + 1; j < d; ++j) P *= ctx->n[j];
    if (use_cs(ctx, k))
      LS_CHECK(launch_mode(ctx, src, ws[k % 2], ctx->Wf_cs[k], ctx->n[k], P, Q, false, nullptr, nullptr, 1));
    else
      LS_CHECK(launch_mode(ctx, src, ws[k % 2], ctx->Wf[k], ctx->n[k], P, Q, false));
    src = ws[k % 2];
  }
  const int k = d - 1;
  uint64_t Q = 1;
  for (int j = 0; j < k; ++j) Q *= ctx->n[j];
  ModeArgs a{};
  a.X = src;
  a.Y = ctx->tmp[5];  // unused by the scattering epilogue (alignment probe only)
  const bool cs = use_cs(ctx, k);
  a.W = cs ? ctx->Wf_cs[k] : ctx->Wf[k];
  a.n = ctx->n[k];
  a.P = uint32_t(rows);
  a.Q = uint32_t(Q);
  a.ncols = uint32_t(rows * Q);
  a.y16 = true;
  a.remote = 1;
  a.peer = peer;
  a.world = world;
  a.me = me;
  a.nt_g = ctx->nt;
  a.Ns_g = ctx->Ns;
  return launch_mode_rd(ctx, a, false, false, cs ? 1 : 0);
}

// time mode of this rank's spatial chunk [n_t][chunk_ld(len)] (spatial offset c0): forward +
// scale locally into `mid`, backward scattering into the owners' slab buffers (a2a_bwd_dest)
static int time_chunk_scatter(ls_ctx* ctx, const double* chunk, int64_t c0, int64_t len, double* mid,
                              double* const* peer, int world, int me) {
  const int64_t ld = chunk_ld(len);
  ModeArgs a{};
  a.X = chunk;
  a.Y = mid;
  a.W = ctx->Wf[3];
  a.lam_a = ctx->lam[3];
  a.lam_c = ctx->lam_s + c0;
  a.n = ctx->nt;
  a.P = 1;
  a.Q = uint32_t(ld);
  a.ncols = uint32_t(len);
  a.y16 = (reinterpret_cast<uintptr_t>(mid) & 15) == 0;
  LS_CHECK(launch_mode_rd(ctx, a, false, true));
  ModeArgs b{};
  b.X = mid;
  b.Y = ctx->tmp[5];
  b.W = ctx->Wb[3];
  b.n = ctx->nt;
  b.P = 1;
  b.Q = uint32_t(ld);
  b.ncols = uint32_t(len);
  b.y16 = true;
  b.remote = 2;
  b.peer = peer;
  b.world = world;
  b.me = me;
  b.nt_g = ctx->nt;
  b.Ns_g = ctx->Ns;
  return launch_mode_rd(ctx, b, false, false);
}

extern "C" int fd_apply_scatter(ls_ctx* ctx, int stage, const double* in, int64_t a, int64_t b, int world, int me,
                                double* const* dst_host) {
  if (!ctx || !in || !dst_host || world < 1 || world > 64 || me < 0 || me >= world || !aligned8(in)) return LS_EINVAL;
  if (ctx->geo) return LS_ENOTSUP;
  if (ctx->d < 2) return LS_ENOTSUP;
  if (!ctx->scatter_tab) {
    LS_CHECK(ctx->alloc(reinterpret_cast<double**>(&ctx->scatter_tab), 64));
    LS_CUDA(cudaMallocHost(&ctx->scatter_stage, 64 * sizeof(double*)));
  }
  LS_CUDA(cudaStreamSynchronize(ctx->stream));  // the staging buffer is free
  for (int h = 0; h < world; ++h) {
    if (!dst_host[h]) return LS_EINVAL;
    ctx->scatter_stage[h] = dst_host[h];
  }
  LS_CUDA(cudaMemcpyAsync(ctx->scatter_tab, ctx->scatter_stage, world * sizeof(double*), cudaMemcpyHostToDevice,
                          ctx->stream));
  int64_t off, len;
  if (stage == 0) {
    split_part(ctx->nt, world, me, &off, &len);
    if (a != len || len < 1 || len > ctx->ntl) return LS_EINVAL;
    return spatial_fwd_scatter(ctx, in, uint64_t(a), ctx->scatter_tab, world, me);
  }
  if (stage == 1) {
    split_part(ctx->Ns, world, me, &off, &len);
    if (a != off || b != len || len < 1) return LS_EINVAL;
    return time_chunk_scatter(ctx, in, a, b, ctx->tmp[3], ctx->scatter_tab, world, me);
  }
  return LS_EINVAL;
}

// distributed fd_apply: slab -> all-to-all -> time mode on spatial chunks -> all-to-all -> slab
int comm_fd_apply(ls_ctx* ctx, const double* r, double* z) {
  Comm& cm = *ctx->comm;
  double* A = ctx->tmp[0];
  double* B = ctx->tmp[1];
  double* C = ctx->tmp[2];
  if (cm.fused) {
    // fused path: the all-to-alls are the epilogues of the last forward spatial mode and of
    // the backward time mode (stores into peer memory), each followed by a cross-GPU
    // barrier.  Receive buffers: B = tmp[1] (chunk), A = tmp[0] (slab); every workspace
    // written locally after a barrier (tmp[2..4]) is never a peer's destination.
    const int64_t c0 = cm.chunk_off[ctx->rank], len = cm.chunk_len[ctx->rank];
    // entry barrier: tmp[0] / tmp[1] are also ls_matvec workspaces, so no rank may scatter
    // into a peer's receive buffers before that peer has finished its previous call
    LS_CHECK(cm.barrier());
    LS_CHECK(spatial_fwd_scatter(ctx, r, uint64_t(ctx->ntl), cm.d_peer_chunk, ctx->world, ctx->rank));
    LS_CHECK(cm.barrier());
    if (len > 0) LS_CHECK(time_chunk_scatter(ctx, B, c0, len, C, cm.d_peer_slab, ctx->world, ctx->rank));
    LS_CHECK(cm.barrier());
    return spatial_modes(ctx, A, z, C, ctx->tmp[3], ctx->ntl, false);
  }
  // NCCL path, pipelined over pieces of consecutive time slices (plan.hpp a2a_piece_plan): the
  // exchange of piece c (comm stream) overlaps the spatial modes of piece c + 1 (compute stream),
  // and on the way back the unpack + backward spatial modes of piece c overlap the exchange of
  // piece c + 1.  A = slab [ntl][Ns], B = chunk [nt][chunk], C = packed staging; the spatial
  // modes of a piece use tmp[3], tmp[4].
  cudaStream_t cs = ctx->comm_stream;
  cudaEvent_t* ev = ctx->cev;  // 0: entry, 1: forward done, 2: time modes done, 3..6 forward pieces, 7..10 backward
  const int P = cm.pieces();
  const int64_t Ns = ctx->Ns, ntl = ctx->ntl;
  double* W0 = ctx->tmp[3];
  double* W1 = ctx->tmp[4];
  LS_CUDA(cudaEventRecord(ev[0], ctx->stream));  // the workspaces' previous users are done
  LS_CUDA(cudaStreamWaitEvent(cs, ev[0], 0));
  for (int c = 0; c < P; ++c) {
    int64_t a, l;
    split_part(ntl, P, c, &a, &l);
    if (l > 0) {
      LS_CHECK(spatial_modes(ctx, r + a * Ns, A + a * Ns, W0, W1, uint64_t(l), true));
      LS_CHECK(cm.pack_piece(true, A, C, c, ctx->stream, ctx->launches));
    }
    LS_CUDA(cudaEventRecord(ev[3 + c], ctx->stream));
    LS_CUDA(cudaStreamWaitEvent(cs, ev[3 + c], 0));
    LS_CHECK(cm.exchange_piece(true, C, B, c, cs));
  }
  LS_CUDA(cudaEventRecord(ev[1], cs));
  LS_CUDA(cudaStreamWaitEvent(ctx->stream, ev[1], 0));
  const int64_t chunk = cm.chunk_len[ctx->rank];
  const int64_t c0 = cm.chunk_off[ctx->rank];
  if (chunk > 0) {
    LS_CHECK(time_modes(ctx, B, C, B, uint64_t(chunk), ctx->lam_s + c0));
  }
  LS_CUDA(cudaEventRecord(ev[2], ctx->stream));
  LS_CUDA(cudaStreamWaitEvent(cs, ev[2], 0));
  for (int c = 0; c < P; ++c) {
    LS_CHECK(cm.exchange_piece(false, B, C, c, cs));
    LS_CUDA(cudaEventRecord(ev[7 + c], cs));
  }
  for (int c = 0; c < P; ++c) {
    int64_t a, l;
    split_part(ntl, P, c, &a, &l);
    LS_CUDA(cudaStreamWaitEvent(ctx->stream, ev[7 + c], 0));
    if (l == 0) continue;
    LS_CHECK(cm.pack_piece(false, C, A, c, ctx->stream, ctx->launches));
    LS_CHECK(spatial_modes(ctx, A + a * Ns, z + a * Ns, W0, W1, uint64_t(l), false));
  }
  return LS_OK;
}

// ------------------------------------------------------------------------------------------
// ls_matvec
// ------------------------------------------------------------------------------------------
static unsigned grid_for(uint64_t total, int threads, int num_sms) {
  uint64_t g = (total + threads - 1) / threads;
  return unsigned(std::min<uint64_t>(g, uint64_t(num_sms) * 16));
}

// ---- banded kernels (matvec_kernels.cuh): dispatch on p (template P) and row blocks RB
template <class Kern>
static int prepare_kernel(Kern k, size_t smem, int* occ, int threads = 256) {
  LS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  LS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, k, threads, smem));
  if (*occ < 1) *occ = 1;
  return LS_OK;
}

template <int P, int RB, int KIND, int NWARPS>
static int launch_tile(ls_ctx* ctx, BandArgs a) {
  using C = BandCfg<P, RB, KIND, 3, NWARPS>;
  static int occ = -1;
  if (occ < 0) LS_CHECK(prepare_kernel(band_tile_kernel<P, RB, KIND, 3, NWARPS>, C::SMEM, &occ, C::THREADS));
  a.ntiles = (a.ncols + C::BN - 1) / C::BN;
  if (a.ntiles == 0) return LS_OK;
  const unsigned grid = std::min<unsigned>(a.ntiles, unsigned(ctx->num_sms * occ));
  LS_CUDA(launch_pdl(band_tile_kernel<P, RB, KIND, 3, NWARPS>, grid, C::THREADS, C::SMEM, ctx->stream, a));
  ctx->launches++;
  LS_CUDA(cudaGetLastError());
  return LS_OK;
}

template <int P, int NMAX>
static int launch_first(ls_ctx* ctx, BandArgs a) {
  using C = FirstCfg<P, NMAX, 2>;
  static int occ = -1;
  if (occ < 0) LS_CHECK(prepare_kernel(band_first_kernel<P, NMAX, 2>, C::SMEM, &occ));
  a.ntiles = (a.ncols + C::BN - 1) / C::BN;
  if (a.ntiles == 0) return LS_OK;
  const unsigned grid = std::min<unsigned>(a.ntiles, unsigned(ctx->num_sms * occ));
  LS_CUDA(launch_pdl(band_first_kernel<P, NMAX, 2>, grid, 256, C::SMEM, ctx->stream, a));
  ctx->launches++;
  LS_CUDA(cudaGetLastError());
  return LS_OK;
}

// kind 0: direction 1 ; kind 1: directions >= 2 ; kind 2: time.  rows = output rows.
template <int P>
static int launch_band_p(ls_ctx* ctx, const BandArgs& a, int kind, int rows) {
  if (kind == 0) {
    if (a.n <= 32) return launch_first<P, 32>(ctx, a);
    if (a.n <= 72) return launch_first<P, 72>(ctx, a);
    if (a.n <= 104) return launch_first<P, 104>(ctx, a);
    return launch_first<P, 136>(ctx, a);
  }
  // (RB rows per warp, warps): rows covered = RB * NW >= rows; <= ~48 doubles of
  // accumulators + window per thread
#define LS_RB(R, NW)                                                                          \
  if (rows <= R * NW) return kind == 1 ? launch_tile<P, R, 1, NW>(ctx, a) : launch_tile<P, R, 2, NW>(ctx, a);
  LS_RB(2, 8) LS_RB(4, 8) LS_RB(8, 8) LS_RB(9, 8) LS_RB(13, 8) LS_RB(17, 8)
#undef LS_RB
  return LS_EINVAL;
}

static int launch_band(ls_ctx* ctx, const BandArgs& a, int kind, int rows) {
  switch (kind == 2 ? ctx->pt : ctx->p) {  // time kernel: p_t; direction kernels: p_s
    case 1: return kind == 2 ? launch_band_p<1>(ctx, a, kind, rows) : LS_ENOTSUP;
    case 2: return launch_band_p<2>(ctx, a, kind, rows);
    case 3: return launch_band_p<3>(ctx, a, kind, rows);
    case 4: return launch_band_p<4>(ctx, a, kind, rows);
    case 5: return launch_band_p<5>(ctx, a, kind, rows);
    case 6: return launch_band_p<6>(ctx, a, kind, rows);
    case 7: return launch_band_p<7>(ctx, a, kind, rows);
    case 8: return launch_band_p<8>(ctx, a, kind, rows);
    default: return LS_ENOTSUP;  // ls_matvec supports p <= 8 (BASELINE configs: p <= 8)
  }
}

// y = A x: spatial sum-factorisation on the `rows` time slices of x (global rows
// [s_first, s_first + rows), halo included), time part on global output rows
// [t_first, t_first + nout) written to y.
static int matvec_block(ls_ctx* ctx, const double* x, double* y, int64_t rows, int64_t s_first,
                        int64_t t_first, int64_t nout) {
  const int d = ctx->d;
  double* S[3] = {ctx->tmp[0], ctx->tmp[1], ctx->tmp[2]};
  double* T[3] = {ctx->tmp[3], ctx->tmp[4], ctx->tmp[5]};
  const uint64_t total = uint64_t(rows) * ctx->Ns;
  for (int k = 0; k < d; ++k) {
    BandArgs a{};
    uint64_t Q = 1;
    for (int j = 0; j < k; ++j) Q *= ctx->n[j];
    a.in[0] = (k == 0) ? x : S[0];
    a.in[1] = (k == 0) ? nullptr : S[1];
    a.in[2] = (k == 0) ? nullptr : S[2];
    for (int m = 0; m < 3; ++m) a.out[m] = T[m];
    a.band[0] = ctx->bM[k];
    a.band[1] = ctx->bK[k];
    a.band[2] = ctx->bJ[k];
    a.n = ctx->n[k];
    a.Q = uint32_t(Q);
    a.ncols = uint32_t(total / ctx->n[k]);
    LS_CHECK(launch_band(ctx, a, k == 0 ? 0 : 1, ctx->n[k]));
    std::swap(S, T);
  }
  // time: y = K_t S_M + M_t S_J + W_t S_K on global output rows [t_first, t_first + nout)
  BandArgs t{};
  t.in[0] = S[0];
  t.in[1] = S[2];
  t.in[2] = S[1];
  t.out[0] = y;
  t.band[0] = ctx->bMt;
  t.band[1] = ctx->bKt;
  t.band[2] = nullptr;
  t.n = ctx->nt;
  t.Q = uint32_t(ctx->Ns);
  t.ncols = uint32_t(ctx->Ns);
  t.t_first = int(t_first);
  t.s_first = int(s_first);
  t.s_rows = int(rows);
  t.nout = int(nout);
  return launch_band(ctx, t, 2, int(nout));
}

// ---- matvec v2 (matvec2_kernels.cuh) ---------------------------------------------------
static void mv_set(MVArgs& a, int slot, const ls_ctx::Split& sp) {
  for (int j = 0; j < MV_MAXW; ++j) a.st[slot][j] = j < int(sp.s.size()) ? sp.s[j] : 0.0;
  a.E[slot] = sp.E;
}

static int mv2_launch(ls_ctx* ctx, const double* x, double* y, int64_t rows, int64_t s_first,
                      int64_t t_first, int64_t nout) {
  const int d = ctx->d, P = ctx->p;
  if (P < 2 || P > 8 || ctx->pt < 2 || ctx->pt > 8) return LS_ENOTSUP;  // ls_matvec supports p <= 8 (BASELINE configs: p <= 8)
  double* Kx = ctx->tmp[0];
  double* Mx = ctx->tmp[1];
  double* A = ctx->tmp[2];
  double* B = ctx->tmp[3];
  double* C = ctx->tmp[4];
  MV2Plan pl{};
  pl.d = d;
  pl.stream = ctx->stream;
  pl.num_sms = ctx->num_sms;
  // time pass on all N_s columns
  {
    MVArgs& a = pl.time;
    mv_set(a, 0, ctx->tsplit.K);
    mv_set(a, 1, ctx->tsplit.M);
    a.r_lo = ctx->tsplit.lo;
    a.r_hi = ctx->tsplit.hi;
    a.in[0] = x;
    a.out[0] = Kx;
    a.out[1] = Mx;
    a.n = ctx->nt;
    a.ncols = uint32_t(ctx->Ns);
    a.t_first = int(t_first);
    a.s_first = int(s_first);
    a.s_rows = int(rows);
    a.nout = int(nout);
    pl.grid_time = nout > 0 ? unsigned((ctx->Ns + 31) / 32) : 0;
  }
  // direction d on [nout][n_d][Q]
  const int kd = d - 1;
  uint64_t Q = 1;
  for (int j = 0; j < kd; ++j) Q *= ctx->n[j];
  {
    MVArgs& a = pl.dir;
    const auto& sp = ctx->dsplit[kd];
    mv_set(a, 0, sp.M);
    mv_set(a, 1, sp.J);
    mv_set(a, 2, sp.K);
    mv_set(a, 3, sp.K2);
    a.r_lo = sp.lo;
    a.r_hi = sp.hi;
    a.in[0] = Kx;
    a.in[1] = Mx;
    a.out[0] = (d == 1) ? y : A;
    a.out[1] = B;
    a.out[2] = C;
    const int64_t tT = (ctx->nt - 1) - t_first;  // local output index of the last time slice
    const bool own_last = tT >= 0 && tT < nout;
    a.tT = own_last ? int(tT) : -1;
    a.xT = own_last ? x + (ctx->nt - 1 - s_first) * ctx->Ns : nullptr;
    a.n = ctx->n[kd];
    a.Q = uint32_t(Q);
    a.ncols = uint32_t(uint64_t(nout) * Q);
    pl.grid_dir = unsigned((a.ncols + 31) / 32);
  }
  // plane pass: directions d-1 .. 1
  if (d >= 2) {
    MVArgs& a = pl.plane;
    const auto& s1 = ctx->dsplit[0];
    mv_set(a, 4, s1.M);
    mv_set(a, 5, s1.J);
    mv_set(a, 6, s1.K);
    a.r_lo1 = s1.lo;
    a.r_hi1 = s1.hi;
    a.n1 = ctx->n[0];
    a.in[0] = A;
    a.in[1] = B;
    a.in[2] = C;
    a.out[0] = y;
    uint64_t items;
    if (d == 3) {
      const auto& s2 = ctx->dsplit[1];
      mv_set(a, 0, s2.M);
      mv_set(a, 1, s2.J);
      mv_set(a, 2, s2.K);
      mv_set(a, 3, s2.K2);
      a.r_lo = s2.lo;
      a.r_hi = s2.hi;
      a.n = ctx->n[1];
      a.ncols = uint32_t(nout * ctx->n[2]);  // planes
      items = uint64_t(a.ncols) * ((ctx->n[1] + MV_PLANE_ROWS - 1) / MV_PLANE_ROWS);
    } else {
      a.n = 1;
      a.ncols = uint32_t(nout * ctx->n[1]);  // rows of [rows][n1]
      items = (uint64_t(a.ncols) + MV_PLANE_ROWS - 1) / MV_PLANE_ROWS;
    }
    pl.smem_plane = size_t(3) * MV_PLANE_ROWS * mv_plane_pitch(ctx->n[0], P) * sizeof(double);
    const int per_sm = int(std::max<size_t>(1, std::min<size_t>(mv_plane_ctas(P), (227 * 1024) / pl.smem_plane)));
    pl.grid_plane = unsigned(std::min<uint64_t>(items, uint64_t(ctx->num_sms) * per_sm));
    // the register sweep (one warp per plane, CW columns per lane; P = 2 only)
    const int cw = std::max(2, (ctx->n[0] + 31) / 32);
    pl.sweep_cw = 0;
    if (d == 3 && P == 2 && ctx->mv2_sweep && cw <= 4) {
      pl.sweep_cw = cw;
      pl.grid_plane = unsigned(std::min<uint64_t>((uint64_t(a.ncols) + 7) / 8, uint64_t(ctx->num_sms)));
    }
  }
  LS_CUDA(mv2_run(P, ctx->pt, pl, &ctx->launches));
  return LS_OK;
}

// ---- matvec v3 (matvec3_kernels.cuh): DMMA band passes time -> d -> ... -> 1 ----------
static int mv3_launch(ls_ctx* ctx, const double* x, double* y, int64_t rows, int64_t s_first,
                      int64_t t_first, int64_t nout) {
  const int d = ctx->d, P = ctx->p, PT = ctx->pt;
  if (P < 2 || P > 8 || PT < 2 || PT > 8) return LS_ENOTSUP;
  double* Kx = ctx->tmp[0];
  double* Mx = ctx->tmp[1];
  double* A = ctx->tmp[2];
  double* B = ctx->tmp[3];
  double* C = ctx->tmp[4];
  MV3Pass ps[4];
  int np = 0;
  const int n1 = ctx->n[0], n1p = ctx->n1p;
  const int64_t Nsp = (ctx->Ns / n1) * n1p;  // padded slice
  const bool own_last_t = (ctx->nt - 1) - t_first >= 0 && (ctx->nt - 1) - t_first < nout;
  if (own_last_t && d >= 2)  // W_t term input in the padded layout
    LS_CUDA(mv3_pad_slice(x + (ctx->nt - 1 - s_first) * ctx->Ns, ctx->xT_pad, Nsp, n1, n1p, ctx->stream,
                          &ctx->launches));
  {  // time
    MV3Pass& q = ps[np++];
    q = MV3Pass{};
    q.kind = MV3_TIME;
    q.mode1 = false;
    MV3Args& a = q.args;
    a.frag = ctx->frag_time;
    a.in[0] = x;
    a.out[0] = Kx;
    a.out[1] = Mx;
    a.n = ctx->nt;
    a.mt = mv3_mt(PT, ctx->nt);
    a.Q = uint32_t(ctx->Ns);
    a.Qout = uint32_t(Nsp);
    a.ncols = uint32_t(Nsp);
    if (n1p != n1 && d >= 2) {
      a.map_n1 = n1;
      a.map_n1p = n1p;
    }
    a.s_first = int(s_first);
    a.s_rows = int(rows);
    a.t_first = int(t_first);
    a.nout = int(nout);
    const int S0 = mv3_s0(PT);  // m-tiles covering the output band rows [t_first, t_first + nout)
    a.mt0 = int((t_first - S0) / 8);
    a.mt1 = int((t_first + nout - S0 + 7) / 8);
  }
  const int kd = d - 1;
  uint64_t Q = 1;
  for (int j = 0; j < kd; ++j) Q *= (j == 0 ? n1p : ctx->n[j]);
  {  // direction d
    MV3Pass& q = ps[np++];
    q = MV3Pass{};
    q.kind = (d == 1) ? MV3_DIR_A : MV3_DIR;
    q.mode1 = (d == 1);
    MV3Args& a = q.args;
    a.frag = ctx->frag_dir[kd];
    a.in[0] = Kx;
    a.in[1] = Mx;
    a.out[0] = (d == 1) ? y : A;
    a.out[1] = B;
    a.out[2] = C;
    const int64_t tT = (ctx->nt - 1) - t_first;
    const bool own_last = tT >= 0 && tT < nout;
    a.tT = own_last ? int(tT) : -1;
    a.xT = own_last ? (d >= 2 ? ctx->xT_pad : x + (ctx->nt - 1 - s_first) * ctx->Ns) : nullptr;
    a.n = ctx->n[kd];
    a.mt = mv3_mt(P, a.n);
    a.Q = uint32_t(Q);
    a.ncols = uint32_t(uint64_t(nout) * Q);
    a.mt0 = 0;
    a.mt1 = a.mt;
    a.in_fiber = a.out_fiber = a.n;  // d = 1 (contiguous, unpadded)
  }
  const double* cur[3] = {A, B, C};
  if (d == 3) {  // direction 2: (A, B, C) -> (A2, B2, C2) in Kx, Mx, tmp[5]
    MV3Pass& q = ps[np++];
    q = MV3Pass{};
    q.kind = MV3_MID;
    q.mode1 = false;
    MV3Args& a = q.args;
    a.frag = ctx->frag_dir[1];
    for (int m = 0; m < 3; ++m) a.in[m] = cur[m];
    a.out[0] = Kx;
    a.out[1] = Mx;
    a.out[2] = ctx->tmp[5];
    a.n = ctx->n[1];
    a.mt = mv3_mt(P, a.n);
    a.Q = uint32_t(n1p);
    a.ncols = uint32_t(uint64_t(nout) * ctx->n[2] * n1p);
    a.tT = -1;
    a.mt0 = 0;
    a.mt1 = a.mt;
    cur[0] = Kx;
    cur[1] = Mx;
    cur[2] = ctx->tmp[5];
  }
  if (d >= 2) {  // direction 1: y = M A + J B + K C
    MV3Pass& q = ps[np++];
    q = MV3Pass{};
    q.kind = MV3_LAST;
    q.mode1 = true;
    MV3Args& a = q.args;
    a.frag = ctx->frag_dir[0];
    for (int m = 0; m < 3; ++m) a.in[m] = cur[m];
    a.out[0] = y;
    a.n = ctx->n[0];
    a.mt = mv3_mt(P, a.n);
    a.Q = 1;
    a.ncols = uint32_t(uint64_t(nout) * (ctx->Ns / ctx->n[0]));
    a.in_fiber = n1p;   // padded intermediates
    a.out_fiber = n1;   // y in the caller's layout
    a.tT = -1;
    a.mt0 = 0;
    a.mt1 = a.mt;
  }
  for (int i = 0; i < np; ++i) ps[i].p = (ps[i].kind == MV3_TIME) ? PT : P;
  LS_CUDA(mv3_run(ps, np, ctx->num_sms, ctx->stream, &ctx->launches));
  return LS_OK;
}

// ---- matvec v4 (mv4_kernels.cuh): plane pass (directions 1 + 2) -> direction 3 -> time ------
// MV4Split: the input rows in three pieces (distributed ls_matvec without the copy into the
// halo-extended buffer): own rows [lo, lo + own) from `x`, halo rows [0, lo) from x_lo and
// [lo + own, rows) from x_hi; the plane pass of the own rows runs first, the halo rows after
// halo_ready (the exchange overlaps it)
struct MV4Split {
  const double* x_lo = nullptr;
  const double* x_hi = nullptr;
  int64_t lo = 0, own = 0, hi = 0;
  cudaEvent_t halo_ready = nullptr;
};

static int mv4_launch(ls_ctx* ctx, const double* x, double* y, int64_t rows, int64_t s_first,
                      int64_t t_first, int64_t nout, const MV4Split* split = nullptr) {
  const int d = ctx->d, P = ctx->p, PT = ctx->pt;
  if (d < 2 || P < 2 || P > 8 || PT < 2 || PT > 8) return LS_ENOTSUP;
  const int n1 = ctx->n[0], n2 = ctx->n[1];
  double *PM = ctx->tmp[0], *PK = ctx->tmp[1], *PJ = ctx->tmp[2];
  const int cw4 = std::max(P, (n1 + 31) / 32);
  const bool sweep = ctx->mv4_sweep && d == 3 && (P == 3 || P == 4) && cw4 <= 4;
  auto plane = [&](const double* src, int64_t row0, int64_t nrows) -> int {
    if (nrows <= 0) return LS_OK;
    if (sweep) {  // DFMA register sweep (matvec2_kernels.cuh mv4_sweep_kernel)
      MVArgs s{};
      const auto& s2 = ctx->dsplit[1];
      const auto& s1 = ctx->dsplit[0];
      mv_set(s, 0, s2.M);
      mv_set(s, 1, s2.J);
      mv_set(s, 2, s2.K);
      mv_set(s, 4, s1.M);
      mv_set(s, 5, s1.J);
      mv_set(s, 6, s1.K);
      s.r_lo = s2.lo;
      s.r_hi = s2.hi;
      s.r_lo1 = s1.lo;
      s.r_hi1 = s1.hi;
      s.in[0] = src;
      s.out[0] = PM + row0 * ctx->Ns;
      s.out[1] = PK + row0 * ctx->Ns;
      s.out[2] = PJ + row0 * ctx->Ns;
      s.n = n2;
      s.n1 = n1;
      s.ncols = uint32_t(nrows * ctx->n[2]);
      LS_CUDA(mv4_sweep_run(s, P, cw4, ctx->num_sms, ctx->stream));
      ctx->launches++;
      return LS_OK;
    }
    MV4PlaneArgs a{};
    a.x = src;
    a.out[0] = PM + row0 * ctx->Ns;
    a.out[1] = PK + row0 * ctx->Ns;
    a.out[2] = PJ + row0 * ctx->Ns;
    a.frag1 = ctx->frag_dir[0];
    a.frag2 = ctx->frag_dir[1];
    a.n1 = n1;
    a.n2 = n2;
    a.mt1 = mv3_mt(P, n1);
    a.mt2 = mv3_mt(P, n2);
    a.nplanes = nrows * (d == 3 ? ctx->n[2] : 1);
    LS_CUDA(mv4_plane_run(a, P, ctx->num_sms, ctx->stream));
    ctx->launches++;
    return LS_OK;
  };
  // p.q (fused dot): p = the own rows of x
  const double* xown = split ? x : x + (t_first - s_first) * ctx->Ns;
  if (!split) {
    LS_CHECK(plane(x, 0, rows));
  } else {
    LS_CHECK(plane(x, split->lo, split->own));
    if (split->halo_ready) LS_CUDA(cudaStreamWaitEvent(ctx->stream, split->halo_ready, 0));
    LS_CHECK(plane(split->x_lo, 0, split->lo));
    LS_CHECK(plane(split->x_hi, split->lo + split->own, split->hi));
  }
  // v5 measured (tools/ab_mv.py, r02): config 3 (p = 3) 0.720 -> 0.610 ms, config 5 p = 4 2.945 ->
  // 2.924 ms; slower at p = 6 (config 4 10.08 -> 13.04 ms) and 8 (3.69 -> 5.18 ms): 255 registers
  // (the 2p+1-row ring) and 8 warps per SM leave its latency exposed
  const bool mv5 = ctx->mv5 == 1 || (ctx->mv5 == 2 && P <= 4);
  if (d == 3 && mv5 && mv5_supported(P, PT) && ctx->tcol) {
    // v5: direction 3 and time in one pass (mv5_kernels.cuh), v1 / v2 stay on chip
    MV5Args a{};
    a.in[0] = PM;
    a.in[1] = PK;
    a.in[2] = PJ;
    a.y = y;
    a.frag3 = ctx->frag_dir[2];
    a.tcol = ctx->tcol;
    a.n3 = ctx->n[2];
    a.mt3 = mv3_mt(P, a.n3);
    a.nt = ctx->nt;
    a.Q = uint32_t(int64_t(n1) * n2);
    a.s_first = int(s_first);
    a.rows = int(rows);
    a.t_first = int(t_first);
    a.nout = int(nout);
    if (ctx->fuse_dot_slot >= 0) {  // p.q in the epilogue: p = the own rows of x
      a.dotp = xown;
      a.dot_part = ctx->partials;
    }
    unsigned grid = 0;
    LS_CUDA(mv5_run(a, P, PT, ctx->num_sms, ctx->stream, &grid));
    ctx->launches++;
    if (ctx->fuse_dot_slot >= 0) {
      LS_CUDA(launch_pdl(reduce_final_kernel, 1, RED_THREADS, 0, ctx->stream, ctx->partials, int(grid), ctx->scal,
                         ctx->fuse_dot_slot));
      ctx->launches++;
      LS_CUDA(cudaGetLastError());
      if (ctx->world > 1) LS_CHECK(ctx->comm->allreduce_scalar(ctx->scal + ctx->fuse_dot_slot));
      ctx->fuse_dot_done = true;
    }
    return LS_OK;
  }
  const int64_t tT = (ctx->nt - 1) - s_first;  // the last time slice among the stored rows
  const bool have_last = tT >= 0 && tT < rows;
  const double *v1 = PM, *v2 = PJ, *v3 = have_last ? PK + tT * ctx->Ns : nullptr;
  if (ctx->mv6 == 1) {
    // v6: the same two passes as DFMA Toeplitz stencils (matvec6_kernels.cuh)
    if (d == 3) {
      MV6Args a{};
      const auto& sp = ctx->dsplit[2];
      mv_set(a.m, 0, sp.M);
      mv_set(a.m, 1, sp.J);
      mv_set(a.m, 2, sp.K);
      mv_set(a.m, 3, sp.K2);
      a.m.r_lo = sp.lo;
      a.m.r_hi = sp.hi;
      a.m.in[0] = PM;
      a.m.in[1] = PK;
      a.m.in[2] = PJ;
      a.m.out[0] = ctx->tmp[3];
      a.m.out[1] = ctx->tmp[4];
      a.m.n = ctx->n[2];
      a.Q = uint32_t(int64_t(n1) * n2);
      a.rows = int(rows);
      a.tT = have_last ? int(tT) : -1;
      a.L = ctx->xT_pad;
      LS_CUDA(mv6_run_d3(a, P, ctx->num_sms, ctx->stream));
      ctx->launches++;
      v1 = ctx->tmp[3];
      v2 = ctx->tmp[4];
      v3 = have_last ? ctx->xT_pad : nullptr;
    }
    MV6Args b{};
    mv_set(b.m, 0, ctx->tsplit.K);
    mv_set(b.m, 1, ctx->tsplit.M);
    b.m.r_lo = ctx->tsplit.lo;
    b.m.r_hi = ctx->tsplit.hi;
    b.m.in[0] = v1;
    b.m.in[1] = v2;
    b.m.xT = v3;
    b.m.out[0] = y;
    b.m.n = ctx->nt;
    b.m.t_first = int(t_first);
    b.m.s_first = int(s_first);
    b.m.s_rows = int(rows);
    b.m.nout = int(nout);
    b.Q = uint32_t(ctx->Ns);
    if (ctx->fuse_dot_slot >= 0) {  // p.q in the epilogue: p = the own rows of x
      b.dotp = xown;
      b.dot_part = ctx->partials;
    }
    unsigned grid = 0;
    LS_CUDA(mv6_run_time(b, PT, ctx->num_sms, ctx->stream, &grid));
    ctx->launches++;
    if (ctx->fuse_dot_slot >= 0) {
      LS_CUDA(launch_pdl(reduce_final_kernel, 1, RED_THREADS, 0, ctx->stream, ctx->partials, int(grid), ctx->scal,
                         ctx->fuse_dot_slot));
      ctx->launches++;
      LS_CUDA(cudaGetLastError());
      if (ctx->world > 1) LS_CHECK(ctx->comm->allreduce_scalar(ctx->scal + ctx->fuse_dot_slot));
      ctx->fuse_dot_done = true;
    }
    return LS_OK;
  }
  MV3Pass ps[2];
  int np = 0;
  if (d == 3) {  // direction 3: (P_M, P_K, P_J) -> v1, v2 (+ v3 on the last slice)
    MV3Pass& q = ps[np++];
    q = MV3Pass{};
    q.kind = MV3_D3;
    q.mode1 = false;
    q.p = P;
    MV3Args& a = q.args;
    a.frag = ctx->frag_dir[2];
    a.in[0] = PM;
    a.in[1] = PK;
    a.in[2] = PJ;
    a.out[0] = ctx->tmp[3];
    a.out[1] = ctx->tmp[4];
    a.v3 = ctx->xT_pad;
    a.tT = have_last ? int(tT) : -1;
    a.n = ctx->n[2];
    a.mt = mv3_mt(P, a.n);
    a.Q = uint32_t(int64_t(n1) * n2);
    a.ncols = uint32_t(rows * a.Q);
    a.mt0 = 0;
    a.mt1 = a.mt;
    v1 = ctx->tmp[3];
    v2 = ctx->tmp[4];
    v3 = have_last ? ctx->xT_pad : nullptr;
  }
  {  // time: y = K_t v1 + M_t v2 + W_t v3 on the output rows [t_first, t_first + nout)
    MV3Pass& q = ps[np++];
    q = MV3Pass{};
    q.kind = MV3_T2;
    q.mode1 = false;
    q.p = PT;
    MV3Args& a = q.args;
    a.frag = ctx->frag_time;
    a.in[0] = v1;
    a.in[1] = v2;
    a.v3 = const_cast<double*>(v3);
    a.out[0] = y;
    a.n = ctx->nt;
    a.mt = mv3_mt(PT, ctx->nt);
    a.Q = uint32_t(ctx->Ns);
    a.ncols = uint32_t(ctx->Ns);
    a.tT = -1;
    a.s_first = int(s_first);
    a.s_rows = int(rows);
    a.t_first = int(t_first);
    a.nout = int(nout);
    const int S0 = mv3_s0(PT);
    a.mt0 = int((t_first - S0) / 8);
    a.mt1 = int((t_first + nout - S0 + 7) / 8);
    if (ctx->fuse_dot_slot >= 0) {  // p.q in the epilogue: p = the own rows of x
      a.dotp = xown;
      a.dot_part = ctx->partials;
    }
  }
  LS_CUDA(mv3_run(ps, np, ctx->num_sms, ctx->stream, &ctx->launches));
  if (ctx->fuse_dot_slot >= 0) {
    LS_CUDA(launch_pdl(reduce_final_kernel, 1, RED_THREADS, 0, ctx->stream, ctx->partials, int(ps[np - 1].grid),
                       ctx->scal, ctx->fuse_dot_slot));
    ctx->launches++;
    LS_CUDA(cudaGetLastError());
    if (ctx->world > 1) LS_CHECK(ctx->comm->allreduce_scalar(ctx->scal + ctx->fuse_dot_slot));
    ctx->fuse_dot_done = true;
  }
  return LS_OK;
}

static int matvec_any(ls_ctx* ctx, const double* x, double* y, int64_t rows, int64_t s_first,
                      int64_t t_first, int64_t nout) {
  // auto (measured, tools/mv_variants.py, r01):
  //   p = 2:  v2 (config 5 p=2: 2.74 ms vs v1 3.07, v3 3.30)
  //   p = 3: v1 (config 3: 0.81 ms vs v3 1.06, v2 1.16)
  //   p >= 4: v3, DMMA band passes (config 4: 12.0 ms vs v1 16.4; config 5 p=8: 5.04 vs 6.49,
  //           p=4: 3.96 vs 4.08)
  //   (v2 / v3 have time passes for p_t >= 2 only; p_t = 1 runs v1)
  // r02 (tools/mv_variants.py, L2 flushed): v4 (plane pass first) for d >= 2, p >= 3: config 4
  //   10.1 ms (v3 11.5), config 5 p = 8 / 4: 3.70 / 2.95 ms (v3 3.95 / 3.33), config 3: 0.73 ms
  //   (v1 0.75); p = 2 stays on v2 (config 5 p = 2: 2.18 ms vs v4 2.55)
  if (ctx->mv_variant == 4 ||
      (ctx->mv_variant == 0 && ctx->d >= 2 && ctx->p >= 3 && ctx->pt >= 2 && ctx->p <= 8 && ctx->pt <= 8))
    return mv4_launch(ctx, x, y, rows, s_first, t_first, nout);
  if (ctx->mv_variant == 3 || (ctx->mv_variant == 0 && ctx->p >= 4 && ctx->pt >= 2))
    return mv3_launch(ctx, x, y, rows, s_first, t_first, nout);
  const bool v2 = ctx->mv_variant == 2 || (ctx->mv_variant == 0 && ctx->p == 2 && ctx->pt >= 2);
  if (!v2) return matvec_block(ctx, x, y, rows, s_first, t_first, nout);
  return mv2_launch(ctx, x, y, rows, s_first, t_first, nout);
}

// extended-slab geometry of this rank (halo rows of the time factors)
static void ext_geom(const ls_ctx* ctx, int64_t* lo, int64_t* hi) {
  int64_t t0, ntl;
  halo_plan(ctx->nt, ctx->world, ctx->rank, ctx->pt, &t0, &ntl, lo, hi);
}

extern "C" int ls_matvec(ls_ctx* ctx, const double* x, double* y) {
  if (!ctx || !x || !y || x == y || !aligned8(x) || !aligned8(y)) return LS_EINVAL;
  if (ctx->geo && ctx->world == 1)
    return geo_matvec(*ctx->geo, ctx->bKt, ctx->bMt, ctx->nt, x, 0, 0, ctx->nt, y, ctx->tmp[3], ctx->tmp[4],
                      ctx->stream, &ctx->launches);
  if (ctx->world == 1) return matvec_any(ctx, x, y, ctx->nt, 0, 0, ctx->nt);
  int64_t lo, hi;
  ext_geom(ctx, &lo, &hi);
  double* own = ctx->pp + lo * ctx->Ns;  // extended buffer [lo | own | hi]
  const bool v4 = !ctx->geo && (ctx->mv_variant == 4 || (ctx->mv_variant == 0 && ctx->d >= 2 && ctx->p >= 3 &&
                                                          ctx->pt >= 2 && ctx->p <= 8 && ctx->pt <= 8));
  if (v4) {
    // no copy of x: the halos arrive in pp's halo rows (comm stream) while the plane pass of the
    // own rows runs; the halo rows' plane pass waits for them
    LS_CUDA(cudaEventRecord(ctx->cev[0], ctx->stream));
    LS_CUDA(cudaStreamWaitEvent(ctx->comm_stream, ctx->cev[0], 0));
    LS_CHECK(ctx->comm->halo_exchange_from(x, ctx->pp, ctx->pt, ctx->comm_stream));
    LS_CUDA(cudaEventRecord(ctx->cev[11], ctx->comm_stream));
    MV4Split sp;
    sp.x_lo = ctx->pp;
    sp.x_hi = own + ctx->ntl * ctx->Ns;
    sp.lo = lo;
    sp.own = ctx->ntl;
    sp.hi = hi;
    sp.halo_ready = ctx->cev[11];
    return mv4_launch(ctx, x, y, lo + ctx->ntl + hi, ctx->t0 - lo, ctx->t0, ctx->ntl, &sp);
  }
  if (x != own)
    LS_CUDA(cudaMemcpyAsync(own, x, size_t(ctx->Nl) * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  LS_CHECK(ctx->comm->halo_exchange(ctx->pp, ctx->pt));
  if (ctx->geo)  // mapped domain: slab-local time band + stencil pass (the spatial factors are replicated)
    return geo_matvec(*ctx->geo, ctx->bKt, ctx->bMt, ctx->nt, ctx->pp, int(ctx->t0 - lo), int(ctx->t0),
                      int(ctx->ntl), y, ctx->tmp[3], ctx->tmp[4], ctx->stream, &ctx->launches);
  return matvec_any(ctx, ctx->pp, y, lo + ctx->ntl + hi, ctx->t0 - lo, ctx->t0, ctx->ntl);
}

extern "C" int ls_matvec_slab(ls_ctx* ctx, const double* x_ext, int64_t s_first, int64_t s_rows,
                              double* y, int64_t t_first, int64_t nout) {
  if (!ctx || !x_ext || !y || !aligned8(x_ext) || !aligned8(y)) return LS_EINVAL;
  const int64_t nt = ctx->nt, p = ctx->pt;  // the time band
  if (nout < 0 || t_first < 0 || t_first + nout > nt || s_rows < 0) return LS_EINVAL;
  if (nout > ctx->ntl) return LS_EINVAL;  // workspaces hold ntl (+ halo) slices
  // the stored rows must cover the time band of every output row (clipped to [0, n_t))
  const int64_t need_lo = std::max<int64_t>(0, t_first - p), need_hi = std::min<int64_t>(nt, t_first + nout + p);
  if (nout > 0 && (s_first > need_lo || s_first + s_rows < need_hi)) return LS_EINVAL;
  if (s_rows > ctx->ntl + 2 * p) return LS_EINVAL;
  if (nout == 0) return LS_OK;
  if (ctx->geo)
    return geo_matvec(*ctx->geo, ctx->bKt, ctx->bMt, int(nt), x_ext, int(s_first), int(t_first), int(nout), y,
                      ctx->tmp[3], ctx->tmp[4], ctx->stream, &ctx->launches);
  return matvec_any(ctx, x_ext, y, s_rows, s_first, t_first, nout);
}

extern "C" int ls_matvec_slab3(ls_ctx* ctx, const double* x_lo, int64_t lo, const double* x_own, int64_t own,
                               const double* x_hi, int64_t hi, int64_t s_first, double* y, int64_t t_first,
                               int64_t nout) {
  if (!ctx || !x_own || !y || lo < 0 || hi < 0 || own < 1 || (lo > 0 && !x_lo) || (hi > 0 && !x_hi)) return LS_EINVAL;
  if (!aligned8(x_own) || !aligned8(y) || (x_lo && !aligned8(x_lo)) || (x_hi && !aligned8(x_hi))) return LS_EINVAL;
  const int64_t nt = ctx->nt, p = ctx->pt, rows = lo + own + hi;
  if (nout < 0 || t_first < 0 || t_first + nout > nt) return LS_EINVAL;
  if (nout > ctx->ntl || rows > ctx->ntl + 2 * p) return LS_EINVAL;
  const int64_t need_lo = std::max<int64_t>(0, t_first - p), need_hi = std::min<int64_t>(nt, t_first + nout + p);
  if (nout > 0 && (s_first > need_lo || s_first + rows < need_hi)) return LS_EINVAL;
  if (nout == 0) return LS_OK;
  const bool v4 = !ctx->geo && (ctx->mv_variant == 4 || (ctx->mv_variant == 0 && ctx->d >= 2 && ctx->p >= 3 &&
                                                          ctx->pt >= 2 && ctx->p <= 8 && ctx->pt <= 8));
  if (v4) {
    MV4Split sp;
    sp.x_lo = x_lo;
    sp.x_hi = x_hi;
    sp.lo = lo;
    sp.own = own;
    sp.hi = hi;
    return mv4_launch(ctx, x_own, y, rows, s_first, t_first, nout, &sp);
  }
  // other paths read one contiguous [rows][N_s] block: gather it into pp
  const size_t rb = size_t(ctx->Ns) * sizeof(double);
  double* ext = ctx->pp;
  if (lo > 0) LS_CUDA(cudaMemcpyAsync(ext, x_lo, lo * rb, cudaMemcpyDeviceToDevice, ctx->stream));
  LS_CUDA(cudaMemcpyAsync(ext + lo * ctx->Ns, x_own, own * rb, cudaMemcpyDeviceToDevice, ctx->stream));
  if (hi > 0) LS_CUDA(cudaMemcpyAsync(ext + (lo + own) * ctx->Ns, x_hi, hi * rb, cudaMemcpyDeviceToDevice, ctx->stream));
  return ls_matvec_slab(ctx, ext, s_first, rows, y, t_first, nout);
}

// ------------------------------------------------------------------------------------------
// ls_rhs (PAPER.md 409; reading c11)
// ------------------------------------------------------------------------------------------
extern "C" int ls_rhs(ls_ctx* ctx, int kind, double* b) {
  if (!ctx || !b || !aligned8(b)) return LS_EINVAL;
  if (ctx->geo) {
    // mapped domains: kind 2 = the 2D quarter-annulus benchmark u = P(x, y) sin(pi t) of
    // PAPER.md 1128-1129 (d = 2); kind 3 = the rotated quarter annulus' f = (P - Lap P) sin z of
    // PAPER.md 1219-1221 with homogeneous data (d = 3, reading c23);
    // b = sum_m G1_m (x) S0_m - G0_m (x) S2_m (geo_rhs_kernel)
    if (kind != 2 && kind != 3) return LS_ENOTSUP;
    LS_CHECK(geo_load(*ctx->geo, *ctx->gmap, ctx->n_el, kind, ctx->stream, &ctx->launches));
    const int nt = ctx->nt, d = ctx->d;
    std::vector<double> G(4 * size_t(nt), 0.0), i0, i1, i2;
    const double pi = 3.14159265358979323846;
    if (kind == 2) {
      load_integrals(int(ctx->n_el[d]), ctx->pt, false, 3, 0.0, i0, i1, i2);  // cos(pi t)
      for (int t = 0; t < nt; ++t) {
        G[t] = pi * i0[t];       // G0_1 = int pi cos(pi t) b_t
        G[nt + t] = pi * i1[t];  // G1_1 = int pi cos(pi t) b_t'
      }
      load_integrals(int(ctx->n_el[d]), ctx->pt, false, 0, 0.0, i0, i1, i2);  // sin(pi t)
      for (int t = 0; t < nt; ++t) {
        G[2 * nt + t] = i0[t];
        G[3 * nt + t] = i1[t];
      }
    } else {
      load_integrals(int(ctx->n_el[d]), ctx->pt, false, 4, 0.0, i0, i1, i2);  // g = 1
      for (int t = 0; t < nt; ++t) {
        G[t] = i0[t];
        G[nt + t] = i1[t];
      }
    }
    LS_CUDA(cudaMemcpyAsync(ctx->rhs_buf, G.data(), G.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    LS_CHECK(geo_rhs(*ctx->geo, ctx->rhs_buf, b, int(ctx->t0), int(ctx->ntl), nt, ctx->stream, &ctx->launches));
    LS_CUDA(cudaStreamSynchronize(ctx->stream));  // G goes out of scope
    return LS_OK;
  }
  if (kind != 0 && kind != 1) return LS_EINVAL;
  const int d = ctx->d;
  std::vector<double> stack(6 * NMAX_STACK, 0.0);  // S0[3], S2[3] ... G0, G1 stacked
  std::vector<double> i0, i1, i2;
  for (int k = 0; k < d; ++k) {
    load_integrals(int(ctx->n_el[k]), ctx->p, true, 0, 0.0, i0, i1, i2);
    std::copy(i0.begin(), i0.end(), stack.begin() + k * NMAX_STACK);
    std::copy(i2.begin(), i2.end(), stack.begin() + (3 + k) * NMAX_STACK);
  }
  const double pi = 3.14159265358979323846;
  load_integrals(int(ctx->n_el[d]), ctx->pt, false, kind == 0 ? 1 : 2, d * pi * pi, i0, i1, i2);
  std::vector<double> G(2 * NMAX_STACK, 0.0);
  std::copy(i0.begin(), i0.end(), G.begin());
  std::copy(i1.begin(), i1.end(), G.begin() + NMAX_STACK);
  // device buffer: [S0 x3 | S2 x3] then G0, G1 reuse a second region
  double* dS = ctx->rhs_buf;
  LS_CUDA(cudaMemcpyAsync(dS, stack.data(), stack.size() * sizeof(double), cudaMemcpyHostToDevice,
                          ctx->stream));
  // G0/G1 are staged in the partials buffer tail (RED_BLOCKS >= 2*NMAX_STACK)
  double* dG = ctx->partials;
  LS_CUDA(cudaMemcpyAsync(dG, G.data(), G.size() * sizeof(double), cudaMemcpyHostToDevice,
                          ctx->stream));
  const uint64_t total = uint64_t(ctx->Nl);
  rhs_outer_kernel<<<grid_for(total, 256, ctx->num_sms), 256, 0, ctx->stream>>>(
      b, dG, dG + NMAX_STACK, dS, dS + 3 * NMAX_STACK, d, ctx->n[0], ctx->n[1], ctx->n[2],
      uint64_t(ctx->Ns), total, uint64_t(ctx->t0));
  ctx->launches++;
  LS_CUDA(cudaGetLastError());
  LS_CUDA(cudaStreamSynchronize(ctx->stream));  // host vectors go out of scope
  return LS_OK;
}

// ------------------------------------------------------------------------------------------
// PCG
// ------------------------------------------------------------------------------------------
static int dot(ls_ctx* ctx, const double* a, const double* b, int slot) {
  LS_CUDA(launch_pdl(dot_partial_kernel, RED_BLOCKS, RED_THREADS, 0, ctx->stream, a, b, uint64_t(ctx->Nl),
                     ctx->partials));
  LS_CUDA(launch_pdl(reduce_final_kernel, 1, RED_THREADS, 0, ctx->stream, ctx->partials, int(RED_BLOCKS), ctx->scal,
                     slot));
  ctx->launches += 2;
  LS_CUDA(cudaGetLastError());
  if (ctx->world > 1) LS_CHECK(ctx->comm->allreduce_scalar(ctx->scal + slot));
  return LS_OK;
}

// q = A p and scal[slot] = p.q: fused into the matvec's last pass when the v4 path runs,
// otherwise ls_matvec + dot
static int matvec_dot(ls_ctx* ctx, const double* p, double* q, int slot) {
  ctx->fuse_dot_slot = (ctx->geo || !ctx->pq_fuse) ? -1 : slot;
  ctx->fuse_dot_done = false;
  const int rc = ls_matvec(ctx, p, q);
  ctx->fuse_dot_slot = -1;
  if (rc != LS_OK) return rc;
  if (ctx->fuse_dot_done) return LS_OK;
  return dot(ctx, p, q, slot);
}

static int read_scal(ls_ctx* ctx) {
  LS_CUDA(cudaMemcpyAsync(ctx->h_scal, ctx->scal, S_NSLOT * sizeof(double), cudaMemcpyDeviceToHost,
                          ctx->stream));
  LS_CUDA(cudaStreamSynchronize(ctx->stream));
  return LS_OK;
}

// The whole single-GPU solve after the b.b test as ONE graph launch (reading c7 order):
//   r = b; z = P r; rho0 = r.z; p = z; q = A p; pq; x += a p, r -= a q; rr; k = 1, test
//   WHILE (test fails): z = P r; rho1 = r.z; p = z + (rho1/rho0) p; rho0 = rho1; q = A p; pq;
//                       x += a p, r -= a q; rr; k += 1, test
//   true residual: z = b - A x; z.z
// The stopping test runs on the device (pcg_check_kernel sets the WHILE condition), so no
// per-iteration host round trip (config 2 is launch / latency bound).  The
// captured kernels and their order are those of the host loop: iterates are bit-identical.
static int pcg_build_graph(ls_ctx* ctx, const double* b, double* x, double tol, int max_iter) {
  if (ctx->pcg_exec) {
    cudaGraphExecDestroy(ctx->pcg_exec);
    ctx->pcg_exec = nullptr;
  }
  if (!ctx->cap_stream) LS_CUDA(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
  if (!ctx->cap_stream2) LS_CUDA(cudaStreamCreateWithFlags(&ctx->cap_stream2, cudaStreamNonBlocking));
  cudaGraph_t g = nullptr;
  LS_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  LS_CUDA(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault));
  cudaStream_t user = ctx->stream;
  const int64_t l0 = ctx->launches;
  const size_t bytes = size_t(ctx->Nl) * sizeof(double);
  double *r = ctx->pr, *z = ctx->pz, *p = ctx->pp, *q = ctx->pq;
  const unsigned gb = RED_BLOCKS;
  int rc = LS_OK;
  auto ck = [&](cudaError_t e) {
    if (rc == LS_OK && e != cudaSuccess) rc = LS_ECUDA;
  };
  // the iteration tail shared by the first iteration and the loop body
  auto tail = [&]() {
    if (rc == LS_OK) rc = matvec_dot(ctx, p, q, S_PQ);
    if (rc != LS_OK) return;
    ck(launch_pdl(update_xr_kernel, gb, RED_THREADS, 0, ctx->stream, x, r, p, q, uint64_t(ctx->Nl), ctx->scal,
                  int(S_RHO0), ctx->partials));
    ck(launch_pdl(reduce_final_kernel, 1, RED_THREADS, 0, ctx->stream, ctx->partials, int(RED_BLOCKS), ctx->scal,
                  int(S_RR)));
    ck(launch_pdl(pcg_check_kernel, 1, 1, 0, ctx->stream, ctx->scal, tol, max_iter, h));
    ctx->launches += 3;
  };
  ctx->stream = ctx->cap_stream;
  ck(cudaStreamBeginCaptureToGraph(ctx->stream, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  const bool capturing = rc == LS_OK;
  // first iteration
  ck(cudaMemcpyAsync(r, b, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  if (rc == LS_OK) rc = fd_apply(ctx, r, z);
  if (rc == LS_OK) rc = dot(ctx, r, z, S_RHO0);
  ck(cudaMemcpyAsync(p, z, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  ck(cudaMemsetAsync(ctx->scal + S_K, 0, sizeof(double), ctx->stream));  // k = 0 (all-zero bits)
  tail();
  // WHILE node after the first test, its body captured on the second stream
  cudaGraphNode_t wn = nullptr;
  if (rc == LS_OK) {
    cudaStreamCaptureStatus cs;
    cudaGraph_t cg = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    ck(cudaStreamGetCaptureInfo(ctx->stream, &cs, nullptr, &cg, &deps, &nd));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    if (rc == LS_OK) ck(cudaGraphAddNode(&wn, cg, deps, nd, &cp));
    if (rc == LS_OK) ck(cudaStreamUpdateCaptureDependencies(ctx->stream, &wn, 1, cudaStreamSetCaptureDependencies));
    if (rc == LS_OK) {
      const int64_t lb = ctx->launches;
      cudaStream_t outer = ctx->stream;
      ctx->stream = ctx->cap_stream2;
      ck(cudaStreamBeginCaptureToGraph(ctx->stream, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                       cudaStreamCaptureModeRelaxed));
      if (rc == LS_OK) rc = fd_apply(ctx, r, z);
      if (rc == LS_OK) rc = dot(ctx, r, z, S_RHO1);
      if (rc == LS_OK) {
        ck(launch_pdl(update_p_kernel, gb, RED_THREADS, 0, ctx->stream, p, z, uint64_t(ctx->Nl), ctx->scal,
                      int(S_RHO1), int(S_RHO0)));
        ck(launch_pdl(copy_slot_kernel, 1, 1, 0, ctx->stream, ctx->scal, int(S_RHO0), int(S_RHO1)));
        ctx->launches += 2;
      }
      tail();
      cudaGraph_t bo = nullptr;
      ck(cudaStreamEndCapture(ctx->stream, &bo));
      ctx->stream = outer;
      ctx->pcg_body_launches = ctx->launches - lb;
    }
  }
  // true residual ||b - A x|| -> scal[S_AUX]
  if (rc == LS_OK) rc = ls_matvec(ctx, x, q);
  if (rc == LS_OK) {
    ck(launch_pdl(sub_kernel, gb, RED_THREADS, 0, ctx->stream, z, b, q, uint64_t(ctx->Nl)));
    ctx->launches++;
  }
  if (rc == LS_OK) rc = dot(ctx, z, z, S_AUX);
  if (capturing) {
    cudaGraph_t out = nullptr;
    ck(cudaStreamEndCapture(ctx->cap_stream, &out));
  }
  ctx->stream = user;
  ctx->pcg_fixed_launches = ctx->launches - l0 - ctx->pcg_body_launches;
  ctx->launches = l0;
  if (rc == LS_OK && cudaGraphInstantiate(&ctx->pcg_exec, g, 0) != cudaSuccess) {
    ctx->pcg_exec = nullptr;
    rc = LS_ECUDA;
  }
  cudaGraphDestroy(g);
  cudaGetLastError();  // a failed capture is not sticky: the host loop takes over
  if (rc != LS_OK) return rc;
  ctx->pcg_key_b = b;
  ctx->pcg_key_x = x;
  ctx->pcg_key_tol = tol;
  ctx->pcg_key_iter = max_iter;
  return LS_OK;
}

extern "C" int pcg_solve(ls_ctx* ctx, const double* b, double* x, double tol, int max_iter,
                         ls_pcg_stats* st) {
  if (!ctx || !b || !x || b == x || !aligned8(b) || !aligned8(x) || !(tol >= 0) || max_iter < 0)
    return LS_EINVAL;  // b == x: x is zeroed before b is read
  ls_pcg_stats s{0, 0.0, 0.0, LS_OK};
  const size_t bytes = size_t(ctx->Nl) * sizeof(double);
  LS_CUDA(cudaMemsetAsync(x, 0, bytes, ctx->stream));
  LS_CHECK(dot(ctx, b, b, S_BB));
  LS_CHECK(read_scal(ctx));
  const double bnorm = std::sqrt(ctx->h_scal[S_BB]);
  if (bnorm == 0.0) {
    if (st) *st = s;
    return LS_OK;
  }
  if (max_iter >= 1 && ctx->world == 1 && ctx->pcg_graph && !ctx->prof) {
    bool ok = ctx->pcg_exec && ctx->pcg_key_b == b && ctx->pcg_key_x == x && ctx->pcg_key_tol == tol &&
              ctx->pcg_key_iter == max_iter;
    if (!ok) ok = pcg_build_graph(ctx, b, x, tol, max_iter) == LS_OK;
    if (ok) {
      LS_CUDA(cudaGraphLaunch(ctx->pcg_exec, ctx->stream));
      LS_CHECK(read_scal(ctx));
      s.iters = int(ctx->h_scal[S_K]);
      ctx->launches += ctx->pcg_fixed_launches + ctx->pcg_body_launches * (s.iters - 1);
      s.rel_res = std::sqrt(ctx->h_scal[S_RR]) / bnorm;
      s.true_rel_res = std::sqrt(ctx->h_scal[S_AUX]) / bnorm;
      s.status = int(ctx->h_scal[S_STAT]);
      if (st) *st = s;
      return s.status;
    }
  }
  int64_t lo = 0, hi = 0;
  if (ctx->world > 1) ext_geom(ctx, &lo, &hi);
  // p lives inside the halo-extended buffer so ls_matvec needs no copy
  double *r = ctx->pr, *z = ctx->pz, *p = ctx->pp + lo * ctx->Ns, *q = ctx->pq;
  LS_CUDA(cudaMemcpyAsync(r, b, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  LS_CHECK(fd_apply(ctx, r, z));
  int cur = S_RHO0, nxt = S_RHO1;
  LS_CHECK(dot(ctx, r, z, cur));
  LS_CUDA(cudaMemcpyAsync(p, z, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  double rel = 1.0;
  int k = 0;
  s.status = LS_ENOCONV;
  const unsigned g = RED_BLOCKS;
  while (k < max_iter) {
    LS_CHECK(matvec_dot(ctx, p, q, S_PQ));
    LS_CUDA(launch_pdl(update_xr_kernel, g, RED_THREADS, 0, ctx->stream, x, r, p, q, uint64_t(ctx->Nl), ctx->scal,
                       cur, ctx->partials));
    LS_CUDA(launch_pdl(reduce_final_kernel, 1, RED_THREADS, 0, ctx->stream, ctx->partials, int(RED_BLOCKS),
                       ctx->scal, int(S_RR)));
    ctx->launches += 2;
    LS_CUDA(cudaGetLastError());
    if (ctx->world > 1) LS_CHECK(ctx->comm->allreduce_scalar(ctx->scal + S_RR));
    LS_CHECK(read_scal(ctx));
    ++k;
    const double rr = ctx->h_scal[S_RR], alpha = ctx->h_scal[S_ALPHA];
    if (!std::isfinite(rr) || !std::isfinite(alpha)) {
      s.status = LS_ENUMERIC;
      break;
    }
    rel = std::sqrt(rr) / bnorm;
    if (rel <= tol) {
      s.status = LS_OK;
      break;
    }
    LS_CHECK(fd_apply(ctx, r, z));
    LS_CHECK(dot(ctx, r, z, nxt));
    LS_CUDA(launch_pdl(update_p_kernel, g, RED_THREADS, 0, ctx->stream, p, z, uint64_t(ctx->Nl), ctx->scal, nxt,
                       cur));
    ctx->launches++;
    LS_CUDA(cudaGetLastError());
    std::swap(cur, nxt);
  }
  s.iters = k;
  s.rel_res = rel;
  // true residual ||b - A x|| / ||b||
  LS_CHECK(ls_matvec(ctx, x, q));
  LS_CUDA(launch_pdl(sub_kernel, g, RED_THREADS, 0, ctx->stream, z, b, q, uint64_t(ctx->Nl)));
  ctx->launches++;
  LS_CHECK(dot(ctx, z, z, S_RR));
  LS_CHECK(read_scal(ctx));
  s.true_rel_res = std::sqrt(ctx->h_scal[S_RR]) / bnorm;
  if (st) *st = s;
  return s.status;
}

// ------------------------------------------------------------------------------------------
// least-squares functional / energy error (PAPER.md 392-410)
// ------------------------------------------------------------------------------------------
extern "C" int ls_energy_error(ls_ctx* ctx, int kind, const double* x, double* out4) {
  if (!ctx || !x || !out4 || !aligned8(x) || kind < 0 || kind > 3) return LS_EINVAL;
  if (ctx->geo ? kind < 2 : kind >= 2) return ctx->geo ? LS_ENOTSUP : LS_EINVAL;
  if (x == ctx->pz || x == ctx->pq) return LS_EINVAL;  // the library's scratch vectors
  const double pi = 3.14159265358979323846;
  const int d = ctx->d;
  // ||f||^2 in closed form (T = 1, unit cube, reading c11): int sin^2(pi x) = 1/2 per direction
  double f2 = std::ldexp(1.0, -d);
  if (kind >= 2) {
    // mapped domains. kind 2, u = P sin(pi t): int_0^1 (pi cos)^2 = pi^2 / 2, int sin^2 = 1/2,
    // cross term 0.  kind 3: f time independent, T = 1.
    LS_CHECK(geo_load(*ctx->geo, *ctx->gmap, ctx->n_el, kind, ctx->stream, &ctx->launches));
    f2 = kind == 2 ? 0.5 * pi * pi * ctx->geo->fint[0] + 0.5 * ctx->geo->fint[1] : ctx->geo->fint[0];
  } else if (kind == 0) {
    f2 *= (std::exp(2.0) - 1.0) / 2.0;
  } else {
    const double c = d * pi * pi;
    f2 *= (0.5 + std::sin(2.0) / 4.0) + c * std::sin(1.0) * std::sin(1.0) + c * c * (0.5 - std::sin(2.0) / 4.0);
  }
  LS_CHECK(ls_rhs(ctx, kind, ctx->pz));         // b_i = F(B_i)
  LS_CHECK(dot(ctx, ctx->pz, x, S_AUX));         // b . x = F(u_h)
  LS_CUDA(cudaStreamSynchronize(ctx->stream));
  LS_CHECK(read_scal(ctx));
  const double bx = ctx->h_scal[S_AUX];
  LS_CHECK(ls_matvec(ctx, x, ctx->pq));          // A x
  LS_CHECK(dot(ctx, x, ctx->pq, S_AUX));         // x . A x = A(u_h, u_h)
  LS_CHECK(read_scal(ctx));
  const double xax = ctx->h_scal[S_AUX];
  out4[0] = f2 - 2.0 * bx + xax;
  out4[1] = f2;
  out4[2] = bx;
  out4[3] = xax;
  return LS_OK;
}

// discretisation-error norms against the exact solution (err.cu)
extern "C" int ls_error_norms(ls_ctx* ctx, int kind, const double* x, double* out8) {
  if (!ctx || !x || !out8 || !aligned8(x)) return LS_EINVAL;
  if (ctx->world != 1) return LS_ENOTSUP;
  ErrSetup es;
  es.d = ctx->d;
  es.ps = ctx->p;
  es.pt = ctx->pt;
  es.kind = kind;
  es.nt = ctx->nt;
  for (int k = 0; k <= ctx->d; ++k) es.n_el[k] = ctx->n_el[k];
  es.gmap = ctx->gmap.get();
  return error_norms(es, x, ctx->stream, &ctx->launches, out8);
}

// ------------------------------------------------------------------------------------------
// host-buffer entry point, introspection, teardown
// ------------------------------------------------------------------------------------------
extern "C" int fd_apply_host(ls_ctx* ctx, const double* r_host, double* z_host) {
  if (!ctx || !r_host || !z_host) return LS_EINVAL;
  const size_t bytes = size_t(ctx->Nl) * sizeof(double);
  constexpr int NCH = 8;
  if (ctx->world == 1 && ctx->ntl >= NCH && !ctx->dm12) {
    // pipelined over NCH time-slice chunks (the spatial modes act slice by slice): the
    // H2D copy of chunk k+1 overlaps the forward spatial modes of chunk k, the D2H copy of
    // chunk k overlaps the backward spatial modes of chunk k+1; the time mode needs all.
    if (!ctx->copy_stream) {
      LS_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
      for (auto& e : ctx->hev) LS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const int64_t Ns = ctx->Ns;
    double *A = ctx->tmp[0], *B = ctx->tmp[1], *C = ctx->tmp[2], *R = ctx->pr, *Z = ctx->pz;
    LS_CUDA(cudaEventRecord(ctx->hev[16], ctx->stream));  // earlier work on the context stream
    LS_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->hev[16], 0));
    for (int k = 0; k < NCH; ++k) {
      int64_t off, rows;
      split_part(ctx->ntl, NCH, k, &off, &rows);
      LS_CUDA(cudaMemcpyAsync(R + off * Ns, r_host + off * Ns, size_t(rows * Ns) * sizeof(double),
                              cudaMemcpyHostToDevice, ctx->copy_stream));
      LS_CUDA(cudaEventRecord(ctx->hev[k], ctx->copy_stream));
      LS_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->hev[k], 0));
      LS_CHECK(spatial_modes(ctx, R + off * Ns, A + off * Ns, B + off * Ns, C + off * Ns, uint64_t(rows), true));
    }
    LS_CHECK(time_modes(ctx, A, B, C, uint64_t(Ns), ctx->lam_s));
    for (int k = 0; k < NCH; ++k) {
      int64_t off, rows;
      split_part(ctx->ntl, NCH, k, &off, &rows);
      LS_CHECK(spatial_modes(ctx, C + off * Ns, Z + off * Ns, A + off * Ns, B + off * Ns, uint64_t(rows), false));
      LS_CUDA(cudaEventRecord(ctx->hev[NCH + k], ctx->stream));
      LS_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->hev[NCH + k], 0));
      LS_CUDA(cudaMemcpyAsync(z_host + off * Ns, Z + off * Ns, size_t(rows * Ns) * sizeof(double),
                              cudaMemcpyDeviceToHost, ctx->copy_stream));
    }
    LS_CUDA(cudaStreamSynchronize(ctx->copy_stream));
    LS_CUDA(cudaStreamSynchronize(ctx->stream));
    return LS_OK;
  }
  LS_CUDA(cudaMemcpyAsync(ctx->pr, r_host, bytes, cudaMemcpyHostToDevice, ctx->stream));
  LS_CHECK(fd_apply(ctx, ctx->pr, ctx->pz));
  LS_CUDA(cudaMemcpyAsync(z_host, ctx->pz, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  LS_CUDA(cudaStreamSynchronize(ctx->stream));
  return LS_OK;
}

// count fd_apply calls on host vectors, pipelined across vectors: two device buffer pairs, the
// H2D copy of vector k + 1 (H2D stream) and the D2H copy of vector k - 1 (D2H stream) run while
// vector k is applied on the context stream (PCIe is full duplex, so both directions overlap).
extern "C" int fd_apply_host_batch(ls_ctx* ctx, const double* const* r_host, double* const* z_host, int64_t count) {
  if (!ctx || count < 0 || (count > 0 && (!r_host || !z_host))) return LS_EINVAL;
  for (int64_t k = 0; k < count; ++k)
    if (!r_host[k] || !z_host[k]) return LS_EINVAL;
  if (count == 0) return LS_OK;
  if (!ctx->hb_r) {
    LS_CHECK(ctx->alloc(&ctx->hb_r, ctx->Nl));
    LS_CHECK(ctx->alloc(&ctx->hb_z, ctx->Nl));
    LS_CUDA(cudaStreamCreateWithFlags(&ctx->h2d_stream, cudaStreamNonBlocking));
    LS_CUDA(cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking));
    for (auto& e : ctx->bev) LS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  const size_t bytes = size_t(ctx->Nl) * sizeof(double);
  double* R[2] = {ctx->pr, ctx->hb_r};
  double* Z[2] = {ctx->pz, ctx->hb_z};
  cudaEvent_t* h2d_done = ctx->bev;      // [2]
  cudaEvent_t* comp_done = ctx->bev + 2;  // [2]
  cudaEvent_t* d2h_done = ctx->bev + 4;   // [2]
  LS_CUDA(cudaEventRecord(ctx->bev[6], ctx->stream));  // earlier work on the context stream
  LS_CUDA(cudaStreamWaitEvent(ctx->h2d_stream, ctx->bev[6], 0));
  LS_CUDA(cudaStreamWaitEvent(ctx->d2h_stream, ctx->bev[6], 0));
  for (int64_t k = 0; k < count; ++k) {
    const int b = int(k & 1);
    if (k >= 2) LS_CUDA(cudaStreamWaitEvent(ctx->h2d_stream, comp_done[b], 0));  // R[b] read by vector k - 2
    LS_CUDA(cudaMemcpyAsync(R[b], r_host[k], bytes, cudaMemcpyHostToDevice, ctx->h2d_stream));
    LS_CUDA(cudaEventRecord(h2d_done[b], ctx->h2d_stream));
    LS_CUDA(cudaStreamWaitEvent(ctx->stream, h2d_done[b], 0));
    if (k >= 2) LS_CUDA(cudaStreamWaitEvent(ctx->stream, d2h_done[b], 0));  // Z[b] copied out
    LS_CHECK(fd_apply(ctx, R[b], Z[b]));
    LS_CUDA(cudaEventRecord(comp_done[b], ctx->stream));
    LS_CUDA(cudaStreamWaitEvent(ctx->d2h_stream, comp_done[b], 0));
    LS_CUDA(cudaMemcpyAsync(z_host[k], Z[b], bytes, cudaMemcpyDeviceToHost, ctx->d2h_stream));
    LS_CUDA(cudaEventRecord(d2h_done[b], ctx->d2h_stream));
  }
  LS_CUDA(cudaStreamSynchronize(ctx->h2d_stream));
  LS_CUDA(cudaStreamSynchronize(ctx->stream));
  LS_CUDA(cudaStreamSynchronize(ctx->d2h_stream));
  return LS_OK;
}

extern "C" int ls_get_factor(const ls_ctx* ctx, int which, int dir, double* out) {
  if (!ctx || !out) return LS_EINVAL;
  const std::vector<double>* v = nullptr;
  const int k = dir - 1;
  const bool sp = (k >= 0 && k < ctx->d);
  switch (which) {
    case 0: v = sp ? &ctx->hM[k] : nullptr; break;
    case 1: v = sp ? &ctx->hK[k] : nullptr; break;
    case 2: v = sp ? &ctx->hJ[k] : nullptr; break;
    case 3: v = &ctx->hMt; break;
    case 4: v = &ctx->hKt; break;
    case 5: v = sp ? &ctx->hlam[k] : nullptr; break;
    case 6: v = &ctx->hlam[3]; break;
    case 7: v = sp ? &ctx->hU[k] : nullptr; break;
    case 8: v = &ctx->hU[3]; break;
    default: return LS_EINVAL;
  }
  if (!v) return LS_EINVAL;
  std::memcpy(out, v->data(), v->size() * sizeof(double));
  return LS_OK;
}

extern "C" int ls_profile(ls_ctx* ctx, int enable) {
  if (!ctx) return LS_EINVAL;
  ctx->prof = enable != 0;
  return LS_OK;
}

extern "C" int ls_profile_read(ls_ctx* ctx, double* total_ms, double* total_flops, int64_t* n) {
  if (!ctx) return LS_EINVAL;
  LS_CUDA(cudaStreamSynchronize(ctx->stream));
  double ms = 0, fl = 0;
  for (auto& r : ctx->prof_recs) {
    float t = 0;
    LS_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    ms += t;
    fl += r.flops;
    ctx->ev_pool.push_back(r.a);
    ctx->ev_pool.push_back(r.b);
  }
  if (total_ms) *total_ms = ms;
  if (total_flops) *total_flops = fl;
  if (n) *n = int64_t(ctx->prof_recs.size());
  ctx->prof_recs.clear();
  return LS_OK;
}

// ---- host-only plan queries (no GPU needed; used by the CPU multi-rank tests) -------------
extern "C" int ls_partition(int64_t total, int world, int part, int64_t* off, int64_t* len) {
  if (world < 1 || part < 0 || part >= world || total < 0 || !off || !len) return LS_EINVAL;
  split_part(total, world, part, off, len);
  return LS_OK;
}

extern "C" int ls_a2a_plan(int64_t nt, int64_t Ns, int world, int rank, int64_t* send_off,
                           int64_t* send_cnt, int64_t* recv_off, int64_t* recv_cnt) {
  if (world < 1 || rank < 0 || rank >= world || !send_off || !send_cnt || !recv_off || !recv_cnt)
    return LS_EINVAL;
  for (int h = 0; h < world; ++h)
    a2a_plan(nt, Ns, world, rank, h, send_off + h, send_cnt + h, recv_off + h, recv_cnt + h);
  return LS_OK;
}

extern "C" int ls_a2a_piece_plan(int64_t nt, int64_t Ns, int world, int rank, int piece, int* pieces,
                                 int64_t* send_off, int64_t* send_cnt, int64_t* recv_off, int64_t* recv_cnt) {
  if (world < 1 || rank < 0 || rank >= world || nt < 1 || !pieces) return LS_EINVAL;
  *pieces = a2a_pieces(nt, world);
  if (piece < 0) return LS_OK;
  if (piece >= *pieces || !send_off || !send_cnt || !recv_off || !recv_cnt) return LS_EINVAL;
  for (int h = 0; h < world; ++h)
    a2a_piece_plan(nt, Ns, world, rank, h, piece, *pieces, send_off + h, send_cnt + h, recv_off + h, recv_cnt + h);
  return LS_OK;
}

extern "C" int ls_pack_map(int64_t ntl, int64_t Ns, int world, int64_t* pos) {
  if (world < 1 || ntl < 0 || Ns < 0 || !pos) return LS_EINVAL;
  for (int64_t e = 0; e < ntl * Ns; ++e) pos[e] = pack_pos(e, ntl, Ns, world);
  return LS_OK;
}

extern "C" int ls_a2a_dest(int64_t nt, int64_t Ns, int world, int rank, int dir, int64_t i, int64_t j, int* peer,
                           int64_t* off) {
  if (world < 1 || rank < 0 || rank >= world || !peer || !off || (dir != 0 && dir != 1)) return LS_EINVAL;
  if (dir == 0) a2a_fwd_dest(i, j, nt, Ns, world, rank, peer, off);
  else a2a_bwd_dest(i, j, nt, Ns, world, rank, peer, off);
  return LS_OK;
}

extern "C" int ls_halo_plan(int64_t nt, int world, int rank, int p, int64_t* t0, int64_t* ntl,
                            int64_t* lo, int64_t* hi) {
  if (world < 1 || rank < 0 || rank >= world || p < 0 || !t0 || !ntl || !lo || !hi) return LS_EINVAL;
  halo_plan(nt, world, rank, p, t0, ntl, lo, hi);
  if (world > 1 && nt / world < p) return LS_EINVAL;  // a slab thinner than the halo
  return LS_OK;
}

extern "C" int64_t ls_kernel_launches(const ls_ctx* ctx) { return ctx ? ctx->launches : -1; }

extern "C" int ls_tune(ls_ctx* ctx, int knob, int value) {
  if (!ctx) return LS_EINVAL;
  if (ctx->pcg_exec) {  // the cached PCG graph holds the kernels chosen so far
    cudaGraphExecDestroy(ctx->pcg_exec);
    ctx->pcg_exec = nullptr;
  }
  switch (knob) {
    case LS_TUNE_FD_KERNEL:
      if (value < 0 || value > 2) return LS_EINVAL;
      ctx->fd_variant = value;
      return LS_OK;
    case LS_TUNE_MATVEC:
      if (value < 0 || value > 4) return LS_EINVAL;
      ctx->mv_variant = value;
      if (ctx->geo) ctx->geo->variant = (value == 1) ? 1 : 0;  // mapped domain: 1 = DFMA stencil
      return LS_OK;
    case LS_TUNE_A2A: {  // collective when enabling: every rank calls it
      if (value == 0) {
        if (ctx->comm) ctx->comm->fused = false;
        return LS_OK;
      }
      if (value != 1 || !ctx->comm || ctx->d < 2) return LS_EINVAL;
      uint64_t Q = 1;
      for (int j = 0; j < ctx->d - 1; ++j) Q *= ctx->n[j];
      if (Q % 4 != 0) return LS_ENOTSUP;  // the scattering epilogue is a FAST-path variant
      return ctx->comm->setup_fused(ctx->tmp[1], ctx->tmp[0]);
    }
    case LS_TUNE_MV4_CTAS:  // process-wide: plane-pass register budget (CTAs per SM)
      if (value != 1 && value != 2) return LS_EINVAL;
      g_mv4_ctas = value;
      return LS_OK;
    case LS_TUNE_FD_TAIL:
      if (value < 0 || value > 2) return LS_EINVAL;
      ctx->fd_tail = value != 0;
      g_rd_tail = value == 2;  // process-wide: the split register-direct kernels (RDCfg::TR)
      return LS_OK;
    case LS_TUNE_MV5:  // v4: direction 3 + time fused into one pass (d = 3, p_s = p_t); 2 = automatic
      if (value < 0 || value > 2) return LS_EINVAL;
      ctx->mv5 = value;
      return LS_OK;
    case LS_TUNE_PQ_FUSE:  // PCG: p.q fused into the matvec's last pass (1) or a separate dot (0)
      if (value != 0 && value != 1) return LS_EINVAL;
      ctx->pq_fuse = value;
      return LS_OK;
    case LS_TUNE_FD_STAGED:  // process-wide: the cp.async-staged split FD kernel where it applies
      if (value != 0 && value != 1) return LS_EINVAL;
      g_rd_staged = value;
      return LS_OK;
    case LS_TUNE_FD_TIME:  // fused time mode (one launch) where n_t <= 104 (1, default) or two launches (0)
      if (value != 0 && value != 1) return LS_EINVAL;
      ctx->fd_time = value;
      return LS_OK;
    case LS_TUNE_MV2_SWEEP:  // v2 (p = 2): the d = 3 plane pass as the register sweep (1, default) or staged (0)
      if (value != 0 && value != 1) return LS_EINVAL;
      ctx->mv2_sweep = value;
      return LS_OK;
    case LS_TUNE_MV4_SWEEP:  // v4's plane pass as the DFMA register sweep (d = 3, p = 3, 4; opt-in)
      if (value != 0 && value != 1) return LS_EINVAL;
      ctx->mv4_sweep = value;
      return LS_OK;
    case LS_TUNE_MV6:  // v4's direction-3 + time passes as DFMA stencils: 0 off (default), 1 on
      if (value != 0 && value != 1) return LS_EINVAL;
      ctx->mv6 = value;
      return LS_OK;
    case LS_TUNE_FD_PLANE:  // spatial modes 1 + 2 as one plane launch where supported (1) or per direction (0, default)
      if (value != 0 && value != 1) return LS_EINVAL;
      ctx->fd_plane = value;
      return LS_OK;
    case LS_TUNE_FD_CS:  // centrosymmetric split of the spatial modes (default 1 where the pencil allows)
      if (value != 0 && value != 1) return LS_EINVAL;
      ctx->fd_cs = value;
      return LS_OK;
    case LS_TUNE_PDL:  // process-wide: programmatic dependent launch of the FD mode kernels
      if (value != 0 && value != 1) return LS_EINVAL;
      g_ls_pdl = value;
      return LS_OK;
    case LS_TUNE_PCG_GRAPH:  // 1 = graph-resident PCG loop (default on one GPU), 0 = host loop
      if (value != 0 && value != 1) return LS_EINVAL;
      ctx->pcg_graph = value;
      return LS_OK;
    case LS_TUNE_MV3_PAD:  // row granularity of the v3 intermediates along direction 1
      if (value != 1 && value != 8 && value != 16) return LS_EINVAL;
      if (ctx->d < 2) return LS_OK;
      ctx->n1p = (ctx->n[0] + value - 1) / value * value;
      return LS_OK;
    default: return LS_EINVAL;
  }
}

extern "C" void ls_destroy(ls_ctx* ctx) {
  if (!ctx) return;
  cudaDeviceSynchronize();
  delete ctx;
}

extern "C" const char* ls_strerror(int code) {
  switch (code) {
    case LS_OK: return "ok";
    case LS_EINVAL: return "invalid argument";
    case LS_ENOTSPD: return "mass matrix not SPD (Cholesky failure in the generalized eigensolver)";
    case LS_ENOCONV: return "PCG did not converge within max_iter";
    case LS_ENUMERIC: return "NaN/Inf in a PCG scalar";
    case LS_ENOMEM: return "not enough device memory";
    case LS_ECUDA: return "CUDA runtime error";
    case LS_ENCCL: return "NCCL error";
    case LS_ENOTSUP: return "operation not supported for this context";
    default: return "unknown error";
  }
}
