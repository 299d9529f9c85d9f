// runtime.cu — context, solver drivers, training loop and the C-ABI.
//
// Host C++ side of the drop-in boundary (include/warmgp_b200.h).  The solver
// drivers restate proj/src/solvers.cpp over a matrix-free device operator;
// the outer loop restates proj/src/optimizer.cpp:81-171 with the solver state
// (warm-start solutions, residuals, directions) resident in HBM across steps.
#include <cublas_v2.h>
#include <cusolverDn.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the entry points are resolved from libnccl.so.2 at run time

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/warmgp_b200.h"
#include "common.cuh"
#include "exact.cuh"
#include "host_rng.hpp"
#include "hv_f64.cuh"
#include "hv_tc.cuh"
#include "kernels.cuh"
#include "solver_kernels.cuh"

namespace wgp {
namespace {

thread_local std::string g_last_error;
constexpr uint64_t kSolverStream = 0x736f6c7665ULL;  // proj/src/optimizer.cpp:15
constexpr double kUScale = kSqrt3 * kLog2e;            // u = sqrt(3) log2(e) r

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  Buf() = default;
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  ~Buf() {
    if (p) cudaFree(p);
  }
  void ensure(size_t b) {
    if (b <= bytes) return;
    if (p) WGP_CUDA(cudaFree(p));
    p = nullptr;
    bytes = 0;
    WGP_CUDA(cudaMalloc(&p, b));
    bytes = b;
    alloc_generation().fetch_add(1);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct PinnedCtrl {
  SolveCtrl* h = nullptr;
  PinnedCtrl() { WGP_CUDA(cudaMallocHost(&h, sizeof(SolveCtrl))); }
  ~PinnedCtrl() {
    if (h) cudaFreeHost(h);
  }
};

// Page-locked host staging that grows on demand (async host -> device copies).
struct PinnedBuf {
  void* p = nullptr;
  size_t bytes = 0;
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  void ensure(size_t b) {
    if (b <= bytes) return;
    if (p) WGP_CUDA(cudaFreeHost(p));
    p = nullptr;
    bytes = 0;
    WGP_CUDA(cudaMallocHost(&p, b));
    bytes = b;
  }
  template <class T>
  T* as() {
    return static_cast<T*>(p);
  }
};

const char* solver_name(int kind) { return kind == 0 ? "cg_solve" : kind == 1 ? "ap_solve" : "sgd_solve"; }

// NCCL, resolved at run time from libnccl.so.2 (the copy torch already
// loaded, when it did, else the system's): a context without a communicator
// never touches it, and the library has no link-time NCCL dependency.
struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  static const NcclApi& get() {
    static const NcclApi api = [] {
      NcclApi a;
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
      if (!h) return a;
      a.get_unique_id = reinterpret_cast<decltype(&ncclGetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
      a.comm_init_rank = reinterpret_cast<decltype(&ncclCommInitRank)>(dlsym(h, "ncclCommInitRank"));
      a.comm_destroy = reinterpret_cast<decltype(&ncclCommDestroy)>(dlsym(h, "ncclCommDestroy"));
      a.all_gather = reinterpret_cast<decltype(&ncclAllGather)>(dlsym(h, "ncclAllGather"));
      a.all_reduce = reinterpret_cast<decltype(&ncclAllReduce)>(dlsym(h, "ncclAllReduce"));
      a.group_start = reinterpret_cast<decltype(&ncclGroupStart)>(dlsym(h, "ncclGroupStart"));
      a.group_end = reinterpret_cast<decltype(&ncclGroupEnd)>(dlsym(h, "ncclGroupEnd"));
      a.error_string = reinterpret_cast<decltype(&ncclGetErrorString)>(dlsym(h, "ncclGetErrorString"));
      return a;
    }();
    if (!api.comm_init_rank || !api.all_gather || !api.all_reduce || !api.group_start)
      throw DeviceError("NCCL (libnccl.so.2) is not available");
    return api;
  }
  void check(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess)
      throw DeviceError(std::string(what) + ": " + (error_string ? error_string(r) : "NCCL error"));
  }
};

// A rank's communicator.  NcclComm (one process per GPU) is the
// product; LocalComm is a host-mediated stand-in for tests on one GPU: N
// contexts driven by N host threads, each collective a host barrier plus
// device copies between the contexts' buffers, so no kernel ever waits on
// another rank's kernel.  Collectives run on the context stream (NCCL's are
// captured into the CG / AP graphs; LocalComm's are not capturable).
struct Comm {
  int rank = 0, nranks = 1;
  virtual ~Comm() = default;
  virtual bool capturable() const = 0;
  // In-place all-gather of row blocks of s columns (column c at base + c ld,
  // rank r's rows at [r blk, (r + 1) blk)).
  virtual void gather_rows(void* base, int64_t ld, int64_t blk, int s, size_t elem, cudaStream_t st) = 0;
  // recv[r * count + k] = rank r's send[k]
  virtual void all_gather(const double* send, double* recv, size_t count, cudaStream_t st) = 0;
  virtual void all_reduce_sum(double* buf, size_t count, cudaStream_t st) = 0;
};

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  NcclComm(int r, int nr, const ncclUniqueId& id) {
    rank = r;
    nranks = nr;
    const NcclApi& a = NcclApi::get();
    a.check(a.comm_init_rank(&comm, nr, id, r), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm) NcclApi::get().comm_destroy(comm);
  }
  static ncclDataType_t type(size_t elem) { return elem == 8 ? ncclFloat64 : ncclFloat32; }
  bool capturable() const override { return true; }
  void gather_rows(void* base, int64_t ld, int64_t blk, int s, size_t elem, cudaStream_t st) override {
    const NcclApi& a = NcclApi::get();
    char* b = static_cast<char*>(base);
    a.check(a.group_start(), "ncclGroupStart");  // one grouped launch for all columns
    for (int c = 0; c < s; ++c) {
      char* col = b + static_cast<size_t>(c) * ld * elem;
      a.check(a.all_gather(col + static_cast<size_t>(rank) * blk * elem, col, static_cast<size_t>(blk), type(elem),
                           comm, st),
              "ncclAllGather");
    }
    a.check(a.group_end(), "ncclGroupEnd");
  }
  void all_gather(const double* send, double* recv, size_t count, cudaStream_t st) override {
    const NcclApi& a = NcclApi::get();
    a.check(a.all_gather(send, recv, count, ncclFloat64, comm, st), "ncclAllGather");
  }
  void all_reduce_sum(double* buf, size_t count, cudaStream_t st) override {
    const NcclApi& a = NcclApi::get();
    a.check(a.all_reduce(buf, buf, count, ncclFloat64, ncclSum, comm, st), "ncclAllReduce");
  }
};

}  // namespace

// The shared state of a LocalComm group (wgp_local_group_create).
struct LocalGroup {
  int nranks = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  std::vector<const void*> slot;
  explicit LocalGroup(int n) : nranks(n), slot(n, nullptr) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = generation;
    if (++arrived == nranks) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != g; });
    }
  }
};

namespace {
struct LocalComm : Comm {
  std::shared_ptr<LocalGroup> g;
  LocalComm(std::shared_ptr<LocalGroup> grp, int r) : g(std::move(grp)) {
    rank = r;
    nranks = g->nranks;
  }
  bool capturable() const override { return false; }
  // publish this rank's pointer once its stream is idle; returns after all did
  void publish(const void* p, cudaStream_t st) {
    WGP_CUDA(cudaStreamSynchronize(st));
    g->slot[rank] = p;
    g->barrier();
  }
  void gather_rows(void* base, int64_t ld, int64_t blk, int s, size_t elem, cudaStream_t st) override {
    publish(base, st);
    for (int r = 0; r < nranks; ++r) {
      if (r == rank) continue;
      const char* src = static_cast<const char*>(g->slot[r]) + static_cast<size_t>(r) * blk * elem;
      char* dst = static_cast<char*>(base) + static_cast<size_t>(r) * blk * elem;
      WGP_CUDA(cudaMemcpy2DAsync(dst, ld * elem, src, ld * elem, blk * elem, s, cudaMemcpyDeviceToDevice, st));
    }
    WGP_CUDA(cudaStreamSynchronize(st));
    g->barrier();  // nobody overwrites its block before every rank copied it
  }
  void all_gather(const double* send, double* recv, size_t count, cudaStream_t st) override {
    publish(send, st);
    for (int r = 0; r < nranks; ++r)
      WGP_CUDA(cudaMemcpyAsync(recv + r * count, g->slot[r], sizeof(double) * count, cudaMemcpyDeviceToDevice, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    g->barrier();
  }
  void all_reduce_sum(double* buf, size_t count, cudaStream_t st) override {
    publish(buf, st);
    std::vector<double> sum(count, 0.0), part(count);
    for (int r = 0; r < nranks; ++r) {  // rank order
      WGP_CUDA(cudaMemcpy(part.data(), g->slot[r], sizeof(double) * count, cudaMemcpyDeviceToHost));
      for (size_t k = 0; k < count; ++k) sum[k] += part[k];
    }
    g->barrier();  // every rank has read every buffer
    WGP_CUDA(cudaMemcpyAsync(buf, sum.data(), sizeof(double) * count, cudaMemcpyHostToDevice, st));
    WGP_CUDA(cudaStreamSynchronize(st));
  }
};

}  // namespace

struct Ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  cublasHandle_t cublas = nullptr;
  cusolverDnHandle_t cusolver = nullptr;
  int hv_impl = WGP_HV_TC;

  int64_t n = 0, n_pad = 0, ld = 0;
  int d = 0, dp = 0;
  Buf X;    // raw inputs, column-major n x d
  Buf xs;   // prepared points [n_pad][dp]
  std::vector<double> mu, ls;
  double sf = 1.0, sigma = 1.0;
  bool have_hyper = false;
  int64_t r0 = 0, r1 = -1;
  int64_t ap_bs = 0;  // block size of the cached AP factors (hbuf), 0: none
  // J splits keyed on the global n (row shards reproduce the full operator's
  // rows bitwise) or on the local rows (wgp_set_split_global(ctx, 0): more
  // CTAs per rank on small row shards, rows equal to fp32 tolerance)
  bool split_global = true;
  TcOperands tc;

  // Row sharding (one process per GPU, wgp_set_comm): rank r owns rows
  // [own0, own1) = [r blk, (r + 1) blk) ∩ [0, n) of every solver vector;
  // vectors keep all n rows (ld = nranks blk) so the all-gathers are in place.
  std::unique_ptr<Comm> comm;
  int rank = 0, nranks = 1;
  int64_t blk = 0, own0 = 0, own1 = 0;
  bool sharded() const { return comm != nullptr; }
  bool graphs_ok() const { return !comm || comm->capturable(); }
  int64_t own_m() const { return own1 - own0; }
  Buf dloc, dall;  // per-rank column totals and their all-gather (dist reductions)

  // workspaces
  Buf ctrl, conv, rs, alpha, beta, bnorm, tol, part, colsum, best, stall, act, Xbest, Rbest;
  Buf P, HP, Rtmp, vel, batch, idx, hbuf, linv, Rb, D64, DX, DXP, XP, PP, lapack_work, info;
  Buf gpart, gout, gtc_ws;
  // fp64 CG (cg_precision == WGP_CG_F64): solver state and the hv_f64 split partials
  Buf B64, X64, R64, P64, HP64, Rt64, Xbest64, Rbest64, hv64_ws;
  Buf linv_ptrs;  // AP: device pointer array of the batched inverse
  Buf sgd_xsq;    // SGD: running ||X||_F^2
  Buf Rpart;      // row-sharded AP: this rank's share of a block residual
  Buf tr_rhs, tr_sol0, tr_sol1, tr_res, tr_sol64a, tr_sol64b;  // train(): solver state across steps
  Buf api_B, api_X0, api_Xs, api_Rs, api_B64;  // wgp_solve staging
  int cg_precision = WGP_CG_F64;
  Buf dhyp;  // device [sf2, a, diag] for the H.V kernels (CUDA-graph friendly)
  Buf hyper_tmp;  // set_hyper staging (centres, scales)
  Buf hx, hx_ws, exv;  // exact path: dense H (fp64), cuSOLVER workspace, vectors
  Buf io_in, io_out;  // staging for the host-pointer entry points
  Buf cublas_ws;  // explicit cuBLAS workspace: no allocation inside a captured AP epoch
  PinnedCtrl hctrl;
  PinnedBuf sgd_hidx;  // SGD minibatch indices, two rounds (double buffer)
  // wgp_hv's row-chunk pipeline: the result's device->host copy of one chunk
  // runs on its own stream under the next chunk's H.V
  cudaStream_t cst = nullptr;
  cudaEvent_t ev_chunk = nullptr, ev_copied = nullptr;
  // wgp_hv upload policy (see wgp_hv): the copy engine's last measured H2D rate and
  // the calls since it was measured
  cudaEvent_t ev_up0 = nullptr, ev_up1 = nullptr;
  double ce_gbps = -1.0;
  int zc_streak = 0;
  const float* v_host_next = nullptr;  // consumed by the next hv(): HvParams::v_host

  ~Ctx() {
    drop_cg_graphs();
    if (ev_chunk) cudaEventDestroy(ev_chunk);
    if (ev_copied) cudaEventDestroy(ev_copied);
    if (ev_up0) cudaEventDestroy(ev_up0);
    if (ev_up1) cudaEventDestroy(ev_up1);
    if (cst) cudaStreamDestroy(cst);
    if (cublas) cublasDestroy(cublas);
    if (cusolver) cusolverDnDestroy(cusolver);
    if (st) cudaStreamDestroy(st);
  }

  float sf2() const { return static_cast<float>(sf * sf); }
  float a_coef() const { return static_cast<float>(sf * sf * kLn2); }
  float noise2() const { return static_cast<float>(sigma * sigma); }

  void require_data() const {
    if (n < 1) throw std::invalid_argument("no training inputs: call wgp_set_data first");
    if (!have_hyper) throw std::invalid_argument("no hyperparameters: call wgp_set_hyper first");
  }

  // ---------------------------------------------------------------- data
  void set_data(const float* Xh, int64_t n_, int d_) {
    if (n_ < 1) throw std::invalid_argument("build_kernel_matrices: need at least one row");
    drop_cg_graphs();  // n and the leading dimension are baked into captured launches
    if (d_ < 1 || d_ > 64) throw std::invalid_argument("input dimension must lie in [1, 64]");
    for (int64_t e = 0; e < n_ * d_; ++e)
      if (!std::isfinite(Xh[e])) throw std::invalid_argument("build_kernel_matrices: non-finite input");
    n = n_;
    d = d_;
    dp = static_cast<int>(round_up(d, 4));
    n_pad = round_up(n, 128);
    ld = n_pad;
    blk = ld;
    own0 = 0;
    own1 = n;
    if (comm) {  // 128-row tiles dealt to the ranks in contiguous blocks
      blk = ceil_div(ceil_div(n, 128), nranks) * 128;
      ld = std::max(n_pad, blk * nranks);
      own0 = std::min<int64_t>(n, rank * blk);
      own1 = std::min<int64_t>(n, (rank + 1) * blk);
    }
    X.ensure(sizeof(float) * n * d);
    WGP_CUDA(cudaMemcpyAsync(X.p, Xh, sizeof(float) * n * d, cudaMemcpyHostToDevice, st));
    mu.assign(d, 0.0);
    for (int k = 0; k < d; ++k) {
      double acc = 0.0;
      for (int64_t i = 0; i < n; ++i) acc += Xh[i + k * n];
      mu[k] = acc / static_cast<double>(n);
    }
    xs.ensure(sizeof(float) * n_pad * dp);
    have_hyper = false;
    r0 = 0;
    r1 = n;
    tc.invalidate();
    WGP_CUDA(cudaStreamSynchronize(st));
  }

  void set_hyper(const double* c) {
    ap_bs = 0;  // cached AP block factors belong to the previous hyperparameters
    if (n < 1) throw std::invalid_argument("no training inputs: call wgp_set_data first");
    for (int k = 0; k < d + 2; ++k)
      if (!(c[k] > 0.0) || !std::isfinite(c[k]))
        throw std::invalid_argument("hyperparameters must be positive and finite");
    ls.assign(c, c + d);
    sf = c[d];
    sigma = c[d + 1];
    std::vector<double> scale(d);
    for (int k = 0; k < d; ++k) scale[k] = kUScale / ls[k];
    Buf& tmp = hyper_tmp;  // persistent: a fresh allocation would invalidate the cached CG graphs
    tmp.ensure(sizeof(double) * 2 * d);
    std::vector<double> h(2 * d);
    std::copy(mu.begin(), mu.end(), h.begin());
    std::copy(scale.begin(), scale.end(), h.begin() + d);
    WGP_CUDA(cudaMemcpyAsync(tmp.p, h.data(), sizeof(double) * 2 * d, cudaMemcpyHostToDevice, st));
    prepare_points(X.as<float>(), n, d, tmp.as<double>(), tmp.as<double>() + d, xs.as<float>(), n_pad,
                   dp, st);
    tc.invalidate();
    const float hh[4] = {sf2(), a_coef(), static_cast<float>(sf * sf + sigma * sigma), 0.f};
    dhyp.ensure(sizeof(float) * 4);
    WGP_CUDA(cudaMemcpyAsync(dhyp.p, hh, sizeof(hh), cudaMemcpyHostToDevice, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    have_hyper = true;
  }

  // ---------------------------------------------------------------- H.V
  void hv(const float* V, int64_t ldv, int s, float* out, int64_t ldo, int mode, const float* B,
          int64_t ldb, int64_t j0, int64_t j1, const int* row_idx, int64_t rr0, int64_t m,
          const int* done = nullptr, bool shard_invariant = true, const float* vplanes = nullptr,
          int64_t vplanes_ld = 0, bool reuse_vsplit = false) {
    HvParams p{};
    p.reuse_vsplit = reuse_vsplit;
    p.v_host = v_host_next;
    v_host_next = nullptr;
    p.vplanes = vplanes;
    p.vplanes_ld = vplanes_ld;
    p.xs = xs.as<float>();
    p.n = n;
    p.dp = dp;
    p.row_idx = row_idx;
    p.r0 = rr0;
    p.m = m;
    p.j0 = j0;
    p.j1 = j1;
    p.V = V;
    p.ldv = ldv;
    p.s = s;
    p.out = out;
    p.ldo = ldo;
    p.B = B;
    p.ldb = ldb;
    p.mode = mode;
    p.sf2 = sf2();
    p.a = a_coef();
    p.noise2 = noise2();
    p.diag = static_cast<float>(sf * sf + sigma * sigma);
    p.hyp = dhyp.as<float>();
    p.done = done;
    // shards of the full operator decompose like the whole (bitwise-equal
    // rows); internal row blocks (AP) split for their own size instead
    p.split_rows = (row_idx || !shard_invariant || !split_global) ? 0 : n;
    if ((hv_impl == WGP_HV_TC || hv_impl == WGP_HV_TC_F16) && hv_tc_supported(d, s)) {
      if (!tc.valid) tc.build(xs.as<float>(), n, dp, d, st);
      hv_tc(tc, p, st, hv_impl == WGP_HV_TC_F16);
    } else {
      hv_simt(p, st);
    }
  }
  // full-operator convenience: out (rows all) = H V
  void hv_all(const float* V, int s, float* out, int mode = kHvStore, const float* B = nullptr,
              const int* done = nullptr, const float* vplanes = nullptr) {
    hv(V, ld, s, out, ld, mode, B, ld, 0, n, nullptr, 0, n, done, true, vplanes, vplanes ? ld : 0);
  }

  // ---------------------------------------------------------------- workspace
  SolveCtrl* dctrl() { return ctrl.as<SolveCtrl>(); }
  void ensure_solver_ws(int s) {
    if (!ctrl.p) {
      ctrl.ensure(sizeof(SolveCtrl));
      WGP_CUDA(cudaMemsetAsync(ctrl.p, 0, sizeof(SolveCtrl), st));
    }
    conv.ensure(sizeof(int) * (s + 1));
    rs.ensure(sizeof(double) * (s + 1));
    alpha.ensure(sizeof(double) * (s + 1));
    beta.ensure(sizeof(double) * (s + 1));
    bnorm.ensure(sizeof(double) * (s + 1));
    tol.ensure(sizeof(double) * (s + 1));
    colsum.ensure(sizeof(double) * (s + 1));
    best.ensure(sizeof(double) * (s + 1));
    stall.ensure(sizeof(int) * (s + 1));
    act.ensure(sizeof(int) * (s + 1));
    part.ensure(sizeof(double) * static_cast<size_t>(reduce_blocks(n)) * std::max(s + 2, 2 * s));
    P.ensure(sizeof(float) * ld * s);
    HP.ensure(sizeof(float) * ld * s);
    Rtmp.ensure(sizeof(float) * ld * s);
    if (sharded()) {
      dloc.ensure(sizeof(double) * 2 * std::max(s + 2, 2 * s));
      dall.ensure(sizeof(double) * 2 * std::max(s + 2, 2 * s) * nranks);
    }
  }
  ColState colstate() {
    ColState c{conv.as<int>(), rs.as<double>(), alpha.as<double>(), beta.as<double>(),
               bnorm.as<double>(), tol.as<double>(), best.as<double>(), stall.as<int>(), act.as<int>()};
    c.dist_loc = sharded() ? dloc.as<double>() : nullptr;
    return c;
  }
  // Row-sharded reduction epilogue: the ranks' column totals (left in dloc by
  // the reduction kernel) are all-gathered and summed in rank order, then
  // `kind`'s epilogue runs -- identically on every rank.
  void dist_reduce(int kind, int w, int s, bool fa = false, bool fb = false, double* out = nullptr) {
    comm->all_gather(dloc.as<double>(), dall.as<double>(), static_cast<size_t>(w), st);
    dist_finish(kind, dall.as<double>(), nranks, w, s, colstate(), dctrl(), out, fa, fb, st);
  }
  // all-gather the own rows of s columns (in place; no-op unsharded)
  template <class T>
  void gather_rows(T* base, int s) {
    if (sharded()) comm->gather_rows(base, ld, blk, s, sizeof(T), st);
  }
  // in-place all-gather of equal contiguous chunks: rank r's at base + r chunk
  void gather_rows_raw(double* base, int64_t chunk) {
    if (sharded()) comm->gather_rows(base, chunk * nranks, chunk, 1, sizeof(double), st);
  }
  // column dots over the own rows, summed over the ranks
  template <class T>
  std::vector<double> dots_own(const T* A, const T* B_, int s) {
    ensure_solver_ws(s);
    col_dots(A + own0, B_ + own0, ld, own_m(), s, part.as<double>(), &dctrl()->ticket, colsum.as<double>(), st);
    if (sharded()) {
      comm->all_gather(colsum.as<double>(), dall.as<double>(), static_cast<size_t>(s), st);
      dist_finish(kDistSum, dall.as<double>(), nranks, s, s, colstate(), dctrl(), colsum.as<double>(), false,
                  false, st);
    }
    std::vector<double> h(s);
    WGP_CUDA(cudaMemcpyAsync(h.data(), colsum.p, sizeof(double) * s, cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    return h;
  }
  // host vector summed over the ranks in rank order (identical on every rank)
  void sum_over_ranks(std::vector<double>& v) {
    if (!sharded() || v.empty()) return;
    const size_t w = v.size();
    Buf& sb = dloc;
    Buf& rb = dall;
    sb.ensure(sizeof(double) * w);
    rb.ensure(sizeof(double) * w * nranks);
    WGP_CUDA(cudaMemcpyAsync(sb.p, v.data(), sizeof(double) * w, cudaMemcpyHostToDevice, st));
    comm->all_gather(sb.as<double>(), rb.as<double>(), w, st);
    std::vector<double> all(w * nranks);
    WGP_CUDA(cudaMemcpyAsync(all.data(), rb.p, sizeof(double) * w * nranks, cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    for (size_t k = 0; k < w; ++k) {
      double t = 0.0;
      for (int r = 0; r < nranks; ++r) t += all[r * w + k];
      v[k] = t;
    }
  }
  // column dots over rows [r, r + m)
  std::vector<double> dots_rows(const float* A, const float* B_, int s, int64_t r, int64_t m) {
    ensure_solver_ws(s);
    col_dots(A + r, B_ + r, ld, m, s, part.as<double>(), &dctrl()->ticket, colsum.as<double>(), st);
    std::vector<double> h(s);
    WGP_CUDA(cudaMemcpyAsync(h.data(), colsum.p, sizeof(double) * s, cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    return h;
  }
  template <class T>
  std::vector<double> dots(const T* A, const T* B_, int s) {
    ensure_solver_ws(s);
    col_dots(A, B_, ld, n, s, part.as<double>(), &dctrl()->ticket, colsum.as<double>(), st);
    std::vector<double> h(s);
    WGP_CUDA(cudaMemcpyAsync(h.data(), colsum.p, sizeof(double) * s, cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    return h;
  }
  void reset_ctrl(int max_it) {
    SolveCtrl h{};
    h.max_it = max_it;
    WGP_CUDA(cudaMemcpyAsync(ctrl.p, &h, sizeof(SolveCtrl), cudaMemcpyHostToDevice, st));
  }
  const SolveCtrl& poll() {
    WGP_CUDA(cudaMemcpyAsync(hctrl.h, ctrl.p, sizeof(SolveCtrl), cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    return *hctrl.h;
  }
  void lazy_handles() {
    if (!cublas) {
      if (cublasCreate(&cublas) != CUBLAS_STATUS_SUCCESS) throw DeviceError("cublasCreate failed");
      cublasSetStream(cublas, st);
      constexpr size_t kWs = size_t(32) << 20;
      cublas_ws.ensure(kWs);
      cublasSetWorkspace(cublas, cublas_ws.p, kWs);
    }
    if (!cusolver) {
      if (cusolverDnCreate(&cusolver) != CUSOLVER_STATUS_SUCCESS) throw DeviceError("cusolverDnCreate failed");
      cusolverDnSetStream(cusolver, st);
    }
  }

  // ---------------------------------------------------------------- solvers
  struct SolveOut {
    int iterations = 0;
    std::vector<double> rel;
    std::vector<int> conv;
    bool r_exact = false;  // the solver's residual at exit is B - H X computed from scratch
  };

  static void validate(const wgp_solver_cfg& c) {  // proj/src/solvers.cpp:31-37
    if (!(c.tol_mean > 0.0 && c.tol_mean < 1.0) || !(c.tol_samples > 0.0 && c.tol_samples < 1.0))
      throw std::invalid_argument("SolverConfig: tolerances must lie in (0, 1)");
    if (c.block_size < 1) throw std::invalid_argument("SolverConfig: block_size must be >= 1");
    if (c.minibatch_size < 1) throw std::invalid_argument("SolverConfig: minibatch_size must be >= 1");
    if (c.max_iterations < 0) throw std::invalid_argument("SolverConfig: max_iterations must be >= 0");
    if (c.kind < 0 || c.kind > 2) throw std::invalid_argument("solve: unknown solver kind");
  }

  [[noreturn]] void fail(const SolveCtrl& h, int kind) {
    const std::string who = solver_name(kind);
    if (h.status == kStatusNotPd)
      throw NumericalError(kind == 0
                               ? "cg_solve: non-positive curvature encountered, H is not positive definite"
                               : who + ": H is not positive definite");
    if (h.status == kStatusNaN)
      throw NumericalError(who + (kind == 1 ? ": NaN in iterate at epoch " : ": NaN in iterate at iteration ") +
                           std::to_string(h.fail_it));
    throw NumericalError("sgd_solve: iterate diverged at step " + std::to_string(h.fail_it) +
                         "; use a smaller learning rate");
  }

  // solve(H, rhs, init, config), proj/src/solvers.cpp:265-279.  Device
  // pointers with leading dimension ld; init == nullptr means zeros.
  // CG with cg_precision == WGP_CG_F64 runs on fp64 solver state over the
  // fp64-accumulating operator (hv_f64.cu) and rounds X / R to fp32 at exit;
  // init64 (optional) is an fp64 initial guess taking precedence over init,
  // and Xo64 (optional) receives the fp64 solutions (the outer loop's warm
  // start keeps them, proj/src/optimizer.cpp:133-135,158).
  SolveOut solve(const wgp_solver_cfg& cfg, const float* B, const float* init, float* Xo, float* Ro,
                 int s, const double* init64 = nullptr, double* Xo64 = nullptr, const double* B64in = nullptr) {
    require_data();
    validate(cfg);
    if (s < 1) throw std::invalid_argument("solve: rhs needs at least one column");
    ensure_solver_ws(s);
    std::vector<double> bn = dots(B, B, s);
    for (double& v : bn) {
      if (!std::isfinite(v)) throw std::invalid_argument("solve: non-finite right-hand side or init");
      v = std::sqrt(v);
    }
    if (init) {
      for (double v : dots(init, init, s))
        if (!std::isfinite(v)) throw std::invalid_argument("solve: non-finite right-hand side or init");
    }
    std::vector<double> tl(s);
    for (int c = 0; c < s; ++c) tl[c] = c == 0 ? cfg.tol_mean : cfg.tol_samples;  // :49-56
    WGP_CUDA(cudaMemcpyAsync(bnorm.p, bn.data(), sizeof(double) * s, cudaMemcpyHostToDevice, st));
    WGP_CUDA(cudaMemcpyAsync(tol.p, tl.data(), sizeof(double) * s, cudaMemcpyHostToDevice, st));
    SolveOut out;
    std::vector<double> en;
    // Row-sharded contexts: rhs and init hold all rows on every rank; the
    // residuals are formed for the rank's rows [own0, own1) only and the
    // solutions end with all rows on every rank.
    const int64_t r = own0, m = own_m();
    if (sharded() && cfg.kind == WGP_SOLVER_SGD)
      throw std::invalid_argument("sgd_solve: not available on a row-sharded context (use CG or AP)");
    if (cfg.kind == WGP_SOLVER_CG && cg_precision == WGP_CG_F64) {
      const size_t bytes = sizeof(double) * ld * s;
      B64.ensure(bytes);
      X64.ensure(bytes);
      R64.ensure(bytes);
      double* b64 = B64.as<double>();
      double* x64 = X64.as<double>();
      double* r64 = R64.as<double>();
      if (B64in)  // an fp64 caller's rhs, unrounded
        WGP_CUDA(cudaMemcpyAsync(b64, B64in, bytes, cudaMemcpyDeviceToDevice, st));
      else
        widen(B, ld, b64, ld, n, s, st);
      if (init64 || init) {
        if (init64) WGP_CUDA(cudaMemcpy2DAsync(x64, sizeof(double) * ld, init64, sizeof(double) * ld,
                                               sizeof(double) * n, s, cudaMemcpyDeviceToDevice, st));
        else widen(init, ld, x64, ld, n, s, st);
        hv64_rows(x64, ld, s, r64 + r, ld, kHv64Residual, b64, ld, r, m, nullptr);
        if (keep_residuals) {  // B - H X0 for warm_distance_res
          wsd_r0.ensure(bytes);
          WGP_CUDA(cudaMemcpyAsync(wsd_r0.p, r64, bytes, cudaMemcpyDeviceToDevice, st));
        }
      } else {
        WGP_CUDA(cudaMemsetAsync(x64, 0, bytes, st));
        WGP_CUDA(cudaMemcpyAsync(r64, b64, bytes, cudaMemcpyDeviceToDevice, st));
      }
      cg<double>(cfg, b64, x64, r64, s, out);
      // finalize_exact_residuals (:69-77) on the fp64 iterate
      Rt64.ensure(bytes);
      double* e64 = Rt64.as<double>();
      hv64_rows(x64, ld, s, e64 + r, ld, kHv64Residual, b64, ld, r, m, nullptr);
      en = dots_own(e64, e64, s);
      wsd_res = WsdRes{e64, 64, init64 || init};
      narrow(x64, ld, Xo, ld, n, s, st);
      narrow(r64 + r, ld, Ro + r, ld, m, s, st);
      if (Xo64) WGP_CUDA(cudaMemcpy2DAsync(Xo64, sizeof(double) * ld, x64, sizeof(double) * ld,
                                           sizeof(double) * n, s, cudaMemcpyDeviceToDevice, st));
    } else {
      // X = init; R = rhs - H X (exactly rhs for a zero init)
      if (init) {
        copy_cols(init, ld, Xo, ld, n, s, st);
        hv(Xo, ld, s, Ro + r, ld, kHvResidual, B, ld, 0, n, nullptr, r, m);
        if (keep_residuals) {
          const size_t bytes = sizeof(float) * ld * s;
          wsd_r0.ensure(bytes);
          WGP_CUDA(cudaMemcpyAsync(wsd_r0.p, Ro, bytes, cudaMemcpyDeviceToDevice, st));
        }
      } else {
        fill_zero(Xo, ld, n, s, st);
        copy_cols(B, ld, Ro, ld, n, s, st);
      }
      if (cfg.kind == WGP_SOLVER_CG) cg<float>(cfg, B, Xo, Ro, s, out);
      else if (cfg.kind == WGP_SOLVER_AP) ap(cfg, B, Xo, Ro, s, out);
      else sgd(cfg, B, Xo, Ro, s, out);
      // finalize_exact_residuals, :69-77 (AP whose last epoch closed with the
      // exact residual: that is this product, same kernel and arguments)
      float* E = Rtmp.as<float>();
      if (out.r_exact) {
        en = dots_own(Ro, Ro, s);
        wsd_res = WsdRes{Ro, 32, init != nullptr};
      } else {
        hv(Xo, ld, s, E + r, ld, kHvResidual, B, ld, 0, n, nullptr, r, m);
        en = dots_own(E, E, s);
        wsd_res = WsdRes{E, 32, init != nullptr};
      }
    }
    out.rel.resize(s);
    for (int c = 0; c < s; ++c) out.rel[c] = bn[c] > 0.0 ? std::sqrt(en[c]) / bn[c] : 0.0;
    out.conv.resize(s);
    WGP_CUDA(cudaMemcpyAsync(out.conv.data(), conv.p, sizeof(int) * s, cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    for (int& c : out.conv) c = c == 1 || c == 2;  // 3: stalled, frozen at its best iterate
    return out;
  }

  // CG iterations as CUDA graphs: after the first 10 iterations (eager, which
  // also sizes every workspace) the loop replays a captured 10-iteration chunk
  // (or its variant whose last iteration is the residual refresh, :111).  At
  // small n a CG iteration is launch-bound (~150 us eager at config 0 for
  // ~10 us of GPU work).  Graphs are cached per (B, X, R, s, hv_impl) across
  // solves -- the H.V kernels read the hyperparameter scalars from device
  // memory -- and re-captured when any device workspace was reallocated.
  struct CgGraph {
    const void* B;
    const void* Xo;
    const void* R;
    int s, impl;
    uint64_t gen;
    cudaGraphExec_t exec[2];
  };
  std::vector<CgGraph> cg_graphs;
  // One AP epoch (every block step + the exact residual + the convergence
  // check) as a graph, cached like the CG ones and keyed on the block size:
  // at config 2 an epoch is 42 blocks of ~6 launches each with only a few us
  // of GPU work per launch.
  struct ApGraph {
    const float* B;
    float* Xo;
    float* R;
    int s, impl;
    int64_t bs;
    int exact;  // the epoch's closing residual from scratch
    uint64_t gen;
    cudaGraphExec_t exec;
  };
  std::list<ApGraph> ap_graphs;  // stable addresses: a solve holds pointers to two of them
  void drop_cg_graphs() {  // and the AP epoch graphs
    for (auto& g : cg_graphs)
      for (auto e : g.exec)
        if (e) cudaGraphExecDestroy(e);
    cg_graphs.clear();
    for (auto& g : ap_graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    ap_graphs.clear();
  }

  // fp64 CG operator: out = H V (store) or B - H V (residual) for output rows
  // [rr0, rr0 + m), fp64 V (all n rows) / out / B (hv_f64.cu).
  Hv64Params hv64_params(const double* V, int64_t ldv, int s, double* out, int64_t ldo, int mode, const double* B,
                         int64_t ldb, int64_t rr0, int64_t m, const int* done) {
    Hv64Params q{};
    q.xs = xs.as<float>();
    q.n = n;
    q.dp = dp;
    q.d = d;
    q.r0 = rr0;
    q.m = m;
    q.V = V;
    q.ldv = ldv;
    q.s = s;
    q.out = out;
    q.ldo = ldo;
    q.B = B;
    q.ldb = ldb;
    q.mode = mode;
    q.hyp = dhyp.as<float>();
    q.done = done;
    return q;
  }
  void hv64_rows(const double* V, int64_t ldv, int s, double* out, int64_t ldo, int mode, const double* B,
                 int64_t ldb, int64_t rr0, int64_t m, const int* done) {
    Hv64Params q{};
    q.xs = xs.as<float>();
    q.n = n;
    q.dp = dp;
    q.d = d;
    q.r0 = rr0;
    q.m = m;
    q.ldv = ldv;
    q.ldo = ldo;
    q.ldb = ldb;
    q.mode = mode;
    q.hyp = dhyp.as<float>();
    q.done = done;
    for (int c0 = 0; c0 < s; c0 += 80) {  // one workspace per chunk of <= 80 columns
      const int sc = std::min(80, s - c0);
      hv64_ws.ensure(hv64_workspace_bytes(n, m, sc));
      Hv64Params r = q;
      r.s = sc;
      r.V = V + c0 * ldv;
      r.out = out + c0 * ldo;
      r.B = B ? B + c0 * ldb : nullptr;
      r.part = hv64_ws.as<double>();
      hv64(r, st);
    }
  }
  void hv64_all(const double* V, int s, double* out, int mode, const double* B, const int* done) {
    hv64_rows(V, ld, s, out, ld, mode, B, ld, 0, n, done);
  }

  // The operator of a CG iteration in the solver-state precision T: float
  // runs the configured fp32 engine (P's tf32 planes kept by the direction
  // kernels), double the fp64-accumulating symmetric engine (hv_f64.cu).
  // (output rows [own0, own1): the rank's rows; out / B indexed by global row)
  void cg_hv(const float* V, int s, float* out, int mode, const float* B, const int* done, const float* vplanes) {
    hv(V, ld, s, out + own0, ld, mode, B, ld, 0, n, nullptr, own0, own_m(), done, true, vplanes,
       vplanes ? ld : 0);
  }
  void cg_hv(const double* V, int s, double* out, int mode, const double* B, const int* done, const float*) {
    hv64_rows(V, ld, s, out + own0, ld, mode == kHvResidual ? kHv64Residual : kHv64Store, B, ld, own0, own_m(),
              done);
  }

  template <class T>
  void cg(const wgp_solver_cfg& cfg, const T* B, T* Xo, T* R, int s, SolveOut& out) {
    constexpr bool f64 = std::is_same<T, double>::value;
    const int max_it = cfg.max_iterations > 0 ? cfg.max_iterations : static_cast<int>(10 * n);
    reset_ctrl(max_it);
    Buf& Pbuf = f64 ? P64 : P;
    Buf& HPbuf = f64 ? HP64 : HP;
    Buf& Rtbuf = f64 ? Rt64 : Rtmp;
    Pbuf.ensure(sizeof(T) * ld * s);
    HPbuf.ensure(sizeof(T) * ld * s);
    Rtbuf.ensure(sizeof(T) * ld * s);
    T* Pp = Pbuf.as<T>();
    T* HPp = HPbuf.as<T>();
    T* Rt = Rtbuf.as<T>();
    const ColState cs = colstate();
    SolveCtrl* c = dctrl();
    double* pt = part.as<double>();
    Buf& Xbbuf = f64 ? Xbest64 : Xbest;
    Buf& Rbbuf = f64 ? Rbest64 : Rbest;
    Xbbuf.ensure(sizeof(T) * ld * s);
    Rbbuf.ensure(sizeof(T) * ld * s);
    T* Xb = Xbbuf.as<T>();
    T* Rb = Rbbuf.as<T>();
    float* PPp = nullptr;
    if (!f64 && !sharded()) {  // (sharded: the H.V splits the gathered P itself -- one all-gather, not three)
      PP.ensure(sizeof(float) * 2 * ld * s);  // P's tf32 planes: the H.V skips its split of P
      PPp = PP.as<float>();
    }
    // Vector work on the rank's rows [own0, own1) (all rows unsharded); a
    // sharded iteration all-gathers the direction before its H.V and the
    // iterate before a residual refresh, and finishes every column reduction
    // on the ranks' rank-order sum (dist_reduce).
    const int64_t r = own0, m = own_m();
    const bool sh = sharded();
    float* PPr = PPp ? PPp + r : nullptr;
    cg_init(R + r, ld, m, s, cs, pt, c, st);
    if (sh) dist_reduce(kDistInit, s, s);
    cg_seed(Pp + r, R + r, ld, m, s, cs.conv, st, PPr);
    cg_snapshot(Xo + r, R + r, Xb + r, Rb + r, ld, m, s, cs, c, true, st);
    const int* done = &c->done;
    static const bool no_fused = getenv("WGP_CG_NO_FUSED") != nullptr;
    bool use_fused = !no_fused;
    auto iteration = [&](bool refresh) {
      if (sh) gather_rows(Pp, s);
      // fp64, unsharded: hv64's split reduction runs inside cg_fused (HvFold)
      static const bool no_fold = getenv("WGP_CG_NO_FOLD") != nullptr;
      if (f64 && !refresh && !sh && use_fused && !no_fold) {
        HvFold fold;
        Hv64Params q = hv64_params(reinterpret_cast<const double*>(Pp), ld, s, reinterpret_cast<double*>(HPp), ld,
                                   kHv64Store, nullptr, ld, 0, n, done);
        hv64_ws.ensure(hv64_workspace_bytes(n, n, s));
        q.part = hv64_ws.as<double>();
        if (hv64_partials(q, st, &fold.splits, &fold.m_pad)) {
          fold.part = q.part;
          fold.hyp = q.hyp;
          if (cg_fused(Xo, R, Pp, HPp, ld, n, s, cs, pt, c, st, PPp, fold)) return;
          use_fused = false;  // (the partials are re-formed below)
        }
      }
      cg_hv(Pp, s, HPp, kHvStore, nullptr, done, PPp);
      if (!refresh && !sh && use_fused) {  // alpha + update + direction in one cooperative kernel
        if (cg_fused(Xo, R, Pp, HPp, ld, n, s, cs, pt, c, st, PPp)) return;
        use_fused = false;
      }
      cg_alpha(Pp + r, HPp + r, ld, m, s, cs, pt, c, st);
      if (sh) dist_reduce(kDistAlpha, s, s);
      if (!refresh) {
        cg_update(Xo + r, R + r, Pp + r, HPp + r, ld, m, s, cs, pt, c, false, st);
        if (sh) dist_reduce(kDistBeta, s, s);
      } else {
        cg_update(Xo + r, R + r, Pp + r, HPp + r, ld, m, s, cs, pt, c, true, st);
        if (sh) gather_rows(Xo, s);
        cg_hv(Xo, s, Rt, kHvResidual, B, done, nullptr);
        cg_refresh_norm(R + r, Rt + r, ld, m, s, cs, pt, c, st);
        if (sh) dist_reduce(kDistRefresh, s, s);
        cg_snapshot(Xo + r, R + r, Xb + r, Rb + r, ld, m, s, cs, c, false, st);
      }
      cg_direction(Pp + r, R + r, ld, m, s, cs, pt, c, st, PPr);
    };
    // every rank ends with all rows of the solutions
    struct GatherAtExit {
      Ctx* self;
      T* X;
      int s;
      ~GatherAtExit() {
        if (self->sharded()) {
          try {
            self->gather_rows(X, s);
          } catch (...) {
          }
        }
      }
    } gather_at_exit{this, Xo, s};
    static const bool no_graphs = getenv("WGP_NO_GRAPHS") != nullptr;
    constexpr int kChunk = 10;
    const int impl = f64 ? -1 : hv_impl;
    int launched = 0;
    const int eager[3] = {2, 4, 4};  // first kChunk iterations, polled early
    for (int e = 0; e < 3; ++e) {
      const SolveCtrl& h = poll();
      if (h.done) {
        if (h.status != kStatusOk) fail(h, 0);
        out.iterations = h.it;
        return;
      }
      for (int k = 0; k < eager[e]; ++k) iteration(++launched % 50 == 0);
    }
    CgGraph* gr = nullptr;
    if (!no_graphs && graphs_ok()) {
      const uint64_t gen = alloc_generation().load();
      for (auto& g : cg_graphs)
        if (g.B == B && g.Xo == Xo && g.R == R && g.s == s && g.impl == impl) gr = &g;
      if (gr && gr->gen != gen) {
        drop_cg_graphs();
        gr = nullptr;
      }
      if (!gr) {
        if (cg_graphs.size() >= 8) drop_cg_graphs();
        CgGraph g{B, Xo, R, s, impl, gen, {nullptr, nullptr}};
        // capture; a failed capture with the cooperative fused kernel is
        // retried once with the three-kernel iteration
        bool ok = false;
        for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
          ok = true;
          for (int v = 0; v < 2 && ok; ++v) {
            cudaGraph_t graph = nullptr;
            WGP_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            for (int k = 0; k < kChunk; ++k) iteration(v == 1 && k == kChunk - 1);
            const cudaError_t ce = cudaStreamEndCapture(st, &graph);
            ok = ce == cudaSuccess && graph && cudaGraphInstantiate(&g.exec[v], graph, 0) == cudaSuccess;
            if (graph) cudaGraphDestroy(graph);
          }
          if (!ok) {
            cudaGetLastError();
            for (auto& e : g.exec)
              if (e) cudaGraphExecDestroy(e), e = nullptr;
            if (!use_fused) break;
            use_fused = false;
          }
        }
        if (!ok) {
          // capture unavailable (e.g. a collective that cannot be captured):
          // eager iterations from here on
        } else if (alloc_generation().load() != gen) {  // a workspace moved while capturing
          for (auto e : g.exec) cudaGraphExecDestroy(e);
        } else {
          cg_graphs.push_back(g);
          gr = &cg_graphs.back();
        }
      }
    }
    while (true) {
      const SolveCtrl& h = poll();
      if (h.done) {
        if (h.status != kStatusOk) fail(h, 0);
        out.iterations = h.it;
        return;
      }
      if (gr) {
        const bool refresh = (launched + kChunk) % 50 == 0;
        WGP_CUDA(cudaGraphLaunch(gr->exec[refresh ? 1 : 0], st));
        launched += kChunk;
      } else {
        for (int k = 0; k < kChunk; ++k) iteration(++launched % 50 == 0);
      }
    }
  }

  // Factor every diagonal block of size bs once (solvers.cpp:151-165): H[b,b]
  // in fp64 (the last, partial block padded with the identity), one batched
  // cuSOLVER Cholesky over all blocks, then the explicit inverses H_bb^-1
  // (hbuf, ap_bs): each Gauss-Seidel step is one DGEMM.  Returns the count.
  int64_t ap_factor(int64_t bs) {
    lazy_handles();
    const int64_t nb = ceil_div(n, bs);
    // Factor every diagonal block once per solve (:151-165): H[b,b] in fp64
    // (the last, partial block padded with the identity), one batched
    // cuSOLVER Cholesky over all blocks, then the explicit inverses below.
    // (Per-block potrf + potri and a symm per step cost ~20 small launches per
    // block and 0.4 ms per symm, measured.)  Row-sharded contexts factor
    // their contiguous share of the blocks and all-gather the inverses (every
    // rank applies every block's solve).
    const bool sh = sharded();
    const int64_t nbr = sh ? ceil_div(nb, nranks) : nb;  // blocks per rank
    const int64_t b0 = sh ? std::min<int64_t>(nb, rank * nbr) : 0, b1 = sh ? std::min<int64_t>(nb, b0 + nbr) : nb;
    const int64_t nown = b1 - b0;
    const size_t bb = static_cast<size_t>(bs) * bs;
    hbuf.ensure(sizeof(double) * bb * static_cast<size_t>(sh ? nbr * nranks : nb));
    info.ensure(sizeof(int) * std::max<int64_t>(1, nown));
    WGP_CUDA(cudaMemsetAsync(info.p, 0, sizeof(int) * std::max<int64_t>(1, nown), st));
    const double sf2d = sf * sf, ad = sf * sf * kLn2, n2d = sigma * sigma;
    std::vector<double*> hptr(std::max<int64_t>(1, nown));
    for (int64_t b = b0; b < b1; ++b) {
      const int64_t start = b * bs, size = std::min(bs, n - start);
      hptr[b - b0] = hbuf.as<double>() + static_cast<size_t>(b) * bb;
      build_block(xs.as<float>(), dp, start, size, bs, sf2d, ad, n2d, hptr[b - b0], st);
    }
    bool failed = false;
    if (nown > 0) {
      lapack_work.ensure(sizeof(double*) * nown);
      WGP_CUDA(cudaMemcpyAsync(lapack_work.p, hptr.data(), sizeof(double*) * nown, cudaMemcpyHostToDevice, st));
      if (cusolverDnDpotrfBatched(cusolver, CUBLAS_FILL_MODE_LOWER, static_cast<int>(bs),
                                  reinterpret_cast<double**>(lapack_work.p), static_cast<int>(bs), info.as<int>(),
                                  static_cast<int>(nown)) != CUSOLVER_STATUS_SUCCESS)
        throw DeviceError("cusolverDnDpotrfBatched failed");
      std::vector<int> hinfo(nown);
      WGP_CUDA(cudaMemcpyAsync(hinfo.data(), info.p, sizeof(int) * nown, cudaMemcpyDeviceToHost, st));
      WGP_CUDA(cudaStreamSynchronize(st));
      for (int v : hinfo) failed = failed || v != 0;
    }
    if (sh) {  // every rank raises the same error
      std::vector<double> f{failed ? 1.0 : 0.0};
      sum_over_ranks(f);
      failed = f[0] > 0.0;
    }
    if (failed) throw NumericalError("ap_solve: diagonal block factorization failed, H is not positive definite");
    // H_bb^-1 = L^-T L^-1 for all blocks: batched triangular solve against the
    // identity, then a strided-batched GEMM (per-block cublasDtrsm in the
    // epoch loop expanded to ~30 kernels, ~0.5 ms per block, measured); each
    // Gauss-Seidel step is then one DGEMM.
    if (nown > 0) {
      linv.ensure(sizeof(double) * bb * nown);
      identities(linv.as<double>(), bs, nown, st);
      std::vector<double*> lptr(nown);
      for (int64_t b = 0; b < nown; ++b) lptr[b] = linv.as<double>() + b * bb;
      Buf& lp = linv_ptrs;  // persistent: a fresh allocation would invalidate the cached graphs
      lp.ensure(sizeof(double*) * nown);
      WGP_CUDA(cudaMemcpyAsync(lp.p, lptr.data(), sizeof(double*) * nown, cudaMemcpyHostToDevice, st));
      const double one_ = 1.0, zero_ = 0.0;
      if (cublasDtrsmBatched(cublas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                             static_cast<int>(bs), static_cast<int>(bs), &one_,
                             reinterpret_cast<const double* const*>(lapack_work.p), static_cast<int>(bs),
                             reinterpret_cast<double* const*>(lp.p), static_cast<int>(bs),
                             static_cast<int>(nown)) != CUBLAS_STATUS_SUCCESS)
        throw DeviceError("cublasDtrsmBatched failed");
      if (cublasDgemmStridedBatched(cublas, CUBLAS_OP_T, CUBLAS_OP_N, static_cast<int>(bs), static_cast<int>(bs),
                                    static_cast<int>(bs), &one_, linv.as<double>(), static_cast<int>(bs),
                                    static_cast<long long>(bb), linv.as<double>(), static_cast<int>(bs),
                                    static_cast<long long>(bb), &zero_, hbuf.as<double>() + b0 * bb,
                                    static_cast<int>(bs), static_cast<long long>(bb),
                                    static_cast<int>(nown)) != CUBLAS_STATUS_SUCCESS)
        throw DeviceError("cublasDgemmStridedBatched failed");
    }
    if (sh) gather_rows_raw(hbuf.as<double>(), nbr * bb);  // rank r's blocks [r nbr, (r + 1) nbr)
    ap_bs = bs;
    return nb;
  }
  // delta = H_bb^-1 R_b for block b of the last ap_factor (device fp64,
  // column-major size x s, leading dimension size).
  void ap_block_solve(int64_t b, const double* Rbp, int s, double* delta) {
    if (ap_bs <= 0) throw std::invalid_argument("ap_block_solve: call ap_factor first");
    const int64_t nb = ceil_div(n, ap_bs);
    if (b < 0 || b >= nb) throw std::invalid_argument("ap_block_solve: block index out of range");
    const int64_t start = b * ap_bs, size = std::min(ap_bs, n - start);
    const double one = 1.0, zero = 0.0;
    const double* Hinv = hbuf.as<double>() + static_cast<size_t>(b) * ap_bs * ap_bs;
    if (cublasDgemm(cublas, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(size), s, static_cast<int>(size), &one, Hinv,
                    static_cast<int>(ap_bs), Rbp, static_cast<int>(size), &zero, delta,
                    static_cast<int>(size)) != CUBLAS_STATUS_SUCCESS)
      throw DeviceError("cublasDgemm failed");
  }

  void ap(const wgp_solver_cfg& cfg, const float* B, float* Xo, float* R, int s, SolveOut& out) {
    lazy_handles();
    const int max_ep = cfg.max_iterations > 0 ? cfg.max_iterations : 1000;
    const int64_t bs = std::min<int64_t>(std::max(cfg.block_size, 1), n);
    const int64_t nb = ap_factor(bs);
    Rb.ensure(sizeof(double) * bs * s);
    constexpr int kSplitK = 4;  // block solve as 4 K-slices (a 1000 x 65 output is only 64 cuBLAS tiles)
    D64.ensure(sizeof(double) * bs * s * kSplitK);
    DX.ensure(sizeof(float) * ld * s);
    DXP.ensure(sizeof(float) * 2 * ld * s);  // tf32 planes of DX (no per-block re-split)
    reset_ctrl(max_ep);
    const ColState cs = colstate();
    SolveCtrl* c = dctrl();
    double* pt = part.as<double>();
    // Row-sharded AP: R holds the exact residual of the rank's rows; X and
    // the epoch's deltas DX stay replicated (every rank applies the same
    // delta_b); block b's residual R_b = R0_b - H[b, 0:start] DX[0:start] is
    // a sum of per-rank shares -- the R0 rows the rank owns minus the
    // contraction over its 1/nranks slice of the columns [0, start) -- summed
    // by an all-reduce, so every rank solves the same delta_b = H_bb^-1 R_b.
    const bool sh = sharded();
    const int64_t r = own0, m = own_m();
    if (sh) {
      Rpart.ensure(sizeof(float) * bs * s);
      fill_zero(DX.as<float>(), ld, n, s, st);  // the column slices read DX rows of any rank
    }
    norms_convergence(R + r, ld, m, s, cs, pt, c, false, true, st);  // :172-178
    if (sh) dist_reduce(kDistNorms, s, s, false, true);
    const double one = 1.0, zero = 0.0;
    // The epoch's closing residual (:188).  `exact`: R = B - H X from scratch
    // (n^2 entries).  Otherwise, unsharded: R = R0 - H dX, completed block by
    // block -- R[b] already holds R0_b - H[b, 0:start] dX[0:start] from the
    // block step, so R[b] -= H[b, start:n] dX[start:n] adds the rest: n^2 / 2
    // entries, an epoch of n^2 instead of 1.5 n^2 (the triangle of the block
    // steps plus this one).  Equal in exact arithmetic; every kApExact-th epoch
    // is exact, so fp32 rounding cannot accumulate across epochs.
    auto epoch = [&](bool exact) {
      for (int64_t b = 0; b < nb; ++b) {  // :183-187
        const int64_t start = b * bs, size = std::min(bs, n - start);
        const double* Hinv = hbuf.as<double>() + static_cast<size_t>(b) * bs * bs;
        if (sh) {
          float* rp = Rpart.as<float>();
          masked_rows(R, ld, start, size, own0, own1, s, rp, c, st);
          const int64_t j0 = start * rank / nranks, j1 = start * (rank + 1) / nranks;
          if (j1 > j0)
            hv(DX.as<float>(), ld, s, rp, size, kHvSubtract, nullptr, 0, j0, j1, nullptr, start, size, &c->done,
               false, DXP.as<float>(), ld);
          widen_block(rp, Rb.as<double>(), size, s, c, st);
          comm->all_reduce_sum(Rb.as<double>(), static_cast<size_t>(size) * s, st);
        } else {
        // Block residual, left-looking over the earlier blocks only: R is the
        // exact residual at the epoch start (R0), and this epoch changed X
        // only in blocks < b, by DX = their deltas, so
        //   R_b = R0_b - H[b, 0:start] DX[0:start]
        // -- the reference's incrementally updated R_b (R -= H[:, b'] delta
        // after every block b', :186) computed when it is needed.  Contracting
        // `size` rows against the `start` earlier points splits into long J
        // ranges (the right-looking update over n rows with only `size`
        // contracted points ran ~32 tiles per CTA, dominated by the per-CTA
        // fixed cost: 0.75 s per config-3 epoch), and the triangle costs
        // n^2 / 2 entries per epoch where B_b - H[b, :] X cost n^2.
        if (b > 0) hv(DX.as<float>(), ld, s, R + start, ld, kHvResidual, R, ld, 0, start, nullptr, start, size,
                      &c->done, false, DXP.as<float>(), ld);
        ap_gather(R, ld, start, size, s, Rb.as<double>(), c, st);
        }
        // delta = H_bb^-1 R_b (:185); full blocks as kSplitK K-slices in one
        // strided-batched DGEMM (partials summed in fixed order by ap_apply):
        // the single DGEMM ran 64 CTAs over K = 1000, ~16 us per block
        int kparts = 1;
        if (size == bs && bs % kSplitK == 0) {
          const int kc = static_cast<int>(bs / kSplitK);
          kparts = kSplitK;
          if (cublasDgemmStridedBatched(cublas, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(size), s, kc, &one, Hinv,
                                        static_cast<int>(bs), static_cast<long long>(kc) * bs, Rb.as<double>(),
                                        static_cast<int>(size), kc, &zero, D64.as<double>(), static_cast<int>(size),
                                        static_cast<long long>(size) * s, kSplitK) != CUBLAS_STATUS_SUCCESS)
            throw DeviceError("cublasDgemmStridedBatched failed (AP block solve)");
        } else {
          if (cublasDgemm(cublas, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(size), s, static_cast<int>(size), &one,
                          Hinv, static_cast<int>(bs), Rb.as<double>(), static_cast<int>(size), &zero,
                          D64.as<double>(), static_cast<int>(size)) != CUBLAS_STATUS_SUCCESS)
            throw DeviceError("cublasDgemm failed (AP block solve)");
        }
        ap_apply(Xo, ld, start, size, s, D64.as<double>(), kparts, DX.as<float>(), DXP.as<float>(), c, st);
      }
      if (exact || sh) {
        hv(Xo, ld, s, R + r, ld, kHvResidual, B, ld, 0, n, nullptr, r, m);  // :188
      } else {
        for (int64_t b = 0; b < nb; ++b) {
          const int64_t start = b * bs, size = std::min(bs, n - start);
          hv(DX.as<float>(), ld, s, R + start, ld, kHvSubtract, nullptr, 0, start, n, nullptr, start, size,
             &c->done, false, DXP.as<float>(), ld);
        }
      }
      norms_convergence(R + r, ld, m, s, cs, pt, c, true, true, st);  // :189-191
      if (sh) dist_reduce(kDistNorms, s, s, true, true);
    };
    static const int kApExact = [] {
      const char* e = getenv("WGP_AP_EXACT_EVERY");  // 1: every epoch exact (the reference's form)
      return e ? std::max(1, atoi(e)) : 10;
    }();
    static const bool no_graphs = getenv("WGP_NO_GRAPHS") != nullptr;
    bool eager_done[2] = {false, false};  // one eager epoch of each form first: every workspace exists
    bool tried[2] = {false, false};       // one capture attempt per form and solve
    ApGraph* gr[2] = {nullptr, nullptr};
    bool last_exact = true;  // R at entry is exact (B - H X0, or B)
    for (int e = 0;; ++e) {
      const SolveCtrl& h = poll();
      if (h.done) {
        if (h.status != kStatusOk) fail(h, 1);
        out.iterations = h.it;
        out.r_exact = last_exact;
        return;
      }
      // exact closing residual every kApExact epochs and in the last epoch of
      // the budget (finalize then reuses it instead of another product)
      const int x = (e % kApExact == kApExact - 1 || e == max_ep - 1 || sh) ? 1 : 0;
      last_exact = x == 1;
      // a workspace grown by an eager epoch of the other form (e.g. the first
      // exact residual over all rows) invalidates the graphs captured before it
      for (int k = 0; k < 2; ++k)
        if (gr[k] && gr[k]->gen != alloc_generation().load()) {
          gr[k] = nullptr;
          tried[k] = false;
          eager_done[k] = false;
        }
      if (!gr[x] && !tried[x] && eager_done[x] && !no_graphs && !tc.profiling && graphs_ok()) {
        tried[x] = true;
        auto ep = [&]() { epoch(x == 1); };
        gr[x] = ap_graph(B, Xo, R, s, bs, x, ep);
      }
      if (gr[x])
        WGP_CUDA(cudaGraphLaunch(gr[x]->exec, st));
      else
        epoch(x == 1);
      eager_done[x] = true;
    }
  }
  template <class F>
  ApGraph* ap_graph(const float* B, float* Xo, float* R, int s, int64_t bs, int exact, F& epoch) {
    const uint64_t gen = alloc_generation().load();
    for (auto& g : ap_graphs)
      if (g.B == B && g.Xo == Xo && g.R == R && g.s == s && g.impl == hv_impl && g.bs == bs && g.exact == exact &&
          g.gen == gen)
        return &g;
    if (ap_graphs.size() >= 6) {  // evict other solves' graphs (this solve may hold the other form's)
      for (auto it = ap_graphs.begin(); it != ap_graphs.end();) {
        if (it->B == B && it->Xo == Xo && it->R == R && it->s == s && it->bs == bs) {
          ++it;
        } else {
          cudaGraphExecDestroy(it->exec);
          it = ap_graphs.erase(it);
        }
      }
    }
    cudaGraph_t graph = nullptr;
    WGP_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    bool ok = true;
    try {
      epoch();
    } catch (...) {
      ok = false;
    }
    const cudaError_t ee = cudaStreamEndCapture(st, &graph);
    cudaGraphExec_t exec = nullptr;
    if (ok && ee == cudaSuccess && graph && alloc_generation().load() == gen)
      ok = cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
    else
      ok = false;
    if (graph) cudaGraphDestroy(graph);
    if (!ok) {  // eager epochs from here on (capture unsupported for a library call, or a workspace moved)
      if (exec) cudaGraphExecDestroy(exec);
      cudaGetLastError();
      return nullptr;
    }
    ap_graphs.push_back(ApGraph{B, Xo, R, s, hv_impl, bs, exact, gen, exec});
    return &ap_graphs.back();
  }

  void sgd(const wgp_solver_cfg& cfg, const float* B, float* Xo, float* R, int s, SolveOut& out) {
    const int64_t m = std::min<int64_t>(std::max(cfg.minibatch_size, 1), n);
    const int max_steps = cfg.max_iterations > 0 ? cfg.max_iterations : static_cast<int>((100 * n) / m);
    vel.ensure(sizeof(float) * ld * s);
    fill_zero(vel.as<float>(), ld, n, s, st);
    // X's tf32 planes, kept current by sgd_scatter: the minibatch H.V then
    // skips re-splitting all of X every step (10 us per config-2 step)
    XP.ensure(sizeof(float) * 2 * ld * s);
    tf32_planes(Xo, ld, n, s, XP.as<float>(), st);
    batch.ensure(sizeof(float) * m * s);
    constexpr int K = 8;  // steps per host round trip
    // two rounds of indices: round r + 1 is drawn on the host (pinned) while
    // the device runs round r, then copied asynchronously
    idx.ensure(sizeof(int) * m * K * 2);
    sgd_hidx.ensure(sizeof(int) * m * K * 2);
    sgd_xsq.ensure(sizeof(double));
    part.ensure(sizeof(double) * static_cast<size_t>(ceil_div(m, 256)) * 2 * s);  // sgd_step's partials
    double* xsq = sgd_xsq.as<double>();
    reset_ctrl(max_steps);
    const ColState cs = colstate();
    SolveCtrl* c = dctrl();
    double* pt = part.as<double>();
    norms_convergence(R, ld, n, s, cs, pt, c, false, true, st);
    std::vector<int64_t> pool(n);
    std::iota(pool.begin(), pool.end(), 0);
    std::mt19937_64 rng(cfg.seed);
    const float gs = static_cast<float>(static_cast<double>(n) / static_cast<double>(m));
    const float ss = static_cast<float>(cfg.learning_rate / static_cast<double>(n));
    // minibatch index stream, partial Fisher-Yates on the persistent pool
    // (:237-240), in the reference's draw order
    auto draw = [&](int* hidx) {
      for (int k = 0; k < K; ++k)
        for (int64_t i = 0; i < m; ++i) {
          const int64_t j = i + static_cast<int64_t>(uniform_below(rng, static_cast<uint64_t>(n - i)));
          std::swap(pool[i], pool[j]);
          hidx[static_cast<size_t>(k) * m + i] = static_cast<int>(pool[i]);
        }
    };
    // One round = the copy of its K index vectors + K steps, each the
    // minibatch residual H.V (batch = B[I] - H[I, :] X, :241-243) and one
    // sgd_step (momentum scatter, :247-252, with the residual-estimate and
    // iterate norms updated from the minibatch rows' changes, then the checks
    // of :254-258).  The norms are recomputed exactly every kResync rounds.
    // After one eager round sizes every workspace, the two rounds (index
    // halves) replay as captured CUDA graphs: a step is launch-bound
    // otherwise (~5 small launches for ~30 us of GPU work at config 2).
    auto round = [&](int h) {
      const size_t off = static_cast<size_t>(h) * m * K;
      WGP_CUDA(cudaMemcpyAsync(idx.as<int>() + off, sgd_hidx.as<int>() + off, sizeof(int) * m * K,
                               cudaMemcpyHostToDevice, st));
      for (int k = 0; k < K; ++k) {
        const int* ik = idx.as<int>() + off + static_cast<size_t>(k) * m;
        hv(Xo, ld, s, batch.as<float>(), m, kHvResidual, B, ld, 0, n, ik, 0, m, &c->done, true, XP.as<float>(),
           ld);
        sgd_step(Xo, R, vel.as<float>(), ld, ik, m, s, batch.as<float>(), static_cast<float>(cfg.momentum), gs, ss,
                 XP.as<float>(), cs, xsq, pt, c, st);
      }
    };
    static const bool no_graphs = getenv("WGP_NO_GRAPHS") != nullptr;
    cudaGraphExec_t graphs[2] = {nullptr, nullptr};
    struct Drop {
      cudaGraphExec_t* g;
      ~Drop() {
        for (int h = 0; h < 2; ++h)
          if (g[h]) cudaGraphExecDestroy(g[h]);
      }
    } drop{graphs};
    bool eager_done = false, tried = false;
    int cur = 0;
    constexpr int kResync = 8;  // rounds between exact norm re-syncs (fp64 running sums drift ~1e-16 per step)
    int64_t rounds = 0;
    draw(sgd_hidx.as<int>());
    while (true) {
      const SolveCtrl& hc = poll();
      if (hc.done) {
        if (hc.status != kStatusOk) fail(hc, 2);
        out.iterations = hc.it;
        return;
      }
      if (eager_done && !tried && !no_graphs && !tc.profiling) {
        tried = true;
        const uint64_t gen = alloc_generation().load();
        bool ok = true;
        for (int h = 0; h < 2 && ok; ++h) {
          cudaGraph_t graph = nullptr;
          WGP_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
          try {
            round(h);
          } catch (...) {
            ok = false;
          }
          const cudaError_t ee = cudaStreamEndCapture(st, &graph);
          ok = ok && ee == cudaSuccess && graph && alloc_generation().load() == gen &&
               cudaGraphInstantiate(&graphs[h], graph, 0) == cudaSuccess;
          if (graph) cudaGraphDestroy(graph);
        }
        if (!ok) {  // eager rounds from here on
          for (int h = 0; h < 2; ++h)
            if (graphs[h]) cudaGraphExecDestroy(graphs[h]);
          graphs[0] = graphs[1] = nullptr;
          cudaGetLastError();
        }
      }
      if (rounds++ % kResync == 0) sgd_norms(Xo, R, ld, n, s, cs, xsq, pt, c, st);
      if (graphs[cur])
        WGP_CUDA(cudaGraphLaunch(graphs[cur], st));
      else
        round(cur);
      eager_done = true;
      // the next round's indices while the device runs this one (its pinned
      // half was last read by the copy two rounds ago, complete at the poll)
      cur ^= 1;
      draw(sgd_hidx.as<int>() + static_cast<size_t>(cur) * m * K);
    }
  }

  // warm_start_distance, proj/src/estimator.cpp:84-95
  double warm_distance(const float* init, const float* sol, int s) {
    ensure_solver_ws(s);
    float* D = P.as<float>();
    float* HD = HP.as<float>();
    sub_into(init, sol, D, ld, n, s, st);
    hv(D, ld, s, HD + own0, ld, kHvStore, nullptr, 0, 0, n, nullptr, own0, own_m());
    const std::vector<double> q = dots_own(D, HD, s);
    double acc = 0.0;
    for (double v : q) acc += v;
    return std::sqrt(std::max(acc / s / static_cast<double>(n), 0.0));
  }

  // The warm-start distance without another product: H (x0 - x*) =
  // (B - H x*) - (B - H x0) = R_end - R_0, both exact residuals the solve
  // formed anyway (its initial residual, kept when keep_residuals, and the
  // finalize_exact_residuals product).  Same quantity as estimator.cpp:84-95.
  struct WsdRes {
    const void* rend = nullptr;  // exact final residual of the last solve (own rows)
    int prec = 0;                // 32 / 64, 0: none
    bool warm = false;           // the last solve started from an init (R_0 kept)
  };
  WsdRes wsd_res;
  bool keep_residuals = false;
  Buf wsd_r0, wsd_d;
  bool warm_distance_res_ok(int prec) const { return keep_residuals && wsd_res.warm && wsd_res.prec == prec; }
  template <class T>
  double warm_distance_res(const T* init, const T* sol, int s) {
    const size_t bytes = sizeof(T) * ld * s;
    wsd_d.ensure(2 * bytes);
    T* D = wsd_d.as<T>();
    T* HD = D + ld * s;
    diff_cols(init, sol, D, ld, n, s, st);                                      // x0 - x*
    diff_cols(static_cast<const T*>(wsd_res.rend), wsd_r0.as<T>(), HD, ld, n, s, st);  // R_end - R_0
    const std::vector<double> q = dots_own(D, HD, s);
    double acc = 0.0;
    for (double v : q) acc += v;
    return std::sqrt(std::max(acc / s / static_cast<double>(n), 0.0));
  }

  // the same on fp64 solver state over the fp64 operator (fp64 CG)
  double warm_distance64(const double* init, const double* sol, int s) {
    ensure_solver_ws(s);
    const size_t bytes = sizeof(double) * ld * s;
    P64.ensure(bytes);
    HP64.ensure(bytes);
    double* D = P64.as<double>();
    double* HD = HP64.as<double>();
    // D = init - sol
    WGP_CUDA(cudaMemcpyAsync(D, init, bytes, cudaMemcpyDeviceToDevice, st));
    axpy_cols(-1.0, sol, D, ld, n, s, st);
    hv64_rows(D, ld, s, HD + own0, ld, kHv64Store, nullptr, ld, own0, own_m(), nullptr);
    const std::vector<double> q = dots_own(D, HD, s);
    double acc = 0.0;
    for (double v : q) acc += v;
    return std::sqrt(std::max(acc / s / static_cast<double>(n), 0.0));
  }

  // ---------------------------------------------------------------- gradient
  // derivative_contractions for A = vy vy^T / 2, B = coef L R^T (device
  // inputs, ld); raw-space outputs on the host.
  // Rows [gr0, gr0 + gm) against all n points (gm < 0: all rows): a row
  // shard's share of every contraction; the shares of a row partition sum to
  // the full gradient (all outputs are linear in the row sums).
  // Row-sharded contexts (reduce_ranks): each rank contracts its rows and
  // the (d + 2)-vectors are summed over the ranks in rank order.
  void grad(int transform, const double* raw, const float* vy, const float* L, const float* R,
            int s, double coef_b, double* out_a, double* out_b, int64_t gr0 = 0, int64_t gm = -1,
            bool reduce_ranks = false) {
    if (gm < 0) gm = n - gr0;
    std::vector<double> cons(d + 2);
    for (int k = 0; k < d + 2; ++k) cons[k] = transform == 1 ? std::exp(raw[k]) : softplus(raw[k]);
    set_hyper(cons.data());
    if (gm <= 0) {  // a rank without rows contributes zeros
      std::fill(out_a, out_a + d + 2, 0.0);
      std::fill(out_b, out_b + d + 2, 0.0);
    } else {
      grad_rows(transform, raw, vy, L, R, s, coef_b, out_a, out_b, gr0, gm);
    }
    if (reduce_ranks && sharded()) {
      std::vector<double> v(out_a, out_a + d + 2);
      v.insert(v.end(), out_b, out_b + d + 2);
      sum_over_ranks(v);
      std::copy(v.begin(), v.begin() + d + 2, out_a);
      std::copy(v.begin() + d + 2, v.end(), out_b);
    }
  }
  void grad_rows(int transform, const double* raw, const float* vy, const float* L, const float* R,
                 int s, double coef_b, double* out_a, double* out_b, int64_t gr0, int64_t gm) {
    // tensor-core engines (TC, TC_F16) use the tcgen05 gradient where it
    // applies; WGP_GRAD_IMPL=simt forces the CUDA-core kernel
    static const bool force_simt = [] {
      const char* e = getenv("WGP_GRAD_IMPL");
      return e && std::string(e) == "simt";
    }();
    const bool use_tc = hv_impl != WGP_HV_SIMT && !force_simt && grad_tc_supported(d, s);
    GradTcPlan plan;
    if (use_tc) plan = grad_tc_plan(n, gm, d, s);
    const int nblk = use_tc ? plan.nblk : grad_blocks(gm);
    const int W = 2 * (d + 1);
    gpart.ensure(sizeof(double) * nblk * W);
    if (use_tc) gtc_ws.ensure(plan.ws_bytes);
    gout.ensure(sizeof(double) * W);
    GradParams gp{};
    gp.xs = xs.as<float>();
    gp.n = n;
    gp.dp = dp;
    gp.d = d;
    gp.vy = vy;
    gp.L = L;
    gp.R = R;
    gp.ld = ld;
    gp.s = s;
    gp.coef_b = static_cast<float>(coef_b);
    gp.sf2 = sf2();
    gp.a = a_coef();
    gp.part = gpart.as<double>();
    gp.r0 = gr0;
    gp.m = gm;
    if (use_tc)
      grad_tc(gp, plan, gtc_ws.p, st);
    else
      grad_simt(gp, st);
    grad_finalize(gpart.as<double>(), nblk, W, gout.as<double>(), st);
    std::vector<double> acc(W);
    WGP_CUDA(cudaMemcpyAsync(acc.data(), gout.p, sizeof(double) * W, cudaMemcpyDeviceToHost, st));
    const std::vector<double> yy = dots_rows(vy, vy, 1, gr0, gm);
    const std::vector<double> lr = dots_rows(L, R, s, gr0, gm);
    double tb = 0.0;
    for (double v : lr) tb += v;
    auto chain = [&](double r) { return transform == 1 ? std::exp(r) : softplus_derivative(r); };
    const double c2 = kUScale * kUScale;
    for (int k = 0; k < d; ++k) {
      const double scale = 3.0 * sf * sf * chain(raw[k]) / (ls[k] * c2);
      out_a[k] = scale * acc[k];
      out_b[k] = scale * acc[d + 1 + k];
    }
    const double csf = 2.0 * chain(raw[d]) / sf;
    out_a[d] = csf * acc[d];
    out_b[d] = csf * acc[d + 1 + d];
    const double dn = 2.0 * sigma * chain(raw[d + 1]);
    out_a[d + 1] = dn * 0.5 * yy[0];
    out_b[d + 1] = dn * coef_b * tb;
  }

  static double softplus(double x) { return x > 0.0 ? x + std::log1p(std::exp(-x)) : std::log1p(std::exp(x)); }
  static double softplus_inverse(double v) {
    if (!(v > 0.0)) throw std::invalid_argument("softplus_inverse: argument must be positive");
    return v > 0.6931471805599453 ? v + std::log1p(-std::exp(-v)) : std::log(std::expm1(v));
  }
  static double softplus_derivative(double x) {
    if (x > 0.0) return 1.0 / (1.0 + std::exp(-x));
    const double e = std::exp(x);
    return e / (1.0 + e);
  }

  // ---------------------------------------------------------------- RFF probes
  struct DevRff {
    int F = 0, s = 0;
    Buf b, w, eps, om;
    RffBase host;
  };
  void rff_upload(DevRff& r, int F, int s, uint64_t seed) {
    r.host = rff_base_host(n, d, F, s, seed, ld);
    r.F = F;
    r.s = s;
    std::vector<float> wf(r.host.w.begin(), r.host.w.end());
    r.b.ensure(sizeof(double) * F);
    r.w.ensure(sizeof(float) * F * s);
    r.eps.ensure(sizeof(float) * ld * s);
    r.om.ensure(sizeof(double) * F * d);
    WGP_CUDA(cudaMemcpyAsync(r.b.p, r.host.b.data(), sizeof(double) * F, cudaMemcpyHostToDevice, st));
    WGP_CUDA(cudaMemcpyAsync(r.w.p, wf.data(), sizeof(float) * F * s, cudaMemcpyHostToDevice, st));
    WGP_CUDA(cudaMemcpyAsync(r.eps.p, r.host.eps.data(), sizeof(float) * ld * s, cudaMemcpyHostToDevice, st));
    WGP_CUDA(cudaStreamSynchronize(st));
  }
  void rff_eval(DevRff& r, float* out) {
    std::vector<double> om(static_cast<size_t>(r.F) * d);
    for (int f = 0; f < r.F; ++f) {
      const double scale = 1.0 / std::sqrt(r.host.chi2[f] / 3.0);
      for (int k = 0; k < d; ++k)
        om[static_cast<size_t>(f) * d + k] = r.host.omega_z[static_cast<size_t>(f) * d + k] * scale / ls[k];
    }
    WGP_CUDA(cudaMemcpyAsync(r.om.p, om.data(), sizeof(double) * om.size(), cudaMemcpyHostToDevice, st));
    for (int c0 = 0; c0 < r.s; c0 += 128) {
      RffParams p{};
      p.x = X.as<float>();
      p.n = n;
      p.d = d;
      p.om = r.om.as<double>();
      p.b = r.b.as<double>();
      p.w = r.w.as<float>() + static_cast<size_t>(c0) * r.F;
      p.eps = r.eps.as<float>() + static_cast<size_t>(c0) * ld;
      p.F = r.F;
      p.s = std::min(128, r.s - c0);
      p.ld = ld;
      p.amp = static_cast<float>(sf * std::sqrt(2.0 / r.F));
      p.sigma = static_cast<float>(sigma);
      p.out = out + static_cast<size_t>(c0) * ld;
      rff_probes(p, st);
    }
    WGP_CUDA(cudaStreamSynchronize(st));  // om host buffer lifetime
  }

  // ---------------------------------------------------------------- training
  double to_c(int tr, double raw) const { return tr == 1 ? std::exp(raw) : softplus(raw); }
  double to_r(int tr, double v) const {
    if (tr == 1) {
      if (!(v > 0.0)) throw std::invalid_argument("log transform: argument must be positive");
      return std::log(v);
    }
    return softplus_inverse(v);
  }

  // ---------------------------------------------------------------- prediction
  // predict / test metrics (proj/src/exact.cpp:52-92) through iterative solves
  // (SURVEY §8f rank 2): alpha = H^-1 y and W = H^-1 K* with the configured
  // solver, K* (train x test) built per chunk of test points;
  // means = K*^T alpha, latent variances = sf^2 - colsum(K* o W).  The
  // reference's -1e-10 negativity guard is for fp64 dense solves; here a
  // variance below -1e-3 sf^2 is a NumericalError and smaller negatives clamp
  // to 0 like the reference.
  Buf xt, kstar, pw, pr, pal, pdots;
  void predict(const float* Xt_h, int64_t m, const float* yh, const wgp_solver_cfg& cfg, double* means,
               double* vars) {
    require_data();
    if (m < 0) throw std::invalid_argument("predict: negative test count");
    if (m == 0) return;
    for (int64_t e = 0; e < m * d; ++e)
      if (!std::isfinite(Xt_h[e])) throw std::invalid_argument("predict: non-finite test input");
    // prepared test points (training centres and scales, hyper_tmp = [mu | scale])
    const int64_t m_pad = round_up(m, 128);
    Buf xraw;
    xraw.ensure(sizeof(float) * m * d);
    WGP_CUDA(cudaMemcpyAsync(xraw.p, Xt_h, sizeof(float) * m * d, cudaMemcpyHostToDevice, st));
    xt.ensure(sizeof(float) * m_pad * dp);
    prepare_points(xraw.as<float>(), m, d, hyper_tmp.as<double>(), hyper_tmp.as<double>() + d, xt.as<float>(), m_pad,
                   dp, st);
    // alpha = H^-1 y
    pal.ensure(sizeof(float) * ld * 2);
    float* yd = pal.as<float>();
    float* alpha = yd + ld;
    WGP_CUDA(cudaMemsetAsync(yd, 0, sizeof(float) * ld, st));
    WGP_CUDA(cudaMemcpyAsync(yd, yh, sizeof(float) * n, cudaMemcpyHostToDevice, st));
    pw.ensure(sizeof(float) * ld * 64);
    pr.ensure(sizeof(float) * ld * 64);
    solve(cfg, yd, nullptr, alpha, pr.as<float>(), 1);
    // test points in chunks of 64 columns (the solver's right-hand sides)
    constexpr int64_t kMc = 64;
    kstar.ensure(sizeof(float) * ld * kMc);
    pdots.ensure(sizeof(double) * kMc);
    const double sfv = sf * sf;
    for (int64_t i0 = 0; i0 < m; i0 += kMc) {
      const int mc = static_cast<int>(std::min(kMc, m - i0));
      float* K = kstar.as<float>();
      cross_matrix(xs.as<float>(), n, xt.as<float>() + i0 * dp, mc, dp, sf2(), a_coef(), K, ld, st);
      colvec_dots(K, ld, n, mc, alpha, pdots.as<double>(), st);
      WGP_CUDA(cudaMemcpyAsync(means + i0, pdots.p, sizeof(double) * mc, cudaMemcpyDeviceToHost, st));
      solve(cfg, K, nullptr, pw.as<float>(), pr.as<float>(), mc);
      const std::vector<double> q = dots(K, pw.as<float>(), mc);
      for (int c = 0; c < mc; ++c) {
        double v = sfv - q[c];
        if (v < -1e-3 * sfv) throw NumericalError("predict: negative predictive variance beyond tolerance");
        vars[i0 + c] = v < 0.0 ? 0.0 : v;
      }
    }
    WGP_CUDA(cudaStreamSynchronize(st));
  }

  // ---------------------------------------------------------------- exact path
  // exact_mll / exact_gradient (proj/src/exact.cpp:25-50) in fp64 on the device:
  // dense H (lower triangle), cuSOLVER potrf / potrs / potri, fused derivative
  // contractions.  grad (raw space, d + 2) may be null (mll only).
  void exact(int transform, const double* raw, const float* yh, double* mll, double* grad_out) {
    if (n < 1) throw std::invalid_argument("no training inputs: call wgp_set_data first");
    const char* who = grad_out ? "exact_gradient" : "exact_mll";
    if (n > kDenseGuard) throw std::invalid_argument(std::string(who) + ": n exceeds the dense guard");
    const int p = d + 2;
    std::vector<double> cons(p);
    for (int k = 0; k < p; ++k) cons[k] = to_c(transform, raw[k]);
    const double sfe = cons[d], sge = cons[d + 1];
    lazy_handles();
    const int parts = exact_grad_parts();
    // device vectors: inv_ls [d] | y -> alpha [n] | logdiag [1] | sums [p] | parts [parts x p]
    const size_t nv = static_cast<size_t>(d) + n + 1 + p + static_cast<size_t>(parts) * p;
    exv.ensure(sizeof(double) * nv);
    double* inv_ls = exv.as<double>();
    double* alpha = inv_ls + d;
    double* logd = alpha + n;
    double* sums = logd + 1;
    double* part = sums + p;
    std::vector<double> hv(d + n);
    for (int k = 0; k < d; ++k) hv[k] = 1.0 / cons[k];
    for (int64_t i = 0; i < n; ++i) hv[d + i] = static_cast<double>(yh[i]);
    WGP_CUDA(cudaMemcpyAsync(inv_ls, hv.data(), sizeof(double) * (d + n), cudaMemcpyHostToDevice, st));
    hx.ensure(sizeof(double) * static_cast<size_t>(n) * n);
    double* H = hx.as<double>();
    exact_build(X.as<float>(), n, d, inv_ls, sfe * sfe, sge * sge, H, st);
    const int ni = static_cast<int>(n);
    int lw1 = 0, lw2 = 0;
    cusolverDnDpotrf_bufferSize(cusolver, CUBLAS_FILL_MODE_LOWER, ni, H, ni, &lw1);
    if (grad_out) cusolverDnDpotri_bufferSize(cusolver, CUBLAS_FILL_MODE_LOWER, ni, H, ni, &lw2);
    hx_ws.ensure(sizeof(double) * std::max(std::max(lw1, lw2), 1) + sizeof(int));
    int* dinfo = reinterpret_cast<int*>(hx_ws.as<double>() + std::max(std::max(lw1, lw2), 1));
    cusolverDnDpotrf(cusolver, CUBLAS_FILL_MODE_LOWER, ni, H, ni, hx_ws.as<double>(), std::max(lw1, 1), dinfo);
    int hinfo = 0;
    WGP_CUDA(cudaMemcpyAsync(&hinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    if (hinfo != 0) throw NumericalError(std::string(who) + ": system matrix is not positive definite");
    cusolverDnDpotrs(cusolver, CUBLAS_FILL_MODE_LOWER, ni, 1, H, ni, alpha, ni, dinfo);
    exact_logdiag(H, n, logd, st);
    std::vector<double> ha(n + 1);
    WGP_CUDA(cudaMemcpyAsync(ha.data(), alpha, sizeof(double) * (n + 1), cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    if (mll) {
      double ya = 0.0;
      for (int64_t i = 0; i < n; ++i) ya += hv[d + i] * ha[i];
      *mll = -0.5 * ya - ha[n] - 0.5 * static_cast<double>(n) * 1.8378770664093453;
    }
    if (!grad_out) return;
    cusolverDnDpotri(cusolver, CUBLAS_FILL_MODE_LOWER, ni, H, ni, hx_ws.as<double>(), std::max(lw2, 1), dinfo);
    WGP_CUDA(cudaMemcpyAsync(&hinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost, st));
    exact_grad_sums(X.as<float>(), n, d, inv_ls, sfe * sfe, alpha, H, part, parts, sums, st);
    std::vector<double> acc(p);
    WGP_CUDA(cudaMemcpyAsync(acc.data(), sums, sizeof(double) * p, cudaMemcpyDeviceToHost, st));
    WGP_CUDA(cudaStreamSynchronize(st));
    if (hinfo != 0) throw NumericalError(std::string(who) + ": system matrix is not positive definite");
    auto chain = [&](double r) { return transform == 1 ? std::exp(r) : softplus_derivative(r); };
    // dk/dl_k = 3 sf^2 e^{-sqrt3 r} dx_k^2 / l_k^3; dH/dsf = 2 k / sf; dH/dsigma = 2 sigma I
    for (int k = 0; k < d; ++k) grad_out[k] = 3.0 * sfe * sfe / cons[k] * acc[k] * chain(raw[k]);
    grad_out[d] = 2.0 / sfe * acc[d] * chain(raw[d]);
    grad_out[d + 1] = 2.0 * sge * acc[d + 1] * chain(raw[d + 1]);
  }

  void train(const float* yh, const wgp_train_cfg& cfg, wgp_trace* tr) {  // optimizer.cpp:81-171
    if (cfg.steps < 1) throw std::invalid_argument("TrainConfig: steps must be >= 1");
    if (cfg.num_probes < 1) throw std::invalid_argument("TrainConfig: num_probes must be >= 1");
    if (!(cfg.learning_rate > 0.0)) throw std::invalid_argument("TrainConfig: learning rate must be positive");
    if (!(cfg.init_constrained > 0.0))
      throw std::invalid_argument("TrainConfig: initial constrained value must be positive");
    validate(cfg.solver);
    if (n < 1) throw std::invalid_argument("train: dataset is empty");
    const int p = d + 2, s = cfg.num_probes, sp = s + 1;
    const int T = cfg.transform;
    std::vector<double> raw(p), m(p, 0.0), v(p, 0.0);
    for (int k = 0; k < d; ++k) raw[k] = to_r(T, cfg.init_constrained);
    raw[d] = to_r(T, cfg.init_signal > 0.0 ? cfg.init_signal : cfg.init_constrained);
    raw[d + 1] = to_r(T, cfg.init_noise > 0.0 ? cfg.init_noise : cfg.init_constrained);
    const bool fixed = cfg.mode != 1, warm = cfg.mode == 0, pathwise = cfg.estimator == 1;
    static const bool no_wsd_res = getenv("WGP_WSD_PRODUCT") != nullptr;  // 1: the explicit H (x0 - x*) product
    const int F = cfg.rff_features > 0 ? cfg.rff_features : 1000;

    // persistent across calls (Ctx members): fresh allocations would bump the
    // allocation generation and force every cached CG / AP graph to re-capture
    Buf& rhs = tr_rhs;
    Buf& sol0 = tr_sol0;
    Buf& sol1 = tr_sol1;
    Buf& Rres = tr_res;
    rhs.ensure(sizeof(float) * ld * sp);
    sol0.ensure(sizeof(float) * ld * sp);
    sol1.ensure(sizeof(float) * ld * sp);
    Rres.ensure(sizeof(float) * ld * sp);
    WGP_CUDA(cudaMemsetAsync(rhs.p, 0, sizeof(float) * ld * sp, st));
    WGP_CUDA(cudaMemcpyAsync(rhs.p, yh, sizeof(float) * n, cudaMemcpyHostToDevice, st));
    float* Z = rhs.as<float>() + ld;
    std::vector<float> hz;
    DevRff rff;
    uint64_t probe_seed = 0;
    auto draw = [&](uint64_t seed) {
      probe_seed = seed;
      if (pathwise) {
        rff_upload(rff, F, s, seed);
      } else {
        hz.assign(static_cast<size_t>(ld) * s, 0.f);
        sample_probes_host(n, s, cfg.probe_distribution, seed, hz.data(), ld);
        WGP_CUDA(cudaMemcpyAsync(Z, hz.data(), sizeof(float) * ld * s, cudaMemcpyHostToDevice, st));
        WGP_CUDA(cudaStreamSynchronize(st));
      }
    };
    if (fixed && !cfg.exact_gradients) draw(derive_seed(cfg.seed, 1));  // optimizer.cpp:99
    float* cur = sol0.as<float>();
    float* prev = sol1.as<float>();
    // fp64 CG keeps the warm-start solutions in fp64 as well (the reference's
    // prev_solutions are MatrixXd, optimizer.cpp:133-135,158)
    const bool keep64 = cfg.solver.kind == WGP_SOLVER_CG && cg_precision == WGP_CG_F64;
    Buf& s64a = tr_sol64a;
    Buf& s64b = tr_sol64b;
    double* cur64 = nullptr;
    double* prev64 = nullptr;
    if (keep64) {
      s64a.ensure(sizeof(double) * ld * sp);
      s64b.ensure(sizeof(double) * ld * sp);
      cur64 = s64a.as<double>();
      prev64 = s64b.as<double>();
    }
    bool have_prev = false;
    cudaEvent_t e0, e1, e1w, e2;
    WGP_CUDA(cudaEventCreate(&e0));
    WGP_CUDA(cudaEventCreate(&e1));
    WGP_CUDA(cudaEventCreate(&e1w));
    WGP_CUDA(cudaEventCreate(&e2));
    try {
      for (int t = 1; t <= cfg.steps; ++t) {
        try {
          std::vector<double> cons(p);
          for (int k = 0; k < p; ++k) cons[k] = to_c(T, raw[k]);
          WGP_CUDA(cudaEventRecord(e0, st));
          if (cfg.exact_gradients) {  // train_exact: the exact Cholesky gradient (optimizer.cpp:117-118)
            std::vector<double> g(p);
            exact(T, raw.data(), yh, nullptr, g.data());
            WGP_CUDA(cudaEventRecord(e1, st));
            adam(raw.data(), g.data(), m.data(), v.data(), p, t, cfg.learning_rate, cfg.adam_beta1,
                 cfg.adam_beta2, cfg.adam_eps);
            WGP_CUDA(cudaEventRecord(e2, st));
            WGP_CUDA(cudaEventSynchronize(e2));
            if (tr) {
              const size_t off = static_cast<size_t>(t - 1) * p;
              if (tr->raw_params) std::memcpy(tr->raw_params + off, raw.data(), sizeof(double) * p);
              if (tr->constrained_params)
                for (int k = 0; k < p; ++k) tr->constrained_params[off + k] = to_c(T, raw[k]);
              if (tr->gradient) std::memcpy(tr->gradient + off, g.data(), sizeof(double) * p);
              if (tr->solver_iterations) tr->solver_iterations[t - 1] = 0;
              if (tr->per_column_relative_residual)
                std::fill(tr->per_column_relative_residual + static_cast<size_t>(t - 1) * sp,
                          tr->per_column_relative_residual + static_cast<size_t>(t) * sp, 0.0);
              if (tr->warm_start_distance) tr->warm_start_distance[t - 1] = 0.0;
              if (tr->probe_seed) tr->probe_seed[t - 1] = 0;
              float ms_a = 0.f, ms_b = 0.f;
              WGP_CUDA(cudaEventElapsedTime(&ms_a, e0, e1));
              WGP_CUDA(cudaEventElapsedTime(&ms_b, e0, e2));
              if (tr->solver_ms) tr->solver_ms[t - 1] = ms_a;
              if (tr->step_ms) tr->step_ms[t - 1] = ms_b;
              if (tr->warm_distance_ms) tr->warm_distance_ms[t - 1] = 0.0;
            }
            continue;
          }
          set_hyper(cons.data());
          if (!fixed) draw(derive_seed(cfg.seed, static_cast<uint64_t>(t)));
          if (pathwise) rff_eval(rff, Z);
          wgp_solver_cfg sc = cfg.solver;
          sc.seed = derive_seed(derive_seed(cfg.seed, kSolverStream), static_cast<uint64_t>(t));
          const bool have_warm = warm && have_prev;
          keep_residuals = have_warm && cfg.warm_start_distance && !no_wsd_res;
          wsd_res = WsdRes{};
          SolveOut so = solve(sc, rhs.as<float>(), have_warm ? prev : nullptr, cur, Rres.as<float>(), sp,
                              have_warm ? prev64 : nullptr, cur64);
          WGP_CUDA(cudaEventRecord(e1, st));
          double wsd = 0.0;
          if (have_warm && cfg.warm_start_distance) {
            if (keep64)
              wsd = warm_distance_res_ok(64) ? warm_distance_res(prev64, cur64, sp) : warm_distance64(prev64, cur64, sp);
            else
              wsd = warm_distance_res_ok(32) ? warm_distance_res(prev, cur, sp) : warm_distance(prev, cur, sp);
          }
          WGP_CUDA(cudaEventRecord(e1w, st));
          if (tr && cfg.record_solver_state) {  // optimizer.cpp:148-151 (fp32 copies)
            const size_t off = static_cast<size_t>(t - 1) * n * sp;
            if (tr->solver_init) {
              if (have_warm)
                WGP_CUDA(cudaMemcpy2DAsync(tr->solver_init + off, sizeof(float) * n, prev, sizeof(float) * ld,
                                           sizeof(float) * n, sp, cudaMemcpyDeviceToHost, st));
              else
                std::fill(tr->solver_init + off, tr->solver_init + off + static_cast<size_t>(n) * sp, 0.f);
            }
            if (tr->solver_solutions)
              WGP_CUDA(cudaMemcpy2DAsync(tr->solver_solutions + off, sizeof(float) * n, cur, sizeof(float) * ld,
                                         sizeof(float) * n, sp, cudaMemcpyDeviceToHost, st));
          }
          std::vector<double> qa(p), qb(p), g(p);
          grad(T, raw.data(), cur, cur + ld, pathwise ? cur + ld : Z, s, 0.5 / s, qa.data(), qb.data(), own0,
               own_m(), true);
          for (int k = 0; k < p; ++k) g[k] = qa[k] - qb[k];
          adam(raw.data(), g.data(), m.data(), v.data(), p, t, cfg.learning_rate, cfg.adam_beta1,
               cfg.adam_beta2, cfg.adam_eps);
          WGP_CUDA(cudaEventRecord(e2, st));
          WGP_CUDA(cudaEventSynchronize(e2));
          if (tr) {
            const size_t off = static_cast<size_t>(t - 1) * p;
            if (tr->raw_params) std::memcpy(tr->raw_params + off, raw.data(), sizeof(double) * p);
            if (tr->constrained_params)
              for (int k = 0; k < p; ++k) tr->constrained_params[off + k] = to_c(T, raw[k]);
            if (tr->gradient) std::memcpy(tr->gradient + off, g.data(), sizeof(double) * p);
            if (tr->solver_iterations) tr->solver_iterations[t - 1] = so.iterations;
            if (tr->per_column_relative_residual)
              std::memcpy(tr->per_column_relative_residual + static_cast<size_t>(t - 1) * sp, so.rel.data(),
                          sizeof(double) * sp);
            if (tr->warm_start_distance) tr->warm_start_distance[t - 1] = wsd;
            if (tr->probe_seed) tr->probe_seed[t - 1] = probe_seed;
            float ms_solve = 0.f, ms_step = 0.f;
            WGP_CUDA(cudaEventElapsedTime(&ms_solve, e0, e1));
            WGP_CUDA(cudaEventElapsedTime(&ms_step, e0, e2));
            if (tr->solver_ms) tr->solver_ms[t - 1] = ms_solve;
            if (tr->step_ms) tr->step_ms[t - 1] = ms_step;
            if (tr->warm_distance_ms) {
              float ms_w = 0.f;
              WGP_CUDA(cudaEventElapsedTime(&ms_w, e1, e1w));
              tr->warm_distance_ms[t - 1] = ms_w;
            }
          }
          std::swap(cur, prev);
          std::swap(cur64, prev64);
          have_prev = true;
        } catch (const NumericalError& e) {
          throw NumericalError("step " + std::to_string(t) + ": " + e.what());
        }
      }
      if (tr && tr->final_solutions) {
        // prev holds the last step's solutions after the swap
        WGP_CUDA(cudaMemcpy2DAsync(tr->final_solutions, sizeof(float) * n, prev, sizeof(float) * ld,
                                   sizeof(float) * n, sp, cudaMemcpyDeviceToHost, st));
        WGP_CUDA(cudaStreamSynchronize(st));
      }
    } catch (...) {
      for (cudaEvent_t e : {e0, e1, e1w, e2}) cudaEventDestroy(e);
      throw;
    }
    for (cudaEvent_t e : {e0, e1, e1w, e2}) cudaEventDestroy(e);
  }

  static void adam(double* raw, const double* g, double* m, double* v, int p, int t, double lr,
                   double b1, double b2, double eps) {  // optimizer.cpp:48-65
    if (t < 1) throw std::invalid_argument("adam_step: t must be >= 1");
    for (int k = 0; k < p; ++k)
      if (!std::isfinite(g[k])) throw NumericalError("adam_step: non-finite gradient at step " + std::to_string(t));
    const double c1 = 1.0 - std::pow(b1, t), c2 = 1.0 - std::pow(b2, t);
    for (int k = 0; k < p; ++k) {
      m[k] = b1 * m[k] + (1.0 - b1) * g[k];
      v[k] = b2 * v[k] + (1.0 - b2) * (g[k] * g[k]);
      raw[k] += lr * (m[k] / c1) / (std::sqrt(v[k] / c2) + eps);
    }
  }
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return WGP_OK;
  } catch (const NumericalError& e) {
    g_last_error = e.what();
    return WGP_NUMERICAL;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return WGP_INVALID;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return WGP_DEVICE;
  }
}

std::atomic<uint64_t>& launch_counter() {
  static std::atomic<uint64_t> c{0};
  return c;
}
std::atomic<uint64_t>& alloc_generation() {
  static std::atomic<uint64_t> c{0};
  return c;
}

}  // namespace wgp

struct wgp_ctx {
  wgp::Ctx c;
};
struct wgp_local_group {
  std::shared_ptr<wgp::LocalGroup> g;
};

using wgp::guarded;

namespace {
// wgp_solve / wgp_solve_f64: host rhs / init (fp32 or fp64) -> device, solve,
// solutions / residuals back in the caller's precision.  With fp64 CG an fp64
// init and the fp64 solutions pass through unrounded.
template <class H, class S>
int solve_host(wgp_ctx* ctx, const wgp_solver_cfg* cfg, const H* rhs, const H* init, int s, S* state) {
  constexpr bool f64 = std::is_same<H, double>::value;
  return guarded([&] {
    wgp::Ctx& c = ctx->c;
    WGP_CUDA(cudaSetDevice(c.device));
    c.require_data();
    if (!cfg) throw std::invalid_argument("solve: null config");
    if (s < 1) throw std::invalid_argument("solve: rhs needs at least one column");
    if (!rhs) throw std::invalid_argument("solve: rhs row count mismatch");
    for (int64_t e = 0; e < c.n * s; ++e)
      if (!std::isfinite(rhs[e]) || (init && !std::isfinite(init[e])))
        throw std::invalid_argument("solve: non-finite right-hand side or init");
    const size_t bytes = sizeof(float) * c.ld * s;
    c.api_B.ensure(bytes);
    c.api_Xs.ensure(bytes);
    c.api_Rs.ensure(bytes);
    float* B = c.api_B.as<float>();
    float* Xs = c.api_Xs.as<float>();
    float* Rs = c.api_Rs.as<float>();
    float* X0 = nullptr;
    double* X0_64 = nullptr;
    double* Xo64 = nullptr;
    // host fp64 -> device fp64 staging, rounded to fp32 where the solver state is fp32
    auto upload = [&](const H* src, float* dst32, double** dst64) {
      WGP_CUDA(cudaMemsetAsync(dst32, 0, bytes, c.st));
      if constexpr (f64) {
        c.io_in.ensure(sizeof(double) * c.ld * s);
        double* tmp = c.io_in.as<double>();
        WGP_CUDA(cudaMemcpy2DAsync(tmp, sizeof(double) * c.ld, src, sizeof(double) * c.n, sizeof(double) * c.n, s,
                                   cudaMemcpyHostToDevice, c.st));
        wgp::narrow(tmp, c.ld, dst32, c.ld, c.n, s, c.st);
        if (dst64) *dst64 = tmp;
      } else {
        WGP_CUDA(cudaMemcpy2DAsync(dst32, sizeof(float) * c.ld, src, sizeof(float) * c.n, sizeof(float) * c.n, s,
                                   cudaMemcpyHostToDevice, c.st));
      }
    };
    upload(rhs, B, nullptr);
    if constexpr (f64) {  // keep the fp64 rhs (io_in is reused for init below)
      c.api_B64.ensure(sizeof(double) * c.ld * s);
      WGP_CUDA(cudaMemcpyAsync(c.api_B64.p, c.io_in.p, sizeof(double) * c.ld * s, cudaMemcpyDeviceToDevice, c.st));
    }
    if (init) {
      c.api_X0.ensure(bytes);
      X0 = c.api_X0.as<float>();
      upload(init, X0, &X0_64);
    }
    const bool keep64 = f64 && cfg->kind == WGP_SOLVER_CG && c.cg_precision == WGP_CG_F64;
    if (keep64) {
      c.io_out.ensure(sizeof(double) * c.ld * s);
      Xo64 = c.io_out.as<double>();
    }
    const wgp::Ctx::SolveOut so =
        c.solve(*cfg, B, X0, Xs, Rs, s, keep64 ? X0_64 : nullptr, Xo64, keep64 ? c.api_B64.as<double>() : nullptr);
    if (state) {
      if constexpr (f64) {
        // solutions in fp64 (fp64 CG: unrounded), residuals widened from fp32
        c.io_in.ensure(sizeof(double) * c.ld * s);
        double* w = c.io_in.as<double>();
        if (state->solutions) {
          const double* src = Xo64;
          if (!src) {
            wgp::widen(Xs, c.ld, w, c.ld, c.n, s, c.st);
            src = w;
          }
          WGP_CUDA(cudaMemcpy2DAsync(state->solutions, sizeof(double) * c.n, src, sizeof(double) * c.ld,
                                     sizeof(double) * c.n, s, cudaMemcpyDeviceToHost, c.st));
          WGP_CUDA(cudaStreamSynchronize(c.st));
        }
        if (state->residuals) {
          wgp::widen(Rs, c.ld, w, c.ld, c.n, s, c.st);
          WGP_CUDA(cudaMemcpy2DAsync(state->residuals, sizeof(double) * c.n, w, sizeof(double) * c.ld,
                                     sizeof(double) * c.n, s, cudaMemcpyDeviceToHost, c.st));
        }
      } else {
        if (state->solutions)
          WGP_CUDA(cudaMemcpy2DAsync(state->solutions, sizeof(float) * c.n, Xs, sizeof(float) * c.ld,
                                     sizeof(float) * c.n, s, cudaMemcpyDeviceToHost, c.st));
        if (state->residuals)
          WGP_CUDA(cudaMemcpy2DAsync(state->residuals, sizeof(float) * c.n, Rs, sizeof(float) * c.ld,
                                     sizeof(float) * c.n, s, cudaMemcpyDeviceToHost, c.st));
      }
      WGP_CUDA(cudaStreamSynchronize(c.st));
      if (state->per_column_relative_residual)
        std::copy(so.rel.begin(), so.rel.end(), state->per_column_relative_residual);
      if (state->converged) std::copy(so.conv.begin(), so.conv.end(), state->converged);
      state->iterations_used = so.iterations;
    }
  });
}
}  // namespace

extern "C" {

const char* wgp_last_error(void) { return wgp::g_last_error.c_str(); }

const char* wgp_version(void) {
  return "warmgp_b200 0.2 (sm_100a; tcgen05 H.V: 3xTF32 Gram + 3xTF32 or fp16x3 K.V, fp64 chunk sums; fp64 DMMA CG operator; SIMT fp32/fp64 kernel)";
}

uint64_t wgp_launch_count(void) { return wgp::launch_counter().load(); }

int wgp_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int wgp_create(int device, wgp_ctx** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("wgp_create: null output pointer");
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
      cudaGetLastError();
      throw wgp::DeviceError("no CUDA device available (warmgp_b200 has no CPU fallback)");
    }
    if (device < 0 || device >= count) throw std::invalid_argument("wgp_create: device out of range");
    WGP_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    WGP_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      throw wgp::DeviceError("warmgp_b200 is built for sm_100a (B200); found sm_" +
                             std::to_string(prop.major) + std::to_string(prop.minor));
    auto* ctx = new wgp_ctx();
    ctx->c.device = device;
    if (cudaStreamCreateWithFlags(&ctx->c.st, cudaStreamNonBlocking) != cudaSuccess) {
      delete ctx;
      throw wgp::DeviceError("cudaStreamCreate failed");
    }
    *out = ctx;
  });
}

int wgp_destroy(wgp_ctx* ctx) {
  return guarded([&] {
    if (ctx) {
      cudaSetDevice(ctx->c.device);
      delete ctx;
    }
  });
}

int wgp_set_hv_impl(wgp_ctx* ctx, int impl) {
  return guarded([&] {
    if (impl != WGP_HV_TC && impl != WGP_HV_SIMT && impl != WGP_HV_TC_F16)
      throw std::invalid_argument("unknown H.V implementation");
    ctx->c.hv_impl = impl;
  });
}

int wgp_set_cg_precision(wgp_ctx* ctx, int precision) {
  return guarded([&] {
    if (precision != WGP_CG_F64 && precision != WGP_CG_F32) throw std::invalid_argument("unknown CG precision");
    ctx->c.cg_precision = precision;
  });
}

int wgp_profile(wgp_ctx* ctx, int enable) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    ctx->c.tc.profiling = enable != 0;
  });
}

int wgp_profile_read(wgp_ctx* ctx, double* kernel_ms, int* launches) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    const double ms = ctx->c.tc.profile_ms(launches);
    if (kernel_ms) *kernel_ms = ms;
  });
}

void* wgp_stream(wgp_ctx* ctx) { return ctx ? static_cast<void*>(ctx->c.st) : nullptr; }

int wgp_set_data(wgp_ctx* ctx, const float* X, int64_t n, int d) {
  return guarded([&] {
    WGP_CUDA(cudaSetDevice(ctx->c.device));
    ctx->c.set_data(X, n, d);
  });
}

int wgp_set_hyper(wgp_ctx* ctx, const double* c) {
  return guarded([&] {
    WGP_CUDA(cudaSetDevice(ctx->c.device));
    ctx->c.set_hyper(c);
  });
}

int wgp_nccl_unique_id(unsigned char* id) {
  return guarded([&] {
    if (!id) throw std::invalid_argument("wgp_nccl_unique_id: null id");
    const wgp::NcclApi& a = wgp::NcclApi::get();
    ncclUniqueId u;
    a.check(a.get_unique_id(&u), "ncclGetUniqueId");
    std::memcpy(id, u.internal, sizeof(u.internal));
  });
}

int wgp_set_comm(wgp_ctx* ctx, int rank, int nranks, const unsigned char* id) {
  return guarded([&] {
    wgp::Ctx& c = ctx->c;
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("wgp_set_comm: bad rank / nranks");
    if (!id) throw std::invalid_argument("wgp_set_comm: null id");
    WGP_CUDA(cudaSetDevice(c.device));
    ncclUniqueId u;
    std::memcpy(u.internal, id, sizeof(u.internal));
    c.drop_cg_graphs();  // captured launches bake in the layout
    c.comm.reset();
    c.comm = std::make_unique<wgp::NcclComm>(rank, nranks, u);
    c.rank = rank;
    c.nranks = nranks;
    c.n = 0;  // the row layout depends on the rank count: wgp_set_data follows
    c.have_hyper = false;
  });
}

int wgp_local_group_create(int nranks, wgp_local_group** out) {
  return guarded([&] {
    if (nranks < 1 || !out) throw std::invalid_argument("wgp_local_group_create: bad arguments");
    *out = new wgp_local_group{std::make_shared<wgp::LocalGroup>(nranks)};
  });
}

int wgp_local_group_destroy(wgp_local_group* g) {
  delete g;
  return WGP_OK;
}

int wgp_set_comm_local(wgp_ctx* ctx, wgp_local_group* g, int rank) {
  return guarded([&] {
    wgp::Ctx& c = ctx->c;
    if (!g || rank < 0 || rank >= g->g->nranks) throw std::invalid_argument("wgp_set_comm_local: bad rank");
    WGP_CUDA(cudaSetDevice(c.device));
    c.drop_cg_graphs();
    c.comm.reset();
    c.comm = std::make_unique<wgp::LocalComm>(g->g, rank);
    c.rank = rank;
    c.nranks = g->g->nranks;
    c.n = 0;
    c.have_hyper = false;
  });
}

int wgp_shard_info(wgp_ctx* ctx, int* rank, int* nranks, int64_t* own0, int64_t* own1, int64_t* ld) {
  return guarded([&] {
    const wgp::Ctx& c = ctx->c;
    if (rank) *rank = c.rank;
    if (nranks) *nranks = c.nranks;
    if (own0) *own0 = c.own0;
    if (own1) *own1 = c.own1;
    if (ld) *ld = c.ld;
  });
}

int wgp_shard_rows(int64_t n, int rank, int nranks, int64_t* own0, int64_t* own1, int64_t* ld) {
  return guarded([&] {
    if (n < 1 || nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("wgp_shard_rows: bad arguments");
    const int64_t blk = wgp::ceil_div(wgp::ceil_div(n, 128), nranks) * 128;
    if (own0) *own0 = std::min<int64_t>(n, rank * blk);
    if (own1) *own1 = std::min<int64_t>(n, (rank + 1) * blk);
    if (ld) *ld = std::max<int64_t>(wgp::round_up(n, 128), blk * nranks);
  });
}

int wgp_set_rows(wgp_ctx* ctx, int64_t r0, int64_t r1) {
  return guarded([&] {
    if (r0 < 0 || r1 > ctx->c.n || r1 <= r0) throw std::invalid_argument("wgp_set_rows: bad row range");
    ctx->c.r0 = r0;
    ctx->c.r1 = r1;
  });
}

// wgp_hv's copy / compute pipeline on the tcgen05 engines: the product in
// row chunks, each chunk's result copy running under the next chunk's launch
// (the short last chunk's copy is the exposed one).  Each launch keys its J
// splits on its own rows, so the result equals the one-launch product to fp32
// rounding.  The cut comes from hv_tc's launch cost model (choose_splits) and
// a PCIe model (D2H 40 GB/s + 10 us): chunks sized to whole waves can even beat the
// one launch's wave tail (config 1: 0.30 vs 0.33 ms end to end, one launch
// 0.178 ms on the device).  Cutting the contracted points instead, so that a
// first J range's launch hides the rest of V's upload, was measured slower
// (0.315 ms at the best cut, 0.62 ms combined with the row chunks).
// WGP_HV_PIPE (read per call): "1" one launch, or comma-separated row fractions.
struct HvPlan {
  std::vector<int64_t> cuts{0};  // row offsets of the launches, then m
};

static HvPlan hv_plan(const wgp::Ctx& c, int64_t m, int s) {
  const char* env = getenv("WGP_HV_PIPE");  // read per call (A/B within one process)
  const std::string spec(env ? env : "");
  HvPlan pl;
  const bool tc = (c.hv_impl == WGP_HV_TC || c.hv_impl == WGP_HV_TC_F16) && wgp::hv_tc_supported(c.d, s);
  if (!tc || s > 96 || m < 8192 || spec == "1") {
    pl.cuts.push_back(m);
    return pl;
  }
  if (!spec.empty()) {  // row fractions
    std::vector<double> fr;
    size_t pos = 0;
    while (pos <= spec.size()) {
      const size_t q = spec.find(',', pos);
      const std::string t = spec.substr(pos, q == std::string::npos ? std::string::npos : q - pos);
      if (!t.empty()) fr.push_back(std::max(0.0, atof(t.c_str())));
      if (q == std::string::npos) break;
      pos = q + 1;
    }
    double tot = 0, acc = 0;
    for (double f : fr) tot += f;
    for (size_t k = 0; k + 1 < fr.size() && tot > 0; ++k) {
      acc += fr[k] / tot;
      const int64_t r = wgp::round_up(static_cast<int64_t>(acc * static_cast<double>(m)), 128);
      if (r > pl.cuts.back() && r < m) pl.cuts.push_back(r);
    }
    pl.cuts.push_back(m);
    return pl;
  }
  const bool f16 = c.hv_impl == WGP_HV_TC_F16;
  // seconds per cost unit (config-1 calibration: 0.166 ms / 213 units fp16,
  // 0.207 ms / 431 units tf32) plus launch overhead
  const double t_unit = f16 ? 0.78e-6 : 0.48e-6, t_launch = 4e-6;
  // D2H 40 GB/s + 10 us per copy: conservative, so the first chunk's copy
  // stays hidden under the second launch (measured: cuts where the model's
  // 50 GB/s said "just hidden" ran ~0.01 ms slower)
  auto d2h = [&](int64_t rows) { return static_cast<double>(rows) * 4.0 * s / 40e9 + 10e-6; };
  auto T = [&](int64_t rows) { return wgp::hv_tc_model_cost(rows, c.n, s, f16) * t_unit + t_launch; };
  double best = T(m) + d2h(m);
  int64_t cut = 0;
  const int64_t step = std::max<int64_t>(128, wgp::round_up(m / 64, 128));
  for (int64_t r = 1024; r <= m - 1024; r += step) {
    const double e1 = T(r);
    const double e = std::max(e1 + T(m - r), e1 + d2h(r)) + d2h(m - r);
    if (e < best - 1e-12) {
      best = e;
      cut = r;
    }
  }
  if (cut > 0) pl.cuts.push_back(cut);
  pl.cuts.push_back(m);
  if (getenv("WGP_HV_PLAN_DEBUG"))
    fprintf(stderr, "[wgp_hv plan] m=%lld n=%lld s=%d cut=%lld model %.1f us\n", (long long)m, (long long)c.n, s,
            (long long)cut, best * 1e6);
  return pl;
}

int wgp_hv(wgp_ctx* ctx, const float* V, int s, float* out) {
  return guarded([&] {
    wgp::Ctx& c = ctx->c;
    WGP_CUDA(cudaSetDevice(c.device));
    c.require_data();
    if (s < 1) throw std::invalid_argument("wgp_hv: s must be >= 1");
    wgp::Buf& dv = c.io_in;
    wgp::Buf& dout = c.io_out;
    // V uploaded as one contiguous copy (leading dimension n: the H.V kernels
    // take any ldv), faster than a pitched copy into the padded layout
    dv.ensure(sizeof(float) * c.ld * s);
    const int64_t ldv = c.n;
    if (c.sharded()) {  // the rank's rows, then the all-gather of the n x s result
      WGP_CUDA(cudaMemcpyAsync(dv.p, V, sizeof(float) * c.n * s, cudaMemcpyHostToDevice, c.st));
      dout.ensure(sizeof(float) * c.ld * s);
      float* o = dout.as<float>();
      c.hv(dv.as<float>(), ldv, s, o + c.own0, c.ld, wgp::kHvStore, nullptr, 0, 0, c.n, nullptr, c.own0,
           c.own_m());
      c.gather_rows(o, s);
      WGP_CUDA(cudaMemcpy2DAsync(out, sizeof(float) * c.n, o, sizeof(float) * c.ld, sizeof(float) * c.n, s,
                                 cudaMemcpyDeviceToHost, c.st));
    } else {
      const int64_t m = c.r1 - c.r0;
      dout.ensure(sizeof(float) * m * s);
      const HvPlan pl = hv_plan(c, m, s);
      if (!c.cst) {
        WGP_CUDA(cudaStreamCreateWithFlags(&c.cst, cudaStreamNonBlocking));
        WGP_CUDA(cudaEventCreateWithFlags(&c.ev_chunk, cudaEventDisableTiming));
        WGP_CUDA(cudaEventCreateWithFlags(&c.ev_copied, cudaEventDisableTiming));
      }
      if (!c.ev_up0) {
        WGP_CUDA(cudaEventCreate(&c.ev_up0));
        WGP_CUDA(cudaEventCreate(&c.ev_up1));
      }
      // Upload of V.  The copy engine reads page-locked memory at ~52 GB/s when the host
      // link is in its fast state, but only 11-21 GB/s in a slow state some hosts fall
      // into for 10-100 ms at a time (DESIGN 4.1); SM loads from the same buffer hold
      // ~42 GB/s in both.  So on the tcgen05 engines the V split can read the caller's
      // page-locked buffer itself (HvParams::v_host, keeping a device copy for the
      // diagonal term): config 1 end to end 0.317 ms in either state, against 0.312
      // (fast) to 0.53 ms (slow) with the copy engine -- the default for page-locked
      // V.  WGP_HV_UPLOAD (read per call): zc (default), ce (always the copy engine),
      // auto (time each copy-engine upload; below 35 GB/s switch to the zero-copy
      // split, re-probing the copy engine every 16th call).
      const float* v_alias = nullptr;
      {
        const char* e = getenv("WGP_HV_UPLOAD");
        const std::string mode(e ? e : "zc");
        const bool tc_eng = (c.hv_impl == WGP_HV_TC || c.hv_impl == WGP_HV_TC_F16) && wgp::hv_tc_supported(c.d, s) &&
                            s <= 96;
        const bool want = mode == "zc" || (mode == "auto" && c.ce_gbps >= 0 && c.ce_gbps < 35.0 && c.zc_streak < 15);
        if (tc_eng && want && sizeof(float) * c.n * s >= (1u << 20)) {
          cudaPointerAttributes at{};
          if (cudaPointerGetAttributes(&at, V) == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer)
            v_alias = static_cast<const float*>(at.devicePointer);
          else
            (void)cudaGetLastError();
        }
      }
      if (v_alias) {
        ++c.zc_streak;
        c.v_host_next = v_alias;
      } else {
        c.zc_streak = 0;
        WGP_CUDA(cudaEventRecord(c.ev_up0, c.st));
        WGP_CUDA(cudaMemcpyAsync(dv.p, V, sizeof(float) * c.n * s, cudaMemcpyHostToDevice, c.st));
        WGP_CUDA(cudaEventRecord(c.ev_up1, c.st));
      }
      const bool timed_upload = !v_alias;
      if (pl.cuts.size() <= 2) {
        c.hv(dv.as<float>(), ldv, s, dout.as<float>(), m, wgp::kHvStore, nullptr, 0, 0, c.n, nullptr, c.r0, m);
        WGP_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(float) * m * s, cudaMemcpyDeviceToHost, c.st));
      } else {
        float* o = dout.as<float>();
        // chunk 0 splits V, the others reuse its planes; chunk k's result copy
        // overlaps chunk k + 1's launch
        // The last chunk's copy is the exposed one: with a page-locked result buffer
        // its launch can store straight into the caller's memory instead (plain
        // coalesced stores in store mode, no read of the destination; same values).
        // Config 1: 0.316 vs 0.321 ms per call.  WGP_HV_DOWNLOAD=ce turns it off (read
        // per call).
        float* out_alias = nullptr;
        {
          const char* e = getenv("WGP_HV_DOWNLOAD");
          if (!e || std::string(e) != "ce") {
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, out) == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer)
              out_alias = static_cast<float*>(at.devicePointer);
            else
              (void)cudaGetLastError();
          }
        }
        for (size_t k = 0; k + 1 < pl.cuts.size(); ++k) {
          const int64_t a = pl.cuts[k], len = pl.cuts[k + 1] - pl.cuts[k];
          if (out_alias && k + 2 == pl.cuts.size()) {
            c.hv(dv.as<float>(), ldv, s, out_alias + a, m, wgp::kHvStore, nullptr, 0, 0, c.n, nullptr, c.r0 + a, len,
                 nullptr, false, nullptr, 0, k > 0);
            break;
          }
          c.hv(dv.as<float>(), ldv, s, o + a, m, wgp::kHvStore, nullptr, 0, 0, c.n, nullptr, c.r0 + a, len, nullptr,
               false, nullptr, 0, k > 0);
          WGP_CUDA(cudaEventRecord(c.ev_chunk, c.st));
          WGP_CUDA(cudaStreamWaitEvent(c.cst, c.ev_chunk, 0));
          WGP_CUDA(cudaMemcpy2DAsync(out + a, sizeof(float) * m, o + a, sizeof(float) * m, sizeof(float) * len, s,
                                     cudaMemcpyDeviceToHost, c.cst));
        }
        WGP_CUDA(cudaEventRecord(c.ev_copied, c.cst));
        WGP_CUDA(cudaStreamWaitEvent(c.st, c.ev_copied, 0));
      }
      WGP_CUDA(cudaStreamSynchronize(c.st));
      c.v_host_next = nullptr;
      if (timed_upload) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, c.ev_up0, c.ev_up1) == cudaSuccess && ms > 0.f)
          c.ce_gbps = static_cast<double>(sizeof(float) * c.n * s) / (ms * 1e-3) / 1e9;
        else
          (void)cudaGetLastError();
      }
      return;
    }
    WGP_CUDA(cudaStreamSynchronize(c.st));
  });
}

int wgp_hv_f64(wgp_ctx* ctx, const double* V, int s, double* out) {
  return guarded([&] {
    wgp::Ctx& c = ctx->c;
    WGP_CUDA(cudaSetDevice(c.device));
    c.require_data();
    if (s < 1) throw std::invalid_argument("wgp_hv: s must be >= 1");
    wgp::Buf& dv = c.io_in;
    wgp::Buf& dout = c.io_out;
    dv.ensure(sizeof(double) * c.ld * s);
    WGP_CUDA(cudaMemcpy2DAsync(dv.p, sizeof(double) * c.ld, V, sizeof(double) * c.n, sizeof(double) * c.n, s,
                               cudaMemcpyHostToDevice, c.st));
    if (c.sharded()) {
      dout.ensure(sizeof(double) * c.ld * s);
      double* o = dout.as<double>();
      c.hv64_rows(dv.as<double>(), c.ld, s, o + c.own0, c.ld, wgp::kHv64Store, nullptr, 0, c.own0, c.own_m(),
                  nullptr);
      c.gather_rows(o, s);
      WGP_CUDA(cudaMemcpy2DAsync(out, sizeof(double) * c.n, o, sizeof(double) * c.ld, sizeof(double) * c.n, s,
                                 cudaMemcpyDeviceToHost, c.st));
    } else {
      const int64_t m = c.r1 - c.r0;
      dout.ensure(sizeof(double) * m * s);
      c.hv64_rows(dv.as<double>(), c.ld, s, dout.as<double>(), m, wgp::kHv64Store, nullptr, 0, c.r0, m, nullptr);
      WGP_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(double) * m * s, cudaMemcpyDeviceToHost, c.st));
    }
    WGP_CUDA(cudaStreamSynchronize(c.st));
  });
}

int wgp_hv_device(wgp_ctx* ctx, const float* V, int64_t ldv, int s, float* out, int64_t ldo) {
  return guarded([&] {
    wgp::Ctx& c = ctx->c;
    c.require_data();
    if (s < 1) throw std::invalid_argument("wgp_hv: s must be >= 1");
    if (c.sharded()) {  // rows [own0, own1) into out, then the in-place all-gather: out holds all rows
      if (ldv < c.n || ldo != c.ld)
        throw std::invalid_argument("wgp_hv: a row-sharded context needs ldo == its leading dimension");
      c.hv(V, ldv, s, out + c.own0, ldo, wgp::kHvStore, nullptr, 0, 0, c.n, nullptr, c.own0, c.own_m());
      c.gather_rows(out, s);
      return;
    }
    if (ldv < c.n || ldo < c.r1 - c.r0) throw std::invalid_argument("wgp_hv: leading dimension too small");
    c.hv(V, ldv, s, out, ldo, wgp::kHvStore, nullptr, 0, 0, c.n, nullptr, c.r0, c.r1 - c.r0);
  });
}

int wgp_solve(wgp_ctx* ctx, const wgp_solver_cfg* cfg, const float* rhs, const float* init, int s,
              wgp_solve_state* state) {
  return solve_host(ctx, cfg, rhs, init, s, state);
}

int wgp_solve_f64(wgp_ctx* ctx, const wgp_solver_cfg* cfg, const double* rhs, const double* init, int s,
                  wgp_solve_state_f64* state) {
  return solve_host(ctx, cfg, rhs, init, s, state);
}

int wgp_grad(wgp_ctx* ctx, int transform, const double* raw, const float* vy, const float* L,
             const float* R, int s, double coef_b, double* out_a, double* out_b) {
  return guarded([&] {
    wgp::Ctx& c = ctx->c;
    WGP_CUDA(cudaSetDevice(c.device));
    if (c.n < 1) throw std::invalid_argument("no training inputs: call wgp_set_data first");
    if (s < 1) throw std::invalid_argument("wgp_grad: s must be >= 1");
    wgp::Buf dvy, dL, dR;
    const size_t bytes = sizeof(float) * c.ld * s;
    dvy.ensure(sizeof(float) * c.ld);
    dL.ensure(bytes);
    dR.ensure(bytes);
    WGP_CUDA(cudaMemsetAsync(dvy.p, 0, sizeof(float) * c.ld, c.st));
    WGP_CUDA(cudaMemsetAsync(dL.p, 0, bytes, c.st));
    WGP_CUDA(cudaMemsetAsync(dR.p, 0, bytes, c.st));
    WGP_CUDA(cudaMemcpyAsync(dvy.p, vy, sizeof(float) * c.n, cudaMemcpyHostToDevice, c.st));
    WGP_CUDA(cudaMemcpy2DAsync(dL.p, sizeof(float) * c.ld, L, sizeof(float) * c.n, sizeof(float) * c.n, s,
                               cudaMemcpyHostToDevice, c.st));
    WGP_CUDA(cudaMemcpy2DAsync(dR.p, sizeof(float) * c.ld, R, sizeof(float) * c.n, sizeof(float) * c.n, s,
                               cudaMemcpyHostToDevice, c.st));
    // rows of the context's row range (wgp_set_rows) against all points;
    // a row-sharded context contracts its rows and sums over the ranks
    if (c.sharded())
      c.grad(transform, raw, dvy.as<float>(), dL.as<float>(), dR.as<float>(), s, coef_b, out_a, out_b, c.own0,
             c.own_m(), true);
    else
      c.grad(transform, raw, dvy.as<float>(), dL.as<float>(), dR.as<float>(), s, coef_b, out_a, out_b, c.r0,
             c.r1 - c.r0);
  });
}

int wgp_sample_probes(int64_t n, int s, int dist, uint64_t seed, float* out) {
  return guarded([&] { wgp::sample_probes_host(n, s, dist, seed, out, n); });
}

int wgp_rff_probes(wgp_ctx* ctx, int F, int s, uint64_t seed, float* out) {
  return guarded([&] {
    wgp::Ctx& c = ctx->c;
    WGP_CUDA(cudaSetDevice(c.device));
    c.require_data();
    if (F < 1 || s < 1) throw std::invalid_argument("rff_probes: F and s must be >= 1");
    wgp::Ctx::DevRff r;
    c.rff_upload(r, F, s, seed);
    wgp::Buf dz;
    dz.ensure(sizeof(float) * c.ld * s);
    c.rff_eval(r, dz.as<float>());
    WGP_CUDA(cudaMemcpy2DAsync(out, sizeof(float) * c.n, dz.p, sizeof(float) * c.ld, sizeof(float) * c.n, s,
                               cudaMemcpyDeviceToHost, c.st));
    WGP_CUDA(cudaStreamSynchronize(c.st));
  });
}

int wgp_train(wgp_ctx* ctx, const float* y, const wgp_train_cfg* cfg, wgp_trace* trace) {
  return guarded([&] {
    WGP_CUDA(cudaSetDevice(ctx->c.device));
    if (ctx->c.n < 1) throw std::invalid_argument("train: dataset is empty");
    ctx->c.train(y, *cfg, trace);
  });
}

int wgp_predict(wgp_ctx* ctx, const float* X_test, int64_t m, const float* y, const wgp_solver_cfg* cfg,
                double* means, double* variances, double* noise_variance) {
  return guarded([&] {
    if (!ctx || !y || !cfg || (m > 0 && (!X_test || !means || !variances)))
      throw std::invalid_argument("wgp_predict: null argument");
    WGP_CUDA(cudaSetDevice(ctx->c.device));
    ctx->c.predict(X_test, m, y, *cfg, means, variances);
    if (noise_variance) *noise_variance = ctx->c.sigma * ctx->c.sigma;
  });
}

int wgp_exact(wgp_ctx* ctx, int transform, const double* raw, const float* y, double* mll, double* grad) {
  return guarded([&] {
    if (!ctx || !raw || !y) throw std::invalid_argument("wgp_exact: null argument");
    WGP_CUDA(cudaSetDevice(ctx->c.device));
    if (transform != WGP_TRANSFORM_SOFTPLUS && transform != WGP_TRANSFORM_LOG)
      throw std::invalid_argument("unknown hyperparameter transform");
    ctx->c.exact(transform, raw, y, mll, grad);
  });
}

int wgp_adam_step(double* raw, const double* grad, double* m, double* v, int p, int t, double lr,
                  double beta1, double beta2, double eps) {
  return guarded([&] { wgp::Ctx::adam(raw, grad, m, v, p, t, lr, beta1, beta2, eps); });
}

uint64_t wgp_derive_seed(uint64_t base, uint64_t stream) { return wgp::derive_seed(base, stream); }

int wgp_set_split_global(wgp_ctx* ctx, int global) {
  return guarded([&] { ctx->c.split_global = global != 0; });
}

int wgp_hv_cols(wgp_ctx* ctx, const float* V, int64_t ldv, int s, int64_t j0, int64_t j1, float* out, int64_t ldo,
                int mode, const float* B, int64_t ldb) {
  return guarded([&] {
    wgp::Ctx& c = ctx->c;
    c.require_data();
    if (s < 1) throw std::invalid_argument("wgp_hv_cols: s must be >= 1");
    if (j0 < 0 || j1 > c.n || j1 <= j0) throw std::invalid_argument("wgp_hv_cols: bad column range");
    if (mode < wgp::kHvStore || mode > wgp::kHvSubtract) throw std::invalid_argument("wgp_hv_cols: bad mode");
    if (mode == wgp::kHvResidual && !B) throw std::invalid_argument("wgp_hv_cols: residual mode needs B");
    if (ldv < j1 - j0 || ldo < c.r1 - c.r0 || (B && ldb < c.r1 - c.r0))
      throw std::invalid_argument("wgp_hv_cols: leading dimension too small");
    // the kernels index V by global point and B by global row
    c.hv(V - j0, ldv, s, out, ldo, mode, B ? B - c.r0 : nullptr, ldb, j0, j1, nullptr, c.r0, c.r1 - c.r0);
  });
}

int wgp_hv_block(wgp_ctx* ctx, int64_t i0, int64_t i1, int64_t j0, int64_t j1, const float* V, int64_t ldv, int s,
                 float* out, int64_t ldo) {
  return guarded([&] {
    wgp::Ctx& c = ctx->c;
    c.require_data();
    if (s < 1) throw std::invalid_argument("wgp_hv_block: s must be >= 1");
    if (i0 < 0 || i1 > c.n || i1 <= i0 || j0 < 0 || j1 > c.n || j1 <= j0)
      throw std::invalid_argument("wgp_hv_block: bad row or column range");
    if (ldv < j1 - j0 || ldo < i1 - i0) throw std::invalid_argument("wgp_hv_block: leading dimension too small");
    // the kernels index V by global point
    c.hv(V - j0, ldv, s, out, ldo, wgp::kHvStore, nullptr, 0, j0, j1, nullptr, i0, i1 - i0, nullptr, false);
  });
}

int wgp_ap_factor(wgp_ctx* ctx, int block_size, int64_t* nblocks) {
  return guarded([&] {
    wgp::Ctx& c = ctx->c;
    c.require_data();
    if (block_size < 1) throw std::invalid_argument("SolverConfig: block_size must be >= 1");
    const int64_t nb = c.ap_factor(std::min<int64_t>(block_size, c.n));
    if (nblocks) *nblocks = nb;
  });
}

int wgp_ap_block_solve(wgp_ctx* ctx, int64_t block, const double* Rb, int s, double* delta) {
  return guarded([&] {
    if (s < 1) throw std::invalid_argument("wgp_ap_block_solve: s must be >= 1");
    ctx->c.ap_block_solve(block, Rb, s, delta);
  });
}

// split_standardize's row permutation (dataset.cpp:118-124): Fisher-Yates
// from the back with mt19937_64(derive_seed(split_seed, 0x5b117)).
int wgp_split_order(int64_t n, uint64_t split_seed, int64_t* order) {
  return guarded([&] {
    if (n < 1 || !order) throw std::invalid_argument("split_order: n must be >= 1");
    for (int64_t i = 0; i < n; ++i) order[i] = i;
    std::mt19937_64 rng(wgp::derive_seed(split_seed, 0x5b117ULL));
    for (int64_t i = n - 1; i > 0; --i) {
      const int64_t j = static_cast<int64_t>(wgp::uniform_below(rng, static_cast<uint64_t>(i) + 1));
      std::swap(order[i], order[j]);
    }
  });
}

}  // extern "C"
