// C ABI (include/qp_b200.h): host orchestration of the single-factorization
// inexact IPM (arXiv 2104.12916) on one B200.  Every arithmetic step runs in
// the kernels of kernels.cu; this file does validation, symbolic planning
// (symbolic.cpp), device memory, and the IPM / PCG control flow.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <cstddef>
#include <functional>
#include <memory>
#include <string>
#include <vector>
#include <random>

#include "../../include/qp_b200.h"
#include "kernels.cuh"
#include "symbolic.h"

using namespace qpb;

namespace {

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// NCCL, loaded on first use (only sharded runs need it; single-GPU builds never touch it).
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  // halo mode of the sharded operator (optional symbols: present in every NCCL ≥ 2.7)
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
};
NcclApi& nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    api.err = std::string("cannot load libnccl.so.2: ") + dlerror();
    return api;
  }
  api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
  api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
  api.all_reduce = (decltype(api.all_reduce))dlsym(h, "ncclAllReduce");
  api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
  api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
  api.send = (decltype(api.send))dlsym(h, "ncclSend");
  api.recv = (decltype(api.recv))dlsym(h, "ncclRecv");
  api.group_start = (decltype(api.group_start))dlsym(h, "ncclGroupStart");
  api.group_end = (decltype(api.group_end))dlsym(h, "ncclGroupEnd");
  api.ok = api.get_unique_id && api.comm_init_rank && api.all_reduce && api.comm_destroy && api.error_string;
  if (!api.ok) api.err = "libnccl.so.2 lacks a required symbol";
  return api;
}

// Contiguous split of the m2 inequality rows over `world` ranks, balancing nnz + 1 per row.
void partition_rows(const int64_t* indptr, int64_t m2, int world, int64_t* bounds) {
  const double total = (double)(indptr[m2] - indptr[0]) + (double)m2;
  bounds[0] = 0;
  int64_t i = 0;
  for (int r = 1; r < world; ++r) {
    const double target = total * r / world;
    while (i < m2 && (double)(indptr[i] - indptr[0]) + (double)i < target) ++i;
    bounds[r] = std::max<int64_t>(i, bounds[r - 1]);
  }
  bounds[world] = m2;
}

struct HostCSR {
  int64_t nrows = 0, ncols = 0;
  std::vector<int64_t> p;
  std::vector<int32_t> i;
  std::vector<double> v;
  int64_t nnz() const { return (int64_t)i.size(); }
};

HostCSR transpose(const HostCSR& A) {
  HostCSR T;
  T.nrows = A.ncols;
  T.ncols = A.nrows;
  T.p.assign(T.nrows + 1, 0);
  for (int32_t c : A.i) T.p[c + 1]++;
  for (int64_t r = 0; r < T.nrows; ++r) T.p[r + 1] += T.p[r];
  T.i.resize(A.nnz());
  T.v.resize(A.nnz());
  std::vector<int64_t> pos(T.p.begin(), T.p.end() - 1);
  for (int64_t r = 0; r < A.nrows; ++r)
    for (int64_t q = A.p[r]; q < A.p[r + 1]; ++q) {
      int64_t d = pos[A.i[q]]++;
      T.i[d] = (int32_t)r;
      T.v[d] = A.v[q];
    }
  return T;
}

// B = A(rowperm, :) with columns renumbered by colmap (old col → new col), rows sorted.
HostCSR permute(const HostCSR& A, const std::vector<int64_t>* rowperm, const std::vector<int64_t>* colmap) {
  HostCSR B;
  B.nrows = A.nrows;
  B.ncols = A.ncols;
  B.p.assign(B.nrows + 1, 0);
  B.i.resize(A.nnz());
  B.v.resize(A.nnz());
  std::vector<std::pair<int32_t, double>> tmp;
  int64_t w = 0;
  for (int64_t r = 0; r < B.nrows; ++r) {
    int64_t ro = rowperm ? (*rowperm)[r] : r;
    tmp.clear();
    for (int64_t q = A.p[ro]; q < A.p[ro + 1]; ++q)
      tmp.emplace_back(colmap ? (int32_t)(*colmap)[A.i[q]] : A.i[q], A.v[q]);
    std::sort(tmp.begin(), tmp.end(), [](auto& a, auto& b) { return a.first < b.first; });
    for (auto& e : tmp) {
      B.i[w] = e.first;
      B.v[w] = e.second;
      ++w;
    }
    B.p[r + 1] = w;
  }
  return B;
}

struct DeviceArena {
  std::vector<void*> ptrs;
  size_t bytes = 0;
  ~DeviceArena() { release(); }
  void release() {
    for (void* p : ptrs) cudaFree(p);
    ptrs.clear();
    bytes = 0;
  }
  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    size_t b = std::max<size_t>(1, n) * sizeof(T);
    if (cudaMalloc(&p, b) != cudaSuccess) throw std::bad_alloc();
    ptrs.push_back(p);
    bytes += b;
    return (T*)p;
  }
  template <class T>
  T* upload(const std::vector<T>& v, cudaStream_t s) {
    T* d = alloc<T>(v.size());
    if (!v.empty()) cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s);
    return d;
  }
  template <class T>
  T* zeros(size_t n, cudaStream_t s) {
    T* d = alloc<T>(n);
    cudaMemsetAsync(d, 0, std::max<size_t>(1, n) * sizeof(T), s);
    return d;
  }
  // Free one allocation early (its size stays counted in `bytes`, an upper bound).
  void free_ptr(void* p) {
    for (size_t i = 0; i < ptrs.size(); ++i)
      if (ptrs[i] == p) {
        cudaFree(p);
        ptrs.erase(ptrs.begin() + (long)i);
        return;
      }
  }
};

// Host construction of a SymvPlan (kernels.cuh) for chunks [c_begin, c_end): chunk i contributes its row
// partial (rows rob[i]) and column partials (output blocks cob0[i] .. cob0[i]+ncob[i]−1); output block o
// (ids ob_lo + o, nob of them) has `width[o]` rows at x0[o].  Each block's slot list is ordered by the
// kind (row partials first) and then by chunk index: the fixed summation order of the reducers.
SymvPlan build_symv_plan(DeviceArena& m, cudaStream_t st, int64_t c_begin, int64_t c_end,
                         const std::vector<int32_t>& rob, const std::vector<int32_t>& cob0,
                         const std::vector<int32_t>& ncob, int32_t ob_lo, int32_t nob,
                         const std::vector<int32_t>& width, const std::vector<int64_t>& x0) {
  const int64_t nc = c_end - c_begin;
  std::vector<int64_t> lptr(nob + 1, 0);
  for (int64_t i = 0; i < nc; ++i) {
    lptr[rob[i] - ob_lo + 1] += 1;
    for (int32_t k = 0; k < ncob[i]; ++k) lptr[cob0[i] + k - ob_lo + 1] += 1;
  }
  for (int32_t o = 0; o < nob; ++o) lptr[o + 1] += lptr[o];
  std::vector<int64_t> woff((size_t)nc * 9, -1), fill(lptr.begin(), lptr.end() - 1);
  for (int64_t i = 0; i < nc; ++i) woff[i * 9] = 64 * fill[rob[i] - ob_lo]++;          // row partials first
  for (int64_t i = 0; i < nc; ++i)
    for (int32_t k = 0; k < ncob[i]; ++k) woff[i * 9 + 1 + k] = 64 * fill[cob0[i] + k - ob_lo]++;
  SymvPlan P{};
  static const bool det = !(std::getenv("QPB_DETERMINISTIC") && std::getenv("QPB_DETERMINISTIC")[0] == '0');
  P.slots = det ? m.zeros<double>((size_t)std::max<int64_t>(1, lptr[nob]) * 64, st) : nullptr;
  P.nob = nob;
  P.lptr = m.upload(lptr, st);
  P.woff = m.upload(woff, st);
  P.width = m.upload(width, st);
  P.x0 = m.upload(x0, st);
  P.c_begin = c_begin;
  P.ob_lo = ob_lo;
  cudaStreamSynchronize(st);   // host vectors
  return P;
}

struct Factor {
  Symbolic S;
  DevFactor d{};
  DeviceArena mem;
  bool ready = false;
  int64_t fs_bytes = 0, ws_bytes = 0;
  // partitioned inverse of big supernodes
  double* xtmp = nullptr;
  int32_t* big = nullptr;
  std::vector<int32_t> big_host;
  int n_big = 0;
  int32_t* sym = nullptr;            // symmetric roots (S⁻¹ stored)
  std::vector<int32_t> sym_host;
  int n_sym = 0;
  std::vector<GemmProb> sym_plan;
  SymvPlan sym_symv{};               // deterministic accumulation plan of k_symroot_gemv
  GemmProb* sym_dev = nullptr;
  int64_t* sym_pref_dev = nullptr;
  int64_t sym_total = 0;
  int64_t max_w2 = 0;
  std::vector<std::vector<GemmProb>> inv_plan;   // per height: [T1 problems..., X21 problems...]
  std::vector<int> inv_split;                    // per height: number of T1 problems
  GemmProb* inv_dev = nullptr;
  int64_t* inv_pref_dev = nullptr;
  std::vector<int64_t> inv_off;                  // per (height, phase) offsets into inv_dev / inv_pref_dev
  std::vector<int64_t> inv_total;
  unsigned long long* tprof_buf = nullptr;
  int32_t* fwd_x = nullptr;      // task queues without the symmetric-root shortcut
  int32_t* bwd_x = nullptr;
  double sym_discrepancy = 0.0;  // ‖y_sym − y_X‖ / ‖y_X‖ measured at factor time
  bool sym_enabled = false;
  double flat_discrepancy = -1.0;  // ‖y_flat − y_sweep‖ / ‖y_sweep‖ at factor time (−1: not tried)
  PiSweep pi{};                    // level products (partitioned inverse by levels)
  double pi_discrepancy = -1.0;    // ‖y_levels − y_sweeps‖ / ‖y_sweeps‖ at factor time (−1: not tried)
  double pi_ms[2] = {0, 0};        // factor-time F-solve medians: [0] task graph, [1] level products
  const int32_t* fwd_sym = nullptr;
  const int32_t* bwd_sym = nullptr;
  int64_t n_fwd_sym = 0, n_bwd_sym = 0, n_fwd_x = 0, n_bwd_x = 0;
  void use_symmetric_roots(bool on) {
    d.use_sym = on ? 1 : 0;
    d.fwd_tasks = on ? fwd_sym : fwd_x;
    d.bwd_tasks = on ? bwd_sym : bwd_x;
    d.n_fwd_tasks = on ? n_fwd_sym : n_fwd_x;
    d.n_bwd_tasks = on ? n_bwd_sym : n_bwd_x;
    sym_enabled = on;
  }
};

DevCSR upload_csr(DeviceArena& mem, const HostCSR& A, cudaStream_t s) {
  DevCSR d;
  d.nrows = A.nrows;
  d.ncols = A.ncols;
  d.nnz = A.nnz();
  d.p = mem.upload(A.p, s);
  d.i = mem.upload(A.i, s);
  d.v = mem.upload(A.v, s);
  return d;
}

}  // namespace

struct qp_ctx {
  std::string err;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int vectors_on_device = 0;
  int rank = 0, world = 1;
  // sharded ν rows: this rank owns inequality rows [row0, row1) of m2_global;
  // x-space work (F-solves, H, A) is replicated; Cᵀ(·) partial products and the PCG / IPM
  // reductions are all-reduced (NCCL, or the caller's qp_allreduce_fn).
  bool sharded = false;
  int64_t m2_global = 0, row0 = 0, row1 = 0;
  ncclComm_t nccl = nullptr;
  qp_allreduce_fn ar_fn = nullptr;
  void* ar_user = nullptr;
  qp_halo_fn halo_fn = nullptr;
  void* halo_user = nullptr;
  // halo plan of the sharded operator (qp_operator_halo_plan): owned boundaries b[0..world], the ranks'
  // windows of p and q, receive scratch
  struct HaloPlan {
    bool planned = false, enabled = false;
    std::vector<int64_t> b, plo, phi, qlo, qhi;
    double *from_prev = nullptr, *from_next = nullptr;
  } halo;
  double* ubuf = nullptr;        // N: all-reduced Cᵀ(·) in factor order (λ part zero)
  int64_t ws_limit = 0;
  int64_t n = 0, m1 = 0, m2 = 0;
  HostCSR H, A, C;
  std::vector<double> g, b, d;
  std::vector<int64_t> xperm_user;
  bool setup_done = false, factored = false, analysed = false;
  int precond = 1;
  int sm_count = 148;
  int vgrid = 148 * 4;     // grid for vector kernels (fixed ⇒ deterministic reductions)
  int tgrid = 148;         // persistent trsv grid

  // ordering + permuted operators
  std::vector<int64_t> perm;  // new → old for x block (n)
  DeviceArena mem;            // problem + vectors
  DevCSR Hf{}, Af{}, Atf{}, Cf{}, Ctf{}, Cnu{};
  double *gf = nullptr, *bv = nullptr, *dv = nullptr;
  int64_t* perm_dev = nullptr;   // N: factor position → original index (x: perm, λ: n+i)
  Factor FF;                     // LDLᵀ of F
  Factor FP;                     // Cholesky (LDLᵀ, positive pivots) of P_H
  // P_H extras
  std::vector<int64_t> perm_ph;
  int64_t* perm_ph_dev = nullptr;
  int64_t* t_row = nullptr;
  int32_t* t_col = nullptr;
  double* t_val = nullptr;
  int64_t nnz_t = 0;
  double* hdiag = nullptr;
  double* D_ph_last = nullptr;   // D of the current P_H numeric factor
  bool ph_valid = false;
  double t_factor_ph = 0;
  int64_t ph_refactors = 0;
  int64_t launches = 0;           // kernel launches issued by this context
  cudaGraphExec_t pcg_graph[4] = {nullptr, nullptr, nullptr, nullptr};   // GCH PCG iterations per
                                                                           // preconditioner; [3]: x-space
  int graph_launches[4] = {0, 0, 0, 0};
  // x-space twin buffers (n in factor order unless noted)
  double *xs_W = nullptr, *xs_p = nullptr, *xs_q = nullptr, *xs_r = nullptr, *xs_x = nullptr;
  double *xs_lam = nullptr /*m1*/, *xs_rhs = nullptr /*N, λ part zero*/;
  bool use_graphs = true;
  int graph_launches_per_chunk = 0;
  double last_eps = 0;            // PCG tolerance of the last IPM iteration

  // vectors
  double *xl = nullptr, *nu = nullptr, *s = nullptr;          // iterate (x_f; λ), ν, s
  double *rgre = nullptr, *rhs2 = nullptr, *xbuf = nullptr;   // (r_g; r_e), recovery rhs, sweep buffer
  double *rc = nullptr, *ra = nullptr, *Dk = nullptr, *rnu = nullptr, *ds = nullptr, *dxl = nullptr;
  double *px = nullptr, *pr = nullptr, *pz = nullptr, *pp = nullptr, *pq = nullptr, *xph = nullptr;
  double *vin = nullptr, *vin2 = nullptr, *vout = nullptr;  // staging for host I/O
  double* partial = nullptr;
  unsigned long long* tl_buf = nullptr;   // qp_debug_timeline
  double* dense_w = nullptr;         // explicit (F⁻¹)₁₁ (build_dense_w), column-major, leading dimension dw_ld
  int64_t dw_ld = 0, dw_nch = 0;
  int64_t dw_c0 = 0, dw_c1 = 0;      // this rank's chunk range (all chunks unless sharded)
  SymvPlan dw_plan_all{}, dw_plan{}; // k_dense_symv accumulation plans: all chunks (guard), this rank's
  double* dense_finv = nullptr;      // small N: the whole F⁻¹ (N × N, ld df_ld), F-solves as one symmetric GEMV
  int64_t df_ld = 0, df_nch = 0;
  const int2* df_chunks = nullptr;
  SymvPlan df_plan{};
  double* df_rhs = nullptr;          // materialised right-hand side (N)
  double df_discrepancy = -1;        // factor-time guard of the dense F⁻¹ (−1: not built)
  bool op_ready = false;             // qp_operator_apply: natural-order device copies of H, C, Cᵀ
  DevCSR opH{}, opC{}, opCt{};
  double *op_D = nullptr, *op_p = nullptr, *op_t = nullptr, *op_q = nullptr;
  double* phinv = nullptr;           // small m2: P_H⁻¹ (m2 × m2, ld pi_ld), rebuilt after every P_H refactor
  bool phinv_ready = false;
  int64_t pi_ld = 0, pi_nch = 0;
  const int2* pi_chunks = nullptr;
  SymvPlan pi_plan{};
  double* pi_unit = nullptr;
  double dw_share = 1.0;             // its share of W's bytes
  const int2* dw_chunks = nullptr;
  double dw_discrepancy = -1.0;
  const int32_t* long_c = nullptr;   // rows of C with > KF_LONG_ROW entries (k_pcg_step)
  int64_t n_long_c = 0;
  PcgState* pst = nullptr;
  IpmState* ist = nullptr;
  PcgState* h_pst = nullptr;  // pinned
  IpmState* h_ist = nullptr;  // pinned

  // IPM control
  qp_ipm_opts opts{};
  bool ipm_initialised = false;
  bool ipm_converged = false;
  int32_t ipm_k = 0;
  std::vector<int32_t> pcg_hist;
  double gmax = 0, bmax = 0, dmax = 0;
  double t_symbolic = 0, t_factor = 0;

  // profiling
  bool prof = false;
  struct Ev { int cls; cudaEvent_t a, b; };
  std::vector<Ev> evs;
  std::vector<cudaEvent_t> pool;
  double prof_ms[10] = {0};
  int64_t prof_cnt[10] = {0};

  cudaEvent_t get_ev() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  int begin(int cls) {
    if (!prof) return -1;
    Ev e{cls, get_ev(), get_ev()};
    cudaEventRecord(e.a, stream);
    evs.push_back(e);
    return (int)evs.size() - 1;
  }
  void end(int h) {
    if (h < 0) return;
    cudaEventRecord(evs[h].b, stream);
  }
  void harvest() {
    if (evs.empty()) return;
    cudaStreamSynchronize(stream);
    for (auto& e : evs) {
      float ms = 0;
      cudaEventElapsedTime(&ms, e.a, e.b);
      prof_ms[e.cls] += ms;
      prof_cnt[e.cls] += 1;
      pool.push_back(e.a);
      pool.push_back(e.b);
    }
    evs.clear();
  }
  // In-place all-reduce of cnt doubles on this context's stream (op: 0 sum, 1 max, 2 min).
  int allreduce(double* buf, int64_t cnt, int op) {
    if (!sharded || cnt <= 0) return 0;
    if (ar_fn) {
      int rc = ar_fn(ar_user, buf, cnt, op, (void*)stream);
      if (rc != 0) err = "qp_allreduce_fn returned " + std::to_string(rc);
      return rc != 0 ? QP_ENCCL : 0;
    }
    const ncclRedOp_t o = op == 0 ? ncclSum : (op == 1 ? ncclMax : ncclMin);
    ncclResult_t r = nccl_api().all_reduce(buf, buf, (size_t)cnt, ncclFloat64, o, nccl, stream);
    if (r != ncclSuccess) {
      err = std::string("ncclAllReduce: ") + nccl_api().error_string(r);
      return QP_ENCCL;
    }
    return 0;
  }
  // Neighbour exchange on this context's stream (see qp_halo_fn); counts of 0 are skipped.
  int exchange(const double* to_prev, int64_t n_tp, const double* to_next, int64_t n_tn, double* from_prev, int64_t n_fp,
               double* from_next, int64_t n_fn) {
    if (halo_fn) {
      int rc = halo_fn(halo_user, to_prev, n_tp, to_next, n_tn, from_prev, n_fp, from_next, n_fn, (void*)stream);
      if (rc != 0) err = "qp_halo_fn returned " + std::to_string(rc);
      return rc != 0 ? QP_ENCCL : 0;
    }
    NcclApi& api = nccl_api();
    if (!nccl || !api.send || !api.recv || !api.group_start || !api.group_end) {
      err = "halo exchange needs NCCL send/recv or opts.halo";
      return QP_ENCCL;
    }
    ncclResult_t r = api.group_start();
    if (r == ncclSuccess && n_tp > 0) r = api.send(to_prev, (size_t)n_tp, ncclFloat64, rank - 1, nccl, stream);
    if (r == ncclSuccess && n_tn > 0) r = api.send(to_next, (size_t)n_tn, ncclFloat64, rank + 1, nccl, stream);
    if (r == ncclSuccess && n_fp > 0) r = api.recv(from_prev, (size_t)n_fp, ncclFloat64, rank - 1, nccl, stream);
    if (r == ncclSuccess && n_fn > 0) r = api.recv(from_next, (size_t)n_fn, ncclFloat64, rank + 1, nccl, stream);
    ncclResult_t r2 = api.group_end();
    if (r == ncclSuccess) r = r2;
    if (r != ncclSuccess) {
      err = std::string("ncclSend/ncclRecv: ") + api.error_string(r);
      return QP_ENCCL;
    }
    return 0;
  }
  ~qp_ctx() {
    harvest();
    if (nccl) nccl_api().comm_destroy(nccl);
    for (auto& g : pcg_graph)
      if (g) cudaGraphExecDestroy(g);
    for (auto e : pool) cudaEventDestroy(e);
    if (h_pst) cudaFreeHost(h_pst);
    if (tl_buf) {
      timeline_enable(nullptr);
      cudaFree(tl_buf);
    }
    if (h_ist) cudaFreeHost(h_ist);
    FF.mem.release();
    FP.mem.release();
    mem.release();
    if (own_stream && stream) cudaStreamDestroy(stream);
  }
};

namespace {

int fail(qp_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

int cuda_check(qp_ctx* c, const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, QP_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
  return QP_OK;
}

int sync_check(qp_ctx* c, const char* where) {
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, QP_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
  return QP_OK;
}

std::string check_csr(const qp_csr* M, int64_t nr, int64_t nc, const char* name, HostCSR& out) {
  if (!M) return std::string(name) + " is NULL";
  if (M->nrows != nr || M->ncols != nc)
    return std::string(name) + " has shape " + std::to_string(M->nrows) + "x" + std::to_string(M->ncols) +
           ", expected " + std::to_string(nr) + "x" + std::to_string(nc);
  if (nr > 0 && (!M->indptr)) return std::string(name) + ": NULL indptr";
  out.nrows = nr;
  out.ncols = nc;
  out.p.assign(M->indptr, M->indptr + nr + 1);
  if (out.p[0] != 0) return std::string(name) + ": indptr[0] != 0";
  for (int64_t r = 0; r < nr; ++r)
    if (out.p[r + 1] < out.p[r]) return std::string(name) + ": indptr not monotone";
  int64_t nnz = out.p[nr];
  if (nnz > 0 && (!M->indices || !M->values)) return std::string(name) + ": NULL indices/values";
  out.i.assign(M->indices, M->indices + nnz);
  out.v.assign(M->values, M->values + nnz);
  for (int64_t r = 0; r < nr; ++r)
    for (int64_t q = out.p[r]; q < out.p[r + 1]; ++q) {
      if (out.i[q] < 0 || out.i[q] >= nc) return std::string(name) + ": column index out of range";
      if (q > out.p[r] && out.i[q] <= out.i[q - 1]) return std::string(name) + ": columns not sorted/unique";
      if (!std::isfinite(out.v[q])) return std::string(name) + ": non-finite value";
    }
  return "";
}

// Upload a symbolic plan and allocate numeric storage for one factor.
std::string upload_factor(qp_ctx* c, Factor& F, int64_t ws_limit) {
  Symbolic& S = F.S;
  cudaStream_t st = c->stream;
  if (S.ws_size * 8 > ws_limit)
    return "multifrontal workspace " + std::to_string(S.ws_size * 8 / (1 << 20)) + " MiB exceeds the limit";
  try {
    DeviceArena& m = F.mem;
    DevFactor& d = F.d;
    d.N = S.N;
    d.ns = S.ns;
    d.nb = S.nb;
    d.n_tiles = (int64_t)S.tile_blk.size();
    d.n_fwd_tasks = (int64_t)S.fwd_tasks.size();
    d.n_bwd_tasks = (int64_t)S.bwd_tasks.size();
    d.sn_start = m.upload(S.sn_start, st);
    d.sn_rowptr = m.upload(S.sn_rowptr, st);
    d.sn_rows = m.upload(S.sn_rows, st);
    d.front_off = m.upload(S.front_off, st);
    d.sn_blk0 = m.upload(S.sn_blk0, st);
    d.blk_col0 = m.upload(S.blk_col0, st);
    d.blk_w = m.upload(S.blk_w, st);
    d.blk_noff = m.upload(S.blk_noff, st);
    d.blk_rows = m.upload(S.blk_rows, st);
    d.blk_inv = m.upload(S.blk_inv, st);
    d.blk_off = m.upload(S.blk_off, st);
    d.tile_blk = m.upload(S.tile_blk, st);
    d.tile_r0 = m.upload(S.tile_r0, st);
    d.tile_nr = m.upload(S.tile_nr, st);
    d.tile_dptr = m.upload(S.tile_dptr, st);
    d.tile_dlist = m.upload(S.tile_dlist, st);
    d.fwd_tasks = m.upload(S.fwd_tasks, st);
    d.bwd_tasks = m.upload(S.bwd_tasks, st);
    F.fwd_x = m.upload(S.fwd_tasks_x, st);
    F.bwd_x = m.upload(S.bwd_tasks_x, st);
    if (S.sym_c1 > S.sym_c0) {   // the symmetric-root GEMV's deterministic accumulation plan
      const int64_t nc = S.sym_c1 - S.sym_c0;
      std::vector<int32_t> rob(nc), cob0(nc), ncob(nc);
      int32_t lo = INT32_MAX, hi = -1;
      for (int64_t i = 0; i < nc; ++i) {
        const int64_t x = S.sym_c0 + i;
        const int32_t bI = S.xt_bI[x], bK = S.xt_bK[x], nK = S.xt_nK[x];
        const int64_t rI = S.blk_col0[bI], cK = S.blk_col0[bK];
        const int64_t ncol = S.blk_col0[bK + nK - 1] + S.blk_w[bK + nK - 1] - cK;
        const int64_t ncol_t = std::min<int64_t>(rI, cK + ncol) - cK;
        rob[i] = bI;
        cob0[i] = bK;
        ncob[i] = (int32_t)(ncol_t / 64);
        lo = std::min({lo, bI, bK});
        hi = std::max(hi, bI);
      }
      const int32_t nob = hi - lo + 1;
      std::vector<int32_t> width(nob);
      std::vector<int64_t> x0(nob);
      for (int32_t o = 0; o < nob; ++o) {
        width[o] = S.blk_w[lo + o];
        x0[o] = S.blk_col0[lo + o];
      }
      F.sym_symv = build_symv_plan(m, st, S.sym_c0, S.sym_c1, rob, cob0, ncob, lo, nob, width, x0);
    }
    d.fwd_expect = m.upload(S.fwd_expect, st);
    d.bwd_expect = m.upload(S.bwd_expect, st);
    d.ws = m.alloc<double>(S.ws_size);
    d.fstore = m.zeros<double>(S.fs_size, st);
    d.Dpiv = m.zeros<double>(S.N, st);
    d.pivsign = m.upload(S.pivsign, st);
    d.acc = m.zeros<double>(S.N, st);
    d.tacc = m.zeros<double>(S.N, st);
    d.cnt_f = m.zeros<unsigned long long>(S.ns, st);
    d.cnt_b = m.zeros<unsigned long long>(S.nb, st);
    d.ready_f = m.zeros<unsigned int>(S.nb, st);
    d.ready_b = m.zeros<unsigned int>(S.nb, st);
    d.sweep = m.zeros<unsigned int>(4, st);
    d.blk_sn = m.upload(S.blk_sn, st);
    d.sn_xinv = m.upload(S.sn_xinv, st);
    d.xt_bI = m.upload(S.xt_bI, st);
    d.xt_bK = m.upload(S.xt_bK, st);
    d.xt_nK = m.upload(S.xt_nK, st);
    d.xb_bK = m.upload(S.xb_bK, st);
    d.xb_bI = m.upload(S.xb_bI, st);
    d.xb_nI = m.upload(S.xb_nI, st);
    d.sn_xtr = m.upload(S.sn_xtr, st);
    d.sn_ldx = m.upload(S.sn_ldx, st);
    d.sn_sinv = m.upload(S.sn_sinv, st);
    d.sn_nblk = m.upload(S.sn_nblk, st);
    d.blk_dptr = m.upload(S.blk_dptr, st);
    d.blk_dest = m.upload(S.blk_dest, st);
    d.mf_group = S.mf_group;
    d.snw_fwd = m.upload(S.snw_fwd, st);
    d.snw_bwd = m.upload(S.snw_bwd, st);
    {
      std::vector<int32_t> desc;
      desc.reserve(S.lvl_blk.size() * 8);
      for (int32_t b : S.lvl_blk) {
        const int64_t lo = S.blk_off[b], io = S.blk_inv[b], ro = S.blk_rows[b];
        desc.insert(desc.end(), {(int32_t)(uint32_t)(lo & 0xffffffffll), (int32_t)(lo >> 32),
                                 (int32_t)(uint32_t)(io & 0xffffffffll), (int32_t)(io >> 32),
                                 (int32_t)(uint32_t)(ro & 0xffffffffll), (int32_t)(ro >> 32), S.blk_col0[b],
                                 (int32_t)(S.blk_w[b] | (S.blk_noff[b] << 6))});
      }
      d.lvl_desc = reinterpret_cast<const int4*>(m.upload(desc, st));
    }
    d.lvl_cut = S.lvl_cut;
    d.lvl_cut = (int32_t)std::min<size_t>(S.lvl_g.size(), (size_t)std::min<int32_t>(S.lvl_cut, LVL_MAX));
    for (int L = 0; L <= d.lvl_cut; ++L) d.lvl_ptr_h[L] = L < (int)S.lvl_ptr.size() ? S.lvl_ptr[L] : 0;
    for (int L = 0; L < d.lvl_cut; ++L) d.lvl_g_h[L] = (int8_t)S.lvl_g[L];
    d.flat = 0;
    if (S.flat) {
      d.fl_rc0 = S.fl_rc0;
      d.fl_roff = m.upload(S.fl_roff, st);
      d.fl_rows = m.upload(S.fl_rows, st);
      d.fl_moff = m.upload(S.fl_moff, st);
      d.fl_mval = m.zeros<double>(S.fl_msize, st);
      d.fl_cp = m.upload(S.fl_cp, st);
      d.fl_ci = m.upload(S.fl_ci, st);
      d.fl_rp = m.upload(S.fl_rp, st);
      d.fl_rj = m.upload(S.fl_rj, st);
      d.fl_r2c = m.upload(S.fl_r2c, st);
      d.fl_nval = m.zeros<double>(S.fl_ci.size(), st);
      d.fl_col2sn = m.upload(S.fl_col2sn, st);
      d.fl_mt_J = m.upload(S.fl_mt_J, st);
      d.fl_mt_q0 = m.upload(S.fl_mt_q0, st);
      d.fl_mt_nq = m.upload(S.fl_mt_nq, st);
      d.fl_nmt = (int64_t)S.fl_mt_J.size();
      d.fl_mr_ptr = m.upload(S.fl_mr_ptr, st);
      d.fl_mr_col = m.upload(S.fl_mr_col, st);
      d.fl_mr_val = m.zeros<double>(S.fl_mr_col.size(), st);
      std::vector<int32_t> units;   // 8 int32 per unit: moff lo, moff hi, roff, col0, ld, rows | cols << 16, 0, 0
      for (size_t t = 0; t < S.fl_mt_J.size(); ++t) {
        const int64_t J = S.fl_mt_J[t], q0 = S.fl_mt_q0[t], nq = S.fl_mt_nq[t];
        const int64_t c0 = S.sn_start[J], w = S.sn_start[J + 1] - c0, nr = S.fl_roff[J + 1] - S.fl_roff[J];
        for (int64_t cg = 0; cg < w; cg += 8)
          for (int64_t rg = 0; rg < nq; rg += 64) {
            const int64_t mo = S.fl_moff[J] + cg * nr + q0 + rg;
            units.insert(units.end(), {(int32_t)(uint32_t)(mo & 0xffffffffll), (int32_t)(mo >> 32),
                                       (int32_t)(S.fl_roff[J] + q0 + rg), (int32_t)(c0 + cg), (int32_t)nr,
                                       (int32_t)(std::min<int64_t>(64, nq - rg) | (std::min<int64_t>(8, w - cg) << 16)),
                                       0, 0});
          }
      }
      d.fl_nunits = (int64_t)units.size() / 8;
      d.fl_units = reinterpret_cast<const int4*>(m.upload(units, st));
      {   // fixed-order reduction lists of the unit partials (no floating-point atomics)
        const int64_t nu = d.fl_nunits, wr = S.N - S.fl_rc0, rc0 = S.fl_rc0;
        std::vector<int64_t> fr_ptr(wr + 1, 0), bc_ptr(rc0 + 1, 0);
        for (int64_t u = 0; u < nu; ++u) {
          const int64_t roff = units[8 * u + 2], col0 = units[8 * u + 3], sh = units[8 * u + 5];
          const int64_t nrows = sh & 0xffff, ncols = sh >> 16;
          for (int64_t k = 0; k < nrows; ++k) fr_ptr[S.fl_rows[roff + k] + 1] += 1;
          for (int64_t k = 0; k < ncols; ++k) bc_ptr[col0 + k + 1] += 1;
        }
        for (int64_t r = 0; r < wr; ++r) fr_ptr[r + 1] += fr_ptr[r];
        for (int64_t c2 = 0; c2 < rc0; ++c2) bc_ptr[c2 + 1] += bc_ptr[c2];
        std::vector<int32_t> fr_src(fr_ptr[wr]), bc_src(bc_ptr[rc0]);
        std::vector<int64_t> ff(fr_ptr.begin(), fr_ptr.end() - 1), bf(bc_ptr.begin(), bc_ptr.end() - 1);
        for (int64_t u = 0; u < nu; ++u) {
          const int64_t roff = units[8 * u + 2], col0 = units[8 * u + 3], sh = units[8 * u + 5];
          const int64_t nrows = sh & 0xffff, ncols = sh >> 16;
          for (int64_t k = 0; k < nrows; ++k) fr_src[ff[S.fl_rows[roff + k]]++] = (int32_t)(u * 64 + k);
          for (int64_t k = 0; k < ncols; ++k) bc_src[bf[col0 + k]++] = (int32_t)(u * 8 + k);
        }
        d.fl_fslot = m.zeros<double>((size_t)std::max<int64_t>(1, nu) * 64, st);
        d.fl_bslot = m.zeros<double>((size_t)std::max<int64_t>(1, nu) * 8, st);
        d.fl_fr_ptr = m.upload(fr_ptr, st);
        d.fl_fr_src = m.upload(fr_src, st);
        d.fl_bc_ptr = m.upload(bc_ptr, st);
        d.fl_bc_src = m.upload(bc_src, st);
        cudaStreamSynchronize(st);   // local host buffers
      }
      cudaStreamSynchronize(st);   // `units` is a local host buffer
    }
    d.ready_sb = m.zeros<unsigned int>(S.ns, st);
    d.sn_done_b = m.zeros<unsigned long long>(S.ns, st);
    d.xexp_f = m.upload(S.xexp_f, st);
    d.xexp_b = m.upload(S.xexp_b, st);
    d.xinv = m.alloc<double>(S.x_size);
    d.vbuf = m.zeros<double>(S.N, st);
    d.cntx_f = m.zeros<unsigned long long>(S.nb, st);
    d.cntx_b = m.zeros<unsigned long long>(S.nb, st);
    d.vready_f = m.zeros<unsigned int>(S.nb, st);
    d.vready_b = m.zeros<unsigned int>(S.nb, st);
    F.xtmp = m.alloc<double>(S.xtmp_size);
    {
      std::vector<int32_t> big;
      int64_t mw2 = 0;
      for (int64_t J = 0; J < S.ns; ++J)
        if (S.sn_xinv[J] >= 0) {
          big.push_back((int32_t)J);
          int64_t w = S.sn_start[J + 1] - S.sn_start[J];
          mw2 = std::max(mw2, w * S.sn_ldx[J]);
        }
      F.n_big = (int)big.size();
      F.max_w2 = mw2;
      F.big = m.upload(big, st);
      F.big_host = big;
      std::vector<int32_t> sym;
      for (int32_t J : big)
        if (S.sn_sinv[J] >= 0) sym.push_back(J);
      F.n_sym = (int)sym.size();
      F.sym = m.upload(sym, st);
      F.sym_host = sym;
    }
    d.asm_dst = m.upload(S.asm_dst, st);
    d.asm_val = m.upload(S.asm_val, st);
    d.asm_src = m.upload(S.asm_src, st);
    d.n_asm = (int64_t)S.asm_dst.size();
    d.diag_dst = m.upload(S.diag_dst, st);
    d.asm_diag = m.upload(S.asm_diag, st);
    d.lev_fronts = m.upload(S.lev_fronts, st);
    d.lev_zpref = m.upload(S.lev_zpref, st);
    d.relind = m.upload(S.relind, st);
    d.relind_off = m.upload(S.relind_off, st);
    d.grp_P = m.upload(S.grp_P, st);
    d.grp_pc = m.upload(S.grp_pc, st);
    d.grp_ptr = m.upload(S.grp_ptr, st);
    d.grp_K = m.upload(S.grp_K, st);
    d.grp_j = m.upload(S.grp_j, st);
    d.act = m.upload(S.act, st);
    d.pan_pref = m.upload(S.pan_pref, st);
    d.upd_pref = m.upload(S.upd_pref, st);
    d.status = m.zeros<int>(1, st);
    d.tprof = nullptr;
    d.use_sym = 0;
    d.sweep_var = getenv("QPB_SWEEP_VAR") ? atoi(getenv("QPB_SWEEP_VAR")) : 1;
    d.l2hint = getenv("QPB_L2HINT") ? atoi(getenv("QPB_L2HINT")) : 0;
    F.fwd_sym = d.fwd_tasks;
    F.bwd_sym = d.bwd_tasks;
    F.n_fwd_sym = d.n_fwd_tasks;
    F.n_bwd_sym = d.n_bwd_tasks;
    F.n_fwd_x = (int64_t)S.fwd_tasks_x.size();
    F.n_bwd_x = (int64_t)S.bwd_tasks_x.size();
    d.ttrace_cap = std::max<int64_t>(std::max(F.n_fwd_sym, F.n_bwd_sym), std::max(F.n_fwd_x, F.n_bwd_x));
    F.tprof_buf = m.alloc<unsigned long long>(80 + 12 * d.ttrace_cap);
    F.fs_bytes = S.fs_size * 8;
    F.ws_bytes = S.ws_size * 8;
  } catch (std::bad_alloc&) {
    return "cudaMalloc failed (factor storage)";
  }
  return "";
}

// Plan of the recursive blocked inversion X_J = L_JJ⁻¹ for every big supernode:
// split the tile range [lo, hi) at mid; X21 = −X22 · (L21 · X11), bottom-up by height.
void plan_inverse(qp_ctx* c, Factor& F) {
  const Symbolic& S = F.S;
  F.inv_plan.clear();
  F.inv_split.clear();
  std::vector<std::vector<GemmProb>> t1, x21;
  for (int32_t J : F.big_host) {
    const int64_t w = S.sn_start[J + 1] - S.sn_start[J];
    const int64_t T = S.sn_blk0[J + 1] - S.sn_blk0[J];
    const int64_t ldx = S.sn_ldx[J];
    double* X = F.d.xinv + S.sn_xinv[J];
    double* tmp = F.xtmp + S.sn_xtmp[J];
    std::vector<int64_t> tmp_used(64, 0);
    auto tb = [&](int64_t t) { return std::min<int64_t>(t * BW, w); };
    std::function<int(int64_t, int64_t)> gen = [&](int64_t lo, int64_t hi) -> int {
      if (hi - lo <= 1) return 0;
      const int64_t mid = lo + (hi - lo) / 2;
      const int h = 1 + std::max(gen(lo, mid), gen(mid, hi));
      if ((int)t1.size() < h) { t1.resize(h); x21.resize(h); }
      if ((int)tmp_used.size() <= h) tmp_used.resize(h + 1, 0);
      const int64_t a = tb(lo), m = tb(mid), e = tb(hi);
      const int M2 = (int)(e - m), M1 = (int)(m - a);
      double* T1 = tmp + tmp_used[h];
      tmp_used[h] += (int64_t)M2 * M1;
      GemmProb p1{X + m + a * ldx, X + a + a * ldx, T1, M2, M1, M1, (int)ldx, (int)ldx, M2, 1.0, 0.0, 2, 0};
      GemmProb p2{X + m + m * ldx, T1, X + m + a * ldx, M2, M1, M2, (int)ldx, M2, (int)ldx, -1.0, 0.0, 1, 0};
      t1[h - 1].push_back(p1);
      x21[h - 1].push_back(p2);
      return h;
    };
    gen(0, T);
  }
  std::vector<GemmProb> all;
  std::vector<int64_t> pref;
  F.inv_off.clear();
  F.inv_total.clear();
  for (size_t h = 0; h < t1.size(); ++h)
    for (int phase = 0; phase < 2; ++phase) {
      const auto& v = phase == 0 ? t1[h] : x21[h];
      F.inv_off.push_back((int64_t)all.size());
      int64_t acc = 0;
      for (const GemmProb& p : v) {
        pref.push_back(acc);
        acc += (int64_t)((p.M + 127) / 128) * ((p.N + 127) / 128);   // k_gemm128 tiles
        all.push_back(p);
      }
      pref.push_back(acc);
      all.push_back(GemmProb{});  // keeps all[] aligned with pref[] (one sentinel per group)
      F.inv_total.push_back(acc);
    }
  F.inv_dev = F.mem.upload(all, c->stream);
  F.inv_pref_dev = F.mem.upload(pref, c->stream);
  F.inv_split.assign(t1.size(), 0);
  for (size_t h = 0; h < t1.size(); ++h) F.inv_split[h] = (int)t1[h].size();
  // S_J⁻¹ = X_Jᵀ (D_J⁻¹ X_J) for the symmetric roots: lower tiles, diagonal tiles full
  std::vector<GemmProb> sp;
  std::vector<int64_t> spref;
  int64_t acc = 0;
  for (int32_t J : F.sym_host) {
    const int64_t w = S.sn_start[J + 1] - S.sn_start[J], ldx = S.sn_ldx[J];
    GemmProb g{F.d.xinv + S.sn_xtr[J], F.d.xinv + S.sn_xinv[J], F.d.xinv + S.sn_sinv[J], (int)w, (int)w, (int)w,
               (int)ldx, (int)ldx, (int)ldx, 1.0, 0.0, 2 | 4 | 8, 0};
    spref.push_back(acc);
    acc += ((w + 127) / 128) * ((w + 127) / 128);
    sp.push_back(g);
  }
  spref.push_back(acc);
  sp.push_back(GemmProb{});
  F.sym_total = acc;
  F.sym_dev = F.mem.upload(sp, c->stream);
  F.sym_pref_dev = F.mem.upload(spref, c->stream);
}

void run_inverse(qp_ctx* c, Factor& F) {
  if (F.n_big == 0) return;
  build_xinv(F.d, F.big, F.n_big, F.max_w2, c->stream);
  for (size_t h = 0; h < F.inv_split.size(); ++h)
    for (int phase = 0; phase < 2; ++phase) {
      const size_t g = 2 * h + phase;
      const int64_t off = F.inv_off[g];
      gemm_batched(F.inv_dev + off, F.inv_pref_dev + off, F.inv_split[h], F.inv_total[g], c->stream);
    }
  transpose_xinv(F.d, F.big, F.n_big, F.max_w2, c->stream);
  if (F.n_sym > 0) {
    scale_xinv_rows(F.d, F.sym, F.n_sym, F.max_w2, false, c->stream);   // X ← D⁻¹X
    gemm_batched(F.sym_dev, F.sym_pref_dev, F.n_sym, F.sym_total, c->stream);
    scale_xinv_rows(F.d, F.sym, F.n_sym, F.max_w2, true, c->stream);    // X restored (X/Xᵀ fallback path)
  }
}

// Numeric multifrontal factorization (assembly → per level: extend-add, blocked steps).
int numeric_factor(qp_ctx* c, Factor& F, const double* src_vals, const double* D, const int64_t* dperm,
                   const char* what) {
  cudaStream_t st = c->stream;
  const Symbolic& S = F.S;
  cudaMemsetAsync(F.d.status, 0, sizeof(int), st);
  size_t si = 0;
  for (int64_t L = 0; L < S.n_levels; ++L) {
    const LevelEA& le = S.level_ea[L];
    mf_assemble_level(F.d, le.fr_off, le.n_fr, S.lev_zpref[le.fr_off + le.n_fr], le.asm_off, le.n_asm, src_vals, D,
                      dperm, st);
    mf_extend_add(F.d, S.level_ea[L].grp_off, S.level_ea[L].n_grp, st);
    while (si < S.steps.size() && S.steps[si].level == L) {
      const StepDesc& sd = S.steps[si];
      mf_step(F.d, sd.k, sd.k0, sd.kind, sd.act_off, sd.n_act, S.pref_off[si], sd.pan_total, sd.upd_total, st);
      ++si;
    }
  }
  run_inverse(c, F);   // partitioned inverse of the big supernodes' diagonal blocks
  int rc = cuda_check(c, what);
  if (rc) return rc;
  int status = 0;
  cudaMemcpyAsync(&status, F.d.status, sizeof(int), cudaMemcpyDeviceToHost, st);
  rc = sync_check(c, what);
  if (rc) return rc;
  if (status) return fail(c, QP_ENOTSPD, std::string(what) + ": pivot of wrong sign / zero (inertia check)");
  F.ready = true;
  return QP_OK;
}

// y = F⁻¹ rhs (factor order, N), forward + backward sweeps.
double* pst_red(qp_ctx* c) { return (double*)((char*)c->pst + offsetof(PcgState, red)); }
double* ist_red(qp_ctx* c) { return (double*)((char*)c->ist + offsetof(IpmState, red)); }

void sym_gemv(qp_ctx* c, Factor& F, double* x, const int* done, const double* sub = nullptr) {
  if (!F.sym_enabled) return;
  c->launches += F.sym_symv.slots ? 2 : 1;
  symroot_gemv(F.d, x, F.S.sym_c0, F.S.sym_c1, &F.sym_symv, done, c->sm_count * 3, c->stream, sub);
}

// One F-solve on the right-hand side described by r: the task-graph sweeps, or — flattened forest —
// forward product, root GEMV, backward product (three dependency-free kernels).
void f_solve_sweeps(qp_ctx* c, const SweepRhs& r, double* out) {
  Factor& F = c->FF;
  if (c->dense_finv) {   // small N: out = F⁻¹ v, one deterministic symmetric GEMV (DESIGN §5 "dense F⁻¹")
    c->launches += c->df_plan.slots ? 3 : 2;
    int h = c->begin(8);
    gather_rhs(r, c->df_rhs, out, F.d.N, c->sm_count, c->stream);
    dense_symv(c->dense_finv, c->df_ld, F.d.N, c->df_chunks, c->df_nch, &c->df_plan, c->df_rhs, out, r.done_flag,
               c->sm_count, c->stream);
    c->end(h);
    return;
  }
  if (F.pi.enabled) {   // level products: leaf levels, one product kernel per upper level, root GEMV, and back
    int nl = 0;
    for (int L = 0; L < F.pi.nlev; ++L) nl += F.pi.lev_ptr[L + 1] > F.pi.lev_ptr[L] ? 1 : 0;
    c->launches += (r.rhs_ready ? 0 : 1) + (F.pi.st_n > 0 ? 2 : 2 * F.d.lvl_cut) + 2 * nl;
    int h = c->begin(0);
    pi_forward(F.d, F.pi, r, out, c->sm_count, c->stream);
    c->end(h);
    h = c->begin(8);
    sym_gemv(c, F, out, r.done_flag, F.d.acc);
    c->end(h);
    h = c->begin(1);
    pi_backward(F.d, F.pi, out, r.done_flag, c->stream);
    c->end(h);
    return;
  }
  c->launches += F.d.flat ? (r.rhs_ready ? 4 : 5) : 2 + 2 * F.d.lvl_cut;
  int h = c->begin(0);
  if (F.d.flat) flat_forward(F.d, r, out, c->sm_count, c->stream);
  else trsv_forward(F.d, r, out, c->tgrid, c->stream);
  c->end(h);
  h = c->begin(8);
  sym_gemv(c, F, out, r.done_flag);
  c->end(h);
  h = c->begin(1);
  if (F.d.flat) flat_backward(F.d, out, r.done_flag, c->sm_count, c->stream);
  else trsv_backward(F.d, out, r.done_flag, c->tgrid, c->stream);
  c->end(h);
}

void f_solve_dev(qp_ctx* c, const double* rhs_f, double* out) {
  SweepRhs r{};
  r.rhs = rhs_f;
  f_solve_sweeps(c, r, out);
}

// q = K_F p (a1–a5): Cᵀp fused into the forward sweep, F-solve, q = D∘p − C w.
constexpr int NT_HOST = 256;   // threads per CTA of the vector kernels (kernels.cuh NT)

static bool pregather_on() {
  static const bool on = !(std::getenv("QPB_PREGATHER") && std::getenv("QPB_PREGATHER")[0] == '0');
  return on;
}

// rhs_ready: the fused PCG step already prepared this F-solve's right-hand side (flat: acc / vbuf / xbuf;
// pregather: ubuf).
int kf_apply_dev(qp_ctx* c, const double* D, const double* p, double* q, bool pcg_mode, bool fsolve_only = false,
                 bool rhs_ready = false) {
  c->launches += fsolve_only ? 0 : 1;
  SweepRhs r{};
  r.done_flag = pcg_mode ? &c->pst->done : nullptr;
  if (c->dense_w && (rhs_ready || pcg_mode)) {   // w = W·Cᵀp
    if (!rhs_ready) {   // (P_H or sharded PCG: not fused) Cᵀp into ubuf, w accumulator zeroed
      spmv(c->Ctf, p, c->ubuf, r.done_flag, c->vgrid, c->stream);
      c->launches += 1;
      if (int rc = c->allreduce(c->ubuf, c->n, 0)) return rc;   // u = Σ_ranks C_gᵀ p_g
      cudaMemsetAsync(c->xbuf, 0, c->n * 8, c->stream);
    }   // else ubuf = Cᵀp and xbuf[0, n) = 0 come from the fused step's phase D
    int h = c->begin(9);
    dense_symv(c->dense_w, c->dw_ld, c->n, c->dw_chunks + c->dw_c0, c->dw_c1 - c->dw_c0, &c->dw_plan, c->ubuf, c->xbuf,
               r.done_flag, c->sm_count, c->stream, false);
    c->end(h);
    h = c->begin(7);   // its fixed-order reduction (profiled apart from the GEMV)
    symv_reduce(&c->dw_plan, c->xbuf, r.done_flag, c->sm_count, c->stream);
    c->end(h);
    c->launches += c->dw_plan.slots ? 2 : 1;   // GEMV (+ its fixed-order reduction)
    if (int rc = c->allreduce(c->xbuf, c->n, 0)) return rc;       // w = Σ_ranks (this rank's chunks)·u
    if (fsolve_only) return 0;
    h = c->begin(2);
    kf_q(c->Cf, c->long_c, c->n_long_c, D, p, c->xbuf, q, c->partial, c->pst, c->vgrid, c->stream, pcg_mode);
    c->end(h);
    if (c->sharded && pcg_mode) {
      if (int rc = c->allreduce(pst_red(c), 1, 0)) return rc;
      finalize(FIN_PCG_PQ, c->pst, c->ist, c->precond, c->stream);
      c->launches += 1;
    }
    return 0;
  }
  r.rhs_ready = rhs_ready && (c->FF.d.flat || (c->FF.pi.enabled && !c->dense_finv)) ? 1 : 0;
  if (rhs_ready && !c->FF.d.flat) {
    r.rhs = c->ubuf;
  } else if (c->sharded || (pregather_on() && !c->FF.d.flat)) {
    // u = Σ_ranks C_gᵀ p_g (one coalesced SpMV before the sweeps: every sweep task then reads its
    // right-hand side with one load), then the replicated F-solve on [u; 0]
    spmv(c->Ctf, p, c->ubuf, r.done_flag, c->vgrid, c->stream);
    c->launches += 1;
    if (int rc = c->allreduce(c->ubuf, c->n, 0)) return rc;
    r.rhs = c->ubuf;
  } else {
    r.ct = c->Ctf;   // Cᵀp fused into the forward sweep (a1)
    r.p = p;
  }
  f_solve_sweeps(c, r, c->xbuf);
  if (fsolve_only) return 0;   // q = D∘p − C w comes from the fused PCG step
  int h = c->begin(2);
  kf_q(c->Cf, c->long_c, c->n_long_c, D, p, c->xbuf, q, c->partial, c->pst, c->vgrid, c->stream, pcg_mode);
  c->end(h);
  if (c->sharded && pcg_mode) {
    if (int rc = c->allreduce(pst_red(c), 1, 0)) return rc;
    finalize(FIN_PCG_PQ, c->pst, c->ist, c->precond, c->stream);
    c->launches += 1;
  }
  return 0;
}

// z = P_H⁻¹ r (a7), P_H factor order via perm_ph.
void ph_apply_dev(qp_ctx* c, const double* r, double* z, const int* done) {
  if (c->phinv_ready) {   // small m2: z = P_H⁻¹ r, one deterministic symmetric GEMV
    c->launches += c->pi_plan.slots ? 3 : 2;
    int h = c->begin(4);
    zero_flag(z, c->m2, done, c->stream);
    dense_symv(c->phinv, c->pi_ld, c->m2, c->pi_chunks, c->pi_nch, &c->pi_plan, r, z, done, c->sm_count, c->stream);
    c->end(h);
    return;
  }
  c->launches += 3 + 2 * c->FP.d.lvl_cut;
  SweepRhs sr{};
  sr.rhs = r;
  sr.in_perm = c->perm_ph_dev;
  sr.done_flag = done;
  int h = c->begin(4);
  trsv_forward(c->FP.d, sr, c->xph, c->tgrid, c->stream);
  trsv_backward(c->FP.d, c->xph, done, c->tgrid, c->stream);
  scatter(z, c->xph, c->perm_ph_dev, c->m2, done, c->stream);
  c->end(h);
}

// Opt-in (QPB_DENSE_PHINV = m2 limit, default 0 = off): P_H⁻¹ formed column by column from the fresh
// factor (m2 sweep pairs on unit vectors), so every P_H apply is one symmetric GEMV — one launch instead
// of two latency-bound sweeps, and bit-reproducible.  Off by default: late in the IPM P_H's condition
// number reaches 1e11 (c0) and an explicit inverse is then a measurably different preconditioner from
// the Cholesky solves (c0 PH-KF iteration 16: 64 PCG iterations against the oracle's 72 in every
// variant), unlike F⁻¹, whose conditioning does not depend on D.
int build_phinv(qp_ctx* c) {
  const char* e = std::getenv("QPB_DENSE_PHINV");
  const int64_t lim = e ? std::atoll(e) : 0;
  const int64_t m2 = c->m2;
  c->phinv_ready = false;
  if (m2 > lim || c->sharded) return QP_OK;
  cudaStream_t st = c->stream;
  if (!c->phinv) {
    const int64_t ld = m2 + (m2 & 1), nb = (m2 + 63) / 64;
    c->phinv = c->mem.zeros<double>((size_t)ld * (size_t)m2, st);
    c->pi_unit = c->mem.zeros<double>(m2, st);
    c->pi_ld = ld;
    std::vector<int32_t> ch, rob, cob0, ncob, width(nb);
    std::vector<int64_t> x0(nb);
    for (int64_t I = 0; I < nb; ++I)
      for (int64_t K0 = 0; K0 <= I; K0 += 8) {
        const int64_t rr = std::min<int64_t>(64, m2 - 64 * I);
        const int64_t ncol = std::min<int64_t>(64 * K0 + 512, 64 * I + rr) - 64 * K0;
        ch.push_back((int32_t)I);
        ch.push_back((int32_t)K0);
        rob.push_back((int32_t)I);
        cob0.push_back((int32_t)K0);
        ncob.push_back((int32_t)(std::min<int64_t>(64 * I - 64 * K0, ncol) / 64));
      }
    for (int64_t o = 0; o < nb; ++o) {
      width[o] = (int32_t)std::min<int64_t>(64, m2 - 64 * o);
      x0[o] = 64 * o;
    }
    c->pi_chunks = reinterpret_cast<const int2*>(c->mem.upload(ch, st));
    c->pi_nch = (int64_t)rob.size();
    c->pi_plan = build_symv_plan(c->mem, st, 0, c->pi_nch, rob, cob0, ncob, 0, (int32_t)nb, width, x0);
    cudaStreamSynchronize(st);   // host vectors
  }
  cudaMemsetAsync(c->pi_unit, 0, m2 * 8, st);
  for (int64_t j = 0; j < m2; ++j) {
    if (j > 0) cudaMemsetAsync(c->pi_unit + j - 1, 0, 8, st);
    flat_set_unit(c->pi_unit, j, st);
    ph_apply_dev(c, c->pi_unit, c->phinv + (size_t)j * c->pi_ld, nullptr);
  }
  w_symmetrize_diag(c->phinv, c->pi_ld, m2, st);
  if (int rc = cuda_check(c, "P_H inverse")) return rc;
  c->phinv_ready = true;
  return QP_OK;
}

int ph_refactor(qp_ctx* c, const double* D) {
  double t0 = now_s();
  int h = c->begin(5);
  int rc = numeric_factor(c, c->FP, c->t_val, D, c->perm_ph_dev, "P_H factorization");
  c->end(h);
  if (rc) return rc;
  cudaMemcpyAsync(c->D_ph_last, D, c->m2 * 8, cudaMemcpyDeviceToDevice, c->stream);
  c->ph_valid = true;
  if (int rc2 = build_phinv(c)) return rc2;
  c->t_factor_ph += now_s() - t0;
  c->ph_refactors++;
  return QP_OK;
}

// PCG on K_F(D) x = b from x = 0.  Result in c->px.
int pcg_dev(qp_ctx* c, const double* D, const double* b, double tol, int maxit, int* iters, double* relres,
            bool refactor_ph) {
  cudaStream_t st = c->stream;
  const int prec = c->precond;
  const int64_t m2 = c->m2;
  if (prec == 2 && refactor_ph) {
    int rc = ph_refactor(c, D);
    if (rc) return rc;
  }
  int h = c->begin(3);
  pcg_init(prec, m2, b, D, c->px, c->pr, c->pz, c->pp, c->partial, c->pst, tol, maxit, c->vgrid, st);
  c->end(h);
  c->launches += 1;
  if (c->sharded) {
    if (int rc = c->allreduce(pst_red(c), 2, 0)) return rc;
    finalize(FIN_PCG_INIT, c->pst, c->ist, prec, st);
    c->launches += 1;
  }
  if (prec == 2) {
    ph_apply_dev(c, c->pr, c->pz, &c->pst->done);
    pcg_init_ph(m2, c->pr, c->pz, c->pp, c->partial, c->pst, c->vgrid, st);
    c->launches += 1;
  }
  // P_L / none on one GPU: a5 + a6 as one cooperative kernel (QPB_FUSED_PCG=0 restores k_kf_q,
  // k_pcg_update1, k_pcg_update2 — equal up to the reduction order: they run on the vector grid)
  static const bool fused_env = !(std::getenv("QPB_FUSED_PCG") && std::getenv("QPB_FUSED_PCG")[0] == '0');
  const bool fused = fused_env && prec != 2 && !c->sharded;
  // its grid: whole multiples of the SM count, about two rows of m2 per thread (fewer blocks make the two
  // grid syncs and the per-block partial sums cheaper on small m2), at most the vector-kernel grid
  static const int rows_per_thread = std::getenv("QPB_STEP_RPT") ? std::max(1, std::atoi(std::getenv("QPB_STEP_RPT"))) : 2;
  const int64_t per_wave = (int64_t)c->sm_count * NT_HOST * rows_per_thread;
  const int step_grid = (int)std::min<int64_t>(
      c->vgrid, (int64_t)c->sm_count * std::max<int64_t>(1, (m2 + per_wave - 1) / per_wave));
  // phase D of the fused step prepares the next iteration's u = Cᵀp (flattened forest or pregathered
  // sweeps); the first iteration's comes from the usual kernel
  const int next_rhs = !fused ? 0 : c->dense_w ? 3 : c->FF.d.flat ? 1 : !pregather_on() ? 0 : c->FF.pi.enabled ? 4 : 2;
  if (next_rhs == 3) {
    spmv(c->Ctf, c->pp, c->ubuf, &c->pst->done, c->vgrid, st);
    cudaMemsetAsync(c->xbuf, 0, c->n * 8, st);
    c->launches += 1;
  } else if (next_rhs == 1) {
    SweepRhs r0{};
    r0.ct = c->Ctf;
    r0.p = c->pp;
    r0.done_flag = &c->pst->done;
    flat_rhs(c->FF.d, r0, c->xbuf, c->sm_count, st);
    c->launches += 1;
  } else if (next_rhs == 2 || next_rhs == 4) {
    spmv(c->Ctf, c->pp, c->ubuf, &c->pst->done, c->vgrid, st);
    c->launches += 1;
    if (next_rhs == 4) {   // level products: accumulators zeroed and the root's right-hand side staged
      SweepRhs r0{};
      r0.rhs = c->ubuf;
      r0.done_flag = &c->pst->done;
      pi_init(c->FF.d, c->FF.pi, r0, c->xbuf, c->sm_count, st);
      c->launches += 1;
    }
  }
  auto body = [&]() -> int {
    if (fused) {
      if (int rc = kf_apply_dev(c, D, c->pp, c->pq, true, true, next_rhs != 0)) return rc;
      int hh = c->begin(2);
      const bool ok = pcg_step(c->Cf, c->long_c, c->n_long_c, prec, D, c->pp, c->xbuf, c->pq, c->px, c->pr, c->pz,
                               c->partial, c->pst, step_grid, st, next_rhs, &c->FF.d, &c->Ctf, c->xbuf, c->ubuf);
      c->end(hh);
      c->launches += 1;
      if (ok) return 0;
      cudaGetLastError();
      return fail(c, QP_ECUDA, "cooperative launch of k_pcg_step failed");
    }
    if (int rc = kf_apply_dev(c, D, c->pp, c->pq, true)) return rc;
    int hh = c->begin(3);
    pcg_update1(prec, m2, D, c->pp, c->pq, c->px, c->pr, c->pz, c->partial, c->pst, c->vgrid, st);
    c->end(hh);
    if (c->sharded) {
      if (int rc = c->allreduce(pst_red(c), 2, 0)) return rc;
      finalize(FIN_PCG_UPD1, c->pst, c->ist, prec, st);
      c->launches += 1;
    }
    if (prec == 2) {
      ph_apply_dev(c, c->pr, c->pz, &c->pst->done);
      pcg_rz_ph(m2, c->pr, c->pz, c->partial, c->pst, c->vgrid, st);
    }
    hh = c->begin(3);
    pcg_update2(m2, c->pz, c->pp, c->pst, c->vgrid, st);
    c->end(hh);
    c->launches += prec == 2 ? 3 : 2;
    return 0;
  };
  // CUDA graph of GCH iterations (kernels exit early once the device `done` flag is set); the
  // operands are the context's fixed buffers, so one graph per preconditioner is reused.
  constexpr int GCH = 8;
  const bool graphs = c->use_graphs && !c->prof && D == c->Dk && !c->sharded;
  if (graphs && !c->pcg_graph[prec]) {
    int64_t l0 = c->launches;
    cudaGraph_t g;
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
      for (int k = 0; k < GCH; ++k) body();
      if (cudaStreamEndCapture(st, &g) == cudaSuccess) {
        if (cudaGraphInstantiate(&c->pcg_graph[prec], g, 0) != cudaSuccess) c->pcg_graph[prec] = nullptr;
        cudaGraphDestroy(g);
      }
    }
    cudaGetLastError();
    c->graph_launches[prec] = (int)(c->launches - l0);
    c->launches = l0;
  }
  int chunk = 2;
  for (int it = 0; it < maxit + 1;) {
    if (graphs && c->pcg_graph[prec] && it >= 2) {
      cudaGraphLaunch(c->pcg_graph[prec], st);
      c->launches += c->graph_launches[prec];
      it += GCH;
    } else {
      for (int k = 0; k < chunk; ++k)
        if (int rc = body()) return rc;
      it += chunk;
    }
    cudaMemcpyAsync(c->h_pst, c->pst, sizeof(PcgState), cudaMemcpyDeviceToHost, st);
    int rc = sync_check(c, "pcg");
    if (rc) return rc;
    if (c->h_pst->done) break;
    chunk = std::min(chunk * 2, 32);
  }
  c->harvest();
  if (!c->h_pst->done) return fail(c, QP_ECUDA, "pcg loop ended without completion (internal error)");
  if (iters) *iters = c->h_pst->iter;
  if (relres) *relres = c->h_pst->bnorm2 > 0 ? std::sqrt(c->h_pst->rr / c->h_pst->bnorm2) : 0.0;
  if (c->h_pst->status == -3) return fail(c, QP_EBREAKDOWN, "PCG breakdown (pᵀq <= 0 or non-finite)");
  return c->h_pst->status == 1 ? QP_MAXIT : QP_OK;
}

// x-space twin: projected CG on G Δx − AᵀΔλ = f, AΔx = e (oracle/xspace.py), G = H + CᵀD⁻¹C.
// fe: [f; e] in factor order (N).  Result in c->xs_x (n) and c->xs_lam (m1).
int pcg_x_dev(qp_ctx* c, const double* D, const double* fe, double tol, int maxit, int* iters, double* relres) {
  cudaStream_t st = c->stream;
  const int64_t n = c->n, m1 = c->m1, N = n + m1;
  const int g = c->vgrid;
  int h = c->begin(3);
  recip(c->m2, D, c->xs_W, g, st);
  c->end(h);
  // particular solution A x₀ = e: F [x₀; ·] = [0; e]
  cudaMemsetAsync(c->xs_rhs, 0, N * 8, st);
  if (m1 > 0) {
    cudaMemcpyAsync(c->xs_rhs + n, fe + n, m1 * 8, cudaMemcpyDeviceToDevice, st);
    f_solve_dev(c, c->xs_rhs, c->xbuf);
    cudaMemcpyAsync(c->xs_x, c->xbuf, n * 8, cudaMemcpyDeviceToDevice, st);
    cudaMemsetAsync(c->xs_rhs + n, 0, m1 * 8, st);
  } else {
    cudaMemsetAsync(c->xs_x, 0, n * 8, st);
  }
  // r = G x₀ − f, first projection, ρ₀, p = −g
  g_apply(c->Hf, c->Cf, c->Ctf, c->xs_W, c->xs_x, c->xs_q, c->partial, c->pst, false, g, st);
  xp_init_r(n, c->xs_q, fe, c->xs_r, c->xs_rhs, g, st);
  c->launches += 3;
  {
    PcgState ps{};
    ps.tol2 = tol * tol;
    ps.maxit = maxit;
    *c->h_pst = ps;
    cudaMemcpyAsync(c->pst, c->h_pst, sizeof(PcgState), cudaMemcpyHostToDevice, st);
  }
  if (m1 > 0) cudaMemsetAsync(c->xs_lam, 0, m1 * 8, st);
  f_solve_dev(c, c->xs_rhs, c->xbuf);
  xp_update2(c->Atf, m1, c->xbuf, c->xs_r, c->xs_lam, c->xs_p, c->partial, c->pst, true, g, st);
  c->launches += 1;
  auto body = [&]() {
    SweepRhs r{};
    r.rhs = c->xs_rhs;
    r.done_flag = &c->pst->done;
    int hh = c->begin(2);
    g_apply(c->Hf, c->Cf, c->Ctf, c->xs_W, c->xs_p, c->xs_q, c->partial, c->pst, true, g, st);
    c->end(hh);
    hh = c->begin(3);
    xp_update1(n, c->xs_p, c->xs_q, c->xs_x, c->xs_r, c->xs_rhs, c->pst, g, st);
    c->end(hh);
    f_solve_sweeps(c, r, c->xbuf);
    hh = c->begin(3);
    xp_update2(c->Atf, m1, c->xbuf, c->xs_r, c->xs_lam, c->xs_p, c->partial, c->pst, false, g, st);
    xp_update3(n, c->xbuf, c->xs_p, c->pst, g, st);
    c->end(hh);
    c->launches += 4;
  };
  constexpr int GCH = 8;
  const bool graphs = c->use_graphs && !c->prof;
  if (graphs && !c->pcg_graph[3]) {
    int64_t l0 = c->launches;
    cudaGraph_t gr;
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
      for (int k = 0; k < GCH; ++k) body();
      if (cudaStreamEndCapture(st, &gr) == cudaSuccess) {
        if (cudaGraphInstantiate(&c->pcg_graph[3], gr, 0) != cudaSuccess) c->pcg_graph[3] = nullptr;
        cudaGraphDestroy(gr);
      }
    }
    cudaGetLastError();
    c->graph_launches[3] = (int)(c->launches - l0);
    c->launches = l0;
  }
  int chunk = 2;
  for (int it = 0; it < maxit + 1;) {
    if (graphs && c->pcg_graph[3] && it >= 2) {
      cudaGraphLaunch(c->pcg_graph[3], st);
      c->launches += c->graph_launches[3];
      it += GCH;
    } else {
      for (int k = 0; k < chunk; ++k) body();
      it += chunk;
    }
    cudaMemcpyAsync(c->h_pst, c->pst, sizeof(PcgState), cudaMemcpyDeviceToHost, st);
    int rc = sync_check(c, "pcg_x");
    if (rc) return rc;
    if (c->h_pst->done) break;
    chunk = std::min(chunk * 2, 32);
  }
  c->harvest();
  if (!c->h_pst->done) return fail(c, QP_ECUDA, "projected CG loop ended without completion (internal error)");
  if (iters) *iters = c->h_pst->iter;
  if (relres) *relres = c->h_pst->bnorm2 > 0 ? std::sqrt(c->h_pst->rr / c->h_pst->bnorm2) : 0.0;
  if (c->h_pst->status == -3) return fail(c, QP_EBREAKDOWN, "projected CG breakdown (pᵀGp <= 0 or non-finite)");
  return c->h_pst->status == 1 ? QP_MAXIT : QP_OK;
}

// Ordering (x block by x_perm or minimum degree on the graph of H, λ last) + symbolic analysis of F.
// When the factor ends in a dense root supernode, the top levels of the supernodal tree (an
// ancestor-closed set) are moved next to it — an equivalent reordering with the same fill — so that
// amalgamation absorbs them into the root: fewer dependent levels for the sweeps, at the price of a
// bounded number of explicit zeros (≤ 2 % of the root's entries).
std::string analyse_F(qp_ctx* c) {
  const int64_t n = c->n, m1 = c->m1;
  double t0 = now_s();
  const bool user = !c->xperm_user.empty();
  std::vector<int64_t> ptr(n + 1, 0);
  std::vector<int32_t> idx;
  if (user) {
    c->perm = c->xperm_user;
  } else {
    idx.reserve(c->H.nnz());
    for (int64_t r = 0; r < n; ++r) {
      for (int64_t q = c->H.p[r]; q < c->H.p[r + 1]; ++q)
        if (c->H.i[q] != r) idx.push_back(c->H.i[q]);
      ptr[r + 1] = (int64_t)idx.size();
    }
    c->perm = min_degree_order(n, ptr, idx);
    if (!std::getenv("QPB_NO_POSTORDER")) c->perm = etree_postorder(n, ptr, idx, c->perm);
  }
  int64_t trailing = -1;
  auto run = [&]() {
    c->FF.S = Symbolic();
    LowerMatrix M = build_F_lower(n, m1, c->H.p.data(), c->H.i.data(), c->H.v.data(), c->A.p.data(),
                                  c->A.i.data(), c->A.v.data(), c->perm);
    return analyse(M, c->FF.S, n, true, trailing);
  };
  std::string e = run();
  if (e.empty() && !user && !std::getenv("QPB_NO_ABSORB")) {
    const Symbolic& S = c->FF.S;
    const int64_t ns = S.ns, root = ns - 1;
    const int64_t wr = S.sn_start[ns] - S.sn_start[root];
    const bool dense_root = ns > 1 && S.sn_parent[root] < 0 && wr > BW &&
                            S.sn_rowptr[root + 1] - S.sn_rowptr[root] == wr;
    if (dense_root && S.n_levels > 3) {
      // choose the lowest cut level L (≥ 1) whose absorbed set costs ≤ 2 % of the root's entries
      const double budget = 0.02 * (double)wr * (double)(wr + 1) / 2;
      int64_t best = S.n_levels - 1;
      for (int64_t L = S.n_levels - 2; L >= 1; --L) {
        double zeros = 0;
        int64_t wsum = 0;
        for (int64_t J = 0; J < root; ++J)
          if (S.sn_level[J] >= L) {
            const int64_t w = S.sn_start[J + 1] - S.sn_start[J], m = S.sn_rowptr[J + 1] - S.sn_rowptr[J];
            wsum += w;
            zeros += (double)w * (double)(wr - (m - w));
          }
        zeros += (double)wsum * (double)wsum / 2;
        if (zeros > budget) break;
        best = L;
      }
      if (best < S.n_levels - 1) {
        // new x order: columns of supernodes below the cut, then the absorbed ones, then the root
        std::vector<int64_t> low, high;
        for (int64_t J = 0; J < root; ++J)
          for (int64_t col = S.sn_start[J]; col < S.sn_start[J + 1]; ++col)
            if (col < n) (S.sn_level[J] >= best ? high : low).push_back(c->perm[col]);
        for (int64_t col = S.sn_start[root]; col < n; ++col) high.push_back(c->perm[col]);
        low.insert(low.end(), high.begin(), high.end());
        if (std::getenv("QPB_VERBOSE"))
          std::fprintf(stderr, "qpb: absorbing levels >= %lld into the root (%zu columns moved)\n", (long long)best,
                       high.size());
        if ((int64_t)low.size() == n) {
          trailing = n - (int64_t)high.size();   // first column of the absorbed block
          c->perm = low;
          e = run();
          if (std::getenv("QPB_VERBOSE"))
            std::fprintf(stderr, "qpb: after absorption: %lld supernodes, %lld levels\n", (long long)c->FF.S.ns,
                         (long long)c->FF.S.n_levels);
        }
      }
    }
  }
  c->t_symbolic = now_s() - t0;
  if (e.empty()) c->analysed = true;
  return e;
}

int require(qp_ctx* c, bool factored) {
  if (!c) return QP_EINVAL;
  if (!c->setup_done) return fail(c, QP_ESTATE, "qp_setup has not completed");
  if (factored && !c->factored) return fail(c, QP_ESTATE, "ipm_factor_once has not completed");
  cudaSetDevice(c->device);
  return QP_OK;
}

// Copy m doubles host/device → device buffer (staging) according to vectors_on_device.
const double* in_vec(qp_ctx* c, const double* v, double* stage, int64_t m) {
  if (c->vectors_on_device) return v;
  cudaMemcpyAsync(stage, v, m * 8, cudaMemcpyHostToDevice, c->stream);
  return stage;
}
void out_vec(qp_ctx* c, double* dst, const double* src_dev, int64_t m) {
  if (!dst) return;
  cudaMemcpyAsync(dst, src_dev, m * 8, c->vectors_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                  c->stream);
}

// μ and the residuals (a9) at the current iterate; sharded: Cᵀν and the reductions all-reduced.
int ipm_eval_residuals(qp_ctx* c) {
  cudaStream_t st = c->stream;
  const int64_t n = c->n;
  int h = c->begin(6);
  ipm_mu(c->m2, c->s, c->nu, c->partial, c->ist, c->vgrid, st);
  c->launches += 2;
  const double* ctnu = nullptr;
  if (c->sharded) {
    if (int rc = c->allreduce(ist_red(c), 1, 0)) return rc;
    finalize(FIN_IPM_MU, c->pst, c->ist, c->precond, st);
    spmv(c->Ctf, c->nu, c->ubuf, nullptr, c->vgrid, st);
    if (int rc = c->allreduce(c->ubuf, n, 0)) return rc;
    ctnu = c->ubuf;
    c->launches += 2;
  }
  ipm_residuals(c->Hf, c->Atf, c->Ctf, c->Af, c->Cf, c->gf, c->bv, c->dv, c->xl, c->xl + n, c->nu, c->s, c->rgre,
                c->rc, c->ra, c->Dk, c->partial, c->ist, c->vgrid, st, ctnu);
  if (c->sharded) {
    if (int rc = c->allreduce(ist_red(c), 3, 1)) return rc;
    finalize(FIN_IPM_RESID, c->pst, c->ist, c->precond, st);
    c->launches += 1;
  }
  c->end(h);
  return 0;
}

int ipm_iteration(qp_ctx* c, bool* converged) {
  cudaStream_t st = c->stream;
  const int64_t n = c->n, m1 = c->m1, m2 = c->m2, N = n + m1;
  int h;
  if (int rc0 = ipm_eval_residuals(c)) return rc0;
  cudaMemcpyAsync(c->h_ist, c->ist, sizeof(IpmState), cudaMemcpyDeviceToHost, st);
  int rc = sync_check(c, "ipm residuals");
  if (rc) return rc;
  const IpmState& S = *c->h_ist;
  const double tol = c->opts.ipm_tol;
  if (S.rg_inf <= tol * (1 + c->gmax) && S.re_inf <= tol * (1 + c->bmax) && S.ri_inf <= tol * (1 + c->dmax) &&
      S.mu <= tol) {
    *converged = true;
    return QP_OK;
  }
  *converged = false;
  double eps_x = c->opts.pcg_forcing ? std::min(c->opts.pcg_tol, S.mu) : c->opts.pcg_tol;
  if (c->opts.space == 1) {
    // x-space twin: [f; e] = [r_g − CᵀD⁻¹r_a; −r_e] → projected CG → Δν = −D⁻¹(r_a + CΔx)
    c->last_eps = eps_x;
    h = c->begin(7);
    x_rhs(c->Ctf, m1, c->rgre, c->ra, c->Dk, c->rhs2, c->vgrid, st);
    c->end(h);
    int itx = 0;
    rc = pcg_x_dev(c, c->Dk, c->rhs2, eps_x, c->opts.pcg_maxit, &itx, nullptr);
    if (rc != QP_OK && rc != QP_MAXIT) return rc;
    c->pcg_hist.push_back(itx);
    h = c->begin(7);
    cudaMemcpyAsync(c->dxl, c->xs_x, n * 8, cudaMemcpyDeviceToDevice, st);
    if (m1 > 0) cudaMemcpyAsync(c->dxl + n, c->xs_lam, m1 * 8, cudaMemcpyDeviceToDevice, st);
    x_dnu(c->Cf, c->ra, c->Dk, c->xs_x, c->px, c->vgrid, st);
    ipm_ds_alpha(m2, c->rc, c->nu, c->Dk, c->px, c->s, c->ds, c->partial, c->ist, c->vgrid, st);
    ipm_update(N, m2, c->dxl, c->px, c->ds, c->xl, c->nu, c->s, c->ist, c->vgrid, st);
    c->end(h);
    c->launches += 5;
    c->ipm_k++;
    return cuda_check(c, "ipm iteration (x-space)");
  }
  // r_ν = −r_a + [C 0] F⁻¹ (r_g; r_e)
  f_solve_dev(c, c->rgre, c->xbuf);
  h = c->begin(7);
  ipm_rnu(c->Cf, c->ra, c->xbuf, c->rnu, c->vgrid, st);
  c->end(h);
  // PCG (reading R4 forcing)
  double eps = c->opts.pcg_forcing ? std::min(c->opts.pcg_tol, S.mu) : c->opts.pcg_tol;
  c->last_eps = eps;
  c->launches += 1 + 1 + 2;   // r_nu, recovery rhs, ds/alpha + update
  int iters = 0;
  rc = pcg_dev(c, c->Dk, c->rnu, eps, c->opts.pcg_maxit, &iters, nullptr, true);
  if (rc != QP_OK && rc != QP_MAXIT) return rc;
  c->pcg_hist.push_back(iters);
  // recovery: F(Δx;Δλ) = −(r_g + CᵀΔν; r_e)
  h = c->begin(7);
  const double* ctdnu = nullptr;
  if (c->sharded) {
    spmv(c->Ctf, c->px, c->ubuf, nullptr, c->vgrid, st);
    if ((rc = c->allreduce(c->ubuf, n, 0))) return rc;
    ctdnu = c->ubuf;
    c->launches += 1;
  }
  ipm_recovery_rhs(c->Ctf, n, m1, c->rgre, c->px, c->rhs2, c->vgrid, st, ctdnu);
  c->end(h);
  f_solve_dev(c, c->rhs2, c->dxl);
  h = c->begin(7);
  ipm_ds_alpha(m2, c->rc, c->nu, c->Dk, c->px, c->s, c->ds, c->partial, c->ist, c->vgrid, st);
  if (c->sharded) {
    if ((rc = c->allreduce(ist_red(c), 1, 2))) return rc;
    finalize(FIN_IPM_ALPHA, c->pst, c->ist, c->precond, st);
    c->launches += 1;
  }
  ipm_update(N, m2, c->dxl, c->px, c->ds, c->xl, c->nu, c->s, c->ist, c->vgrid, st);
  c->end(h);
  c->ipm_k++;
  return cuda_check(c, "ipm iteration");
}

void fill_result(qp_ctx* c, qp_ipm_result* r) {
  if (!r) return;
  cudaStream_t st = c->stream;
  const int64_t n = c->n;
  ipm_objective(c->Hf, c->gf, c->xl, c->partial, c->ist, c->vgrid, st);
  cudaMemcpyAsync(c->h_ist, c->ist, sizeof(IpmState), cudaMemcpyDeviceToHost, st);
  if (r->x) {
    scatter(c->vout, c->xl, c->perm_dev, n, nullptr, st);  // x[perm[i]] = x_f[i]
    out_vec(c, r->x, c->vout, n);
  }
  out_vec(c, r->lam, c->xl + n, c->m1);
  out_vec(c, r->nu, c->nu, c->m2);
  out_vec(c, r->s, c->s, c->m2);
  cudaStreamSynchronize(st);
  r->objective = c->h_ist->objective;
  r->n_ipm = c->ipm_k;
  r->status = c->ipm_converged ? QP_OK : QP_MAXIT;
  int64_t tot = 0;
  for (size_t i = 0; i < c->pcg_hist.size(); ++i) {
    if (r->pcg_iters && (int32_t)i < c->opts.max_ipm) r->pcg_iters[i] = c->pcg_hist[i];
    tot += c->pcg_hist[i];
  }
  r->pcg_total = (int32_t)tot;
  r->t_setup_s = c->t_symbolic + c->t_factor;
  r->mu = c->h_ist->mu;
  r->rg_inf = c->h_ist->rg_inf;
  r->re_inf = c->h_ist->re_inf;
  r->ri_inf = c->h_ist->ri_inf;
  r->alpha = c->h_ist->alpha;
}

}  // namespace

// ============================================================================ C ABI
extern "C" {

int qp_analyse(qp_ctx** out, const qp_csr* H, const qp_csr* A, const int64_t* x_perm) {
  if (!out || !H || !A) return QP_EINVAL;
  std::unique_ptr<qp_ctx> c(new qp_ctx());
  const int64_t n = H->nrows, m1 = A->nrows;
  std::string e = n > 0 && m1 >= 0 && m1 <= n ? "" : "need n >= 1 and 0 <= m1 <= n";
  if (e.empty()) e = check_csr(H, n, n, "H", c->H);
  if (e.empty()) e = check_csr(A, m1, n, "A", c->A);
  c->n = n;
  c->m1 = m1;
  if (e.empty() && x_perm) c->xperm_user.assign(x_perm, x_perm + n);
  if (e.empty()) e = analyse_F(c.get());
  *out = c.release();
  return e.empty() ? QP_OK : fail(*out, QP_EINVAL, e);
}

int qp_setup(qp_ctx** out, const qp_csr* H, const qp_csr* A, const qp_csr* C, const double* g, const double* b,
             const double* d, const qp_setup_opts* opts) {
  if (!out) return QP_EINVAL;
  *out = nullptr;
  std::unique_ptr<qp_ctx> c(new qp_ctx());
  if (!H || !A || !C) return QP_EINVAL;
  const int64_t n = H->nrows, m1 = A->nrows, m2 = C->nrows;
  if (n <= 0 || m2 <= 0 || m1 < 0 || m1 > n) {
    *out = c.release();
    return fail(*out, QP_EINVAL, "need n >= 1, m2 >= 1, 0 <= m1 <= n");
  }
  std::string e = check_csr(H, n, n, "H", c->H);
  if (e.empty()) e = check_csr(A, m1, n, "A", c->A);
  if (e.empty()) e = check_csr(C, m2, n, "C", c->C);
  if (e.empty()) {
    // H symmetric (both triangles stored)
    HostCSR Ht = transpose(c->H);
    if (Ht.p != c->H.p || Ht.i != c->H.i) e = "H pattern is not symmetric (store both triangles)";
    else
      for (int64_t q = 0; q < c->H.nnz() && e.empty(); ++q)
        if (Ht.v[q] != c->H.v[q]) e = "H values are not symmetric";
  }
  c->n = n;
  c->m1 = m1;
  c->m2 = m2;
  if (e.empty() && (!g || (m1 > 0 && !b) || !d)) e = "NULL g / b / d";
  if (e.empty()) {
    c->g.assign(g, g + n);
    c->b.assign(b ? b : g, (b ? b : g) + m1);
    c->d.assign(d, d + m2);
    for (double v : c->g) if (!std::isfinite(v)) e = "non-finite g";
    for (double v : c->b) if (!std::isfinite(v)) e = "non-finite b";
    for (double v : c->d) if (!std::isfinite(v)) e = "non-finite d";
  }
  if (!e.empty()) {
    *out = c.release();
    return fail(*out, QP_EINVAL, e);
  }
  qp_setup_opts o{};
  if (opts) o = *opts;
  c->device = o.device;
  c->vectors_on_device = o.vectors_on_device;
  c->rank = o.rank;
  c->world = o.world <= 0 ? 1 : o.world;
  c->ws_limit = o.workspace_limit_bytes > 0 ? o.workspace_limit_bytes : (int64_t)120 << 30;
  c->sharded = c->world > 1 || o.allreduce != nullptr || o.nccl_uid != nullptr;
  c->m2_global = m2;
  c->row0 = 0;
  c->row1 = m2;
  if (c->sharded) {
    if (c->rank < 0 || c->rank >= c->world || m2 < c->world) {
      *out = c.release();
      return fail(*out, QP_EINVAL, "sharded setup needs 0 <= rank < world <= m2");
    }
    if (!o.allreduce && !o.nccl_uid) {
      *out = c.release();
      return fail(*out, QP_EINVAL, "world > 1 needs opts.nccl_uid (qp_nccl_unique_id) or opts.allreduce");
    }
    std::vector<int64_t> bounds(c->world + 1);
    partition_rows(c->C.p.data(), m2, c->world, bounds.data());
    c->row0 = bounds[c->rank];
    c->row1 = bounds[c->rank + 1];
    // keep only this rank's rows of C and d (global |d|max first: the stopping test is global)
    c->dmax = 0;
    for (double v : c->d) c->dmax = std::max(c->dmax, std::fabs(v));
    HostCSR Cl;
    Cl.nrows = c->row1 - c->row0;
    Cl.ncols = n;
    const int64_t q0 = c->C.p[c->row0], q1 = c->C.p[c->row1];
    Cl.p.resize(Cl.nrows + 1);
    for (int64_t i = 0; i <= Cl.nrows; ++i) Cl.p[i] = c->C.p[c->row0 + i] - q0;
    Cl.i.assign(c->C.i.begin() + q0, c->C.i.begin() + q1);
    Cl.v.assign(c->C.v.begin() + q0, c->C.v.begin() + q1);
    c->C = std::move(Cl);
    c->d = std::vector<double>(c->d.begin() + c->row0, c->d.begin() + c->row1);
    c->m2 = c->row1 - c->row0;
  }
  if (o.x_perm) {
    c->xperm_user.assign(o.x_perm, o.x_perm + n);
    std::vector<char> seen(n, 0);
    for (int64_t v : c->xperm_user) {
      if (v < 0 || v >= n || seen[v]) {
        *out = c.release();
        return fail(*out, QP_EINVAL, "x_perm is not a permutation of 0..n-1");
      }
      seen[v] = 1;
    }
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= c->device) {
    cudaGetLastError();
    *out = c.release();
    return fail(*out, QP_ECUDA, "no CUDA device available (this library has no CPU fallback)");
  }
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, c->device);
  if (prop.major < 10) {
    *out = c.release();
    return fail(*out, QP_ECUDA, "device is not sm_100 class (Blackwell) — the kernels are built for sm_100a only");
  }
  cudaSetDevice(c->device);
  c->sm_count = prop.multiProcessorCount;
  c->vgrid = c->sm_count * 4;
  if (o.stream) {
    c->stream = (cudaStream_t)o.stream;
  } else {
    cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    c->own_stream = true;
  }
  c->tgrid = trsv_grid(c->device);
  c->use_graphs = std::getenv("QPB_NO_GRAPH") == nullptr;
  if (std::getenv("QPB_VERBOSE")) std::fprintf(stderr, "qpb: trsv grid %d CTAs on %d SMs\n", c->tgrid, c->sm_count);
  cudaMallocHost(&c->h_pst, sizeof(PcgState));
  cudaMallocHost(&c->h_ist, sizeof(IpmState));
  c->gmax = 0;
  for (double v : c->g) c->gmax = std::max(c->gmax, std::fabs(v));
  c->bmax = 0;
  for (double v : c->b) c->bmax = std::max(c->bmax, std::fabs(v));
  if (!c->sharded) {
    c->dmax = 0;
    for (double v : c->d) c->dmax = std::max(c->dmax, std::fabs(v));
  }
  if (c->sharded) {
    c->use_graphs = false;   // host-side collectives between the PCG kernels
    if (!o.allreduce) {
      NcclApi& api = nccl_api();
      if (!api.ok) {
        *out = c.release();
        return fail(*out, QP_ENCCL, api.err);
      }
      ncclUniqueId uid;
      std::memcpy(&uid, o.nccl_uid, sizeof(uid));
      ncclResult_t r = api.comm_init_rank(&c->nccl, c->world, uid, c->rank);
      if (r != ncclSuccess) {
        *out = c.release();
        return fail(*out, QP_ENCCL, std::string("ncclCommInitRank: ") + api.error_string(r));
      }
    } else {
      c->ar_fn = o.allreduce;
      c->ar_user = o.allreduce_user;
    }
    c->halo_fn = o.halo;
    c->halo_user = o.halo_user;
  }
  int rc = cuda_check(c.get(), "qp_setup");
  c->setup_done = rc == QP_OK;
  *out = c.release();
  return rc;
}

// Level products: plan and build Z_J = [X_J; L_ext,J X_J] for every supernode of F between the
// leaf phase and the symmetric root, level by level (tiles of ≤ 512 rows × ≤ 64 columns, larger first).
// Leaves F.pi.enabled = 0; the caller enables it after the accuracy guard.
int build_pi(qp_ctx* c, bool allow_subtrees = true) {
  Factor& F = c->FF;
  const Symbolic& S = F.S;
  const int64_t ns = S.ns, Jr = ns - 1;
  F.pi = PiSweep{};
  const int64_t min_n = std::getenv("QPB_PI_MINN") ? std::atoll(std::getenv("QPB_PI_MINN")) : 4096;   // tests: 0
  if (Jr < 1 || S.sn_sinv[Jr] < 0 || F.n_sym != 1 || S.N <= min_n) return QP_OK;
  // ---- subtrees below the level products (kernels.cuh StHdr): maximal subtrees of single-block supernodes of
  // ≤ 32 columns whose entries fit QPB_ST_KB (default 96 KB) and whose frame fits ST_FRAME
  std::vector<char> in_st(ns, 0);
  std::vector<StHdr> hdr;
  std::vector<int32_t> sdesc, slptr, sloc;
  int st_g = 16;
  {
    const char* se = std::getenv("QPB_ST");
    const int64_t budget = (std::getenv("QPB_ST_KB") ? std::atoll(std::getenv("QPB_ST_KB")) : 96) * 128;   // doubles
    std::vector<int64_t> sub(ns, 0), cols(ns, 0), cnt(ns, 0);
    std::vector<char> ok(ns, 1), fits(ns, 0);
    bool post = true;
    for (int64_t J = 0; J < ns && post; ++J) post = S.sn_parent[J] < 0 || S.sn_parent[J] > J;
    for (int64_t J = 0; post && allow_subtrees && !(se && se[0] == '0') && J < ns; ++J) {
      const int64_t w = S.sn_start[J + 1] - S.sn_start[J], m = S.sn_rowptr[J + 1] - S.sn_rowptr[J], noff = m - w;
      const bool elig = J != Jr && S.sn_blk0[J + 1] - S.sn_blk0[J] == 1 && w <= 32 && S.sn_xinv[J] < 0 &&
                        noff < (int64_t(1) << 25);
      sub[J] += w * w + noff * w;
      cols[J] += w;
      cnt[J] += 1;
      ok[J] = ok[J] && elig;
      bool f = ok[J] && sub[J] <= budget && cols[J] + noff <= ST_FRAME && S.sn_level[J] < 30 && cnt[J] <= J + 1 &&
               cnt[J] <= ST_MAXSN;
      if (f) {   // the subtree's supernodes and columns are the contiguous ranges ending at J (postorder)
        const int64_t K0 = J - cnt[J] + 1;
        f = S.sn_start[J + 1] - cols[J] == S.sn_start[K0];
        for (int64_t K = K0; f && K < J; ++K) f = S.sn_parent[K] > K && S.sn_parent[K] <= J;
      }
      fits[J] = f;
      const int64_t p = S.sn_parent[J];
      if (p >= 0) {
        sub[p] += sub[J];
        cols[p] += cols[J];
        cnt[p] += cnt[J];
        if (!ok[J]) ok[p] = 0;
      }
    }
    std::vector<int32_t> roots;
    for (int64_t J = 0; J < ns; ++J)
      if (fits[J] && (S.sn_parent[J] < 0 || !fits[S.sn_parent[J]])) roots.push_back((int32_t)J);
    const int64_t st_min = std::getenv("QPB_ST_MIN") ? std::atoll(std::getenv("QPB_ST_MIN")) : 64;
    if ((int64_t)roots.size() < st_min) roots.clear();   // too few to fill the GPU: keep the leaf phase
    std::stable_sort(roots.begin(), roots.end(), [&](int32_t a, int32_t b) { return sub[a] > sub[b]; });
    for (int32_t Jt : roots) {
      const int64_t K0 = Jt - cnt[Jt] + 1;
      const int64_t c_lo = S.sn_start[K0], c_hi = S.sn_start[Jt + 1];
      const int64_t wt = S.sn_start[Jt + 1] - S.sn_start[Jt];
      const int32_t* rr = S.sn_rows.data() + S.sn_rowptr[Jt] + wt;
      const int64_t next = S.sn_rowptr[Jt + 1] - S.sn_rowptr[Jt] - wt;
      std::vector<int32_t> mem;
      for (int64_t K = K0; K <= Jt; ++K) mem.push_back((int32_t)K);
      std::stable_sort(mem.begin(), mem.end(), [&](int32_t a, int32_t b) { return S.sn_level[a] < S.sn_level[b]; });
      StHdr h{};
      h.d0 = (int32_t)(sdesc.size() / 8);
      h.nlev = (int32_t)S.sn_level[Jt] + 1;
      h.c_lo = (int32_t)c_lo;
      h.ncols = (int32_t)(c_hi - c_lo);
      h.next = (int32_t)next;
      h.lptr = (int32_t)slptr.size();
      h.rootrows = S.sn_rowptr[Jt] + wt;
      h.fslo = S.blk_inv[S.sn_blk0[K0]];
      h.fslen = (int32_t)(S.blk_off[S.sn_blk0[Jt]] + next * wt - h.fslo);
      size_t q = 0;
      for (int32_t l = 0; l <= h.nlev; ++l) {
        while (l < h.nlev && q < mem.size() && S.sn_level[mem[q]] < l) ++q;
        slptr.push_back(l < h.nlev ? (int32_t)q : (int32_t)mem.size());
      }
      for (int32_t K : mem) {
        in_st[K] = 1;
        const int64_t w = S.sn_start[K + 1] - S.sn_start[K], m = S.sn_rowptr[K + 1] - S.sn_rowptr[K], noff = m - w;
        if (w > 16) st_g = 32;
        const int32_t b = S.sn_blk0[K];
        const int64_t lo = S.blk_off[b], io = S.blk_inv[b], ro = (int64_t)sloc.size();
        for (int64_t e = 0; e < noff; ++e) {
          const int32_t g = S.sn_rows[S.sn_rowptr[K] + w + e];
          if (g < c_hi) {
            sloc.push_back((int32_t)(g - c_lo));
          } else {
            const int32_t* it = std::lower_bound(rr, rr + next, g);
            if (it == rr + next || *it != g) return fail(c, QP_EINVAL, "subtree plan: row outside the root's row list");
            sloc.push_back((int32_t)(h.ncols + (it - rr)));
          }
        }
        sdesc.insert(sdesc.end(), {(int32_t)(uint32_t)(lo & 0xffffffffll), (int32_t)(lo >> 32),
                                   (int32_t)(uint32_t)(io & 0xffffffffll), (int32_t)(io >> 32),
                                   (int32_t)(uint32_t)(ro & 0xffffffffll), (int32_t)(ro >> 32), (int32_t)S.sn_start[K],
                                   (int32_t)(w | (noff << 6))});
      }
      hdr.push_back(h);
    }
  }
  const bool use_st = !hdr.empty();
  const int lcut = use_st ? 0 : F.d.lvl_cut;
  auto in_pi = [&](int64_t J) { return J < Jr && (use_st ? !in_st[J] : S.sn_level[J] >= lcut); };
  int64_t top = -1;
  for (int64_t J = 0; J < Jr; ++J)
    if (in_pi(J)) top = std::max<int64_t>(top, S.sn_level[J]);
  if (top < lcut || top - lcut + 1 > PI_MAXLEV) return QP_OK;
  const int nlev = (int)(top - lcut + 1);
  std::vector<std::vector<int32_t>> by(nlev);
  for (int64_t J = 0; J < Jr; ++J)
    if (in_pi(J)) by[S.sn_level[J] - lcut].push_back((int32_t)J);
  std::vector<int64_t> zoffJ(ns, -1);
  std::vector<PiTile> tiles;
  std::vector<int32_t> tile_J;
  int64_t zs = 0;
  F.pi.lev_ptr[0] = 0;
  // Tile shapes: a supernode with ≤ `short` rows is cut into strips of 64 rows (a warp each, 8 per CTA); taller
  // ones into CTA tiles of 512 rows × 64 columns.  The backward product takes strips up to 640 rows (a CTA
  // tile there first gathers its 512 inputs, then streams), the forward product up to 320 (measured on c2).
  const int64_t short_f = std::getenv("QPB_PI_SHORT") ? std::atoll(std::getenv("QPB_PI_SHORT")) : 320;
  const int64_t short_b = std::getenv("QPB_PI_SHORT_B") ? std::atoll(std::getenv("QPB_PI_SHORT_B")) : 640;
  // CTA-tile width: 64 columns, halved (to ≥ 16) while a level has fewer than 2 CTA tiles per SM: a lone CTA
  // keeps only 32 KB in flight, so a level of one or two wide supernodes (the top of the tree) is bound by
  // per-CTA memory parallelism, not bandwidth (c4s: 13 → 7 µs per top level, 0.59 → 0.49 ms per PCG
  // iteration; c2's levels 18–19 11.7 → 9.4 µs forward, 18.8 → 13.5 µs backward).  Levels that already fill
  // the GPU get slower with narrower tiles (every tile re-gathers its inputs).  QPB_PI_NC forces a width.
  const int64_t nc_force = std::getenv("QPB_PI_NC") ? std::max<int64_t>(16, std::min<int64_t>(64, std::atoll(std::getenv("QPB_PI_NC")))) : 0;
  std::vector<PiTile> btiles;
  bool too_big = false;
  auto plan = [&](int64_t pi_short, std::vector<PiTile>& out, std::vector<int32_t>* outJ, int64_t* ptr, int64_t* sptr,
                  bool set_z) {
    int64_t z = 0;
    ptr[0] = 0;
    for (int L = 0; L < nlev; ++L) {
      std::vector<std::pair<PiTile, int32_t>> lt, ls;
      int64_t ncw = nc_force > 0 ? nc_force : 64;
      for (; nc_force == 0 && ncw > 16; ncw /= 2) {
        int64_t nt = 0;
        for (int32_t J : by[L]) {
          const int64_t w = S.sn_start[J + 1] - S.sn_start[J], m = S.sn_rowptr[J + 1] - S.sn_rowptr[J];
          if (m <= pi_short) continue;
          for (int64_t c0 = 0; c0 < w; c0 += ncw) nt += (m - (c0 & ~int64_t(63)) + 511) / 512;
        }
        if (nt == 0 || nt >= 2 * (int64_t)c->sm_count) break;
      }
      for (int32_t J : by[L]) {
        const int64_t w = S.sn_start[J + 1] - S.sn_start[J], m = S.sn_rowptr[J + 1] - S.sn_rowptr[J];
        const int64_t ld = (m + 1) & ~int64_t(1);
        if (ld > INT32_MAX) too_big = true;
        if (set_z) zoffJ[J] = z;
        const bool strip = m <= pi_short;
        const int64_t cw = strip ? 64 : ncw, rh = strip ? 64 : 512;
        for (int64_t c0 = 0; c0 < w; c0 += cw) {
          const int64_t nc = std::min<int64_t>(cw, w - c0);
          for (int64_t r0 = c0 & ~int64_t(63); r0 < m; r0 += rh) {   // rows above the diagonal block are zero
            const int64_t nr = std::min<int64_t>(rh, m - r0);
            PiTile t{};
            t.zoff = z + r0 + c0 * ld;
            t.roff = S.sn_rowptr[J] + r0;
            t.ld = (int32_t)ld;
            t.col0 = (int32_t)(S.sn_start[J] + c0);
            t.nr = (int16_t)nr;
            t.nc = (int16_t)nc;
            t.wx = (int16_t)std::max<int64_t>(0, std::min<int64_t>(nr, w - r0));
            (strip ? ls : lt).push_back({t, J});
          }
        }
        z += ld * w;
      }
      auto bigger = [](const std::pair<PiTile, int32_t>& a, const std::pair<PiTile, int32_t>& b) {
        return (int)a.first.nr * a.first.nc > (int)b.first.nr * b.first.nc;
      };
      std::stable_sort(lt.begin(), lt.end(), bigger);
      std::stable_sort(ls.begin(), ls.end(), bigger);
      for (auto& q : lt) {
        out.push_back(q.first);
        if (outJ) outJ->push_back(q.second);
      }
      sptr[L] = (int64_t)out.size();
      for (auto& q : ls) {
        out.push_back(q.first);
        if (outJ) outJ->push_back(q.second);
      }
      ptr[L + 1] = (int64_t)out.size();
    }
    return z;
  };
  zs = plan(short_f, tiles, &tile_J, F.pi.lev_ptr, F.pi.lev_sptr, true);
  plan(short_b, btiles, nullptr, F.pi.blev_ptr, F.pi.blev_sptr, false);
  if (too_big) {
    F.pi = PiSweep{};
    return QP_OK;
  }
  // before the wait: 2 (default) = the lines of each thread's first batch of loads and whole strips into L2 (c4s 0.489 -> 0.472 ms,
  // c2 0.898 -> 0.896 ms); 1 = the whole CTA tile (c2 0.917 -> 0.981 ms: it floods L2 ahead of the streaming loads); 0 = none
  F.pi.prefetch = std::getenv("QPB_PI_PF") ? std::atoi(std::getenv("QPB_PI_PF")) : 2;
  if (tiles.empty()) return QP_OK;
  cudaStream_t st = c->stream;
  int64_t* zoff_dev = nullptr;
  try {
    F.pi.Z = F.mem.alloc<double>((size_t)zs);
    F.pi.tiles = F.mem.upload(tiles, st);
    F.pi.tile_J = F.mem.upload(tile_J, st);
    F.pi.btiles = F.mem.upload(btiles, st);
    zoff_dev = F.mem.upload(zoffJ, st);
    if (use_st) {
      F.pi.st_hdr = F.mem.upload(hdr, st);
      F.pi.st_desc = reinterpret_cast<const int4*>(F.mem.upload(sdesc, st));
      F.pi.st_lptr = F.mem.upload(slptr, st);
      F.pi.st_loc = F.mem.upload(sloc, st);
      F.pi.st_n = (int64_t)hdr.size();
      F.pi.st_g = st_g;
    }
  } catch (std::bad_alloc&) {
    cudaGetLastError();
    F.pi = PiSweep{};
    return QP_OK;   // not enough memory for Z: keep the sweeps
  }
  F.pi.nlev = nlev;
  F.pi.z_size = zs;
  F.pi.root0 = S.sn_start[Jr];
  if (!F.d.flat) F.d.fl_rc0 = F.pi.root0;   // the fused PCG step's phase D (next_rhs = 4) stages vbuf from here
  pi_build(F.d, F.pi, zoff_dev, st);
  int rc = sync_check(c, "level-product build");   // host vectors
  if (std::getenv("QPB_VERBOSE"))
    std::fprintf(stderr, "qpb: level products: %d levels above %s (%d / %zu), %zu tiles, Z %.1f MB\n", nlev,
                 use_st ? "the subtrees" : "the leaf levels", lcut, hdr.size(), tiles.size(), zs * 8e-6);
  return rc;
}

// Sharded mode: turn a per-rank yes/no into one decision shared by every rank (min over ranks of 0/1),
// through the same collective the PCG uses.  Uses xbuf[0] as device scratch (free at setup).
static int agree_all(qp_ctx* c, bool& ok) {
  double v = ok ? 1.0 : 0.0;
  cudaMemcpyAsync(c->xbuf, &v, 8, cudaMemcpyHostToDevice, c->stream);
  if (int rc = c->allreduce(c->xbuf, 1, 2)) return rc;
  cudaMemcpyAsync(&v, c->xbuf, 8, cudaMemcpyDeviceToHost, c->stream);
  if (int rc = sync_check(c, "rank agreement")) return rc;
  ok = v > 0.5;
  return QP_OK;
}

// Explicit x-block of F⁻¹ (DESIGN §5 "dense W"): W = (F⁻¹)₁₁ = −H⁻¹ + H⁻¹Aᵀ(AH⁻¹Aᵀ)⁻¹AH⁻¹ (n × n, factor
// order, the block form of P:L757–787), so that the K_F product inside PCG is w = W·Cᵀp, one symmetric
// GEMV reading 8·n(n+1)/2 bytes.  Used when that is fewer bytes than one F-solve (c0, c1) and W fits the
// budget; built column by column from F-solves on unit vectors, then checked against an F-solve on a
// random right-hand side (≤ 1e-10 relative) before it is used.  QPB_DENSE_W=0 disables it, =2 forces it
// whenever it fits (tests).
int build_dense_w(qp_ctx* c) {
  if (c->dense_w) return QP_OK;
  const char* e = std::getenv("QPB_DENSE_W");
  if (e && e[0] == '0') return QP_OK;
  qp_stats s{};
  qp_get_stats(c, &s);
  const int64_t n = c->n, N = c->n + c->m1;
  // Small problems (N ≤ QPB_DENSE_FINV, default 4 096): the whole F⁻¹ is formed (N F-solves on unit
  // vectors) and every F-solve becomes one symmetric GEMV; W = (F⁻¹)₁₁ is its top-left block.  At this
  // size the sweeps are latency-bound (tens of µs through a few dependency levels) while the GEMV is one
  // launch, and the GEMV's fixed-order reduction makes every F-solve and K_F product bit-reproducible.
  const char* ef = std::getenv("QPB_DENSE_FINV");
  const int64_t finv_max = ef ? std::atoll(ef) : 4096;
  const bool small = N <= finv_max && N >= 1;
  const int64_t ld = small ? N + (N & 1) : n + (n & 1);
  const double wbytes = 8.0 * (double)n * (double)(n + 1) / 2.0;
  const bool force = e && e[0] == '2';   // QPB_DENSE_W=2: whenever it fits (tests)
  if (!small && (n < 64 || !(force || wbytes < s.fsolve_bytes_F) || 8.0 * (double)ld * (double)n > 16e9))
    return QP_OK;
  cudaStream_t st = c->stream;
  double* W = nullptr;
  try {
    W = c->mem.zeros<double>((size_t)ld * (size_t)(small ? N : n), st);
  } catch (std::bad_alloc&) {
    cudaGetLastError();
    W = nullptr;    // no room: keep the F-solve path (sharded: every rank must agree, below)
  }
  if (c->sharded && c->world > 1) {
    // The two K_F paths issue different collectives (W: all-reduce of u and of w; F-solve: of u only),
    // so all ranks must take the same one: agree on the allocation first (min over ranks).
    bool ok = W != nullptr;
    if (int rc = agree_all(c, ok)) return rc;
    if (!ok) {
      if (W) c->mem.free_ptr(W);
      return QP_OK;
    }
  } else if (!W) {
    return QP_OK;
  }
  // Flattened forest with a symmetric root J0 = columns [r0, N): for a root column j the F-solve is
  // x2 = S⁻¹e_j, so W's root block is S⁻¹'s x-part, copied from its lower storage; only the forest
  // columns [0, r0) need F-solves (c1: 3 761 instead of 20 000).  The diagonal 64-blocks (the GEMV reads
  // them full) are then completed from their lower triangles.
  const Symbolic& S = c->FF.S;
  const int64_t J0 = S.ns - 1;
  const bool fast = !small && c->FF.d.flat && c->FF.sym_enabled && J0 >= 0 && S.sn_sinv[J0] >= 0 &&
                    S.sn_start[J0] == c->FF.d.fl_rc0 && S.sn_start[J0 + 1] == N && S.sn_start[J0] < n;
  const int64_t r0 = small ? N : fast ? S.sn_start[J0] : n;
  const int64_t rows = small ? N : n;   // entries kept per column
  cudaMemsetAsync(c->rhs2, 0, N * 8, st);
  for (int64_t j = 0; j < r0; ++j) {
    if (j > 0) cudaMemsetAsync(c->rhs2 + j - 1, 0, 8, st);
    flat_set_unit(c->rhs2, j, st);
    f_solve_dev(c, c->rhs2, c->xbuf);
    cudaMemcpyAsync(W + (size_t)j * ld, c->xbuf, rows * 8, cudaMemcpyDeviceToDevice, st);
  }
  cudaMemsetAsync(c->rhs2, 0, N * 8, st);
  if (fast) w_copy_root(c->FF.d.xinv + S.sn_sinv[J0], S.sn_ldx[J0], W, ld, r0, n, st);
  w_symmetrize_diag(W, ld, small ? N : n, st);   // the GEMV reads the diagonal 64-blocks full
  if (int rc = cuda_check(c, "dense W columns")) return rc;
  if (small) {   // the whole F⁻¹: its own chunk list and plan over N, guarded against an F-solve by the sweeps
    std::vector<int32_t> chF, rob, cob0, ncob;
    const int64_t nbF = (N + 63) / 64;
    for (int64_t I = 0; I < nbF; ++I)
      for (int64_t K0 = 0; K0 <= I; K0 += 8) {
        const int64_t rr = std::min<int64_t>(64, N - 64 * I);
        const int64_t ncol = std::min<int64_t>(64 * K0 + 512, 64 * I + rr) - 64 * K0;
        chF.push_back((int32_t)I);
        chF.push_back((int32_t)K0);
        rob.push_back((int32_t)I);
        cob0.push_back((int32_t)K0);
        ncob.push_back((int32_t)(std::min<int64_t>(64 * I - 64 * K0, ncol) / 64));
      }
    std::vector<int32_t> width(nbF);
    std::vector<int64_t> x0(nbF);
    for (int64_t o = 0; o < nbF; ++o) {
      width[o] = (int32_t)std::min<int64_t>(64, N - 64 * o);
      x0[o] = 64 * o;
    }
    c->df_chunks = reinterpret_cast<const int2*>(c->mem.upload(chF, st));
    c->df_nch = (int64_t)rob.size();
    c->df_plan = build_symv_plan(c->mem, st, 0, c->df_nch, rob, cob0, ncob, 0, (int32_t)nbF, width, x0);
    c->df_rhs = c->mem.zeros<double>(N, st);
    c->df_ld = ld;
    std::vector<double> u(N), y1(N), y2(N);
    std::mt19937_64 g(9);
    std::normal_distribution<double> nd;
    for (auto& v : u) v = nd(g);
    cudaMemcpyAsync(c->rhs2, u.data(), N * 8, cudaMemcpyHostToDevice, st);
    f_solve_dev(c, c->rhs2, c->xbuf);                                   // the sweeps
    cudaMemcpyAsync(y2.data(), c->xbuf, N * 8, cudaMemcpyDeviceToHost, st);
    cudaMemsetAsync(c->xbuf, 0, N * 8, st);
    dense_symv(W, ld, N, c->df_chunks, c->df_nch, &c->df_plan, c->rhs2, c->xbuf, nullptr, c->sm_count, st);
    cudaMemcpyAsync(y1.data(), c->xbuf, N * 8, cudaMemcpyDeviceToHost, st);
    cudaMemsetAsync(c->rhs2, 0, N * 8, st);
    if (int rc = sync_check(c, "dense F^-1 guard")) return rc;
    double fd = 0, fn = 0;
    for (int64_t i = 0; i < N; ++i) {
      fd += (y1[i] - y2[i]) * (y1[i] - y2[i]);
      fn += y2[i] * y2[i];
    }
    c->df_discrepancy = fn > 0 ? std::sqrt(fd / fn) : 0.0;
    if (c->df_discrepancy <= 1e-10) c->dense_finv = W;
  }
  // chunk list: row block I, first column block K0 (≤ 8 blocks of 64 columns up to the diagonal block)
  std::vector<int32_t> ch;
  std::vector<double> cb;   // bytes per chunk (rows × columns read), for the sharded split below
  const int64_t nb = (n + 63) / 64;
  for (int64_t I = 0; I < nb; ++I)
    for (int64_t K0 = 0; K0 <= I; K0 += 8) {
      ch.push_back((int32_t)I);
      ch.push_back((int32_t)K0);
      const int64_t rows = std::min<int64_t>(64, n - 64 * I);
      cb.push_back((double)rows * (double)(std::min<int64_t>(64 * K0 + 512, 64 * I + rows) - 64 * K0));
    }
  c->dw_chunks = reinterpret_cast<const int2*>(c->mem.upload(ch, st));
  c->dw_nch = (int64_t)ch.size() / 2;
  // Sharded rows: W is replicated like the F factor, and rank g applies only the contiguous run of
  // chunks [dw_c0, dw_c1) holding its 1/world of the lower triangle's bytes; its partial w (both the
  // x_I and the transposed x_K contributions) is summed over ranks by one all-reduce of n doubles.
  c->dw_c0 = 0;
  c->dw_c1 = c->dw_nch;
  if (c->sharded && c->world > 1) {
    double tot = 0;
    for (double v : cb) tot += v;
    double acc = 0;
    int64_t c0 = -1, c1 = c->dw_nch;
    for (int64_t i = 0; i < c->dw_nch; ++i) {
      const int owner = std::min<int>(c->world - 1, (int)(acc * c->world / tot));
      if (owner == c->rank && c0 < 0) c0 = i;
      if (owner > c->rank) {
        c1 = i;
        break;
      }
      acc += cb[i];
    }
    c->dw_c0 = c0 < 0 ? c1 : c0;
    c->dw_c1 = c1;
  }
  {
    double tot = 0, mine = 0;
    for (int64_t i = 0; i < c->dw_nch; ++i) {
      tot += cb[i];
      if (i >= c->dw_c0 && i < c->dw_c1) mine += cb[i];
    }
    c->dw_share = tot > 0 ? mine / tot : 1.0;
  }
  {   // deterministic accumulation plans (all chunks for the guard below; this rank's for the PCG)
    std::vector<int32_t> rob(c->dw_nch), cob0(c->dw_nch), ncob(c->dw_nch), width(nb);
    std::vector<int64_t> x0(nb);
    for (int64_t i = 0; i < c->dw_nch; ++i) {
      const int64_t I = ch[2 * i], K0 = ch[2 * i + 1], rows = std::min<int64_t>(64, n - 64 * I);
      const int64_t ncol = std::min<int64_t>(64 * K0 + 512, 64 * I + rows) - 64 * K0;
      const int64_t ncol_t = std::min<int64_t>(64 * I - 64 * K0, ncol);
      rob[i] = (int32_t)I;
      cob0[i] = (int32_t)K0;
      ncob[i] = (int32_t)(ncol_t / 64);
    }
    for (int64_t o = 0; o < nb; ++o) {
      width[o] = (int32_t)std::min<int64_t>(64, n - 64 * o);
      x0[o] = 64 * o;
    }
    c->dw_plan_all = build_symv_plan(c->mem, st, 0, c->dw_nch, rob, cob0, ncob, 0, (int32_t)nb, width, x0);
    if (c->dw_c0 == 0 && c->dw_c1 == c->dw_nch) {
      c->dw_plan = c->dw_plan_all;
    } else {
      std::vector<int32_t> r2(rob.begin() + c->dw_c0, rob.begin() + c->dw_c1),
          k2(cob0.begin() + c->dw_c0, cob0.begin() + c->dw_c1), n2(ncob.begin() + c->dw_c0, ncob.begin() + c->dw_c1);
      c->dw_plan = build_symv_plan(c->mem, st, 0, c->dw_c1 - c->dw_c0, r2, k2, n2, 0, (int32_t)nb, width, x0);
    }
  }
  cudaStreamSynchronize(st);
  // accuracy guard: W·u against the x-part of an F-solve on [u; 0]
  std::vector<double> u(N, 0.0), y1(n), y2(n);
  std::mt19937_64 g(7);
  std::normal_distribution<double> nd;
  for (int64_t i = 0; i < n; ++i) u[i] = nd(g);
  cudaMemcpyAsync(c->rhs2, u.data(), N * 8, cudaMemcpyHostToDevice, st);
  f_solve_dev(c, c->rhs2, c->xbuf);
  cudaMemcpyAsync(y2.data(), c->xbuf, n * 8, cudaMemcpyDeviceToHost, st);
  cudaMemsetAsync(c->xbuf, 0, n * 8, st);
  dense_symv(W, ld, n, c->dw_chunks, c->dw_nch, &c->dw_plan_all, c->rhs2, c->xbuf, nullptr, c->sm_count, st);
  cudaMemcpyAsync(y1.data(), c->xbuf, n * 8, cudaMemcpyDeviceToHost, st);
  cudaMemsetAsync(c->rhs2, 0, N * 8, st);
  if (int rc = sync_check(c, "dense W guard")) return rc;
  double fd = 0, fn = 0;
  for (int64_t i = 0; i < n; ++i) {
    fd += (y1[i] - y2[i]) * (y1[i] - y2[i]);
    fn += y2[i] * y2[i];
  }
  c->dw_discrepancy = fn > 0 ? std::sqrt(fd / fn) : 0.0;
  if (std::getenv("QPB_VERBOSE"))
    std::fprintf(stderr, "qpb: dense W (n = %lld, %.3g GB read per product) guard %.2e\n", (long long)n,
                 wbytes / 1e9, c->dw_discrepancy);
  bool ok = c->dw_discrepancy <= 1e-10;
  if (c->sharded && c->world > 1)
    if (int rc = agree_all(c, ok)) return rc;   // one decision for every rank (guard min over ranks)
  if (!ok) {
    cudaStreamSynchronize(st);
    c->mem.free_ptr(W);
    return QP_OK;
  }
  c->dense_w = W;
  c->dw_ld = ld;
  return QP_OK;
}

int ipm_factor_once(qp_ctx* c, const double* D0, qp_precond p) {
  int rc = require(c, false);
  if (rc) return rc;
  if (c->factored) return fail(c, QP_ESTATE, "ipm_factor_once already called (the factor of F is computed once)");
  if (p < QP_PREC_NONE || p > QP_PREC_HIGH) return fail(c, QP_EINVAL, "unknown preconditioner");
  if (c->sharded && p == QP_PREC_HIGH)
    return fail(c, QP_EINVAL, "P_H couples all inequality rows: not available with sharded rows (DESIGN.md §7)");
  c->precond = (int)p;
  cudaStream_t st = c->stream;
  const int64_t n = c->n, m1 = c->m1, m2 = c->m2, N = n + m1;
  double t0 = now_s();
  std::string e = analyse_F(c);
  if (!e.empty()) return fail(c, QP_EINVAL, "symbolic analysis of F: " + e);
  std::vector<int64_t> pinv(n);
  for (int64_t i = 0; i < n; ++i) pinv[c->perm[i]] = i;
  e = upload_factor(c, c->FF, c->ws_limit);
  if (!e.empty()) return fail(c, QP_ENOMEM, e);
  plan_inverse(c, c->FF);
  // ---- permuted operators (factor order for the x block)
  try {
    HostCSR Hf = permute(c->H, &c->perm, &pinv);
    HostCSR Af = permute(c->A, nullptr, &pinv);
    HostCSR Cf = permute(c->C, nullptr, &pinv);
    HostCSR Atf = transpose(Af), Ctf = transpose(Cf);
    c->Hf = upload_csr(c->mem, Hf, st);
    c->Af = upload_csr(c->mem, Af, st);
    c->Cf = upload_csr(c->mem, Cf, st);
    {   // rows of C longer than 32 entries (power-law degrees, c3/c3s): warp per row in the fused PCG step
      std::vector<int32_t> lr;
      for (int64_t r = 0; r < Cf.nrows; ++r)
        if (Cf.p[r + 1] - Cf.p[r] > KF_LONG_ROW) lr.push_back((int32_t)r);
      c->n_long_c = (int64_t)lr.size();
      c->long_c = c->mem.upload(lr, st);
      cudaStreamSynchronize(st);
    }
    c->Atf = upload_csr(c->mem, Atf, st);
    c->Ctf = upload_csr(c->mem, Ctf, st);
    std::vector<double> gf(n);
    for (int64_t i = 0; i < n; ++i) gf[i] = c->g[c->perm[i]];
    c->gf = c->mem.upload(gf, st);
    c->bv = c->mem.upload(c->b, st);
    c->dv = c->mem.upload(c->d, st);
    std::vector<int64_t> pf(N);
    for (int64_t i = 0; i < n; ++i) pf[i] = c->perm[i];
    for (int64_t i = 0; i < m1; ++i) pf[n + i] = n + i;
    c->perm_dev = c->mem.upload(pf, st);
    int64_t V = std::max<int64_t>(N, m2);
    c->xl = c->mem.zeros<double>(N, st);
    c->nu = c->mem.zeros<double>(m2, st);
    c->s = c->mem.zeros<double>(m2, st);
    c->rgre = c->mem.zeros<double>(N, st);
    c->rhs2 = c->mem.zeros<double>(N, st);
    c->xbuf = c->mem.zeros<double>(N, st);
    c->dxl = c->mem.zeros<double>(N, st);
    c->rc = c->mem.zeros<double>(m2, st);
    c->ra = c->mem.zeros<double>(m2, st);
    c->Dk = c->mem.zeros<double>(m2, st);
    c->rnu = c->mem.zeros<double>(m2, st);
    c->ds = c->mem.zeros<double>(m2, st);
    c->px = c->mem.zeros<double>(m2, st);
    c->pr = c->mem.zeros<double>(m2, st);
    c->pz = c->mem.zeros<double>(m2, st);
    c->pp = c->mem.zeros<double>(m2, st);
    c->pq = c->mem.zeros<double>(m2, st);
    c->vin = c->mem.zeros<double>(V, st);
    c->vin2 = c->mem.zeros<double>(V, st);
    c->vout = c->mem.zeros<double>(V, st);
    c->partial = c->mem.zeros<double>(4 * (size_t)std::max(c->vgrid, 1), st);
    c->pst = c->mem.zeros<PcgState>(1, st);
    c->ist = c->mem.zeros<IpmState>(1, st);
    c->ubuf = c->mem.zeros<double>(N, st);
    c->xs_W = c->mem.zeros<double>(m2, st);
    c->xs_p = c->mem.zeros<double>(n, st);
    c->xs_q = c->mem.zeros<double>(n, st);
    c->xs_r = c->mem.zeros<double>(n, st);
    c->xs_x = c->mem.zeros<double>(n, st);
    c->xs_lam = c->mem.zeros<double>(std::max<int64_t>(m1, 1), st);
    c->xs_rhs = c->mem.zeros<double>(N, st);
    PcgState ps{};
    ps.defer = c->sharded ? 1 : 0;
    cudaMemcpyAsync(c->pst, &ps, sizeof(PcgState), cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);   // ps is a stack object
  } catch (std::bad_alloc&) {
    return fail(c, QP_ENOMEM, "cudaMalloc failed (problem / vectors)");
  }
  rc = cuda_check(c, "upload");
  if (rc) return rc;
  // ---- numeric LDLᵀ of F, once
  double t1 = now_s();
  rc = numeric_factor(c, c->FF, nullptr, nullptr, nullptr, "F factorization");
  c->t_factor = now_s() - t1;
  if (rc) return rc;
  c->FF.use_symmetric_roots(false);
  if (c->FF.n_sym > 0) {
    // accuracy guard for the symmetric-root shortcut: one F-solve through S⁻¹ vs through X/Xᵀ
    std::vector<double> r(N), y1(N), y2(N);
    uint64_t st64 = 0x9E3779B97F4A7C15ull;
    for (int64_t i = 0; i < N; ++i) {
      st64 = st64 * 6364136223846793005ull + 1442695040888963407ull;
      r[i] = (double)((st64 >> 11) & ((1ull << 52) - 1)) / (double)(1ull << 52) - 0.5;
    }
    cudaMemcpyAsync(c->rhs2, r.data(), N * 8, cudaMemcpyHostToDevice, st);
    c->FF.use_symmetric_roots(true);
    f_solve_dev(c, c->rhs2, c->xbuf);
    cudaMemcpyAsync(y1.data(), c->xbuf, N * 8, cudaMemcpyDeviceToHost, st);
    c->FF.use_symmetric_roots(false);
    f_solve_dev(c, c->rhs2, c->xbuf);
    cudaMemcpyAsync(y2.data(), c->xbuf, N * 8, cudaMemcpyDeviceToHost, st);
    rc = sync_check(c, "symmetric-root guard");
    if (rc) return rc;
    double dn = 0, nn = 0;
    for (int64_t i = 0; i < N; ++i) {
      dn += (y1[i] - y2[i]) * (y1[i] - y2[i]);
      nn += y2[i] * y2[i];
    }
    c->FF.sym_discrepancy = nn > 0 ? std::sqrt(dn / nn) : 0.0;
    c->FF.use_symmetric_roots(c->FF.sym_discrepancy <= 1e-10 && std::isfinite(c->FF.sym_discrepancy));
    // flattened forest: M = L21 L11⁻¹ and L11⁻¹ column by column from forward sweeps on unit vectors
    // (the sweep kernels already validated above), then the same accuracy guard against the sweeps
    Factor& F = c->FF;
    const char* fe = std::getenv("QPB_FLAT");
    if (F.S.flat && F.sym_enabled && !(fe && fe[0] == '0')) {
      if (std::getenv("QPB_VERBOSE")) {   // M-tile shape statistics
        const auto& S = F.S;
        int64_t ent = 0, warps = 0, hist[5] = {0, 0, 0, 0, 0};
        for (size_t t = 0; t < S.fl_mt_J.size(); ++t) {
          const int64_t J = S.fl_mt_J[t], w = S.sn_start[J + 1] - S.sn_start[J], nq = S.fl_mt_nq[t];
          ent += w * nq;
          warps += (nq + 63) / 64;
          hist[w <= 2 ? 0 : w <= 8 ? 1 : w <= 16 ? 2 : w <= 32 ? 3 : 4]++;
        }
        std::fprintf(stderr, "qpb: flat %lld units; ", (long long)F.d.fl_nunits);
        std::fprintf(stderr, "qpb: flat rc0 %lld, %zu M tiles, %lld entries, %.2f busy warps per tile, "
                     "w<=2/8/16/32/64: %lld %lld %lld %lld %lld tiles\n", (long long)S.fl_rc0, S.fl_mt_J.size(),
                     (long long)ent, S.fl_mt_J.empty() ? 0.0 : (double)warps / S.fl_mt_J.size(), (long long)hist[0],
                     (long long)hist[1], (long long)hist[2], (long long)hist[3], (long long)hist[4]);
      }
      cudaMemsetAsync(c->rhs2, 0, N * 8, st);
      SweepRhs ur{};
      ur.rhs = c->rhs2;
      for (int64_t col = 0; col < F.S.fl_rc0; ++col) {
        flat_set_unit(c->rhs2, col, st);
        trsv_forward(F.d, ur, c->xbuf, c->tgrid, st);
        flat_extract(F.d, col, c->xbuf, c->rhs2, col, st);
      }
      {
        DeviceArena tmp;
        const int32_t* src = tmp.upload(F.S.fl_mr_src, st);
        flat_fill_rows(F.d, src, (int64_t)F.S.fl_mr_src.size(), st);
        cudaStreamSynchronize(st);
        tmp.release();
      }
      cudaMemsetAsync(F.d.acc, 0, N * 8, st);
      rc = cuda_check(c, "flattened forest extraction");
      if (rc) return rc;
      cudaMemcpyAsync(c->rhs2, r.data(), N * 8, cudaMemcpyHostToDevice, st);
      f_solve_dev(c, c->rhs2, c->xbuf);
      cudaMemcpyAsync(y2.data(), c->xbuf, N * 8, cudaMemcpyDeviceToHost, st);
      F.d.flat = 1;
      f_solve_dev(c, c->rhs2, c->xbuf);
      cudaMemcpyAsync(y1.data(), c->xbuf, N * 8, cudaMemcpyDeviceToHost, st);
      rc = sync_check(c, "flattened-forest guard");
      if (rc) return rc;
      double fd = 0, fn = 0;
      for (int64_t i = 0; i < N; ++i) {
        fd += (y1[i] - y2[i]) * (y1[i] - y2[i]);
        fn += y2[i] * y2[i];
      }
      F.flat_discrepancy = fn > 0 ? std::sqrt(fd / fn) : 0.0;
      F.d.flat = (F.flat_discrepancy <= 1e-10 && std::isfinite(F.flat_discrepancy)) ? 1 : 0;
      if (!F.d.flat) cudaMemsetAsync(F.d.acc, 0, N * 8, st);   // the sweeps expect zero accumulators
    }
    // level products (deep forests: c2, c3s, c4s): the same guard against the sweeps, then the fastest of up
    // to three paths is kept by TIMING them on this factor (median of 5 F-solves after 2 warm-ups each): the
    // task graph, the level products over subtrees, and the level products over the leaf phase's level
    // kernels.  Which wins depends on the tree — c2 (deep nested dissection): 1.34 / 0.81 / 0.88 ms; c3s (a
    // shallow, unbalanced minimum-degree forest under a dominant root: its 8 291 subtrees are long chains
    // of supernodes, 65 µs per sweep in one warp each): 0.166 / 0.210 / ≈ 0.12 ms.  QPB_PI=2 skips the task
    // graph, QPB_ST=0 the subtrees, QPB_ST=2 the leaf-phase variant.
    const char* pe = std::getenv("QPB_PI");
    if (F.sym_enabled && !F.d.flat && !(pe && pe[0] == '0')) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto time_path = [&]() -> double {
        std::vector<float> ts;
        for (int rep = 0; rep < 7; ++rep) {
          cudaEventRecord(e0, st);
          f_solve_dev(c, c->rhs2, c->xbuf);
          cudaEventRecord(e1, st);
          cudaEventSynchronize(e1);
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          if (rep >= 2) ts.push_back(ms);
        }
        std::sort(ts.begin(), ts.end());
        return ts[ts.size() / 2];
      };
      auto zero_acc = [&]() {   // the sweeps expect zero accumulators
        cudaMemsetAsync(F.d.acc, 0, N * 8, st);
        cudaMemsetAsync(F.d.tacc, 0, N * 8, st);
      };
      // reference: the task graph
      F.pi = PiSweep{};
      cudaMemcpyAsync(c->rhs2, r.data(), N * 8, cudaMemcpyHostToDevice, st);
      f_solve_dev(c, c->rhs2, c->xbuf);
      cudaMemcpyAsync(y2.data(), c->xbuf, N * 8, cudaMemcpyDeviceToHost, st);
      rc = sync_check(c, "level-product reference");
      if (rc) return rc;
      const bool force = pe && pe[0] == '2';
      const bool only_st = std::getenv("QPB_ST") && std::getenv("QPB_ST")[0] == '2';   // tests: subtrees or nothing
      double best_ms = force ? 1e30 : time_path();
      F.pi_ms[0] = force ? 0.0 : best_ms;
      PiSweep best{};
      double best_disc = -1.0;
      for (int cand = 0; cand < 2; ++cand) {   // 0: over subtrees, 1: over the leaf phase
        rc = build_pi(c, cand == 0);
        if (rc) return rc;
        PiSweep P = F.pi;
        if (P.nlev <= 0 || (cand == 1 && best.nlev > 0 && best.st_n == 0)) {   // nothing built / same plan as candidate 0
          F.pi = best;
          if (cand == 0) continue;
          break;
        }
        F.pi.enabled = 1;
        f_solve_dev(c, c->rhs2, c->xbuf);
        cudaMemcpyAsync(y1.data(), c->xbuf, N * 8, cudaMemcpyDeviceToHost, st);
        rc = sync_check(c, "level-product guard");
        if (rc) return rc;
        double fd = 0, fn = 0;
        for (int64_t i = 0; i < N; ++i) {
          fd += (y1[i] - y2[i]) * (y1[i] - y2[i]);
          fn += y2[i] * y2[i];
        }
        const double disc = fn > 0 ? std::sqrt(fd / fn) : 0.0;
        const bool ok = disc <= 1e-10 && std::isfinite(disc);
        const double ms = ok ? time_path() : 1e30;
        if (ok && (F.pi_ms[1] == 0.0 || ms < F.pi_ms[1])) F.pi_ms[1] = ms;   // the faster level-product variant
        rc = cuda_check(c, "level-product timing");
        if (rc) return rc;
        if (std::getenv("QPB_VERBOSE"))
          std::fprintf(stderr, "qpb: level products over %s: guard %.3e, F-solve %.3f ms (task graph %.3f ms)\n",
                       P.st_n > 0 ? "subtrees" : "the leaf phase", disc, ok ? ms : -1.0, F.pi_ms[0]);
        if (cand == 0 || best.nlev == 0) F.pi_discrepancy = disc;
        bool better = ok && ms < best_ms;
        if (c->sharded)
          if (int rc3 = agree_all(c, better)) return rc3;
        if (better) {
          if (best.Z) F.mem.free_ptr(best.Z);
          best = F.pi;
          best.enabled = 1;
          best_ms = ms;
          best_disc = disc;
        } else if (P.Z) {
          F.mem.free_ptr(P.Z);
        }
        F.pi = PiSweep{};
        if (cand == 0 && (P.st_n == 0 || only_st)) break;   // no subtrees planned (the second candidate is the same plan) / QPB_ST=2
      }
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      F.pi = best;
      if (best.enabled) {
        F.pi_discrepancy = best_disc;
        if (!F.d.flat) F.d.fl_rc0 = F.pi.root0;
      }
      zero_acc();
      if (std::getenv("QPB_VERBOSE"))
        std::fprintf(stderr, "qpb: F-solve path: %s\n", !F.pi.enabled ? "task graph" : F.pi.st_n > 0
                     ? "level products over subtrees" : "level products over the leaf phase");
    }
  }
  if (int rc2 = build_dense_w(c)) return rc2;   // explicit W / small-N F⁻¹ (with or without a symmetric root)
  // ---- P_H: T = C diag(H)⁻¹ Cᵀ pattern (host) and values (device), symbolic of D + T
  if (p == QP_PREC_HIGH) {
    const bool verbose = std::getenv("QPB_VERBOSE") != nullptr;
    double tph0 = now_s();
    HostCSR Ct = transpose(c->C);
    std::vector<int64_t> tp(m2 + 1, 0);
    std::vector<int32_t> ti;
    std::vector<int64_t> mark(m2, -1);
    std::vector<int32_t> rowbuf;
    for (int64_t i = 0; i < m2; ++i) {
      rowbuf.clear();
      for (int64_t q = c->C.p[i]; q < c->C.p[i + 1]; ++q) {
        int32_t k = c->C.i[q];
        for (int64_t u = Ct.p[k]; u < Ct.p[k + 1]; ++u) {
          int32_t j = Ct.i[u];
          if (mark[j] != i) { mark[j] = i; rowbuf.push_back(j); }
        }
      }
      if (mark[i] != i) rowbuf.push_back((int32_t)i);  // empty C row: keep the diagonal of D
      std::sort(rowbuf.begin(), rowbuf.end());
      ti.insert(ti.end(), rowbuf.begin(), rowbuf.end());
      tp[i + 1] = (int64_t)ti.size();
    }
    c->nnz_t = (int64_t)ti.size();
    std::vector<int64_t> trow(c->nnz_t);
    for (int64_t i = 0; i < m2; ++i)
      for (int64_t q = tp[i]; q < tp[i + 1]; ++q) trow[q] = i;
    if (verbose) std::fprintf(stderr, "qpb: P_H pattern of T (%lld entries) %.2f s\n", (long long)c->nnz_t, now_s() - tph0);
    // ordering of P_H: minimum degree on the pattern of T (or nested dissection, below)
    std::vector<int64_t> ph_ptr;
    std::vector<int32_t> ph_idx;
    {
      std::vector<int64_t> ptr(m2 + 1, 0);
      std::vector<int32_t> idx;
      idx.reserve(c->nnz_t);
      for (int64_t r = 0; r < m2; ++r) {
        for (int64_t q = tp[r]; q < tp[r + 1]; ++q)
          if (ti[q] != r) idx.push_back(ti[q]);
        ptr[r + 1] = (int64_t)idx.size();
      }
      // the tail of P_H's elimination is dense (C diag(H)⁻¹ Cᵀ couples rows through shared columns):
      // stop the minimum-degree search once the minimum degree reaches half the remaining nodes
      const double ds = std::getenv("QPB_PH_DENSE_STOP") ? std::atof(std::getenv("QPB_PH_DENSE_STOP")) : 0.5;
      c->perm_ph = etree_postorder(m2, ptr, idx, min_degree_order(m2, ptr, idx, ds));
      ph_ptr.swap(ptr);
      ph_idx.swap(idx);
    }
    // P_H is refactored at every D: no symmetric root, and supernodes capped at 4096 columns so the
    // partitioned inverses of its sweeps cost Σ B³/6 per refactor instead of w³/6 (QPB_PH_MAXW)
    const int64_t ph_maxw = std::getenv("QPB_PH_MAXW") ? std::atoll(std::getenv("QPB_PH_MAXW")) : 4096;
    // lower pattern of P_H in the order `perm` (+ source index of every entry in T's values)
    auto build_pm = [&](const std::vector<int64_t>& perm, LowerMatrix& PM) {
      std::vector<int64_t> pinv_ph(m2);
      for (int64_t i = 0; i < m2; ++i) pinv_ph[perm[i]] = i;
      PM = LowerMatrix();
      PM.N = m2;
      PM.colptr.assign(m2 + 1, 0);
      PM.diag_src.assign(m2, -1);
      for (int64_t i = 0; i < m2; ++i)
        for (int64_t q = tp[i]; q < tp[i + 1]; ++q) {
          int64_t a2 = pinv_ph[i], bb = pinv_ph[ti[q]];
          if (a2 > bb) PM.colptr[bb + 1]++;
          else if (a2 == bb) PM.diag_src[a2] = q;
        }
      for (int64_t j = 0; j < m2; ++j) PM.colptr[j + 1] += PM.colptr[j];
      PM.rowind.resize(PM.colptr[m2]);
      PM.src.resize(PM.colptr[m2]);
      std::vector<int64_t> pos(PM.colptr.begin(), PM.colptr.end() - 1);
      for (int64_t i = 0; i < m2; ++i)
        for (int64_t q = tp[i]; q < tp[i + 1]; ++q) {
          int64_t a2 = pinv_ph[i], bb = pinv_ph[ti[q]];
          if (a2 > bb) {
            int64_t w = pos[bb]++;
            PM.rowind[w] = (int32_t)a2;
            PM.src[w] = q;
          }
        }
      std::vector<std::pair<int32_t, int64_t>> tmp;
      for (int64_t j = 0; j < m2; ++j) {
        tmp.clear();
        for (int64_t q = PM.colptr[j]; q < PM.colptr[j + 1]; ++q) tmp.emplace_back(PM.rowind[q], PM.src[q]);
        std::sort(tmp.begin(), tmp.end());
        for (int64_t q = PM.colptr[j]; q < PM.colptr[j + 1]; ++q) {
          PM.rowind[q] = tmp[q - PM.colptr[j]].first;
          PM.src[q] = tmp[q - PM.colptr[j]].second;
        }
      }
    };
    // model time of one IPM iteration's P_H work: the refactor (c_fact at ~20 TFLOP/s) plus ~50 PCG
    // iterations of two sweeps (the stored entries at ~6 TB/s, plus ~20 µs per supernodal level and sweep:
    // c4s's minimum-degree P_H measured 17 ms per sweep over 825 levels)
    auto ph_cost = [](const Symbolic& S) {
      return S.c_fact / 20e12 + 50.0 * (16.0 * (double)S.nnz_stored / 6e12 + 2.0 * 20e-6 * (double)S.n_levels);
    };
    LowerMatrix PM;
    build_pm(c->perm_ph, PM);
    e = analyse(PM, c->FP.S, 0, /*allow_symroot=*/false, -1, ph_maxw);
    // the minimum-degree order can leave a long chain of narrow supernodes (a banded T: c4s); when its
    // supernodal tree is deep, try nested dissection by level structures and keep the cheaper order by
    // the model above (QPB_PH_ND=0: never, =2: always)
    const char* nde = std::getenv("QPB_PH_ND");
    const int ndm = nde ? std::atoi(nde) : 1;
    if (e.empty() && ndm != 0 && (ndm == 2 || c->FP.S.n_levels > 64)) {
      std::vector<int64_t> nd = etree_postorder(m2, ph_ptr, ph_idx, nested_dissection_order(m2, ph_ptr, ph_idx, 64));
      LowerMatrix PM2;
      build_pm(nd, PM2);
      Symbolic S2;
      std::string e2 = analyse(PM2, S2, 0, false, -1, ph_maxw);
      const double cm = ph_cost(c->FP.S), cn = e2.empty() ? ph_cost(S2) : 1e30;
      if (verbose)
        std::fprintf(stderr, "qpb: P_H orders: min degree %lld levels, %.3g stored, model %.3g s; nested dissection "
                     "%lld levels, %.3g stored, model %.3g s %s\n", (long long)c->FP.S.n_levels,
                     (double)c->FP.S.nnz_stored, cm, (long long)S2.n_levels, (double)S2.nnz_stored, cn, e2.c_str());
      if (ndm == 2 ? e2.empty() : cn < cm) {
        c->perm_ph = nd;
        c->FP.S = std::move(S2);
      }
    }
    if (!e.empty()) return fail(c, QP_EINVAL, "symbolic analysis of P_H: " + e);
    if (verbose) std::fprintf(stderr, "qpb: P_H symbolic %.2f s\n", now_s() - tph0);
    e = upload_factor(c, c->FP, c->ws_limit);
    if (!e.empty()) return fail(c, QP_ENOMEM, e);
    plan_inverse(c, c->FP);
    try {
      c->t_row = c->mem.upload(trow, st);
      c->t_col = c->mem.upload(ti, st);
      c->t_val = c->mem.zeros<double>(c->nnz_t, st);
      std::vector<double> hd(n, 0.0);
      for (int64_t r = 0; r < n; ++r)
        for (int64_t q = c->H.p[r]; q < c->H.p[r + 1]; ++q)
          if (c->H.i[q] == r) hd[r] = c->H.v[q];
      c->hdiag = c->mem.upload(hd, st);
      HostCSR Cn = c->C;
      c->Cnu = upload_csr(c->mem, Cn, st);
      c->perm_ph_dev = c->mem.upload(c->perm_ph, st);
      c->xph = c->mem.zeros<double>(m2, st);
      c->D_ph_last = c->mem.zeros<double>(m2, st);
    } catch (std::bad_alloc&) {
      return fail(c, QP_ENOMEM, "cudaMalloc failed (P_H)");
    }
    t_values(c->Cnu, c->hdiag, c->t_row, c->t_col, c->nnz_t, c->t_val, st);  // T once
    std::vector<double> ones(m2, 1.0);
    const double* D0d;
    if (D0) {
      D0d = in_vec(c, D0, c->vin, m2);
    } else {
      cudaMemcpyAsync(c->vin, ones.data(), m2 * 8, cudaMemcpyHostToDevice, st);
      D0d = c->vin;
    }
    rc = ph_refactor(c, D0d);
    if (rc) return rc;
  }
  c->factored = true;
  return sync_check(c, "ipm_factor_once");
}

int pcg_solve(qp_ctx* c, const double* D_k, const double* rhs, double tol, int32_t maxit, double* dnu_out,
              int32_t* iters, double* relres) {
  int rc = require(c, true);
  if (rc) return rc;
  if (!D_k || !rhs) return fail(c, QP_EINVAL, "NULL D_k / rhs");
  const int64_t m2 = c->m2;
  const double* Dd = in_vec(c, D_k, c->vin, m2);
  const double* bd = in_vec(c, rhs, c->vin2, m2);
  // copy D into the IPM D buffer so P_H change detection compares stable storage
  cudaMemcpyAsync(c->Dk, Dd, m2 * 8, cudaMemcpyDeviceToDevice, c->stream);
  bool refac = false;
  if (c->precond == 2) {
    std::vector<double> a(m2), b(m2);
    cudaMemcpyAsync(a.data(), c->Dk, m2 * 8, cudaMemcpyDeviceToHost, c->stream);
    cudaMemcpyAsync(b.data(), c->D_ph_last, m2 * 8, cudaMemcpyDeviceToHost, c->stream);
    cudaStreamSynchronize(c->stream);
    refac = !c->ph_valid || a != b;
  }
  int it = 0;
  double rr = 0;
  rc = pcg_dev(c, c->Dk, bd, tol, maxit, &it, &rr, refac);
  if (iters) *iters = it;
  if (relres) *relres = rr;
  if (rc != QP_OK && rc != QP_MAXIT) return rc;
  out_vec(c, dnu_out, c->px, m2);
  int rc2 = sync_check(c, "pcg_solve");
  return rc2 ? rc2 : rc;
}

int pcg_solve_x(qp_ctx* c, const double* D_k, const double* f, const double* e, double tol, int32_t maxit,
                double* dx_out, double* dlam_out, int32_t* iters, double* relres) {
  int rc = require(c, true);
  if (rc) return rc;
  if (c->sharded) return fail(c, QP_EINVAL, "the x-space twin is not available with sharded rows");
  if (!D_k || !f || (c->m1 > 0 && !e)) return fail(c, QP_EINVAL, "NULL D_k / f / e");
  const int64_t n = c->n, m1 = c->m1;
  const double* Dd = in_vec(c, D_k, c->vin, c->m2);
  cudaMemcpyAsync(c->Dk, Dd, c->m2 * 8, cudaMemcpyDeviceToDevice, c->stream);
  const double* fd = in_vec(c, f, c->vin2, n);
  gather(c->rhs2, fd, c->perm_dev, n, nullptr, c->stream);    // f into factor order
  if (m1 > 0) {
    const double* ed = in_vec(c, e, c->vin, m1);              // D_k already copied out of vin
    cudaMemcpyAsync(c->rhs2 + n, ed, m1 * 8, cudaMemcpyDeviceToDevice, c->stream);
  }
  int it = 0;
  double rr = 0;
  rc = pcg_x_dev(c, c->Dk, c->rhs2, tol, maxit, &it, &rr);
  if (iters) *iters = it;
  if (relres) *relres = rr;
  if (rc != QP_OK && rc != QP_MAXIT) return rc;
  scatter(c->vout, c->xs_x, c->perm_dev, n, nullptr, c->stream);
  out_vec(c, dx_out, c->vout, n);
  if (m1 > 0) out_vec(c, dlam_out, c->xs_lam, m1);
  int rc2 = sync_check(c, "pcg_solve_x");
  return rc2 ? rc2 : rc;
}

int qp_ipm_init(qp_ctx* c, const qp_ipm_opts* o) {
  int rc = require(c, true);
  if (rc) return rc;
  qp_ipm_opts d{1e-8, 1e-3, 0.1, 0.995, 100, 2000, 1, 0};
  c->opts = o ? *o : d;
  if (c->opts.space != 0 && c->opts.space != 1) return fail(c, QP_EINVAL, "qp_ipm_opts.space must be 0 or 1");
  if (c->opts.space == 1 && c->sharded) return fail(c, QP_EINVAL, "the x-space twin is not available with sharded rows");
  if (c->opts.max_ipm <= 0) c->opts.max_ipm = 100;
  if (c->opts.pcg_maxit <= 0) c->opts.pcg_maxit = 2000;
  const int64_t n = c->n, m1 = c->m1, m2 = c->m2;
  cudaStream_t st = c->stream;
  // x = 0, λ = 0, ν = 1, s = |d| + 1 (reading R3 start)
  cudaMemsetAsync(c->xl, 0, (n + m1) * 8, st);
  std::vector<double> ones(m2, 1.0), s0(m2);
  for (int64_t i = 0; i < m2; ++i) s0[i] = std::fabs(c->d[i]) + 1.0;
  cudaMemcpyAsync(c->nu, ones.data(), m2 * 8, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(c->s, s0.data(), m2 * 8, cudaMemcpyHostToDevice, st);
  IpmState is{};
  is.sigma = c->opts.sigma;
  is.tau = c->opts.tau;
  is.defer = c->sharded ? 1 : 0;
  is.m2_total = (double)c->m2_global;
  cudaMemcpyAsync(c->ist, &is, sizeof(IpmState), cudaMemcpyHostToDevice, st);
  c->ipm_k = 0;
  c->ipm_converged = false;
  c->pcg_hist.clear();
  c->ipm_initialised = true;
  return sync_check(c, "qp_ipm_init");
}

int qp_ipm_iterate(qp_ctx* c, int32_t nsteps, qp_ipm_result* r, int32_t* done) {
  int rc = require(c, true);
  if (rc) return rc;
  if (!c->ipm_initialised) return fail(c, QP_ESTATE, "qp_ipm_init has not been called");
  for (int32_t k = 0; k < nsteps && !c->ipm_converged && c->ipm_k < c->opts.max_ipm; ++k) {
    bool conv = false;
    rc = ipm_iteration(c, &conv);
    if (rc) return rc;
    if (conv) c->ipm_converged = true;
  }
  if (!c->ipm_converged && c->ipm_k >= c->opts.max_ipm) {
    // final residual evaluation at the last iterate
    if ((rc = ipm_eval_residuals(c))) return rc;

  }
  if (done) *done = c->ipm_converged ? 1 : 0;
  fill_result(c, r);
  return sync_check(c, "qp_ipm_iterate");
}

int ipm_solve(qp_ctx* c, const qp_ipm_opts* o, qp_ipm_result* r) {
  double t0 = now_s();
  int rc = qp_ipm_init(c, o);
  if (rc) return rc;
  int32_t done = 0;
  rc = qp_ipm_iterate(c, c->opts.max_ipm + 1, r, &done);
  if (r) r->t_solve_s = now_s() - t0;
  if (rc) return rc;
  return done ? QP_OK : QP_MAXIT;
}

int qp_f_solve(qp_ctx* c, const double* rhs, double* out) {
  int rc = require(c, true);
  if (rc) return rc;
  const int64_t N = c->n + c->m1;
  const double* in = in_vec(c, rhs, c->vin, N);
  gather(c->rhs2, in, c->perm_dev, N, nullptr, c->stream);   // factor order
  f_solve_dev(c, c->rhs2, c->xbuf);
  scatter(c->vout, c->xbuf, c->perm_dev, N, nullptr, c->stream);
  out_vec(c, out, c->vout, N);
  rc = sync_check(c, "qp_f_solve");
  c->harvest();
  return rc;
}

int qp_kf_apply(qp_ctx* c, const double* D, const double* p, double* q) {
  int rc = require(c, true);
  if (rc) return rc;
  const int64_t m2 = c->m2;
  const double* Dd = in_vec(c, D, c->vin, m2);
  const double* pd = in_vec(c, p, c->vin2, m2);
  rc = kf_apply_dev(c, Dd, pd, c->vout, false);
  if (rc) return rc;
  out_vec(c, q, c->vout, m2);
  rc = sync_check(c, "qp_kf_apply");
  c->harvest();
  return rc;
}

static int ensure_op(qp_ctx* c) {
  if (c->op_ready) return QP_OK;
  cudaStream_t st = c->stream;
  try {
    c->opH = upload_csr(c->mem, c->H, st);
    c->opC = upload_csr(c->mem, c->C, st);
    c->opCt = upload_csr(c->mem, transpose(c->C), st);
    c->op_D = c->mem.zeros<double>(std::max<int64_t>(1, c->m2), st);
    c->op_t = c->mem.zeros<double>(std::max<int64_t>(1, c->m2), st);
    c->op_p = c->mem.zeros<double>(c->n, st);
    c->op_q = c->mem.zeros<double>(c->n, st);
  } catch (std::bad_alloc&) {
    return fail(c, QP_ENOMEM, "cudaMalloc failed (operator copies)");
  }
  c->op_ready = true;
  return QP_OK;
}

int qp_operator_apply(qp_ctx* c, const double* D, const double* p, double* q) {
  if (!c) return QP_EINVAL;
  if (!c->setup_done) return fail(c, QP_ESTATE, "qp_setup has not completed");
  cudaSetDevice(c->device);
  cudaStream_t st = c->stream;
  if (int rc = ensure_op(c)) return rc;
  const double* Dd = in_vec(c, D, c->op_D, c->m2);
  const double* pd = in_vec(c, p, c->op_p, c->n);
  double* qd = c->vectors_on_device ? q : c->op_q;
  op_apply(c->opH, c->opC, c->opCt, Dd, pd, c->op_t, qd, !c->sharded || c->rank == 0, c->sm_count, st);
  c->launches += 2;
  if (c->sharded)
    if (int rc = c->allreduce(qd, c->n, 0)) return rc;   // Σ_ranks of the rows' partial products
  if (!c->vectors_on_device) out_vec(c, q, c->op_q, c->n);
  return sync_check(c, "qp_operator_apply");
}

// Small all-gather through the all-reduce: every rank contributes `per` values at its own offset.
static int gather_small(qp_ctx* c, const std::vector<double>& mine, std::vector<double>& all) {
  const int64_t per = (int64_t)mine.size(), tot = per * c->world;
  all.assign(tot, 0.0);
  for (int64_t k = 0; k < per; ++k) all[c->rank * per + k] = mine[k];
  cudaMemcpyAsync(c->op_q, all.data(), tot * 8, cudaMemcpyHostToDevice, c->stream);
  if (int rc = c->allreduce(c->op_q, tot, 0)) return rc;
  cudaMemcpyAsync(all.data(), c->op_q, tot * 8, cudaMemcpyDeviceToHost, c->stream);
  return sync_check(c, "halo plan gather");
}

int qp_operator_halo_plan(qp_ctx* c, int64_t* info) {
  if (!c || !info) return QP_EINVAL;
  if (!c->setup_done) return fail(c, QP_ESTATE, "qp_setup has not completed");
  cudaSetDevice(c->device);
  if (int rc = ensure_op(c)) return rc;
  auto& P = c->halo;
  const int W = c->world, g = c->rank;
  const int64_t n = c->n;
  if (!P.planned) {
    P.enabled = false;
    if (c->sharded && W >= 2 && n >= 4 * (int64_t)W) {
      // columns this rank's rows of C touch
      double cmin = (double)n, cmax = -1.0;
      for (int32_t j : c->C.i) {
        cmin = std::min(cmin, (double)j);
        cmax = std::max(cmax, (double)j);
      }
      std::vector<double> all;
      if (int rc = gather_small(c, {cmin, cmax}, all)) return rc;
      // owned boundaries: b_0 = 0, b_W = n, b_g = the midpoint between the last column rank g − 1 touches
      // and the first column rank g touches (rounded down), made monotone
      P.b.assign(W + 1, 0);
      P.b[W] = n;
      bool ok = true;
      for (int r = 1; r < W; ++r) {
        const double hi_prev = all[2 * (r - 1) + 1], lo_here = all[2 * r];
        if (hi_prev < 0 || lo_here >= (double)n) ok = false;   // a rank without entries
        int64_t mid = (int64_t)std::floor((hi_prev + 1.0 + lo_here) / 2.0);
        P.b[r] = std::max<int64_t>(P.b[r - 1], std::min<int64_t>(n, std::max<int64_t>(0, mid)));
      }
      for (int r = 0; r < W; ++r) ok = ok && P.b[r + 1] > P.b[r];
      // this rank's windows: q = owned ∪ C's columns; p = q ∪ the columns of H's owned rows
      int64_t qlo = std::min<int64_t>(P.b[g], (int64_t)cmin), qhi = std::max<int64_t>(P.b[g + 1], (int64_t)cmax + 1);
      int64_t plo = qlo, phi = qhi;
      for (int64_t i = P.b[g]; ok && i < P.b[g + 1]; ++i)
        for (int64_t e = c->H.p[i]; e < c->H.p[i + 1]; ++e) {
          plo = std::min<int64_t>(plo, c->H.i[e]);
          phi = std::max<int64_t>(phi, (int64_t)c->H.i[e] + 1);
        }
      std::vector<double> wall;
      if (int rc = gather_small(c, {(double)plo, (double)phi, (double)qlo, (double)qhi}, wall)) return rc;
      P.plo.resize(W); P.phi.resize(W); P.qlo.resize(W); P.qhi.resize(W);
      for (int r = 0; r < W; ++r) {
        P.plo[r] = (int64_t)wall[4 * r];
        P.phi[r] = (int64_t)wall[4 * r + 1];
        P.qlo[r] = (int64_t)wall[4 * r + 2];
        P.qhi[r] = (int64_t)wall[4 * r + 3];
        // only the two neighbours' owned ranges may be reached
        const int64_t left = P.b[std::max(0, r - 1)], right = P.b[std::min(W, r + 2)];
        ok = ok && P.plo[r] >= left && P.phi[r] <= right && P.qlo[r] >= left && P.qhi[r] <= right;
      }
      {   // one decision for every rank (xbuf may not exist yet: through the small gather)
        std::vector<double> oks;
        if (int rc = gather_small(c, {ok ? 1.0 : 0.0}, oks)) return rc;
        for (double v : oks) ok = ok && v > 0.5;
      }
      if (ok) {
        const int64_t nfp = g > 0 ? std::max<int64_t>(0, P.qhi[g - 1] - P.b[g]) : 0;
        const int64_t nfn = g + 1 < W ? std::max<int64_t>(0, P.b[g + 1] - P.qlo[g + 1]) : 0;
        try {
          P.from_prev = c->mem.zeros<double>((size_t)std::max<int64_t>(1, nfp), c->stream);
          P.from_next = c->mem.zeros<double>((size_t)std::max<int64_t>(1, nfn), c->stream);
        } catch (std::bad_alloc&) {
          return fail(c, QP_ENOMEM, "cudaMalloc failed (halo buffers)");
        }
      }
      P.enabled = ok;
    }
    P.planned = true;
  }
  for (int k = 0; k < 8; ++k) info[k] = 0;
  info[0] = P.enabled ? 1 : 0;
  if (P.enabled) {
    info[1] = P.b[g];
    info[2] = P.b[g + 1];
    info[3] = P.plo[g];
    info[4] = P.phi[g];
    info[5] = P.qlo[g];
    info[6] = P.qhi[g];
    int64_t sent = 0;
    if (g > 0) sent += std::max<int64_t>(0, P.phi[g - 1] - P.b[g]) + std::max<int64_t>(0, P.b[g] - P.qlo[g]);
    if (g + 1 < W) sent += std::max<int64_t>(0, P.b[g + 1] - P.plo[g + 1]) + std::max<int64_t>(0, P.qhi[g] - P.b[g + 1]);
    info[7] = sent;
  }
  return QP_OK;
}

int qp_operator_apply_halo(qp_ctx* c, const double* D, double* p, double* q) {
  if (!c) return QP_EINVAL;
  if (!c->setup_done) return fail(c, QP_ESTATE, "qp_setup has not completed");
  auto& P = c->halo;
  if (!P.planned || !P.enabled) return fail(c, QP_ESTATE, "no halo plan (qp_operator_halo_plan) or not band-local");
  cudaSetDevice(c->device);
  cudaStream_t st = c->stream;
  const int W = c->world, g = c->rank;
  const double* Dd = in_vec(c, D, c->op_D, c->m2);
  double* pd = c->vectors_on_device ? p : c->op_p;
  double* qd = c->vectors_on_device ? q : c->op_q;
  if (!c->vectors_on_device)
    cudaMemcpyAsync(pd + P.b[g], p + P.b[g], (P.b[g + 1] - P.b[g]) * 8, cudaMemcpyHostToDevice, st);
  // 1. boundary entries of p: my owned entries inside the neighbours' windows go out, my window's
  //    entries outside my owned range come in (in place: all ranges are contiguous)
  const int64_t tp = g > 0 ? std::max<int64_t>(0, P.phi[g - 1] - P.b[g]) : 0;
  const int64_t tn = g + 1 < W ? std::max<int64_t>(0, P.b[g + 1] - P.plo[g + 1]) : 0;
  const int64_t fp = std::max<int64_t>(0, P.b[g] - P.plo[g]), fn = std::max<int64_t>(0, P.phi[g] - P.b[g + 1]);
  if (int rc = c->exchange(pd + P.b[g], tp, pd + (P.b[g + 1] - tn), tn, pd + P.plo[g], fp, pd + P.b[g + 1], fn)) return rc;
  // 2. local products on the windows
  op_apply_range(c->opH, c->opC, c->opCt, Dd, pd, c->op_t, qd, P.qlo[g], P.qhi[g], P.b[g], P.b[g + 1], c->sm_count, st);
  c->launches += 2;
  // 3. q outside the owned range goes to its owner and is added there
  const int64_t qtp = std::max<int64_t>(0, P.b[g] - P.qlo[g]), qtn = std::max<int64_t>(0, P.qhi[g] - P.b[g + 1]);
  const int64_t qfp = g > 0 ? std::max<int64_t>(0, P.qhi[g - 1] - P.b[g]) : 0;
  const int64_t qfn = g + 1 < W ? std::max<int64_t>(0, P.b[g + 1] - P.qlo[g + 1]) : 0;
  if (int rc = c->exchange(qd + P.qlo[g], qtp, qd + P.b[g + 1], qtn, P.from_prev, qfp, P.from_next, qfn)) return rc;
  add_range(qd + P.b[g], P.from_prev, qfp, st);
  add_range(qd + (P.b[g + 1] - qfn), P.from_next, qfn, st);
  c->launches += (qfp > 0) + (qfn > 0);
  if (!c->vectors_on_device) {
    cudaMemcpyAsync(p + P.plo[g], pd + P.plo[g], (P.phi[g] - P.plo[g]) * 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(q + P.b[g], qd + P.b[g], (P.b[g + 1] - P.b[g]) * 8, cudaMemcpyDeviceToHost, st);
  }
  return sync_check(c, "qp_operator_apply_halo");
}

int qp_get_structure(qp_ctx* c, int32_t which, int64_t* out, int64_t* len) {
  if (!c) return QP_EINVAL;
  if (!c->analysed) return fail(c, QP_ESTATE, "no symbolic analysis yet (qp_analyse or ipm_factor_once)");
  const Symbolic& S = which >= 10 ? c->FP.S : c->FF.S;
  if (which >= 10 && c->precond != 2) return fail(c, QP_ESTATE, "no P_H factor (precond != HIGH)");
  std::vector<int64_t> v;
  switch (which % 10) {
    case 0:
      if (which >= 10) v = c->perm_ph;
      else {
        v = c->perm;
        for (int64_t i = 0; i < c->m1; ++i) v.push_back(c->n + i);
      }
      break;
    case 1: v = S.parent; break;
    case 2: v = S.colcount; break;
    case 3: v = S.sn_start; break;
    case 4: v = S.sn_parent; break;
    case 5: v = S.sn_level; break;
    case 6: v = S.sn_rowptr; break;
    case 7: v.assign(S.sn_rows.begin(), S.sn_rows.end()); break;
    case 8: v = S.rowlev; break;
    case 9: v = {S.trailing_from}; break;
    default: return fail(c, QP_EINVAL, "unknown structure id");
  }
  if (!len) return QP_EINVAL;
  if (out) {
    if (*len < (int64_t)v.size()) return fail(c, QP_EINVAL, "buffer too small");
    std::memcpy(out, v.data(), v.size() * 8);
  }
  *len = (int64_t)v.size();
  return QP_OK;
}

int qp_get_stats(qp_ctx* c, qp_stats* s) {
  if (!c || !s) return QP_EINVAL;
  std::memset(s, 0, sizeof(*s));
  s->n = c->n;
  s->m1 = c->m1;
  s->m2 = c->m2;
  s->nnz_H = c->H.nnz();
  s->nnz_A = c->A.nnz();
  s->nnz_C = c->C.nnz();
  if (c->analysed) {
    const Symbolic& S = c->FF.S;
    s->nnz_LF = S.nnz_L;
    s->nnz_LF_stored = S.nnz_stored;
    s->workspace_bytes = S.ws_size * 8;
    s->factor_bytes = S.fs_size * 8;
    s->n_supernodes_F = S.ns;
    s->n_blocks_F = S.nb;
    s->n_levels_F = S.n_levels;
    s->row_levels_F = S.n_rowlev;
    s->c_fact_F = S.c_fact;
    s->workspace_bytes = S.ws_size * 8 + c->FP.S.ws_size * 8;
    s->factor_bytes = S.fs_size * 8 + c->FP.S.fs_size * 8;
    if (c->precond == 2) {
      s->nnz_LPH = c->FP.S.nnz_L;
      s->n_supernodes_PH = c->FP.S.ns;
      s->c_fact_PH = c->FP.S.c_fact;
    }
    s->t_symbolic_s = c->t_symbolic;
    s->t_factor_s = c->t_factor;
    s->t_factor_ph_s = c->ph_refactors ? c->t_factor_ph / (double)c->ph_refactors : 0.0;
    const double n = (double)c->n, m1 = (double)c->m1, m2 = (double)c->m2;
    s->pcg_bytes_per_iter = 16.0 * (double)S.nnz_L + 24.0 * (double)c->C.nnz() + 8.0 * (15.0 * m2 + 6.0 * (n + m1)) +
                            16.0 * (double)s->nnz_LPH;
    s->pcg_flops_per_iter = 4.0 * (double)S.nnz_L + 4.0 * (double)c->C.nnz() + 4.0 * (double)s->nnz_LPH;
    s->sweep_bytes_F = 8.0 * (double)S.nnz_L;
    s->fsolve_bytes_F = c->FF.sym_enabled || !c->factored
                            ? 8.0 * (2.0 * (double)(S.nnz_L - S.sym_true) + (double)S.sym_lower)
                            : 16.0 * (double)S.nnz_L;
    if (c->FF.d.flat)   // forest read as M (twice) and L11⁻¹ (twice) instead of L11, L21
      s->fsolve_bytes_F = 8.0 * ((double)S.sym_lower + 2.0 * (double)S.fl_msize + 2.0 * (double)S.fl_ci.size());
    s->sym_discrepancy = c->FF.sym_discrepancy;
    s->lvl_levels_F = S.lvl_cut;
    s->lvl_supernodes_F = S.lvl_blk.size();
    s->lvl_levels_PH = c->FP.S.lvl_cut;
    s->lvl_supernodes_PH = c->FP.S.lvl_blk.size();
    s->pi_enabled = c->FF.pi.enabled ? 1.0 : 0.0;
    s->pi_discrepancy = c->FF.pi_discrepancy;
    s->pi_levels = 0;
    for (int L = 0; c->FF.pi.enabled && L < c->FF.pi.nlev; ++L)
      s->pi_levels += c->FF.pi.lev_ptr[L + 1] > c->FF.pi.lev_ptr[L] ? 1 : 0;   // non-empty levels = launches per sweep
    s->pi_subtrees = c->FF.pi.enabled ? (double)c->FF.pi.st_n : 0.0;
    s->pi_fsolve_ms = c->FF.pi_ms[1];
    s->sweep_fsolve_ms = c->FF.pi_ms[0];
    s->sym_enabled = c->FF.sym_enabled ? 1.0 : 0.0;
    s->flat_discrepancy = c->FF.flat_discrepancy;
    s->flat_enabled = c->FF.d.flat ? 1.0 : 0.0;
    s->flat_nnz_M = (double)S.fl_msize;
    s->dense_w_enabled = c->dense_w ? 1.0 : 0.0;
    s->dense_w_discrepancy = c->dw_discrepancy;
    s->kf_bytes_W = c->dense_w ? 4.0 * (double)c->n * (double)(c->n + 1) * c->dw_share : 0.0;
    s->dense_finv_enabled = c->dense_finv ? 1.0 : 0.0;
    s->dense_finv_discrepancy = c->df_discrepancy;
  }
  return QP_OK;
}

int qp_ipm_last_system(qp_ctx* c, double* D, double* rnu, double* eps) {
  int rc = require(c, true);
  if (rc) return rc;
  if (c->ipm_k == 0) return fail(c, QP_ESTATE, "no IPM iteration has run");
  out_vec(c, D, c->Dk, c->m2);
  out_vec(c, rnu, c->rnu, c->m2);
  if (eps) *eps = c->last_eps;
  return sync_check(c, "qp_ipm_last_system");
}

int64_t qp_launch_count(const qp_ctx* c) { return c ? c->launches : -1; }

int qp_profile(qp_ctx* c, int32_t enable) {
  if (!c) return QP_EINVAL;
  c->harvest();
  c->prof = enable != 0;
  if (!enable) {
    std::memset(c->prof_ms, 0, sizeof(c->prof_ms));
    std::memset(c->prof_cnt, 0, sizeof(c->prof_cnt));
  }
  return QP_OK;
}

int qp_profile_read(qp_ctx* c, double* ms, int64_t* count) {
  if (!c) return QP_EINVAL;
  c->harvest();
  for (int i = 0; i < 10; ++i) {
    if (ms) ms[i] = c->prof_ms[i];
    if (count) count[i] = c->prof_cnt[i];
  }
  return QP_OK;
}

// Debug: sweep instrumentation of the F factor. enable=1 resets and turns it on;
// enable=0 copies [2 sweeps][8 task types][count, wait ns, busy ns, first, last] into out (80 int64).
// QPB_TRACE_PH=1 selects the P_H factor's sweeps instead of F's (debug only).
static bool trace_ph(qp_ctx* c) {
  const char* e = getenv("QPB_TRACE_PH");
  return e && atoi(e) != 0 && c->FP.tprof_buf != nullptr;
}

int qp_debug_sweep_profile(qp_ctx* c, int32_t enable, int64_t* out) {
  if (!c || !c->factored) return QP_ESTATE;
  Factor& F = trace_ph(c) ? c->FP : c->FF;
  if (enable) {
    std::vector<unsigned long long> init(80 + 12 * F.d.ttrace_cap, 0);
    for (int i = 0; i < 16; ++i) init[i * 5 + 3] = ~0ull;
    cudaMemcpyAsync(F.tprof_buf, init.data(), init.size() * 8, cudaMemcpyHostToDevice, c->stream);
    F.d.tprof = F.tprof_buf;
  } else {
    if (out) cudaMemcpyAsync(out, F.tprof_buf, 80 * 8, cudaMemcpyDeviceToHost, c->stream);
    F.d.tprof = nullptr;
  }
  return sync_check(c, "qp_debug_sweep_profile");
}

// Debug: per-task trace of the last profiled sweeps (after qp_debug_sweep_profile(…, 0)).
// out[cap][6] = [task | smid << 32, start, dependency met, marker a, marker b, end] (ns) by ticket; the
// number of records written (the sweep's task count) or a negative status.
int64_t qp_debug_sweep_trace(qp_ctx* c, int32_t sweep, int64_t* out, int64_t cap) {
  if (!c || !c->factored || sweep < 0 || sweep > 1) return QP_ESTATE;
  Factor& F = trace_ph(c) ? c->FP : c->FF;
  const int64_t n = std::min<int64_t>(cap, sweep == 0 ? F.d.n_fwd_tasks : F.d.n_bwd_tasks);
  if (n > 0 && out)
    cudaMemcpyAsync(out, F.tprof_buf + 80 + sweep * F.d.ttrace_cap * 6, n * 48, cudaMemcpyDeviceToHost, c->stream);
  int st = sync_check(c, "qp_debug_sweep_trace");
  return st != QP_OK ? st : n;
}

// Debug: launch timeline of the instrumented kernels (kernels.cuh TL_K / TL_RING).  enable = 1 allocates
// (once), resets and turns it on; enable = 0 copies the buffer to out (host, 2·TL_K + 2·TL_K·TL_RING uint64)
// and turns it off.  Returns the number of words, or a negative status.
int64_t qp_debug_timeline(qp_ctx* c, int32_t enable, int64_t* out, int64_t cap) {
  if (!c) return QP_EINVAL;
  const int64_t words = 2 * TL_K + 2 * (int64_t)TL_K * TL_RING;
  if (enable) {
    if (!c->tl_buf) {
      if (cudaMalloc(&c->tl_buf, words * 8) != cudaSuccess) return fail(c, QP_ENOMEM, "timeline buffer");
    }
    std::vector<unsigned long long> init(words, 0ull);
    for (int64_t i = 2 * TL_K; i < 2 * TL_K + (int64_t)TL_K * TL_RING; ++i) init[i] = ~0ull;
    cudaMemcpyAsync(c->tl_buf, init.data(), words * 8, cudaMemcpyHostToDevice, c->stream);
    cudaStreamSynchronize(c->stream);
    timeline_enable(c->tl_buf);
    int st = sync_check(c, "qp_debug_timeline");
    return st != QP_OK ? st : words;
  }
  if (!c->tl_buf) return QP_ESTATE;
  cudaStreamSynchronize(c->stream);
  timeline_enable(nullptr);
  if (out) cudaMemcpy(out, c->tl_buf, std::min(cap, words) * 8, cudaMemcpyDeviceToHost);
  int st = sync_check(c, "qp_debug_timeline");
  return st != QP_OK ? st : words;
}

int qp_partition_rows(const int64_t* indptr, int64_t m2, int32_t world, int64_t* bounds) {
  if (!indptr || !bounds || m2 < 0 || world < 1) return QP_EINVAL;
  partition_rows(indptr, m2, world, bounds);
  return QP_OK;
}

int qp_get_partition(qp_ctx* c, int64_t* row0, int64_t* row1, int64_t* m2_global) {
  if (!c) return QP_EINVAL;
  if (row0) *row0 = c->row0;
  if (row1) *row1 = c->row1;
  if (m2_global) *m2_global = c->m2_global;
  return QP_OK;
}

int qp_nccl_unique_id(void* out) {
  if (!out) return QP_EINVAL;
  NcclApi& api = nccl_api();
  if (!api.ok) return QP_ENCCL;
  ncclUniqueId uid;
  if (api.get_unique_id(&uid) != ncclSuccess) return QP_ENCCL;
  std::memcpy(out, &uid, sizeof(uid));
  return QP_OK;
}

const char* qp_last_error(const qp_ctx* c) { return c ? c->err.c_str() : "NULL context"; }

void qp_free(qp_ctx* c) { delete c; }

}  // extern "C"
