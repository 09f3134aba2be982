// sm_100a fp64 kernels for the single-factorization inexact IPM (arXiv 2104.12916).
//
//  * multifrontal numeric LDLᵀ / Cholesky (setup of F; P_H refactor
//    every IPM iteration): assemble → extend-add → per-level blocked
//    partial factorization (DIAG / PANEL / UPDATE tile kernels), deterministic
//    owner-computes, no atomics;
//  * forward / backward triangular sweeps with L (c_trsv) as persistent
//    task-graph kernels: tasks are claimed from a ticket counter in topological
//    order, dependencies are tracked with per-block counters/flags, so there is
//    no level barrier; the K_F product's Cᵀp SpMV is fused into the
//    forward sweep's diagonal tasks;
//  * K_F's q = D∘p − C·w SpMV with the pᵀq reduction, fused PCG vector updates
//    with deterministic warp-shuffle + block + last-block reductions
//    (P:L284–285);
//  * IPM rhs / r_ν / recovery / Δs / step kernels (P:L65–69, P:L473–505,
//    P:L727–752).
#include <atomic>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
#include "kernels.cuh"

#include <cfloat>
#include <cmath>
#include <algorithm>
#include <cstdlib>

namespace qpb {

// ------------------------------------------------------------------------- helpers
__device__ __forceinline__ unsigned ld_acq_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acq_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long atom_acqrel_add_u64(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
// Programmatic dependent launch (the level-product chain): wait for the previous grid in the stream to
// complete and flush, then let the next grid's CTAs be scheduled as this grid's CTAs drain (they block in
// their own grid_dep_wait).  Both are no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// Block reduction (NT threads); result valid in every thread.
template <int OP>
__device__ double block_reduce(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = OP == 0 ? warp_sum(v) : (OP == 1 ? warp_max(v) : warp_min(v));
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double init = OP == 0 ? 0.0 : (OP == 1 ? -DBL_MAX : DBL_MAX);
  v = (lane < NT / 32) ? sh[lane] : init;
  v = OP == 0 ? warp_sum(v) : (OP == 1 ? warp_max(v) : warp_min(v));
  return v;
}
// Last-block detection after each block stored its partials.
__device__ bool is_last_block(unsigned int* arrive) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(arrive, 1u) == gridDim.x - 1);
  __syncthreads();
  return last;
}
// Deterministic sum of partial[0..n) by one block (fixed assignment).
template <int OP>
__device__ double reduce_partials(const double* part, int n, double* sh) {
  double init = OP == 0 ? 0.0 : (OP == 1 ? -DBL_MAX : DBL_MAX);
  double v = init;
  for (int i = threadIdx.x; i < n; i += NT) {
    double x = __ldcg(part + i);
    v = OP == 0 ? v + x : (OP == 1 ? fmax(v, x) : fmin(v, x));
  }
  return block_reduce<OP>(v, sh);
}
// One row of a CSR product, B entries per batch so their index, value and gather loads overlap
// (short rows — C has 4–6 entries per row, Cᵀ about 12 — then cost one dependent load round).
template <int B = 4>
__device__ __forceinline__ double csr_dot(const DevCSR& M, int64_t row, const double* x) {
  double s = 0.0;
  const int64_t q0 = M.p[row], q1 = M.p[row + 1];
  for (int64_t q = q0; q < q1; q += B) {
    double v[B];
    int32_t c[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const bool ok = q + u < q1;
      v[u] = ok ? M.v[q + u] : 0.0;
      c[u] = ok ? M.i[q + u] : 0;
    }
#pragma unroll
    for (int u = 0; u < B; ++u) s += v[u] * __ldg(x + c[u]);
  }
  return s;
}
// Front tile boundaries: pivot blocks of 64, then the update rows in tiles of 64.
__device__ __forceinline__ int64_t tile_begin(int64_t t, int64_t nk, int64_t w, int64_t m) {
  int64_t v = t < nk ? (int64_t)MF_BW * t : w + (int64_t)MF_BW * (t - nk);
  return v < m ? v : m;
}
__device__ __forceinline__ int find_seg(const int64_t* pref, int n, int64_t x) {
  int lo = 0, hi = n - 1;  // largest a with pref[a] <= x
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (pref[mid] <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// 8-byte global→shared asynchronous copies (zero fill when !ok)
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int n = ok ? 8 : 0;   // src-size 0 ⇒ zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(n));
}
// 16-byte copy (two rows of one column) when the global address is 16-byte aligned and both rows are in
// range; otherwise two 8-byte copies (zero fill for rows out of range)
__device__ __forceinline__ void cp_async_pair(double* smem, const double* gmem, bool ok0, bool ok1) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  if (ok0 && ok1 && ((reinterpret_cast<uintptr_t>(gmem) & 15) == 0)) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(ok0 ? 8 : 0));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa + 8), "l"(ok1 ? gmem + 1 : gmem), "r"(ok1 ? 8 : 0));
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// ------------------------------------------------------------------------- multifrontal
__global__ void k_mf_zero_fronts(DevFactor F, int64_t fr_off, int n_fr, int64_t total) {
  const int32_t* fr = F.lev_fronts + fr_off;
  const int64_t* zp = F.lev_zpref + fr_off;
  for (int64_t e = blockIdx.x * (int64_t)NT + threadIdx.x; e < total; e += (int64_t)gridDim.x * NT) {
    const int a = find_seg(zp, n_fr + 1, e);
    F.ws[F.front_off[fr[a]] + (e - zp[a])] = 0.0;
  }
}

__global__ void k_mf_assemble(DevFactor F, int64_t off, int64_t n, const double* src_vals, const double* D,
                              const int64_t* perm) {
  for (int64_t e = off + blockIdx.x * (int64_t)NT + threadIdx.x; e < off + n; e += (int64_t)gridDim.x * NT) {
    double v = F.asm_val[e];
    if (src_vals != nullptr) {
      int64_t s = F.asm_src[e];
      v = s >= 0 ? src_vals[s] : 0.0;
    }
    if (D != nullptr) {
      const int32_t c = F.asm_diag[e];
      if (c >= 0) v += D[perm[c]];
    }
    F.ws[F.asm_dst[e]] = v;
  }
}

// One warp per (parent front, parent column) group; children in fixed order.
__global__ void k_mf_extend_add(DevFactor F, int64_t grp_off, int64_t n_grp) {
  const int lane = threadIdx.x & 31;
  const int64_t g = grp_off + (blockIdx.x * (int64_t)NT + threadIdx.x) / 32;
  if (g >= grp_off + n_grp) return;
  const int32_t P = F.grp_P[g];
  const int64_t mP = F.sn_rowptr[P + 1] - F.sn_rowptr[P];
  double* col = F.ws + F.front_off[P] + (int64_t)F.grp_pc[g] * mP;
  for (int64_t e = F.grp_ptr[g]; e < F.grp_ptr[g + 1]; ++e) {
    const int32_t K = F.grp_K[e];
    const int64_t j = F.grp_j[e];
    const int64_t mK = F.sn_rowptr[K + 1] - F.sn_rowptr[K];
    const int64_t wK = F.sn_start[K + 1] - F.sn_start[K];
    const int32_t* ri = F.relind + F.relind_off[K] - wK;
    const double* u = F.ws + F.front_off[K] + j * mK;
    for (int64_t i = j + lane; i < mK; i += 32) col[ri[i]] += u[i];
  }
}

// DIAG: LDLᵀ of the 64×64 pivot tile (static 1×1 pivots), sign check, L⁻¹.
__global__ void __launch_bounds__(NT) k_mf_diag(DevFactor F, int k, int64_t act_off) {
  extern __shared__ double dsm[];
  double* a = dsm;
  double* xi = dsm + 64 * 65;
  const int J = F.act[act_off + blockIdx.x];
  const int64_t c0 = F.sn_start[J], w = F.sn_start[J + 1] - c0;
  const int64_t m = F.sn_rowptr[J + 1] - F.sn_rowptr[J];
  const int64_t fo = F.front_off[J];
  const int64_t p0 = (int64_t)MF_BW * k;
  const int wk = (int)(w - p0 < MF_BW ? w - p0 : MF_BW);
  const int b = F.sn_blk0[J] + k;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < wk * wk; idx += NT) {
    int c = idx / wk, r = idx % wk;
    a[c * 65 + r] = F.ws[fo + (p0 + c) * m + p0 + r];
    xi[c * 65 + r] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int j = 0; j < wk; ++j) {
    const double d = a[j * 65 + j];
    if (tid == 0) {
      F.Dpiv[c0 + p0 + j] = d;
      const signed char sg = F.pivsign[c0 + p0 + j];
      if (!(isfinite(d)) || d == 0.0 || (sg < 0 && d > 0.0) || (sg > 0 && d < 0.0)) atomicExch(F.status, 1);
    }
    const int rem = wk - j - 1;
    const double inv = 1.0 / d;
    for (int idx = tid; idx < rem * rem; idx += NT) {
      int i = j + 1 + idx % rem, c = j + 1 + idx / rem;
      if (c <= i) a[c * 65 + i] -= a[j * 65 + i] * a[j * 65 + c] * inv;
    }
    __syncthreads();
    for (int i = j + 1 + tid; i < wk; i += NT) a[j * 65 + i] *= inv;
    __syncthreads();
  }
  // X = L⁻¹ (unit lower) by column-oriented forward substitution
  for (int j = 0; j + 1 < wk; ++j) {
    const int rem = wk - j - 1;
    for (int idx = tid; idx < rem * (j + 1); idx += NT) {
      int i = j + 1 + idx % rem, c = idx / rem;
      xi[c * 65 + i] -= a[j * 65 + i] * xi[c * 65 + j];
    }
    __syncthreads();
  }
  double* inv = F.fstore + F.blk_inv[b];
  for (int idx = tid; idx < wk * wk; idx += NT) {
    int c = idx / wk, r = idx % wk;
    inv[idx] = r >= c ? xi[c * 65 + r] : 0.0;
  }
}

// PANEL: L_tk = A_tk · L_kk⁻ᵀ · D_k⁻¹ for the row tiles below the pivot block.
__global__ void __launch_bounds__(NT) k_mf_panel(DevFactor F, int k, int64_t act_off, int n_act,
                                                 int64_t pref_off) {
  extern __shared__ double dsm[];
  double* Ls = dsm;
  double* At = dsm + 64 * 65;
  double* Dk = dsm + 2 * 64 * 65;
  const int64_t* pref = F.pan_pref + pref_off;
  const int a = find_seg(pref, n_act + 1, blockIdx.x);
  const int J = F.act[act_off + a];
  const int64_t c0 = F.sn_start[J], w = F.sn_start[J + 1] - c0;
  const int64_t m = F.sn_rowptr[J + 1] - F.sn_rowptr[J];
  const int64_t fo = F.front_off[J];
  const int64_t nk = (w + MF_BW - 1) / MF_BW;
  const int64_t t = k + 1 + (blockIdx.x - pref[a]);
  const int64_t p0 = (int64_t)MF_BW * k;
  const int wk = (int)(w - p0 < MF_BW ? w - p0 : MF_BW);
  const int b = F.sn_blk0[J] + k;
  const int64_t tb = tile_begin(t, nk, w, m), te = tile_begin(t + 1, nk, w, m);
  const int R = (int)(te - tb);
  const int tid = threadIdx.x;
  const double* inv = F.fstore + F.blk_inv[b];
  for (int idx = tid; idx < wk * wk; idx += NT) {
    int c = idx / wk, r = idx % wk;
    Ls[c * 65 + r] = inv[idx];
  }
  for (int idx = tid; idx < R * wk; idx += NT) {
    int c = idx / R, r = idx % R;
    At[c * 65 + r] = F.ws[fo + (p0 + c) * m + tb + r];
  }
  if (tid < wk) Dk[tid] = F.Dpiv[c0 + p0 + tid];
  __syncthreads();
  const int64_t noff = F.blk_noff[b];
  double* L = F.fstore + F.blk_off[b] + (tb - (p0 + wk));
  for (int idx = tid; idx < R * wk; idx += NT) {
    int r = idx % R, c = idx / R;
    double s = 0.0;
    for (int j = 0; j <= c; ++j) s += At[j * 65 + r] * Ls[j * 65 + c];  // Linv(c, j)
    L[r + (int64_t)c * noff] = s / Dk[c];
  }
}

// UPDATE: A_ij −= L_ik D_k L_jkᵀ on the trailing tiles (i ≥ j > k) of each front.
// UPDATE A_ij −= L_ik D_k L_jkᵀ over the trailing lower triangle of each active front: one 64×64 tile
// per 256-thread CTA, 4×4 outputs per thread (rows tx·2 + {0,1} + {0,32}: a warp's stores cover 32
// consecutive rows of a column; columns likewise from ty) so
// the fragments are conflict-free 128-bit shared loads (4 per 16 DFMA), the ≤ 64 pivot columns staged
// by cp.async in double-buffered chunks of 16 (≈ 80 registers: 3 CTAs per SM overlap their epilogues),
// D_k applied to the column operand once per landed chunk in shared memory.
// mode 1: block k on the tiles i ≥ j ≥ k+1; 2: block k on the column strip j = k+1 (i ≥ k+1);
// 3: blocks k and k+1 (≤ 128 pivot columns) on the tiles i ≥ j ≥ k+2.
__global__ void __launch_bounds__(NT) k_mf_update(DevFactor F, int k, int k0g, int mode, int64_t act_off, int n_act,
                                                  int64_t pref_off) {
  constexpr int KC = 16, LD = 64 + 4;
  __shared__ __align__(16) double As[2][KC * LD];
  __shared__ __align__(16) double Bs[2][KC * LD];
  __shared__ double Dk[4 * MF_BW];
  const int64_t* pref = F.upd_pref + pref_off;
  const int a = find_seg(pref, n_act + 1, blockIdx.x);
  const int J = F.act[act_off + a];
  const int64_t c0 = F.sn_start[J], w = F.sn_start[J + 1] - c0;
  const int64_t m = F.sn_rowptr[J + 1] - F.sn_rowptr[J];
  const int64_t fo = F.front_off[J];
  const int64_t nk = (w + MF_BW - 1) / MF_BW;
  const int64_t ntile = nk + (m - w + MF_BW - 1) / MF_BW;
  const int64_t e = min((int64_t)k0g + F.mf_group, nk) - 1;   // last pivot block of this front's group
  int64_t q = blockIdx.x - pref[a];
  int64_t ti, tj;
  int kfirst, nblk;   // pivot blocks kfirst .. kfirst + nblk − 1 are applied
  if (mode == 2) {    // band: block k on block columns k+1 .. e, rows ≥ the column
    tj = k + 1;
    while (q >= ntile - tj) {
      q -= ntile - tj;
      ++tj;
    }
    ti = tj + q;
    kfirst = k;
    nblk = 1;
  } else {            // trailing triangle from block column e+1, all the group's blocks
    int64_t ii = (int64_t)((sqrt(8.0 * (double)q + 1.0) - 1.0) * 0.5);
    while (ii * (ii + 1) / 2 > q) --ii;
    while ((ii + 1) * (ii + 2) / 2 <= q) ++ii;
    const int64_t jj = q - ii * (ii + 1) / 2;
    ti = e + 1 + ii;
    tj = e + 1 + jj;
    kfirst = k0g;
    nblk = (int)(e - k0g + 1);
  }
  const int64_t p0 = (int64_t)MF_BW * kfirst;
  const int kt = (int)(min((int64_t)MF_BW * (kfirst + nblk), w) - p0);   // pivot columns applied
  const int b0 = F.sn_blk0[J] + kfirst;
  const int64_t ib = tile_begin(ti, nk, w, m), ie = tile_begin(ti + 1, nk, w, m);
  const int64_t jb = tile_begin(tj, nk, w, m), je = tile_begin(tj + 1, nk, w, m);
  const int Ri = (int)(ie - ib), Rj = (int)(je - jb);
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  if (tid < kt) Dk[tid] = F.Dpiv[c0 + p0 + tid];
  {   // pull the C tile into L2 now so the read-modify-write epilogue does not wait on HBM
    const int cc = tid >> 2, seg = tid & 3;   // 64 columns × 4 lines of 16 doubles
    if (cc < Rj && seg * 16 < Ri) prefetch_l2(F.ws + fo + (jb + cc) * m + ib + seg * 16);
  }
  auto load = [&](int buf, int kc0) {   // chunk of 16 pivot columns: block kfirst + kc0/64 (all but the last are 64 wide)
    const int bi = kc0 / MF_BW, kb = kc0 - bi * MF_BW;
    const int64_t pb = p0 + (int64_t)bi * MF_BW;
    const int wl = (int)(min(pb + MF_BW, w) - pb);
    const int64_t ns = F.blk_noff[b0 + bi];
    const double* Ls = F.fstore + F.blk_off[b0 + bi] - (pb + wl);   // index by front row
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = tid + NT * u;
      const int r = idx & 63, c = idx >> 6;
      const bool oka = r < Ri && kb + c < wl, okb = r < Rj && kb + c < wl;
      cp_async8(&As[buf][c * LD + r], Ls + (oka ? ib + r + (int64_t)(kb + c) * ns : 0), oka);
      cp_async8(&Bs[buf][c * LD + r], Ls + (okb ? jb + r + (int64_t)(kb + c) * ns : 0), okb);
    }
    cp_async_commit();
  };
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  load(0, 0);
  int buf = 0;
  for (int k0 = 0; k0 < kt; k0 += KC) {
    cp_async_wait_all();
    __syncthreads();
    {   // B ← B·D_k on the landed chunk (4 DMUL per thread per chunk instead of 4 per k-step)
      double* bw = Bs[buf];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = tid + NT * u;
        const int r = idx & 63, c = idx >> 6;
        const int kc = k0 + c;
        bw[c * LD + r] *= kc < kt ? Dk[kc] : 0.0;
      }
    }
    __syncthreads();
    if (k0 + KC < kt) load(buf ^ 1, k0 + KC);
    const double* as = As[buf];
    const double* bs = Bs[buf];
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      const double2 a0 = *reinterpret_cast<const double2*>(as + kk * LD + tx * 2);
      const double2 a1 = *reinterpret_cast<const double2*>(as + kk * LD + 32 + tx * 2);
      const double2 b0 = *reinterpret_cast<const double2*>(bs + kk * LD + ty * 2);
      const double2 b1 = *reinterpret_cast<const double2*>(bs + kk * LD + 32 + ty * 2);
      const double av[4] = {a0.x, a0.y, a1.x, a1.y};
      const double bv[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    buf ^= 1;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int s = (j >> 1) * 32 + ty * 2 + (j & 1);
    if (s >= Rj) continue;
    double* col = F.ws + fo + (jb + s) * m + ib;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = (i >> 1) * 32 + tx * 2 + (i & 1);
      if (r < Ri) col[r] -= acc[i][j];
    }
  }
}

// The same UPDATE with 128 threads, 8 × 4 outputs per thread (QPB_UPD=2, default; 1 = 256 threads, 4 × 4):
// c1 P_H refactor 1.120 -> 1.064 s.  Twice the FMAs per shared-memory
// fragment and per thread, for the FP64-pipe occupancy ncu found at 48 % with 4 × 4.
__global__ void __launch_bounds__(128) k_mf_update8x4(DevFactor F, int k, int k0g, int mode, int64_t act_off, int n_act,
                                                  int64_t pref_off) {
  constexpr int KC = 16, LD = 64 + 4;
  __shared__ __align__(16) double As[2][KC * LD];
  __shared__ __align__(16) double Bs[2][KC * LD];
  __shared__ double Dk[4 * MF_BW];
  const int64_t* pref = F.upd_pref + pref_off;
  const int a = find_seg(pref, n_act + 1, blockIdx.x);
  const int J = F.act[act_off + a];
  const int64_t c0 = F.sn_start[J], w = F.sn_start[J + 1] - c0;
  const int64_t m = F.sn_rowptr[J + 1] - F.sn_rowptr[J];
  const int64_t fo = F.front_off[J];
  const int64_t nk = (w + MF_BW - 1) / MF_BW;
  const int64_t ntile = nk + (m - w + MF_BW - 1) / MF_BW;
  const int64_t e = min((int64_t)k0g + F.mf_group, nk) - 1;   // last pivot block of this front's group
  int64_t q = blockIdx.x - pref[a];
  int64_t ti, tj;
  int kfirst, nblk;   // pivot blocks kfirst .. kfirst + nblk − 1 are applied
  if (mode == 2) {    // band: block k on block columns k+1 .. e, rows ≥ the column
    tj = k + 1;
    while (q >= ntile - tj) {
      q -= ntile - tj;
      ++tj;
    }
    ti = tj + q;
    kfirst = k;
    nblk = 1;
  } else {            // trailing triangle from block column e+1, all the group's blocks
    int64_t ii = (int64_t)((sqrt(8.0 * (double)q + 1.0) - 1.0) * 0.5);
    while (ii * (ii + 1) / 2 > q) --ii;
    while ((ii + 1) * (ii + 2) / 2 <= q) ++ii;
    const int64_t jj = q - ii * (ii + 1) / 2;
    ti = e + 1 + ii;
    tj = e + 1 + jj;
    kfirst = k0g;
    nblk = (int)(e - k0g + 1);
  }
  const int64_t p0 = (int64_t)MF_BW * kfirst;
  const int kt = (int)(min((int64_t)MF_BW * (kfirst + nblk), w) - p0);   // pivot columns applied
  const int b0 = F.sn_blk0[J] + kfirst;
  const int64_t ib = tile_begin(ti, nk, w, m), ie = tile_begin(ti + 1, nk, w, m);
  const int64_t jb = tile_begin(tj, nk, w, m), je = tile_begin(tj + 1, nk, w, m);
  const int Ri = (int)(ie - ib), Rj = (int)(je - jb);
  constexpr int UT = 128;
  const int tid = threadIdx.x, tx = tid & 7, ty = tid >> 3;
  for (int t = tid; t < kt; t += UT) Dk[t] = F.Dpiv[c0 + p0 + t];
  {   // pull the C tile into L2 now so the read-modify-write epilogue does not wait on HBM
    for (int t = tid; t < 256; t += UT) {   // 64 columns × 4 lines of 16 doubles
      const int cc = t >> 2, seg = t & 3;
      if (cc < Rj && seg * 16 < Ri) prefetch_l2(F.ws + fo + (jb + cc) * m + ib + seg * 16);
    }
  }
  auto load = [&](int buf, int kc0) {   // chunk of 16 pivot columns: block kfirst + kc0/64 (all but the last are 64 wide)
    const int bi = kc0 / MF_BW, kb = kc0 - bi * MF_BW;
    const int64_t pb = p0 + (int64_t)bi * MF_BW;
    const int wl = (int)(min(pb + MF_BW, w) - pb);
    const int64_t ns = F.blk_noff[b0 + bi];
    const double* Ls = F.fstore + F.blk_off[b0 + bi] - (pb + wl);   // index by front row
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = tid + UT * u;
      const int r = idx & 63, c = idx >> 6;
      const bool oka = r < Ri && kb + c < wl, okb = r < Rj && kb + c < wl;
      cp_async8(&As[buf][c * LD + r], Ls + (oka ? ib + r + (int64_t)(kb + c) * ns : 0), oka);
      cp_async8(&Bs[buf][c * LD + r], Ls + (okb ? jb + r + (int64_t)(kb + c) * ns : 0), okb);
    }
    cp_async_commit();
  };
  double acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  load(0, 0);
  int buf = 0;
  for (int k0 = 0; k0 < kt; k0 += KC) {
    cp_async_wait_all();
    __syncthreads();
    {   // B ← B·D_k on the landed chunk (4 DMUL per thread per chunk instead of 4 per k-step)
      double* bw = Bs[buf];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int idx = tid + UT * u;
        const int r = idx & 63, c = idx >> 6;
        const int kc = k0 + c;
        bw[c * LD + r] *= kc < kt ? Dk[kc] : 0.0;
      }
    }
    __syncthreads();
    if (k0 + KC < kt) load(buf ^ 1, k0 + KC);
    const double* as = As[buf];
    const double* bs = Bs[buf];
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      double av[8], bv[4];
#pragma unroll
      for (int i2 = 0; i2 < 4; ++i2) {   // rows 2tx + 16 i2 + {0, 1}
        const double2 a = *reinterpret_cast<const double2*>(as + kk * LD + 16 * i2 + tx * 2);
        av[2 * i2] = a.x;
        av[2 * i2 + 1] = a.y;
      }
#pragma unroll
      for (int j2 = 0; j2 < 2; ++j2) {   // columns 2ty + 32 j2 + {0, 1}
        const double2 b = *reinterpret_cast<const double2*>(bs + kk * LD + 32 * j2 + ty * 2);
        bv[2 * j2] = b.x;
        bv[2 * j2 + 1] = b.y;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    buf ^= 1;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int s = (j >> 1) * 32 + ty * 2 + (j & 1);
    if (s >= Rj) continue;
    double* col = F.ws + fo + (jb + s) * m + ib;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = (i >> 1) * 16 + tx * 2 + (i & 1);
      if (r < Ri) col[r] -= acc[i][j];
    }
  }
}

// Default UPDATE (QPB_UPD=4): k_mf_update8x4 with D_k applied to the B fragments in registers (4 DMUL per
// k-step) instead of a shared-memory scaling pass and its barrier per chunk, and 16-byte cp.async for row
// pairs where the column's address allows
// (c1 P_H refactor 1.064 → 1.008 s; ncu had the scaling pass at 17 % and the cp.async at 22 % of the
// instructions; 16-byte read-modify-writes in the epilogue were measured slower, 1.054 s).
__global__ void __launch_bounds__(128, 4) k_mf_update8x4r(DevFactor F, int k, int k0g, int mode, int64_t act_off, int n_act,
                                                  int64_t pref_off) {
  constexpr int KC = 16, LD = 64 + 4;
  __shared__ __align__(16) double As[2][KC * LD];
  __shared__ __align__(16) double Bs[2][KC * LD];
  __shared__ __align__(16) double Dk[4 * MF_BW + KC];
  const int64_t* pref = F.upd_pref + pref_off;
  const int a = find_seg(pref, n_act + 1, blockIdx.x);
  const int J = F.act[act_off + a];
  const int64_t c0 = F.sn_start[J], w = F.sn_start[J + 1] - c0;
  const int64_t m = F.sn_rowptr[J + 1] - F.sn_rowptr[J];
  const int64_t fo = F.front_off[J];
  const int64_t nk = (w + MF_BW - 1) / MF_BW;
  const int64_t ntile = nk + (m - w + MF_BW - 1) / MF_BW;
  const int64_t e = min((int64_t)k0g + F.mf_group, nk) - 1;   // last pivot block of this front's group
  int64_t q = blockIdx.x - pref[a];
  int64_t ti, tj;
  int kfirst, nblk;   // pivot blocks kfirst .. kfirst + nblk − 1 are applied
  if (mode == 2) {    // band: block k on block columns k+1 .. e, rows ≥ the column
    tj = k + 1;
    while (q >= ntile - tj) {
      q -= ntile - tj;
      ++tj;
    }
    ti = tj + q;
    kfirst = k;
    nblk = 1;
  } else {            // trailing triangle from block column e+1, all the group's blocks
    int64_t ii = (int64_t)((sqrt(8.0 * (double)q + 1.0) - 1.0) * 0.5);
    while (ii * (ii + 1) / 2 > q) --ii;
    while ((ii + 1) * (ii + 2) / 2 <= q) ++ii;
    const int64_t jj = q - ii * (ii + 1) / 2;
    ti = e + 1 + ii;
    tj = e + 1 + jj;
    kfirst = k0g;
    nblk = (int)(e - k0g + 1);
  }
  const int64_t p0 = (int64_t)MF_BW * kfirst;
  const int kt = (int)(min((int64_t)MF_BW * (kfirst + nblk), w) - p0);   // pivot columns applied
  const int b0 = F.sn_blk0[J] + kfirst;
  const int64_t ib = tile_begin(ti, nk, w, m), ie = tile_begin(ti + 1, nk, w, m);
  const int64_t jb = tile_begin(tj, nk, w, m), je = tile_begin(tj + 1, nk, w, m);
  const int Ri = (int)(ie - ib), Rj = (int)(je - jb);
  constexpr int UT = 128;
  const int tid = threadIdx.x, tx = tid & 7, ty = tid >> 3;
  for (int t = tid; t < 4 * MF_BW + KC; t += UT) Dk[t] = t < kt ? F.Dpiv[c0 + p0 + t] : 0.0;   // zero past kt
  {   // pull the C tile into L2 now so the read-modify-write epilogue does not wait on HBM
    for (int t = tid; t < 256; t += UT) {   // 64 columns × 4 lines of 16 doubles
      const int cc = t >> 2, seg = t & 3;
      if (cc < Rj && seg * 16 < Ri) prefetch_l2(F.ws + fo + (jb + cc) * m + ib + seg * 16);
    }
  }
  auto load = [&](int buf, int kc0) {   // chunk of 16 pivot columns: block kfirst + kc0/64 (all but the last are 64 wide)
    const int bi = kc0 / MF_BW, kb = kc0 - bi * MF_BW;
    const int64_t pb = p0 + (int64_t)bi * MF_BW;
    const int wl = (int)(min(pb + MF_BW, w) - pb);
    const int64_t ns = F.blk_noff[b0 + bi];
    const double* Ls = F.fstore + F.blk_off[b0 + bi] - (pb + wl);   // index by front row
#pragma unroll
    for (int u = 0; u < 4; ++u) {   // row pairs: 16-byte copies where the column's address allows
      const int idx = tid + UT * u;
      const int r = (idx & 31) * 2, c = idx >> 5;
      const bool okc = kb + c < wl;
      const int64_t co = (int64_t)(kb + c) * ns;
      cp_async_pair(&As[buf][c * LD + r], Ls + (okc ? ib + r + co : 0), okc && r < Ri, okc && r + 1 < Ri);
      cp_async_pair(&Bs[buf][c * LD + r], Ls + (okc ? jb + r + co : 0), okc && r < Rj, okc && r + 1 < Rj);
    }
    cp_async_commit();
  };
  double acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  load(0, 0);
  int buf = 0;
  for (int k0 = 0; k0 < kt; k0 += KC) {
    cp_async_wait_all();
    __syncthreads();
    if (k0 + KC < kt) load(buf ^ 1, k0 + KC);
    const double* as = As[buf];
    const double* bs = Bs[buf];
    double2 dk2;   // D_k of k-steps kk, kk + 1 (one 16-byte shared load per two k-steps)
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      double av[8], bv[4];
#pragma unroll
      for (int i2 = 0; i2 < 4; ++i2) {   // rows 2tx + 16 i2 + {0, 1}
        const double2 a = *reinterpret_cast<const double2*>(as + kk * LD + 16 * i2 + tx * 2);
        av[2 * i2] = a.x;
        av[2 * i2 + 1] = a.y;
      }
      const double dk = (kk & 1) ? dk2.y : (dk2 = *reinterpret_cast<const double2*>(Dk + k0 + kk)).x;   // D_k in registers
#pragma unroll
      for (int j2 = 0; j2 < 2; ++j2) {   // columns 2ty + 32 j2 + {0, 1}
        const double2 b = *reinterpret_cast<const double2*>(bs + kk * LD + 32 * j2 + ty * 2);
        bv[2 * j2] = b.x * dk;
        bv[2 * j2 + 1] = b.y * dk;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    buf ^= 1;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int s = (j >> 1) * 32 + ty * 2 + (j & 1);
    if (s >= Rj) continue;
    double* col = F.ws + fo + (jb + s) * m + ib;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = (i >> 1) * 16 + tx * 2 + (i & 1);
      if (r < Ri) col[r] -= acc[i][j];
    }
  }
}

void mf_assemble_level(const DevFactor& F, int64_t fr_off, int64_t n_fr, int64_t zero_total, int64_t asm_off,
                       int64_t n_asm, const double* src_vals, const double* D, const int64_t* perm, cudaStream_t s) {
  if (zero_total > 0) {
    int grid = (int)std::min<int64_t>((zero_total + NT - 1) / NT, 148 * 16);
    k_mf_zero_fronts<<<grid, NT, 0, s>>>(F, fr_off, (int)n_fr, zero_total);
  }
  if (n_asm > 0) {
    int grid = (int)std::min<int64_t>((n_asm + NT - 1) / NT, 148 * 16);
    k_mf_assemble<<<grid, NT, 0, s>>>(F, asm_off, n_asm, src_vals, D, perm);
  }
}
void mf_extend_add(const DevFactor& F, int64_t grp_off, int64_t n_grp, cudaStream_t s) {
  if (n_grp == 0) return;
  int64_t grid = (n_grp * 32 + NT - 1) / NT;
  k_mf_extend_add<<<(unsigned)grid, NT, 0, s>>>(F, grp_off, n_grp);
}
void mf_step(const DevFactor& F, int k, int k0, int kind, int64_t act_off, int n_act, int64_t pref_off,
             int64_t pan_total, int64_t upd_total, cudaStream_t s) {
  if (n_act == 0) return;
  // The shared-memory attribute is per device: set it once per device (several contexts on several
  // devices, or threads, may call this concurrently).
  static std::atomic<uint8_t> attr[64];
  const size_t sd = 2 * 64 * 65 * 8, sp = (2 * 64 * 65 + 64) * 8;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr[dev].load(std::memory_order_acquire)) {
    cudaFuncSetAttribute(k_mf_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sd);
    cudaFuncSetAttribute(k_mf_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp);
    if (dev >= 0 && dev < 64) attr[dev].store(1, std::memory_order_release);
  }
  if (kind == 0) {
    k_mf_diag<<<n_act, NT, sd, s>>>(F, k, act_off);
    if (pan_total > 0) k_mf_panel<<<(unsigned)pan_total, NT, sp, s>>>(F, k, act_off, n_act, pref_off);
  } else if (upd_total > 0) {
    static const int var = std::getenv("QPB_UPD") ? std::atoi(std::getenv("QPB_UPD")) : 4;
    if (var == 4) k_mf_update8x4r<<<(unsigned)upd_total, 128, 0, s>>>(F, k, k0, kind, act_off, n_act, pref_off);
    else if (var == 2) k_mf_update8x4<<<(unsigned)upd_total, 128, 0, s>>>(F, k, k0, kind, act_off, n_act, pref_off);
    else k_mf_update<<<(unsigned)upd_total, NT, 0, s>>>(F, k, k0, kind, act_off, n_act, pref_off);
  }
}

// ------------------------------------------------------------------------- triangular sweeps
// Task types (symbolic.h): 0 DIAG(b), 1 TILE(t), 2 PREP(b), 3 XTILE(x); index in the low 29 bits.
struct SweepShared {
  int task;
  unsigned ticket;
  unsigned epoch;
  double rhs[64];
  double y[64];
  double red[4 * 64];
  int rows[512];
  double xr[512];
};

__device__ __forceinline__ void spin_u64(const unsigned long long* p, unsigned long long target) {
  if (ld_acq_u64(p) >= target) return;
  unsigned ns = 8;
  while (ld_acq_u64(p) < target) {
    __nanosleep(ns);
    if (ns < 64) ns <<= 1;
  }
}
__device__ __forceinline__ void spin_u32(const unsigned* p, unsigned target) {
  if (ld_acq_u32(p) == target) return;
  unsigned ns = 8;
  while (ld_acq_u32(p) != target) {
    __nanosleep(ns);
    if (ns < 64) ns <<= 1;
  }
}

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Launch timeline (debug, qp_debug_timeline): for instrumented kernel k and its launch number s < TL_RING
// (later launches are counted, not recorded), the earliest block start and the latest block end
// (globaltimer ns), so the host can
// rebuild the per-launch durations AND the gaps between dependent launches (inside CUDA graphs too).
// Layout of g_tl: [TL_K launch counters][TL_K arrival counters][TL_K][TL_RING] starts, [TL_K][TL_RING] ends.
__device__ unsigned long long* g_tl = nullptr;
__device__ __forceinline__ unsigned tl_begin(int k) {
  unsigned long long* t = g_tl;
  if (t == nullptr || threadIdx.x != 0) return 0;
  const unsigned long long n = *((volatile unsigned long long*)(t + k));
  if (n >= TL_RING) return TL_RING;   // ring full: only the first TL_RING launches are kept
  atomicMin(t + 2 * TL_K + k * TL_RING + n, gtime());
  return (unsigned)n;
}
__device__ __forceinline__ void tl_end(int k, unsigned s) {
  unsigned long long* t = g_tl;
  if (t == nullptr) return;
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (s < TL_RING) atomicMax(t + 2 * TL_K + TL_K * TL_RING + k * TL_RING + s, gtime());
  __threadfence();
  if (atomicAdd(t + TL_K + k, 1ull) == gridDim.x - 1) {
    t[TL_K + k] = 0;
    __threadfence();
    atomicAdd(t + k, 1ull);
  }
}
void timeline_enable(unsigned long long* buf) { cudaMemcpyToSymbol(g_tl, &buf, sizeof(buf)); }

// instrumentation: per sweep (0 fwd, 1 bwd) and task type: count, wait ns, busy ns, first start, last end
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void tprof_add(unsigned long long* tp, int sweep, int type, unsigned long long t0,
                                          unsigned long long t1, unsigned long long t2, int task = 0,
                                          unsigned ticket = 0, int64_t cap = 0, unsigned long long ta = 0,
                                          unsigned long long tb = 0) {
  if (tp == nullptr || threadIdx.x != 0) return;
  if ((int64_t)ticket < cap) {  // per-task trace: [task | smid<<32, t0, t1, ta, tb, t2]
    unsigned long long* r = tp + 80 + ((int64_t)sweep * cap + ticket) * 6;
    r[0] = (unsigned long long)(unsigned)task | ((unsigned long long)smid() << 32);
    r[1] = t0;
    r[2] = t1;
    r[3] = ta;
    r[4] = tb;
    r[5] = t2;
  }
  unsigned long long* q = tp + (sweep * 8 + type) * 5;
  atomicAdd(q + 0, 1ull);
  atomicAdd(q + 1, t1 - t0);
  atomicAdd(q + 2, t2 - t1);
  atomicMin(q + 3, t0);
  atomicMax(q + 4, t2);
}

// Load a R×W column-major tile (leading dimension ld, R·W ≤ 4096) into smem with padding R+1.
__device__ __forceinline__ void load_tile(double* sm, const double* g, int R, int W, int64_t ld) {
  const int ldp = R + 1;
  const int n = R * W;
#pragma unroll 4
  for (int idx = threadIdx.x; idx < n; idx += NT) {
    const int c = idx / R, r = idx - c * R;
    sm[c * ldp + r] = __ldg(g + r + (int64_t)c * ld);
  }
}
// Prefetch the lines of a R×W column-major block into L2 (fire and forget).
__device__ __forceinline__ void prefetch_block(const double* g, int64_t R, int W, int64_t ld) {
  const int64_t lines = (R + 15) / 16;  // 128-byte lines per column
  for (int64_t e = threadIdx.x; e < lines * W; e += NT) {
    const int64_t c = e / lines, l = e - c * lines;
    prefetch_l2(g + l * 16 + c * ld);
  }
}
// out[r] = Σ_c T(r,c) v[c]   (T in smem, R×W, ld R+1); result for r < R in S.red[r] (after sync)
__device__ __forceinline__ void tile_gemv(const double* sm, int R, int W, const double* v, double* red) {
  const int ldp = R + 1;
  if (R <= 64) {
    const int r = threadIdx.x & 63, g = threadIdx.x >> 6;
    double s = 0.0;
    if (r < R)
      for (int c = g; c < W; c += 4) s += sm[c * ldp + r] * v[c];
    red[g * 64 + r] = s;
    __syncthreads();
    if (threadIdx.x < R) red[threadIdx.x] = red[threadIdx.x] + red[64 + threadIdx.x] + red[128 + threadIdx.x] +
                                            red[192 + threadIdx.x];
  } else {
    // caller handles R > 64 inline (rows per thread); not used with red
  }
  __syncthreads();
}
// out[c] = Σ_r T(r,c) v[r]   (transpose), result in red[c] for c < W (after sync)
__device__ __forceinline__ void tile_gemv_t(const double* sm, int R, int W, const double* v, double* red) {
  const int ldp = R + 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int P = W >= 8 ? 1 : 8 / W;
  __shared__ double part[64];
  for (int it = wid; it < W * P; it += NT / 32) {
    const int c = it / P, pr = it % P;
    double s = 0.0;
    for (int r = pr * 32 + lane; r < R; r += 32 * P) s += sm[c * ldp + r] * v[r];
    s = warp_sum(s);
    if (lane == 0) part[it] = s;
  }
  __syncthreads();
  if (threadIdx.x < W) {
    double s = 0.0;
    for (int pr = 0; pr < P; ++pr) s += part[threadIdx.x * P + pr];
    red[threadIdx.x] = s;
  }
  __syncthreads();
}

// Spin (by threads 0..n-1, one flag each) until every flag equals E; then barrier.
__device__ __forceinline__ void wait_flags(const unsigned* flags, int n, unsigned E) {
  if (threadIdx.x < n) spin_u32(flags + threadIdx.x, E);
}

// Streaming GEMV over a chunk of a big supernode's X_J (or X_Jᵀ): R ≤ 64 rows,
// ncol columns, leading dimension ld (multiple of 8, zero padding rows):
// red[512 + r] = Σ_c M(r, c)·v[c].  Lane l owns rows 2l, 2l+1 (128-bit loads);
// the 8 warps split the columns; 8 columns of loads in flight per thread.
__device__ __forceinline__ void xchunk_gemv(const double* __restrict__ M, int64_t ld, int R, int ncol,
                                            const double* v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool ok = 2 * lane < R;
  const double2* base = reinterpret_cast<const double2*>(M + 2 * lane);
  const int64_t ld2 = ld >> 1;
  double a0 = 0.0, a1 = 0.0;
  int c = wid;
  if (ok) {
    for (; c + 56 < ncol; c += 64) {
      double2 q[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) q[u] = __ldg(base + (int64_t)(c + 8 * u) * ld2);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double vc = v[c + 8 * u];
        a0 = fma(q[u].x, vc, a0);
        a1 = fma(q[u].y, vc, a1);
      }
    }
    for (; c < ncol; c += 8) {
      const double2 q = __ldg(base + (int64_t)c * ld2);
      const double vc = v[c];
      a0 = fma(q.x, vc, a0);
      a1 = fma(q.y, vc, a1);
    }
  }
  red[wid * 64 + 2 * lane] = a0;
  red[wid * 64 + 2 * lane + 1] = a1;
  __syncthreads();
  if (threadIdx.x < 64) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += red[k * 64 + threadIdx.x];
    red[512 + threadIdx.x] = s;
  }
  __syncthreads();
}

// L2 eviction-priority hints (createpolicy + ld.global.nc.L2::cache_hint): the root GEMV's one-pass
// stream of S⁻¹ (1.8 GB on c1) is marked evict_first so it does not push the flattened-forest arrays
// (re-read by every F-solve, ≈0.1 GB) out of L2; those are marked evict_last.
__device__ __forceinline__ uint64_t l2pol_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2pol_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2pol_normal() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ldg_pol(const double2* a, uint64_t pol) {
  double2 v;
  asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ldg_pol(const double* a, uint64_t pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ int32_t ldg_pol(const int32_t* a, uint64_t pol) {
  int32_t v;
  asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ int64_t ldg_pol(const int64_t* a, uint64_t pol) {
  int64_t v;
  asm("ld.global.nc.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}

// Symmetric-root chunk: rows R ≤ 64 of block I, ncol columns of blocks K0..;
// red[512 + r] = Σ_c S(r,c)·vK[c] (all columns) and colv[c] = Σ_r S(r,c)·vI[r] for c < ncol_t
// (the columns strictly before block I).  One read of the chunk serves both products.
template <int U = 8>
__device__ __forceinline__ void schunk_gemv(const double* __restrict__ M, int64_t ld, int R, int ncol, int ncol_t,
                                            const double* vK, const double* vI, double* red, double* colv,
                                            uint64_t pol) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool ok = 2 * lane < R;
  const double2* base = reinterpret_cast<const double2*>(M + 2 * lane);
  const int64_t ld2 = ld >> 1;
  const double vi0 = ok ? vI[2 * lane] : 0.0, vi1 = (2 * lane + 1 < R) ? vI[2 * lane + 1] : 0.0;
  double a0 = 0.0, a1 = 0.0;
  int c = wid;
  for (; c + 8 * (U - 1) < ncol; c += 8 * U) {
    double2 q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) q[u] = ok ? ldg_pol(base + (int64_t)(c + 8 * u) * ld2, pol) : make_double2(0.0, 0.0);
    double t[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double vc = vK[c + 8 * u];
      a0 = fma(q[u].x, vc, a0);
      a1 = fma(q[u].y, vc, a1);
      t[u] = q[u].x * vi0 + q[u].y * vi1;
    }
    if constexpr (U == 8) {
      // transpose-reduce: 8 column partials over 32 lanes in 4+2+1+1+1 shuffles (not 5·8); lane bits
      // 4,3,2 select the column a lane ends up holding, bits 1,0 finish the sum
      const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
      double a4[4], a2[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double recv = __shfl_xor_sync(0xffffffffu, h16 ? t[i] : t[i + 4], 16);
        a4[i] = (h16 ? t[i + 4] : t[i]) + recv;
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const double recv = __shfl_xor_sync(0xffffffffu, h8 ? a4[i] : a4[i + 2], 8);
        a2[i] = (h8 ? a4[i + 2] : a4[i]) + recv;
      }
      double a1 = (h4 ? a2[1] : a2[0]) + __shfl_xor_sync(0xffffffffu, h4 ? a2[0] : a2[1], 4);
      a1 += __shfl_xor_sync(0xffffffffu, a1, 2);
      a1 += __shfl_xor_sync(0xffffffffu, a1, 1);
      const int col = (h16 ? 4 : 0) + (h8 ? 2 : 0) + (h4 ? 1 : 0);
      if ((lane & 3) == 0 && c + 8 * col < ncol_t) colv[c + 8 * col] = a1;
    } else if constexpr (U == 16) {
      // the same transpose-reduce for 16 columns: 8+4+2+1 shuffles, bits 4..1 pick the column
      const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4, h2 = lane & 2;
      double a8[8], a4[4], a2[2];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        a8[i] = (h16 ? t[i + 8] : t[i]) + __shfl_xor_sync(0xffffffffu, h16 ? t[i] : t[i + 8], 16);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        a4[i] = (h8 ? a8[i + 4] : a8[i]) + __shfl_xor_sync(0xffffffffu, h8 ? a8[i] : a8[i + 4], 8);
#pragma unroll
      for (int i = 0; i < 2; ++i)
        a2[i] = (h4 ? a4[i + 2] : a4[i]) + __shfl_xor_sync(0xffffffffu, h4 ? a4[i] : a4[i + 2], 4);
      double a1 = (h2 ? a2[1] : a2[0]) + __shfl_xor_sync(0xffffffffu, h2 ? a2[0] : a2[1], 2);
      a1 += __shfl_xor_sync(0xffffffffu, a1, 1);
      const int col = (h16 ? 8 : 0) + (h8 ? 4 : 0) + (h4 ? 2 : 0) + (h2 ? 1 : 0);
      if ((lane & 1) == 0 && c + 8 * col < ncol_t) colv[c + 8 * col] = a1;
    } else {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int u = 0; u < U; ++u) t[u] += __shfl_xor_sync(0xffffffffu, t[u], o);
      if (lane == 0)
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (c + 8 * u < ncol_t) colv[c + 8 * u] = t[u];
    }
  }
  for (; c < ncol; c += 8) {
    const double2 q = ok ? ldg_pol(base + (int64_t)c * ld2, pol) : make_double2(0.0, 0.0);
    const double vc = vK[c];
    a0 = fma(q.x, vc, a0);
    a1 = fma(q.y, vc, a1);
    double t = warp_sum(q.x * vi0 + q.y * vi1);
    if (lane == 0 && c < ncol_t) colv[c] = t;
  }
  red[wid * 64 + 2 * lane] = a0;
  red[wid * 64 + 2 * lane + 1] = a1;
  __syncthreads();
  if (threadIdx.x < 64) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += red[k * 64 + threadIdx.x];
    red[512 + threadIdx.x] = s;
  }
  __syncthreads();
}

// Right-hand side of block columns c0..c0+wk-1 into rhs[] (visible after the caller's barrier):
// either the given vector, or (Cᵀp)_c gathered warp-per-column so all the CTA's loads are in flight.
__device__ __forceinline__ void sweep_rhs(const SweepRhs& R, int64_t c0, int wk, double* rhs) {
  const int tid = threadIdx.x;
  if (R.ct.p == nullptr) {
    if (tid < wk) {
      const int64_t c = c0 + tid;
      rhs[tid] = R.rhs[R.in_perm ? R.in_perm[c] : c];
    }
    return;
  }
  const int lane = tid & 31, wid = tid >> 5;
  for (int j = wid; j < wk; j += NT / 32) {
    const int64_t c = c0 + j;
    double v = 0.0;
    if (c < R.ct.nrows) {
      const int64_t q0 = __ldg(R.ct.p + c), q1 = __ldg(R.ct.p + c + 1);
      for (int64_t q = q0 + lane; q < q1; q += 32) v += __ldg(R.ct.v + q) * __ldg(R.p + __ldg(R.ct.i + q));
      v = warp_sum(v);
    }
    if (lane == 0) rhs[j] = v;
  }
}

// ---- SNW: one tiny single-block supernode per warp (w ≤ 32, noff ≤ 256, w·noff ≤ 1024)
// forward: y = L_bb⁻¹ (rhs − acc), acc[rows] += L_rows·y, then release the destination counters.
__device__ __forceinline__ void snw_forward(const DevFactor& F, const SweepRhs& R, double* x, int b, unsigned E,
                                            unsigned long long& ta, unsigned long long& tb) {
  const int lane = threadIdx.x & 31;
  const int J = F.blk_sn[b];
  const int wk = F.blk_w[b];
  const int64_t c0 = F.blk_col0[b];
  const int64_t noff = F.blk_noff[b];
  const double* L = F.fstore + F.blk_off[b];
  const double* inv = F.fstore + F.blk_inv[b];
  const int32_t* rows = F.sn_rows + F.blk_rows[b];
  // independent of the dependency: pull L_bb⁻¹, the L rows and their indices into L2
  for (int64_t e = (int64_t)lane * 16; e < (int64_t)wk * wk; e += 32 * 16) prefetch_l2(inv + e);
  for (int64_t e = (int64_t)lane * 16; e < noff * wk; e += 32 * 16) prefetch_l2(L + e);
  if (lane * 32 < noff) prefetch_l2(rows + lane * 32);
  double v = 0.0;
  if (lane < wk) {
    const int64_t c = c0 + lane;
    if (R.ct.p != nullptr) v = c < R.ct.nrows ? csr_dot(R.ct, c, R.p) : 0.0;
    else v = R.rhs[R.in_perm ? R.in_perm[c] : c];
  }
  if (lane == 0) spin_u64(F.cnt_f + J, (unsigned long long)E * (unsigned long long)F.fwd_expect[J]);
  __syncwarp();
  if (lane < wk) {
    double* ap = F.acc + c0 + lane;
    v -= __ldcg(ap);
    *ap = 0.0;
  }
  double y = 0.0;   // y_i = Σ_{j ≤ i} L⁻¹(i, j) v_j,  L⁻¹(i, j) = inv[j·wk + i]
#pragma unroll 8
  for (int j = 0; j < wk; ++j) {
    const double a = (lane < wk && j <= lane) ? __ldg(inv + j * wk + lane) : 0.0;
    y += a * __shfl_sync(0xffffffffu, v, j);
  }
  if (lane < wk) x[c0 + lane] = y;
  if (F.tprof && threadIdx.x == 0) ta = gtime();
  for (int r0 = 0; r0 < noff; r0 += 32) {
    const int r = r0 + lane;
    const bool ok = r < noff;
    const int32_t row = ok ? __ldg(rows + r) : 0;
    double s = 0.0;
#pragma unroll 8
    for (int c = 0; c < wk; ++c) {
      const double l = ok ? __ldg(L + r + (int64_t)c * noff) : 0.0;
      s += l * __shfl_sync(0xffffffffu, y, c);
    }
    if (ok) atomicAdd(F.acc + row, s);
  }
  // publish: every lane fences its own atomics into acc (in parallel, one fence latency), then the lanes
  // release the destination counters in parallel (the warp barrier orders all lanes' fenced writes
  // before every release).  One fence per destination by lane 0 cost ~11 µs per task on c2's leaves.
  if (F.blk_dptr[b + 1] > F.blk_dptr[b]) __threadfence();
  __syncwarp();
  if (F.tprof && threadIdx.x == 0) tb = gtime();
  for (int64_t k = F.blk_dptr[b] + lane; k < F.blk_dptr[b + 1]; k += 32)
    red_release_add_u64(F.cnt_f + F.blk_dest[k], 1ull);
}
// backward: t = L_rowsᵀ x_rows, x_b = L_bb⁻ᵀ (D⁻¹ y_b − t), publish the supernode.
__device__ __forceinline__ void snw_backward(const DevFactor& F, double* x, int b, unsigned E) {
  const int lane = threadIdx.x & 31;
  const int J = F.blk_sn[b];
  const int wk = F.blk_w[b];
  const int64_t c0 = F.blk_col0[b];
  const int64_t noff = F.blk_noff[b];
  const double* L = F.fstore + F.blk_off[b];
  const double* inv = F.fstore + F.blk_inv[b];
  const int32_t* rows = F.sn_rows + F.blk_rows[b];
  for (int64_t e = (int64_t)lane * 16; e < (int64_t)wk * wk; e += 32 * 16) prefetch_l2(inv + e);
  for (int64_t e = (int64_t)lane * 16; e < noff * wk; e += 32 * 16) prefetch_l2(L + e);
  const double dinv = lane < wk ? 1.0 / F.Dpiv[c0 + lane] : 0.0;
  for (int64_t k = F.blk_dptr[b] + lane; k < F.blk_dptr[b + 1]; k += 32) spin_u32(F.ready_sb + F.blk_dest[k], E);
  __syncwarp();
  double t = 0.0;   // lane j < wk: t_j = Σ_r L(r, j) x_{rows[r]}
  for (int r0 = 0; r0 < noff; r0 += 32) {
    const int r = r0 + lane;
    const double xr = r < noff ? __ldcg(x + __ldg(rows + r)) : 0.0;
#pragma unroll 4
    for (int j = 0; j < wk; ++j) {
      double p = r < noff ? __ldg(L + r + (int64_t)j * noff) * xr : 0.0;
      p = warp_sum(p);
      if (lane == j) t += p;
    }
  }
  double rhs = 0.0;
  if (lane < wk) rhs = __ldcg(x + c0 + lane) * dinv - t;
  double xi = 0.0;  // x_i = Σ_{j ≥ i} L⁻¹(j, i) rhs_j,  L⁻¹(j, i) = inv[i·wk + j]
#pragma unroll 8
  for (int j = 0; j < wk; ++j) {
    const double a = (lane < wk && j >= lane) ? __ldg(inv + lane * wk + j) : 0.0;
    xi += a * __shfl_sync(0xffffffffu, rhs, j);
  }
  if (lane < wk) x[c0 + lane] = xi;
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    st_rel_u32(F.ready_sb + J, E);
  }
}

// ---- leaf phase: one level of single-block supernodes (≤ G columns), a group of G lanes per supernode.
// Every load that does not depend on the solve — the right-hand side, the accumulator, the group's column of
// L_bb⁻¹ and the first G rows of L_rows with their indices — is issued before any arithmetic, so a supernode
// costs about one memory round trip.  Forward: y = L_bb⁻¹ (b − acc), acc[rows] += L_rows·y (the level below
// has finished: kernel order replaces the task graph's counters).
template <int G>
__device__ __forceinline__ unsigned lvl_mask() {
  return G == 32 ? 0xffffffffu : (0xffffu << (threadIdx.x & 16));
}
template <int G>
__global__ void __launch_bounds__(NT, G == 16 ? 3 : 2) k_lvl_fwd(DevFactor F, SweepRhs R, double* x, int64_t i0,
                                                                 int64_t i1) {
  if (R.done_flag != nullptr && *((volatile const int*)R.done_flag)) return;
  const unsigned tls = tl_begin(8);
  const int64_t i = i0 + ((int64_t)blockIdx.x * NT + threadIdx.x) / G;
  if (i < i1) {   // whole groups take the same branch
    const unsigned gm = lvl_mask<G>();
    const int lane = threadIdx.x & (G - 1);
    const int4 d0 = __ldg(F.lvl_desc + 2 * i), d1 = __ldg(F.lvl_desc + 2 * i + 1);   // one round trip
    const double* L = F.fstore + ((int64_t)(uint32_t)d0.x | ((int64_t)d0.y << 32));
    const double* inv = F.fstore + ((int64_t)(uint32_t)d0.z | ((int64_t)d0.w << 32));
    const int32_t* rows = F.sn_rows + ((int64_t)(uint32_t)d1.x | ((int64_t)d1.y << 32));
    const int64_t c0 = d1.z;
    const int wk = d1.w & 63, noff = (int)((unsigned)d1.w >> 6);
    if (noff > G)
      for (int64_t e = (int64_t)lane * 16; e < (int64_t)noff * wk; e += G * 16) prefetch_l2(L + e);
    double v = 0.0, a = 0.0;
    if (lane < wk) {
      const int64_t c = c0 + lane;
      if (R.ct.p != nullptr) v = c < R.ct.nrows ? csr_dot(R.ct, c, R.p) : 0.0;
      else v = R.rhs[R.in_perm ? R.in_perm[c] : c];
      a = __ldcg(F.acc + c);
    }
    double iv[G];   // lane i: L_bb⁻¹(i, j) = inv[j·wk + i], j ≤ i
#pragma unroll
    for (int j = 0; j < G; ++j) iv[j] = (j < wk && j <= lane && lane < wk) ? __ldg(inv + j * wk + lane) : 0.0;
    const bool rok = lane < noff;
    const int32_t row = rok ? __ldg(rows + lane) : 0;
    double lr[G];   // lane r: L(r, c)
#pragma unroll
    for (int c = 0; c < G; ++c) lr[c] = (c < wk && rok) ? __ldg(L + lane + (int64_t)c * noff) : 0.0;
    if (lane < wk) F.acc[c0 + lane] = 0.0;
    v -= a;
    double y = 0.0;
#pragma unroll
    for (int j = 0; j < G; ++j) y += iv[j] * __shfl_sync(gm, v, j, G);
    if (lane < wk) x[c0 + lane] = y;
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < G; ++c) s += lr[c] * __shfl_sync(gm, y, c, G);
    if (rok) atomicAdd(F.acc + row, s);
    for (int r0 = G; r0 < noff; r0 += G) {
      const int r = r0 + lane;
      const bool ok = r < noff;
      const int32_t rw = ok ? __ldg(rows + r) : 0;
      double s2 = 0.0;
#pragma unroll
      for (int c = 0; c < G; ++c) {
        const double l = (c < wk && ok) ? __ldg(L + r + (int64_t)c * noff) : 0.0;
        s2 += l * __shfl_sync(gm, y, c, G);
      }
      if (ok) atomicAdd(F.acc + rw, s2);
    }
  }
  tl_end(8, tls);
}
// Transpose-reduce over a group of G lanes: lane l ends with Σ_lanes t[l] (G−1 shuffles for G columns).
template <int G>
__device__ __forceinline__ double group_treduce(double (&t)[G], int lane, unsigned gm) {
#pragma unroll
  for (int h = G / 2; h >= 1; h >>= 1) {
    const bool up = lane & h;
#pragma unroll
    for (int k = 0; k < h; ++k) {
      const double send = up ? t[k] : t[k + h];
      const double keep = up ? t[k + h] : t[k];
      t[k] = keep + __shfl_xor_sync(gm, send, h, G);
    }
  }
  return t[0];
}
// Backward: t = L_rowsᵀ x_rows (the rows belong to higher levels, already final), x_b = L_bb⁻ᵀ (D⁻¹y_b − t).
// Fixed-order arithmetic (no atomics): bit-reproducible.
template <int G>
__global__ void __launch_bounds__(NT, G == 16 ? 3 : 2) k_lvl_bwd(DevFactor F, double* x, const int* done_flag,
                                                                 int64_t i0, int64_t i1) {
  if (done_flag != nullptr && *((volatile const int*)done_flag)) return;
  const unsigned tls = tl_begin(9);
  const int64_t i = i0 + ((int64_t)blockIdx.x * NT + threadIdx.x) / G;
  if (i < i1) {
    const unsigned gm = lvl_mask<G>();
    const int lane = threadIdx.x & (G - 1);
    const int4 d0 = __ldg(F.lvl_desc + 2 * i), d1 = __ldg(F.lvl_desc + 2 * i + 1);
    const double* L = F.fstore + ((int64_t)(uint32_t)d0.x | ((int64_t)d0.y << 32));
    const double* inv = F.fstore + ((int64_t)(uint32_t)d0.z | ((int64_t)d0.w << 32));
    const int32_t* rows = F.sn_rows + ((int64_t)(uint32_t)d1.x | ((int64_t)d1.y << 32));
    const int64_t c0 = d1.z;
    const int wk = d1.w & 63, noff = (int)((unsigned)d1.w >> 6);
    if (noff > G)
      for (int64_t e = (int64_t)lane * 16; e < (int64_t)noff * wk; e += G * 16) prefetch_l2(L + e);
    double yv = 0.0, dinv = 0.0;
    if (lane < wk) {
      yv = __ldcg(x + c0 + lane);
      dinv = 1.0 / __ldg(F.Dpiv + c0 + lane);
    }
    double ivt[G];   // lane i: L_bb⁻¹(j, i) = inv[i·wk + j], j ≥ i (one contiguous run per lane)
#pragma unroll
    for (int j = 0; j < G; ++j) ivt[j] = (j < wk && j >= lane && lane < wk) ? __ldg(inv + lane * wk + j) : 0.0;
    double t[G];
#pragma unroll
    for (int c = 0; c < G; ++c) t[c] = 0.0;
    for (int r0 = 0; r0 < noff; r0 += G) {
      const int r = r0 + lane;
      const bool ok = r < noff;
      const double xr = ok ? __ldcg(x + __ldg(rows + r)) : 0.0;
#pragma unroll
      for (int c = 0; c < G; ++c) t[c] += ((c < wk && ok) ? __ldg(L + r + (int64_t)c * noff) : 0.0) * xr;
    }
    const double tc = group_treduce<G>(t, lane, gm);
    const double rhs = lane < wk ? yv * dinv - tc : 0.0;
    double xi = 0.0;
#pragma unroll
    for (int j = 0; j < G; ++j) xi += ivt[j] * __shfl_sync(gm, rhs, j, G);
    if (lane < wk) x[c0 + lane] = xi;
  }
  tl_end(9, tls);
}

// Forward sweep L y = b (unit lower L, factor order); y written to x.
__global__ void __launch_bounds__(NT) k_trsv_fwd(DevFactor F, SweepRhs R, double* x) {
  extern __shared__ double sm[];
  __shared__ SweepShared S;
  const int tid = threadIdx.x;
  if (R.done_flag != nullptr && *((volatile const int*)R.done_flag)) return;
  if (tid == 0) S.epoch = *((volatile unsigned*)(F.sweep + 2)) + 1u;
  __syncthreads();
  const unsigned E = S.epoch;
  const unsigned tls = tl_begin(5);
  while (true) {
    if (tid == 0) {
      unsigned t = atomicAdd(F.sweep + 0, 1u);
      S.task = t < (unsigned)F.n_fwd_tasks ? F.fwd_tasks[t] : -1;
      S.ticket = t;
    }
    __syncthreads();
    const int task = S.task;
    __syncthreads();
    if (task < 0) break;
    const int type = task >> 28, idx = task & ((1 << 28) - 1);
    const unsigned long long t0 = F.tprof ? gtime() : 0ull;
    unsigned long long t1 = t0, ta = 0, tb = 0;
    if (type == 0 || type == 2) {
      // ---------------- DIAG(b) / PREP(b): v = b_b − Σ updates into supernode J
      const int b = idx;
      const int J = F.blk_sn[b];
      const int wk = F.blk_w[b];
      const int64_t c0 = F.blk_col0[b];
      if (type == 0) {
        const double* inv = F.fstore + F.blk_inv[b];
        for (int i2 = tid; i2 < wk * wk; i2 += NT) {
          int c = i2 / wk, r = i2 - c * wk;
          sm[c * 65 + r] = __ldg(inv + i2);
        }
      }
      sweep_rhs(R, c0, wk, S.rhs);
      if (tid == 0) {
        spin_u64(F.cnt_f + J, (unsigned long long)E * (unsigned long long)F.fwd_expect[J]);
        if (F.tprof) t1 = gtime();
      }
      __syncthreads();
      if (tid < wk) {
        double* ap = F.acc + c0 + tid;
        S.rhs[tid] -= __ldcg(ap);
        *ap = 0.0;
      }
      __syncthreads();
      if (type == 0) {
        const int i = tid & 63, g = tid >> 6;
        double s = 0.0;
        if (i < wk)
          for (int j = g; j <= i; j += 4) s += sm[j * 65 + i] * S.rhs[j];
        S.red[g * 64 + i] = s;
        __syncthreads();
        if (tid < wk) x[c0 + tid] = S.red[tid] + S.red[64 + tid] + S.red[128 + tid] + S.red[192 + tid];
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          st_rel_u32(F.ready_f + b, E);
        }
      } else {
        if (tid < wk) {
          F.vbuf[c0 + tid] = S.rhs[tid];
          x[c0 + tid] = 0.0;
        }
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          // keep the X-path counters in step when the symmetric root bypasses them
          if (F.use_sym && F.sn_sinv[J] >= 0) atomicAdd(F.cntx_f + b, (unsigned long long)F.xexp_f[b]);
          st_rel_u32(F.vready_f + b, E);
        }
      }
    } else if (type == 4) {
      // ---------------- SNF(b): small supernode in one task — y_b = L_bb⁻¹ v, then acc[rows] += L_rows·y_b
      const int b = idx;
      const int J = F.blk_sn[b];
      const int wk = F.blk_w[b];
      const int64_t c0 = F.blk_col0[b];
      const int64_t noff = F.blk_noff[b];
      const double* L = F.fstore + F.blk_off[b];
      const int32_t* rows = F.sn_rows + F.blk_rows[b];
      const int Rc = wk > 4 ? 4096 / wk : 1024;
      // independent of the dependency: L_bb⁻¹ → smem[0, 4160); a first L chunk (≤ 2048 doubles,
      // ≤ 512 rows) and its row indices → smem; otherwise the whole L block is prefetched into L2
      double* Ls = sm + 4160;
      const double* inv = F.fstore + F.blk_inv[b];
      for (int i2 = tid; i2 < wk * wk; i2 += NT) {
        int c = i2 / wk, r = i2 - c * wk;
        sm[c * 65 + r] = __ldg(inv + i2);
      }
      const int R0 = (int)(noff < Rc ? noff : Rc);
      const bool one_chunk = noff <= 512 && wk * (noff + 1) <= 1024;
      if (one_chunk) {
        for (int i2 = tid; i2 < wk * R0; i2 += NT) {
          int c = i2 / R0, r = i2 - c * R0;
          Ls[c * (R0 + 1) + r] = __ldg(L + r + (int64_t)c * noff);
        }
        for (int r = tid; r < R0; r += NT) S.rows[r] = __ldg(rows + r);
      } else {
        prefetch_block(L, noff, wk, noff);
        for (int64_t r = (int64_t)tid * 32; r < noff; r += (int64_t)NT * 32) prefetch_l2(rows + r);
      }
      sweep_rhs(R, c0, wk, S.rhs);
      if (tid == 0) {
        spin_u64(F.cnt_f + J, (unsigned long long)E * (unsigned long long)F.fwd_expect[J]);
        if (F.tprof) t1 = gtime();
      }
      __syncthreads();
      if (tid < wk) {
        double* ap = F.acc + c0 + tid;
        S.rhs[tid] -= __ldcg(ap);
        *ap = 0.0;
      }
      __syncthreads();
      {
        const int i = tid & 63, g = tid >> 6;
        double s = 0.0;
        if (i < wk)
          for (int j = g; j <= i; j += 4) s += sm[j * 65 + i] * S.rhs[j];
        S.red[g * 64 + i] = s;
      }
      __syncthreads();
      if (tid < wk) {
        const double yv = S.red[tid] + S.red[64 + tid] + S.red[128 + tid] + S.red[192 + tid];
        S.y[tid] = yv;
        x[c0 + tid] = yv;
      }
      __syncthreads();
      if (F.tprof && tid == 0) ta = gtime();
      if (one_chunk) {
        for (int r = tid; r < R0; r += NT) {
          double s = 0.0;
          for (int c = 0; c < wk; ++c) s += Ls[c * (R0 + 1) + r] * S.y[c];
          atomicAdd(F.acc + S.rows[r], s);
        }
      } else {
        for (int64_t r0 = 0; r0 < noff; r0 += Rc) {
          const int Rn = (int)(noff - r0 < Rc ? noff - r0 : Rc);
          __syncthreads();
          load_tile(sm, L + r0, Rn, wk, noff);
          __syncthreads();
          for (int r = tid; r < Rn; r += NT) {
            double s = 0.0;
            for (int c = 0; c < wk; ++c) s += sm[c * (Rn + 1) + r] * S.y[c];
            atomicAdd(F.acc + __ldg(rows + r0 + r), s);
          }
        }
      }
      __syncthreads();
      if (F.tprof && tid == 0) tb = gtime();
      for (int64_t k = F.blk_dptr[b] + tid; k < F.blk_dptr[b + 1]; k += NT) {
        __threadfence();
        red_release_add_u64(F.cnt_f + F.blk_dest[k], 1ull);
      }
    } else if (type == 7) {
      // ---------------- SNW: up to 8 tiny supernodes of one level, one warp each
      const int bw = F.snw_fwd[idx * 8 + (tid >> 5)];
      if (bw >= 0) snw_forward(F, R, x, bw, E, ta, tb);
    } else if (type == 5) {
      // ---------------- SCHUNK: symmetric root — x_I += S_IK v_K, x_K += S_IKᵀ v_I (K < I)
      const int bI = F.xt_bI[idx], bK = F.xt_bK[idx], nK = F.xt_nK[idx];
      const int J = F.blk_sn[bI];
      const int64_t cJ = F.sn_start[J];
      const int64_t rI = F.blk_col0[bI], cK = F.blk_col0[bK];
      const int Rn = F.blk_w[bI];
      const int ncol = (int)(F.blk_col0[bK + nK - 1] + F.blk_w[bK + nK - 1] - cK);
      const int ncol_t = (int)((rI < cK + ncol ? rI : cK + ncol) - cK);   // columns before block I
      if (tid < nK) spin_u32(F.vready_f + bK + tid, E);
      if (tid == 64) spin_u32(F.vready_f + bI, E);
      if (F.tprof && tid == 0) t1 = gtime();
      __syncthreads();
      double* vK = sm;              // ≤ 512
      double* vI = sm + 512;        // 64
      double* red = sm + 576;       // 8·64 + 64
      double* colv = sm + 576 + 576;  // ≤ 512
      for (int c = tid; c < ncol; c += NT) vK[c] = __ldcg(F.vbuf + cK + c);
      if (tid < Rn) vI[tid] = __ldcg(F.vbuf + rI + tid);
      __syncthreads();
      const int64_t ldx = F.sn_ldx[J];
      schunk_gemv(F.xinv + F.sn_sinv[J] + (rI - cJ) + (cK - cJ) * ldx, ldx, Rn, ncol, ncol_t, vK, vI, red, colv,
                  (F.l2hint & 1) ? l2pol_first() : l2pol_normal());
      if (tid < Rn) atomicAdd(x + rI + tid, red[512 + tid]);
      for (int c = tid; c < ncol_t; c += NT) atomicAdd(x + cK + c, colv[c]);
    } else if (type == 3) {
      // ---------------- XCHUNK: x[I] += X_{I,K0..K0+nK} · v[K0..]
      const int bI = F.xt_bI[idx], bK = F.xt_bK[idx], nK = F.xt_nK[idx];
      const int J = F.blk_sn[bI];
      const int64_t cJ = F.sn_start[J];
      const int64_t rI = F.blk_col0[bI], cK = F.blk_col0[bK];
      const int Rn = F.blk_w[bI];
      const int ncol = (int)(F.blk_col0[bK + nK - 1] + F.blk_w[bK + nK - 1] - cK);
      if (tid < nK) spin_u32(F.vready_f + bK + tid, E);
      if (tid == 64) spin_u32(F.vready_f + bI, E);
      if (F.tprof && tid == 0) t1 = gtime();
      __syncthreads();
      for (int c = tid; c < ncol; c += NT) sm[c] = __ldcg(F.vbuf + cK + c);
      __syncthreads();
      double* red = sm + 512;
      const int64_t ldx = F.sn_ldx[J];
      xchunk_gemv(F.xinv + F.sn_xinv[J] + (rI - cJ) + (cK - cJ) * ldx, ldx, Rn, ncol, sm, red);
      if (tid < Rn) atomicAdd(x + rI + tid, red[512 + tid]);
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        unsigned long long old = atomicAdd(F.cntx_f + bI, 1ull);
        if (old + 1 == (unsigned long long)E * (unsigned long long)F.xexp_f[bI]) {
          __threadfence();
          st_rel_u32(F.ready_f + bI, E);
        }
      }
    } else {
      // ---------------- TILE: acc[rows] += L_tile · y_b  (rows in the supernodes tile_dlist[tile_dptr[ti] ..])
      const int ti = idx;
      const int b = F.tile_blk[ti];
      const int wk = F.blk_w[b];
      const int Rn = F.tile_nr[ti];
      const int r0 = F.tile_r0[ti];
      const int64_t noff = F.blk_noff[b];
      const int64_t c0 = F.blk_col0[b];
      const bool longt = Rn * wk > 4096;   // a long tile of a full-width block: straight from global memory
      const double* Lt = F.fstore + F.blk_off[b] + r0;
      if (!longt) load_tile(sm, Lt, Rn, wk, noff);   // long tiles stream after the wait (an L2 prefetch of
      // 256 KB per task was evicted before use and doubled the DRAM reads)
      if (tid == 0) {
        spin_u32(F.ready_f + b, E);
        if (F.tprof) t1 = gtime();
      }
      __syncthreads();
      if (tid < wk) S.y[tid] = __ldcg(x + c0 + tid);
      __syncthreads();
      const int32_t* rows = F.sn_rows + F.blk_rows[b] + r0;
      if (longt) {
        // warp w: rows 64w + lane and 64w + 32 + lane; all 64 columns, 8 in flight
        const int lane = tid & 31, wid = tid >> 5;
        for (int rb = wid * 64; rb < Rn; rb += NT * 2) {
          const int ra = rb + lane, rc = rb + 32 + lane;
          double s0 = 0.0, s1 = 0.0;
#pragma unroll 8
          for (int c = 0; c < wk; ++c) {
            const double yc = S.y[c];
            if (ra < Rn) s0 += __ldg(Lt + ra + (int64_t)c * noff) * yc;
            if (rc < Rn) s1 += __ldg(Lt + rc + (int64_t)c * noff) * yc;
          }
          if (ra < Rn) atomicAdd(F.acc + rows[ra], s0);
          if (rc < Rn) atomicAdd(F.acc + rows[rc], s1);
        }
      } else if (Rn <= 64) {
        tile_gemv(sm, Rn, wk, S.y, S.red);
        if (tid < Rn) atomicAdd(F.acc + rows[tid], S.red[tid]);
      } else {
        const int ld = Rn + 1;
        for (int r = tid; r < Rn; r += NT) {
          double s = 0.0;
          for (int c = 0; c < wk; ++c) s += sm[c * ld + r] * S.y[c];
          atomicAdd(F.acc + rows[r], s);
        }
      }
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        for (int64_t q = F.tile_dptr[ti]; q < F.tile_dptr[ti + 1]; ++q) atomicAdd(F.cnt_f + F.tile_dlist[q], 1ull);
      }
    }
    if (F.tprof) tprof_add(F.tprof, 0, type, t0, t1, gtime(), task, S.ticket, F.ttrace_cap, ta, tb);
  }
  if (tid == 0) {
    unsigned d = atomicAdd(F.sweep + 1, 1u);
    if (d == gridDim.x - 1) {
      F.sweep[0] = 0u;
      F.sweep[1] = 0u;
      F.sweep[2] = E;
      __threadfence();
    }
  }
  tl_end(5, tls);
}

// Backward sweep Lᵀ x = D⁻¹ y (in place in x).
__global__ void __launch_bounds__(NT, 4) k_trsv_bwd(DevFactor F, double* x, const int* done_flag) {
  extern __shared__ double sm[];
  __shared__ SweepShared S;
  const int tid = threadIdx.x;
  if (done_flag != nullptr && *((volatile const int*)done_flag)) return;
  if (tid == 0) S.epoch = *((volatile unsigned*)(F.sweep + 3)) + 1u;
  __syncthreads();
  const unsigned E = S.epoch;
  const unsigned tls = tl_begin(6);
  while (true) {
    if (tid == 0) {
      unsigned t = atomicAdd(F.sweep + 0, 1u);
      S.task = t < (unsigned)F.n_bwd_tasks ? F.bwd_tasks[t] : -1;
      S.ticket = t;
    }
    __syncthreads();
    const int task = S.task;
    __syncthreads();
    if (task < 0) break;
    const int type = task >> 28, idx = task & ((1 << 28) - 1);
    const unsigned long long t0 = F.tprof ? gtime() : 0ull;
    unsigned long long t1 = t0, ta = 0, tb = 0;
    if (type == 0 || type == 2) {
      const int b = idx;
      const int wk = F.blk_w[b];
      const int64_t c0 = F.blk_col0[b];
      if (type == 0) {
        const double* inv = F.fstore + F.blk_inv[b];
        for (int i2 = tid; i2 < wk * wk; i2 += NT) {
          int c = i2 / wk, r = i2 - c * wk;
          sm[c * 65 + r] = __ldg(inv + i2);
        }
      }
      double dinv = 0.0;
      if (tid < wk) dinv = 1.0 / F.Dpiv[c0 + tid];
      if (tid == 0) {
        spin_u64(F.cnt_b + b, (unsigned long long)E * (unsigned long long)F.bwd_expect[b]);
        if (F.tprof) t1 = gtime();
      }
      __syncthreads();
      if (tid < wk) {
        double* tp = F.tacc + c0 + tid;
        S.rhs[tid] = __ldcg(x + c0 + tid) * dinv - __ldcg(tp);
        *tp = 0.0;
      }
      __syncthreads();
      if (type == 0) {
        const int i = tid & 63, g = tid >> 6;
        double s = 0.0;
        if (i < wk)
          for (int j = i + g; j < wk; j += 4) s += sm[i * 65 + j] * S.rhs[j];  // Linv(j, i)
        S.red[g * 64 + i] = s;
        __syncthreads();
        if (tid < wk) x[c0 + tid] = S.red[tid] + S.red[64 + tid] + S.red[128 + tid] + S.red[192 + tid];
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          st_rel_u32(F.ready_sb + F.blk_sn[b], E);
        }
      } else {
        if (tid < wk) {
          F.vbuf[c0 + tid] = S.rhs[tid];
          x[c0 + tid] = 0.0;
        }
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          st_rel_u32(F.vready_b + b, E);
        }
      }
    } else if (type == 4) {
      // ---------------- SNF(b) backward: t = L_rowsᵀ x_rows (gather), x_b = L_bb⁻ᵀ (D⁻¹ y_b − t)
      const int b = idx;
      const int J = F.blk_sn[b];
      const int wk = F.blk_w[b];
      const int64_t c0 = F.blk_col0[b];
      const int64_t noff = F.blk_noff[b];
      const double* L = F.fstore + F.blk_off[b];
      const int32_t* rows = F.sn_rows + F.blk_rows[b];
      double dinv = 0.0;
      if (tid < wk) dinv = 1.0 / F.Dpiv[c0 + tid];
      // independent of the dependencies: L_bb⁻¹, a single L chunk and its row indices → smem
      const bool one_chunk = noff <= 512 && wk * (noff + 1) <= 1024;
      const int R0 = (int)noff;
      double* Ls = sm + 4160;
      const double* inv = F.fstore + F.blk_inv[b];
      for (int i2 = tid; i2 < wk * wk; i2 += NT) {
        int c = i2 / wk, r = i2 - c * wk;
        sm[c * 65 + r] = __ldg(inv + i2);
      }
      if (one_chunk) {
        for (int i2 = tid; i2 < wk * R0; i2 += NT) {
          int c = i2 / R0, r = i2 - c * R0;
          Ls[c * (R0 + 1) + r] = __ldg(L + r + (int64_t)c * noff);
        }
        for (int r = tid; r < R0; r += NT) S.rows[r] = __ldg(rows + r);
      } else {
        prefetch_block(L, noff, wk, noff);
        for (int64_t r = (int64_t)tid * 32; r < noff; r += (int64_t)NT * 32) prefetch_l2(rows + r);
      }
      for (int64_t k = F.blk_dptr[b] + tid; k < F.blk_dptr[b + 1]; k += NT) spin_u32(F.ready_sb + F.blk_dest[k], E);
      if (F.tprof && tid == 0) t1 = gtime();
      __syncthreads();
      double tsum = 0.0;
      if (one_chunk) {
        for (int r = tid; r < R0; r += NT) S.xr[r] = __ldcg(x + S.rows[r]);
        __syncthreads();
        tile_gemv_t(Ls, R0, wk, S.xr, S.red);
        if (tid < wk) tsum = S.red[tid];
        __syncthreads();
      } else {
        double* Lc = sm + 4160;   // chunk tiles must not overwrite L_bb⁻¹: use a second pass below
        (void)Lc;
        const int Rc = wk > 4 ? 4096 / wk : 1024;
        for (int64_t r0 = 0; r0 < noff; r0 += Rc) {
          const int Rn = (int)(noff - r0 < Rc ? noff - r0 : Rc);
          __syncthreads();
          load_tile(sm, L + r0, Rn, wk, noff);
          double* xr = sm + wk * (Rn + 1);
          for (int r = tid; r < Rn; r += NT) xr[r] = __ldcg(x + __ldg(rows + r0 + r));
          __syncthreads();
          tile_gemv_t(sm, Rn, wk, xr, S.red);
          if (tid < wk) tsum += S.red[tid];
        }
        __syncthreads();
        for (int i2 = tid; i2 < wk * wk; i2 += NT) {
          int c = i2 / wk, r = i2 - c * wk;
          sm[c * 65 + r] = __ldg(inv + i2);
        }
      }
      if (tid < wk) S.rhs[tid] = __ldcg(x + c0 + tid) * dinv - tsum;
      __syncthreads();
      {
        const int i = tid & 63, g = tid >> 6;
        double s = 0.0;
        if (i < wk)
          for (int j = i + g; j < wk; j += 4) s += sm[i * 65 + j] * S.rhs[j];
        S.red[g * 64 + i] = s;
      }
      __syncthreads();
      if (tid < wk) x[c0 + tid] = S.red[tid] + S.red[64 + tid] + S.red[128 + tid] + S.red[192 + tid];
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        st_rel_u32(F.ready_sb + J, E);
      }
    } else if (type == 7) {
      // ---------------- SNW backward
      const int bw = F.snw_bwd[idx * 8 + (tid >> 5)];
      if (bw >= 0) snw_backward(F, x, bw, E);
    } else if (type == 6) {
      // ---------------- ROOTB: the symmetric root's x = S⁻¹ v was completed by the forward sweep
      const int J = idx;
      for (int b = F.sn_blk0[J] + tid; b < F.sn_blk0[J + 1]; b += NT)
        atomicAdd(F.cntx_b + b, (unsigned long long)F.xexp_b[b]);   // keep X-path counters in step
      __syncthreads();
      if (tid == 0) {
        atomicAdd(F.sn_done_b + J, (unsigned long long)F.sn_nblk[J]);
        st_rel_u32(F.ready_sb + J, E);
      }
    } else if (type == 3) {
      // ---------------- XCHUNK (backward): x[K] += (X_Jᵀ)_{K, I0..I0+nI} · v[I0..]
      const int bK = F.xb_bK[idx], bI = F.xb_bI[idx], nI = F.xb_nI[idx];
      const int J = F.blk_sn[bK];
      const int64_t cJ = F.sn_start[J];
      const int64_t rK = F.blk_col0[bK], cI = F.blk_col0[bI];
      const int Rn = F.blk_w[bK];
      const int ncol = (int)(F.blk_col0[bI + nI - 1] + F.blk_w[bI + nI - 1] - cI);
      if (tid < nI) spin_u32(F.vready_b + bI + tid, E);
      if (tid == 64) spin_u32(F.vready_b + bK, E);
      if (F.tprof && tid == 0) t1 = gtime();
      __syncthreads();
      for (int c = tid; c < ncol; c += NT) sm[c] = __ldcg(F.vbuf + cI + c);
      __syncthreads();
      double* red = sm + 512;
      const int64_t ldx = F.sn_ldx[J];
      xchunk_gemv(F.xinv + F.sn_xtr[J] + (rK - cJ) + (cI - cJ) * ldx, ldx, Rn, ncol, sm, red);
      if (tid < Rn) atomicAdd(x + rK + tid, red[512 + tid]);
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        unsigned long long old = atomicAdd(F.cntx_b + bK, 1ull);
        if (old + 1 == (unsigned long long)E * (unsigned long long)F.xexp_b[bK]) {
          __threadfence();
          unsigned long long d = atomicAdd(F.sn_done_b + J, 1ull);
          if (d + 1 == (unsigned long long)E * (unsigned long long)F.sn_nblk[J]) {
            __threadfence();
            st_rel_u32(F.ready_sb + J, E);
          }
        }
      }
    } else {
      const int ti = idx;
      const int b = F.tile_blk[ti];
      const int wk = F.blk_w[b];
      const int Rn = F.tile_nr[ti];
      const int r0 = F.tile_r0[ti];
      const int64_t noff = F.blk_noff[b];
      const int64_t c0 = F.blk_col0[b];
      const double* Lt = F.fstore + F.blk_off[b] + r0;
      const bool longt = Rn * wk > 4096;
      if (!longt) load_tile(sm, Lt, Rn, wk, noff);   // long tiles stream after the wait (an L2 prefetch of
      // 256 KB per task was evicted before use and doubled the DRAM reads)
      if (tid == 0) {
        for (int64_t q = F.tile_dptr[ti]; q < F.tile_dptr[ti + 1]; ++q) spin_u32(F.ready_sb + F.tile_dlist[q], E);
        if (F.tprof) t1 = gtime();
      }
      __syncthreads();
      const int32_t* rows = F.sn_rows + F.blk_rows[b] + r0;
      if (longt) {
        // straight from global memory: x of the tile's rows staged once in shared memory, warp w sums
        // columns 8w..8w+7 over all rows (coalesced along rows, 8 loads in flight per row), then a
        // transpose-reduce of the 8 column partials across the warp
        for (int r = tid; r < Rn; r += NT) sm[r] = __ldcg(x + rows[r]);
        __syncthreads();
        const int lane = tid & 31, cw = (tid >> 5) * 8;
        double t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) t[u] = 0.0;
        int r = lane;
        if (wk == 64 && (F.sweep_var & 1)) {   // full-width block: two rows per lane in flight (16 loads)
          const double* Lc = Lt + (int64_t)cw * noff;
          for (; r + 32 < Rn; r += 64) {
            const double xa = sm[r], xb = sm[r + 32];
            double va[8], vb[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              va[u] = __ldg(Lc + r + (int64_t)u * noff);
              vb[u] = __ldg(Lc + r + 32 + (int64_t)u * noff);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) t[u] += va[u] * xa + vb[u] * xb;
          }
        }
        for (; r < Rn; r += 32) {
          const double xv = sm[r];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (cw + u < wk) t[u] += __ldg(Lt + r + (int64_t)(cw + u) * noff) * xv;
        }
        const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
        double a4[4], a2[2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          a4[i] = (h16 ? t[i + 4] : t[i]) + __shfl_xor_sync(0xffffffffu, h16 ? t[i] : t[i + 4], 16);
#pragma unroll
        for (int i = 0; i < 2; ++i)
          a2[i] = (h8 ? a4[i + 2] : a4[i]) + __shfl_xor_sync(0xffffffffu, h8 ? a4[i] : a4[i + 2], 8);
        double a1 = (h4 ? a2[1] : a2[0]) + __shfl_xor_sync(0xffffffffu, h4 ? a2[0] : a2[1], 4);
        a1 += __shfl_xor_sync(0xffffffffu, a1, 2);
        a1 += __shfl_xor_sync(0xffffffffu, a1, 1);
        const int col = cw + (h16 ? 4 : 0) + (h8 ? 2 : 0) + (h4 ? 1 : 0);
        if ((lane & 3) == 0 && col < wk) atomicAdd(F.tacc + c0 + col, a1);
      } else {
        double* xr = sm + wk * (Rn + 1);
        for (int r = tid; r < Rn; r += NT) xr[r] = __ldcg(x + rows[r]);
        __syncthreads();
        tile_gemv_t(sm, Rn, wk, xr, S.red);
        if (tid < wk) atomicAdd(F.tacc + c0 + tid, S.red[tid]);
      }
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(F.cnt_b + b, 1ull);
      }
    }
    if (F.tprof) tprof_add(F.tprof, 1, type, t0, t1, gtime(), task, S.ticket, F.ttrace_cap, ta, tb);
  }
  if (tid == 0) {
    unsigned d = atomicAdd(F.sweep + 1, 1u);
    if (d == gridDim.x - 1) {
      F.sweep[0] = 0u;
      F.sweep[1] = 0u;
      F.sweep[3] = E;
      __threadfence();
    }
  }
  tl_end(6, tls);
}

// ------------------------------------------------------------------------- partitioned inverse
// Batched C = α·A·B + β·C (column-major) on CUDA-core fp64: 128×128 C tile per 256-thread CTA,
// 8×8 outputs per thread (rows tx·2 + {0,1} + {0,32,64,96}: coalesced column stores; columns likewise
// from ty) so every
// shared-memory fragment load is a conflict-free 128-bit read, K in chunks of 8 staged by cp.async
// into a double buffer (loads of chunk k+1 overlap the 64 DFMA per k-step of chunk k).
constexpr int G_T = 128, G_K = 8, G_LD = G_T + 4;
__global__ void __launch_bounds__(256, 1) k_gemm128(const GemmProb* probs, const int64_t* pref, int nprob) {
  __shared__ __align__(16) double As[2][G_K * G_LD];
  __shared__ __align__(16) double Bs[2][G_K * G_LD];
  const int p = find_seg(pref, nprob + 1, blockIdx.x);
  const GemmProb P = probs[p];
  const int64_t t = blockIdx.x - pref[p];
  const int tilesM = (P.M + G_T - 1) / G_T;
  const int ti = (int)(t % tilesM), tj = (int)(t / tilesM);
  if ((P.flags & 8) && tj > ti) return;
  const int r0 = ti * G_T, c0 = tj * G_T;
  int kmin = (P.flags & 2) ? c0 : 0;
  if (P.flags & 4) kmin = max(kmin, r0);
  const int kmax = (P.flags & 1) ? min(P.K, r0 + G_T) : P.K;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  double acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
  // chunk loader: A(r0 + m, k0 + k) → As[k][m];  B(k0 + k, c0 + n) → Bs[k][n]  (4 + 4 per thread)
  auto load = [&](int buf, int k0) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = tid + 256 * u;
      const int m = idx & (G_T - 1), k = idx >> 7;
      const bool ok = r0 + m < P.M && k0 + k < kmax;
      cp_async8(&As[buf][k * G_LD + m], P.A + (ok ? (int64_t)(r0 + m) + (int64_t)(k0 + k) * P.lda : 0), ok);
      const int kk = idx & (G_K - 1), n = idx >> 3;
      const bool okb = c0 + n < P.N && k0 + kk < kmax;
      cp_async8(&Bs[buf][kk * G_LD + n], P.B + (okb ? (int64_t)(k0 + kk) + (int64_t)(c0 + n) * P.ldb : 0), okb);
    }
    cp_async_commit();
  };
  if (kmin < kmax) load(0, kmin);
  int buf = 0;
  for (int k0 = kmin; k0 < kmax; k0 += G_K) {
    cp_async_wait_all();
    __syncthreads();
    if (k0 + G_K < kmax) load(buf ^ 1, k0 + G_K);
    const double* as = As[buf];
    const double* bs = Bs[buf];
#pragma unroll 4
    for (int k = 0; k < G_K; ++k) {
      double a[8], b[8];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const double2 va = *reinterpret_cast<const double2*>(as + k * G_LD + g * 32 + tx * 2);
        const double2 vb = *reinterpret_cast<const double2*>(bs + k * G_LD + g * 32 + ty * 2);
        a[2 * g] = va.x;
        a[2 * g + 1] = va.y;
        b[2 * g] = vb.x;
        b[2 * g + 1] = vb.y;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    buf ^= 1;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int c = c0 + (j >> 1) * 32 + ty * 2 + (j & 1);
    if (c >= P.N) continue;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = r0 + (i >> 1) * 32 + tx * 2 + (i & 1);
      if (r >= P.M) continue;
      double* cp = P.C + r + (int64_t)c * P.ldc;
      *cp = P.alpha * acc[i][j] + (P.beta != 0.0 ? P.beta * *cp : 0.0);
    }
  }
}

void gemm_batched(const GemmProb* probs, const int64_t* tile_pref, int nprob, int64_t total_tiles,
                  cudaStream_t s) {
  if (total_tiles <= 0) return;
  k_gemm128<<<(unsigned)total_tiles, 256, 0, s>>>(probs, tile_pref, nprob);   // tile_pref counts 128×128 tiles
}

// X_J := unit-lower L_JJ below the diagonal tiles, L_kk⁻¹ on the 64×64 diagonal tiles, 0 above.
__global__ void k_build_xinv(DevFactor F, const int32_t* big, int n_big) {
  const int J = big[blockIdx.y];
  const int64_t cJ = F.sn_start[J], w = F.sn_start[J + 1] - cJ, ldx = F.sn_ldx[J];
  double* X = F.xinv + F.sn_xinv[J];
  for (int64_t e = blockIdx.x * (int64_t)NT + threadIdx.x; e < ldx * w; e += (int64_t)gridDim.x * NT) {
    const int64_t c = e / ldx, r = e - c * ldx;
    if (r >= w) {
      X[e] = 0.0;
      continue;
    }
    double v = 0.0;
    const int64_t kc = c / MF_BW, kr = r / MF_BW;
    const int b = F.sn_blk0[J] + (int)kc;
    const int wk = F.blk_w[b];
    if (kr == kc) {
      if (r >= c) v = F.fstore[F.blk_inv[b] + (c - kc * MF_BW) * wk + (r - kc * MF_BW)];
    } else if (r > c) {
      const int64_t noff = F.blk_noff[b];
      v = F.fstore[F.blk_off[b] + (r - (kc * MF_BW + wk)) + (c - kc * MF_BW) * noff];
    }
    X[e] = v;
  }
}

// X_Jᵀ (same padded layout) by 32×32 smem tiles; padding rows of X_Jᵀ are zero.
__global__ void k_transpose_xinv(DevFactor F, const int32_t* big) {
  __shared__ double t[32][33];
  const int J = big[blockIdx.z];
  const int64_t w = F.sn_start[J + 1] - F.sn_start[J], ldx = F.sn_ldx[J];
  const double* X = F.xinv + F.sn_xinv[J];
  double* XT = F.xinv + F.sn_xtr[J];
  const int64_t nt = (ldx + 31) / 32;
  for (int64_t tile = blockIdx.x; tile < nt * nt; tile += gridDim.x) {
    const int64_t bi = tile % nt, bj = tile / nt;   // X rows bi*32.., cols bj*32..
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 × 8
    for (int k = ty; k < 32; k += 8) {
      const int64_t r = bi * 32 + tx, c = bj * 32 + k;
      t[k][tx] = (r < ldx && c < w) ? X[r + c * ldx] : 0.0;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
      const int64_t r = bj * 32 + tx, c = bi * 32 + k;   // XT(r, c) = X(c, r)
      if (r < ldx && c < w) XT[r + c * ldx] = r < w ? t[tx][k] : 0.0;
    }
    __syncthreads();
  }
}

__global__ void k_scale_xinv_rows(DevFactor F, const int32_t* sns, int multiply) {
  const int J = sns[blockIdx.y];
  const int64_t cJ = F.sn_start[J], w = F.sn_start[J + 1] - cJ, ldx = F.sn_ldx[J];
  double* X = F.xinv + F.sn_xinv[J];
  for (int64_t e = blockIdx.x * (int64_t)NT + threadIdx.x; e < ldx * w; e += (int64_t)gridDim.x * NT) {
    const int64_t r = e % ldx;
    if (r < w) X[e] = multiply ? X[e] * F.Dpiv[cJ + r] : X[e] / F.Dpiv[cJ + r];
  }
}

void scale_xinv_rows(const DevFactor& F, const int32_t* sns, int n, int64_t max_w2, bool multiply, cudaStream_t s) {
  if (n == 0) return;
  dim3 grid((unsigned)std::min<int64_t>((max_w2 + NT - 1) / NT, 148 * 8), (unsigned)n);
  k_scale_xinv_rows<<<grid, NT, 0, s>>>(F, sns, multiply ? 1 : 0);
}

void transpose_xinv(const DevFactor& F, const int32_t* big_sns, int n_big, int64_t max_w2, cudaStream_t s) {
  if (n_big == 0) return;
  dim3 grid((unsigned)std::min<int64_t>((max_w2 + 1023) / 1024 + 1, 148 * 8), 1, (unsigned)n_big);
  k_transpose_xinv<<<grid, NT, 0, s>>>(F, big_sns);
}

void build_xinv(const DevFactor& F, const int32_t* big_sns, int n_big, int64_t max_w2, cudaStream_t s) {
  if (n_big == 0) return;
  dim3 grid((unsigned)std::min<int64_t>((max_w2 + NT - 1) / NT, 148 * 8), (unsigned)n_big);
  k_build_xinv<<<grid, NT, 0, s>>>(F, big_sns, n_big);
}

// Epilogue of a symmetric-GEMV chunk (see SymvPlan): the chunk's row partial (red_row, Rn rows, output
// block rob) and column partials (colv, ncol_t = 64·ncob columns, output blocks cob0 …) go to their slots;
// k_symv_reduce then sums every output block's slots in the plan's fixed order.  (A last-arriver
// reduction inside the GEMV — counters, fences, the arriving CTA reducing — made it 4× slower on c1.)
__device__ __forceinline__ void symv_epilogue(const SymvPlan& P, int64_t idx, int Rn, int rob, int ncol_t, int cob0,
                                              const double* red_row, const double* colv, double* x) {
  const int tid = threadIdx.x;
  if (P.slots == nullptr) {   // QPB_DETERMINISTIC=0: fp64 atomics (rounding order varies run to run)
    if (tid < Rn) atomicAdd(x + P.x0[rob - P.ob_lo] + tid, red_row[tid]);
    const int64_t xc = P.x0[cob0 - P.ob_lo];
    for (int c = tid; c < ncol_t; c += NT) atomicAdd(x + xc + c, colv[c]);
    return;
  }
  const int64_t* wo = P.woff + (idx - P.c_begin) * 9;
  if (tid < Rn) P.slots[wo[0] + tid] = red_row[tid];
  for (int c = tid; c < ncol_t; c += NT) P.slots[wo[1 + (c >> 6)] + (c & 63)] = colv[c];
}

// x[block o] += Σ of its contributions, which are contiguous (64 doubles each) in the plan's fixed order:
// CTA of 1 024 threads per output block, 16 groups of 64 (one thread per row) stride the list with 8
// independent partial sums each; the 128 partials of a row are combined in a fixed order (bit-reproducible).
constexpr int RED_NT = 1024;
__global__ void __launch_bounds__(RED_NT) k_symv_reduce(SymvPlan P, int32_t nob, double* x, const int* done_flag) {
  __shared__ double red[RED_NT];
  if (done_flag != nullptr && *((volatile const int*)done_flag)) return;
  const int tid = threadIdx.x, i = tid & 63, g = tid >> 6;
  for (int ob = blockIdx.x; ob < nob; ob += gridDim.x) {
    const int w = P.width[ob];
    const int64_t e0 = P.lptr[ob], e1 = P.lptr[ob + 1];
    double a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = 0.0;
    if (i < w)
      for (int64_t e = e0 + g; e < e1; e += 128) {   // entries e + 16u: 8 loads in flight per thread
        const double* q = P.slots + 64 * e + i;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (e + 16 * u < e1) a[u] += __ldcg(q + 64 * 16 * u);
      }
    red[g * 64 + i] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    __syncthreads();
    if (tid < w) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < 16; ++k) t += red[k * 64 + tid];
      x[P.x0[ob] + tid] += t;
    }
    __syncthreads();
  }
}
void symv_reduce(const SymvPlan* P, double* x, const int* done_flag, int sms, cudaStream_t s) {
  if (P == nullptr || P->slots == nullptr || P->nob <= 0) return;
  k_symv_reduce<<<(unsigned)std::min<int64_t>(P->nob, (int64_t)sms * 2), RED_NT, 0, s>>>(*P, P->nob, x, done_flag);
}

// Symmetric-root GEMV as its own kernel (between the forward and backward sparse sweeps):
// x_J += S_J⁻¹ v_J over the chunks (I, K0..K0+nK) of every symmetric root, grid-stride, no flags.
template <int U, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_symroot_gemv(DevFactor F, double* x, int64_t c_begin, int64_t c_end,
                                                           SymvPlan P, const int* done_flag, const double* sub) {
  __shared__ double vK[512];
  __shared__ double vI[64];
  __shared__ double red[576];
  __shared__ double colv[512];
  if (done_flag != nullptr && *((volatile const int*)done_flag)) return;
  const unsigned tls = tl_begin(2);
  const int tid = threadIdx.x;
  const uint64_t pol = (F.l2hint & 1) ? l2pol_first() : l2pol_normal();
  for (int64_t idx = c_begin + blockIdx.x; idx < c_end; idx += gridDim.x) {
    const int bI = F.xt_bI[idx], bK = F.xt_bK[idx], nK = F.xt_nK[idx];
    const int J = F.blk_sn[bI];
    const int64_t cJ = F.sn_start[J];
    const int64_t rI = F.blk_col0[bI], cK = F.blk_col0[bK];
    const int Rn = F.blk_w[bI];
    const int ncol = (int)(F.blk_col0[bK + nK - 1] + F.blk_w[bK + nK - 1] - cK);
    const int ncol_t = (int)((rI < cK + ncol ? rI : cK + ncol) - cK);
    const int64_t ldx = F.sn_ldx[J];
    const double* Mc = F.xinv + F.sn_sinv[J] + (rI - cJ) + (cK - cJ) * ldx;
    __syncthreads();
    if (sub != nullptr) {
      for (int c = tid; c < ncol; c += NT) vK[c] = F.vbuf[cK + c] - sub[cK + c];
      if (tid < Rn) vI[tid] = F.vbuf[rI + tid] - sub[rI + tid];
    } else {
      for (int c = tid; c < ncol; c += NT) vK[c] = F.vbuf[cK + c];
      if (tid < Rn) vI[tid] = F.vbuf[rI + tid];
    }
    __syncthreads();
    schunk_gemv<U>(Mc, ldx, Rn, ncol, ncol_t, vK, vI, red, colv, pol);
    __syncthreads();
    symv_epilogue(P, idx, Rn, bI, ncol_t, bK, red + 512, colv, x);
  }
  tl_end(2, tls);
}

// Dense symmetric GEMV x += W v on the explicit x-block W = (F⁻¹)₁₁ (column-major, leading dimension ld,
// full storage, lower triangle read): chunks (row block I, ≤ 8 column blocks from K0 up to the diagonal
// block) through schunk_gemv, so each lower tile is read once for x_I += W_IK v_K and x_K += W_IKᵀ v_I.
template <int U, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_dense_symv(const double* W, int64_t ld, int64_t n, const int2* chunks,
                                                         int64_t nch, SymvPlan P, const double* v, double* x,
                                                         const int* done_flag) {
  __shared__ double vK[512];
  __shared__ double vI[64];
  __shared__ double red[576];
  __shared__ double colv[512];
  if (done_flag != nullptr && *((volatile const int*)done_flag)) return;
  const unsigned tls = tl_begin(2);
  const int tid = threadIdx.x;
  const uint64_t pol = l2pol_normal();
  for (int64_t idx = blockIdx.x; idx < nch; idx += gridDim.x) {
    const int2 ch = __ldg(chunks + idx);
    const int64_t rI = 64 * (int64_t)ch.x, cK = 64 * (int64_t)ch.y;
    const int Rn = (int)(n - rI < 64 ? n - rI : 64);
    const int64_t cEnd = (cK + 512 < rI + Rn) ? cK + 512 : rI + Rn;
    const int ncol = (int)(cEnd - cK);
    const int ncol_t = (int)(rI - cK < ncol ? rI - cK : ncol);
    __syncthreads();
    for (int c = tid; c < ncol; c += NT) vK[c] = v[cK + c];
    if (tid < Rn) vI[tid] = v[rI + tid];
    __syncthreads();
    schunk_gemv<U>(W + rI + cK * ld, ld, Rn, ncol, ncol_t, vK, vI, red, colv, pol);
    __syncthreads();
    symv_epilogue(P, P.c_begin + idx, Rn, ch.x, ncol_t, ch.y, red + 512, colv, x);
  }
  tl_end(2, tls);
}

// v[c] = the F-solve right-hand side described by R, for every c < N (dense F⁻¹ mode: the GEMV needs it
// materialised): R.rhs (optionally gathered through in_perm), or (Cᵀp)_c fused (warp per row).
__global__ void k_gather_rhs(SweepRhs R, double* v, double* out, int64_t N) {
  if (R.done_flag != nullptr && *((volatile const int*)R.done_flag)) return;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (NT / 32);
  for (int64_t c = blockIdx.x * (int64_t)(NT / 32) + (threadIdx.x >> 5); c < N; c += nw) {
    double x = 0.0;
    if (R.ct.p == nullptr) {
      if (lane == 0) x = R.rhs[R.in_perm ? R.in_perm[c] : c];
    } else if (c < R.ct.nrows) {
      const int64_t q0 = __ldg(R.ct.p + c), q1 = __ldg(R.ct.p + c + 1);
      for (int64_t q = q0 + lane; q < q1; q += 32) x += __ldg(R.ct.v + q) * __ldg(R.p + __ldg(R.ct.i + q));
      x = warp_sum(x);
    }
    if (lane == 0) {
      v[c] = x;
      out[c] = 0.0;   // the GEMV's reducers accumulate into out
    }
  }
}
__global__ void k_zero_flag(double* v, int64_t n, const int* done_flag) {
  if (done_flag != nullptr && *((volatile const int*)done_flag)) return;
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) v[i] = 0.0;
}
void zero_flag(double* v, int64_t n, const int* done_flag, cudaStream_t s) {
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((n + NT - 1) / NT, 148 * 8));
  k_zero_flag<<<g, NT, 0, s>>>(v, n, done_flag);
}
void gather_rhs(const SweepRhs& r, double* v, double* out, int64_t N, int sms, cudaStream_t s) {
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((N + 7) / 8, (int64_t)sms * 8));
  k_gather_rhs<<<g, NT, 0, s>>>(r, v, out, N);
}

// W[r0 + a, r0 + b] = S⁻¹(a, b) for a ≥ b (x-part of the symmetric root, lower storage Sinv with ldx).
__global__ void k_w_copy_root(const double* Sinv, int64_t ldx, double* W, int64_t ld, int64_t r0, int64_t n) {
  const int64_t m = n - r0;
  for (int64_t b = blockIdx.x; b < m; b += gridDim.x)
    for (int64_t a = b + threadIdx.x; a < m; a += NT) W[(r0 + a) + (r0 + b) * ld] = Sinv[a + b * ldx];
}
void w_copy_root(const double* Sinv, int64_t ldx, double* W, int64_t ld, int64_t r0, int64_t n, cudaStream_t s) {
  if (n > r0) k_w_copy_root<<<148 * 8, NT, 0, s>>>(Sinv, ldx, W, ld, r0, n);
}
// Upper triangle of every diagonal 64-block from its lower triangle (k_dense_symv reads them full).
__global__ void k_w_symmetrize_diag(double* W, int64_t ld, int64_t n) {
  const int64_t c0 = 64 * (int64_t)blockIdx.x;
  for (int t = threadIdx.x; t < 64 * 64; t += NT) {
    const int64_t i = c0 + (t & 63), j = c0 + (t >> 6);
    if (i < j && j < n) W[i + j * ld] = W[j + i * ld];
  }
}
void w_symmetrize_diag(double* W, int64_t ld, int64_t n, cudaStream_t s) {
  if (n > 0) k_w_symmetrize_diag<<<(unsigned)((n + 63) / 64), NT, 0, s>>>(W, ld, n);
}

void dense_symv(const double* W, int64_t ld, int64_t n, const int2* chunks, int64_t nch, const SymvPlan* plan,
                const double* v, double* x, const int* done_flag, int sms, cudaStream_t s, bool reduce) {
  if (nch <= 0) return;
  k_dense_symv<16, 3><<<sms * 3, NT, 0, s>>>(W, ld, n, chunks, nch, *plan, v, x, done_flag);
  if (reduce) symv_reduce(plan, x, done_flag, sms, s);
}

void symroot_gemv(const DevFactor& F, double* x, int64_t c_begin, int64_t c_end, const SymvPlan* plan,
                  const int* done_flag, int grid, cudaStream_t s, const double* sub) {
  if (c_end <= c_begin) return;
  static int variant = std::getenv("QPB_GEMV_VARIANT") ? std::atoi(std::getenv("QPB_GEMV_VARIANT")) : 3;
  static int sms = 0;
  if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  switch (variant) {
    case 1: k_symroot_gemv<8, 4><<<sms * 4, NT, 0, s>>>(F, x, c_begin, c_end, *plan, done_flag, sub); break;
    case 2: k_symroot_gemv<16, 2><<<sms * 2, NT, 0, s>>>(F, x, c_begin, c_end, *plan, done_flag, sub); break;
    case 3: k_symroot_gemv<16, 3><<<sms * 3, NT, 0, s>>>(F, x, c_begin, c_end, *plan, done_flag, sub); break;
    case 4: k_symroot_gemv<4, 4><<<sms * 4, NT, 0, s>>>(F, x, c_begin, c_end, *plan, done_flag, sub); break;
    default: k_symroot_gemv<8, 3><<<sms * 3, NT, 0, s>>>(F, x, c_begin, c_end, *plan, done_flag, sub); break;
  }
  symv_reduce(plan, x, done_flag, sms, s);
  (void)grid;
}


// ------------------------------------------------------------------------- flattened forest
// Right-hand side of a flattened F-solve: b_c = (Cᵀp)_c or rhs_c (warp per column); forest columns
// → acc[0, rc0) (b1), root columns → vbuf (the root GEMV's right-hand side before − M b1); x = 0.
__global__ void __launch_bounds__(NT) k_flat_rhs(DevFactor F, SweepRhs R, double* x) {
  if (R.done_flag != nullptr && *((volatile const int*)R.done_flag)) return;
  const unsigned tls = tl_begin(0);
  const int lane = threadIdx.x & 31;
  const int64_t rc0 = F.fl_rc0, N = F.N;
  for (int64_t c = (blockIdx.x * (int64_t)NT + threadIdx.x) >> 5; c < N; c += ((int64_t)gridDim.x * NT) >> 5) {
    double v;
    if (R.ct.p != nullptr) {
      v = 0.0;
      if (c < R.ct.nrows) {
        const int64_t q0 = __ldg(R.ct.p + c), q1 = __ldg(R.ct.p + c + 1);
        for (int64_t q = q0 + lane; q < q1; q += 32) v += __ldg(R.ct.v + q) * __ldg(R.p + __ldg(R.ct.i + q));
        v = warp_sum(v);
      }
    } else {
      v = R.rhs[R.in_perm ? R.in_perm[c] : c];
    }
    if (lane == 0) {
      if (c < rc0) {
        F.acc[c] = v;
        F.vbuf[c] = 0.0;   // y1 accumulator (k_flat_fwd)
      } else {
        F.vbuf[c] = v;
      }
      x[c] = 0.0;
    }
  }
  tl_end(0, tls);
}

// Forward product: tasks [0, nY) — 8 forest columns each (warp per column c), vbuf[rows of L11⁻¹(:,c)]
// += L11⁻¹(:,c) b1_c (y1 = L11⁻¹ b1; vbuf[0, rc0) zeroed by k_flat_rhs); tasks [nY, nY + nRr) — 8 root
// rows each (warp per row r): vbuf[r] = b2_r − M(r,:) b1, a fixed-order dot product (no atomics).
__global__ void __launch_bounds__(NT) k_flat_fwd(DevFactor F, const int* done_flag, int64_t nY, int64_t total) {
  if (done_flag != nullptr && *((volatile const int*)done_flag)) return;
  const unsigned tls = tl_begin(1);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t rc0 = F.fl_rc0, wr = F.N - rc0;
  const uint64_t pol = (F.l2hint & 2) ? l2pol_last() : l2pol_normal();
  for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
    if (t < nY) {
      const int64_t c = t * 8 + wid;
      if (c < rc0) {
        const double bc = F.acc[c];
        const int64_t e1 = ldg_pol(F.fl_cp + c + 1, pol);
        for (int64_t e = ldg_pol(F.fl_cp + c, pol) + lane; e < e1; e += 32)
          atomicAdd(F.vbuf + ldg_pol(F.fl_ci + e, pol), ldg_pol(F.fl_nval + e, pol) * bc);
      }
    } else {
      const int64_t r = (t - nY) * 8 + wid;
      if (r < wr) {
        const int64_t e0 = ldg_pol(F.fl_mr_ptr + r, pol), e1 = ldg_pol(F.fl_mr_ptr + r + 1, pol);
        double s = 0.0;
        for (int64_t e = e0 + lane; e < e1; e += 256) {   // 8 entries per lane in flight (predicated tail)
          double v[8];
          int cc[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const bool ok = e + 32 * u < e1;
            v[u] = ok ? ldg_pol(F.fl_mr_val + e + 32 * u, pol) : 0.0;
            cc[u] = ok ? ldg_pol(F.fl_mr_col + e + 32 * u, pol) : 0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) s += v[u] * F.acc[cc[u]];
        }
        s = warp_sum(s);
        if (lane == 0) F.vbuf[rc0 + r] -= s;
      }
    }
  }
  tl_end(1, tls);
}

// ---- M products by units (QPB_FLAT_TILES=1, default).  M_J (nr rows × w columns, column-major) is cut into
// units of ≤ 64 rows × ≤ 8 columns, each described by 32 bytes built once at setup (fl_units: offset of
// its first entry, offset of its row indices, first column, leading dimension, rows | columns << 16).
// Warps take units grid-stride (about two per warp on c1), so a unit costs one descriptor load, one
// round of matrix / row-index loads (two rows per lane, 8 columns in flight) and, backward, one gather.
// Forward: s_r = Σ_c M(r,c) b1_c, one atomic per row into the root right-hand side.  Backward:
// x_c −= Σ_r M(r,c) x_root(r): the 8 column partials combined by a transpose-reduce (4+2+1+1+1 shuffles),
// one atomic per column and unit.  Forest columns (L11⁻¹ products) follow as warp-per-column units.
// Transpose-reduce of 8 per-lane values over a warp: returns the warp sum of t[lane >> 2] in every lane
// with (lane & 3) == 0.
__device__ __forceinline__ double transpose_reduce8(const double (&t)[8], int lane) {
  const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
  double a4[4], a2[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) a4[i] = (h16 ? t[i + 4] : t[i]) + __shfl_xor_sync(0xffffffffu, h16 ? t[i] : t[i + 4], 16);
#pragma unroll
  for (int i = 0; i < 2; ++i) a2[i] = (h8 ? a4[i + 2] : a4[i]) + __shfl_xor_sync(0xffffffffu, h8 ? a4[i] : a4[i + 2], 8);
  double a1 = (h4 ? a2[1] : a2[0]) + __shfl_xor_sync(0xffffffffu, h4 ? a2[0] : a2[1], 4);
  a1 += __shfl_xor_sync(0xffffffffu, a1, 2);
  a1 += __shfl_xor_sync(0xffffffffu, a1, 1);
  return a1;
}

struct FlatUnit {
  int64_t moff;
  int32_t roff, col0, ld, shape;
};
__device__ __forceinline__ FlatUnit load_unit(const int4* U, int64_t u) {
  const int4 a = __ldg(U + 2 * u), b = __ldg(U + 2 * u + 1);
  FlatUnit f;
  f.moff = (int64_t)(uint32_t)a.x | ((int64_t)a.y << 32);
  f.roff = a.z;
  f.col0 = a.w;
  f.ld = b.x;
  f.shape = b.y;
  return f;
}

__global__ void __launch_bounds__(NT) k_flat_fwd_t(DevFactor F, const int* done_flag) {
  if (done_flag != nullptr && *((volatile const int*)done_flag)) return;
  const unsigned tls = tl_begin(1);
  const int lane = threadIdx.x & 31;
  const int64_t nu = F.fl_nunits, total = nu;
  const int64_t nw = (int64_t)gridDim.x * (NT / 32);
  for (int64_t u = blockIdx.x * (int64_t)(NT / 32) + (threadIdx.x >> 5); u < total; u += nw) {
    {
      const FlatUnit f = load_unit(F.fl_units, u);
      const int nrows = f.shape & 0xffff, ncols = f.shape >> 16;
      if (lane >= nrows) continue;
      const bool okb = lane + 32 < nrows;
      const double* Mu = F.fl_mval + f.moff;
      double ma[8], mb[8], bv[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const bool okc = c < ncols;
        ma[c] = okc ? __ldg(Mu + (int64_t)c * f.ld + lane) : 0.0;
        mb[c] = okc && okb ? __ldg(Mu + (int64_t)c * f.ld + lane + 32) : 0.0;
        bv[c] = okc ? F.acc[f.col0 + c] : 0.0;
      }
      double sa = 0.0, sb = 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        sa = fma(ma[c], bv[c], sa);
        sb = fma(mb[c], bv[c], sb);
      }
      F.fl_fslot[u * 64 + lane] = sa;              // reduced per root row, in unit order, by k_flat_fwd_red
      if (okb) F.fl_fslot[u * 64 + 32 + lane] = sb;
    }
  }
  tl_end(1, tls);
}

// Forward reductions (fixed order, no atomics): forest row i — y1_i = Σ_j L11⁻¹(i, j) b1_j (row form of
// L11⁻¹); root row r — vbuf[rc0 + r] −= Σ of its unit partials in unit order.  Warp per row.
__global__ void __launch_bounds__(NT) k_flat_fwd_red(DevFactor F, const int* done_flag) {
  if (done_flag != nullptr && *((volatile const int*)done_flag)) return;
  const int lane = threadIdx.x & 31;
  const int64_t rc0 = F.fl_rc0, N = F.N;
  const int64_t nw = (int64_t)gridDim.x * (NT / 32);
  for (int64_t t = blockIdx.x * (int64_t)(NT / 32) + (threadIdx.x >> 5); t < N; t += nw) {
    double v = 0.0;
    if (t < rc0) {
      for (int64_t e = F.fl_rp[t] + lane; e < F.fl_rp[t + 1]; e += 32)
        v += F.fl_nval[F.fl_r2c[e]] * F.acc[F.fl_rj[e]];
    } else {
      const int64_t r = t - rc0;
      for (int64_t e = F.fl_fr_ptr[r] + lane; e < F.fl_fr_ptr[r + 1]; e += 32) v += __ldcg(F.fl_fslot + F.fl_fr_src[e]);
    }
    v = warp_sum(v);
    if (lane == 0) {
      if (t < rc0) F.vbuf[t] = v;
      else F.vbuf[t] -= v;
    }
  }
}

__global__ void __launch_bounds__(NT) k_flat_bwd_t(DevFactor F, double* x, const int* done_flag) {
  if (done_flag != nullptr && *((volatile const int*)done_flag)) return;
  const unsigned tls = tl_begin(3);
  const int lane = threadIdx.x & 31;
  const int64_t rc0 = F.fl_rc0, nu = F.fl_nunits, total = nu;
  const int64_t nw = (int64_t)gridDim.x * (NT / 32);
  for (int64_t u = blockIdx.x * (int64_t)(NT / 32) + (threadIdx.x >> 5); u < total; u += nw) {
    {   // warp-uniform: the shuffles below need all 32 lanes
      const FlatUnit f = load_unit(F.fl_units, u);
      const int nrows = f.shape & 0xffff, ncols = f.shape >> 16;
      const bool oka = lane < nrows, okb = lane + 32 < nrows;
      const int32_t ia = oka ? __ldg(F.fl_rows + f.roff + lane) : 0;
      const int32_t ib = okb ? __ldg(F.fl_rows + f.roff + lane + 32) : 0;
      const double* Mu = F.fl_mval + f.moff;
      double ma[8], mb[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const bool okc = c < ncols;
        ma[c] = okc && oka ? __ldg(Mu + (int64_t)c * f.ld + lane) : 0.0;
        mb[c] = okc && okb ? __ldg(Mu + (int64_t)c * f.ld + lane + 32) : 0.0;
      }
      const double xa = oka ? x[rc0 + ia] : 0.0, xb = okb ? x[rc0 + ib] : 0.0;
      double tt[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) tt[c] = ma[c] * xa + mb[c] * xb;
      const double s = transpose_reduce8(tt, lane);
      const int col = lane >> 2;
      if ((lane & 3) == 0 && col < ncols) F.fl_bslot[u * 8 + col] = s;   // reduced by k_flat_bwd_red
    }
  }
  tl_end(3, tls);
}

// Backward reduction (fixed order, no atomics), warp per forest column c:
// x_c += Σ_i L11⁻¹(i, c) y1_i / d_i − Σ of its unit partials (Mᵀ x_root) in unit order.
__global__ void __launch_bounds__(NT) k_flat_bwd_red(DevFactor F, double* x, const int* done_flag) {
  if (done_flag != nullptr && *((volatile const int*)done_flag)) return;
  const int lane = threadIdx.x & 31;
  const int64_t rc0 = F.fl_rc0;
  const int64_t nw = (int64_t)gridDim.x * (NT / 32);
  for (int64_t c = blockIdx.x * (int64_t)(NT / 32) + (threadIdx.x >> 5); c < rc0; c += nw) {
    double v = 0.0, t = 0.0;
    for (int64_t e = F.fl_cp[c] + lane; e < F.fl_cp[c + 1]; e += 32) {
      const int32_t i = F.fl_ci[e];
      v += F.fl_nval[e] * F.vbuf[i] / F.Dpiv[i];
    }
    for (int64_t e = F.fl_bc_ptr[c] + lane; e < F.fl_bc_ptr[c + 1]; e += 32) t += __ldcg(F.fl_bslot + F.fl_bc_src[e]);
    v = warp_sum(v);
    t = warp_sum(t);
    if (lane == 0) x[c] += v - t;
  }
}

__global__ void k_flat_fill_rows(DevFactor F, const int32_t* src, int64_t nnz) {
  for (int64_t k = blockIdx.x * (int64_t)NT + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * NT)
    F.fl_mr_val[k] = F.fl_mval[src[k]];
}
void flat_fill_rows(const DevFactor& F, const int32_t* src, int64_t nnz, cudaStream_t s) {
  k_flat_fill_rows<<<148 * 8, NT, 0, s>>>(F, src, nnz);
}

// Backward product: the M tiles — x[cols of J] −= M_J(tile)ᵀ x_root(tile rows) (root values gathered
// once per tile into shared memory, warp per column); tasks [nmt, nmt + nX): 8 forest columns each,
// x_c += Σ_i L11⁻¹(i,c) y1_i / d_i.  x[0, rc0) was zeroed by k_flat_rhs.
__global__ void __launch_bounds__(NT) k_flat_bwd(DevFactor F, double* x, const int* done_flag, int64_t nX, int64_t t0) {
  __shared__ double xr[512];
  if (done_flag != nullptr && *((volatile const int*)done_flag)) return;
  const unsigned tls = tl_begin(3);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t rc0 = F.fl_rc0, N = F.N;
  const int64_t total = F.fl_nmt + nX;
  const uint64_t pol = (F.l2hint & 2) ? l2pol_last() : l2pol_normal();
  for (int64_t t = t0 + blockIdx.x; t < total; t += gridDim.x) {
    if (t < F.fl_nmt) {
      const int J = F.fl_mt_J[t], q0 = F.fl_mt_q0[t], nq = F.fl_mt_nq[t];
      const int64_t c0 = F.sn_start[J];
      const int w = (int)(F.sn_start[J + 1] - c0);
      const int64_t nr = F.fl_roff[J + 1] - F.fl_roff[J];
      const int32_t* rows = F.fl_rows + F.fl_roff[J] + q0;
      __syncthreads();
      for (int q = tid; q < nq; q += NT) xr[q] = x[rc0 + ldg_pol(rows + q, pol)];   // nq ≤ 2·NT
      __syncthreads();
      const double* Mj = F.fl_mval + F.fl_moff[J] + q0;
      for (int c = wid; c < w; c += NT / 32) {
        const double* Mc = Mj + (int64_t)c * nr;
        double s = 0.0;
        for (int q0 = lane; q0 < nq; q0 += 256) {   // predicated batches of 8 loads per lane
          double mv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) mv[u] = q0 + 32 * u < nq ? ldg_pol(Mc + q0 + 32 * u, pol) : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u) s += q0 + 32 * u < nq ? mv[u] * xr[q0 + 32 * u] : 0.0;
        }
        s = warp_sum(s);
        if (lane == 0) atomicAdd(x + c0 + c, -s);
      }
    } else {
      const int64_t c = (t - F.fl_nmt) * 8 + wid;
      if (c < rc0) {
        double u = 0.0;
        const int64_t e1 = ldg_pol(F.fl_cp + c + 1, pol);
        for (int64_t e = ldg_pol(F.fl_cp + c, pol) + lane; e < e1; e += 32) {
          const int32_t i = ldg_pol(F.fl_ci + e, pol);
          u += ldg_pol(F.fl_nval + e, pol) * F.vbuf[i] / F.Dpiv[i];
        }
        u = warp_sum(u);
        if (lane == 0) atomicAdd(x + c, u);
      }
    }
  }
  tl_end(3, tls);
}

// Extraction of forest column `col` after a forward sweep with rhs = e_col (symmetric-root mode):
// vbuf[root] = −M e_col and x[forest] = L11⁻¹ e_col.  Also moves the unit entry: unit[prev] = 0.
__global__ void k_flat_extract(DevFactor F, int64_t col, const double* x, double* unit, int64_t prev) {
  const int tid = threadIdx.x;
  const int64_t rc0 = F.fl_rc0;
  const int J = F.fl_col2sn[col];
  const int64_t nr = F.fl_roff[J + 1] - F.fl_roff[J];
  double* Mc = F.fl_mval + F.fl_moff[J] + (col - F.sn_start[J]) * nr;
  const int32_t* rows = F.fl_rows + F.fl_roff[J];
  for (int64_t q = blockIdx.x * (int64_t)NT + tid; q < nr; q += (int64_t)gridDim.x * NT) Mc[q] = -F.vbuf[rc0 + rows[q]];
  for (int64_t e = F.fl_cp[col] + blockIdx.x * (int64_t)NT + tid; e < F.fl_cp[col + 1]; e += (int64_t)gridDim.x * NT)
    F.fl_nval[e] = x[F.fl_ci[e]];
  if (blockIdx.x == 0 && tid == 0) {
    if (prev >= 0) unit[prev] = 0.0;
  }
}
__global__ void k_set_unit(double* unit, int64_t col) { unit[col] = 1.0; }

void flat_rhs(const DevFactor& F, const SweepRhs& r, double* x, int sms, cudaStream_t s) {
  const int g0 = (int)std::max<int64_t>(1, std::min<int64_t>((F.N * 32 + NT - 1) / NT, (int64_t)sms * 8));
  k_flat_rhs<<<g0, NT, 0, s>>>(F, r, x);
}
void flat_forward(const DevFactor& F, const SweepRhs& r, double* x, int sms, cudaStream_t s) {
  if (!r.rhs_ready) flat_rhs(F, r, x, sms, s);
  static const bool tiles = !(std::getenv("QPB_FLAT_TILES") && std::getenv("QPB_FLAT_TILES")[0] == '0');
  if (tiles) {
    const int gt = (int)std::max<int64_t>(1, std::min<int64_t>((F.fl_nunits + 7) / 8, (int64_t)sms * 8));
    k_flat_fwd_t<<<gt, NT, 0, s>>>(F, r.done_flag);
    const int gr = (int)std::max<int64_t>(1, std::min<int64_t>((F.N + 7) / 8, (int64_t)sms * 8));
    k_flat_fwd_red<<<gr, NT, 0, s>>>(F, r.done_flag);
    return;
  }
  const int64_t nY = (F.fl_rc0 + 7) / 8, nRr = (F.N - F.fl_rc0 + 7) / 8;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nY + nRr, (int64_t)sms * 8));
  if (nY + nRr > 0) k_flat_fwd<<<grid, NT, 0, s>>>(F, r.done_flag, nY, nY + nRr);
}
void flat_backward(const DevFactor& F, double* x, const int* done_flag, int sms, cudaStream_t s) {
  static const bool tiles = !(std::getenv("QPB_FLAT_TILES") && std::getenv("QPB_FLAT_TILES")[0] == '0');
  if (tiles) {
    const int gt = (int)std::max<int64_t>(1, std::min<int64_t>((F.fl_nunits + 7) / 8, (int64_t)sms * 8));
    k_flat_bwd_t<<<gt, NT, 0, s>>>(F, x, done_flag);
    const int gr = (int)std::max<int64_t>(1, std::min<int64_t>((F.fl_rc0 + 7) / 8, (int64_t)sms * 8));
    k_flat_bwd_red<<<gr, NT, 0, s>>>(F, x, done_flag);
    return;
  }
  const int64_t nX = (F.fl_rc0 + 7) / 8;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(F.fl_nmt + nX, 1), (int64_t)sms * 8));
  k_flat_bwd<<<grid, NT, 0, s>>>(F, x, done_flag, nX, 0);
}
void flat_extract(const DevFactor& F, int64_t col, const double* x, double* unit, int64_t prev, cudaStream_t s) {
  k_flat_extract<<<8, NT, 0, s>>>(F, col, x, unit, prev);
}
void flat_set_unit(double* unit, int64_t col, cudaStream_t s) { k_set_unit<<<1, 1, 0, s>>>(unit, col); }

__global__ void k_lvl16_fwd(DevFactor F, SweepRhs R, double* x, int64_t i0, int64_t i1);
__global__ void k_lvl16_bwd(DevFactor F, double* x, const int* done_flag, int64_t i0, int64_t i1);
// QPB_LVL16=0: the 16-lane level kernels instead of the warp-per-supernode ones (A/B)
static bool lvl16_on() {
  static const bool on = !(std::getenv("QPB_LVL16") && std::getenv("QPB_LVL16")[0] == '0');
  return on;
}
static size_t trsv_smem_bytes() { return sizeof(double) * (size_t)TRSV_SMEM_DBL; }

int trsv_grid(int device) {
  static std::atomic<int> cached[64];
  if (device >= 0 && device < 64 && cached[device].load()) return cached[device].load();
  int sms = 148, occ = 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaFuncSetAttribute(k_trsv_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)trsv_smem_bytes());
  cudaFuncSetAttribute(k_trsv_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)trsv_smem_bytes());
  int o1 = 1, o2 = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_trsv_fwd, NT, trsv_smem_bytes());
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_trsv_bwd, NT, trsv_smem_bytes());
  occ = std::max(1, std::min(o1, o2));
  int g = sms * occ;
  if (device >= 0 && device < 64) cached[device].store(g);
  return g;
}

void trsv_forward(const DevFactor& F, const SweepRhs& r, double* x, int grid, cudaStream_t s) {
  for (int L = 0; L < F.lvl_cut; ++L) {   // leaf phase, bottom level first
    const int64_t i0 = F.lvl_ptr_h[L], i1 = F.lvl_ptr_h[L + 1];
    const int G = F.lvl_g_h[L];
    const int g = (int)((i1 - i0) * G + NT - 1) / NT;
    if (G == 16 && lvl16_on()) k_lvl16_fwd<<<(unsigned)(((i1 - i0) * 32 + NT - 1) / NT), NT, 0, s>>>(F, r, x, i0, i1);
    else if (G == 16) k_lvl_fwd<16><<<g, NT, 0, s>>>(F, r, x, i0, i1);
    else k_lvl_fwd<32><<<g, NT, 0, s>>>(F, r, x, i0, i1);
  }
  k_trsv_fwd<<<grid, NT, trsv_smem_bytes(), s>>>(F, r, x);
}
void trsv_backward(const DevFactor& F, double* x, const int* done_flag, int grid, cudaStream_t s) {
  k_trsv_bwd<<<grid, NT, trsv_smem_bytes(), s>>>(F, x, done_flag);
  for (int L = F.lvl_cut - 1; L >= 0; --L) {   // leaf phase, top level first
    const int64_t i0 = F.lvl_ptr_h[L], i1 = F.lvl_ptr_h[L + 1];
    const int G = F.lvl_g_h[L];
    const int g = (int)((i1 - i0) * G + NT - 1) / NT;
    if (G == 16 && lvl16_on()) k_lvl16_bwd<<<(unsigned)(((i1 - i0) * 32 + NT - 1) / NT), NT, 0, s>>>(F, x, done_flag, i0, i1);
    else if (G == 16) k_lvl_bwd<16><<<g, NT, 0, s>>>(F, x, done_flag, i0, i1);
    else k_lvl_bwd<32><<<g, NT, 0, s>>>(F, x, done_flag, i0, i1);
  }
}

// ------------------------------------------------------------------------- level products (PiSweep)
// Z_J = [X_J; L_ext,J X_J] per supernode; one kernel per elimination-tree level, a CTA per tile.
__device__ __forceinline__ PiTile pi_load_tile(const PiTile* t) {
  const int4 a = __ldg(reinterpret_cast<const int4*>(t)), b = __ldg(reinterpret_cast<const int4*>(t) + 1);
  PiTile T;
  T.zoff = (int64_t)(uint32_t)a.x | ((int64_t)a.y << 32);
  T.roff = (int64_t)(uint32_t)a.z | ((int64_t)a.w << 32);
  T.ld = b.x;
  T.col0 = b.y;
  T.nr = (int16_t)(b.z & 0xffff);
  T.nc = (int16_t)((unsigned)b.z >> 16);
  T.wx = (int16_t)(b.w & 0xffff);
  T.pad = 0;
  return T;
}
// X part of Z_J: rows [0, w) of the tile's columns, copied from L_bb⁻¹ (single block) or X_J (big supernode).
__global__ void __launch_bounds__(NT) k_pi_build_x(DevFactor F, const PiTile* tiles, const int32_t* tile_J, double* Z,
                                                   int64_t ntiles) {
  const int64_t ti = blockIdx.x;
  if (ti >= ntiles) return;
  const PiTile T = pi_load_tile(tiles + ti);
  if (T.wx <= 0) return;
  const int J = tile_J[ti];
  const int64_t cJ = F.sn_start[J], w = F.sn_start[J + 1] - cJ;
  const int64_t r0 = T.roff - F.sn_rowptr[J], c0 = T.col0 - cJ;
  const bool big = F.sn_xinv[J] >= 0;
  const double* X = big ? F.xinv + F.sn_xinv[J] : F.fstore + F.blk_inv[F.sn_blk0[J]];
  const int64_t ldx = big ? F.sn_ldx[J] : w;
  for (int i = threadIdx.x; i < (int)T.wx * T.nc; i += NT) {
    const int c = i / T.wx, r = i - c * T.wx;
    const int64_t gr = r0 + r, gc = c0 + c;
    Z[T.zoff + r + (int64_t)c * T.ld] = gr >= gc ? X[gr + gc * ldx] : 0.0;
  }
}
// Y part: Y(e, c) = Σ_{k ≥ c} L_ext(e, k) X(k, c), a thread per external row, the tile's columns in registers.
__global__ void __launch_bounds__(NT) k_pi_build_y(DevFactor F, const PiTile* tiles, const int32_t* tile_J, double* Z,
                                                   const int64_t* zoffJ, int64_t ntiles) {
  const int64_t ti = blockIdx.x;
  if (ti >= ntiles) return;
  const PiTile T = pi_load_tile(tiles + ti);
  if (T.wx >= T.nr) return;
  const int J = tile_J[ti];
  const int64_t cJ = F.sn_start[J], w = F.sn_start[J + 1] - cJ;
  const int64_t r0 = T.roff - F.sn_rowptr[J], c0 = T.col0 - cJ;
  const int b0 = F.sn_blk0[J];
  const double* Zx = Z + zoffJ[J];   // X_J: rows [0, w), leading dimension T.ld
  for (int r = T.wx + threadIdx.x; r < T.nr; r += NT) {
    const int64_t e = r0 + r - w;    // external row
    double a[64];
#pragma unroll
    for (int c = 0; c < 64; ++c) a[c] = 0.0;
    for (int64_t k = c0; k < w; ++k) {
      const int b = b0 + (int)(k >> 6), kk = (int)(k & 63);
      const int64_t noff = F.blk_noff[b];
      const int64_t local = w + e - (((k >> 6) << 6) + F.blk_w[b]);
      const double l = F.fstore[F.blk_off[b] + local + (int64_t)kk * noff];
      const double* xr = Zx + k;
#pragma unroll
      for (int c = 0; c < 64; ++c)
        if (c < T.nc && c0 + c <= k) a[c] += l * xr[(c0 + c) * (int64_t)T.ld];
    }
#pragma unroll
    for (int c = 0; c < 64; ++c)
      if (c < T.nc) Z[T.zoff + r + (int64_t)c * T.ld] = a[c];
  }
}
// Start of a level-product F-solve: acc = tacc = x = 0; the root's right-hand side into vbuf.
__global__ void __launch_bounds__(NT) k_pi_init(DevFactor F, SweepRhs R, double* x, int64_t root0) {
  if (R.done_flag != nullptr && *((volatile const int*)R.done_flag)) return;
  for (int64_t c = blockIdx.x * (int64_t)NT + threadIdx.x; c < F.N; c += (int64_t)gridDim.x * NT) {
    F.acc[c] = 0.0;
    F.tacc[c] = 0.0;
    x[c] = 0.0;
    if (c >= root0) {
      double v;
      if (R.ct.p != nullptr) v = c < R.ct.nrows ? csr_dot(R.ct, c, R.p) : 0.0;
      else v = R.rhs[R.in_perm ? R.in_perm[c] : c];
      F.vbuf[c] = v;
    }
  }
}
// Forward, one level: v = b − acc on the tile's columns; [y; u] += Z_tile v (y into tacc, u into acc).
// Blocks [0, nbig) take one CTA tile each (≤ 512 rows, two per thread); the remaining blocks take 8 strips
// each (≤ 64 rows of a short supernode, a warp per strip, v in registers): a short supernode no longer
// occupies a CTA with most of its threads idle.
// A CTA tile's part of Z into L2 (one 128-byte line per lane and column, 8 columns per warp), issued before
// the loads the tile's input depends on: the DRAM fetch then overlaps the gather of v / s.
__device__ __forceinline__ void pi_prefetch(const double* Z, const PiTile& T) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int c = wid; c < T.nc; c += NT / 32)
    for (int r = lane * 16; r < T.nr; r += 32 * 16) prefetch_l2(Z + T.zoff + r + (int64_t)c * T.ld);
}
__device__ __forceinline__ double pi_rhs(const SweepRhs& R, int64_t c) {
  if (R.ct.p != nullptr) return c < R.ct.nrows ? csr_dot(R.ct, c, R.p) : 0.0;
  return R.rhs[R.in_perm ? R.in_perm[c] : c];
}
__device__ __forceinline__ void pi_prefetch_strip(const double* Z, const PiTile& T) {
  const int lane = threadIdx.x & 31;   // 64 rows = 4 lines per column
  for (int i = lane; i < T.nc * 4; i += 32)
    if ((i & 3) * 16 < T.nr) prefetch_l2(Z + T.zoff + (int64_t)(i >> 2) * T.ld + (i & 3) * 16);
}
// Everything that does not depend on the previous level — the tile descriptor, the row indices and (pf) an
// L2 prefetch of the tile's part of Z — happens BEFORE griddepcontrol.wait: with programmatic dependent
// launch the next level's CTAs are already resident while the current level drains, and what remains after
// the wait is the dependent gather and a stream from L2.
__global__ void __launch_bounds__(NT, 4) k_pi_fwd(DevFactor F, SweepRhs R, const PiTile* tiles, int nbig, int nstrip,
                                                  const double* Z, int pf) {
  grid_dep_launch();
  __shared__ double v[64];
  const int tid = threadIdx.x;
  unsigned tls = 0;
  if ((int)blockIdx.x < nbig) {
    const PiTile T = pi_load_tile(tiles + blockIdx.x);
    const int r = 2 * tid;
    const bool ok = r < T.nr, two = r + 1 < T.nr;
    const int32_t* rows = F.sn_rows + T.roff + r;
    const int32_t g0 = ok ? __ldg(rows) : 0, g1 = two ? __ldg(rows + 1) : 0;
    if (pf == 1) pi_prefetch(Z, T);
    if (pf == 2 && ok && (tid & 7) == 0) {   // the lines of the first batch of loads only (one lane per 128-byte line)
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < T.nc) prefetch_l2(Z + T.zoff + r + (int64_t)c * T.ld);
    }
    grid_dep_wait();
    if (R.done_flag != nullptr && *((volatile const int*)R.done_flag)) return;
    tls = tl_begin(5);
    if (tid < T.nc) {
      const int64_t c = (int64_t)T.col0 + tid;
      v[tid] = pi_rhs(R, c) - __ldcg(F.acc + c);
    }
    __syncthreads();
    if (ok) {
      const double* zp = Z + T.zoff + r;
      double s0 = 0.0, s1 = 0.0;
      const int64_t ld = T.ld;
#pragma unroll 8
      for (int c = 0; c < T.nc; ++c) {
        const double2 z = __ldg(reinterpret_cast<const double2*>(zp + c * ld));
        const double vc = v[c];
        s0 += z.x * vc;
        s1 += z.y * vc;
      }
      atomicAdd((r < T.wx ? F.tacc : F.acc) + g0, s0);
      if (two) atomicAdd((r + 1 < T.wx ? F.tacc : F.acc) + g1, s1);
    }
  } else {
    const int lane = tid & 31;
    const int si = ((int)blockIdx.x - nbig) * (NT / 32) + (tid >> 5);
    const bool live = si < nstrip;
    PiTile T{};
    int32_t g0 = 0, g1 = 0;
    if (live) {
      T = pi_load_tile(tiles + nbig + si);
      const int32_t* rows = F.sn_rows + T.roff + 2 * lane;
      g0 = 2 * lane < T.nr ? __ldg(rows) : 0;
      g1 = 2 * lane + 1 < T.nr ? __ldg(rows + 1) : 0;
      if (pf) pi_prefetch_strip(Z, T);
    }
    grid_dep_wait();
    if (R.done_flag != nullptr && *((volatile const int*)R.done_flag)) return;
    tls = tl_begin(5);
    if (live) {
      const int64_t c = (int64_t)T.col0 + lane;
      const double vlo = lane < T.nc ? pi_rhs(R, c) - __ldcg(F.acc + c) : 0.0;
      const double vhi = lane + 32 < T.nc ? pi_rhs(R, c + 32) - __ldcg(F.acc + c + 32) : 0.0;
      const int r = 2 * lane;
      const bool ok = r < T.nr, two = r + 1 < T.nr;
      const double* zp = Z + T.zoff + (ok ? r : 0);
      double s0 = 0.0, s1 = 0.0;
      const int64_t ld = T.ld;
#pragma unroll 8
      for (int cc = 0; cc < T.nc; ++cc) {
        const double vc = __shfl_sync(0xffffffffu, cc < 32 ? vlo : vhi, cc & 31);
        if (ok) {
          const double2 z = __ldg(reinterpret_cast<const double2*>(zp + cc * ld));
          s0 += z.x * vc;
          s1 += z.y * vc;
        }
      }
      if (ok) atomicAdd((r < T.wx ? F.tacc : F.acc) + g0, s0);
      if (two) atomicAdd((r + 1 < T.wx ? F.tacc : F.acc) + g1, s1);
    }
  }
  tl_end(5, tls);
}
// Backward, one level: s = D⁻¹y on the tile's own rows, −x on its external rows; x_cols += Z_tileᵀ s.
__device__ __forceinline__ double pi_sval_g(const DevFactor& F, const PiTile& T, const double* x, int r, int32_t g) {
  return r < T.wx ? __ldcg(F.tacc + g) / __ldg(F.Dpiv + g) : -__ldcg(x + g);
}
__global__ void __launch_bounds__(NT, 4) k_pi_bwd(DevFactor F, const PiTile* tiles, int nbig, int nstrip, const double* Z,
                                                  double* x, const int* done_flag, int pf) {
  grid_dep_launch();
  __shared__ double s[512 + 2];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  unsigned tls = 0;
  if ((int)blockIdx.x < nbig) {
    const PiTile T = pi_load_tile(tiles + blockIdx.x);
    const int32_t ga = tid < T.nr ? __ldg(F.sn_rows + T.roff + tid) : 0;
    const int32_t gb = tid + NT < T.nr ? __ldg(F.sn_rows + T.roff + tid + NT) : 0;
    if (pf == 1) pi_prefetch(Z, T);
    if (pf == 2 && (lane & 7) == 0 && 2 * lane < T.nr) {   // first batch: rows 2·lane.., columns wid + 8k
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (wid + 8 * k < T.nc) prefetch_l2(Z + T.zoff + 2 * lane + (int64_t)(wid + 8 * k) * T.ld);
    }
    grid_dep_wait();
    if (done_flag != nullptr && *((volatile const int*)done_flag)) return;
    tls = tl_begin(6);
    s[tid] = tid < T.nr ? pi_sval_g(F, T, x, tid, ga) : 0.0;
    s[tid + NT] = tid + NT < T.nr ? pi_sval_g(F, T, x, tid + NT, gb) : 0.0;
    __syncthreads();
    double t[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) t[k] = 0.0;
    const int64_t ld = T.ld;
    const double* zp = Z + T.zoff + (int64_t)wid * ld;
    for (int rb = 2 * lane; rb < T.nr; rb += 64) {
      const double s0 = s[rb], s1 = s[rb + 1];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (wid + 8 * k < T.nc) {
          const double2 z = __ldg(reinterpret_cast<const double2*>(zp + rb + 8 * k * ld));
          t[k] += z.x * s0 + z.y * s1;
        }
      }
    }
    // 8 column sums over 32 lanes: fold 8 → 1 values over xor 16, 8, 4, then two plain stages
#pragma unroll
    for (int h = 4, m = 16; h >= 1; h >>= 1, m >>= 1) {
      const bool up = lane & m;
#pragma unroll
      for (int k = 0; k < h; ++k) {
        const double send = up ? t[k] : t[k + h];
        const double keep = up ? t[k + h] : t[k];
        t[k] = keep + __shfl_xor_sync(0xffffffffu, send, m);
      }
    }
    double r0 = t[0];
    r0 += __shfl_xor_sync(0xffffffffu, r0, 2);
    r0 += __shfl_xor_sync(0xffffffffu, r0, 1);
    // lane bits (16, 8, 4) select k = 4·b16 + 2·b8 + b4
    if ((lane & 3) == 0) {
      const int k = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
      const int c = wid + 8 * k;
      if (c < T.nc) atomicAdd(x + T.col0 + c, r0);
    }
  } else {
    const int si = ((int)blockIdx.x - nbig) * (NT / 32) + wid;
    const bool live = si < nstrip;
    PiTile T{};
    int32_t g0 = 0, g1 = 0;
    if (live) {
      T = pi_load_tile(tiles + nbig + si);
      g0 = 2 * lane < T.nr ? __ldg(F.sn_rows + T.roff + 2 * lane) : 0;
      g1 = 2 * lane + 1 < T.nr ? __ldg(F.sn_rows + T.roff + 2 * lane + 1) : 0;
      if (pf) pi_prefetch_strip(Z, T);
    }
    grid_dep_wait();
    if (done_flag != nullptr && *((volatile const int*)done_flag)) return;
    tls = tl_begin(6);
    if (live) {
      const int r = 2 * lane;
      const bool ok = r < T.nr;
      const double s0 = ok ? pi_sval_g(F, T, x, r, g0) : 0.0;
      const double s1 = r + 1 < T.nr ? pi_sval_g(F, T, x, r + 1, g1) : 0.0;
      const double* zp = Z + T.zoff + (ok ? r : 0);
      const int64_t ld = T.ld;
      for (int cb = 0; cb < T.nc; cb += 16) {
        double t[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          double tv = 0.0;
          if (ok && cb + k < T.nc) {
            const double2 z = __ldg(reinterpret_cast<const double2*>(zp + (cb + k) * ld));
            tv = z.x * s0 + z.y * s1;
          }
          t[k] = tv;
        }
        // 16 column sums over 32 lanes: fold 16 → 1 values over xor 16, 8, 4, 2, then one plain stage
#pragma unroll
        for (int h = 8, m = 16; h >= 1; h >>= 1, m >>= 1) {
          const bool up = lane & m;
#pragma unroll
          for (int k = 0; k < h; ++k) {
            const double send = up ? t[k] : t[k + h];
            const double keep = up ? t[k + h] : t[k];
            t[k] = keep + __shfl_xor_sync(0xffffffffu, send, m);
          }
        }
        double r0 = t[0];
        r0 += __shfl_xor_sync(0xffffffffu, r0, 1);
        if ((lane & 1) == 0) {   // lane bits (16, 8, 4, 2) select k = 8·b16 + 4·b8 + 2·b4 + b2
          const int k = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
          if (cb + k < T.nc) atomicAdd(x + T.col0 + cb + k, r0);
        }
      }
    }
  }
  tl_end(6, tls);
}
// ---- small supernodes (≤ 16 columns), one WARP per supernode, every load issued before any arithmetic.
// The 16-lane kernels above (k_lvl_fwd / k_lvl_bwd) load the first 16 rows of L_rows up front and the rest in
// passes of 16 after the solve: with 40–90 rows per supernode that is 4–6 dependent memory round trips, and
// the round trips, not the bytes, set the time of a level (c2: 23 µs forward / 30 µs backward per level for
// 47 MB).  Here lane ↔ row (two passes of 32 rows in registers, further passes looped), the two half-warps
// split the columns of L_bb⁻¹, and a supernode costs one round trip.
// LOCAL: accumulators / x of the rows live in a shared-memory frame (subtrees), rows are frame indices.
constexpr int SNW_P = 2;   // row passes held in registers
template <bool LOCAL>
__device__ __forceinline__ void sn16_fwd(const double* __restrict__ L, const double* __restrict__ inv,
                                         const int32_t* __restrict__ rows, int wk, int noff, double b,
                                         const double* accp /* this supernode's accumulators (lane & 15) */,
                                         double* accw /* base for the row updates */, double* xdst) {
  const int wl = threadIdx.x & 31, i = wl & 15, h = wl >> 4;
  double a = 0.0;
  if (i < wk) a = LOCAL ? accp[i] : __ldcg(accp + i);
  double iv[8];   // half h: L_bb⁻¹(i, j), j = 8h + k
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int j = 8 * h + k;
    iv[k] = (j < wk && j <= i && i < wk) ? __ldg(inv + j * wk + i) : 0.0;
  }
  double lr[SNW_P][16];
  int32_t rw[SNW_P];
#pragma unroll
  for (int p = 0; p < SNW_P; ++p) {
    const int r = wl + 32 * p;
    const bool ok = r < noff;
    rw[p] = ok ? __ldg(rows + r) : 0;
#pragma unroll
    for (int c = 0; c < 16; ++c) lr[p][c] = (ok && c < wk) ? __ldg(L + r + (int64_t)c * noff) : 0.0;
  }
  const double v = b - a;
  double y = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) y += iv[k] * __shfl_sync(0xffffffffu, v, 8 * h + k);
  y += __shfl_xor_sync(0xffffffffu, y, 16);
  if (wl < wk) xdst[wl] = y;
  double sacc[SNW_P];
#pragma unroll
  for (int p = 0; p < SNW_P; ++p) sacc[p] = 0.0;
#pragma unroll
  for (int c = 0; c < 16; ++c) {   // y_c broadcast once per column, used by every pass (no y array in registers)
    const double yc = __shfl_sync(0xffffffffu, y, c);
#pragma unroll
    for (int p = 0; p < SNW_P; ++p) sacc[p] = fma(lr[p][c], yc, sacc[p]);
  }
#pragma unroll
  for (int p = 0; p < SNW_P; ++p)
    if (wl + 32 * p < noff) atomicAdd(accw + rw[p], sacc[p]);
  for (int r0 = 32 * SNW_P; r0 < noff; r0 += 32) {
    const int r = r0 + wl;
    const bool ok = r < noff;
    const int32_t g = ok ? __ldg(rows + r) : 0;
    double s2 = 0.0;
#pragma unroll
    for (int c = 0; c < 16; ++c)
      s2 += ((ok && c < wk) ? __ldg(L + r + (int64_t)c * noff) : 0.0) * __shfl_sync(0xffffffffu, y, c);
    if (ok) atomicAdd(accw + g, s2);
  }
}
template <bool LOCAL>
__device__ __forceinline__ double sn16_bwd(const double* __restrict__ L, const double* __restrict__ inv,
                                           const int32_t* __restrict__ rows, int wk, int noff, double yv, double dpiv,
                                           const double* xr_base) {
  const int wl = threadIdx.x & 31, i = wl & 15, h = wl >> 4;
  double ivt[8];   // half h: L_bb⁻¹(j, i), j = 8h + k ≥ i
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int j = 8 * h + k;
    ivt[k] = (j < wk && j >= i && i < wk) ? __ldg(inv + i * wk + j) : 0.0;
  }
  double lr[SNW_P][16];
  double xr[SNW_P];
#pragma unroll
  for (int p = 0; p < SNW_P; ++p) {
    const int r = wl + 32 * p;
    const bool ok = r < noff;
    const int32_t g = ok ? __ldg(rows + r) : 0;
#pragma unroll
    for (int c = 0; c < 16; ++c) lr[p][c] = (ok && c < wk) ? __ldg(L + r + (int64_t)c * noff) : 0.0;
    xr[p] = ok ? (LOCAL ? xr_base[g] : __ldcg(xr_base + g)) : 0.0;
  }
  double t[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    t[c] = 0.0;
#pragma unroll
    for (int p = 0; p < SNW_P; ++p) t[c] = fma(lr[p][c], xr[p], t[c]);
  }
  for (int r0 = 32 * SNW_P; r0 < noff; r0 += 32) {
    const int r = r0 + wl;
    const bool ok = r < noff;
    const int32_t g = ok ? __ldg(rows + r) : 0;
    const double xv = ok ? (LOCAL ? xr_base[g] : __ldcg(xr_base + g)) : 0.0;
#pragma unroll
    for (int c = 0; c < 16; ++c) t[c] += ((ok && c < wk) ? __ldg(L + r + (int64_t)c * noff) : 0.0) * xv;
  }
  // 16 column sums over 32 lanes: halves added, then the transpose-reduce inside each half
#pragma unroll
  for (int c = 0; c < 16; ++c) t[c] += __shfl_xor_sync(0xffffffffu, t[c], 16);
  const double tc = group_treduce<16>(t, i, 0xffffffffu);
  const double rhs = i < wk ? yv / dpiv - tc : 0.0;
  double xi = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) xi += ivt[k] * __shfl_sync(0xffffffffu, rhs, 8 * h + k);
  xi += __shfl_xor_sync(0xffffffffu, xi, 16);
  return xi;   // x_i in lanes i and i + 16
}
// One level of the leaf phase, warp per supernode (levels whose supernodes have ≤ 16 columns).
__global__ void __launch_bounds__(NT, 2) k_lvl16_fwd(DevFactor F, SweepRhs R, double* x, int64_t i0, int64_t i1) {
  if (R.done_flag != nullptr && *((volatile const int*)R.done_flag)) return;
  const unsigned tls = tl_begin(8);
  const int64_t i = i0 + ((int64_t)blockIdx.x * NT + threadIdx.x) / 32;
  if (i < i1) {
    const int4 d0 = __ldg(F.lvl_desc + 2 * i), d1 = __ldg(F.lvl_desc + 2 * i + 1);
    const double* L = F.fstore + ((int64_t)(uint32_t)d0.x | ((int64_t)d0.y << 32));
    const double* inv = F.fstore + ((int64_t)(uint32_t)d0.z | ((int64_t)d0.w << 32));
    const int32_t* rows = F.sn_rows + ((int64_t)(uint32_t)d1.x | ((int64_t)d1.y << 32));
    const int64_t c0 = d1.z;
    const int wk = d1.w & 63, noff = (int)((unsigned)d1.w >> 6);
    const int li = threadIdx.x & 15;
    double b = 0.0;
    if (li < wk) {
      const int64_t c = c0 + li;
      if (R.ct.p != nullptr) b = c < R.ct.nrows ? csr_dot(R.ct, c, R.p) : 0.0;
      else b = R.rhs[R.in_perm ? R.in_perm[c] : c];
    }
    sn16_fwd<false>(L, inv, rows, wk, noff, b, F.acc + c0, F.acc, x + c0);
    __syncwarp();
    if ((threadIdx.x & 31) < wk) F.acc[c0 + (threadIdx.x & 31)] = 0.0;
  }
  tl_end(8, tls);
}
__global__ void __launch_bounds__(NT, 2) k_lvl16_bwd(DevFactor F, double* x, const int* done_flag, int64_t i0,
                                                     int64_t i1) {
  if (done_flag != nullptr && *((volatile const int*)done_flag)) return;
  const unsigned tls = tl_begin(9);
  const int64_t i = i0 + ((int64_t)blockIdx.x * NT + threadIdx.x) / 32;
  if (i < i1) {
    const int4 d0 = __ldg(F.lvl_desc + 2 * i), d1 = __ldg(F.lvl_desc + 2 * i + 1);
    const double* L = F.fstore + ((int64_t)(uint32_t)d0.x | ((int64_t)d0.y << 32));
    const double* inv = F.fstore + ((int64_t)(uint32_t)d0.z | ((int64_t)d0.w << 32));
    const int32_t* rows = F.sn_rows + ((int64_t)(uint32_t)d1.x | ((int64_t)d1.y << 32));
    const int64_t c0 = d1.z;
    const int wk = d1.w & 63, noff = (int)((unsigned)d1.w >> 6);
    const int li = threadIdx.x & 15;
    double yv = 0.0, dp = 1.0;
    if (li < wk) {
      yv = __ldcg(x + c0 + li);
      dp = __ldg(F.Dpiv + c0 + li);
    }
    const double xi = sn16_bwd<false>(L, inv, rows, wk, noff, yv, dp, x);
    if ((threadIdx.x & 31) < wk) x[c0 + (threadIdx.x & 31)] = xi;
  }
  tl_end(9, tls);
}

// ---- subtrees: one WARP per subtree (StHdr), groups of G lanes per supernode, the frame in shared memory.
// A CTA-wide version (a CTA per subtree, __syncthreads between local levels) left most of its threads idle
// above the subtree's leaves and took 37 µs per subtree (c2: 357 µs forward against 163 µs for the level
// kernels); with a warp per subtree nearly every subtree is resident at once and the per-subtree latency
// overlaps across warps.
constexpr int ST_WPB = NT / 32;   // subtrees per CTA
template <int G>
__global__ void __launch_bounds__(NT, G == 16 ? 3 : 2) k_st_fwd(DevFactor F, SweepRhs R, PiSweep P, double* x) {
  if (R.done_flag != nullptr && *((volatile const int*)R.done_flag)) return;
  const unsigned tls = tl_begin(8);
  __shared__ double frs[ST_WPB][ST_FRAME];
  __shared__ int4 sds[ST_WPB][2 * ST_MAXSN];
  const int tid = threadIdx.x, wl = tid & 31, wid = tid >> 5;
  const int64_t t = (int64_t)blockIdx.x * ST_WPB + wid;
  if (t < P.st_n) {
    double* fr = frs[wid];
    const StHdr* hp = P.st_hdr + t;
    const int d0 = __ldg(&hp->d0), nlev = __ldg(&hp->nlev), c_lo = __ldg(&hp->c_lo), ncols = __ldg(&hp->ncols);
    const int next = __ldg(&hp->next), lp = __ldg(&hp->lptr), fslen = __ldg(&hp->fslen);
    const int64_t fslo = __ldg(&hp->fslo);
    for (int64_t e = (int64_t)wl * 16; e < fslen; e += 32 * 16) prefetch_l2(F.fstore + fslo + e);
    // the subtree's descriptors and level pointers staged once (one round trip instead of one per supernode)
    int4* sd = sds[wid];
    const int lpv = wl <= nlev ? __ldg(P.st_lptr + lp + wl) : 0;
    const int nsn = __shfl_sync(0xffffffffu, lpv, nlev);
    for (int i = wl; i < 2 * nsn; i += 32) sd[i] = __ldg(P.st_desc + 2 * (int64_t)d0 + i);
    for (int i = wl; i < ncols + next; i += 32) fr[i] = 0.0;
    __syncwarp();
    {
      const int4 f1 = sd[1], l1 = sd[2 * nsn - 1];
      const int64_t lo0 = (int64_t)(uint32_t)f1.x | ((int64_t)f1.y << 32);
      const int64_t lo1 = ((int64_t)(uint32_t)l1.x | ((int64_t)l1.y << 32)) + (int64_t)((unsigned)l1.w >> 6);
      for (int64_t e = lo0 + (int64_t)wl * 32; e < lo1; e += 32 * 32) prefetch_l2(P.st_loc + e);
    }
    const unsigned gm = lvl_mask<G>();
    const int lane = tid & (G - 1), grp = wl / G;
    for (int l = 0; l < nlev; ++l) {
      const int i0 = __shfl_sync(0xffffffffu, lpv, l), i1 = __shfl_sync(0xffffffffu, lpv, l + 1);
      for (int i = i0 + grp; i < i1; i += 32 / G) {
        const int4 a0 = sd[2 * i], a1 = sd[2 * i + 1];
        const double* L = F.fstore + ((int64_t)(uint32_t)a0.x | ((int64_t)a0.y << 32));
        const double* inv = F.fstore + ((int64_t)(uint32_t)a0.z | ((int64_t)a0.w << 32));
        const int32_t* loc = P.st_loc + ((int64_t)(uint32_t)a1.x | ((int64_t)a1.y << 32));
        const int c0 = a1.z;
        const int wk = a1.w & 63, noff = (int)((unsigned)a1.w >> 6);
        double v = 0.0;
        if (lane < wk) {
          const int64_t c = (int64_t)c0 + lane;
          if (R.ct.p != nullptr) v = c < R.ct.nrows ? csr_dot(R.ct, c, R.p) : 0.0;
          else v = R.rhs[R.in_perm ? R.in_perm[c] : c];
        }
        double iv[G];   // lane i: L_bb⁻¹(i, j) = inv[j·wk + i], j ≤ i
#pragma unroll
        for (int j = 0; j < G; ++j) iv[j] = (j < wk && j <= lane && lane < wk) ? __ldg(inv + j * wk + lane) : 0.0;
        const bool rok = lane < noff;
        const int32_t row = rok ? __ldg(loc + lane) : 0;
        double lr[G];   // lane r: L(r, c)
#pragma unroll
        for (int c = 0; c < G; ++c) lr[c] = (c < wk && rok) ? __ldg(L + lane + (int64_t)c * noff) : 0.0;
        if (lane < wk) v -= fr[c0 - c_lo + lane];
        double y = 0.0;
#pragma unroll
        for (int j = 0; j < G; ++j) y += iv[j] * __shfl_sync(gm, v, j, G);
        if (lane < wk) x[c0 + lane] = y;
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < G; ++c) s += lr[c] * __shfl_sync(gm, y, c, G);
        if (rok) atomicAdd(fr + row, s);
        for (int r0 = G; r0 < noff; r0 += G) {
          const int r = r0 + lane;
          const bool ok = r < noff;
          const int32_t rw = ok ? __ldg(loc + r) : 0;
          double s2 = 0.0;
#pragma unroll
          for (int c = 0; c < G; ++c) {
            const double lv = (c < wk && ok) ? __ldg(L + r + (int64_t)c * noff) : 0.0;
            s2 += lv * __shfl_sync(gm, y, c, G);
          }
          if (ok) atomicAdd(fr + rw, s2);
        }
      }
      __syncwarp();
    }
    const int32_t* rr = F.sn_rows + __ldg(&hp->rootrows);
    for (int e = wl; e < next; e += 32) atomicAdd(F.acc + __ldg(rr + e), fr[ncols + e]);
  }
  tl_end(8, tls);
}
template <int G>
__global__ void __launch_bounds__(NT, G == 16 ? 3 : 2) k_st_bwd(DevFactor F, PiSweep P, double* x, const int* done_flag) {
  if (done_flag != nullptr && *((volatile const int*)done_flag)) return;
  const unsigned tls = tl_begin(9);
  __shared__ double frs[ST_WPB][ST_FRAME];
  __shared__ int4 sds[ST_WPB][2 * ST_MAXSN];
  const int tid = threadIdx.x, wl = tid & 31, wid = tid >> 5;
  const int64_t t = (int64_t)blockIdx.x * ST_WPB + wid;
  if (t < P.st_n) {
    double* fr = frs[wid];
    const StHdr* hp = P.st_hdr + t;
    const int d0 = __ldg(&hp->d0), nlev = __ldg(&hp->nlev), c_lo = __ldg(&hp->c_lo), ncols = __ldg(&hp->ncols);
    const int next = __ldg(&hp->next), lp = __ldg(&hp->lptr), fslen = __ldg(&hp->fslen);
    const int64_t fslo = __ldg(&hp->fslo);
    for (int64_t e = (int64_t)wl * 16; e < fslen; e += 32 * 16) prefetch_l2(F.fstore + fslo + e);
    int4* sd = sds[wid];
    const int lpv = wl <= nlev ? __ldg(P.st_lptr + lp + wl) : 0;
    const int nsn = __shfl_sync(0xffffffffu, lpv, nlev);
    for (int i = wl; i < 2 * nsn; i += 32) sd[i] = __ldg(P.st_desc + 2 * (int64_t)d0 + i);
    const int32_t* rr = F.sn_rows + __ldg(&hp->rootrows);
    for (int e = wl; e < next; e += 32) fr[ncols + e] = __ldcg(x + __ldg(rr + e));
    __syncwarp();
    {
      const int4 f1 = sd[1], l1 = sd[2 * nsn - 1];
      const int64_t lo0 = (int64_t)(uint32_t)f1.x | ((int64_t)f1.y << 32);
      const int64_t lo1 = ((int64_t)(uint32_t)l1.x | ((int64_t)l1.y << 32)) + (int64_t)((unsigned)l1.w >> 6);
      for (int64_t e = lo0 + (int64_t)wl * 32; e < lo1; e += 32 * 32) prefetch_l2(P.st_loc + e);
    }
    const unsigned gm = lvl_mask<G>();
    const int lane = tid & (G - 1), grp = wl / G;
    for (int l = nlev - 1; l >= 0; --l) {
      const int i0 = __shfl_sync(0xffffffffu, lpv, l), i1 = __shfl_sync(0xffffffffu, lpv, l + 1);
      for (int i = i0 + grp; i < i1; i += 32 / G) {
        const int4 a0 = sd[2 * i], a1 = sd[2 * i + 1];
        const double* L = F.fstore + ((int64_t)(uint32_t)a0.x | ((int64_t)a0.y << 32));
        const double* inv = F.fstore + ((int64_t)(uint32_t)a0.z | ((int64_t)a0.w << 32));
        const int32_t* loc = P.st_loc + ((int64_t)(uint32_t)a1.x | ((int64_t)a1.y << 32));
        const int c0 = a1.z;
        const int wk = a1.w & 63, noff = (int)((unsigned)a1.w >> 6);
        double yv = 0.0, dinv = 0.0;
        if (lane < wk) {
          yv = __ldcg(x + c0 + lane);
          dinv = 1.0 / __ldg(F.Dpiv + c0 + lane);
        }
        double ivt[G];   // lane i: L_bb⁻¹(j, i) = inv[i·wk + j], j ≥ i
#pragma unroll
        for (int j = 0; j < G; ++j) ivt[j] = (j < wk && j >= lane && lane < wk) ? __ldg(inv + lane * wk + j) : 0.0;
        double tt[G];
#pragma unroll
        for (int c = 0; c < G; ++c) tt[c] = 0.0;
        for (int r0 = 0; r0 < noff; r0 += G) {
          const int r = r0 + lane;
          const bool ok = r < noff;
          const double xr = ok ? fr[__ldg(loc + r)] : 0.0;
#pragma unroll
          for (int c = 0; c < G; ++c) tt[c] += ((c < wk && ok) ? __ldg(L + r + (int64_t)c * noff) : 0.0) * xr;
        }
        const double tc = group_treduce<G>(tt, lane, gm);
        const double rhs = lane < wk ? yv * dinv - tc : 0.0;
        double xi = 0.0;
#pragma unroll
        for (int j = 0; j < G; ++j) xi += ivt[j] * __shfl_sync(gm, rhs, j, G);
        if (lane < wk) {
          x[c0 + lane] = xi;
          fr[c0 - c_lo + lane] = xi;
        }
      }
      __syncwarp();
    }
  }
  tl_end(9, tls);
}
// Subtrees of ≤ 16-column supernodes: a warp per subtree, the whole warp on one supernode at a time
// (sn16_fwd / sn16_bwd: one round trip per supernode, served by L2 after the subtree's prefetch).  128 registers,
// 2 CTAs per SM: at 3 CTAs per SM (80 registers, 152 bytes of spills) the kernels took 208 / 179 µs on c2 instead of
// 110 / 111 µs.
__global__ void __launch_bounds__(NT, 2) k_st16_fwd(DevFactor F, SweepRhs R, PiSweep P, double* x) {
  grid_dep_wait();
  grid_dep_launch();
  if (R.done_flag != nullptr && *((volatile const int*)R.done_flag)) return;
  const unsigned tls = tl_begin(8);
  __shared__ double frs[ST_WPB][ST_FRAME];
  __shared__ int4 sds[ST_WPB][2 * ST_MAXSN];
  const int tid = threadIdx.x, wl = tid & 31, wid = tid >> 5;
  const int64_t t = (int64_t)blockIdx.x * ST_WPB + wid;
  if (t < P.st_n) {
    double* fr = frs[wid];
    const StHdr* hp = P.st_hdr + t;
    const int d0 = __ldg(&hp->d0), nlev = __ldg(&hp->nlev), c_lo = __ldg(&hp->c_lo), ncols = __ldg(&hp->ncols);
    const int next = __ldg(&hp->next), lp = __ldg(&hp->lptr), fslen = __ldg(&hp->fslen);
    const int64_t fslo = __ldg(&hp->fslo);
    for (int64_t e = (int64_t)wl * 16; e < fslen; e += 32 * 16) prefetch_l2(F.fstore + fslo + e);
    int4* sd = sds[wid];
    const int lpv = wl <= nlev ? __ldg(P.st_lptr + lp + wl) : 0;
    const int nsn = __shfl_sync(0xffffffffu, lpv, nlev);
    for (int i = wl; i < 2 * nsn; i += 32) sd[i] = __ldg(P.st_desc + 2 * (int64_t)d0 + i);
    for (int i = wl; i < ncols + next; i += 32) fr[i] = 0.0;
    __syncwarp();
    {
      const int4 f1 = sd[1], l1 = sd[2 * nsn - 1];
      const int64_t lo0 = (int64_t)(uint32_t)f1.x | ((int64_t)f1.y << 32);
      const int64_t lo1 = ((int64_t)(uint32_t)l1.x | ((int64_t)l1.y << 32)) + (int64_t)((unsigned)l1.w >> 6);
      for (int64_t e = lo0 + (int64_t)wl * 32; e < lo1; e += 32 * 32) prefetch_l2(P.st_loc + e);
    }
    for (int l = 0; l < nlev; ++l) {
      const int i0 = __shfl_sync(0xffffffffu, lpv, l), i1 = __shfl_sync(0xffffffffu, lpv, l + 1);
      for (int i = i0; i < i1; ++i) {
        const int4 a0 = sd[2 * i], a1 = sd[2 * i + 1];
        const double* L = F.fstore + ((int64_t)(uint32_t)a0.x | ((int64_t)a0.y << 32));
        const double* inv = F.fstore + ((int64_t)(uint32_t)a0.z | ((int64_t)a0.w << 32));
        const int32_t* loc = P.st_loc + ((int64_t)(uint32_t)a1.x | ((int64_t)a1.y << 32));
        const int c0 = a1.z;
        const int wk = a1.w & 63, noff = (int)((unsigned)a1.w >> 6);
        double b = 0.0;
        if ((wl & 15) < wk) {
          const int64_t c = (int64_t)c0 + (wl & 15);
          if (R.ct.p != nullptr) b = c < R.ct.nrows ? csr_dot(R.ct, c, R.p) : 0.0;
          else b = R.rhs[R.in_perm ? R.in_perm[c] : c];
        }
        sn16_fwd<true>(L, inv, loc, wk, noff, b, fr + (c0 - c_lo), fr, x + c0);
      }
      __syncwarp();
    }
    const int32_t* rr = F.sn_rows + __ldg(&hp->rootrows);
    for (int e = wl; e < next; e += 32) atomicAdd(F.acc + __ldg(rr + e), fr[ncols + e]);
  }
  tl_end(8, tls);
}
__global__ void __launch_bounds__(NT, 2) k_st16_bwd(DevFactor F, PiSweep P, double* x, const int* done_flag) {
  grid_dep_wait();
  grid_dep_launch();
  if (done_flag != nullptr && *((volatile const int*)done_flag)) return;
  const unsigned tls = tl_begin(9);
  __shared__ double frs[ST_WPB][ST_FRAME];
  __shared__ int4 sds[ST_WPB][2 * ST_MAXSN];
  const int tid = threadIdx.x, wl = tid & 31, wid = tid >> 5;
  const int64_t t = (int64_t)blockIdx.x * ST_WPB + wid;
  if (t < P.st_n) {
    double* fr = frs[wid];
    const StHdr* hp = P.st_hdr + t;
    const int d0 = __ldg(&hp->d0), nlev = __ldg(&hp->nlev), c_lo = __ldg(&hp->c_lo), ncols = __ldg(&hp->ncols);
    const int next = __ldg(&hp->next), lp = __ldg(&hp->lptr), fslen = __ldg(&hp->fslen);
    const int64_t fslo = __ldg(&hp->fslo);
    for (int64_t e = (int64_t)wl * 16; e < fslen; e += 32 * 16) prefetch_l2(F.fstore + fslo + e);
    int4* sd = sds[wid];
    const int lpv = wl <= nlev ? __ldg(P.st_lptr + lp + wl) : 0;
    const int nsn = __shfl_sync(0xffffffffu, lpv, nlev);
    for (int i = wl; i < 2 * nsn; i += 32) sd[i] = __ldg(P.st_desc + 2 * (int64_t)d0 + i);
    const int32_t* rr = F.sn_rows + __ldg(&hp->rootrows);
    for (int e = wl; e < next; e += 32) fr[ncols + e] = __ldcg(x + __ldg(rr + e));
    __syncwarp();
    {
      const int4 f1 = sd[1], l1 = sd[2 * nsn - 1];
      const int64_t lo0 = (int64_t)(uint32_t)f1.x | ((int64_t)f1.y << 32);
      const int64_t lo1 = ((int64_t)(uint32_t)l1.x | ((int64_t)l1.y << 32)) + (int64_t)((unsigned)l1.w >> 6);
      for (int64_t e = lo0 + (int64_t)wl * 32; e < lo1; e += 32 * 32) prefetch_l2(P.st_loc + e);
    }
    for (int l = nlev - 1; l >= 0; --l) {
      const int i0 = __shfl_sync(0xffffffffu, lpv, l), i1 = __shfl_sync(0xffffffffu, lpv, l + 1);
      for (int i = i0; i < i1; ++i) {
        const int4 a0 = sd[2 * i], a1 = sd[2 * i + 1];
        const double* L = F.fstore + ((int64_t)(uint32_t)a0.x | ((int64_t)a0.y << 32));
        const double* inv = F.fstore + ((int64_t)(uint32_t)a0.z | ((int64_t)a0.w << 32));
        const int32_t* loc = P.st_loc + ((int64_t)(uint32_t)a1.x | ((int64_t)a1.y << 32));
        const int c0 = a1.z;
        const int wk = a1.w & 63, noff = (int)((unsigned)a1.w >> 6);
        double yv = 0.0, dp = 1.0;
        if ((wl & 15) < wk) {
          yv = __ldcg(x + c0 + (wl & 15));
          dp = __ldg(F.Dpiv + c0 + (wl & 15));
        }
        const double xi = sn16_bwd<true>(L, inv, loc, wk, noff, yv, dp, fr);
        if (wl < wk) {
          x[c0 + wl] = xi;
          fr[c0 - c_lo + wl] = xi;
        }
      }
      __syncwarp();
    }
  }
  tl_end(9, tls);
}
// Launch with programmatic stream serialization (QPB_PDL=0: a plain launch): the kernel must start with
// grid_dep_wait().
static bool pdl_on() {
  static const bool on = !(std::getenv("QPB_PDL") && std::getenv("QPB_PDL")[0] == '0');
  return on;
}
template <class... KA, class... A>
static void launch_dep(void (*k)(KA...), unsigned grid, cudaStream_t s, A... a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, a...);
}
void pi_build(const DevFactor& F, const PiSweep& P, const int64_t* zoffJ, cudaStream_t s) {
  const int64_t nt = P.lev_ptr[P.nlev];
  if (nt <= 0) return;
  cudaMemsetAsync(P.Z, 0, (size_t)P.z_size * sizeof(double), s);
  k_pi_build_x<<<(unsigned)nt, NT, 0, s>>>(F, P.tiles, P.tile_J, P.Z, nt);
  k_pi_build_y<<<(unsigned)nt, NT, 0, s>>>(F, P.tiles, P.tile_J, P.Z, zoffJ, nt);
}
void pi_init(const DevFactor& F, const PiSweep& P, const SweepRhs& r, double* x, int sms, cudaStream_t s) {
  k_pi_init<<<sms * 4, NT, 0, s>>>(F, r, x, P.root0);
}
void pi_forward(const DevFactor& F, const PiSweep& P, const SweepRhs& r, double* x, int sms, cudaStream_t s) {
  if (!r.rhs_ready) k_pi_init<<<sms * 4, NT, 0, s>>>(F, r, x, P.root0);
  if (P.st_n > 0) {
    if (P.st_g == 16 && lvl16_on()) launch_dep(k_st16_fwd, (unsigned)((P.st_n + ST_WPB - 1) / ST_WPB), s, F, r, P, x);
    else if (P.st_g == 16) k_st_fwd<16><<<(unsigned)((P.st_n + ST_WPB - 1) / ST_WPB), NT, 0, s>>>(F, r, P, x);
    else k_st_fwd<32><<<(unsigned)((P.st_n + ST_WPB - 1) / ST_WPB), NT, 0, s>>>(F, r, P, x);
  }
  for (int L = 0; P.st_n == 0 && L < F.lvl_cut; ++L) {   // leaf phase, bottom level first
    const int64_t i0 = F.lvl_ptr_h[L], i1 = F.lvl_ptr_h[L + 1];
    const int G = F.lvl_g_h[L];
    const int g = (int)((i1 - i0) * G + NT - 1) / NT;
    if (G == 16 && lvl16_on()) k_lvl16_fwd<<<(unsigned)(((i1 - i0) * 32 + NT - 1) / NT), NT, 0, s>>>(F, r, x, i0, i1);
    else if (G == 16) k_lvl_fwd<16><<<g, NT, 0, s>>>(F, r, x, i0, i1);
    else k_lvl_fwd<32><<<g, NT, 0, s>>>(F, r, x, i0, i1);
  }
  for (int L = 0; L < P.nlev; ++L) {
    const int64_t nbig = P.lev_sptr[L] - P.lev_ptr[L], nstrip = P.lev_ptr[L + 1] - P.lev_sptr[L];
    const int64_t n = nbig + (nstrip + NT / 32 - 1) / (NT / 32);
    if (n > 0) launch_dep(k_pi_fwd, (unsigned)n, s, F, r, P.tiles + P.lev_ptr[L], (int)nbig, (int)nstrip, (const double*)P.Z, P.prefetch);
  }
}
void pi_backward(const DevFactor& F, const PiSweep& P, double* x, const int* done_flag, cudaStream_t s) {
  for (int L = P.nlev - 1; L >= 0; --L) {
    const int64_t nbig = P.blev_sptr[L] - P.blev_ptr[L], nstrip = P.blev_ptr[L + 1] - P.blev_sptr[L];
    const int64_t n = nbig + (nstrip + NT / 32 - 1) / (NT / 32);
    if (n > 0)
      launch_dep(k_pi_bwd, (unsigned)n, s, F, P.btiles + P.blev_ptr[L], (int)nbig, (int)nstrip, (const double*)P.Z, x,
                 done_flag, P.prefetch);
  }
  if (P.st_n > 0) {
    if (P.st_g == 16 && lvl16_on()) launch_dep(k_st16_bwd, (unsigned)((P.st_n + ST_WPB - 1) / ST_WPB), s, F, P, x, done_flag);
    else if (P.st_g == 16) k_st_bwd<16><<<(unsigned)((P.st_n + ST_WPB - 1) / ST_WPB), NT, 0, s>>>(F, P, x, done_flag);
    else k_st_bwd<32><<<(unsigned)((P.st_n + ST_WPB - 1) / ST_WPB), NT, 0, s>>>(F, P, x, done_flag);
  }
  for (int L = P.st_n > 0 ? -1 : F.lvl_cut - 1; L >= 0; --L) {   // leaf phase, top level first
    const int64_t i0 = F.lvl_ptr_h[L], i1 = F.lvl_ptr_h[L + 1];
    const int G = F.lvl_g_h[L];
    const int g = (int)((i1 - i0) * G + NT - 1) / NT;
    if (G == 16 && lvl16_on()) k_lvl16_bwd<<<(unsigned)(((i1 - i0) * 32 + NT - 1) / NT), NT, 0, s>>>(F, x, done_flag, i0, i1);
    else if (G == 16) k_lvl_bwd<16><<<g, NT, 0, s>>>(F, x, done_flag, i0, i1);
    else k_lvl_bwd<32><<<g, NT, 0, s>>>(F, x, done_flag, i0, i1);
  }
}

// ------------------------------------------------------------------------- reduction finalizers
// Each takes the GLOBAL reduced values (local ones when not sharded) and updates the state.
__device__ void fin_pcg_init(PcgState* st, double bb, double rz) {
  st->bnorm2 = bb;
  st->rr = bb;
  st->rho = rz;
  st->done = (bb == 0.0) ? 1 : 0;
  if (st->maxit <= 0 && bb != 0.0) {
    st->done = 1;
    st->status = 1;
  }
}
__device__ void fin_pcg_pq(PcgState* st, double pq) {
  st->pq = pq;
  if (!(pq > 0.0) || !isfinite(pq)) {
    st->status = -3;
    st->done = 1;
  } else {
    st->alpha = st->rho / pq;
  }
}
__device__ void fin_pcg_upd1(PcgState* st, double rr, double rz, int prec) {
  st->iter += 1;
  st->rr = rr;
  if (!isfinite(rr)) {
    st->status = -3;
    st->done = 1;
  } else if (rr <= st->tol2 * st->bnorm2) {
    st->done = 1;
  } else if (st->iter >= st->maxit) {
    st->done = 1;
    st->status = 1;
  } else if (prec != 2) {
    st->beta = rz / st->rho;
    st->rho = rz;
    st->rz = rz;
  }
}
__device__ void fin_pcg_rz_ph(PcgState* st, double rz) {
  st->beta = rz / st->rho;
  st->rho = rz;
  st->rz = rz;
}
__device__ void fin_ipm_mu(IpmState* st, double smu) {
  st->mu = smu / st->m2_total;   // μ = sᵀν / m2
  st->sigma_mu = st->sigma * st->mu;
}
__device__ void fin_ipm_resid(IpmState* st, double a1, double a2, double a3) {
  st->rg_inf = a1;
  st->re_inf = a2;
  st->ri_inf = a3;
}
__device__ void fin_ipm_alpha(IpmState* st, double a) {
  st->alpha_max = a;
  st->alpha = fmin(1.0, st->tau * a);
}

__global__ void k_finalize(int kind, PcgState* ps, IpmState* is, int prec) {
  if (threadIdx.x != 0) return;
  if (kind <= FIN_PCG_RZ_PH && *((volatile int*)&ps->done) && kind != FIN_PCG_INIT) return;
  switch (kind) {
    case FIN_PCG_INIT: fin_pcg_init(ps, ps->red[0], ps->red[1]); break;
    case FIN_PCG_PQ: fin_pcg_pq(ps, ps->red[0]); break;
    case FIN_PCG_UPD1: fin_pcg_upd1(ps, ps->red[0], ps->red[1], prec); break;
    case FIN_PCG_INIT_PH: ps->rho = ps->red[0]; break;
    case FIN_PCG_RZ_PH: fin_pcg_rz_ph(ps, ps->red[0]); break;
    case FIN_IPM_MU: fin_ipm_mu(is, is->red[0]); break;
    case FIN_IPM_RESID: fin_ipm_resid(is, is->red[0], is->red[1], is->red[2]); break;
    case FIN_IPM_ALPHA: fin_ipm_alpha(is, is->red[0]); break;
  }
}
void finalize(int kind, PcgState* ps, IpmState* is, int prec, cudaStream_t s) {
  k_finalize<<<1, 32, 0, s>>>(kind, ps, is, prec);
}

__global__ void k_spmv(DevCSR M, const double* x, double* y, const int* done) {
  if (done != nullptr && *((volatile const int*)done)) return;
  const unsigned tls = tl_begin(7);
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < M.nrows; i += (int64_t)gridDim.x * NT)
    y[i] = csr_dot(M, i, x);
  tl_end(7, tls);
}
void spmv(const DevCSR& M, const double* x, double* y, const int* done, int grid, cudaStream_t s) {
  k_spmv<<<grid, NT, 0, s>>>(M, x, y, done);
}

// ------------------------------------------------------------------------- K_F product and PCG
// q = D∘p − C_f·z (a5) with the pᵀq reduction; last block: α = ρ / pᵀq.
// Row part of q = D∘p − C·z shared by k_kf_q and k_pcg_step: rows with ≤ KF_LONG_ROW entries thread per
// row, the listed long rows (power-law degrees) warp per row with 4 loads in flight per lane; returns the
// thread's share of pᵀq.
template <int B = 4>
__device__ __forceinline__ double kf_rows(const DevCSR& Cf, const int32_t* longr, int64_t nlong, const double* D,
                                          const double* p, const double* z, double* q) {
  const int64_t i0 = blockIdx.x * (int64_t)NT + threadIdx.x, stride = (int64_t)gridDim.x * NT;
  double loc = 0.0;
  for (int64_t i = i0; i < Cf.nrows; i += stride) {
    if (nlong > 0 && Cf.p[i + 1] - Cf.p[i] > KF_LONG_ROW) continue;
    const double pi = p[i];
    const double qi = D[i] * pi - csr_dot<B>(Cf, i, z);
    q[i] = qi;
    loc += pi * qi;
  }
  const int lane = threadIdx.x & 31;
  for (int64_t j = (i0 >> 5); j < nlong; j += stride >> 5) {
    const int64_t i = longr[j];
    const int64_t e0 = Cf.p[i], e1 = Cf.p[i + 1];
    double s = 0.0;
    for (int64_t e = e0 + lane; e < e1; e += 128) {
      double v4[4];
      int32_t c4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool ok = e + 32 * u < e1;
        v4[u] = ok ? Cf.v[e + 32 * u] : 0.0;
        c4[u] = ok ? Cf.i[e + 32 * u] : 0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) s += v4[u] * __ldg(z + c4[u]);
    }
    s = warp_sum(s);
    if (lane == 0) {
      const double pi = p[i];
      const double qi = D[i] * pi - s;
      q[i] = qi;
      loc += pi * qi;
    }
  }
  return loc;
}

__global__ void __launch_bounds__(NT) k_kf_q(DevCSR Cf, const int32_t* longr, int64_t nlong, const double* D,
                                             const double* p, const double* z, double* q, double* partial,
                                             PcgState* st, int pcg_mode) {
  __shared__ double sh[32];
  if (pcg_mode && *((volatile int*)&st->done)) return;
  const double loc = kf_rows(Cf, longr, nlong, D, p, z, q);
  if (!pcg_mode) return;
  double v = block_reduce<0>(loc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
  if (is_last_block(&st->arrive)) {
    double pq = reduce_partials<0>(partial, gridDim.x, sh);
    if (threadIdx.x == 0) {
      if (st->defer) st->red[0] = pq;
      else fin_pcg_pq(st, pq);
      st->arrive = 0;
    }
  }
}

// init: x = 0, r = b, z = M⁻¹ r, p = z, ρ = rᵀz, ‖b‖²
__global__ void __launch_bounds__(NT) k_pcg_init(int prec, int64_t m2, const double* b, const double* D,
                                                 double* x, double* r, double* z, double* p, double* partial,
                                                 PcgState* st, double tol, int maxit) {
  __shared__ double sh[32];
  double bb = 0.0, rz = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < m2; i += (int64_t)gridDim.x * NT) {
    const double bi = b[i];
    x[i] = 0.0;
    r[i] = bi;
    bb += bi * bi;
    if (prec != 2) {
      const double zi = prec == 1 ? bi / D[i] : bi;
      z[i] = zi;
      p[i] = zi;
      rz += bi * zi;
    }
  }
  double v1 = block_reduce<0>(bb, sh);
  double v2 = block_reduce<0>(rz, sh);
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = v1;
    partial[gridDim.x + blockIdx.x] = v2;
  }
  if (is_last_block(&st->arrive)) {
    double s1 = reduce_partials<0>(partial, gridDim.x, sh);
    double s2 = reduce_partials<0>(partial + gridDim.x, gridDim.x, sh);
    if (threadIdx.x == 0) {
      st->tol2 = tol * tol;
      st->iter = 0;
      st->maxit = maxit;
      st->status = 0;
      if (st->defer) {
        st->red[0] = s1;
        st->red[1] = s2;
        st->done = 0;
      } else {
        fin_pcg_init(st, s1, s2);
      }
      st->arrive = 0;
    }
  }
}

// P_H init (after z = P_H⁻¹ r): p = z, ρ = rᵀz
__global__ void __launch_bounds__(NT) k_pcg_init_ph(int64_t m2, const double* r, const double* z, double* p,
                                                    double* partial, PcgState* st) {
  __shared__ double sh[32];
  if (*((volatile int*)&st->done)) return;
  double rz = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < m2; i += (int64_t)gridDim.x * NT) {
    p[i] = z[i];
    rz += r[i] * z[i];
  }
  double v = block_reduce<0>(rz, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
  if (is_last_block(&st->arrive)) {
    double s = reduce_partials<0>(partial, gridDim.x, sh);
    if (threadIdx.x == 0) {
      if (st->defer) st->red[0] = s;
      else st->rho = s;
      st->arrive = 0;
    }
  }
}

// x += αp; r −= αq; z = M⁻¹r (P_L / none); reductions ‖r‖², rᵀz; convergence; β.
__global__ void __launch_bounds__(NT) k_pcg_update1(int prec, int64_t m2, const double* D, const double* p,
                                                    const double* q, double* x, double* r, double* z,
                                                    double* partial, PcgState* st) {
  __shared__ double sh[32];
  if (*((volatile int*)&st->done)) return;
  const double alpha = st->alpha;
  double rr = 0.0, rz = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < m2; i += (int64_t)gridDim.x * NT) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    rr += ri * ri;
    if (prec != 2) {
      const double zi = prec == 1 ? ri / D[i] : ri;
      z[i] = zi;
      rz += ri * zi;
    }
  }
  double v1 = block_reduce<0>(rr, sh);
  double v2 = block_reduce<0>(rz, sh);
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = v1;
    partial[gridDim.x + blockIdx.x] = v2;
  }
  if (is_last_block(&st->arrive)) {
    double s1 = reduce_partials<0>(partial, gridDim.x, sh);
    double s2 = reduce_partials<0>(partial + gridDim.x, gridDim.x, sh);
    if (threadIdx.x == 0) {
      if (st->defer) {
        st->red[0] = s1;
        st->red[1] = s2;
      } else {
        fin_pcg_upd1(st, s1, s2, prec);
      }
      st->arrive = 0;
    }
  }
}

// P_H: ρ' = rᵀz after z = P_H⁻¹ r; β = ρ'/ρ.
__global__ void __launch_bounds__(NT) k_pcg_rz_ph(int64_t m2, const double* r, const double* z, double* partial,
                                                  PcgState* st) {
  __shared__ double sh[32];
  if (*((volatile int*)&st->done)) return;
  double rz = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < m2; i += (int64_t)gridDim.x * NT)
    rz += r[i] * z[i];
  double v = block_reduce<0>(rz, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
  if (is_last_block(&st->arrive)) {
    double s = reduce_partials<0>(partial, gridDim.x, sh);
    if (threadIdx.x == 0) {
      if (st->defer) st->red[0] = s;
      else fin_pcg_rz_ph(st, s);
      st->arrive = 0;
    }
  }
}

__global__ void __launch_bounds__(NT) k_pcg_update2(int64_t m2, const double* z, double* p, PcgState* st) {
  if (*((volatile int*)&st->done)) return;
  const double beta = st->beta;
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < m2; i += (int64_t)gridDim.x * NT)
    p[i] = z[i] + beta * p[i];
}

// Fused PCG tail for P_L / no preconditioner on one GPU (a5 + a6 in one cooperative launch):
//   q = D∘p − C·w, pᵀq  | grid sync |  α = ρ/pᵀq, x += αp, r −= αq, z = M⁻¹r, ‖r‖², rᵀz  | grid sync |
//   convergence test, β = ρ'/ρ, p = z + βp.
// The per-block partials are those of k_kf_q / k_pcg_update1 (same grid, same order), and every block
// reduces them itself with reduce_partials, so all blocks take the same decision without another
// round trip; the result equals the three-kernel sequence's up to the reduction order (those kernels
// run on the vector grid, this one on its own grid); block 0 writes the state.
// Phase A's partials live in partial[0, G), phase B's in partial[G, 3G), so no block overwrites a
// partial another block is still reading.
// QPB_STEP_B4=0: the large-m2 fused step one row per loop trip (A/B)
__device__ int g_step_b4 = 1;
__device__ __forceinline__ bool step_batch4() { return g_step_b4 != 0; }
// Four rows of a CSR product at once (rows r[u], valid where ok[u]): the four rows' pointer, entry and gather
// loads are issued together, so a thread that owns many rows of a grid-stride loop pays one dependent round
// trip per FOUR rows instead of per row (the large-m2 fused step was bound by exactly these round trips).
__device__ __forceinline__ void csr_dot4(const DevCSR& M, const int64_t (&r)[4], const bool (&ok)[4], const double* x,
                                         double (&s)[4]) {
  int64_t q0[4], q1[4];
  int64_t len = 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    q0[u] = ok[u] ? M.p[r[u]] : 0;
    q1[u] = ok[u] ? M.p[r[u] + 1] : 0;
    s[u] = 0.0;
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) len = q1[u] - q0[u] > len ? q1[u] - q0[u] : len;
  for (int64_t k = 0; k < len; ++k) {
    double v[4];
    int32_t c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool in = q0[u] + k < q1[u];
      v[u] = in ? M.v[q0[u] + k] : 0.0;
      c[u] = in ? M.i[q0[u] + k] : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) s[u] += v[u] * __ldg(x + c[u]);
  }
}
// kf_rows with the short rows taken four at a time (see csr_dot4); the long rows as in kf_rows.
__device__ __forceinline__ double kf_rows4(const DevCSR& Cf, const int32_t* longr, int64_t nlong, const double* D,
                                           const double* p, const double* z, double* q) {
  const int64_t i0 = blockIdx.x * (int64_t)NT + threadIdx.x, stride = (int64_t)gridDim.x * NT;
  double loc = 0.0;
  for (int64_t i = i0; i < Cf.nrows; i += 4 * stride) {
    int64_t r[4];
    bool ok[4];
    double pv[4], dv[4], s[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      r[u] = i + u * stride;
      ok[u] = r[u] < Cf.nrows;
      if (ok[u] && nlong > 0 && Cf.p[r[u] + 1] - Cf.p[r[u]] > KF_LONG_ROW) ok[u] = false;
      pv[u] = ok[u] ? p[r[u]] : 0.0;
      dv[u] = ok[u] ? D[r[u]] : 0.0;
    }
    csr_dot4(Cf, r, ok, z, s);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (ok[u]) {
        const double qi = dv[u] * pv[u] - s[u];
        q[r[u]] = qi;
        loc += pv[u] * qi;
      }
    }
  }
  const int lane = threadIdx.x & 31;
  for (int64_t j = (i0 >> 5); j < nlong; j += stride >> 5) {
    const int64_t i = longr[j];
    const int64_t e0 = Cf.p[i], e1 = Cf.p[i + 1];
    double s = 0.0;
    for (int64_t e = e0 + lane; e < e1; e += 128) {
      double v4[4];
      int32_t c4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool in = e + 32 * u < e1;
        v4[u] = in ? Cf.v[e + 32 * u] : 0.0;
        c4[u] = in ? Cf.i[e + 32 * u] : 0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) s += v4[u] * __ldg(z + c4[u]);
    }
    s = warp_sum(s);
    if (lane == 0) {
      const double pi = p[i];
      const double qi = D[i] * pi - s;
      q[i] = qi;
      loc += pi * qi;
    }
  }
  return loc;
}
template <int BA, int BD, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_pcg_step(DevCSR Cf, const int32_t* longr, int64_t nlong, int prec,
                                                 const double* D, double* p, const double* w, double* q, double* x,
                                                 double* r, double* z, double* partial, PcgState* st, int next_rhs,
                                                 DevFactor F, DevCSR Ct, double* xout, double* ubuf) {
  __shared__ double sh[32];
  if (*((volatile int*)&st->done)) return;   // every block reads the flag before the first grid sync
  cg::grid_group grid = cg::this_grid();
  const unsigned tls = tl_begin(4);
  const double rho = st->rho, tol2 = st->tol2, bnorm2 = st->bnorm2;
  const int iter = st->iter, maxit = st->maxit;
  const int64_t m2 = Cf.nrows, G = gridDim.x;
  const int64_t i0 = blockIdx.x * (int64_t)NT + threadIdx.x, stride = G * NT;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  const bool b4 = BA == 4 && step_batch4();   // large-m2 variant: four rows per loop trip in every phase
  const double loc = b4 ? kf_rows4(Cf, longr, nlong, D, p, w, q) : kf_rows<BA>(Cf, longr, nlong, D, p, w, q);
  double v = block_reduce<0>(loc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
  grid.sync();
  const double pq = reduce_partials<0>(partial, (int)G, sh);
  if (leader) fin_pcg_pq(st, pq);
  if (!(pq > 0.0) || !isfinite(pq)) {   // breakdown: fin_pcg_pq set status and done
    tl_end(4, tls);
    return;
  }
  const double alpha = rho / pq;
  double rr = 0.0, rz = 0.0;
  if (b4) {
    for (int64_t i = i0; i < m2; i += 4 * stride) {
      double xv[4], pv[4], rv[4], qv[4], dv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t j = i + u * stride;
        const bool ok = j < m2;
        xv[u] = ok ? x[j] : 0.0;
        pv[u] = ok ? p[j] : 0.0;
        rv[u] = ok ? r[j] : 0.0;
        qv[u] = ok ? q[j] : 0.0;
        dv[u] = ok && prec == 1 ? D[j] : 1.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t j = i + u * stride;
        if (j < m2) {
          x[j] = xv[u] + alpha * pv[u];
          const double ri = rv[u] - alpha * qv[u];
          r[j] = ri;
          rr += ri * ri;
          const double zi = prec == 1 ? ri / dv[u] : ri;
          z[j] = zi;
          rz += ri * zi;
        }
      }
    }
  } else {
    for (int64_t i = i0; i < m2; i += stride) {
      x[i] += alpha * p[i];
      const double ri = r[i] - alpha * q[i];
      r[i] = ri;
      rr += ri * ri;
      const double zi = prec == 1 ? ri / D[i] : ri;
      z[i] = zi;
      rz += ri * zi;
    }
  }
  const double v1 = block_reduce<0>(rr, sh);
  const double v2 = block_reduce<0>(rz, sh);
  if (threadIdx.x == 0) {
    partial[G + blockIdx.x] = v1;
    partial[2 * G + blockIdx.x] = v2;
  }
  grid.sync();
  const double s1 = reduce_partials<0>(partial + G, (int)G, sh);
  const double s2 = reduce_partials<0>(partial + 2 * G, (int)G, sh);
  if (leader) fin_pcg_upd1(st, s1, s2, prec);
  // the same decision as fin_pcg_upd1, from the values read at entry
  if (!isfinite(s1) || s1 <= tol2 * bnorm2 || iter + 1 >= maxit) {
    tl_end(4, tls);
    return;
  }
  const double beta = s2 / rho;
  if (b4) {
    for (int64_t i = i0; i < m2; i += 4 * stride) {
      double zv[4], pv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t j = i + u * stride;
        zv[u] = j < m2 ? z[j] : 0.0;
        pv[u] = j < m2 ? p[j] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t j = i + u * stride;
        if (j < m2) p[j] = zv[u] + beta * pv[u];
      }
    }
  } else {
    for (int64_t i = i0; i < m2; i += stride) p[i] = z[i] + beta * p[i];
  }
  if (next_rhs) {   // phase D: the next F-solve's right-hand side u = Cᵀp (p complete after the sync)
    grid.sync();
    const int64_t N = (next_rhs == 1 || next_rhs == 4) ? F.N : Ct.nrows, rc0 = F.fl_rc0;
    if (b4 && (next_rhs == 2 || next_rhs == 4)) {
      for (int64_t cI = i0; cI < N; cI += 4 * stride) {
        int64_t rr4[4];
        bool ok[4];
        double s4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          rr4[u] = cI + u * stride;
          ok[u] = rr4[u] < Ct.nrows;
        }
        csr_dot4(Ct, rr4, ok, p, s4);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t j = rr4[u];
          if (j < N) {
            const double v = ok[u] ? s4[u] : 0.0;
            ubuf[j] = v;
            if (next_rhs == 4) {
              F.acc[j] = 0.0;
              F.tacc[j] = 0.0;
              xout[j] = 0.0;
              if (j >= rc0) F.vbuf[j] = v;
            }
          }
        }
      }
      tl_end(4, tls);
      return;
    }
    for (int64_t cI = i0; cI < N; cI += stride) {
      const double v = cI < Ct.nrows ? csr_dot<BD>(Ct, cI, p) : 0.0;
      if (next_rhs == 4) {   // level products: what k_pi_init does, with u = Cᵀp as the right-hand side
        ubuf[cI] = v;
        F.acc[cI] = 0.0;
        F.tacc[cI] = 0.0;
        xout[cI] = 0.0;
        if (cI >= rc0) F.vbuf[cI] = v;
      } else if (next_rhs >= 2) {
        ubuf[cI] = v;
        if (next_rhs == 3) xout[cI] = 0.0;   // dense W: the GEMV accumulates into xout[0, n)
      } else {
        if (cI < rc0) {
          F.acc[cI] = v;
          F.vbuf[cI] = 0.0;
        } else {
          F.vbuf[cI] = v;
        }
        xout[cI] = 0.0;
      }
    }
  }
  tl_end(4, tls);
}

bool pcg_step(const DevCSR& Cf, const int32_t* longr, int64_t nlong, int prec, const double* D, double* p,
              const double* w, double* q, double* x, double* r, double* z, double* partial, PcgState* st, int grid,
              cudaStream_t s, int next_rhs, const DevFactor* Fp, const DevCSR* Ctp, double* xout, double* ubuf) {
  // small m2 (grid ≤ 2 CTAs per SM): wide CSR batches (one load round per row of C and of Cᵀ, 94 registers);
  // large m2: 4-entry batches at 4 CTAs per SM (more rows in flight)
  static int sms = 0, max_wide = 0, max_narrow = 0;
  if (!sms) {
    if (std::getenv("QPB_STEP_B4") && std::getenv("QPB_STEP_B4")[0] == '0') {
      const int zero = 0;
      cudaMemcpyToSymbol(g_step_b4, &zero, sizeof(int));
    }
    int dev = 0, o1 = 0, o2 = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_pcg_step<8, 16, 2>, NT, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_pcg_step<4, 4, 3>, NT, 0);
    max_wide = sms * o1;
    max_narrow = sms * o2;
  }
  const bool wide = grid <= 2 * sms;
  const int max_grid = wide ? max_wide : max_narrow;
  if (grid > max_grid) grid = max_grid;   // co-residency bound of the cooperative launch (grid-stride loops)
  DevCSR C = Cf;
  DevFactor F{};
  DevCSR Ct{};
  if (Fp) F = *Fp;
  if (Ctp) Ct = *Ctp;
  if (next_rhs && (!Ctp || ((next_rhs == 1 || next_rhs == 4) && !Fp) || (next_rhs >= 3 && !xout))) next_rhs = 0;
  void* args[] = {&C, &longr, &nlong, &prec, &D, &p, &w, &q, &x, &r, &z, &partial, &st, &next_rhs, &F, &Ct, &xout,
                  &ubuf};
  const void* fn = wide ? (const void*)k_pcg_step<8, 16, 2> : (const void*)k_pcg_step<4, 4, 3>;
  return cudaLaunchCooperativeKernel(fn, grid, NT, args, 0, s) == cudaSuccess;
}

void kf_q(const DevCSR& Cf, const int32_t* longr, int64_t nlong, const double* D, const double* p, const double* z,
          double* q, double* partial, PcgState* st, int grid, cudaStream_t s, bool pcg_mode) {
  k_kf_q<<<grid, NT, 0, s>>>(Cf, longr, nlong, D, p, z, q, partial, st, pcg_mode ? 1 : 0);
}
void pcg_init(int prec, int64_t m2, const double* b, const double* D, double* x, double* r, double* z,
              double* p, double* partial, PcgState* st, double tol, int maxit, int grid, cudaStream_t s) {
  k_pcg_init<<<grid, NT, 0, s>>>(prec, m2, b, D, x, r, z, p, partial, st, tol, maxit);
}
void pcg_init_ph(int64_t m2, const double* r, const double* z, double* p, double* partial, PcgState* st,
                 int grid, cudaStream_t s) {
  k_pcg_init_ph<<<grid, NT, 0, s>>>(m2, r, z, p, partial, st);
}
void pcg_update1(int prec, int64_t m2, const double* D, const double* p, const double* q, double* x,
                 double* r, double* z, double* partial, PcgState* st, int grid, cudaStream_t s) {
  k_pcg_update1<<<grid, NT, 0, s>>>(prec, m2, D, p, q, x, r, z, partial, st);
}
void pcg_rz_ph(int64_t m2, const double* r, const double* z, double* partial, PcgState* st, int grid,
               cudaStream_t s) {
  k_pcg_rz_ph<<<grid, NT, 0, s>>>(m2, r, z, partial, st);
}
void pcg_update2(int64_t m2, const double* z, double* p, PcgState* st, int grid, cudaStream_t s) {
  k_pcg_update2<<<grid, NT, 0, s>>>(m2, z, p, st);
}

__global__ void k_gather(double* out, const double* in, const int64_t* idx, int64_t n, const int* done) {
  if (done != nullptr && *((volatile const int*)done)) return;
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT)
    out[i] = in[idx[i]];
}
__global__ void k_scatter(double* out, const double* in, const int64_t* idx, int64_t n, const int* done) {
  if (done != nullptr && *((volatile const int*)done)) return;
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT)
    out[idx[i]] = in[i];
}
void gather(double* out, const double* in, const int64_t* idx, int64_t n, const int* done, cudaStream_t s) {
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + NT - 1) / NT, 148 * 8));
  k_gather<<<grid, NT, 0, s>>>(out, in, idx, n, done);
}
void scatter(double* out, const double* in, const int64_t* idx, int64_t n, const int* done, cudaStream_t s) {
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + NT - 1) / NT, 148 * 8));
  k_scatter<<<grid, NT, 0, s>>>(out, in, idx, n, done);
}


// ------------------------------------------------------------------------- the x-space operator alone
// G p = H p + Cᵀ(D⁻¹ ∘ (C p)) (the north_star's "H·p + Cᵀ(D·(C·p))" with D = V⁻¹S) at any
// size, without a factorization: two streaming passes — t = D⁻¹∘(C p) over the rows of C, then
// q = H p + Cᵀ t over the rows of H and Cᵀ — each a quad of lanes per row (4 consecutive entries per
// load round: full 32-byte sectors on the short rows of these matrices).  Sharded rows: every rank
// applies its rows of C (and H once, on rank 0); the caller all-reduces q.
__global__ void __launch_bounds__(NT) k_op_t(DevCSR Cf, const double* D, const double* p, double* t) {
  const int q4 = threadIdx.x & 3;
  const int64_t nq = ((int64_t)gridDim.x * NT) >> 2;
  for (int64_t k = (blockIdx.x * (int64_t)NT + threadIdx.x) >> 2; k < Cf.nrows; k += nq) {
    double s = 0.0;
    for (int64_t e = __ldg(Cf.p + k) + q4; e < __ldg(Cf.p + k + 1); e += 4) s += __ldg(Cf.v + e) * __ldg(p + __ldg(Cf.i + e));
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (q4 == 0) t[k] = s / D[k];
  }
}
__global__ void __launch_bounds__(NT) k_op_q(DevCSR Hf, DevCSR Ctf, const double* p, const double* t, double* q,
                                             int with_h) {
  const int q4 = threadIdx.x & 3;
  const int64_t nq = ((int64_t)gridDim.x * NT) >> 2;
  for (int64_t i = (blockIdx.x * (int64_t)NT + threadIdx.x) >> 2; i < Ctf.nrows; i += nq) {
    double s = 0.0;
    if (with_h)
      for (int64_t e = __ldg(Hf.p + i) + q4; e < __ldg(Hf.p + i + 1); e += 4) s += __ldg(Hf.v + e) * __ldg(p + __ldg(Hf.i + e));
    for (int64_t e = __ldg(Ctf.p + i) + q4; e < __ldg(Ctf.p + i + 1); e += 4) s += __ldg(Ctf.v + e) * __ldg(t + __ldg(Ctf.i + e));
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (q4 == 0) q[i] = s;
  }
}
__global__ void __launch_bounds__(NT) k_op_q_range(DevCSR Hf, DevCSR Ctf, const double* p, const double* t, double* q,
                                                   int64_t q_lo, int64_t q_hi, int64_t h_lo, int64_t h_hi) {
  const int q4 = threadIdx.x & 3;
  const int64_t nq = ((int64_t)gridDim.x * NT) >> 2;
  for (int64_t i = q_lo + ((blockIdx.x * (int64_t)NT + threadIdx.x) >> 2); i < q_hi; i += nq) {
    double s = 0.0;
    if (i >= h_lo && i < h_hi)
      for (int64_t e = __ldg(Hf.p + i) + q4; e < __ldg(Hf.p + i + 1); e += 4) s += __ldg(Hf.v + e) * __ldg(p + __ldg(Hf.i + e));
    for (int64_t e = __ldg(Ctf.p + i) + q4; e < __ldg(Ctf.p + i + 1); e += 4) s += __ldg(Ctf.v + e) * __ldg(t + __ldg(Ctf.i + e));
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (q4 == 0) q[i] = s;
  }
}
__global__ void __launch_bounds__(NT) k_add_range(double* dst, const double* src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) dst[i] += src[i];
}
void op_apply_range(const DevCSR& Hf, const DevCSR& Cf, const DevCSR& Ctf, const double* D, const double* p, double* t,
                    double* q, int64_t q_lo, int64_t q_hi, int64_t h_lo, int64_t h_hi, int sms, cudaStream_t s) {
  const int g = sms * 8;
  k_op_t<<<g, NT, 0, s>>>(Cf, D, p, t);
  k_op_q_range<<<g, NT, 0, s>>>(Hf, Ctf, p, t, q, q_lo, q_hi, h_lo, h_hi);
}
void add_range(double* dst, const double* src, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((n + NT - 1) / NT, 148 * 8));
  k_add_range<<<g, NT, 0, s>>>(dst, src, n);
}
void op_apply(const DevCSR& Hf, const DevCSR& Cf, const DevCSR& Ctf, const double* D, const double* p, double* t,
              double* q, bool with_h, int sms, cudaStream_t s) {
  const int g = sms * 8;
  k_op_t<<<g, NT, 0, s>>>(Cf, D, p, t);
  k_op_q<<<g, NT, 0, s>>>(Hf, Ctf, p, t, q, with_h ? 1 : 0);
}

// ------------------------------------------------------------------------- x-space twin (K_C, PPCG)
// q = G p = H p + Cᵀ(W∘(C p)) in ONE kernel (the north_star's fused SpMV chain): warp per x-row i,
// lanes over H's row, then over Cᵀ's row where each lane forms its (C p)_k on the fly (C rows are
// short; the redundancy is nnz(C)·(column count of C) FMAs, all from L2).  Fused pᵀq reduction;
// pcg_mode: the last block sets α = ρ / pᵀq (fin_pcg_pq).
__global__ void __launch_bounds__(NT) k_g_apply(DevCSR Hf, DevCSR Cf, DevCSR Ctf, const double* W, const double* p,
                                                double* q, double* partial, PcgState* st, int pcg_mode) {
  __shared__ double sh[32];
  if (pcg_mode && *((volatile int*)&st->done)) return;
  const int lane = threadIdx.x & 31;
  double loc = 0.0;
  const int64_t nw = ((int64_t)gridDim.x * NT) >> 5;
  for (int64_t i = (blockIdx.x * (int64_t)NT + threadIdx.x) >> 5; i < Hf.nrows; i += nw) {
    double s = 0.0;
    for (int64_t e = Hf.p[i] + lane; e < Hf.p[i + 1]; e += 32) s += Hf.v[e] * __ldg(p + Hf.i[e]);
    for (int64_t e = Ctf.p[i] + lane; e < Ctf.p[i + 1]; e += 32) {
      const int32_t k = Ctf.i[e];
      s += Ctf.v[e] * W[k] * csr_dot(Cf, k, p);
    }
    s = warp_sum(s);
    if (lane == 0) {
      q[i] = s;
      loc += p[i] * s;
    }
  }
  if (!pcg_mode) return;
  const double v = block_reduce<0>(loc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
  if (is_last_block(&st->arrive)) {
    const double pq = reduce_partials<0>(partial, gridDim.x, sh);
    if (threadIdx.x == 0) {
      fin_pcg_pq(st, pq);
      st->arrive = 0;
    }
  }
}

// x += αp; r += αq; rhs[0, n) = −r (the projection's right-hand side; rhs[n, N) stays 0)
__global__ void k_xp_update1(int64_t n, const double* p, const double* q, double* x, double* r, double* rhs,
                             const PcgState* st) {
  if (*((volatile const int*)&st->done)) return;
  const double a = st->alpha;
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
    x[i] += a * p[i];
    const double ri = r[i] + a * q[i];
    r[i] = ri;
    rhs[i] = -ri;
  }
}

// After the projection F [g; v] = [−r; 0] (so H g + Aᵀw = r with w = −v): r −= Aᵀw, λ += w, ρ' = rᵀg;
// the last block applies the PCG decision of fin_pcg_upd1 with ‖·‖ = √(rᵀg) (stop: √(ρ'/ρ₀) ≤ ε).
// init = 1: the first projection — ρ₀ = rᵀg, p = −g, iteration counter reset (fin_pcg_init).
__global__ void __launch_bounds__(NT) k_xp_update2(DevCSR Atf, int64_t m1, const double* sol, double* r, double* lam,
                                                   double* p, double* partial, PcgState* st, int init) {
  __shared__ double sh[32];
  if (!init && *((volatile int*)&st->done)) return;
  const int64_t n = Atf.nrows;
  const double* g = sol;
  const double* v = sol + n;
  double rg = 0.0;
  for (int64_t t = blockIdx.x * (int64_t)NT + threadIdx.x; t < n + m1; t += (int64_t)gridDim.x * NT) {
    if (t < n) {
      const double ri = r[t] + csr_dot(Atf, t, v);   // r − Aᵀw, w = −v
      r[t] = ri;
      rg += ri * g[t];
      if (init) p[t] = -g[t];
    } else {
      lam[t - n] -= v[t - n];                        // λ += w
    }
  }
  const double s = block_reduce<0>(rg, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
  if (is_last_block(&st->arrive)) {
    const double t = reduce_partials<0>(partial, gridDim.x, sh);
    if (threadIdx.x == 0) {
      if (init) {
        st->iter = 0;
        st->status = 0;
        fin_pcg_init(st, fabs(t), t);
        if (!(t > 0.0)) st->done = 1;
      } else {
        fin_pcg_upd1(st, fabs(t), t, 0);
      }
      st->arrive = 0;
    }
  }
}

// p = −g + βp
__global__ void k_xp_update3(int64_t n, const double* g, double* p, const PcgState* st) {
  if (*((volatile const int*)&st->done)) return;
  const double b = st->beta;
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) p[i] = -g[i] + b * p[i];
}

// r = q − f;  rhs[0, n) = −r
__global__ void k_xp_init_r(int64_t n, const double* q, const double* f, double* r, double* rhs) {
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
    const double ri = q[i] - f[i];
    r[i] = ri;
    rhs[i] = -ri;
  }
}

// IPM x-space right-hand side: f = r_g − CᵀW r_a (factor order, n), e = −r_e (m1) → rhs_f = [f; e]
__global__ void k_x_rhs(DevCSR Ctf, int64_t m1, const double* rg_re, const double* ra, const double* D, double* fe) {
  const int64_t n = Ctf.nrows;
  for (int64_t t = blockIdx.x * (int64_t)NT + threadIdx.x; t < n + m1; t += (int64_t)gridDim.x * NT) {
    if (t < n) {
      double s = 0.0;
      for (int64_t e = Ctf.p[t]; e < Ctf.p[t + 1]; ++e) s += Ctf.v[e] * ra[Ctf.i[e]] / D[Ctf.i[e]];
      fe[t] = rg_re[t] - s;
    } else {
      fe[t] = -rg_re[t];
    }
  }
}

// Δν = −D⁻¹(r_a + CΔx)
__global__ void k_x_dnu(DevCSR Cf, const double* ra, const double* D, const double* dx, double* dnu) {
  for (int64_t k = blockIdx.x * (int64_t)NT + threadIdx.x; k < Cf.nrows; k += (int64_t)gridDim.x * NT)
    dnu[k] = -(ra[k] + csr_dot(Cf, k, dx)) / D[k];
}
__global__ void k_recip(int64_t m, const double* D, double* W) {
  for (int64_t k = blockIdx.x * (int64_t)NT + threadIdx.x; k < m; k += (int64_t)gridDim.x * NT) W[k] = 1.0 / D[k];
}

void g_apply(const DevCSR& Hf, const DevCSR& Cf, const DevCSR& Ctf, const double* W, const double* p, double* q,
             double* partial, PcgState* st, bool pcg_mode, int grid, cudaStream_t s) {
  k_g_apply<<<grid, NT, 0, s>>>(Hf, Cf, Ctf, W, p, q, partial, st, pcg_mode ? 1 : 0);
}
void xp_update1(int64_t n, const double* p, const double* q, double* x, double* r, double* rhs, const PcgState* st,
                int grid, cudaStream_t s) {
  k_xp_update1<<<grid, NT, 0, s>>>(n, p, q, x, r, rhs, st);
}
void xp_update2(const DevCSR& Atf, int64_t m1, const double* sol, double* r, double* lam, double* p, double* partial,
                PcgState* st, bool init, int grid, cudaStream_t s) {
  k_xp_update2<<<grid, NT, 0, s>>>(Atf, m1, sol, r, lam, p, partial, st, init ? 1 : 0);
}
void xp_update3(int64_t n, const double* g, double* p, const PcgState* st, int grid, cudaStream_t s) {
  k_xp_update3<<<grid, NT, 0, s>>>(n, g, p, st);
}
void xp_init_r(int64_t n, const double* q, const double* f, double* r, double* rhs, int grid, cudaStream_t s) {
  k_xp_init_r<<<grid, NT, 0, s>>>(n, q, f, r, rhs);
}
void x_rhs(const DevCSR& Ctf, int64_t m1, const double* rg_re, const double* ra, const double* D, double* fe,
           int grid, cudaStream_t s) {
  k_x_rhs<<<grid, NT, 0, s>>>(Ctf, m1, rg_re, ra, D, fe);
}
void x_dnu(const DevCSR& Cf, const double* ra, const double* D, const double* dx, double* dnu, int grid,
           cudaStream_t s) {
  k_x_dnu<<<grid, NT, 0, s>>>(Cf, ra, D, dx, dnu);
}
void recip(int64_t m, const double* D, double* W, int grid, cudaStream_t s) { k_recip<<<grid, NT, 0, s>>>(m, D, W); }

// ------------------------------------------------------------------------- IPM kernels
__global__ void __launch_bounds__(NT) k_ipm_mu(int64_t m2, const double* s_, const double* nu, double* partial,
                                               IpmState* st) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < m2; i += (int64_t)gridDim.x * NT)
    v += s_[i] * nu[i];
  v = block_reduce<0>(v, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
  if (is_last_block(&st->arrive)) {
    double s = reduce_partials<0>(partial, gridDim.x, sh);
    if (threadIdx.x == 0) {
      if (st->defer) st->red[0] = s;
      else fin_ipm_mu(st, s);
      st->arrive = 0;
    }
  }
}

// Rows [0,n): r_g = −(Hx + g − Aᵀλ − Cᵀν) (reading R1) → rhs_f[i];
// rows [n,n+m1): r_e = Ax − b → rhs_f[i];
// rows [n+m1, n+m1+m2): r_i = Cx − s − d, r_c = s∘ν − σμ, r_a = r_i + r_c/ν, D = s/ν.
__global__ void __launch_bounds__(NT) k_ipm_resid(DevCSR Hf, DevCSR Atf, DevCSR Ctf, DevCSR Af, DevCSR Cf,
                                                  const double* gf, const double* b, const double* d,
                                                  const double* x, const double* lam, const double* nu,
                                                  const double* s_, double* rhs_f, double* rc, double* ra,
                                                  double* D, double* partial, IpmState* st, const double* ctnu) {
  __shared__ double sh[32];
  const int64_t n = Hf.nrows, m1 = Af.nrows, m2 = Cf.nrows;
  const double smu = st->sigma_mu;
  double mg = 0.0, me = 0.0, mi = 0.0;
  for (int64_t t = blockIdx.x * (int64_t)NT + threadIdx.x; t < n + m1 + m2; t += (int64_t)gridDim.x * NT) {
    if (t < n) {
      const double grad = csr_dot(Hf, t, x) + gf[t] - csr_dot(Atf, t, lam) -
                          (ctnu != nullptr ? ctnu[t] : csr_dot(Ctf, t, nu));
      rhs_f[t] = -grad;
      mg = fmax(mg, fabs(grad));
    } else if (t < n + m1) {
      const int64_t i = t - n;
      const double re = csr_dot(Af, i, x) - b[i];
      rhs_f[t] = re;
      me = fmax(me, fabs(re));
    } else {
      const int64_t i = t - n - m1;
      const double si = s_[i], ni = nu[i];
      const double ri = csr_dot(Cf, i, x) - si - d[i];
      const double rci = si * ni - smu;
      rc[i] = rci;
      ra[i] = ri + rci / ni;
      D[i] = si / ni;
      mi = fmax(mi, fabs(ri));
    }
  }
  double v1 = block_reduce<1>(mg, sh);
  double v2 = block_reduce<1>(me, sh);
  double v3 = block_reduce<1>(mi, sh);
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = v1;
    partial[gridDim.x + blockIdx.x] = v2;
    partial[2 * gridDim.x + blockIdx.x] = v3;
  }
  if (is_last_block(&st->arrive)) {
    double a1 = reduce_partials<1>(partial, gridDim.x, sh);
    double a2 = reduce_partials<1>(partial + gridDim.x, gridDim.x, sh);
    double a3 = reduce_partials<1>(partial + 2 * gridDim.x, gridDim.x, sh);
    if (threadIdx.x == 0) {
      if (st->defer) {
        st->red[0] = a1;
        st->red[1] = a2;
        st->red[2] = a3;
      } else {
        fin_ipm_resid(st, a1, a2, a3);
      }
      st->arrive = 0;
    }
  }
}

// r_ν = −r_a + C·y_x
__global__ void k_ipm_rnu(DevCSR Cf, const double* ra, const double* y, double* rnu) {
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < Cf.nrows; i += (int64_t)gridDim.x * NT)
    rnu[i] = -ra[i] + csr_dot(Cf, i, y);
}

// rhs of F(Δx;Δλ) = −(r_g + CᵀΔν; r_e); rg_re holds (r_g; r_e) in factor order.
__global__ void k_ipm_recrhs(DevCSR Ctf, int64_t n, int64_t m1, const double* rg_re, const double* dnu,
                             double* rhs_f, const double* ctdnu) {
  for (int64_t t = blockIdx.x * (int64_t)NT + threadIdx.x; t < n + m1; t += (int64_t)gridDim.x * NT)
    rhs_f[t] = t < n ? -(rg_re[t] + (ctdnu != nullptr ? ctdnu[t] : csr_dot(Ctf, t, dnu))) : -rg_re[t];
}

// Δs = −V⁻¹r_c − DΔν; α_max over s, ν; α = min(1, τ α_max) (reading R3).
__global__ void __launch_bounds__(NT) k_ipm_ds_alpha(int64_t m2, const double* rc, const double* nu,
                                                     const double* D, const double* dnu, const double* s_,
                                                     double* ds, double* partial, IpmState* st) {
  __shared__ double sh[32];
  double amin = DBL_MAX;
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < m2; i += (int64_t)gridDim.x * NT) {
    const double dsi = -rc[i] / nu[i] - D[i] * dnu[i];
    ds[i] = dsi;
    if (dsi < 0.0) amin = fmin(amin, -s_[i] / dsi);
    const double dn = dnu[i];
    if (dn < 0.0) amin = fmin(amin, -nu[i] / dn);
  }
  double v = block_reduce<2>(amin, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
  if (is_last_block(&st->arrive)) {
    double a = reduce_partials<2>(partial, gridDim.x, sh);
    if (threadIdx.x == 0) {
      if (st->defer) st->red[0] = a;
      else fin_ipm_alpha(st, a);
      st->arrive = 0;
    }
  }
}

__global__ void k_ipm_update(int64_t N, int64_t m2, const double* dxl, const double* dnu, const double* ds,
                             double* xl, double* nu, double* s_, const IpmState* st) {
  const double a = st->alpha;
  for (int64_t t = blockIdx.x * (int64_t)NT + threadIdx.x; t < N + m2; t += (int64_t)gridDim.x * NT) {
    if (t < N) {
      xl[t] += a * dxl[t];
    } else {
      const int64_t i = t - N;
      nu[i] += a * dnu[i];
      s_[i] += a * ds[i];
    }
  }
}

__global__ void __launch_bounds__(NT) k_ipm_objective(DevCSR Hf, const double* gf, const double* x,
                                                      double* partial, IpmState* st) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < Hf.nrows; i += (int64_t)gridDim.x * NT)
    v += x[i] * (0.5 * csr_dot(Hf, i, x) + gf[i]);
  v = block_reduce<0>(v, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
  if (is_last_block(&st->arrive)) {
    double s = reduce_partials<0>(partial, gridDim.x, sh);
    if (threadIdx.x == 0) {
      st->objective = s;
      st->arrive = 0;
    }
  }
}

void ipm_mu(int64_t m2, const double* s_, const double* nu, double* partial, IpmState* st, int grid,
            cudaStream_t s) {
  k_ipm_mu<<<grid, NT, 0, s>>>(m2, s_, nu, partial, st);
}
void ipm_residuals(const DevCSR& Hf, const DevCSR& Atf, const DevCSR& Ctf, const DevCSR& Af, const DevCSR& Cf,
                   const double* gf, const double* b, const double* d, const double* x, const double* lam,
                   const double* nu, const double* s_, double* rhs_f, double* rc, double* ra, double* D,
                   double* partial, IpmState* st, int grid, cudaStream_t s, const double* ctnu) {
  k_ipm_resid<<<grid, NT, 0, s>>>(Hf, Atf, Ctf, Af, Cf, gf, b, d, x, lam, nu, s_, rhs_f, rc, ra, D, partial, st,
                                  ctnu);
}
void ipm_rnu(const DevCSR& Cf, const double* ra, const double* y, double* rnu, int grid, cudaStream_t s) {
  k_ipm_rnu<<<grid, NT, 0, s>>>(Cf, ra, y, rnu);
}
void ipm_recovery_rhs(const DevCSR& Ctf, int64_t n, int64_t m1, const double* rg_re, const double* dnu,
                      double* rhs_f, int grid, cudaStream_t s, const double* ctdnu) {
  k_ipm_recrhs<<<grid, NT, 0, s>>>(Ctf, n, m1, rg_re, dnu, rhs_f, ctdnu);
}
void ipm_ds_alpha(int64_t m2, const double* rc, const double* nu, const double* D, const double* dnu,
                  const double* s_, double* ds, double* partial, IpmState* st, int grid, cudaStream_t s) {
  k_ipm_ds_alpha<<<grid, NT, 0, s>>>(m2, rc, nu, D, dnu, s_, ds, partial, st);
}
void ipm_update(int64_t N, int64_t m2, const double* dxl, const double* dnu, const double* ds, double* xl,
                double* nu, double* s_, const IpmState* st, int grid, cudaStream_t s) {
  k_ipm_update<<<grid, NT, 0, s>>>(N, m2, dxl, dnu, ds, xl, nu, s_, st);
}
void ipm_objective(const DevCSR& Hf, const double* gf, const double* x, double* partial, IpmState* st, int grid,
                   cudaStream_t s) {
  k_ipm_objective<<<grid, NT, 0, s>>>(Hf, gf, x, partial, st);
}

// ------------------------------------------------------------------------- T = C diag(H)⁻¹ Cᵀ values
// One thread per stored entry (i, j): sparse dot of C rows i and j weighted by 1/H_kk.
__global__ void k_t_values(DevCSR C, const double* hdiag, const int64_t* t_row, const int32_t* t_col,
                           int64_t nnz, double* t_val) {
  for (int64_t e = blockIdx.x * (int64_t)NT + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * NT) {
    const int64_t i = t_row[e], j = t_col[e];
    int64_t a = C.p[i], ae = C.p[i + 1], b = C.p[j], be = C.p[j + 1];
    double s = 0.0;
    while (a < ae && b < be) {
      const int32_t ca = C.i[a], cb = C.i[b];
      if (ca == cb) {
        s += C.v[a] * C.v[b] / hdiag[ca];
        ++a;
        ++b;
      } else if (ca < cb) {
        ++a;
      } else {
        ++b;
      }
    }
    t_val[e] = s;
  }
}
void t_values(const DevCSR& Cnu, const double* hdiag, const int64_t* t_row, const int32_t* t_col, int64_t nnz_t,
              double* t_val, cudaStream_t s) {
  if (nnz_t == 0) return;
  int grid = (int)std::min<int64_t>((nnz_t + NT - 1) / NT, 148 * 16);
  k_t_values<<<grid, NT, 0, s>>>(Cnu, hdiag, t_row, t_col, nnz_t, t_val);
}

}  // namespace qpb
