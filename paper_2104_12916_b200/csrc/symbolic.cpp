// Host symbolic analysis (see symbolic.h).  Plain C++; runs once per factor.
//
// Definitions follow SURVEY.md §8(c) c4 / DESIGN.md §Structures:
//   etree      Liu's algorithm on the lower pattern (parent(j) = min{i>j: L_ij≠0})
//   colcounts  row-subtree traversal: row i of L = ∪ paths k→i in the etree
//              over F_ik ≠ 0, k < i (O(nnz(L)))
//   rowlev     lev(i) = 1 + max{lev(j): L_ij ≠ 0, j<i}, 0 without off-diagonals
//   supernodes j joins j−1 iff parent(j−1)=j and cc(j−1)=cc(j)+1
//   sn levels  0 for leaves, 1 + max over children
#include "symbolic.h"

#include <algorithm>
#include <cstdio>
#include <iterator>
#include <cmath>
#include <numeric>
#include <stdexcept>
#include <cstdlib>

namespace qpb {

LowerMatrix build_F_lower(int64_t n, int64_t m1, const int64_t* Hp, const int32_t* Hi, const double* Hx,
                          const int64_t* Ap, const int32_t* Ai, const double* Ax,
                          const std::vector<int64_t>& xperm) {
  LowerMatrix M;
  const int64_t N = n + m1;
  M.N = N;
  std::vector<int64_t> pinv(n);
  for (int64_t i = 0; i < n; ++i) pinv[xperm[i]] = i;
  M.diag.assign(N, 0.0);
  std::vector<int64_t> cnt(N + 1, 0);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = Hp[i]; p < Hp[i + 1]; ++p) {
      int64_t j = Hi[p];
      if (pinv[i] > pinv[j]) cnt[pinv[j] + 1]++;
      else if (i == j) M.diag[pinv[i]] = -Hx[p];  // (1,1) block of F is −H
    }
  for (int64_t i = 0; i < m1; ++i)
    for (int64_t p = Ap[i]; p < Ap[i + 1]; ++p) cnt[pinv[Ai[p]] + 1]++;  // A in rows n+i
  for (int64_t j = 0; j < N; ++j) cnt[j + 1] += cnt[j];
  M.colptr = cnt;
  M.rowind.resize(cnt[N]);
  M.val.resize(cnt[N]);
  std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = Hp[i]; p < Hp[i + 1]; ++p) {
      int64_t j = Hi[p];
      if (pinv[i] > pinv[j]) {
        int64_t q = pos[pinv[j]]++;
        M.rowind[q] = (int32_t)pinv[i];
        M.val[q] = -Hx[p];
      }
    }
  for (int64_t i = 0; i < m1; ++i)
    for (int64_t p = Ap[i]; p < Ap[i + 1]; ++p) {
      int64_t q = pos[pinv[Ai[p]]]++;
      M.rowind[q] = (int32_t)(n + i);
      M.val[q] = Ax[p];
    }
  // sort rows inside each column
  std::vector<std::pair<int32_t, double>> tmp;
  for (int64_t j = 0; j < N; ++j) {
    int64_t a = M.colptr[j], b = M.colptr[j + 1];
    tmp.clear();
    for (int64_t q = a; q < b; ++q) tmp.emplace_back(M.rowind[q], M.val[q]);
    std::sort(tmp.begin(), tmp.end(), [](auto& x, auto& y) { return x.first < y.first; });
    for (int64_t q = a; q < b; ++q) { M.rowind[q] = tmp[q - a].first; M.val[q] = tmp[q - a].second; }
  }
  return M;
}

static inline int64_t tile_begin(int64_t t, int64_t nk, int64_t w, int64_t m) {
  int64_t v = t < nk ? (int64_t)BW * t : w + (int64_t)BW * (t - nk);
  return v < m ? v : m;
}

std::string analyse(const LowerMatrix& M, Symbolic& S, int64_t n_negative, bool allow_symroot, int64_t trailing_from,
                    int64_t max_sn_width) {
  const int64_t N = M.N;
  S.N = N;
  // ---------------------------------------------------------------- row form of the strict lower part
  std::vector<int64_t> rp(N + 1, 0);
  for (int64_t q = 0; q < (int64_t)M.rowind.size(); ++q) rp[M.rowind[q] + 1]++;
  for (int64_t i = 0; i < N; ++i) rp[i + 1] += rp[i];
  std::vector<int32_t> rc(rp[N]);
  {
    std::vector<int64_t> pos(rp.begin(), rp.end() - 1);
    for (int64_t j = 0; j < N; ++j)
      for (int64_t q = M.colptr[j]; q < M.colptr[j + 1]; ++q) rc[pos[M.rowind[q]]++] = (int32_t)j;
  }
  // ---------------------------------------------------------------- elimination tree (Liu)
  S.parent.assign(N, -1);
  {
    std::vector<int64_t> anc(N, -1);
    for (int64_t i = 0; i < N; ++i) {
      for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
        int64_t r = rc[q];
        while (anc[r] != -1 && anc[r] != i) {
          int64_t t = anc[r];
          anc[r] = i;
          r = t;
        }
        if (anc[r] == -1) {
          anc[r] = i;
          S.parent[r] = i;
        }
      }
    }
  }
  // ---------------------------------------------------------------- column counts + row levels
  S.colcount.assign(N, 0);
  S.rowlev.assign(N, 0);
  {
    std::vector<int64_t> mark(N, -1);
    for (int64_t i = 0; i < N; ++i) {
      mark[i] = i;
      S.colcount[i] += 1;
      int64_t lev = 0;
      for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
        int64_t j = rc[q];
        while (mark[j] != i) {
          mark[j] = i;
          S.colcount[j] += 1;
          lev = std::max(lev, S.rowlev[j] + 1);
          j = S.parent[j];
          if (j < 0) return "etree walk escaped the tree (internal error)";
        }
      }
      S.rowlev[i] = lev;
    }
  }
  S.nnz_L = 0;
  S.c_fact = 0;
  S.n_rowlev = 0;
  for (int64_t j = 0; j < N; ++j) {
    S.nnz_L += S.colcount[j];
    S.c_fact += (double)S.colcount[j] * (double)S.colcount[j];
    S.n_rowlev = std::max(S.n_rowlev, S.rowlev[j] + 1);
  }
  // ---------------------------------------------------------------- fundamental supernodes
  std::vector<int64_t> fs_start;
  fs_start.push_back(0);
  for (int64_t j = 1; j < N; ++j)
    if (!(S.parent[j - 1] == j && S.colcount[j - 1] == S.colcount[j] + 1)) fs_start.push_back(j);
  fs_start.push_back(N);
  const int64_t nf = (int64_t)fs_start.size() - 1;
  std::vector<int64_t> col2sn(N);
  for (int64_t J = 0; J < nf; ++J)
    for (int64_t c = fs_start[J]; c < fs_start[J + 1]; ++c) col2sn[c] = J;
  std::vector<int64_t> fparent(nf, -1);
  for (int64_t J = 0; J < nf; ++J) {
    int64_t p = S.parent[fs_start[J + 1] - 1];
    if (p >= 0) fparent[J] = col2sn[p];
  }
  std::vector<std::vector<int32_t>> fchildren(nf);
  for (int64_t J = 0; J < nf; ++J)
    if (fparent[J] >= 0) fchildren[fparent[J]].push_back((int32_t)J);
  // rows strictly below each fundamental supernode's columns
  std::vector<int64_t> fb_ptr(nf + 1, 0);
  std::vector<int32_t> fb_rows;
  {
    std::vector<int64_t> mark(N, -1);
    std::vector<int32_t> buf;
    for (int64_t J = 0; J < nf; ++J) {
      const int64_t c0 = fs_start[J], c1 = fs_start[J + 1];
      buf.clear();
      for (int64_t c = c0; c < c1; ++c)
        for (int64_t q = M.colptr[c]; q < M.colptr[c + 1]; ++q) {
          int64_t r = M.rowind[q];
          if (r >= c1 && mark[r] != J) { mark[r] = J; buf.push_back((int32_t)r); }
        }
      for (int32_t K : fchildren[J])
        for (int64_t q = fb_ptr[K]; q < fb_ptr[K + 1]; ++q) {
          int64_t r = fb_rows[q];
          if (r >= c1 && mark[r] != J) { mark[r] = J; buf.push_back((int32_t)r); }
        }
      std::sort(buf.begin(), buf.end());
      fb_rows.insert(fb_rows.end(), buf.begin(), buf.end());
      fb_ptr[J + 1] = (int64_t)fb_rows.size();
      if ((c1 - c0) + (int64_t)buf.size() != S.colcount[c0])
        return "supernode structure does not match column count (internal error)";
    }
  }
  // ---------------------------------------------------------------- relaxed amalgamation
  // Merge supernode J into its parent P when J's columns immediately precede
  // P's and the explicit zeros stay small (thresholds of DESIGN.md §Structures:
  // width ≤ 4 always; ≤ 16 if zeros ≤ 80%; ≤ 48 if ≤ 10%; else ≤ 5%).
  std::vector<int64_t> rc0(nf), rw(nf), rm(nf), rtrue(nf);
  std::vector<char> alive(nf, 1);
  for (int64_t J = 0; J < nf; ++J) {
    rc0[J] = fs_start[J];
    rw[J] = fs_start[J + 1] - fs_start[J];
    rm[J] = rw[J] + (fb_ptr[J + 1] - fb_ptr[J]);
    int64_t t = 0;
    for (int64_t c = fs_start[J]; c < fs_start[J + 1]; ++c) t += S.colcount[c];
    rtrue[J] = t;
  }
  // passes over the current partition until no merge happens (a merged parent may now be
  // contiguous with, and cheap enough for, its own parent)
  {
    std::vector<int64_t> colown(N);
    while (true) {
      for (int64_t J = 0; J < nf; ++J)
        if (alive[J])
          for (int64_t c = rc0[J]; c < rc0[J] + rw[J]; ++c) colown[c] = J;
      int64_t merged = 0;
      for (int64_t J = 0; J < nf; ++J) {
        if (!alive[J]) continue;
        const int64_t pc = S.parent[rc0[J] + rw[J] - 1];
        if (pc < 0) continue;
        const int64_t P = colown[pc];
        if (!alive[P] || rc0[J] + rw[J] != rc0[P]) continue;
        const int64_t w = rw[J] + rw[P];
        const int64_t m = rw[J] + rm[P];
        const int64_t stored = w * m - w * (w - 1) / 2;
        const int64_t zeros = stored - (rtrue[J] + rtrue[P]);
        bool merge = w <= 4 || (w <= 16 && 100 * zeros <= 80 * stored) || (w <= 48 && 100 * zeros <= 10 * stored) ||
                     (100 * zeros <= 5 * stored);
        if (!merge) continue;
        rc0[P] = rc0[J];
        rw[P] = w;
        rm[P] = m;
        rtrue[P] += rtrue[J];
        alive[J] = 0;
        for (int64_t c = rc0[J]; c < rc0[J] + rw[J]; ++c) colown[c] = P;
        ++merged;
      }
      if (merged == 0) break;
    }
  }
  // forced dense trailing supernode (absorbed top of the tree, see api.cu analyse_F)
  S.trailing_from = trailing_from;
  if (trailing_from >= 0 && trailing_from < N) {
    int64_t last = -1, first = -1;
    for (int64_t J = 0; J < nf; ++J)
      if (alive[J]) {
        if (rc0[J] + rw[J] > trailing_from && first < 0) first = J;
        last = J;
      }
    if (first >= 0 && last >= 0 && first != last) {
      int64_t t = 0, wsum = 0;
      for (int64_t J = first; J <= last; ++J)
        if (alive[J]) {
          t += rtrue[J];
          wsum += rw[J];
          if (J != last) alive[J] = 0;
        }
      rc0[last] = N - wsum;
      rw[last] = wsum;
      rm[last] = wsum;
      rtrue[last] = t;
      if (fb_ptr[last + 1] != fb_ptr[last]) return "trailing merge: last supernode has rows below (internal error)";
    }
  }
  // relaxed partition (alive supernodes, in column order).  max_sn_width > 0 splits wider supernodes
  // into a chain of pieces (multiples of BW columns): piece i keeps every later column of the original
  // supernode as dense rows, so its parent is piece i+1 and the partitioned inverses of the sweeps
  // are formed per piece (Σ B³/6 instead of w³/6 flops; used for P_H, refactored every IPM iteration).
  S.sn_start.clear();
  std::vector<int64_t> rep;       // fundamental id that carries each relaxed supernode's below-rows
  std::vector<int64_t> sn_end;    // end column of the original relaxed supernode of each piece
  const int64_t cap = max_sn_width > 0 ? std::max<int64_t>(BW, max_sn_width / BW * BW) : 0;
  for (int64_t J = 0; J < nf; ++J)
    if (alive[J]) {
      const int64_t a = rc0[J], e = rc0[J] + rw[J];
      for (int64_t c = a; c < e; c += (cap > 0 ? cap : e - a)) {
        S.sn_start.push_back(c);
        rep.push_back(J);
        sn_end.push_back(e);
      }
    }
  S.sn_start.push_back(N);
  const int64_t ns = (int64_t)S.sn_start.size() - 1;
  S.ns = ns;
  for (int64_t J = 0; J < ns; ++J)
    for (int64_t c = S.sn_start[J]; c < S.sn_start[J + 1]; ++c) col2sn[c] = J;
  S.sn_parent.assign(ns, -1);
  for (int64_t J = 0; J < ns; ++J) {
    if (S.sn_start[J + 1] < sn_end[J]) {   // a piece: the next piece holds its first below-rows
      S.sn_parent[J] = J + 1;
      continue;
    }
    int64_t p = S.parent[S.sn_start[J + 1] - 1];
    if (p >= 0) S.sn_parent[J] = col2sn[p];
  }
  S.sn_level.assign(ns, 0);
  for (int64_t J = 0; J < ns; ++J)
    if (S.sn_parent[J] >= 0)
      S.sn_level[S.sn_parent[J]] = std::max(S.sn_level[S.sn_parent[J]], S.sn_level[J] + 1);
  S.n_levels = 0;
  for (int64_t J = 0; J < ns; ++J) S.n_levels = std::max(S.n_levels, S.sn_level[J] + 1);
  std::vector<std::vector<int32_t>> children(ns);
  for (int64_t J = 0; J < ns; ++J)
    if (S.sn_parent[J] >= 0) children[S.sn_parent[J]].push_back((int32_t)J);
  // ---------------------------------------------------------------- relaxed supernode row structures
  S.sn_rowptr.assign(ns + 1, 0);
  S.sn_rows.clear();
  for (int64_t J = 0; J < ns; ++J) {
    for (int64_t c = S.sn_start[J]; c < sn_end[J]; ++c) S.sn_rows.push_back((int32_t)c);
    const int64_t F0 = rep[J];
    S.sn_rows.insert(S.sn_rows.end(), fb_rows.begin() + fb_ptr[F0], fb_rows.begin() + fb_ptr[F0 + 1]);
    S.sn_rowptr[J + 1] = (int64_t)S.sn_rows.size();
  }
  S.nnz_stored = 0;
  for (int64_t J = 0; J < ns; ++J) {
    const int64_t w = S.sn_start[J + 1] - S.sn_start[J], m = S.sn_rowptr[J + 1] - S.sn_rowptr[J];
    S.nnz_stored += w * m - w * (w - 1) / 2;
  }
  // ---------------------------------------------------------------- fronts: liveness-based memory plan
  // Levels are factored bottom-up; the fronts of level L are allocated before level L
  // (first fit), and a front is released once its parent's level has extend-added it.
  std::vector<std::vector<int32_t>> by_level(S.n_levels);
  for (int64_t J = 0; J < ns; ++J) by_level[S.sn_level[J]].push_back((int32_t)J);
  S.front_off.assign(ns, 0);
  S.ws_size = 0;
  S.ws_naive = 0;
  {
    std::vector<std::pair<int64_t, int64_t>> freel;  // (offset, size), sorted by offset
    int64_t top = 0;
    auto alloc = [&](int64_t sz) -> int64_t {
      for (size_t i = 0; i < freel.size(); ++i)
        if (freel[i].second >= sz) {
          int64_t off = freel[i].first;
          freel[i].first += sz;
          freel[i].second -= sz;
          if (freel[i].second == 0) freel.erase(freel.begin() + i);
          return off;
        }
      int64_t off = top;
      top += sz;
      return off;
    };
    auto release = [&](int64_t off, int64_t sz) {
      auto it = std::lower_bound(freel.begin(), freel.end(), std::make_pair(off, (int64_t)0));
      it = freel.insert(it, {off, sz});
      size_t i = it - freel.begin();
      if (i + 1 < freel.size() && freel[i].first + freel[i].second == freel[i + 1].first) {
        freel[i].second += freel[i + 1].second;
        freel.erase(freel.begin() + i + 1);
      }
      if (i > 0 && freel[i - 1].first + freel[i - 1].second == freel[i].first) {
        freel[i - 1].second += freel[i].second;
        freel.erase(freel.begin() + i);
      }
      if (!freel.empty() && freel.back().first + freel.back().second == top) {
        top = freel.back().first;
        freel.pop_back();
      }
    };
    auto fsize = [&](int64_t J) {
      const int64_t m = S.sn_rowptr[J + 1] - S.sn_rowptr[J];
      return (m * m + 1) & ~int64_t(1);
    };
    for (int64_t L = 0; L < S.n_levels; ++L) {
      for (int32_t J : by_level[L]) {
        S.front_off[J] = alloc(fsize(J));
        S.ws_size = std::max(S.ws_size, top);
        S.ws_naive += fsize(J);
      }
      for (int32_t J : by_level[L])
        for (int32_t K : children[J]) release(S.front_off[K], fsize(K));
    }
  }
  // ---------------------------------------------------------------- blocks + factor storage
  S.sn_blk0.assign(ns + 1, 0);
  S.blk_col0.clear(); S.blk_w.clear(); S.blk_sn.clear(); S.blk_noff.clear();
  S.blk_rows.clear(); S.blk_inv.clear(); S.blk_off.clear();
  S.fs_size = 0;
  for (int64_t J = 0; J < ns; ++J) {
    const int64_t c0 = S.sn_start[J], w = S.sn_start[J + 1] - c0;
    const int64_t m = S.sn_rowptr[J + 1] - S.sn_rowptr[J];
    S.sn_blk0[J] = (int32_t)S.blk_col0.size();
    for (int64_t k = 0; k * BW < w; ++k) {
      int64_t wk = std::min<int64_t>(BW, w - k * BW);
      int64_t noff = m - k * BW - wk;
      S.blk_col0.push_back((int32_t)(c0 + k * BW));
      S.blk_w.push_back((int32_t)wk);
      S.blk_sn.push_back((int32_t)J);
      S.blk_noff.push_back((int32_t)noff);
      S.blk_rows.push_back(S.sn_rowptr[J] + k * BW + wk);
      S.blk_inv.push_back(S.fs_size);
      S.fs_size += wk * wk;
      S.fs_size = (S.fs_size + 1) & ~int64_t(1);
      S.blk_off.push_back(S.fs_size);
      S.fs_size += noff * wk;
      S.fs_size = (S.fs_size + 1) & ~int64_t(1);
    }
  }
  S.sn_blk0[ns] = (int32_t)S.blk_col0.size();
  S.nb = (int64_t)S.blk_col0.size();
  S.col2blk.assign(N, 0);
  for (int64_t b = 0; b < S.nb; ++b)
    for (int64_t c = S.blk_col0[b]; c < S.blk_col0[b] + S.blk_w[b]; ++c) S.col2blk[c] = (int32_t)b;
  // ---------------------------------------------------------------- trsv tiles and task queues
  // Big supernodes (more than one 64-column block) are swept through X_J = L_JJ⁻¹
  // (partitioned inverse): their intra-supernode rows are not tiled.
  S.tile_blk.clear(); S.tile_r0.clear(); S.tile_nr.clear(); S.tile_dlist.clear();
  S.tile_dptr.assign(1, 0);
  const bool split_dest = std::getenv("QPB_TILE_SPLIT") && std::atoi(std::getenv("QPB_TILE_SPLIT")) != 0;
  S.fwd_expect.assign(ns, 0);
  S.bwd_expect.assign(S.nb, 0);
  S.blk_big.assign(S.nb, 0);
  S.sn_xinv.assign(ns, -1);
  S.sn_sinv.assign(ns, -1);
  S.sym_true = 0;
  S.sym_lower = 0;
  S.sn_xtr.assign(ns, -1);
  S.sn_ldx.assign(ns, 0);
  S.sn_xtmp.assign(ns, -1);
  S.x_size = 0;
  S.xtmp_size = 0;
  for (int64_t J = 0; J < ns; ++J) {
    const int64_t w = S.sn_start[J + 1] - S.sn_start[J];
    if (w > BW) {
      const int64_t ldx = (w + 7) & ~int64_t(7);
      S.sn_ldx[J] = ldx;
      S.sn_xinv[J] = S.x_size;
      S.x_size += ldx * w;
      S.sn_xtr[J] = S.x_size;
      S.x_size += ldx * w;
      const int64_t m = S.sn_rowptr[J + 1] - S.sn_rowptr[J];
      if (allow_symroot && S.sn_parent[J] < 0 && m == w && !std::getenv("QPB_NO_SYMROOT")) {
        S.sn_sinv[J] = S.x_size;
        S.x_size += ldx * w;
        for (int64_t c = S.sn_start[J]; c < S.sn_start[J + 1]; ++c) S.sym_true += S.colcount[c];
        S.sym_lower += w * (w + 1) / 2;
      }
      S.sn_xtmp[J] = S.xtmp_size;
      S.xtmp_size += (w / 2 + BW) * (w / 2 + BW);
      for (int64_t b = S.sn_blk0[J]; b < S.sn_blk0[J + 1]; ++b) S.blk_big[b] = 1;
    }
  }
  // ---------------------------------------------------------------- leaf phase (level-synchronous)
  // The bottom levels of a nested-dissection tree hold tens of thousands of tiny supernodes (c2: 63 000 of
  // ≤ 16 columns in levels 0–6).  In the task graph each one costs a dependency hand-off (counter, fence,
  // release), and the leaves took ~300 µs of c2's 750 µs forward sweep at 0.7 TB/s.  Swept level by level
  // instead — one launch per level, a group of 16/32 lanes per supernode issuing all of its loads at once, no
  // counters — a level costs one memory round trip plus its bytes.  A level joins while every supernode in
  // it is a single block of ≤ 32 columns and it has ≥ LVL_MIN supernodes (QPB_LVL_MIN; QPB_LVL=0 disables).
  S.lvl_cut = 0;
  S.lvl_ptr.assign(1, 0);
  S.lvl_blk.clear();
  S.lvl_g.clear();
  std::vector<char> lvl_sn(ns, 0);
  {
    const char* e = std::getenv("QPB_LVL");
    const bool on = !(e && e[0] == '0');
    const int64_t lmin = std::getenv("QPB_LVL_MIN") ? std::max<int64_t>(1, std::atoll(std::getenv("QPB_LVL_MIN")))
                                                    : LVL_MIN;
    for (int64_t L = 0; on && L < S.n_levels && L < LVL_MAX; ++L) {
      const auto& sn = by_level[L];
      if ((int64_t)sn.size() < lmin) break;
      int64_t wmax = 0;
      bool ok = true;
      for (int32_t J : sn) {
        const int64_t w = S.sn_start[J + 1] - S.sn_start[J];
        const int64_t m = S.sn_rowptr[J + 1] - S.sn_rowptr[J];
        if (S.sn_blk0[J + 1] - S.sn_blk0[J] != 1 || w > 32 || S.sn_xinv[J] >= 0 || m - w >= (int64_t(1) << 25)) {
          ok = false;
          break;
        }
        wmax = std::max(wmax, w);
      }
      if (!ok) break;
      for (int32_t J : sn) {
        S.lvl_blk.push_back(S.sn_blk0[J]);
        lvl_sn[J] = 1;
      }
      S.lvl_ptr.push_back((int64_t)S.lvl_blk.size());
      S.lvl_g.push_back(wmax <= 16 ? 16 : 32);
      S.lvl_cut = (int32_t)(L + 1);
    }
  }
  std::vector<int64_t> blk_tile0(S.nb + 1, 0);
  std::vector<char> fused(S.nb, 0);
  // Root-row tiles: with a symmetric root R (the last supernode, columns [rc_split, N)), the rows of a
  // forest block that lie in R only feed R's right-hand side, which nothing but R reads.  Those rows get
  // tiles of their own.  Forward they are dispatched after every forest task, just before R, so the
  // level-by-level forest sweep no longer shares its CTAs and dispatch order with them and they stream at
  // the end with every dependency met (c2: 88 M of the forest's 145 M entries are root rows; forward sweep
  // 888 → 740 µs).  Backward they keep their place before their block's DIAG: there they fill the CTAs the
  // latency-bound top levels leave idle (all first: 680 → 745 µs; a quarter of the CTAs serving them from
  // a second queue: 1 050 µs).  QPB_ROOT_TILES=0 keeps them in place in both sweeps.
  const int64_t Jr = ns - 1;
  const bool root_tiles = Jr >= 0 && S.sn_sinv[Jr] >= 0 &&
                          !(std::getenv("QPB_ROOT_TILES") && std::getenv("QPB_ROOT_TILES")[0] == '0');
  const int64_t rc_split = root_tiles ? S.sn_start[Jr] : N;
  std::vector<char> tile_root;
  const int64_t fuse_elems = std::getenv("QPB_FUSE_ELEMS") ? std::atoll(std::getenv("QPB_FUSE_ELEMS")) : FUSE_ELEMS;
  S.blk_dptr.assign(S.nb + 1, 0);
  S.blk_dest.clear();
  for (int64_t b = 0; b < S.nb; ++b) {
    blk_tile0[b] = (int64_t)S.tile_blk.size();
    const int64_t J = S.blk_sn[b];
    const int64_t wk = S.blk_w[b], noff = S.blk_noff[b];
    if (lvl_sn[J]) {   // leaf phase: swept by the level kernels, no tiles, no counter contributions
      S.blk_dptr[b + 1] = (int64_t)S.blk_dest.size();
      continue;
    }
    if (!S.blk_big[b] && wk * noff <= fuse_elems) {
      fused[b] = 1;
      int64_t last = -1;
      for (int64_t r = 0; r < noff; ++r) {
        int64_t dsn = col2sn[S.sn_rows[S.blk_rows[b] + r]];
        if (dsn != last) {   // rows are sorted, so destination supernodes are non-decreasing
          S.blk_dest.push_back((int32_t)dsn);
          S.fwd_expect[dsn] += 1;
          last = dsn;
        }
      }
      S.blk_dptr[b + 1] = (int64_t)S.blk_dest.size();
      continue;
    }
    S.blk_dptr[b + 1] = (int64_t)S.blk_dest.size();
    // tiles fit the sweep's shared-memory staging (TILE_ELEMS); full-width blocks take long tiles of up to
    // LONG_TILE rows instead, swept straight from global memory (fewer tasks, counters and atomics)
    const int64_t cap = wk == BW ? LONG_TILE : std::max<int64_t>(1, std::min<int64_t>(1024, TILE_ELEMS / wk));
    // first off-diagonal row below the supernode's own columns
    // A tile may span several destination supernodes (rows are sorted, so they form runs): it bumps each
    // destination's forward counter once and, backward, waits for each destination's ready flag.  Tiles
    // split only by size, into equal parts: fewer tasks, so fewer CTAs parked on a dependency
    // (QPB_TILE_SPLIT=1 restores one destination per tile).
    const int64_t rstart = S.blk_big[b] ? (S.sn_start[J + 1] - (S.blk_col0[b] + wk)) : 0;
    int64_t nx = noff;   // rows are sorted: [0, nx) below rc_split, [nx, noff) in the symmetric root
    if (J != Jr)
      while (nx > 0 && S.sn_rows[S.blk_rows[b] + nx - 1] >= rc_split) --nx;
    const int64_t split = std::max(rstart, nx);
    for (int part = 0; part < 2; ++part) {
      int64_t r = part == 0 ? rstart : split;
      const int64_t rend = part == 0 ? split : noff;
      if (r >= rend) continue;
      const int64_t ntl = (rend - r + cap - 1) / cap, per = ntl > 0 ? (rend - r + ntl - 1) / ntl : cap;
      while (r < rend) {
        int64_t e = std::min(rend, r + per);
        if (split_dest) {
          const int64_t d0 = col2sn[S.sn_rows[S.blk_rows[b] + r]];
          e = r + 1;
          while (e < rend && e - r < cap && col2sn[S.sn_rows[S.blk_rows[b] + e]] == d0) ++e;
        }
        S.tile_blk.push_back((int32_t)b);
        S.tile_r0.push_back((int32_t)r);
        S.tile_nr.push_back((int32_t)(e - r));
        tile_root.push_back((char)part);   // part 1 = rows of the symmetric root
        int64_t last = -1;
        for (int64_t q = r; q < e; ++q) {
          const int64_t dsn = col2sn[S.sn_rows[S.blk_rows[b] + q]];
          if (dsn != last) {
            S.tile_dlist.push_back((int32_t)dsn);
            S.fwd_expect[dsn] += 1;
            last = dsn;
          }
        }
        S.tile_dptr.push_back((int64_t)S.tile_dlist.size());
        S.bwd_expect[b] += 1;
        r = e;
      }
    }
  }
  blk_tile0[S.nb] = (int64_t)S.tile_blk.size();
  auto enc = [](int type, int64_t idx) { return (int32_t)(((int64_t)type << TASK_SHIFT) | idx); };
  S.xt_bI.clear();
  S.xt_bK.clear();
  S.xt_nK.clear();
  S.xb_bK.clear();
  S.xb_bI.clear();
  S.xb_nI.clear();
  std::vector<int64_t> sn_xb0(ns + 1, 0);
  S.xexp_f.assign(S.nb, 0);
  S.xexp_b.assign(S.nb, 0);
  S.sexp.assign(S.nb, 0);
  S.sn_nblk.assign(ns, 0);
  std::vector<int64_t> sn_xt0(ns + 1, 0);
  for (int64_t J = 0; J < ns; ++J) {
    sn_xt0[J] = (int64_t)S.xt_bI.size();
    sn_xb0[J] = (int64_t)S.xb_bK.size();
    S.sn_nblk[J] = S.sn_blk0[J + 1] - S.sn_blk0[J];
    if (S.sn_xinv[J] < 0) continue;
    const int64_t b0 = S.sn_blk0[J], b1 = S.sn_blk0[J + 1], T = b1 - b0;
    for (int64_t I = 0; I < T; ++I)
      for (int64_t K = 0; K <= I; K += XCH) {
        S.xt_bI.push_back((int32_t)(b0 + I));
        S.xt_bK.push_back((int32_t)(b0 + K));
        S.xt_nK.push_back((int32_t)std::min<int64_t>(XCH, I + 1 - K));
      }
    for (int64_t K = 0; K < T; ++K)
      for (int64_t I = K; I < T; I += XCH) {
        S.xb_bK.push_back((int32_t)(b0 + K));
        S.xb_bI.push_back((int32_t)(b0 + I));
        S.xb_nI.push_back((int32_t)std::min<int64_t>(XCH, T - I));
      }
    for (int64_t I = 0; I < T; ++I) {
      S.xexp_f[b0 + I] = (int32_t)((I + XCH) / XCH);           // forward chunks covering row-block I
      S.xexp_b[b0 + I] = (int32_t)((T - I + XCH - 1) / XCH);   // backward chunks of output block K = I
      if (S.sn_sinv[J] >= 0) S.sexp[b0 + I] = (int32_t)((I + XCH) / XCH + (T - 1 - I));
    }
  }
  sn_xt0[ns] = (int64_t)S.xt_bI.size();
  sn_xb0[ns] = (int64_t)S.xb_bK.size();
  if ((int64_t)S.xt_bI.size() >= (int64_t(1) << TASK_SHIFT) || (int64_t)S.tile_blk.size() >= (int64_t(1) << TASK_SHIFT))
    return "too many sweep tasks for the 28-bit task encoding";
  // Level-major dispatch: the forward queue by height (leaves first), the backward queue by depth
  // (root first), each stable in postorder.  Every dependency of a task is dispatched before it,
  // and no CTA holding a waiting task blocks the dispatch of a task of an earlier wave.
  std::vector<int32_t> fwd_order(ns), bwd_order(ns);
  {
    std::vector<int64_t> depth(ns, 0);
    for (int64_t J = ns - 1; J >= 0; --J)
      if (S.sn_parent[J] >= 0) depth[J] = depth[S.sn_parent[J]] + 1;
    for (int64_t J = 0; J < ns; ++J) fwd_order[J] = bwd_order[J] = (int32_t)J;
    std::stable_sort(fwd_order.begin(), fwd_order.end(),
                     [&](int32_t a, int32_t b) { return S.sn_level[a] < S.sn_level[b]; });
    std::stable_sort(bwd_order.begin(), bwd_order.end(),
                     [&](int32_t a, int32_t b) { return depth[a] < depth[b]; });
  }
  // Tiny single-block supernodes (w ≤ 32, noff ≤ 256, w·noff ≤ 1024) are swept WARP-wide: groups of
  // up to 8 from the same level (height forward, depth backward) form one task (type 7), one warp each.
  // (Measured slower: chaining whole subtrees of them through one warp — c2 forward 740 → 810 µs, c4s
  // 284 → 373 µs, the per-supernode latency, not the dependency hops, bounds this phase — and one claim
  // queue per level from which every warp of ⌈count/8⌉ tasks takes supernodes one at a time — c2 forward
  // 748 → 757 µs.)
  std::vector<int32_t> tiny_f(ns, -1), tiny_b(ns, -1);   // group id of J, set on every member
  std::vector<char> first_f(ns, 0), first_b(ns, 0);
  {
    auto tiny = [&](int64_t J) {
      if (S.sn_blk0[J + 1] - S.sn_blk0[J] != 1 || lvl_sn[J]) return false;
      const int64_t b = S.sn_blk0[J];
      const int64_t w = S.blk_w[b], noff = S.blk_noff[b];
      return fused[b] && w <= 32 && noff <= 256 && w * noff <= 1024 && S.sn_xinv[J] < 0;
    };
    auto group = [&](const std::vector<int32_t>& order, const std::vector<int64_t>& key,
                     std::vector<int32_t>& gid, std::vector<char>& first, std::vector<int32_t>& out) {
      out.clear();
      int64_t cur_key = -1, fill = 8;
      for (int32_t J : order) {
        if (!tiny(J)) continue;
        if (key[J] != cur_key || fill == 8) {
          out.resize(out.size() + 8, -1);
          cur_key = key[J];
          fill = 0;
          first[J] = 1;
        }
        const int64_t g = (int64_t)out.size() / 8 - 1;
        out[g * 8 + fill++] = S.sn_blk0[J];
        gid[J] = (int32_t)g;
      }
    };
    std::vector<int64_t> height(S.sn_level.begin(), S.sn_level.end()), depth(ns, 0);
    for (int64_t J = ns - 1; J >= 0; --J)
      if (S.sn_parent[J] >= 0) depth[J] = depth[S.sn_parent[J]] + 1;
    group(fwd_order, height, tiny_f, first_f, S.snw_fwd);
    group(bwd_order, depth, tiny_b, first_b, S.snw_bwd);
  }
  // root-row tiles (see rc_split above), in block order
  std::vector<int64_t> rtiles;
  for (int64_t t = 0; t < (int64_t)tile_root.size(); ++t)
    if (tile_root[t]) rtiles.push_back(t);
  auto build_queues = [&](bool use_sym, std::vector<int32_t>& fq, std::vector<int32_t>& bq) {
    fq.clear();
    bq.clear();
    for (int32_t J : fwd_order) {
      const int64_t b0 = S.sn_blk0[J], b1 = S.sn_blk0[J + 1];
      const bool sym = use_sym && S.sn_sinv[J] >= 0;
      if (J == Jr)   // every forest task is dispatched: now the root-row tiles, then the root
        for (int64_t t : rtiles) fq.push_back(enc(1, t));
      if (lvl_sn[J]) continue;
      if (tiny_f[J] >= 0) {
        if (first_f[J]) fq.push_back(enc(7, tiny_f[J]));
        continue;
      }
      if (S.sn_xinv[J] < 0) {
        for (int64_t b = b0; b < b1; ++b) {
          fq.push_back(enc(fused[b] ? 4 : 0, b));
          for (int64_t t = blk_tile0[b]; t < blk_tile0[b + 1]; ++t)
            if (!tile_root[t]) fq.push_back(enc(1, t));
        }
      } else {
        for (int64_t b = b0; b < b1; ++b) fq.push_back(enc(2, b));
        if (!sym)
          for (int64_t x = sn_xt0[J]; x < sn_xt0[J + 1]; ++x) fq.push_back(enc(3, x));
        for (int64_t b = b0; b < b1; ++b)
          for (int64_t t = blk_tile0[b]; t < blk_tile0[b + 1]; ++t)
            if (!tile_root[t]) fq.push_back(enc(1, t));
      }
    }
    for (int32_t J : bwd_order) {
      const int64_t b0 = S.sn_blk0[J], b1 = S.sn_blk0[J + 1];
      const bool sym = use_sym && S.sn_sinv[J] >= 0;
      if (lvl_sn[J]) continue;
      if (tiny_b[J] >= 0) {
        if (first_b[J]) bq.push_back(enc(7, tiny_b[J]));
        continue;
      }
      if (S.sn_xinv[J] < 0) {
        for (int64_t b = b1 - 1; b >= b0; --b) {
          for (int64_t t = blk_tile0[b + 1] - 1; t >= blk_tile0[b]; --t) bq.push_back(enc(1, t));
          bq.push_back(enc(fused[b] ? 4 : 0, b));
        }
      } else {
        if (sym) {
          bq.push_back(enc(6, J));
        } else {
          for (int64_t b = b1 - 1; b >= b0; --b)
            for (int64_t t = blk_tile0[b + 1] - 1; t >= blk_tile0[b]; --t) bq.push_back(enc(1, t));
          for (int64_t b = b0; b < b1; ++b) bq.push_back(enc(2, b));
          for (int64_t x = sn_xb0[J]; x < sn_xb0[J + 1]; ++x) bq.push_back(enc(3, x));
        }
      }
    }
  };
  build_queues(true, S.fwd_tasks, S.bwd_tasks);

  S.sym_c0 = S.sym_c1 = 0;
  for (int64_t J = 0; J < ns; ++J)
    if (S.sn_sinv[J] >= 0) {   // symmetric roots are etree roots: at most one chunk range per root, roots last
      if (S.sym_c1 == 0) S.sym_c0 = sn_xt0[J];
      S.sym_c1 = sn_xt0[J + 1];
    }
  build_queues(false, S.fwd_tasks_x, S.bwd_tasks_x);
  // ---------------------------------------------------------------- assembly map (grouped by level), relative indices
  S.asm_dst.clear();
  S.asm_val.clear();
  S.asm_src.clear();
  S.asm_diag.clear();
  S.diag_dst.assign(N, 0);
  S.relind.clear();
  S.relind_off.assign(ns, -1);
  S.level_ea.assign(S.n_levels, LevelEA{0, 0, 0, 0, 0, 0});
  S.lev_fronts.clear();
  S.lev_zpref.clear();
  {
    std::vector<int32_t> posmap(N, -1);
    for (int64_t L = 0; L < S.n_levels; ++L) {
      S.level_ea[L].asm_off = (int64_t)S.asm_dst.size();
      S.level_ea[L].fr_off = (int64_t)S.lev_zpref.size();
      S.level_ea[L].n_fr = (int64_t)by_level[L].size();
      int64_t zacc = 0;
      for (int32_t J : by_level[L]) {
        S.lev_fronts.push_back(J);
        S.lev_zpref.push_back(zacc);
        const int64_t mJ = S.sn_rowptr[J + 1] - S.sn_rowptr[J];
        zacc += mJ * mJ;
      }
      S.lev_fronts.push_back(-1);   // keeps lev_fronts aligned with lev_zpref
      S.lev_zpref.push_back(zacc);
      for (int32_t J : by_level[L]) {
        const int64_t c0 = S.sn_start[J], c1 = S.sn_start[J + 1];
        const int64_t r0 = S.sn_rowptr[J], m = S.sn_rowptr[J + 1] - r0;
        for (int64_t q = 0; q < m; ++q) posmap[S.sn_rows[r0 + q]] = (int32_t)q;
        for (int64_t c = c0; c < c1; ++c) {
          const int64_t colbase = S.front_off[J] + (c - c0) * m;
          S.diag_dst[c] = colbase + posmap[c];
          S.asm_dst.push_back(colbase + posmap[c]);
          S.asm_val.push_back(M.diag.empty() ? 0.0 : M.diag[c]);
          S.asm_src.push_back(M.diag_src.empty() ? -1 : M.diag_src[c]);
          S.asm_diag.push_back((int32_t)c);
          for (int64_t q = M.colptr[c]; q < M.colptr[c + 1]; ++q) {
            S.asm_dst.push_back(colbase + posmap[M.rowind[q]]);
            S.asm_val.push_back(M.val.empty() ? 0.0 : M.val[q]);
            S.asm_src.push_back(M.src.empty() ? -1 : M.src[q]);
            S.asm_diag.push_back(-1);
          }
        }
        for (int32_t K : children[J]) {
          const int64_t k0 = S.sn_rowptr[K], mK = S.sn_rowptr[K + 1] - k0;
          const int64_t wK = S.sn_start[K + 1] - S.sn_start[K];
          S.relind_off[K] = (int64_t)S.relind.size();
          for (int64_t q = wK; q < mK; ++q) {
            int32_t p = posmap[S.sn_rows[k0 + q]];
            if (p < 0) return "child row missing from parent front (internal error)";
            S.relind.push_back(p);
          }
        }
        for (int64_t q = 0; q < m; ++q) posmap[S.sn_rows[r0 + q]] = -1;
      }
      S.level_ea[L].n_asm = (int64_t)S.asm_dst.size() - S.level_ea[L].asm_off;
    }
  }
  // ---------------------------------------------------------------- levels: extend-add groups and steps
  S.grp_P.clear(); S.grp_pc.clear(); S.grp_K.clear(); S.grp_j.clear();
  S.grp_ptr.assign(1, 0);
  S.steps.clear();
  S.act.clear();
  S.pan_pref.clear();
  S.upd_pref.clear();
  S.pref_off.clear();
  std::vector<std::pair<int32_t, std::pair<int32_t, int32_t>>> ent;  // (pc, (K, j))
  for (int64_t L = 0; L < S.n_levels; ++L) {
    S.level_ea[L].grp_off = (int64_t)S.grp_P.size();
    for (int32_t P : by_level[L]) {
      ent.clear();
      for (int32_t K : children[P]) {
        const int64_t mK = S.sn_rowptr[K + 1] - S.sn_rowptr[K];
        const int64_t wK = S.sn_start[K + 1] - S.sn_start[K];
        for (int64_t j = wK; j < mK; ++j)
          ent.push_back({S.relind[S.relind_off[K] + (j - wK)], {K, (int32_t)j}});
      }
      std::stable_sort(ent.begin(), ent.end(), [](auto& a, auto& b) { return a.first < b.first; });
      for (size_t e = 0; e < ent.size();) {
        size_t f = e;
        while (f < ent.size() && ent[f].first == ent[e].first) {
          S.grp_K.push_back(ent[f].second.first);
          S.grp_j.push_back(ent[f].second.second);
          ++f;
        }
        S.grp_P.push_back(P);
        S.grp_pc.push_back(ent[e].first);
        S.grp_ptr.push_back((int64_t)S.grp_K.size());
        e = f;
      }
    }
    S.level_ea[L].n_grp = (int64_t)S.grp_P.size() - S.level_ea[L].grp_off;
    // steps
    int64_t max_nk = 0;
    for (int32_t J : by_level[L]) {
      int64_t w = S.sn_start[J + 1] - S.sn_start[J];
      max_nk = std::max(max_nk, (w + BW - 1) / BW);
    }
    // Steps, in groups of G pivot blocks k0 .. e (e = min(k0 + G, nk) − 1 per front): for each block g
    // of the group, DIAG+PANEL(g), then (g < e) UPDATE of the group's remaining block columns g+1 .. e by
    // block g (kind 2, a narrow band); after the group, ONE UPDATE of the trailing triangle (block columns
    // > e) with all the group's pivot columns (kind 3, up to 64·G of them).  The trailing matrix is then
    // read and written once per G blocks.  QPB_GROUP = G (default 4; 1 = one block per update).
    const int64_t G = std::getenv("QPB_GROUP") ? std::max<int64_t>(1, std::min<int64_t>(4, std::atoll(std::getenv("QPB_GROUP"))))
                                               : 4;
    S.mf_group = (int32_t)G;
    auto add_step = [&](int64_t k, int64_t k0, int kind, auto select) {
      StepDesc sd;
      sd.level = (int)L;
      sd.k = (int)k;
      sd.k0 = (int)k0;
      sd.kind = kind;
      sd.act_off = (int64_t)S.act.size();
      S.pref_off.push_back((int64_t)S.pan_pref.size());
      S.pan_pref.push_back(0);
      S.upd_pref.push_back(0);
      int n_act = 0;
      for (int32_t J : by_level[L]) {
        const int64_t w = S.sn_start[J + 1] - S.sn_start[J];
        const int64_t m = S.sn_rowptr[J + 1] - S.sn_rowptr[J];
        const int64_t nk = (w + BW - 1) / BW;
        if (!select(nk)) continue;
        const int64_t ntile = nk + (m - w + BW - 1) / BW;
        const int64_t e = std::min(k0 + G, nk) - 1;   // last block of this front's group
        int64_t pan = 0, upd = 0;
        if (kind == 0) {
          pan = ntile - k - 1;
        } else if (kind == 2) {
          for (int64_t tj = k + 1; tj <= e; ++tj) upd += ntile - tj;
        } else {
          const int64_t T = ntile - e - 1;
          upd = T * (T + 1) / 2;
        }
        if (kind != 0 && upd == 0) continue;
        S.act.push_back(J);
        S.pan_pref.push_back(S.pan_pref.back() + pan);
        S.upd_pref.push_back(S.upd_pref.back() + upd);
        ++n_act;
      }
      sd.n_act = n_act;
      sd.pan_total = S.pan_pref.back();
      sd.upd_total = S.upd_pref.back();
      if (n_act > 0) S.steps.push_back(sd);
      else {
        S.pref_off.pop_back();
        S.pan_pref.pop_back();
        S.upd_pref.pop_back();
      }
    };
    for (int64_t k0 = 0; k0 < max_nk; k0 += G) {
      for (int64_t g = k0; g < std::min(k0 + G, max_nk); ++g) {
        add_step(g, k0, 0, [&](int64_t nk) { return nk > g; });
        add_step(g, k0, 2, [&](int64_t nk) { return nk > g + 1 && g + 1 < k0 + G; });
      }
      add_step(k0, k0, 3, [&](int64_t nk) { return nk > k0; });
    }
  }
  S.pivsign.assign(N, 1);
  for (int64_t c = 0; c < std::min(N, n_negative); ++c) S.pivsign[c] = -1;
  (void)tile_begin;
  if (allow_symroot) plan_flat(S);
  return "";
}

void plan_flat(Symbolic& S, int64_t max_cols, double max_rel_root) {
  S.flat = false;
  const bool verbose = std::getenv("QPB_VERBOSE") != nullptr;
  auto no = [&](const char* why) {
    if (verbose) std::fprintf(stderr, "qpb: flattened forest not used: %s\n", why);
  };
  const int64_t ns = S.ns;
  if (ns < 1) return no("empty");
  const int64_t J0 = ns - 1;
  if (S.sn_sinv[J0] < 0 || S.sn_parent[J0] >= 0) return no("last supernode is not a symmetric root");
  const int64_t rc0 = S.sn_start[J0];
  const int64_t wr = S.N - rc0;
  if (rc0 > max_cols) return no("forest too wide");
  for (int64_t J = 0; J < J0; ++J) {
    if (S.sn_sinv[J] >= 0 || S.sn_start[J + 1] - S.sn_start[J] > BW) return no("forest supernode wider than 64");
  }
  // R_J = ∪ root rows of the supernodes on the path J → root (children before parents in index
  // order, so the parent's set is complete when J is processed top-down)
  std::vector<std::vector<int32_t>> R(J0);
  for (int64_t J = J0 - 1; J >= 0; --J) {
    std::vector<int32_t> own;
    for (int64_t q = S.sn_rowptr[J]; q < S.sn_rowptr[J + 1]; ++q)
      if (S.sn_rows[q] >= rc0) own.push_back((int32_t)(S.sn_rows[q] - rc0));
    const int64_t P = S.sn_parent[J];   // −1: a separate tree (no root rows above it)
    if (P >= 0 && P != J0) {
      std::vector<int32_t> u;
      std::set_union(own.begin(), own.end(), R[P].begin(), R[P].end(), std::back_inserter(u));
      R[J].swap(u);
    } else {
      R[J].swap(own);
    }
  }
  int64_t nnzM = 0;
  for (int64_t J = 0; J < J0; ++J) nnzM += (int64_t)R[J].size() * (S.sn_start[J + 1] - S.sn_start[J]);
  if ((double)nnzM > max_rel_root * (double)wr * (double)(wr + 1) / 2) return no("M too large");
  if (verbose) std::fprintf(stderr, "qpb: flattened forest: %lld columns, nnz(M) = %lld\n", (long long)rc0,
                            (long long)nnzM);
  S.flat = true;
  S.fl_rc0 = rc0;
  S.fl_roff.assign(J0 + 1, 0);
  S.fl_moff.assign(J0 + 1, 0);
  S.fl_rows.clear();
  for (int64_t J = 0; J < J0; ++J) {
    S.fl_rows.insert(S.fl_rows.end(), R[J].begin(), R[J].end());
    S.fl_roff[J + 1] = (int64_t)S.fl_rows.size();
    S.fl_moff[J + 1] = S.fl_moff[J] + (int64_t)R[J].size() * (S.sn_start[J + 1] - S.sn_start[J]);
  }
  S.fl_msize = S.fl_moff[J0];
  // L11⁻¹ column patterns: column c of supernode J → J's columns ≥ c, then every forest ancestor's columns
  S.fl_col2sn.assign(rc0, 0);
  S.fl_cp.assign(rc0 + 1, 0);
  S.fl_ci.clear();
  for (int64_t J = 0; J < J0; ++J)
    for (int64_t c = S.sn_start[J]; c < S.sn_start[J + 1]; ++c) {
      S.fl_col2sn[c] = (int32_t)J;
      for (int64_t r = c; r < S.sn_start[J + 1]; ++r) S.fl_ci.push_back((int32_t)r);
      for (int64_t K = S.sn_parent[J]; K >= 0 && K != J0; K = S.sn_parent[K])
        for (int64_t r = S.sn_start[K]; r < S.sn_start[K + 1]; ++r) S.fl_ci.push_back((int32_t)r);
      S.fl_cp[c + 1] = (int64_t)S.fl_ci.size();
    }
  // row form with the index of each entry in the column-ordered values
  S.fl_rp.assign(rc0 + 1, 0);
  for (int32_t r : S.fl_ci) S.fl_rp[r + 1]++;
  for (int64_t r = 0; r < rc0; ++r) S.fl_rp[r + 1] += S.fl_rp[r];
  S.fl_rj.assign(S.fl_ci.size(), 0);
  S.fl_r2c.assign(S.fl_ci.size(), 0);
  {
    std::vector<int64_t> pos(S.fl_rp.begin(), S.fl_rp.end() - 1);
    for (int64_t c = 0; c < rc0; ++c)
      for (int64_t e = S.fl_cp[c]; e < S.fl_cp[c + 1]; ++e) {
        const int64_t d = pos[S.fl_ci[e]]++;
        S.fl_rj[d] = (int32_t)c;
        S.fl_r2c[d] = e;
      }
  }
  // row form of M for the forward product (no atomics: one dot product per root row)
  S.fl_mr_ptr.assign(wr + 1, 0);
  for (int64_t J = 0; J < J0; ++J)
    for (int32_t r : R[J]) S.fl_mr_ptr[r + 1] += S.sn_start[J + 1] - S.sn_start[J];
  for (int64_t r = 0; r < wr; ++r) S.fl_mr_ptr[r + 1] += S.fl_mr_ptr[r];
  S.fl_mr_col.assign(S.fl_mr_ptr[wr], 0);
  S.fl_mr_src.assign(S.fl_mr_ptr[wr], 0);
  {
    std::vector<int64_t> pos(S.fl_mr_ptr.begin(), S.fl_mr_ptr.end() - 1);
    for (int64_t J = 0; J < J0; ++J) {
      const int64_t w = S.sn_start[J + 1] - S.sn_start[J], nr = (int64_t)R[J].size();
      for (int64_t t = 0; t < w; ++t)
        for (int64_t q = 0; q < nr; ++q) {
          const int64_t d = pos[R[J][q]]++;
          S.fl_mr_col[d] = (int32_t)(S.sn_start[J] + t);
          S.fl_mr_src[d] = (int32_t)(S.fl_moff[J] + t * nr + q);
        }
    }
  }
  // backward M tiles
  S.fl_mt_J.clear();
  S.fl_mt_q0.clear();
  S.fl_mt_nq.clear();
  for (int64_t J = 0; J < J0; ++J) {
    const int64_t w = S.sn_start[J + 1] - S.sn_start[J], nr = (int64_t)R[J].size();
    // ≤ 2 rows per thread of a 256-thread CTA: every load of a tile is in flight at once
    const int64_t cap = std::min<int64_t>(512, std::max<int64_t>(1, TILE_ELEMS / std::max<int64_t>(1, w)));
    for (int64_t q = 0; q < nr; q += cap) {
      S.fl_mt_J.push_back((int32_t)J);
      S.fl_mt_q0.push_back((int32_t)q);
      S.fl_mt_nq.push_back((int32_t)std::min(cap, nr - q));
    }
  }
}

}  // namespace qpb

namespace qpb {

// Approximate minimum degree on the quotient graph (element absorption,
// aggressive absorption of elements contained in the new element, AMD-style
// external degree bound d_i ≤ |A_i| + |L_p \ i| + Σ_{e∈E_i\p} |L_e \ L_p|).
// A fill-reducing heuristic for the x block of F and for P_H; the paper does
// not fix an ordering (it used dense SYTRF).  Deterministic.
std::vector<int64_t> min_degree_order(int64_t n, const std::vector<int64_t>& ptr, const std::vector<int32_t>& idx,
                                      double dense_stop) {
  std::vector<std::vector<int32_t>> Av(n), Ev(n), Le(n);
  std::vector<int64_t> deg(n);
  for (int64_t i = 0; i < n; ++i) {
    Av[i].assign(idx.begin() + ptr[i], idx.begin() + ptr[i + 1]);
    std::sort(Av[i].begin(), Av[i].end());
    Av[i].erase(std::unique(Av[i].begin(), Av[i].end()), Av[i].end());
    Av[i].erase(std::remove(Av[i].begin(), Av[i].end(), (int32_t)i), Av[i].end());
    deg[i] = (int64_t)Av[i].size();
  }
  // degree buckets (doubly linked)
  std::vector<int64_t> head(n + 1, -1), nxt(n, -1), prv(n, -1);
  auto insert = [&](int64_t i) {
    int64_t d = deg[i];
    nxt[i] = head[d];
    prv[i] = -1;
    if (head[d] >= 0) prv[head[d]] = i;
    head[d] = i;
  };
  auto remove = [&](int64_t i) {
    if (prv[i] >= 0) nxt[prv[i]] = nxt[i];
    else head[deg[i]] = nxt[i];
    if (nxt[i] >= 0) prv[nxt[i]] = prv[i];
    nxt[i] = prv[i] = -1;
  };
  for (int64_t i = n - 1; i >= 0; --i) insert(i);
  std::vector<char> state(n, 0);  // 0 variable, 1 element, 2 absorbed / dead
  std::vector<int64_t> mark(n, -1), wstamp(n, -1), w(n, 0);
  std::vector<int64_t> order;
  order.reserve(n);
  std::vector<int32_t> Lp, tmp;
  int64_t mind = 0;
  for (int64_t k = 0; k < n; ++k) {
    while (mind <= n && head[mind] < 0) ++mind;
    if (mind > n) break;
    if (n - k > 64 && (mind >= n - k - 1 || (dense_stop < 1.0 && (double)mind >= dense_stop * (double)(n - k - 1)))) {
      // every remaining variable has (approximate) external degree n-k-1: the rest is a
      // clique, its internal order does not change the fill — append in index order.  With
      // dense_stop < 1 the same is done once the minimum degree reaches that fraction of the
      // remaining nodes (the tail then factors as one dense block anyway)
      for (int64_t i = 0; i < n; ++i)
        if (state[i] == 0) order.push_back(i);
      break;
    }
    const int64_t p = head[mind];
    remove(p);
    // new element L_p
    Lp.clear();
    mark[p] = k;
    for (int32_t v : Av[p])
      if (state[v] == 0 && mark[v] != k) { mark[v] = k; Lp.push_back(v); }
    for (int32_t e : Ev[p]) {
      if (state[e] != 1) continue;
      for (int32_t v : Le[e])
        if (state[v] == 0 && mark[v] != k) { mark[v] = k; Lp.push_back(v); }
      state[e] = 2;
      std::vector<int32_t>().swap(Le[e]);
    }
    state[p] = 1;
    std::vector<int32_t>().swap(Av[p]);
    std::vector<int32_t>().swap(Ev[p]);
    Le[p] = Lp;
    order.push_back(p);
    // |L_e \ L_p| for elements adjacent to L_p
    for (int32_t i : Lp)
      for (int32_t e : Ev[i]) {
        if (state[e] != 1) continue;
        if (wstamp[e] != k) { wstamp[e] = k; w[e] = (int64_t)Le[e].size(); }
        w[e] -= 1;
      }
    const int64_t nrem = n - k - 1;
    const int64_t lp = (int64_t)Lp.size();
    for (int32_t i : Lp) {
      tmp.clear();
      int64_t ext = 0;
      for (int32_t e : Ev[i]) {
        if (state[e] != 1 || e == p) continue;
        if (wstamp[e] == k && w[e] == 0) {  // L_e ⊆ L_p: aggressive absorption
          state[e] = 2;
          std::vector<int32_t>().swap(Le[e]);
          continue;
        }
        tmp.push_back(e);
        ext += wstamp[e] == k ? w[e] : (int64_t)Le[e].size();
      }
      tmp.push_back((int32_t)p);
      Ev[i].swap(tmp);
      tmp.clear();
      for (int32_t v : Av[i])
        if (state[v] == 0 && mark[v] != k) tmp.push_back(v);
      Av[i].swap(tmp);
      int64_t d = (int64_t)Av[i].size() + (lp - 1) + ext;
      d = std::min(d, deg[i] + lp - 1);
      d = std::min(d, nrem - 1 < 0 ? 0 : nrem - 1);
      if (d < 0) d = 0;
      remove(i);
      deg[i] = d;
      insert(i);
      if (d < mind) mind = d;
    }
  }
  return order;
}

}  // namespace qpb

namespace qpb {

// Postorder the elimination tree of the symmetric pattern (ptr, idx) under the
// ordering `order` (new→old): an equivalent reordering (same fill) that makes
// every last child contiguous with its parent, so chains of supernodes can be
// amalgamated.  Returns the composed order (new→old).
// Nested dissection by level structures (George's method): in each connected part, a BFS from a
// pseudo-peripheral node splits the part at its middle level; the two sides are ordered recursively and
// the separator level last.  Parts of at most `leaf` nodes keep their input order.  Its elimination tree
// has logarithmic depth on band- and grid-like graphs, where minimum degree can leave a long chain of
// narrow supernodes (c4s's P_H: the banded T = C diag(H)⁻¹ Cᵀ).
std::vector<int64_t> nested_dissection_order(int64_t n, const std::vector<int64_t>& ptr,
                                             const std::vector<int32_t>& idx, int64_t leaf) {
  std::vector<int64_t> order;
  order.reserve(n);
  std::vector<int64_t> part(n, 0);        // current part id of every unordered node; −1 = ordered
  std::vector<int64_t> level(n, -1);
  int64_t next_id = 1;
  // explicit stack of (part id, node list)
  std::vector<std::pair<int64_t, std::vector<int64_t>>> st;
  {
    std::vector<int64_t> all(n);
    for (int64_t i = 0; i < n; ++i) all[i] = i;
    st.push_back({0, std::move(all)});
  }
  // deferred output: a separator must follow both of its sides, so push markers
  struct Item { bool sep; int64_t id; std::vector<int64_t> nodes; };
  std::vector<Item> work;
  work.push_back({false, 0, std::move(st.back().second)});
  st.clear();
  auto bfs = [&](int64_t src, int64_t pid, std::vector<int64_t>& seen) {
    seen.clear();
    seen.push_back(src);
    level[src] = 0;
    for (size_t h = 0; h < seen.size(); ++h) {
      const int64_t u = seen[h];
      for (int64_t q = ptr[u]; q < ptr[u + 1]; ++q) {
        const int64_t v = idx[q];
        if (part[v] == pid && level[v] < 0) {
          level[v] = level[u] + 1;
          seen.push_back(v);
        }
      }
    }
  };
  std::vector<int64_t> seen;
  while (!work.empty()) {
    Item it = std::move(work.back());
    work.pop_back();
    if (it.sep) {
      for (int64_t v : it.nodes) {
        order.push_back(v);
        part[v] = -1;
      }
      continue;
    }
    std::vector<int64_t>& S = it.nodes;
    if ((int64_t)S.size() <= leaf) {
      std::sort(S.begin(), S.end());
      for (int64_t v : S) {
        order.push_back(v);
        part[v] = -1;
      }
      continue;
    }
    const int64_t pid = it.id;
    // connected component of S[0]; the rest of S is a separate part (pushed back)
    bfs(S[0], pid, seen);
    if (seen.size() < S.size()) {
      std::vector<int64_t> rest;
      for (int64_t v : S)
        if (level[v] < 0) rest.push_back(v);
      for (int64_t v : seen) level[v] = -1;
      const int64_t id2 = next_id++;
      for (int64_t v : rest) part[v] = id2;
      std::vector<int64_t> comp(seen);
      work.push_back({false, id2, std::move(rest)});
      work.push_back({false, pid, std::move(comp)});
      continue;
    }
    // pseudo-peripheral node: repeat BFS from the last (deepest) node while the depth grows
    int64_t src = seen.back(), depth = level[seen.back()];
    for (int rep = 0; rep < 4; ++rep) {
      for (int64_t v : seen) level[v] = -1;
      bfs(src, pid, seen);
      const int64_t d = level[seen.back()];
      if (d <= depth && rep > 0) break;
      depth = d;
      src = seen.back();
    }
    if (depth < 2) {   // (nearly) a clique: no useful separator
      std::sort(S.begin(), S.end());
      for (int64_t v : seen) level[v] = -1;
      for (int64_t v : S) {
        order.push_back(v);
        part[v] = -1;
      }
      continue;
    }
    // middle level by node count
    std::vector<int64_t> cnt(depth + 1, 0);
    for (int64_t v : seen) cnt[level[v]]++;
    int64_t acc = 0, mid = 1;
    for (int64_t l = 0; l <= depth; ++l) {
      acc += cnt[l];
      if (2 * acc >= (int64_t)seen.size()) {
        mid = std::max<int64_t>(1, std::min<int64_t>(l, depth - 1));
        break;
      }
    }
    std::vector<int64_t> A, B, Sep;
    for (int64_t v : seen) (level[v] < mid ? A : level[v] > mid ? B : Sep).push_back(v);
    for (int64_t v : seen) level[v] = -1;
    const int64_t ia = next_id++, ib = next_id++;
    for (int64_t v : A) part[v] = ia;
    for (int64_t v : B) part[v] = ib;
    for (int64_t v : Sep) part[v] = -2;   // not in any part any more
    std::sort(Sep.begin(), Sep.end());
    work.push_back({true, -2, std::move(Sep)});
    work.push_back({false, ib, std::move(B)});
    work.push_back({false, ia, std::move(A)});
  }
  return order;
}

std::vector<int64_t> etree_postorder(int64_t n, const std::vector<int64_t>& ptr, const std::vector<int32_t>& idx,
                                     const std::vector<int64_t>& order) {
  std::vector<int64_t> pinv(n);
  for (int64_t i = 0; i < n; ++i) pinv[order[i]] = i;
  std::vector<int64_t> parent(n, -1), anc(n, -1);
  // Liu's algorithm over rows of the permuted lower triangle
  std::vector<int64_t> rp(n + 1, 0);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t q = ptr[i]; q < ptr[i + 1]; ++q)
      if (pinv[idx[q]] < pinv[i]) rp[pinv[i] + 1]++;
  for (int64_t i = 0; i < n; ++i) rp[i + 1] += rp[i];
  std::vector<int64_t> rc(rp[n]);
  {
    std::vector<int64_t> pos(rp.begin(), rp.end() - 1);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t q = ptr[i]; q < ptr[i + 1]; ++q)
        if (pinv[idx[q]] < pinv[i]) rc[pos[pinv[i]]++] = pinv[idx[q]];
  }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
      int64_t r = rc[q];
      while (anc[r] != -1 && anc[r] != i) {
        int64_t t = anc[r];
        anc[r] = i;
        r = t;
      }
      if (anc[r] == -1) {
        anc[r] = i;
        parent[r] = i;
      }
    }
  // children lists (increasing), iterative DFS from roots in increasing order
  std::vector<int64_t> head(n, -1), next(n, -1);
  for (int64_t j = n - 1; j >= 0; --j)
    if (parent[j] >= 0) {
      next[j] = head[parent[j]];
      head[parent[j]] = j;
    }
  std::vector<int64_t> post;
  post.reserve(n);
  std::vector<int64_t> stack;
  for (int64_t r = 0; r < n; ++r) {
    if (parent[r] >= 0) continue;
    stack.push_back(r);
    while (!stack.empty()) {
      int64_t p = stack.back();
      int64_t c = head[p];
      if (c >= 0) {
        head[p] = next[c];
        stack.push_back(c);
      } else {
        stack.pop_back();
        post.push_back(p);
      }
    }
  }
  std::vector<int64_t> out(n);
  for (int64_t k = 0; k < n; ++k) out[k] = order[post[k]];
  return out;
}

}  // namespace qpb
