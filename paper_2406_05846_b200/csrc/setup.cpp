#include <cstdlib>
#include <cstdio>
// Host setup of libstrom: SDP assembly/validation and the one-time factorisation
// of eps I + AA* (eq:strom:gpu:cholesky).
//
// Ordering. The rows of A fall into three classes read off
// the chain structure (Fig. 1):
//   leaf rows   -- interior rows with two nonzeros in one block (the A_mom
//                  "occurrence - canonical" rows, and similar
//                  pair rows), grouped by shared columns into groups of <= 4;
//                  their Gram block K_LL is block diagonal;
//   R_k         -- the remaining rows touching only stage k;
//   S_j         -- separator rows touching stages j and j+1 (A_sen).
// Block elimination K = [K_LL K_LQ; K_QL K_QQ]: K' = K_QQ - K_QL K_LL^{-1} K_LQ keeps
// the chain pattern; K'_RR is block diagonal by stage (dense L_k, explicit L_k^{-1});
// the separator Schur complement T = K'_SS - sum F_k^T F_k is factored densely.
// Identical stage blocks (time-invariant dynamics) share one factor.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <unordered_map>

#include "host.h"

namespace strom {

static const int kLeafGroupMax = 4;

strom_status build_sdp(Sdp &s, int32_t nblocks, const strom_block *blocks, int32_t m,
                       const double *b) {
  if (nblocks <= 0 || m <= 0 || !blocks || !b) {
    set_error("strom_sdp_create: nblocks, m must be > 0 and pointers non-NULL");
    return STROM_EINVAL;
  }
  s.nblocks = nblocks; s.m = m;
  s.bn.resize(nblocks); s.bstage.resize(nblocks); s.boff.assign(nblocks + 1, 0);
  int prev_stage = 0;
  for (int k = 0; k < nblocks; ++k) {
    const strom_block &B = blocks[k];
    if (B.n <= 0 || B.nrows < 0 || B.stage < 0 || (B.nrows > 0 && (!B.rows || !B.rowptr))) {
      set_error("strom_sdp_create: block " + std::to_string(k) + " has invalid n/nrows/stage");
      return STROM_EINVAL;
    }
    if (B.stage < prev_stage || B.stage > prev_stage + 1) {
      set_error("strom_sdp_create: block stages must be non-decreasing and contiguous from 0");
      return STROM_EINVAL;
    }
    if (k == 0 && B.stage != 0) {
      set_error("strom_sdp_create: first block must have stage 0");
      return STROM_EINVAL;
    }
    prev_stage = B.stage;
    s.bn[k] = B.n; s.bstage[k] = B.stage;
    s.boff[k + 1] = s.boff[k] + (int64_t)B.n * (B.n + 1) / 2;
  }
  s.nstages = prev_stage + 1;
  s.n = s.boff[nblocks];
  if (s.n >= (int64_t)INT32_MAX) { set_error("strom_sdp_create: n too large for int32 columns"); return STROM_EINVAL; }
  // count entries per global row
  std::vector<int64_t> cnt(m + 1, 0);
  for (int k = 0; k < nblocks; ++k) {
    const strom_block &B = blocks[k];
    if (B.nrows == 0) continue;
    if (B.rowptr[0] != 0) { set_error("strom_sdp_create: rowptr[0] != 0"); return STROM_EINVAL; }
    const int64_t L = (int64_t)B.n * (B.n + 1) / 2;
    for (int i = 0; i < B.nrows; ++i) {
      const int r = B.rows[i];
      if (r < 0 || r >= m || (i > 0 && r <= B.rows[i - 1])) {
        set_error("strom_sdp_create: block " + std::to_string(k) + " rows must be strictly ascending in [0,m)");
        return STROM_EINVAL;
      }
      const int64_t a = B.rowptr[i], e = B.rowptr[i + 1];
      if (e < a) { set_error("strom_sdp_create: rowptr not monotone"); return STROM_EINVAL; }
      for (int64_t t = a; t < e; ++t)
        if (B.col[t] < 0 || B.col[t] >= L) {
          set_error("strom_sdp_create: block " + std::to_string(k) + " col out of range");
          return STROM_EINVAL;
        }
      cnt[r + 1] += e - a;
    }
  }
  s.rowptr.assign(m + 1, 0);
  for (int i = 0; i < m; ++i) s.rowptr[i + 1] = s.rowptr[i] + cnt[i + 1];
  const int64_t nnz = s.rowptr[m];
  s.col.resize(nnz); s.val.resize(nnz);
  std::vector<int64_t> fill(s.rowptr.begin(), s.rowptr.end() - 1);
  for (int k = 0; k < nblocks; ++k) {  // blocks ascend in svec offset -> columns ascend
    const strom_block &B = blocks[k];
    for (int i = 0; i < B.nrows; ++i) {
      const int r = B.rows[i];
      for (int64_t t = B.rowptr[i]; t < B.rowptr[i + 1]; ++t) {
        s.col[fill[r]] = (int32_t)(s.boff[k] + B.col[t]);
        s.val[fill[r]] = B.val[t];
        ++fill[r];
      }
    }
  }
  // sort columns within each row (blocks were processed in order; within a
  // block the caller's order is kept -> sort to be safe)
  for (int i = 0; i < m; ++i) {
    const int64_t a = s.rowptr[i], e = s.rowptr[i + 1];
    bool sorted = true;
    for (int64_t t = a + 1; t < e; ++t) if (s.col[t] <= s.col[t - 1]) { sorted = false; break; }
    if (!sorted) {
      std::vector<std::pair<int32_t, double>> tmp;
      for (int64_t t = a; t < e; ++t) tmp.push_back({s.col[t], s.val[t]});
      std::sort(tmp.begin(), tmp.end(), [](auto &x, auto &y) { return x.first < y.first; });
      for (int64_t t = a; t < e; ++t) {
        if (t > a && tmp[t - a].first == tmp[t - a - 1].first) {
          set_error("strom_sdp_create: duplicate column in a row"); return STROM_EINVAL;
        }
        s.col[t] = tmp[t - a].first; s.val[t] = tmp[t - a].second;
      }
    }
  }
  s.b.assign(b, b + m);
  s.C.assign(s.n, 0.0);
  for (int k = 0; k < nblocks; ++k)
    if (blocks[k].C_svec)
      std::memcpy(s.C.data() + s.boff[k], blocks[k].C_svec,
                  sizeof(double) * (size_t)(s.boff[k + 1] - s.boff[k]));
  // chain check: a row may touch at most two adjacent stages
  std::vector<int32_t> col_stage(s.n);
  for (int k = 0; k < nblocks; ++k)
    for (int64_t c = s.boff[k]; c < s.boff[k + 1]; ++c) col_stage[c] = s.bstage[k];
  for (int i = 0; i < m; ++i) {
    if (s.rowptr[i + 1] == s.rowptr[i]) { set_error("strom_sdp_create: empty row " + std::to_string(i)); return STROM_EINVAL; }
    int lo = INT32_MAX, hi = -1;
    for (int64_t t = s.rowptr[i]; t < s.rowptr[i + 1]; ++t) {
      lo = std::min(lo, col_stage[s.col[t]]); hi = std::max(hi, col_stage[s.col[t]]);
    }
    if (hi - lo > 1) {
      set_error("strom_sdp_create: row " + std::to_string(i) + " touches non-adjacent stages (not a chain)");
      return STROM_EINVAL;
    }
  }
  return STROM_OK;
}

namespace {

struct UF {
  std::vector<int32_t> p;
  explicit UF(size_t n) : p(n) { std::iota(p.begin(), p.end(), 0); }
  int32_t find(int32_t x) { while (p[x] != x) { p[x] = p[p[x]]; x = p[x]; } return x; }
  void unite(int32_t a, int32_t b) { a = find(a); b = find(b); if (a != b) p[a] = b; }
};

// K = AA* (without eps), symmetric CSR in ORIGINAL row numbering.
void build_AAt(const Sdp &s, std::vector<int64_t> &Kp, std::vector<int32_t> &Ki,
               std::vector<double> &Kv) {
  const int m = s.m;
  // A^T structure
  std::vector<int64_t> cp(s.n + 1, 0);
  for (int64_t t = 0; t < (int64_t)s.col.size(); ++t) cp[s.col[t] + 1]++;
  for (int64_t c = 0; c < s.n; ++c) cp[c + 1] += cp[c];
  std::vector<int32_t> cr(s.col.size());
  std::vector<double> cv(s.col.size());
  {
    std::vector<int64_t> f(cp.begin(), cp.end() - 1);
    for (int i = 0; i < m; ++i)
      for (int64_t t = s.rowptr[i]; t < s.rowptr[i + 1]; ++t) {
        cr[f[s.col[t]]] = i; cv[f[s.col[t]]] = s.val[t]; f[s.col[t]]++;
      }
  }
  std::vector<std::vector<int32_t>> rows_i(m);
  std::vector<std::vector<double>> rows_v(m);
#pragma omp parallel
  {
    std::vector<double> acc(m, 0.0);
    std::vector<char> mark(m, 0);
    std::vector<int32_t> list;
#pragma omp for schedule(dynamic, 64)
    for (int i = 0; i < m; ++i) {
      list.clear();
      for (int64_t t = s.rowptr[i]; t < s.rowptr[i + 1]; ++t) {
        const int32_t c = s.col[t];
        const double a = s.val[t];
        for (int64_t u = cp[c]; u < cp[c + 1]; ++u) {
          const int32_t j = cr[u];
          if (!mark[j]) { mark[j] = 1; list.push_back(j); acc[j] = 0.0; }
          acc[j] += a * cv[u];
        }
      }
      std::sort(list.begin(), list.end());
      rows_i[i] = list;
      rows_v[i].resize(list.size());
      for (size_t q = 0; q < list.size(); ++q) { rows_v[i][q] = acc[list[q]]; mark[list[q]] = 0; }
    }
  }
  Kp.assign(m + 1, 0);
  for (int i = 0; i < m; ++i) Kp[i + 1] = Kp[i] + rows_i[i].size();
  Ki.resize(Kp[m]); Kv.resize(Kp[m]);
  for (int i = 0; i < m; ++i) {
    std::copy(rows_i[i].begin(), rows_i[i].end(), Ki.begin() + Kp[i]);
    std::copy(rows_v[i].begin(), rows_v[i].end(), Kv.begin() + Kp[i]);
  }
}

uint64_t fnv(const void *p, size_t n, uint64_t h = 1469598103934665603ULL) {
  const unsigned char *c = (const unsigned char *)p;
  for (size_t i = 0; i < n; ++i) { h ^= c[i]; h *= 1099511628211ULL; }
  return h;
}

bool small_chol_inv(int g, const double *K, double *Kinv, double rel_floor) {
  // Cholesky of g x g SPD, then full inverse; refuse ill-conditioned groups.
  double L[kLeafGroupMax * kLeafGroupMax] = {0};
  double dmax = 0.0;
  for (int i = 0; i < g; ++i) dmax = std::max(dmax, K[i * g + i]);
  for (int j = 0; j < g; ++j) {
    double d = K[j * g + j];
    for (int k = 0; k < j; ++k) d -= L[j * g + k] * L[j * g + k];
    if (!(d > rel_floor * dmax)) return false;
    L[j * g + j] = std::sqrt(d);
    for (int i = j + 1; i < g; ++i) {
      double s2 = K[i * g + j];
      for (int k = 0; k < j; ++k) s2 -= L[i * g + k] * L[j * g + k];
      L[i * g + j] = s2 / L[j * g + j];
    }
  }
  // inverse via L^{-T} L^{-1} columns
  for (int c = 0; c < g; ++c) {
    double x[kLeafGroupMax];
    for (int i = 0; i < g; ++i) {
      double s2 = (i == c) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) s2 -= L[i * g + k] * x[k];
      x[i] = s2 / L[i * g + i];
    }
    for (int i = g - 1; i >= 0; --i) {
      double s2 = x[i];
      for (int k = i + 1; k < g; ++k) s2 -= L[k * g + i] * x[k];
      x[i] = s2 / L[i * g + i];
    }
    for (int i = 0; i < g; ++i) Kinv[i * g + c] = x[i];
  }
  return true;
}

}  // namespace

// STROM_PROF_SETUP=1: wall time of the build_factor phases on stderr
static std::chrono::steady_clock::time_point g_prof_t;
static void prof_lap(int phase) {
  static const bool on = getenv("STROM_PROF_SETUP") != nullptr;
  if (!on) return;
  const auto now = std::chrono::steady_clock::now();
  if (phase > 0)
    fprintf(stderr, "[strom setup] phase %d: %.1f ms\n", phase - 1,
            std::chrono::duration<double, std::milli>(now - g_prof_t).count());
  g_prof_t = now;
}

strom_status build_factor(const Sdp &s, double eps_rel, double eps_abs, Factor &f) {
  prof_lap(0);
  const int m = s.m;
  const int P = s.nstages;
  f.m = m; f.P = P;
  // ---- classify rows ------------------------------------------------------
  std::vector<int32_t> col_block(s.n);
  for (int k = 0; k < s.nblocks; ++k)
    for (int64_t c = s.boff[k]; c < s.boff[k + 1]; ++c) col_block[c] = k;
  std::vector<int32_t> owner(m);
  std::vector<char> is_sep(m, 0), leaf_cand(m, 0);
  for (int i = 0; i < m; ++i) {
    int lo = INT32_MAX, hi = -1;
    for (int64_t t = s.rowptr[i]; t < s.rowptr[i + 1]; ++t) {
      const int st = s.bstage[col_block[s.col[t]]];
      lo = std::min(lo, st); hi = std::max(hi, st);
    }
    owner[i] = lo;
    is_sep[i] = (hi == lo + 1);
  }
  // A leaf candidate is a two-term row inside one block that owns a private column
  // (referenced by no other row) -- the non-canonical occurrence of an A_mom row
  // (PAPER.md:344). Groups then form only through the shared canonical column.
  std::vector<int32_t> col_count(s.n, 0);
  for (int64_t t = 0; t < (int64_t)s.col.size(); ++t) col_count[s.col[t]]++;
  for (int i = 0; i < m; ++i) {
    const int64_t a = s.rowptr[i];
    if (!is_sep[i] && s.rowptr[i + 1] - a == 2 && col_block[s.col[a]] == col_block[s.col[a + 1]] &&
        (col_count[s.col[a]] == 1 || col_count[s.col[a + 1]] == 1))
      leaf_cand[i] = 1;
  }
  prof_lap(0);
  // ---- K = AA* + eps I ----------------------------------------------------
  std::vector<int64_t> Kp; std::vector<int32_t> Ki; std::vector<double> Kv;
  build_AAt(s, Kp, Ki, Kv);
  double dmax = 0.0;
  for (int i = 0; i < m; ++i)
    for (int64_t t = Kp[i]; t < Kp[i + 1]; ++t)
      if (Ki[t] == i) dmax = std::max(dmax, Kv[t]);
  f.eps = eps_abs > 0.0 ? eps_abs : eps_rel * dmax;
  if (!(f.eps > 0.0)) { set_error("strom_admm_setup: eps must be > 0"); return STROM_EINVAL; }
  for (int i = 0; i < m; ++i)
    for (int64_t t = Kp[i]; t < Kp[i + 1]; ++t)
      if (Ki[t] == i) Kv[t] += f.eps;
  auto Kget = [&](int i, int j) -> double {
    const int32_t *b0 = Ki.data() + Kp[i], *e0 = Ki.data() + Kp[i + 1];
    const int32_t *p = std::lower_bound(b0, e0, j);
    return (p != e0 && *p == j) ? Kv[p - Ki.data()] : 0.0;
  };
  prof_lap(1);
  // ---- leaf groups --------------------------------------------------------
  UF uf(s.n);
  for (int i = 0; i < m; ++i)
    if (leaf_cand[i]) uf.unite(s.col[s.rowptr[i]], s.col[s.rowptr[i] + 1]);
  std::unordered_map<int32_t, std::vector<int32_t>> groups;
  std::vector<int32_t> group_order;
  for (int i = 0; i < m; ++i)
    if (leaf_cand[i]) {
      const int32_t root = uf.find(s.col[s.rowptr[i]]);
      auto it = groups.find(root);
      if (it == groups.end()) { groups[root] = {i}; group_order.push_back(root); }
      else it->second.push_back(i);
    }
  // groups in stage order (a leaf row lies in one block, so in one stage): the leaf rows
  // of a contiguous stage range are contiguous, as the horizon partition needs
  std::stable_sort(group_order.begin(), group_order.end(), [&](int32_t x, int32_t y) {
    return owner[groups[x][0]] < owner[groups[y][0]];
  });
  std::vector<std::vector<int32_t>> leaf_groups;
  std::vector<std::vector<double>> leaf_kinv;
  std::vector<char> is_leaf(m, 0);
  for (int32_t root : group_order) {
    const auto &g = groups[root];
    const int gs = (int)g.size();
    if (gs > kLeafGroupMax) continue;
    std::vector<double> Kg(gs * gs), Kinv(gs * gs);
    for (int a = 0; a < gs; ++a)
      for (int c = 0; c < gs; ++c) Kg[a * gs + c] = Kget(g[a], g[c]);
    if (!small_chol_inv(gs, Kg.data(), Kinv.data(), 1e-8)) continue;  // ill-conditioned -> stays in R
    for (int r : g) is_leaf[r] = 1;
    leaf_groups.push_back(g);
    leaf_kinv.push_back(Kinv);
  }
  prof_lap(2);
  // ---- internal order ------------------------------------------------------
  f.perm.clear(); f.perm.reserve(m);
  f.gptr.assign(1, 0); f.goff.assign(1, 0); f.gKinv.clear();
  for (size_t q = 0; q < leaf_groups.size(); ++q) {
    for (int r : leaf_groups[q]) f.perm.push_back(r);
    f.gptr.push_back((int32_t)f.perm.size());
    f.gKinv.insert(f.gKinv.end(), leaf_kinv[q].begin(), leaf_kinv[q].end());
    f.goff.push_back((int64_t)f.gKinv.size());
  }
  f.nL = (int32_t)f.perm.size();
  f.L_off.assign(P + 1, f.nL);
  for (int l = f.nL - 1; l >= 0; --l) f.L_off[owner[f.perm[l]]] = l;
  for (int k = P - 1; k >= 0; --k) f.L_off[k] = std::min(f.L_off[k], f.L_off[k + 1]);
  f.R_off.assign(P + 1, 0);
  std::vector<std::vector<int32_t>> Rrows(P), Srows(std::max(P - 1, 0));
  for (int i = 0; i < m; ++i) {
    if (is_leaf[i]) continue;
    if (is_sep[i]) Srows[owner[i]].push_back(i); else Rrows[owner[i]].push_back(i);
  }
  for (int k = 0; k < P; ++k) {
    f.R_off[k] = (int32_t)f.perm.size();
    f.perm.insert(f.perm.end(), Rrows[k].begin(), Rrows[k].end());
  }
  f.R_off[P] = (int32_t)f.perm.size();
  f.S_off.assign(P, 0);
  for (int j = 0; j + 1 < P; ++j) {
    f.S_off[j] = (int32_t)f.perm.size();
    f.perm.insert(f.perm.end(), Srows[j].begin(), Srows[j].end());
  }
  if (P >= 1) f.S_off[P - 1] = (int32_t)f.perm.size();
  f.iperm.assign(m, -1);
  for (int i = 0; i < m; ++i) f.iperm[f.perm[i]] = i;
  const int nL = f.nL, nQ = m - nL;
  std::vector<int32_t> leaf_group_of(nL);
  for (size_t q = 0; q + 1 < f.gptr.size(); ++q)
    for (int r = f.gptr[q]; r < f.gptr[q + 1]; ++r) leaf_group_of[r] = (int32_t)q;
  prof_lap(3);
  // ---- G = K_QL K_LL^{-1} (CSR by Q row, leaf internal columns) -----------
  std::vector<std::vector<int32_t>> Gi(nQ);
  std::vector<std::vector<double>> Gv(nQ);
#pragma omp parallel for schedule(dynamic, 64)
  for (int qi = 0; qi < nQ; ++qi) {
    const int orow = f.perm[nL + qi];
    // leaf neighbours grouped by leaf group
    std::vector<std::pair<int32_t, double>> nb;  // (leaf internal idx, K value)
    for (int64_t t = Kp[orow]; t < Kp[orow + 1]; ++t) {
      const int li = f.iperm[Ki[t]];
      if (li < nL) nb.push_back({li, Kv[t]});
    }
    std::sort(nb.begin(), nb.end());
    size_t p = 0;
    while (p < nb.size()) {
      const int g = leaf_group_of[nb[p].first];
      const int g0 = f.gptr[g], gs = f.gptr[g + 1] - g0;
      double kq[kLeafGroupMax] = {0};
      while (p < nb.size() && leaf_group_of[nb[p].first] == g) { kq[nb[p].first - g0] = nb[p].second; ++p; }
      const double *Kinv = f.gKinv.data() + f.goff[g];
      for (int c = 0; c < gs; ++c) {
        double v = 0.0;
        for (int a = 0; a < gs; ++a) v += kq[a] * Kinv[a * gs + c];
        if (v != 0.0) { Gi[qi].push_back(g0 + c); Gv[qi].push_back(v); }
      }
    }
  }
  f.G_ptr.assign(nQ + 1, 0);
  for (int qi = 0; qi < nQ; ++qi) f.G_ptr[qi + 1] = f.G_ptr[qi] + Gi[qi].size();
  f.G_col.resize(f.G_ptr[nQ]); f.G_val.resize(f.G_ptr[nQ]);
  for (int qi = 0; qi < nQ; ++qi) {
    std::copy(Gi[qi].begin(), Gi[qi].end(), f.G_col.begin() + f.G_ptr[qi]);
    std::copy(Gv[qi].begin(), Gv[qi].end(), f.G_val.begin() + f.G_ptr[qi]);
  }
  // G^T by leaf row, columns = absolute internal Q index
  f.Gt_ptr.assign(nL + 1, 0);
  for (int64_t t = 0; t < f.G_ptr[nQ]; ++t) f.Gt_ptr[f.G_col[t] + 1]++;
  for (int l = 0; l < nL; ++l) f.Gt_ptr[l + 1] += f.Gt_ptr[l];
  f.Gt_col.resize(f.G_ptr[nQ]); f.Gt_val.resize(f.G_ptr[nQ]);
  {
    std::vector<int64_t> fl(f.Gt_ptr.begin(), f.Gt_ptr.end() - 1);
    for (int qi = 0; qi < nQ; ++qi)
      for (int64_t t = f.G_ptr[qi]; t < f.G_ptr[qi + 1]; ++t) {
        const int l = f.G_col[t];
        f.Gt_col[fl[l]] = nL + qi; f.Gt_val[fl[l]] = f.G_val[t]; fl[l]++;
      }
  }
  prof_lap(4);
  // ---- K' = K_QQ - G K_LQ, rows restricted to Q (sparse, internal Q index) ---
  std::vector<std::vector<int32_t>> KPi(nQ);
  std::vector<std::vector<double>> KPv(nQ);
#pragma omp parallel
  {
    std::vector<double> acc(nQ, 0.0);
    std::vector<char> mark(nQ, 0);
    std::vector<int32_t> list;
#pragma omp for schedule(dynamic, 64)
    for (int qi = 0; qi < nQ; ++qi) {
      list.clear();
      auto add = [&](int qj, double v) {
        if (!mark[qj]) { mark[qj] = 1; acc[qj] = 0.0; list.push_back(qj); }
        acc[qj] += v;
      };
      const int orow = f.perm[nL + qi];
      for (int64_t t = Kp[orow]; t < Kp[orow + 1]; ++t) {
        const int ii = f.iperm[Ki[t]];
        if (ii >= nL) add(ii - nL, Kv[t]);
      }
      for (int64_t t = f.G_ptr[qi]; t < f.G_ptr[qi + 1]; ++t) {
        const int l = f.G_col[t];
        const double gv = f.G_val[t];
        const int lrow = f.perm[l];
        for (int64_t u = Kp[lrow]; u < Kp[lrow + 1]; ++u) {
          const int ii = f.iperm[Ki[u]];
          if (ii >= nL) add(ii - nL, -gv * Kv[u]);
        }
      }
      std::sort(list.begin(), list.end());
      KPi[qi] = list;
      KPv[qi].resize(list.size());
      for (size_t q = 0; q < list.size(); ++q) { KPv[qi][q] = acc[list[q]]; mark[list[q]] = 0; }
    }
  }
  prof_lap(5);
  // ---- per-stage dense factors with dedup ------------------------------------
  const int S0 = f.R_off[P];
  const int nS = m - S0;
  f.stage_uid.assign(P, -1); f.stage_wl.assign(P, 0); f.stage_wr.assign(P, 0);
  // Dedup on the sparse rows of K'_{R_k R_k} and K'_{R_k, [S_{k-1} S_k]} (the dense blocks
  // are built only for unique stages: time-invariant chains have a handful)
  struct Sig { int nk, wl, wr; std::vector<int32_t> ij; std::vector<double> v; uint64_t h; };
  std::vector<Sig> uid_sig;
  std::vector<std::vector<int32_t>> stage_cmap(P);
  for (int k = 0; k < P; ++k) {
    const int r0 = f.R_off[k], nk = f.R_off[k + 1] - r0;
    const int wl = (k >= 1) ? f.S_off[k] - f.S_off[k - 1] : 0;
    const int wr = (k + 1 < P) ? f.S_off[k + 1] - f.S_off[k] : 0;
    f.stage_wl[k] = wl; f.stage_wr[k] = wr;
    std::vector<int32_t> &cmap = stage_cmap[k];  // F column -> position in T (0-based in S)
    for (int c = 0; c < wl; ++c) cmap.push_back(f.S_off[k - 1] - S0 + c);
    for (int c = 0; c < wr; ++c) cmap.push_back(f.S_off[k] - S0 + c);
    Sig sg{nk, wl, wr, {}, {}, 0};
    for (int i = 0; i < nk; ++i) {               // (row, column code) with code < nk interior,
      const int qi = r0 + i - nL;                // nk + c the separator column c of [S_{k-1} S_k]
      for (size_t t = 0; t < KPi[qi].size(); ++t) {
        const int qj = KPi[qi][t] + nL;  // absolute internal
        int code;
        if (qj >= r0 && qj < r0 + nk) code = qj - r0;
        else if (wl && qj >= f.S_off[k - 1] && qj < f.S_off[k]) code = nk + qj - f.S_off[k - 1];
        else if (wr && qj >= f.S_off[k] && qj < f.S_off[k + 1]) code = nk + wl + qj - f.S_off[k];
        else if (qj < S0) {
          set_error("strom_admm_setup: interior rows of different stages coupled (not a chain)");
          return STROM_EINVAL;
        } else continue;
        sg.ij.push_back(i); sg.ij.push_back(code); sg.v.push_back(KPv[qi][t]);
      }
    }
    sg.h = fnv(sg.ij.data(), sg.ij.size() * 4, fnv(sg.v.data(), sg.v.size() * 8) ^ (uint64_t)(nk * 7919 + wl * 1000003 + wr));
    int found = -1;
    for (size_t u = 0; u < uid_sig.size(); ++u) {
      const Sig &o = uid_sig[u];
      if (o.h == sg.h && o.nk == nk && o.wl == wl && o.wr == wr && o.ij == sg.ij &&
          std::memcmp(o.v.data(), sg.v.data(), sg.v.size() * 8) == 0 && o.v.size() == sg.v.size()) {
        found = (int)u; break;
      }
    }
    if (found >= 0) { f.stage_uid[k] = found; continue; }
    Dense Kd; Kd.rows = Kd.cols = nk; Kd.a.assign((size_t)nk * nk, 0.0);
    Dense Bd; Bd.rows = nk; Bd.cols = wl + wr; Bd.a.assign((size_t)nk * (wl + wr), 0.0);
    for (size_t t = 0; t < sg.v.size(); ++t) {
      const int i = sg.ij[2 * t], code = sg.ij[2 * t + 1];
      if (code < nk) Kd.row(i)[code] = sg.v[t];
      else Bd.row(i)[code - nk] = sg.v[t];
    }
    f.stage_uid[k] = (int)f.uK.size();
    f.uK.push_back(std::move(Kd)); f.uB.push_back(std::move(Bd));
    uid_sig.push_back(std::move(sg));
  }
  f.stage_cmap = stage_cmap;
  prof_lap(6);
  // ---- separator block K'_SS (its Schur complement T is formed by the backend) -----
  f.T0.rows = f.T0.cols = nS; f.T0.a.assign((size_t)nS * nS, 0.0);
  for (int si = 0; si < nS; ++si) {
    const int qi = S0 + si - nL;
    for (size_t t = 0; t < KPi[qi].size(); ++t) {
      const int qj = KPi[qi][t] + nL;
      if (qj >= S0) f.T0.row(si)[qj - S0] = KPv[qi][t];
    }
  }
  prof_lap(8);
  if (getenv("STROM_VERBOSE")) {
    fprintf(stderr, "[strom] m=%d leaf=%d R=%d S=%d stages=%d unique dense=%zu:", m, nL, S0 - nL, nS, P,
            f.uK.size());
    for (size_t u = 0; u < f.uK.size(); ++u) {
      int cnt = 0;
      for (int k = 0; k < P; ++k) cnt += (f.stage_uid[k] == (int)u);
      fprintf(stderr, " [n=%d w=%d x%d]", f.uK[u].rows, f.uB[u].cols, cnt);
    }
    int64_t gmax = 0, gtmax = 0, amax = 0;
    for (int qi = 0; qi < nQ; ++qi) gmax = std::max<int64_t>(gmax, f.G_ptr[qi + 1] - f.G_ptr[qi]);
    for (int l = 0; l < nL; ++l) gtmax = std::max<int64_t>(gtmax, f.Gt_ptr[l + 1] - f.Gt_ptr[l]);
    for (int i = 0; i < m; ++i) amax = std::max<int64_t>(amax, s.rowptr[i + 1] - s.rowptr[i]);
    fprintf(stderr, "\n[strom] G nnz %lld (max/row %lld, mean %.2f), G^T max/row %lld, A max/row %lld\n",
            (long long)f.G_ptr[nQ], (long long)gmax, nQ ? (double)f.G_ptr[nQ] / nQ : 0.0, (long long)gtmax,
            (long long)amax);
  }
  return STROM_OK;
}

// Host backend of the dense factorisation (tests and small problems):
// L_u = chol(K'_u), L_u^{-1}, F_u = L_u^{-1} B_u; T = K'_SS - sum F^T F, L_T^{-1}.
strom_status host_factor_dense(Factor &f) {
  f.Linv.clear(); f.F.clear();
  for (size_t u = 0; u < f.uK.size(); ++u) {
    Dense L = f.uK[u];
    if (L.rows > 0 && !dense_cholesky_lower(L)) {
      set_error("strom_admm_setup: non-positive pivot in a stage interior block");
      return STROM_EFACTOR;
    }
    Dense Li; dense_trinv_lower(L, Li);
    Dense Fk; dense_gemm_lowertri(Li, f.uB[u], Fk);
    f.Linv.push_back(std::move(Li));
    f.F.push_back(std::move(Fk));
  }
  Dense T = f.T0;
  for (int k = 0; k < f.P; ++k)
    if (!f.stage_cmap[k].empty() && f.R_off[k + 1] > f.R_off[k])
      dense_sub_AtA(T, f.F[f.stage_uid[k]], f.stage_cmap[k]);
  if (T.rows > 0) {
    if (!dense_cholesky_lower(T)) {
      set_error("strom_admm_setup: non-positive pivot in the separator Schur complement");
      return STROM_EFACTOR;
    }
    dense_trinv_lower(T, f.LTinv);
  }
  return STROM_OK;
}

// Reference execution of the factored solve on the host (test hook). Same
// phases as the device, in the same order.
void host_solve(const Factor &f, const double *r_orig, double *y_orig) {
  const int m = f.m, nL = f.nL, P = f.P;
  std::vector<double> r(m), u(m), y(m, 0.0);
  for (int i = 0; i < m; ++i) r[i] = r_orig[f.perm[i]];
  // P1: u_Q = r_Q - G r_L
  for (int qi = 0; qi < m - nL; ++qi) {
    double s = r[nL + qi];
    for (int64_t t = f.G_ptr[qi]; t < f.G_ptr[qi + 1]; ++t) s -= f.G_val[t] * r[f.G_col[t]];
    u[nL + qi] = s;
  }
  // P2: v_k = L_k^{-1} u_Rk
  std::vector<double> v(m, 0.0);
  for (int k = 0; k < P; ++k) {
    const Dense &Li = f.Linv[f.stage_uid[k]];
    const int r0 = f.R_off[k];
    for (int i = 0; i < Li.rows; ++i) {
      double s = 0.0;
      for (int j = 0; j <= i; ++j) s += Li.row(i)[j] * u[r0 + j];
      v[r0 + i] = s;
    }
  }
  // P3: u_S' = u_S - sum_k F_k^T v_k
  const int S0 = f.R_off[P], nS = m - S0;
  std::vector<double> us(nS);
  for (int si = 0; si < nS; ++si) us[si] = u[S0 + si];
  for (int k = 0; k < P; ++k) {
    const Dense &F = f.F[f.stage_uid[k]];
    const int r0 = f.R_off[k], wl = f.stage_wl[k];
    for (int c = 0; c < F.cols; ++c) {
      const int si = (c < wl) ? f.S_off[k - 1] - S0 + c : f.S_off[k] - S0 + (c - wl);
      double s = 0.0;
      for (int i = 0; i < F.rows; ++i) s += F.row(i)[c] * v[r0 + i];
      us[si] -= s;
    }
  }
  // P4, P5: y_S = L_T^{-T} L_T^{-1} u_S'
  std::vector<double> z(nS, 0.0), ys(nS, 0.0);
  for (int i = 0; i < nS; ++i) {
    double s = 0.0;
    for (int j = 0; j <= i; ++j) s += f.LTinv.row(i)[j] * us[j];
    z[i] = s;
  }
  for (int i = 0; i < nS; ++i) {
    double s = 0.0;
    for (int j = i; j < nS; ++j) s += f.LTinv.row(j)[i] * z[j];
    ys[i] = s;
  }
  for (int si = 0; si < nS; ++si) y[S0 + si] = ys[si];
  // P6: y_Rk = L_k^{-T} (v_k - F_k y_S,adj)
  for (int k = 0; k < P; ++k) {
    const Dense &Li = f.Linv[f.stage_uid[k]];
    const Dense &F = f.F[f.stage_uid[k]];
    const int r0 = f.R_off[k], nk = Li.rows, wl = f.stage_wl[k];
    std::vector<double> t(nk);
    for (int i = 0; i < nk; ++i) {
      double s = v[r0 + i];
      for (int c = 0; c < F.cols; ++c) {
        const int si = (c < wl) ? f.S_off[k - 1] - S0 + c : f.S_off[k] - S0 + (c - wl);
        s -= F.row(i)[c] * ys[si];
      }
      t[i] = s;
    }
    for (int i = 0; i < nk; ++i) {
      double s = 0.0;
      for (int j = i; j < nk; ++j) s += Li.row(j)[i] * t[j];
      y[r0 + i] = s;
    }
  }
  // P7: y_L = K_LL^{-1} r_L - G^T y_Q
  for (size_t g = 0; g + 1 < f.gptr.size(); ++g) {
    const int g0 = f.gptr[g], gs = f.gptr[g + 1] - g0;
    const double *Kinv = f.gKinv.data() + f.goff[g];
    for (int a = 0; a < gs; ++a) {
      double s = 0.0;
      for (int c = 0; c < gs; ++c) s += Kinv[a * gs + c] * r[g0 + c];
      const int l = g0 + a;
      for (int64_t t = f.Gt_ptr[l]; t < f.Gt_ptr[l + 1]; ++t) s -= f.Gt_val[t] * y[f.Gt_col[t]];
      y[l] = s;
    }
  }
  for (int i = 0; i < m; ++i) y_orig[f.perm[i]] = y[i];
}

}  // namespace strom
