// Fast relaxation generator (NEXT-3; the paper's STROM converter is C++,
// PAPER.md:81, 1082-1099): the kappa-th order sparse moment relaxation of a chain POP as
// the standard multi-block SDP, the same rows in the same order with
// the same floating-point operations as strom_inputs.relax.compile_relaxation (the Python
// reference, which the tests compare byte for byte). Input side of the build: holds none
// of the sGS-ADMM arithmetic. Cliques are processed in parallel (OpenMP).
//
// Row families per clique k: norm M_1(1,1) = 1; mom occurrence -
// canonical = 0 (A_mom); ineq L(r,c) - sum_a g_a M(canon(a + B_r + B_c)) = 0;
// eq sum_a h_a M(canon(a + mu)) = 0 for mu in [z]_{2 kappa - deg h}; sen canon_k(m) -
// canon_{k+1}(m) = 0 for the monomials of the shared variables. svec SDPT3 (Q4),
// canonical = first occurrence in svec order (Q5).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <unordered_map>
#include <vector>

#include <omp.h>
#include <sched.h>

#include "../../include/strom_gen.h"

namespace {

// threads: the CPUs this process may run on (the default team size can be the host's full
// core count inside a container, which oversubscribes the few allowed cores badly)
int gen_threads(int work) {
  cpu_set_t set;
  int ncpu = 1;
  if (sched_getaffinity(0, sizeof(set), &set) == 0) ncpu = CPU_COUNT(&set);
  return std::max(1, std::min({ncpu, omp_get_max_threads(), work}));
}

constexpr int kBits = 3;                  // exponent <= 7 per variable, <= 21 variables
using Key = uint64_t;

inline Key key_of(const uint8_t *e, int nv) {
  Key k = 0;
  for (int i = 0; i < nv; ++i) k |= (Key)e[i] << (kBits * i);
  return k;
}

// [z]_deg over nv ordered variables, graded lex (degree major, then the lexicographic order
// of sorted index tuples: itertools.combinations_with_replacement), as exponent keys
void basis(int nv, int deg, std::vector<Key> &out) {
  out.clear();
  std::vector<int> idx;
  for (int d = 0; d <= deg; ++d) {
    idx.assign(d, 0);
    while (true) {
      Key k = 0;
      for (int v : idx) k += (Key)1 << (kBits * v);
      out.push_back(k);
      int p = d - 1;                     // next non-decreasing tuple
      while (p >= 0 && idx[p] == nv - 1) --p;
      if (p < 0) break;
      const int val = idx[p] + 1;
      for (int q = p; q < d; ++q) idx[q] = val;
    }
  }
}

int degree_of(Key k, int nv) {
  int d = 0;
  for (int i = 0; i < nv; ++i) d += (int)((k >> (kBits * i)) & 7u);
  return d;
}

struct Poly { std::vector<Key> mono; std::vector<double> coef; int deg = 0; };

struct Table {                              // per clique monomial bookkeeping
  int nv = 0, nM = 0;
  std::vector<Key> B;
  std::unordered_map<Key, int> canon;       // monomial -> first svec position
  std::vector<std::vector<int>> occ;        // occurrences per canonical monomial, in svec order
  std::vector<int> occ_order;               // canonical monomials in order of first occurrence
  std::vector<double> ec;                   // entry coefficient per svec position (1 or 1/sqrt2)
};

inline int svec_index(int r, int c) { return c * (c + 1) / 2 + r; }

struct Row { std::vector<int64_t> col; std::vector<double> val; int8_t fam; double rhs; };

// accumulate entries in insertion order (the Python dict's arithmetic order), then drop
// zeros and sort by column
struct Acc {
  std::vector<int64_t> c; std::vector<double> v;
  void add(int64_t col, double x) {
    for (size_t i = 0; i < c.size(); ++i) if (c[i] == col) { v[i] += x; return; }
    c.push_back(col); v.push_back(0.0 + x);
  }
  void sub(int64_t col, double x) {
    for (size_t i = 0; i < c.size(); ++i) if (c[i] == col) { v[i] -= x; return; }
    c.push_back(col); v.push_back(0.0 - x);
  }
  bool emit(std::vector<Row> &rows, int8_t fam, double rhs = 0.0) {
    std::vector<std::pair<int64_t, double>> e;
    for (size_t i = 0; i < c.size(); ++i) if (v[i] != 0.0) e.push_back({c[i], v[i]});
    c.clear(); v.clear();
    if (e.empty()) return false;
    std::sort(e.begin(), e.end(), [](auto &a, auto &b) { return a.first < b.first; });
    Row r; r.fam = fam; r.rhs = rhs;
    for (auto &p : e) { r.col.push_back(p.first); r.val.push_back(p.second); }
    rows.push_back(std::move(r));
    return true;
  }
};

}  // namespace

struct strom_gen_result {
  std::vector<int32_t> block_n, block_stage;
  std::vector<int8_t> block_kind, row_family;
  std::vector<int64_t> block_offset, indptr;
  std::vector<int32_t> indices, row_stage;
  std::vector<double> data, b, C;
  int64_t n = 0;
};

extern "C" {

int32_t strom_gen_compile(int32_t ncliques, const strom_gen_clique *cl, int32_t kappa, strom_gen_result **out) {
  if (!out || !cl || ncliques <= 0 || kappa < 1 || kappa > 3) return -1;
  *out = nullptr;
  const int N = ncliques;
  auto read_poly = [](int nv, int nt, const uint8_t *e, const double *c) {
    Poly p;
    for (int t = 0; t < nt; ++t) {
      const Key k = key_of(e + (size_t)t * nv, nv);
      p.mono.push_back(k); p.coef.push_back(c[t]);
      p.deg = std::max(p.deg, degree_of(k, nv));
    }
    return p;
  };
  std::vector<std::vector<Poly>> g(N), h(N);
  std::vector<Poly> f(N);
  for (int k = 0; k < N; ++k) {
    const strom_gen_clique &q = cl[k];
    if (q.nvars <= 0 || q.nvars > 21) return -2;
    f[k] = read_poly(q.nvars, q.f_nterms, q.f_exp, q.f_coef);
    int64_t t0 = 0;
    for (int i = 0; i < q.ng; ++i) {
      g[k].push_back(read_poly(q.nvars, q.g_nterms[i], q.g_exp + t0 * q.nvars, q.g_coef + t0));
      t0 += q.g_nterms[i];
    }
    t0 = 0;
    for (int j = 0; j < q.nh; ++j) {
      h[k].push_back(read_poly(q.nvars, q.h_nterms[j], q.h_exp + t0 * q.nvars, q.h_coef + t0));
      t0 += q.h_nterms[j];
    }
  }
  // ---- blocks (clique-major: M_k then L_{k,i}) ----------------------------------------
  std::unique_ptr<strom_gen_result> R(new strom_gen_result);
  std::vector<int> mom_block(N);
  std::vector<std::vector<int>> loc_block(N), loc_deg(N);
  std::vector<Table> T(N);
  const int nthr = gen_threads(N);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthr)
  for (int k = 0; k < N; ++k) {
    Table &t = T[k];
    t.nv = cl[k].nvars;
    basis(t.nv, kappa, t.B);
    t.nM = (int)t.B.size();
    const int L = t.nM * (t.nM + 1) / 2;
    t.ec.assign(L, 0.0);
    std::unordered_map<Key, int> slot;       // monomial -> index in occ
    t.canon.reserve(L);
    for (int c = 0; c < t.nM; ++c)
      for (int r = 0; r <= c; ++r) {
        const int s = svec_index(r, c);
        const Key m = t.B[r] + t.B[c];
        auto it = slot.find(m);
        if (it == slot.end()) {
          slot.emplace(m, (int)t.occ.size());
          t.canon.emplace(m, s);
          t.occ.push_back({s});
          t.occ_order.push_back((int)t.occ.size() - 1);
        } else {
          t.occ[it->second].push_back(s);
        }
        t.ec[s] = (r == c) ? 1.0 : 1.0 / std::sqrt(2.0);   // relax._ISQ2
      }
  }
  const double isq2 = 1.0 / std::sqrt(2.0);
  for (int k = 0; k < N; ++k) {
    mom_block[k] = (int)R->block_n.size();
    R->block_n.push_back(T[k].nM); R->block_stage.push_back(k); R->block_kind.push_back(0);
    for (const Poly &gi : g[k]) {
      const int dg = (gi.deg + 1) / 2;
      if (dg > kappa) return -3;
      std::vector<Key> B1;
      basis(T[k].nv, kappa - dg, B1);
      loc_block[k].push_back((int)R->block_n.size());
      loc_deg[k].push_back(kappa - dg);
      R->block_n.push_back((int)B1.size()); R->block_stage.push_back(k); R->block_kind.push_back(1);
    }
  }
  const int nb = (int)R->block_n.size();
  R->block_offset.assign(nb + 1, 0);
  for (int i = 0; i < nb; ++i)
    R->block_offset[i + 1] = R->block_offset[i] + (int64_t)R->block_n[i] * (R->block_n[i] + 1) / 2;
  R->n = R->block_offset[nb];
  // ---- rows, per clique in parallel ---------------------------------------------------
  std::vector<std::vector<Row>> rows(N);
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad) num_threads(nthr)
  for (int k = 0; k < N; ++k) {
    const Table &t = T[k];
    const int64_t offM = R->block_offset[mom_block[k]];
    std::vector<Row> &rw = rows[k];
    Acc acc;
    if (k == 0) { acc.add(offM + 0, 1.0); acc.emit(rw, 0, 1.0); }
    for (int oi : t.occ_order) {                               // mom
      const auto &lst = t.occ[oi];
      const int s0 = lst[0];
      for (size_t j = 1; j < lst.size(); ++j) {
        acc.add(offM + lst[j], t.ec[lst[j]]);
        acc.add(offM + s0, -t.ec[s0]);
        acc.emit(rw, 1);
      }
    }
    for (size_t i = 0; i < g[k].size(); ++i) {                 // ineq
      const Poly &gi = g[k][i];
      const int64_t offL = R->block_offset[loc_block[k][i]];
      std::vector<Key> B1;
      basis(t.nv, loc_deg[k][i], B1);
      const int nL = (int)B1.size();
      for (int c = 0; c < nL; ++c)
        for (int r = 0; r <= c; ++r) {
          acc.add(offL + svec_index(r, c), r == c ? 1.0 : isq2);
          const Key base = B1[r] + B1[c];
          for (size_t a = 0; a < gi.mono.size(); ++a) {
            auto it = t.canon.find(gi.mono[a] + base);
            if (it == t.canon.end()) { bad |= 1; continue; }
            const int s = it->second;
            acc.sub(offM + s, gi.coef[a] * t.ec[s]);
          }
          acc.emit(rw, 2);
        }
    }
    for (const Poly &hj : h[k]) {                              // eq
      if (hj.deg > 2 * kappa) { bad |= 2; continue; }
      std::vector<Key> mus;
      basis(t.nv, 2 * kappa - hj.deg, mus);
      for (Key mu : mus) {
        for (size_t a = 0; a < hj.mono.size(); ++a) {
          auto it = t.canon.find(hj.mono[a] + mu);
          if (it == t.canon.end()) { bad |= 1; continue; }
          const int s = it->second;
          acc.add(offM + s, hj.coef[a] * t.ec[s]);
        }
        acc.emit(rw, 3);
      }
    }
    if (k + 1 < N) {                                           // sen with clique k+1
      const Table &t1 = T[k + 1];
      const int64_t offM1 = R->block_offset[mom_block[k + 1]];
      std::vector<int> pos0, pos1;
      for (int a = 0; a < cl[k].nvars; ++a)
        for (int b2 = 0; b2 < cl[k + 1].nvars; ++b2)
          if (cl[k].vars[a] == cl[k + 1].vars[b2]) { pos0.push_back(a); pos1.push_back(b2); break; }
      std::vector<Key> ms;
      const int ns = (int)pos0.size();
      basis(ns, 2 * kappa, ms);
      for (Key m : ms) {
        Key e0 = 0, e1 = 0;
        for (int j = 0; j < ns; ++j) {
          const Key p = (m >> (kBits * j)) & 7u;
          e0 += p << (kBits * pos0[j]);
          e1 += p << (kBits * pos1[j]);
        }
        const int s0 = t.canon.at(e0), s1 = t1.canon.at(e1);
        acc.add(offM + s0, t.ec[s0]);
        acc.add(offM1 + s1, -t1.ec[s1]);
        acc.emit(rw, 4);
      }
    }
  }
  if (bad) return -4;
  // ---- concatenate (clique-major) -------------------------------------------------------
  int64_t m = 0, nnz = 0;
  for (auto &rw : rows) { m += (int64_t)rw.size(); for (auto &r : rw) nnz += (int64_t)r.col.size(); }
  R->indptr.assign(m + 1, 0);
  R->indices.resize(nnz); R->data.resize(nnz);
  R->b.resize(m); R->row_family.resize(m); R->row_stage.resize(m);
  int64_t i = 0, t = 0;
  for (int k = 0; k < N; ++k)
    for (auto &r : rows[k]) {
      for (size_t q = 0; q < r.col.size(); ++q) { R->indices[t] = (int32_t)r.col[q]; R->data[t] = r.val[q]; ++t; }
      R->b[i] = r.rhs; R->row_family[i] = r.fam; R->row_stage[i] = k;
      R->indptr[++i] = t;
    }
  // ---- objective on canonical occurrences (reading Q11) ---------------------------------
  R->C.assign(R->n, 0.0);
  for (int k = 0; k < N; ++k) {
    const int64_t offM = R->block_offset[mom_block[k]];
    for (size_t a = 0; a < f[k].mono.size(); ++a) {
      auto it = T[k].canon.find(f[k].mono[a]);
      if (it == T[k].canon.end()) return -4;
      R->C[offM + it->second] += f[k].coef[a] * T[k].ec[it->second];
    }
  }
  *out = R.release();
  return 0;
}

void strom_gen_sizes(const strom_gen_result *r, int32_t *nblocks, int64_t *n, int64_t *m, int64_t *nnz) {
  if (nblocks) *nblocks = (int32_t)r->block_n.size();
  if (n) *n = r->n;
  if (m) *m = (int64_t)r->b.size();
  if (nnz) *nnz = (int64_t)r->indices.size();
}

void strom_gen_copy(const strom_gen_result *r, int32_t *block_n, int32_t *block_stage, int8_t *block_kind,
                    int64_t *block_offset, int64_t *indptr, int32_t *indices, double *data, double *b, double *C,
                    int8_t *row_family, int32_t *row_stage) {
  std::copy(r->block_n.begin(), r->block_n.end(), block_n);
  std::copy(r->block_stage.begin(), r->block_stage.end(), block_stage);
  std::copy(r->block_kind.begin(), r->block_kind.end(), block_kind);
  std::copy(r->block_offset.begin(), r->block_offset.end(), block_offset);
  std::copy(r->indptr.begin(), r->indptr.end(), indptr);
  std::copy(r->indices.begin(), r->indices.end(), indices);
  std::copy(r->data.begin(), r->data.end(), data);
  std::copy(r->b.begin(), r->b.end(), b);
  std::copy(r->C.begin(), r->C.end(), C);
  std::copy(r->row_family.begin(), r->row_family.end(), row_family);
  std::copy(r->row_stage.begin(), r->row_stage.end(), row_stage);
}

void strom_gen_free(strom_gen_result *r) { delete r; }

}  // extern "C"
