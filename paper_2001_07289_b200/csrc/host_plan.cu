// Native host symbolic work of the setup (the cold start): the lower CSR pattern of the
// coarse matrix S_0 in elimination order with its segmented contribution lists, and the
// CSR -> front position map. Same output as symbolic.coarse_csr (the numpy statement it
// replaces, kept as the checker: tests/test_host_plan.py), O(contributions) with a
// counting sort by row and a stable per-row sort by column, rows split over host threads.
//
// Reference: the coarse COO -> CSR assembly of build_bddc (bddc.py:494-505), whose
// duplicate summation order (ascending subdomain) the device segmented sum reproduces.
#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bddcso_b200.h"

namespace {

template <class F>
void parallel_for(long long n, F&& f) {
  unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n < 4096) nt = 1;
  std::vector<std::thread> th;
  std::atomic<long long> next{0};
  const long long chunk = std::max<long long>(1024, n / (nt * 16));
  auto work = [&] {
    for (;;) {
      const long long a = next.fetch_add(chunk);
      if (a >= n) break;
      const long long b = std::min(n, a + chunk);
      for (long long i = a; i < b; ++i) f(i);
    }
  };
  for (unsigned t = 1; t < nt; ++t) th.emplace_back(work);
  work();
  for (auto& t : th) t.join();
}

}  // namespace

extern "C" {

// Inputs: nsub subdomains, constraints of subdomain p = sub_con_ids[sub_con_ptr[p] ..
// sub_con_ptr[p+1]) (coarse ids, local order), iperm (coarse id -> elimination position, n),
// nc_pad; the nested-dissection fronts (sep_start, sep_size, bnd_ptr, bnd_idx ascending).
// Outputs (caller-allocated, capacity = number of lower contributions incl. the diagonal):
// csr_row / csr_col (elimination positions, row-major, columns ascending), csr_node, frow,
// fcol (front positions), seg_ptr [nnz + 1], contrib (sub * nc_pad^2 + k + l * nc_pad, by
// entry then ascending subdomain). Returns nnz, or -1 on an entry outside its front.
long long bddc_coarse_pattern(int nsub, const long long* sub_con_ptr, const long long* sub_con_ids,
                              const long long* iperm, long long n, int nc_pad, int nnodes,
                              const long long* sep_start, const long long* sep_size, const long long* bnd_ptr,
                              const long long* bnd_idx, long long* csr_row, long long* csr_col,
                              long long* csr_node, long long* frow, long long* fcol, long long* seg_ptr,
                              int* contrib) {
  // 1. contributions per row (counting sort): row = max position of the pair, col = min
  std::vector<long long> rcount(n + 1, 0);
  for (int p = 0; p < nsub; ++p) {
    const long long a = sub_con_ptr[p], m = sub_con_ptr[p + 1] - a;
    for (long long k = 0; k < m; ++k) {
      const long long ek = iperm[sub_con_ids[a + k]];
      for (long long l = 0; l < m; ++l)
        if (ek >= iperm[sub_con_ids[a + l]]) rcount[ek + 1]++;
    }
  }
  for (long long r = 0; r < n; ++r) rcount[r + 1] += rcount[r];
  const long long ncontrib = rcount[n];
  std::vector<long long> ccol(ncontrib);
  std::vector<int> cidx(ncontrib);
  {
    std::vector<long long> fill(rcount.begin(), rcount.end() - 1);
    for (int p = 0; p < nsub; ++p) {  // ascending subdomain: per row, subdomain order is kept
      const long long a = sub_con_ptr[p], m = sub_con_ptr[p + 1] - a;
      const long long base = (long long)p * nc_pad * nc_pad;
      for (long long k = 0; k < m; ++k) {
        const long long ek = iperm[sub_con_ids[a + k]];
        for (long long l = 0; l < m; ++l) {
          const long long el = iperm[sub_con_ids[a + l]];
          if (ek < el) continue;
          const long long q = fill[ek]++;
          ccol[q] = el;
          cidx[q] = (int)(base + k + l * nc_pad);
        }
      }
    }
  }
  // 2. per row: stable sort by column (keeps ascending subdomain inside an entry), count the
  // distinct columns
  std::vector<long long> rnnz(n + 1, 0);
  parallel_for(n, [&](long long r) {
    const long long a = rcount[r], b = rcount[r + 1];
    if (b - a > 1) {
      std::vector<std::pair<long long, int>> v(b - a);
      for (long long q = a; q < b; ++q) v[q - a] = {ccol[q], cidx[q]};
      std::stable_sort(v.begin(), v.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
      for (long long q = a; q < b; ++q) { ccol[q] = v[q - a].first; cidx[q] = v[q - a].second; }
    }
    long long u = 0;
    for (long long q = a; q < b; ++q) u += (q == a || ccol[q] != ccol[q - 1]);
    rnnz[r + 1] = u;
  });
  for (long long r = 0; r < n; ++r) rnnz[r + 1] += rnnz[r];
  const long long nnz = rnnz[n];
  // node of every elimination position
  std::vector<int> node_of(n);
  for (int i = 0; i < nnodes; ++i)
    for (long long q = sep_start[i]; q < sep_start[i] + sep_size[i]; ++q) node_of[q] = i;
  std::atomic<int> bad{0};
  parallel_for(n, [&](long long r) {
    long long e = rnnz[r];
    const long long a = rcount[r], b = rcount[r + 1];
    for (long long q = a; q < b; ++q) {
      if (q != a && ccol[q] == ccol[q - 1]) continue;
      const long long c = ccol[q];
      const int nd = node_of[c];
      csr_row[e] = r;
      csr_col[e] = c;
      csr_node[e] = nd;
      fcol[e] = c - sep_start[nd];
      if (r < sep_start[nd] + sep_size[nd]) {
        frow[e] = r - sep_start[nd];
      } else {
        const long long* b0 = bnd_idx + bnd_ptr[nd];
        const long long* b1 = bnd_idx + bnd_ptr[nd + 1];
        const long long* it = std::lower_bound(b0, b1, r);
        if (it == b1 || *it != r) bad = 1;
        frow[e] = sep_size[nd] + (it - b0);
      }
      seg_ptr[e] = q;
      ++e;
    }
  });
  seg_ptr[nnz] = ncontrib;
  for (long long q = 0; q < ncontrib; ++q) contrib[q] = cidx[q];
  return bad ? -1 : nnz;
}

}  // extern "C"

// ---- nested-dissection symbolic analysis of the coarse problem (symbolic.analyze, native) ----
// Same tree, elimination order, boundaries and extend-add maps as the numpy statement
// (symbolic.py: nested_dissection + analyze, the checker in tests/test_host_plan.py): the
// subdomain lattice box is halved along its longest axis (first on ties) at ext / 2; the
// coarse dofs whose owners straddle the cut are the separator, the others go to the halves
// (order kept); a cell box holds a leaf; a separator-free cut with one non-empty half is
// skipped. Children before parents (postorder).
namespace {

struct NdPlan {
  std::vector<long long> perm, sep_start, sep_size, level, parent, bnd_ptr, bnd_idx, rmap;
};

struct NdBuilder {
  int dim, W;
  const int* owners;
  std::vector<int> lo, hi;  // per dof, per axis: owner bounding box in lattice coordinates
  std::vector<std::vector<long long>> seps;
  std::vector<std::vector<int>> kids;
  int rec(const int* blo, const int* bhi, std::vector<long long>& idx) {
    if (idx.empty()) return -1;
    int ext[3] = {0, 0, 0};
    long long vol = 1;
    for (int d = 0; d < dim; ++d) ext[d] = bhi[d] - blo[d], vol *= ext[d];
    if (vol <= 1) {
      std::sort(idx.begin(), idx.end());
      seps.push_back(std::move(idx));
      kids.emplace_back();
      return (int)seps.size() - 1;
    }
    int ax = 0;
    for (int d = 1; d < dim; ++d)
      if (ext[d] > ext[ax]) ax = d;
    const int mid = blo[ax] + ext[ax] / 2;
    std::vector<long long> left, right, sep;
    for (long long i : idx) {
      const int l = lo[i * dim + ax], h = hi[i * dim + ax];
      if (h < mid) left.push_back(i);
      else if (l >= mid) right.push_back(i);
      else sep.push_back(i);
    }
    idx.clear();
    idx.shrink_to_fit();
    int lhi[3] = {bhi[0], bhi[1], bhi[2]}, rlo[3] = {blo[0], blo[1], blo[2]};
    lhi[ax] = mid;
    rlo[ax] = mid;
    std::vector<int> ks;
    const int a = rec(blo, lhi, left);
    if (a >= 0) ks.push_back(a);
    const int b = rec(rlo, bhi, right);
    if (b >= 0) ks.push_back(b);
    if (sep.empty() && ks.size() == 1) return ks[0];
    std::sort(sep.begin(), sep.end());
    seps.push_back(std::move(sep));
    kids.push_back(std::move(ks));
    return (int)seps.size() - 1;
  }
};

}  // namespace

struct bddc_nd {
  NdPlan p;
};

extern "C" {

// owners [n * W] (-1 padded owner subdomains of every coarse dof), sub_coords [nsub * dim]
// lattice coordinates, subs [dim], sub_con_ptr / sub_con_ids: CSR subdomain -> its coarse ids.
// Returns 0 (handle in *out) or 1 (inconsistent input; msg in err).
int bddc_nd_build(long long n, int W, const int* owners, int nsub, int dim, const int* sub_coords, const int* subs,
                  const long long* sub_con_ptr, const long long* sub_con_ids, bddc_nd** out, char* err, size_t errlen) {
  auto fail = [&](const char* m) {
    if (err && errlen) {
      snprintf(err, errlen, "%s", m);
    }
    return 1;
  };
  if (!out || dim < 1 || dim > 3) return fail("invalid argument");
  *out = nullptr;
  NdBuilder B;
  B.dim = dim;
  B.W = W;
  B.owners = owners;
  B.lo.assign(n * dim, INT32_MAX);
  B.hi.assign(n * dim, -1);
  for (long long i = 0; i < n; ++i)
    for (int k = 0; k < W; ++k) {
      const int p = owners[i * W + k];
      if (p < 0) continue;
      for (int d = 0; d < dim; ++d) {
        const int c = sub_coords[(long long)p * dim + d];
        B.lo[i * dim + d] = std::min(B.lo[i * dim + d], c);
        B.hi[i * dim + d] = std::max(B.hi[i * dim + d], c);
      }
    }
  std::vector<long long> all(n);
  for (long long i = 0; i < n; ++i) all[i] = i;
  const int blo[3] = {0, 0, 0};
  int bhi[3] = {1, 1, 1};
  for (int d = 0; d < dim; ++d) bhi[d] = subs[d];
  B.rec(blo, bhi, all);
  const int N = (int)B.seps.size();
  bddc_nd* h = new bddc_nd;
  NdPlan& P = h->p;
  P.sep_size.resize(N);
  P.sep_start.resize(N);
  P.parent.assign(N, -1);
  P.level.assign(N, 0);
  long long acc = 0;
  for (int i = 0; i < N; ++i) {
    P.sep_start[i] = acc;
    P.sep_size[i] = (long long)B.seps[i].size();
    acc += P.sep_size[i];
    for (long long v : B.seps[i]) P.perm.push_back(v);
  }
  if (acc != n) {
    delete h;
    return fail("nested dissection lost coarse dofs");
  }
  std::vector<long long> iperm(n);
  for (long long q = 0; q < n; ++q) iperm[P.perm[q]] = q;
  for (int i = 0; i < N; ++i)
    for (int k : B.kids[i]) {
      P.parent[k] = i;
      P.level[i] = std::max(P.level[i], P.level[k] + 1);
    }
  // boundaries, bottom-up: own subdomains' constraints and the children's boundaries
  std::vector<std::vector<long long>> bnd(N);
  std::vector<int> own;
  std::vector<long long> cand;
  for (int i = 0; i < N; ++i) {
    const long long end = P.sep_start[i] + P.sep_size[i];
    own.clear();
    for (long long v : B.seps[i])
      for (int k = 0; k < W; ++k)
        if (owners[v * W + k] >= 0) own.push_back(owners[v * W + k]);
    std::sort(own.begin(), own.end());
    own.erase(std::unique(own.begin(), own.end()), own.end());
    cand.clear();
    for (int p : own)
      for (long long q = sub_con_ptr[p]; q < sub_con_ptr[p + 1]; ++q) {
        const long long e = iperm[sub_con_ids[q]];
        if (e >= end) cand.push_back(e);
      }
    for (int k : B.kids[i])
      for (long long e : bnd[k])
        if (e >= end) cand.push_back(e);
    std::sort(cand.begin(), cand.end());
    cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
    bnd[i] = cand;
  }
  P.bnd_ptr.assign(N + 1, 0);
  for (int i = 0; i < N; ++i) P.bnd_ptr[i + 1] = P.bnd_ptr[i] + (long long)bnd[i].size();
  P.bnd_idx.reserve(P.bnd_ptr[N]);
  for (int i = 0; i < N; ++i) P.bnd_idx.insert(P.bnd_idx.end(), bnd[i].begin(), bnd[i].end());
  P.rmap.assign(P.bnd_ptr[N], 0);
  for (int i = 0; i < N; ++i) {
    const long long p = P.parent[i];
    if (p < 0) {
      if (!bnd[i].empty()) {
        delete h;
        return fail("root front has a boundary");
      }
      continue;
    }
    const long long s0 = P.sep_start[p], ss = P.sep_size[p];
    for (size_t q = 0; q < bnd[i].size(); ++q) {
      const long long e = bnd[i][q];
      long long pos;
      if (e >= s0 && e < s0 + ss) {
        pos = e - s0;
      } else {
        auto it = std::lower_bound(bnd[p].begin(), bnd[p].end(), e);
        if (it == bnd[p].end() || *it != e) {
          delete h;
          return fail("child boundary not contained in parent front");
        }
        pos = ss + (it - bnd[p].begin());
      }
      P.rmap[P.bnd_ptr[i] + q] = pos;
    }
  }
  *out = h;
  return 0;
}

long long bddc_nd_size(const bddc_nd* h, const char* what) {
  if (!h || !what) return -1;
  const std::string w(what);
  if (w == "nnodes") return (long long)h->p.sep_size.size();
  if (w == "nbnd") return (long long)h->p.bnd_idx.size();
  if (w == "n") return (long long)h->p.perm.size();
  return -1;
}

// int64 arrays by name: perm, sep_start, sep_size, level, parent, bnd_ptr, bnd_idx, rmap
int bddc_nd_copy(const bddc_nd* h, const char* name, long long* host, long long count) {
  if (!h || !name) return 1;
  const NdPlan& P = h->p;
  const std::string n(name);
  const std::vector<long long>* v = n == "perm" ? &P.perm : n == "sep_start" ? &P.sep_start
                                  : n == "sep_size" ? &P.sep_size : n == "level" ? &P.level
                                  : n == "parent" ? &P.parent : n == "bnd_ptr" ? &P.bnd_ptr
                                  : n == "bnd_idx" ? &P.bnd_idx : n == "rmap" ? &P.rmap : nullptr;
  if (!v || (long long)v->size() != count) return 1;
  std::copy(v->begin(), v->end(), host);
  return 0;
}

void bddc_nd_free(bddc_nd* h) { delete h; }

}  // extern "C"
