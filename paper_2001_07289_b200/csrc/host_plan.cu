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
