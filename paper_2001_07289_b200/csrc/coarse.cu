// Coarse problem: CSR assembly of S_0 = sum_i R_i^T (Psi_i^T A_i Psi_i) R_i by a segmented
// (deterministic, atomic-free) sum, the multifrontal factorization (one cooperative launch,
// coarse_coop.cu) and the solve plan. Replaces bddc.py:494-511 (COO -> CSR -> SuperLU
// spd_factor) and the coarse solve of bddc.py:362-364.
#include <algorithm>
#include <climits>

#include "bddc_internal.cuh"

namespace bddc {

void coop_build(Ctx& c);
void coop_factor(Ctx& c, cudaStream_t s, int prog);
void coop_solve(Ctx& c, const double* rhs, double* sol, cudaStream_t s, const TvArgs* tv, int queue);

namespace {

__global__ void csr_segsum_kernel(long long nnz, const long long* __restrict__ seg,
                                  const int* __restrict__ contrib, const double* __restrict__ Sloc,
                                  double* __restrict__ val, long long nloc) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (long long k = seg[e]; k < seg[e + 1]; ++k) {
      BDDC_CHECK(contrib[k] >= 0 && contrib[k] < nloc);
      acc += Sloc[contrib[k]];
    }
    val[e] = acc;
  }
}

__global__ void csr_to_front_kernel(long long nnz, const long long* __restrict__ pos,
                                    const double* __restrict__ val, double* __restrict__ fronts,
                                    long long pool) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x) {
    BDDC_CHECK(pos[e] >= 0 && pos[e] < pool);
    fronts[pos[e]] = val[e];
  }
}

}  // namespace

// Solve plan. Every front holds [X; L21] (X = L11^{-1}, the partitioned inverse of the pivot
// block); fronts with s <= coarse_w21_max_sep() also keep W21 = L21 X (scratch pool).
// W21 fronts, one GEMV phase per direction:
//   forward  y_s = X v, upd = gathered - W21 v  (v = rhs + child updates)
//   backward x_s = X^T y_s - W21^T x_bnd
//   * s <= 64 ("row" tasks, mode 1): 256 rows x all separator columns, one thread per row;
//   * otherwise 64 rows x 64 (256) columns (mode 0 / 3); the row (column) chunk's partials
//     are summed by the last task to arrive (fixed order).
// L21 fronts (the top of the tree), two phases per direction with per-chunk dependencies:
//   forward  y_s = X v (mode 0, rows < s), then upd = gathered - L21 y_s (mode 4: column chunk
//            c0 waits for y_s chunk c0 only)
//   backward t = -L21^T x_bnd (mode 2), then x_s = X^T (y_s + t) (mode 3: row chunk r0 waits
//            for t chunk r0 only)
void build_level_schedule(Ctx& c) {
  LevelSchedule& ls = c.sched;
  ls = LevelSchedule{};
  FrontPlan& fp = c.fp;
  const int L = fp.nlevels;
  // gather maps: front position of every node <- child update entries (child order)
  std::vector<long long> goff(fp.nnodes);
  std::vector<int> gptr;
  std::vector<int> gsrc;
  std::vector<std::vector<int>> per_pos;
  for (int nd = 0; nd < fp.nnodes; ++nd) {
    const int f = fp.sep_size[nd] + fp.bnd_size[nd];
    per_pos.assign(f, {});
    for (int q = fp.child_ptr[nd]; q < fp.child_ptr[nd + 1]; ++q) {
      const int ch = fp.child_list[q];
      for (int i = 0; i < fp.bnd_size[ch]; ++i)
        per_pos[fp.rmap_host[fp.bnd_ptr[ch] + i]].push_back((int)(fp.upd_off[ch] + i));
    }
    goff[nd] = (long long)gptr.size();
    int acc = (int)gsrc.size();
    for (int pos = 0; pos < f; ++pos) {
      gptr.push_back(acc);
      for (int v : per_pos[pos]) gsrc.push_back(v);
      acc = (int)gsrc.size();
    }
    gptr.push_back(acc);
  }
  HostTimer ht;
  ht.mark("schedule: solve gather maps");
  ls.gat_ptr = c.upload<int>(gptr.data(), gptr.size());
  ls.gat_src = c.upload<int>(gsrc.data(), std::max<size_t>(gsrc.size(), 1));

  ls.fwd_t.assign(L, nullptr); ls.bwd_t.assign(L, nullptr);
  ls.fwd_r.assign(L, nullptr); ls.bwd_r.assign(L, nullptr);
  ls.n_fwd_t.assign(L, 0); ls.n_bwd_t.assign(L, 0); ls.n_fwd_r.assign(L, 0); ls.n_bwd_r.assign(L, 0);
  std::vector<CsTask> ft, bt;
  std::vector<CsRed> fr, br;
  std::vector<size_t> ft_off(L + 1), bt_off(L + 1), fr_off(L + 1), br_off(L + 1);
  int max_parts = 0;
  std::vector<long long> l_inv, l_y, l_w;
  std::vector<int> l_ldw;
  coarse_df_layout(fp, l_inv, l_y, l_w, l_ldw);  // W21 fronts: l_ldw > 0
  auto base = [&](int nd) {
    CsTask t{};
    t.front_off = fp.front_off[nd];
    t.gat_base = goff[nd];
    t.upd_off = fp.upd_off[nd];
    t.node = nd;
    t.s = fp.sep_size[nd];
    t.f = t.s + fp.bnd_size[nd];
    t.ld = fp.ld[nd];
    t.s0 = fp.sep_start[nd];
    t.red = -1;
    t.np = 1;
    t.w_off = l_w[nd];
    t.ldw = l_ldw[nd];
    t.span = 256;
    return t;
  };
  // partial slots are unique over the whole solve (the dataflow solve overlaps levels)
  std::vector<int> nfch(fp.nnodes, 0), nbch(fp.nnodes, 0);  // finalized chunks per node
  // L21 fronts: per-chunk counters of y_s (forward) and t (backward), chunk = 64 rows / columns
  std::vector<int> ych(fp.nnodes, -1), tch(fp.nnodes, -1);
  int nchunk_ctr = 0;
  int pf = 0, pb = 0;
  // 256-wide tasks for the X / W21 rows of fronts with s >= this (0: always 64): at cfg5 the
  // coarse solve drops from 17.0 to 11.6 ms with every front wide (tools/gpu_ab2.sh)
  const char* we = getenv("BDDC_SOLVE_WIDE_SEP");
  const int wide_sep = we ? atoi(we) : 128;
  // 512-wide tasks for fronts with s >= BDDC_SOLVE_512_SEP (default 2048; 0: never): cfg5
  // coarse solve 11.5 -> 11.4 ms, neutral on cfg3 / cfg2 (tools/gpu_ab4.sh)
  const char* se = getenv("BDDC_SOLVE_512_SEP");
  const int span_sep = se ? (atoi(se) > 0 ? atoi(se) : INT_MAX) : 2048;
  // one reduction chunk: tasks [first, end) share partials (np > 1) or write directly
  auto close_chunk = [](std::vector<CsTask>& v, std::vector<CsRed>& red, size_t first, int p0, int t0) {
    const int cnt = (int)(v.size() - first);
    for (size_t q = first; q < v.size(); ++q) {
      v[q].np = cnt;
      v[q].red = cnt > 1 ? (int)red.size() : -1;
    }
    if (cnt > 1) red.push_back(CsRed{t0, p0, cnt});
    return cnt;
  };
  for (int l = 0; l < L; ++l) {
    ft_off[l] = ft.size(); bt_off[l] = bt.size(); fr_off[l] = fr.size(); br_off[l] = br.size();
    for (int i = fp.level_ptr[l]; i < fp.level_ptr[l + 1]; ++i) {
      const int nd = fp.level_list[i];
      const int sz = fp.sep_size[nd], f = sz + fp.bnd_size[nd];
      const bool wf = l_ldw[nd] > 0 || fp.bnd_size[nd] == 0;  // W21 front (or no boundary)
      if (!wf) {
        if (sz < 128) throw CudaError("coarse solve plan: L21 fronts need s >= 128");
        ych[nd] = nchunk_ctr; nchunk_ctr += ceil_div(sz, 64);
        tch[nd] = nchunk_ctr; nchunk_ctr += ceil_div(sz, 64);
      }
      if (sz <= 64) {
        for (int r0 = 0; r0 < f; r0 += 256) {
          CsTask t = base(nd);
          t.r0 = r0;
          t.rend = std::min(r0 + 256, f);
          t.mode = 1;
          ft.push_back(t);
          nfch[nd]++;
        }
      } else {
        // large separators (the top of the tree, where the level chain is the critical path):
        // narrow tasks whose front entries are all in flight before the dependency wait
        // wide (256-column) tasks for the X / W21 rows of very large fronts: fewer, longer
        // streams where the dependency resolves long before the task starts (BDDC_SOLVE_WIDE_SEP)
        const int cw = sz >= 128 ? (wide_sep > 0 && sz >= wide_sep ? (sz >= span_sep ? 512 : 256) : 64) : 256;
        for (int pass = 0; pass < (wf ? 1 : 2); ++pass) {  // [X; W21] rows | X rows, then L21 rows
          const int rbeg = pass ? sz : 0, rlim = (pass || wf) ? f : sz;
          for (int r0 = rbeg; r0 < rlim; r0 += 64) {
            const size_t first = ft.size();
            const int p0 = pf;
            const int rend = std::min(r0 + 64, rlim);
            const int cwp = pass ? 64 : cw;
            for (int c0 = 0; c0 < sz; c0 += cwp) {
              if (!pass && r0 < sz && c0 > std::min(rend, sz) - 1) break;  // X is lower triangular
              CsTask t = base(nd);
              t.r0 = r0;
              t.rend = rend;
              t.c0 = c0;
              t.part = pf++;
              t.mode = pass ? 4 : 0;
              t.span = pass ? 64 : cw;  // L21 rows wait for one 64-column y_s chunk
              ft.push_back(t);
            }
            if (close_chunk(ft, fr, first, p0, r0) > 0) nfch[nd]++;
          }
        }
      }
      const int rw0 = sz >= 128 ? (wide_sep > 0 && sz >= wide_sep ? (sz >= span_sep ? 512 : 256) : 64) : 256;
      for (int pass = (wf ? 1 : 0); pass < 2; ++pass) {  // (L21: t = -L21^T x_bnd), then x_s
        const int rw = (pass && !wf) ? 64 : rw0;  // L21 fronts' x_s rows wait for one t chunk
        for (int c0 = 0; c0 < sz; c0 += 64) {
          const size_t first = bt.size();
          const int p0 = pb;
          const int rbeg = pass ? (c0 / rw) * rw : sz, rlim = (pass && !wf) ? sz : f;
          for (int r0 = rbeg; r0 < rlim; r0 += rw) {
            CsTask t = base(nd);
            t.r0 = r0;
            t.rend = std::min(r0 + rw, rlim);
            t.c0 = c0;
            t.span = rw;
            t.part = pb++;
            t.mode = pass ? 3 : 2;
            bt.push_back(t);
          }
          if (close_chunk(bt, br, first, p0, c0) > 0 && pass) nbch[nd]++;
        }
      }
    }
  }
  for (auto& t : bt) t.part += pf;  // backward partials after the forward ones
  for (auto& r : br) r.p0 += pf;
  max_parts = pf + pb;
  ft_off[L] = ft.size(); bt_off[L] = bt.size(); fr_off[L] = fr.size(); br_off[L] = br.size();
  CsTask* dft = c.upload<CsTask>(ft.data(), std::max<size_t>(ft.size(), 1));
  CsTask* dbt = c.upload<CsTask>(bt.data(), std::max<size_t>(bt.size(), 1));
  CsRed* dfr = c.upload<CsRed>(fr.data(), std::max<size_t>(fr.size(), 1));
  CsRed* dbr = c.upload<CsRed>(br.data(), std::max<size_t>(br.size(), 1));
  for (int l = 0; l < L; ++l) {
    ls.fwd_t[l] = dft + ft_off[l]; ls.n_fwd_t[l] = (int)(ft_off[l + 1] - ft_off[l]);
    ls.bwd_t[l] = dbt + bt_off[l]; ls.n_bwd_t[l] = (int)(bt_off[l + 1] - bt_off[l]);
    ls.fwd_r[l] = dfr + fr_off[l]; ls.n_fwd_r[l] = (int)(fr_off[l + 1] - fr_off[l]);
    ls.bwd_r[l] = dbr + br_off[l]; ls.n_bwd_r[l] = (int)(br_off[l + 1] - br_off[l]);
  }
  ls.partial = c.alloc<double>((size_t)std::max(max_parts, 1) * 64);
  ls.ybuf = c.alloc<double>((size_t)std::max(fp.n_coarse, 1));
  ls.tbuf = c.alloc<double>((size_t)std::max(fp.n_coarse, 1));
  BDDC_CUDA(cudaMemset(ls.tbuf, 0, sizeof(double) * std::max(fp.n_coarse, 1)));  // stays 0 where b = 0
  ls.red_cnt = c.alloc<int>(fr.size() + br.size() + 1);
  BDDC_CUDA(cudaMemset(ls.red_cnt, 0, sizeof(int) * (fr.size() + br.size() + 1)));
  {
    // dataflow solve queue. Counters: [0, N) finalized forward chunks of each node's children,
    // [N, 2N) own forward chunks, [2N, 3N) own x_s chunks, then per 64-chunk y_s / t counters
    // of the L21 fronts.
    const int N = fp.nnodes;
    std::vector<int> need(N, 0);
    for (int nd = 0; nd < N; ++nd)
      if (fp.parent[nd] >= 0) need[fp.parent[nd]] += nfch[nd];
    std::vector<SdTask> q;
    q.reserve(ft.size() + bt.size() + (c.geo.s_hi - c.geo.s_lo));
    // v = T rho tasks (no dependencies), in slices before each of the top K forward and top K
    // backward levels: the CTAs take them while the chains at the top of the tree leave them
    // idle, and each slice drains in about one level's latency
    const bool tv = c.geo.nG_pad > 0 && c.geo.nG_pad <= 256;
    const int K = std::min(8, L);
    const int nsl = std::max(2 * K, 1);
    const int nl = c.geo.s_hi - c.geo.s_lo;
    int next_sub = c.geo.s_lo, slice = 0;
    ls.n_tv = 0;
    auto emit_tv = [&](bool last) {
      if (!tv) return;
      const int upto = last ? c.geo.s_hi : c.geo.s_lo + (int)((long long)nl * (slice + 1) / nsl);
      ++slice;
      for (; next_sub < upto; ++next_sub) {
        SdTask d{};
        d.t.node = next_sub;
        d.dir = 2;
        d.dep = d.sig0 = d.sig1 = d.sig2 = -1;
        q.push_back(d);
        ls.n_tv++;
      }
    };
    const int C0 = 3 * N;  // per-chunk counters of the L21 fronts start here
    for (int l = 0; l < L; ++l) {  // forward: level order, bottom-up
      if (l >= L - K) emit_tv(false);
      for (size_t i = ft_off[l]; i < ft_off[l + 1]; ++i) {
        const CsTask& t = ft[i];
        SdTask d{};
        d.t = t;
        d.dir = 0;
        d.sig2 = -1;
        if (t.mode == 4) {  // L21 rows x y_s chunk c0 (cw = 64)
          d.dep = C0 + ych[t.node] + t.c0 / 64;
          d.tgt = 1;
        } else {
          d.dep = need[t.node] > 0 ? t.node : -1;
          d.tgt = need[t.node];
          if (ych[t.node] >= 0) d.sig2 = C0 + ych[t.node] + t.r0 / 64;  // y_s chunk final
        }
        d.sig0 = fp.parent[t.node] >= 0 ? fp.parent[t.node] : -1;
        d.sig1 = N + t.node;
        q.push_back(d);
      }
    }
    for (int l = L - 1; l >= 0; --l) {  // backward: top-down
      if (l >= L - K) emit_tv(l == L - K);
      for (size_t i = bt_off[l]; i < bt_off[l + 1]; ++i) {
        const CsTask& t = bt[i];
        SdTask d{};
        d.t = t;
        d.dir = 1;
        d.sig1 = d.sig2 = -1;
        if (t.mode == 3 && tch[t.node] >= 0) {  // X^T (y + t), rows r0: after t chunk r0 (rw = 64)
          d.dep = C0 + tch[t.node] + t.r0 / 64;
          d.tgt = 1;
        } else {  // the nearest ancestor's x_s final (without one: the front's own forward)
          int anc = fp.parent[t.node];
          while (anc >= 0 && nbch[anc] == 0) anc = fp.parent[anc];
          d.dep = anc >= 0 ? 2 * N + anc : N + t.node;
          d.tgt = anc >= 0 ? nbch[anc] : nfch[t.node];
          if (d.tgt <= 0) d.dep = -1;
        }
        if (t.mode == 3) d.sig0 = 2 * N + t.node;
        else d.sig0 = C0 + tch[t.node] + t.c0 / 64;  // t chunk final
        q.push_back(d);
      }
    }
    emit_tv(true);  // (L == 0)
    ls.queues.clear();
    if (!c.dist.on) {
      ls.queues.push_back({c.upload<SdTask>(q.data(), std::max<size_t>(q.size(), 1)), (int)q.size()});
    } else {
      // distributed: three launches with exchanges between them: this rank's
      // subtrees forward (+ the v = T rho tasks), the replicated top forward + backward, this
      // rank's subtrees backward. A dependency on a node of an earlier launch is dropped (its
      // data is final and exchanged before the next launch); another rank's nodes are skipped.
      const std::vector<int>& ph = c.dist.phase;
      std::vector<int> need_d(N, 0);
      for (int nd = 0; nd < N; ++nd)
        if (fp.parent[nd] >= 0 && ph[nd] == ph[fp.parent[nd]]) need_d[fp.parent[nd]] += nfch[nd];
      std::vector<SdTask> qq[3];
      for (SdTask d : q) {
        if (d.dir == 2) {
          qq[0].push_back(d);
          continue;
        }
        const int nd = d.t.node, p = ph[nd];
        if (p < 0) continue;
        const int qi = d.dir == 0 ? (p == 0 ? 0 : 1) : (p == 0 ? 2 : 1);
        if (d.dir == 0 && d.t.mode != 4) {
          d.dep = need_d[nd] > 0 ? nd : -1;
          d.tgt = need_d[nd];
        } else if (d.dir == 1 && !(d.t.mode == 3 && tch[nd] >= 0)) {
          int anc = fp.parent[nd];
          while (anc >= 0 && nbch[anc] == 0) anc = fp.parent[anc];
          if (anc >= 0 ? ph[anc] != p : p == 0) d.dep = -1;
        }
        qq[qi].push_back(d);
      }
      for (auto& v : qq) ls.queues.push_back({c.upload<SdTask>(v.data(), std::max<size_t>(v.size(), 1)), (int)v.size()});
    }
    ls.df_tasks = ls.queues[0].first;
    ls.n_df = ls.queues[0].second;
    ls.n_ctr = 3 * N + nchunk_ctr;
    ls.df_ctr = c.alloc<int>(ls.n_ctr + 2);  // + queue head + error flag
    BDDC_CUDA(cudaMemset(ls.df_ctr, 0, sizeof(int) * (ls.n_ctr + 2)));
  }
  ht.mark("schedule: solve tasks + queue");
  coop_build(c);
  ht.mark("schedule: factor program (total)");
}

void coarse_assemble_and_factor(Ctx& c) {
  FrontPlan& fp = c.fp;
  FrontDev& fd = fp.d;
  if (fp.n_coarse == 0) return;
  cudaStream_t s = c.stream;
  PhaseScope ps(c.prof, "setup.coarse", s);
  const int th = 256;
  { csr_segsum_kernel<<<std::min<long long>((fp.nnz + th - 1) / th, 148 * 16), th, 0, s>>>(
      fp.nnz, fp.seg_ptr, fp.contrib, c.Sloc, fp.csr_val,
      (long long)c.geo.nsub * c.geo.nc_pad * c.geo.nc_pad); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
  front_memset(c, s);
  { csr_to_front_kernel<<<std::min<long long>((fp.nnz + th - 1) / th, 148 * 16), th, 0, s>>>(
      fp.nnz, fp.csr_front_pos, fp.csr_val, fd.fronts, fp.front_pool); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
  // multifrontal factorization + partitioned inverse: one cooperative launch
  if (!c.dist.on) {
    coop_factor(c, s, 0);
    front_pool_mark_clean(c);
    return;
  }
  // distributed: this rank's subtrees, the subtree roots' update blocks to
  // every rank, then the replicated top of the tree
  coop_factor(c, s, 0);
  std::vector<ExSeg> segs;
  const DistCoarse& D = c.dist;
  for (size_t i = 0; i < D.roots.size(); ++i) {
    const int r = D.roots[i], sz = fp.sep_size[r], b = fp.bnd_size[r], ld = fp.ld[r];
    if (b > 0) segs.push_back(ExSeg{fd.fronts + fp.front_off[r] + sz + (long long)sz * ld, 0, D.root_owner[i], 1, b, ld});
  }
  allgather_segments(c, segs, s);
  coop_factor(c, s, 1);
  front_pool_mark_clean(c);
}

void coarse_solve(Ctx& c, const double* rhs, double* sol, cudaStream_t s, const TvArgs* tv) {
  if (!c.dist.on) {
    coop_solve(c, rhs, sol, s, tv, 0);
    return;
  }
  const FrontPlan& fp = c.fp;
  const DistCoarse& D = c.dist;
  coop_solve(c, rhs, sol, s, tv, 0);  // this rank's subtrees, forward
  std::vector<ExSeg> segs;  // the subtree roots' update vectors
  for (size_t i = 0; i < D.roots.size(); ++i) {
    const int r = D.roots[i];
    if (fp.bnd_size[r] > 0) segs.push_back(ExSeg{fp.d.upd + fp.upd_off[r], fp.bnd_size[r], D.root_owner[i], 0, 0, 0});
  }
  allgather_segments(c, segs, s);
  coop_solve(c, rhs, sol, s, nullptr, 1);  // the top, forward + backward (replicated)
  coop_solve(c, rhs, sol, s, nullptr, 2);  // this rank's subtrees, backward
  segs.clear();  // every subtree's solution (a contiguous range of elimination positions)
  for (size_t i = 0; i < D.roots.size(); ++i) {
    const long long a = fp.sep_start[D.sub_lo[i]], e = fp.sep_start[D.sub_hi[i]] + fp.sep_size[D.sub_hi[i]];
    if (e > a) segs.push_back(ExSeg{sol + a, e - a, D.root_owner[i], 0, 0, 0});
  }
  allgather_segments(c, segs, s);
}

}  // namespace bddc
