// Coarse problem: CSR assembly of S_0 = sum_i R_i^T (Psi_i^T A_i Psi_i) R_i by a segmented
// (deterministic, atomic-free) sum, then a multifrontal Cholesky over a geometric
// nested-dissection tree of the subdomain lattice, and the forward/backward solves.
// Replaces bddc.py:494-511 (COO -> CSR -> SuperLU spd_factor) and the coarse solve of
// bddc.py:362-364.
#include <algorithm>
#include <climits>

#include "bddc_internal.cuh"

namespace bddc {

void coop_build(Ctx& c);
void coop_factor(Ctx& c, cudaStream_t s);
void coop_solve(Ctx& c, const double* rhs, double* sol, cudaStream_t s);

namespace {

__global__ void csr_segsum_kernel(long long nnz, const long long* __restrict__ seg,
                                  const int* __restrict__ contrib, const double* __restrict__ Sloc,
                                  double* __restrict__ val) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (long long k = seg[e]; k < seg[e + 1]; ++k) acc += Sloc[contrib[k]];
    val[e] = acc;
  }
}

__global__ void csr_to_front_kernel(long long nnz, const long long* __restrict__ pos,
                                    const double* __restrict__ val, double* __restrict__ fronts) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x)
    fronts[pos[e]] = val[e];
}

// Extend-add the update (Schur) block of child #k of every node in `nodes` into its front.
__global__ void extend_add_kernel(const int* __restrict__ nodes, int k, const int* __restrict__ child_ptr,
                                  const int* __restrict__ child_list, const int* __restrict__ sep_size,
                                  const int* __restrict__ bnd_size, const int* __restrict__ ld,
                                  const long long* __restrict__ front_off,
                                  const int* __restrict__ rmap, const int* __restrict__ rmap_ptr,
                                  double* fronts) {
  const int node = nodes[blockIdx.y];
  const int c0 = child_ptr[node], c1 = child_ptr[node + 1];
  if (k >= c1 - c0) return;
  const int ch = child_list[c0 + k];
  const int b = bnd_size[ch], s = sep_size[ch], lc = ld[ch], lp = ld[node];
  const double* U = fronts + front_off[ch] + s + (long long)s * lc;
  double* F = fronts + front_off[node];
  const int* rm = rmap + rmap_ptr[ch];
  const long long total = (long long)b * b;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx % b), j = (int)(idx / b);
    if (i < j) continue;
    F[rm[i] + (long long)rm[j] * lp] += U[i + (long long)j * lc];
  }
}

// ---- partitioned-inverse preparation: copy L11 to scratch, replace it by the identity ----
__global__ void inv_prep_kernel(const InvTask* __restrict__ tasks, FrontDev fd, double* scratch) {
  const InvTask t = tasks[blockIdx.y];
  const int s = fd.sep_size[t.node], ld = fd.ld[t.node];
  double* F = fd.fronts + fd.front_off[t.node];
  double* S = scratch + t.scr;
  const long long total = (long long)s * s;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx % s), j = (int)(idx / s);
    double* fp = F + i + (long long)j * ld;
    S[i + (long long)j * t.lds] = i >= j ? *fp : 0.0;  // each element copied, then reset,
    *fp = i == j ? 1.0 : 0.0;                          // by the same thread
  }
}

// Sum of the children update entries landing on front position `pos` of `node`.
__device__ __forceinline__ double gather_children(const LevelView& lv, const double* __restrict__ upd,
                                                  int node, int pos) {
  const int* gp = lv.gat_ptr + lv.gat_off[node];
  double acc = 0.0;
  for (int q = gp[pos]; q < gp[pos + 1]; ++q) acc += upd[lv.gat_src[q]];
  return acc;
}

// Forward tile: partial[r] = sum_{k in [c0, c0+256)} F'[r][k] v_S[k] for rows [r0, r0+64),
// F' = [L11^{-1}; L21 L11^{-1}], v_S = rhs(sep) + children updates.
__global__ void __launch_bounds__(256) cs_fwd_partial_kernel(const CsTask* __restrict__ tasks, FrontDev fd,
                                                             LevelView lv, const double* __restrict__ rhs,
                                                             double* __restrict__ partial) {
  __shared__ double vs[256];
  __shared__ double red[4][64];
  const CsTask t = tasks[blockIdx.x];
  const int node = t.node, s = fd.sep_size[node], f = s + fd.bnd_size[node];
  const long long ld = fd.ld[node];
  const int s0 = fd.sep_start[node];
  const double* F = fd.fronts + fd.front_off[node];
  for (int k = threadIdx.x; k < 256; k += blockDim.x) {
    const int kk = t.c0 + k;
    vs[k] = kk < s ? rhs[s0 + kk] + gather_children(lv, fd.upd, node, kk) : 0.0;
  }
  __syncthreads();
  const int rr = threadIdx.x & 63, grp = threadIdx.x >> 6;
  const int r = t.r0 + rr;
  double a0 = 0.0, a1 = 0.0;
  if (r < f) {
    int kb = t.c0 + grp * 64;
    int ke = min(kb + 64, s);
    if (r < s) ke = min(ke, r + 1);  // L11^{-1} is lower triangular
    int k = kb;
    for (; k + 1 < ke; k += 2) {
      a0 += F[r + k * ld] * vs[k - t.c0];
      a1 += F[r + (k + 1) * ld] * vs[k + 1 - t.c0];
    }
    if (k < ke) a0 += F[r + k * ld] * vs[k - t.c0];
  }
  red[grp][rr] = a0 + a1;
  __syncthreads();
  if (threadIdx.x < 64)
    partial[(long long)t.part * 64 + threadIdx.x] = red[0][threadIdx.x] + red[1][threadIdx.x] +
                                                   red[2][threadIdx.x] + red[3][threadIdx.x];
}

// Forward reduction: y_S -> sol(sep); update of the boundary -> upd pool.
__global__ void cs_fwd_reduce_kernel(const CsRed* __restrict__ reds, FrontDev fd, LevelView lv,
                                     const double* __restrict__ partial, double* __restrict__ sol) {
  const CsRed t = reds[blockIdx.x];
  const int node = t.node, s = fd.sep_size[node], f = s + fd.bnd_size[node];
  const int r = t.t0 + threadIdx.x;
  if (threadIdx.x >= 64 || r >= f) return;
  double acc = 0.0;
  for (int p = 0; p < t.np; ++p) acc += partial[(long long)(t.p0 + p) * 64 + threadIdx.x];
  if (r < s) sol[fd.sep_start[node] + r] = acc;
  else fd.upd[fd.upd_off[node] + (r - s)] = gather_children(lv, fd.upd, node, r) - acc;
}

// Backward tile: partial[k] = sum_{r in [r0, r0+256)} F'[r][k] w[r] for columns [c0, c0+64),
// w = [y_S; -x_B].
__global__ void __launch_bounds__(256) cs_bwd_partial_kernel(const CsTask* __restrict__ tasks, FrontDev fd,
                                                             const double* __restrict__ sol,
                                                             double* __restrict__ partial) {
  __shared__ double w[256];
  const CsTask t = tasks[blockIdx.x];
  const int node = t.node, s = fd.sep_size[node], f = s + fd.bnd_size[node];
  const long long ld = fd.ld[node];
  const int s0 = fd.sep_start[node];
  const int* bidx = fd.bnd_idx + fd.bnd_ptr[node];
  const double* F = fd.fronts + fd.front_off[node];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    const int r = t.r0 + i;
    w[i] = r < s ? sol[s0 + r] : (r < f ? -sol[bidx[r - s]] : 0.0);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int cc = 0; cc < 8; ++cc) {
    const int kl = warp * 8 + cc, k = t.c0 + kl;
    double acc = 0.0;
    if (k < s) {
      const double* col = F + k * ld;
      for (int i = lane; i < 256; i += 32) {
        const int r = t.r0 + i;
        if (r < f && (r >= s || r >= k)) acc += col[r] * w[i];
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) partial[(long long)t.part * 64 + kl] = acc;
  }
}

__global__ void cs_bwd_reduce_kernel(const CsRed* __restrict__ reds, FrontDev fd,
                                     const double* __restrict__ partial, double* __restrict__ sol) {
  const CsRed t = reds[blockIdx.x];
  const int node = t.node, s = fd.sep_size[node];
  const int k = t.t0 + threadIdx.x;
  if (threadIdx.x >= 64 || k >= s) return;
  double acc = 0.0;
  for (int p = 0; p < t.np; ++p) acc += partial[(long long)(t.p0 + p) * 64 + threadIdx.x];
  sol[fd.sep_start[node] + k] = acc;
}

}  // namespace

void build_level_schedule(Ctx& c) {
  LevelSchedule& ls = c.sched;
  ls = LevelSchedule{};
  FrontPlan& fp = c.fp;
  const int L = fp.nlevels;
  ls.steps.assign(L, {});
  std::vector<int> flat;
  ls.nodes_off.assign(L + 1, 0);
  for (int l = 0; l < L; ++l) {
    ls.nodes_off[l] = (int)flat.size();
    for (int i = fp.level_ptr[l]; i < fp.level_ptr[l + 1]; ++i) flat.push_back(fp.level_list[i]);
  }
  ls.nodes_off[L] = (int)flat.size();
  ls.d_nodes = c.upload<int>(flat.data(), flat.size());
  for (int n = 0; n < fp.nnodes; ++n)
    ls.max_children = std::max(ls.max_children, fp.child_ptr[n + 1] - fp.child_ptr[n]);
  // ---- factorization + partitioned inverse, per level and 64-column step ----
  // factor step k:  potrf(diag) ; trtri(diag -> scratch slot) ; L21 <- L21 inv^T ; A22 -= L21 L21^T
  // inverse step t (panel P = [I; L21] after inv_prep, L11 copy in inv_scratch), kb from last:
  //                 trtri(L11[kb,kb]) ; P[:,kb] <- P[:,kb] inv ; P[:,0:k] -= P[:,kb] L11[kb,0:k]
  std::vector<TileTask> potrf_all, trtri_all;
  std::vector<GemmTask> ts_all, g_all;
  struct Ref {
    int l; bool inv;
    size_t p0, r0, t0, g0;
    int np, nr, nt, ng, tsM, tsN, gM, gN;
  };
  std::vector<Ref> refs;
  std::vector<InvTask> prep_all;
  std::vector<size_t> prep_off(L + 1, 0);
  long long scr_max = 0;
  std::vector<long long> scr_of(fp.nnodes, 0);
  std::vector<int> lds_of(fp.nnodes, 0);
  size_t max_slots = 1;
  const long long IS = kTileInvStride;
  std::vector<std::pair<size_t, long long>> slot_fix_trtri;  // (task idx, slot) patched later
  std::vector<std::pair<size_t, long long>> slot_fix_ts;     // GemmTask B = slot
  std::vector<std::pair<size_t, long long>> scr_fix_trtri;   // TileTask L = inv_scratch offset
  std::vector<std::pair<size_t, long long>> scr_fix_g;       // GemmTask B = inv_scratch offset
  for (int l = 0; l < L; ++l) {
    int max_s = 0;
    for (int i = fp.level_ptr[l]; i < fp.level_ptr[l + 1]; ++i)
      max_s = std::max(max_s, fp.sep_size[fp.level_list[i]]);
    for (int k = 0; k < max_s; k += kTile) {
      Ref r{l, false, potrf_all.size(), trtri_all.size(), ts_all.size(), g_all.size(), 0, 0, 0, 0, 0, 0, 0, 0};
      size_t slot = 0;
      for (int i = fp.level_ptr[l]; i < fp.level_ptr[l + 1]; ++i) {
        const int nd = fp.level_list[i];
        const int s = fp.sep_size[nd], f = s + fp.bnd_size[nd], ld = fp.ld[nd];
        if (s <= k) continue;
        double* F = fp.d.fronts + fp.front_off[nd];
        const int nb = std::min(kTile, s - k), rest = f - k - nb;
        TileTask t{};
        t.L = F + k + (long long)k * ld; t.n = nb; t.ldl = ld; t.id = nd; t.offset = fp.sep_start[nd] + k;
        potrf_all.push_back(t);
        if (rest > 0) {
          slot_fix_trtri.push_back({trtri_all.size(), (long long)slot});
          trtri_all.push_back(t);
          GemmTask ts{};
          ts.A = F + (k + nb) + (long long)k * ld; ts.lda = ld;
          ts.ldb = kTile;
          ts.C = F + (k + nb) + (long long)k * ld; ts.ldc = ld;
          ts.M = rest; ts.N = nb; ts.K = nb;
          slot_fix_ts.push_back({ts_all.size(), (long long)slot});
          ts_all.push_back(ts);
          r.tsM = std::max(r.tsM, rest); r.tsN = std::max(r.tsN, nb);
          ++slot;
          GemmTask g{};
          g.A = F + (k + nb) + (long long)k * ld; g.lda = ld;
          g.B = g.A; g.ldb = ld;
          g.C = F + (k + nb) + (long long)(k + nb) * ld; g.ldc = ld;
          g.M = rest; g.N = rest; g.K = nb;
          g_all.push_back(g);
          r.gM = std::max(r.gM, rest); r.gN = std::max(r.gN, rest);
        }
      }
      max_slots = std::max(max_slots, slot);
      r.np = (int)(potrf_all.size() - r.p0); r.nr = (int)(trtri_all.size() - r.r0);
      r.nt = (int)(ts_all.size() - r.t0); r.ng = (int)(g_all.size() - r.g0);
      refs.push_back(r);
    }
    // partitioned inverse of this level
    prep_off[l] = prep_all.size();
    long long scr = 0;
    int max_np = 0;
    for (int i = fp.level_ptr[l]; i < fp.level_ptr[l + 1]; ++i) {
      const int nd = fp.level_list[i];
      const int sz = fp.sep_size[nd];
      if (sz <= 0) continue;
      const int lds = (int)round_up(sz, 2);
      scr_of[nd] = scr;
      lds_of[nd] = lds;
      prep_all.push_back(InvTask{nd, scr, lds});
      scr += round_up((long long)lds * sz, 2);
      max_np = std::max(max_np, ceil_div(sz, kTile));
    }
    scr_max = std::max(scr_max, scr);
    for (int t = 0; t < max_np; ++t) {
      Ref r{l, true, potrf_all.size(), trtri_all.size(), ts_all.size(), g_all.size(), 0, 0, 0, 0, 0, 0, 0, 0};
      size_t slot = 0;
      for (int i = fp.level_ptr[l]; i < fp.level_ptr[l + 1]; ++i) {
        const int nd = fp.level_list[i];
        const int sz = fp.sep_size[nd];
        const int np = ceil_div(sz, kTile);
        if (t >= np) continue;
        const int kb = np - 1 - t, k = kb * kTile, nb = std::min(kTile, sz - k);
        const int f = sz + fp.bnd_size[nd], ld = fp.ld[nd], lds = lds_of[nd];
        double* F = fp.d.fronts + fp.front_off[nd];
        TileTask tt{};
        tt.n = nb; tt.ldl = lds; tt.id = nd;
        scr_fix_trtri.push_back({trtri_all.size(), scr_of[nd] + k + (long long)k * lds});
        slot_fix_trtri.push_back({trtri_all.size(), (long long)slot});
        trtri_all.push_back(tt);
        GemmTask ts{};
        ts.A = F + (long long)k * ld; ts.lda = ld;
        ts.ldb = kTile;
        ts.C = F + (long long)k * ld; ts.ldc = ld;
        ts.M = f; ts.N = nb; ts.K = nb;
        slot_fix_ts.push_back({ts_all.size(), (long long)slot});
        ts_all.push_back(ts);
        r.tsM = std::max(r.tsM, f); r.tsN = std::max(r.tsN, nb);
        ++slot;
        if (k > 0) {
          GemmTask g{};
          g.A = F + (long long)k * ld; g.lda = ld;
          g.ldb = lds;
          g.C = F; g.ldc = ld;
          g.M = f; g.N = k; g.K = nb;
          scr_fix_g.push_back({g_all.size(), scr_of[nd] + k});
          g_all.push_back(g);
          r.gM = std::max(r.gM, f); r.gN = std::max(r.gN, k);
        }
      }
      max_slots = std::max(max_slots, slot);
      r.np = 0; r.nr = (int)(trtri_all.size() - r.r0);
      r.nt = (int)(ts_all.size() - r.t0); r.ng = (int)(g_all.size() - r.g0);
      refs.push_back(r);
    }
  }
  prep_off[L] = prep_all.size();
  ls.inv_scratch = c.alloc<double>(std::max<long long>(scr_max, 2));
  ls.tile_scratch = c.alloc<double>(max_slots * IS);
  for (auto& pr : slot_fix_trtri) trtri_all[pr.first].inv = ls.tile_scratch + pr.second * IS;
  for (auto& pr : slot_fix_ts) ts_all[pr.first].B = ls.tile_scratch + pr.second * IS;
  for (auto& pr : scr_fix_trtri) trtri_all[pr.first].L = ls.inv_scratch + pr.second;
  for (auto& pr : scr_fix_g) g_all[pr.first].B = ls.inv_scratch + pr.second;
  TileTask* dp = c.upload<TileTask>(potrf_all.data(), potrf_all.size());
  TileTask* dr = c.upload<TileTask>(trtri_all.data(), trtri_all.size());
  GemmTask* dt = c.upload<GemmTask>(ts_all.data(), ts_all.size());
  GemmTask* dg = c.upload<GemmTask>(g_all.data(), g_all.size());
  ls.inv_steps.assign(L, {});
  ls.inv_prep.assign(L, nullptr);
  ls.n_inv_prep.assign(L, 0);
  for (const Ref& r : refs) {
    LevelSchedule::Step st;
    st.potrf = dp + r.p0; st.n_potrf = r.np;
    st.trtri = dr + r.r0; st.n_trtri = r.nr;
    st.tsolve = dt + r.t0; st.n_tsolve = r.nt; st.ts_M = r.tsM; st.ts_N = r.tsN;
    st.gemm = dg + r.g0; st.n_gemm = r.ng; st.g_M = r.gM; st.g_N = r.gN;
    (r.inv ? ls.inv_steps : ls.steps)[r.l].push_back(st);
  }
  InvTask* dprep = c.upload<InvTask>(prep_all.data(), prep_all.size());
  for (int l = 0; l < L; ++l) {
    ls.inv_prep[l] = dprep + prep_off[l];
    ls.n_inv_prep[l] = (int)(prep_off[l + 1] - prep_off[l]);
  }
  // ---- solve plan: GEMV tiles + reductions per level, gather maps ----
  ls.fwd_t.assign(L, nullptr); ls.bwd_t.assign(L, nullptr);
  ls.fwd_r.assign(L, nullptr); ls.bwd_r.assign(L, nullptr);
  ls.n_fwd_t.assign(L, 0); ls.n_bwd_t.assign(L, 0); ls.n_fwd_r.assign(L, 0); ls.n_bwd_r.assign(L, 0);
  std::vector<CsTask> ft, bt;
  std::vector<CsRed> fr, br;
  std::vector<size_t> ft_off(L + 1), bt_off(L + 1), fr_off(L + 1), br_off(L + 1);
  int max_parts = 0;
  for (int l = 0; l < L; ++l) {
    ft_off[l] = ft.size(); bt_off[l] = bt.size(); fr_off[l] = fr.size(); br_off[l] = br.size();
    int pf = 0, pb = 0;
    for (int i = fp.level_ptr[l]; i < fp.level_ptr[l + 1]; ++i) {
      const int nd = fp.level_list[i];
      const int sz = fp.sep_size[nd], f = sz + fp.bnd_size[nd];
      for (int r0 = 0; r0 < f; r0 += 64) {
        const int p0 = pf;
        int cnt = 0;
        for (int c0 = 0; c0 < sz; c0 += 256) {
          if (r0 < sz && c0 > r0 + 63) break;  // above the lower-triangular L11^{-1}
          ft.push_back(CsTask{nd, r0, c0, pf++, (int)fr.size()});
          ++cnt;
        }
        fr.push_back(CsRed{nd, r0, p0, cnt});
      }
      for (int c0 = 0; c0 < sz; c0 += 64) {
        const int p0 = pb;
        int cnt = 0;
        for (int r0 = (c0 / 256) * 256; r0 < f; r0 += 256) {
          bt.push_back(CsTask{nd, r0, c0, pb++, (int)br.size()});
          ++cnt;
        }
        br.push_back(CsRed{nd, c0, p0, cnt});
      }
    }
    max_parts = std::max(max_parts, std::max(pf, pb));
  }
  ft_off[L] = ft.size(); bt_off[L] = bt.size(); fr_off[L] = fr.size(); br_off[L] = br.size();
  CsTask* dft = c.upload<CsTask>(ft.data(), ft.size());
  CsTask* dbt = c.upload<CsTask>(bt.data(), bt.size());
  CsRed* dfr = c.upload<CsRed>(fr.data(), fr.size());
  CsRed* dbr = c.upload<CsRed>(br.data(), br.size());
  for (int l = 0; l < L; ++l) {
    ls.fwd_t[l] = dft + ft_off[l]; ls.n_fwd_t[l] = (int)(ft_off[l + 1] - ft_off[l]);
    ls.bwd_t[l] = dbt + bt_off[l]; ls.n_bwd_t[l] = (int)(bt_off[l + 1] - bt_off[l]);
    ls.fwd_r[l] = dfr + fr_off[l]; ls.n_fwd_r[l] = (int)(fr_off[l + 1] - fr_off[l]);
    ls.bwd_r[l] = dbr + br_off[l]; ls.n_bwd_r[l] = (int)(br_off[l + 1] - br_off[l]);
  }
  ls.partial = c.alloc<double>((size_t)std::max(max_parts, 1) * 64);
  ls.ybuf = c.alloc<double>((size_t)std::max(fp.n_coarse, 1));
  ls.red_cnt = c.alloc<int>(fr.size() + br.size() + 1);
  BDDC_CUDA(cudaMemset(ls.red_cnt, 0, sizeof(int) * (fr.size() + br.size() + 1)));
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
  ls.gat_ptr = c.upload<int>(gptr.data(), gptr.size());
  ls.gat_off = c.upload<long long>(goff.data(), goff.size());
  ls.gat_src = c.upload<int>(gsrc.data(), std::max<size_t>(gsrc.size(), 1));
  coop_build(c);
}

void coarse_assemble_and_factor(Ctx& c) {
  FrontPlan& fp = c.fp;
  FrontDev& fd = fp.d;
  if (fp.n_coarse == 0) return;
  cudaStream_t s = c.stream;
  LevelSchedule& ls = c.sched;
  PhaseScope ps(c.prof, "setup.coarse", s);
  const int th = 256;
  { csr_segsum_kernel<<<std::min<long long>((fp.nnz + th - 1) / th, 148 * 16), th, 0, s>>>(
      fp.nnz, fp.seg_ptr, fp.contrib, c.Sloc, fp.csr_val); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
  BDDC_CUDA(cudaMemsetAsync(fd.fronts, 0, sizeof(double) * fp.front_pool, s));
  { csr_to_front_kernel<<<std::min<long long>((fp.nnz + th - 1) / th, 148 * 16), th, 0, s>>>(
      fp.nnz, fp.csr_front_pos, fp.csr_val, fd.fronts); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
  // multifrontal factorization + partitioned inverse: one cooperative launch
  coop_factor(c, s);
}

void coarse_solve(Ctx& c, const double* rhs, double* sol, cudaStream_t s) {
  coop_solve(c, rhs, sol, s);
}

}  // namespace bddc
