// Coarse problem: CSR assembly of S_0 = sum_i R_i^T (Psi_i^T A_i Psi_i) R_i by a segmented
// (deterministic, atomic-free) sum, then a multifrontal Cholesky over a geometric
// nested-dissection tree of the subdomain lattice, and the forward/backward solves.
// Replaces bddc.py:494-511 (COO -> CSR -> SuperLU spd_factor) and the coarse solve of
// bddc.py:362-364.
#include <algorithm>
#include <climits>

#include "bddc_internal.cuh"
#include "trsv.cuh"

namespace bddc {

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

// Forward solve of one level: v = [rhs(sep); 0] + sum_children ext(upd_c);
// y = L11^{-1} v_sep; v_bnd -= L21 y; sol(sep) = y; upd_node = v_bnd.
__global__ void front_fwd_kernel(const int* __restrict__ nodes, FrontDev fd,
                                 const double* __restrict__ rhs, double* __restrict__ sol) {
  extern __shared__ double sm[];
  double* dblk = sm;
  double* v = sm + kTrsvB * kTrsvP;
  const int node = nodes[blockIdx.x];
  const int s = fd.sep_size[node], b = fd.bnd_size[node], f = s + b;
  const int s0 = fd.sep_start[node];
  for (int i = threadIdx.x; i < f; i += blockDim.x) v[i] = i < s ? rhs[s0 + i] : 0.0;
  __syncthreads();
  const int c0 = fd.child_ptr[node], c1 = fd.child_ptr[node + 1];
  for (int c = c0; c < c1; ++c) {
    const int ch = fd.child_list[c];
    const int bc = fd.bnd_size[ch];
    const int* rm = fd.rmap + fd.rmap_ptr[ch];
    const double* u = fd.upd + fd.upd_off[ch];
    for (int i = threadIdx.x; i < bc; i += blockDim.x) v[rm[i]] += u[i];
    __syncthreads();
  }
  const double* F = fd.fronts + fd.front_off[node];
  cta_trsv_fwd(F, fd.ld[node], f, s, v, dblk);
  for (int i = threadIdx.x; i < f; i += blockDim.x) {
    if (i < s) sol[s0 + i] = v[i];
    else fd.upd[fd.upd_off[node] + (i - s)] = v[i];
  }
}

// Backward solve of one level: x_sep = L11^{-T} (y - L21^T x_bnd).
__global__ void front_bwd_kernel(const int* __restrict__ nodes, FrontDev fd, double* __restrict__ sol) {
  extern __shared__ double sm[];
  double* dblk = sm;
  double* v = sm + kTrsvB * kTrsvP;
  const int node = nodes[blockIdx.x];
  const int s = fd.sep_size[node], b = fd.bnd_size[node], f = s + b;
  const int s0 = fd.sep_start[node];
  const int* bidx = fd.bnd_idx + fd.bnd_ptr[node];
  for (int i = threadIdx.x; i < f; i += blockDim.x) v[i] = i < s ? sol[s0 + i] : sol[bidx[i - s]];
  __syncthreads();
  const double* F = fd.fronts + fd.front_off[node];
  cta_trsv_bwd(F, fd.ld[node], f, s, v, dblk);
  for (int i = threadIdx.x; i < s; i += blockDim.x) sol[s0 + i] = v[i];
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
  std::vector<TileTask> potrf_all, trsm_all;
  std::vector<GemmTask> gemm_all;
  struct Ref { int l, k; size_t p0, t0, g0; int np, nt, ng, mt, mg; };
  std::vector<Ref> refs;
  for (int l = 0; l < L; ++l) {
    int max_s = 0;
    for (int i = fp.level_ptr[l]; i < fp.level_ptr[l + 1]; ++i)
      max_s = std::max(max_s, fp.sep_size[fp.level_list[i]]);
    for (int k = 0; k < max_s; k += kTile) {
      Ref r{l, k, potrf_all.size(), trsm_all.size(), gemm_all.size(), 0, 0, 0, 0, 0};
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
          TileTask tt = t;
          tt.B = F + (k + nb) + (long long)k * ld; tt.ldb = ld; tt.nvec = rest;
          trsm_all.push_back(tt);
          r.mt = std::max(r.mt, rest);
          GemmTask g{};
          g.A = F + (k + nb) + (long long)k * ld; g.lda = ld;
          g.B = g.A; g.ldb = ld;
          g.C = F + (k + nb) + (long long)(k + nb) * ld; g.ldc = ld;
          g.M = rest; g.N = rest; g.K = nb;
          gemm_all.push_back(g);
          r.mg = std::max(r.mg, rest);
        }
      }
      r.np = (int)(potrf_all.size() - r.p0);
      r.nt = (int)(trsm_all.size() - r.t0);
      r.ng = (int)(gemm_all.size() - r.g0);
      refs.push_back(r);
    }
  }
  TileTask* dp = c.upload<TileTask>(potrf_all.data(), potrf_all.size());
  TileTask* dt = c.upload<TileTask>(trsm_all.data(), trsm_all.size());
  GemmTask* dg = c.upload<GemmTask>(gemm_all.data(), gemm_all.size());
  for (const Ref& r : refs) {
    LevelSchedule::Step st;
    st.potrf = dp + r.p0; st.n_potrf = r.np;
    st.trsm = dt + r.t0; st.n_trsm = r.nt; st.max_trsm = r.mt;
    st.gemm = dg + r.g0; st.n_gemm = r.ng; st.max_gemm = r.mg;
    ls.steps[r.l].push_back(st);
  }
  ls.max_fwd_smem = sizeof(double) * ((size_t)kTrsvB * kTrsvP + fp.max_front);
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
  for (int l = 0; l < fp.nlevels; ++l) {
    const int nn = ls.nodes_off[l + 1] - ls.nodes_off[l];
    const int* nodes = ls.d_nodes + ls.nodes_off[l];
    if (l > 0) {
      for (int k = 0; k < ls.max_children; ++k) {
        dim3 grid(64, nn);
        { extend_add_kernel<<<grid, 256, 0, s>>>(nodes, k, fd.child_ptr, fd.child_list,
                                               fd.sep_size, fd.bnd_size, fd.ld,
                                               fd.front_off, fd.rmap, fd.rmap_ptr, fd.fronts); BDDC_COUNT(); }
        BDDC_LAUNCH_CHECK();
      }
    }
    for (const auto& st : ls.steps[l]) {
      TileArgs pa;
      pa.tasks = st.potrf; pa.count = st.n_potrf; pa.info = fp.info;
      potrf_tile(pa, s);
      if (st.n_trsm) {
        TileArgs ta;
        ta.tasks = st.trsm; ta.count = st.n_trsm; ta.max_nvec = st.max_trsm;
        trsm_tile(ta, TRSM_RLT, s);
      }
      if (st.n_gemm) {
        GemmArgs ga;
        ga.tasks = st.gemm; ga.count = st.n_gemm; ga.max_M = st.max_gemm; ga.max_N = st.max_gemm;
        ga.alpha = -1.0; ga.beta = 1.0; ga.lower = 1;
        gemm(ga, false, true, s);
      }
    }
  }
}

void coarse_solve(Ctx& c, const double* rhs, double* sol, cudaStream_t s) {
  FrontPlan& fp = c.fp;
  FrontDev& fd = fp.d;
  LevelSchedule& ls = c.sched;
  const size_t smem = ls.max_fwd_smem;
  static size_t attr = 0;
  if (smem > attr) {
    BDDC_CUDA(cudaFuncSetAttribute(front_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    BDDC_CUDA(cudaFuncSetAttribute(front_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  for (int l = 0; l < fp.nlevels; ++l) {
    const int nn = ls.nodes_off[l + 1] - ls.nodes_off[l];
    { front_fwd_kernel<<<nn, 256, smem, s>>>(ls.d_nodes + ls.nodes_off[l], fd, rhs, sol); BDDC_COUNT(); }
    BDDC_LAUNCH_CHECK();
  }
  for (int l = fp.nlevels - 1; l >= 0; --l) {
    const int nn = ls.nodes_off[l + 1] - ls.nodes_off[l];
    { front_bwd_kernel<<<nn, 256, smem, s>>>(ls.d_nodes + ls.nodes_off[l], fd, sol); BDDC_COUNT(); }
    BDDC_LAUNCH_CHECK();
  }
}

}  // namespace bddc
