// Per-subdomain setup (the batched half of build_bddc, bddc.py:419-492).
//
// For every subdomain i (all at once, in chunks that fit the workspace):
//   1. assemble the local Neumann pieces from alpha (bddc.py:427): block-tridiagonal A_II,
//      dense A_I,Gamma (into E), dense A_Gamma,Gamma (into LS), s_i = mean|diag A_i|
//   2. block-tridiagonal Cholesky of A_II (interior factor, bddc.py:436-440)
//   3. E = L_I^{-1} A_I,Gamma;  S_Gamma = A_GammaGamma - E^T E  (DMMA GEMM)
//   4. S_K = S_Gamma + s_i C^T C, Cholesky (replaces the KKT LU of linalg.py:175-208;
//      same constrained solution because C u = 0 there)
//   5. G = L_S^{-1} C^T, S_C = G^T G, Phi = L_S^{-T} G S_C^{-1}  (energy-minimal basis,
//      C Phi = I);  Psi = c_i Phi with c_i = 1/s_i^2 ("reference", reproducing
//      linalg.py:165-171 + bddc.py:457) or 1 ("spec")
//   6. local coarse block c_i^2 * sym(Phi^T S_Gamma Phi)  (= Psi^T A Psi, bddc.py:464-466)
#include "stencil.cuh"

namespace bddc {

bool schur2d_supported(const Geometry& G);
bool schur2d(const Ctx& c, int sub0, int cnt, const double* Wd, const double* Wo, const double* E,
             cudaStream_t s);
bool schur3d_supported(const Geometry& G);
void schur3d(const Ctx& c, int sub0, int cnt, double* Rt, double* Ht, long long sE, int* klo,
             cudaStream_t s);

namespace {

// DENSE: also write the interior blocks T_j / B_j and A_IG densely (generic path); the fused
// 2D path generates them from the stencil on chip and only needs A_GG and s_i here.
// ADD (fused 3D): A_GG is added to LS, which already holds -R~^T H~ (no memset of LS).
// AGG = false (fused 2D): s_i only; the Schur kernel generates A_GG in its epilogue.
template <int DIM, bool DENSE, bool ADD = false, bool AGG = true>
__global__ void __launch_bounds__(256) assemble_local_kernel(Geometry G, const double* __restrict__ alpha,
                                                             LocalTables lt, int sub0, double* Wd,
                                                             double* Wo, double* E, double* LS,
                                                             double* diag_s) {
  const int sub = sub0 + blockIdx.x;
  const long long b = blockIdx.x;
  int p[3];
  sub_coords(G, sub, p);
  const long long mm = (long long)G.m_pad * G.m_pad;
  double* wd = Wd + b * G.nblk * mm;
  double* wo = Wo + b * G.nblk * mm;
  double* e = E + b * (long long)G.nI_pad * G.nG_pad;
  double* ls = LS + (long long)sub * G.nG_pad * G.nG_pad;
  constexpr int NOFF = DIM == 3 ? 27 : 9;
  double dsum = 0.0;
  int nfree_loc = 0;
  if (!DENSE) {
    // A_GG only: the couplings of the surface slots among themselves, then the diagonal of
    // every local node for s_i (interior couplings are generated on chip by the fused kernels)
    const int tot1 = AGG ? G.nG * NOFF : 0;
    for (int idx = threadIdx.x; idx < tot1 + G.nloc_nodes; idx += blockDim.x) {
      if (idx < tot1) {
        const int slot = idx / NOFF, o = idx % NOFF;
        const int node = lt.slot_node[slot];
        int a[3], d[3] = {o % 3 - 1, (o / 3) % 3 - 1, DIM == 3 ? o / 9 - 1 : 0};
        local_coords(G, node, a);
        const int bn[3] = {a[0] + d[0], a[1] + d[1], a[2] + d[2]};
        if (bn[0] < 0 || bn[0] > G.blk[0] || bn[1] < 0 || bn[1] > G.blk[1]) continue;
        if (DIM == 3 && (bn[2] < 0 || bn[2] > G.blk[2])) continue;
        const int nb = bn[0] + (G.blk[0] + 1) * (bn[1] + (G.blk[1] + 1) * bn[2]);
        const int cb = lt.node_code[nb];
        if (cb >= 0) continue;  // interior neighbour: A_IG, generated on chip
        const long long pos = slot + (long long)(-cb - 1) * G.nG_pad;
        if (local_to_free(G, p, a) < 0 || local_to_free(G, p, bn) < 0) {
          if (node == nb) {
            if (ADD) ls[pos] += 1.0;
            else ls[pos] = 1.0;
          }
          continue;
        }
        const double v = local_coef<DIM>(G, alpha, p, a, d);
        if (ADD) ls[pos] += v;
        else ls[pos] = v;
      } else {
        const int node = idx - tot1;
        int a[3];
        local_coords(G, node, a);
        if (local_to_free(G, p, a) < 0) continue;
        const int d0[3] = {0, 0, 0};
        dsum += fabs(local_coef<DIM>(G, alpha, p, a, d0));
        nfree_loc += 1;
      }
    }
  }
  const int total = DENSE ? G.nloc_nodes * NOFF : 0;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int node = idx / NOFF, o = idx % NOFF;
    int a[3], d[3] = {o % 3 - 1, (o / 3) % 3 - 1, DIM == 3 ? o / 9 - 1 : 0};
    local_coords(G, node, a);
    int bn[3] = {a[0] + d[0], a[1] + d[1], a[2] + d[2]};
    if (bn[0] < 0 || bn[0] > G.blk[0] || bn[1] < 0 || bn[1] > G.blk[1]) continue;
    if (DIM == 3 && (bn[2] < 0 || bn[2] > G.blk[2])) continue;
    const int nb = bn[0] + (G.blk[0] + 1) * (bn[1] + (G.blk[1] + 1) * bn[2]);
    const bool dir_a = local_to_free(G, p, a) < 0;
    const bool dir_b = local_to_free(G, p, bn) < 0;
    const int ca = lt.node_code[node], cb = lt.node_code[nb];
    if (dir_a || dir_b) {
      if (node == nb && ca < 0) {
        const int s = -ca - 1;
        if (ADD) ls[s + (long long)s * G.nG_pad] += 1.0;
        else ls[s + (long long)s * G.nG_pad] = 1.0;
      }
      continue;
    }
    const double v = local_coef<DIM>(G, alpha, p, a, d);
    if (node == nb) {
      dsum += fabs(v);
      nfree_loc += 1;
    }
    if (!DENSE) {
      if (ca < 0 && cb < 0) {
        if (ADD) ls[(-ca - 1) + (long long)(-cb - 1) * G.nG_pad] += v;
        else ls[(-ca - 1) + (long long)(-cb - 1) * G.nG_pad] = v;
      }
      continue;
    }
    if (ca >= 0 && cb >= 0) {
      const int ja = ca / G.m_pad, jb = cb / G.m_pad, ra = ca % G.m_pad, rb = cb % G.m_pad;
      if (ja == jb) wd[ja * mm + ra + (long long)rb * G.m_pad] = v;
      else if (ja == jb + 1) wo[ja * mm + ra + (long long)rb * G.m_pad] = v;
    } else if (ca >= 0 && cb < 0) {
      e[ca + (long long)(-cb - 1) * G.nI_pad] = v;
    } else if (ca < 0 && cb < 0) {
      ls[(-ca - 1) + (long long)(-cb - 1) * G.nG_pad] = v;
    }
  }
  // identity on padding
  for (int idx = threadIdx.x; DENSE && idx < G.nblk * (G.m_pad - G.m); idx += blockDim.x) {
    const int j = idx / (G.m_pad - G.m), r = G.m + idx % (G.m_pad - G.m);
    wd[j * mm + r + (long long)r * G.m_pad] = 1.0;
  }
  for (int s = G.nG + threadIdx.x; AGG && s < G.nG_pad; s += blockDim.x) {
    if (ADD) ls[s + (long long)s * G.nG_pad] += 1.0;
    else ls[s + (long long)s * G.nG_pad] = 1.0;
  }
  // s_i = mean |diag A_i| over local free nodes
  __shared__ double red[256];
  __shared__ int cnt[256];
  red[threadIdx.x] = dsum;
  cnt[threadIdx.x] = nfree_loc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      red[threadIdx.x] += red[threadIdx.x + w];
      cnt[threadIdx.x] += cnt[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) diag_s[sub] = cnt[0] ? red[0] / cnt[0] : 1.0;
}

// Block-tridiagonal Cholesky of A_II, one CTA per subdomain (blocks of m_pad <= 64):
//   Lo_j = B_j Linv_{j-1}^T ;  Ld_j = chol(T_j - Lo_j Lo_j^T) ;  Linv_j = Ld_j^{-1}
// In: T_j in Wd[j], B_j in Wo[j] (dense m_pad^2, setup workspace).
// Out: Linv_j dense in Wd[j], Lo_j dense in Wo[j] (workspace, for E = L^{-1} A_IG),
//      Linv_j packed + the coupling stencil Bc_j in LI (persistent, for the apply).
__global__ void __launch_bounds__(128) btchol_kernel(Geometry G, int sub0, double* Wd, double* Wo,
                                                     double* LI, int* info) {
  extern __shared__ double sm[];
  const int M = G.m_pad, P = M + 1;  // odd pitch
  double* prev = sm;          // Linv_{j-1}
  double* cur = sm + M * P;   // S_j -> Ld_j
  double* off = sm + 2 * M * P;
  double* inv = sm + 3 * M * P;
  const int b = blockIdx.x, sub = sub0 + b;
  const long long mm = (long long)M * M;
  double* wd = Wd + (long long)b * G.nblk * mm;
  double* wo = Wo + (long long)b * G.nblk * mm;
  double* li = LI + (long long)sub * G.li_stride;
  double* bc = li + (long long)G.nblk * G.Tm;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int px = G.blk[0] - 1;  // in-plane row length
  const int py = G.dim == 3 ? G.blk[1] - 1 : 1;
  __shared__ int failed;
  if (tid == 0) failed = -1;
  for (int j = 0; j < G.nblk; ++j) {
    for (int idx = tid; idx < M * M; idx += nt) cur[idx % M + (idx / M) * P] = wd[j * mm + idx];
    if (j > 0)
      for (int idx = tid; idx < M * M; idx += nt) off[idx % M + (idx / M) * P] = wo[j * mm + idx];
    __syncthreads();
    if (j > 0) {
      // coupling stencil of B_j (rows: plane j, cols: plane j-1) before it is overwritten
      for (int idx = tid; idx < M * G.nbo; idx += nt) {
        const int r = idx / G.nbo, k = idx % G.nbo;
        double v = 0.0;
        if (r < G.m) {
          const int x = r % px + G.bo_dx[k], y = r / px + G.bo_dy[k];
          if (x >= 0 && x < px && y >= 0 && y < py) v = off[r + (x + y * px) * P];
        }
        bc[((long long)j * M + r) * G.nbo + k] = v;
      }
      // off <- B_j Linv_{j-1}^T  (row r: sum_k B[r][k] Linv[c][k], k <= c)
      for (int idx = tid; idx < M * M; idx += nt) {
        const int r = idx % M, c = idx / M;
        double acc = 0.0;
        for (int k = 0; k <= c; ++k) acc += off[r + k * P] * prev[c + k * P];
        inv[r + c * P] = acc;
      }
      __syncthreads();
      for (int idx = tid; idx < M * M; idx += nt) off[idx % M + (idx / M) * P] = inv[idx % M + (idx / M) * P];
      __syncthreads();
      // cur -= off off^T (lower)
      for (int idx = tid; idx < M * M; idx += nt) {
        const int r = idx % M, c = idx / M;
        if (r < c) continue;
        double acc = 0.0;
        for (int k = 0; k < M; ++k) acc += off[r + k * P] * off[c + k * P];
        cur[r + c * P] -= acc;
      }
      __syncthreads();
    } else {
      for (int idx = tid; idx < M * G.nbo; idx += nt) bc[idx] = 0.0;
    }
    // Cholesky of cur (lower), right-looking in shared memory
    for (int c = 0; c < M; ++c) {
      if (tid == 0) {
        double d = cur[c + c * P];
        if (!(d > 0.0)) {
          if (failed < 0) failed = j * M + c;
          d = 1.0;
        }
        cur[c + c * P] = sqrt(d);
      }
      __syncthreads();
      const double iv = 1.0 / cur[c + c * P];
      for (int r = c + 1 + tid; r < M; r += nt) cur[r + c * P] *= iv;
      __syncthreads();
      const int rr = M - c - 1;
      for (int idx = tid; idx < rr * rr; idx += nt) {
        const int i = c + 1 + idx % rr, k = c + 1 + idx / rr;
        if (i >= k) cur[i + k * P] -= cur[i + c * P] * cur[k + c * P];
      }
      __syncthreads();
    }
    // inv = cur^{-1}: thread per column c, forward substitution down the column
    for (int c = tid; c < M; c += nt) {
      for (int i = 0; i < c; ++i) inv[i + c * P] = 0.0;
      for (int i = c; i < M; ++i) {
        double acc = i == c ? 1.0 : 0.0;
        for (int k = c; k < i; ++k) acc -= cur[i + k * P] * inv[k + c * P];
        inv[i + c * P] = acc / cur[i + i * P];
      }
    }
    __syncthreads();
    // outputs: packed W_j = S_j^{-1} = Linv^T Linv (apply), dense Linv / Lo (workspace)
    double* pk = li + (long long)j * G.Tm;
    for (int c = 0; c < M; ++c) {
      const long long cs = (long long)c * M - (long long)c * (c - 1) / 2;  // packed column start
      for (int r = c + tid; r < M; r += nt) {
        double a = 0.0;
        for (int k = r; k < M; ++k) a += inv[k + r * P] * inv[k + c * P];
        pk[cs + (r - c)] = a;
      }
    }
    for (int idx = tid; idx < M * M; idx += nt) {
      const int r = idx % M, c = idx / M;
      wd[j * mm + idx] = inv[r + c * P];
      if (j > 0) wo[j * mm + idx] = off[r + c * P];
    }
    __syncthreads();
    double* t = prev;
    prev = inv;
    inv = t;
  }
  if (tid == 0 && failed >= 0) atomicMin(info + sub, failed);
}

// S += s_i C^T C (one CTA per subdomain): entries of slots sharing a constraint.
__global__ void add_ctc_kernel(Geometry G, int sub0, SubTables st, const double* diag_s, double* LS) {
  const int sub = sub0 + blockIdx.x;
  __shared__ int con[1024];
  __shared__ double coef[1024];
  for (int s = threadIdx.x; s < G.nG_pad; s += blockDim.x) {
    con[s] = st.slot_con[(long long)sub * G.nG_pad + s];
    coef[s] = st.slot_coef[(long long)sub * G.nG_pad + s];
  }
  __syncthreads();
  const double rho = diag_s[sub];
  double* ls = LS + (long long)sub * G.nG_pad * G.nG_pad;
  for (int a = threadIdx.x; a < G.nG_pad; a += blockDim.x) {
    const int ka = con[a];
    if (ka < 0) continue;
    for (int b = 0; b < G.nG_pad; ++b)
      if (con[b] == ka) ls[a + (long long)b * G.nG_pad] += rho * coef[a] * coef[b];
  }
}

// G = C^T (dense nG_pad x nc_pad)
__global__ void build_ct_kernel(Geometry G, int sub0, SubTables st, double* Gm) {
  const int sub = sub0 + blockIdx.x;
  double* g = Gm + (long long)sub * G.nG_pad * G.nc_pad;
  for (int s = threadIdx.x; s < G.nG_pad; s += blockDim.x) {
    const int k = st.slot_con[(long long)sub * G.nG_pad + s];
    if (k >= 0) g[s + (long long)k * G.nG_pad] = st.slot_coef[(long long)sub * G.nG_pad + s];
  }
}

// B = I (n x n, per batch entry)
__global__ void identity_kernel(double* B, int n, long long stride) {
  double* b = B + (long long)blockIdx.x * stride;
  for (long long idx = threadIdx.x; idx < (long long)n * n; idx += blockDim.x)
    b[idx] = (idx % n == idx / n) ? 1.0 : 0.0;
}

// G = L_S^{-1} C^T without a GEMM: C^T is one nonzero per constrained slot, so column k of
// G is the coefficient-weighted sum of the columns of L_S^{-1} at the slots of constraint k
// (ascending slot order: deterministic). Warp per constraint; lane owns rows lane + 32 r.
// LOWER: LIv is L^{-1} with only its diagonal 64-tiles' upper parts zeroed (the blocks above
// them are never written): column s is read from row 64 floor(s / 64) on.
template <int RPL, bool LOWER>
__global__ void __launch_bounds__(256) g_gather_kernel(Geometry G, int sub0, SubTables st,
                                                       const double* __restrict__ LIv, long long sL,
                                                       double* __restrict__ X, long long sX) {
  __shared__ int con[1024];
  __shared__ double cf[1024];
  const int b = blockIdx.x, sub = sub0 + b, n = G.nG_pad, nc = G.nc_pad;
  for (int s = threadIdx.x; s < n; s += blockDim.x) {
    con[s] = st.slot_con[(long long)sub * n + s];
    cf[s] = st.slot_coef[(long long)sub * n + s];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double* li = LIv + b * sL;
  double* x = X + b * sX;
  for (int k = warp; k < nc; k += nw) {
    double acc[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) acc[r] = 0.0;
    for (int s0 = 0; s0 < n; s0 += 32) {
      unsigned mask = __ballot_sync(0xffffffffu, s0 + lane < n && con[s0 + lane] == k);
      while (mask) {
        const int s = s0 + __ffs(mask) - 1;
        mask &= mask - 1;
        const double c = cf[s];
        const double* col = li + (long long)s * n;
        const int i0 = LOWER ? (s & ~63) : 0;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int i = lane + 32 * r;
          if (i < n && i >= i0) acc[r] += c * col[i];
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      if (i < n) x[i + (long long)k * n] = acc[r];
    }
  }
}

bool g_gather(const Geometry& G, int sub0, int cnt, const SubTables& st, const double* LIv, long long sL,
              double* X, long long sX, cudaStream_t s, bool lower) {
  const int rpl = ceil_div(G.nG_pad, 32);
#define BDDC_GG(R) \
  if (rpl <= R) { \
    if (lower) g_gather_kernel<R, true><<<cnt, 256, 0, s>>>(G, sub0, st, LIv, sL, X, sX); \
    else g_gather_kernel<R, false><<<cnt, 256, 0, s>>>(G, sub0, st, LIv, sL, X, sX); \
    BDDC_COUNT(); BDDC_LAUNCH_CHECK(); return true; }
  BDDC_GG(1) BDDC_GG(2) BDDC_GG(4) BDDC_GG(8) BDDC_GG(13) BDDC_GG(16)
#undef BDDC_GG
  return false;
}

// identity on padded constraints of S_C
__global__ void sc_pad_kernel(Geometry G, int sub0, SubTables st, double* SC) {
  const int b = blockIdx.x, sub = sub0 + b;
  double* sc = SC + (long long)b * G.nc_pad * G.nc_pad;
  for (int k = threadIdx.x; k < G.nc_pad; k += blockDim.x)
    if (st.con_coarse[(long long)sub * G.nc_pad + k] < 0) sc[k + (long long)k * G.nc_pad] = 1.0;
}

// Local coarse matrix P = Phi^T S_Gamma Phi without forming S_Gamma Phi: with
// S_K = S_Gamma + s C^T C, Phi = S_K^{-1} C^T S_C^{-1} and C Phi = I,
//   S_Gamma Phi = C^T S_C^{-1} - s C^T   =>   Phi^T S_Gamma Phi = S_C^{-1} - s I
// (zero on padded constraints, where Phi has zero columns). Then, as the reference scales
// it, Sloc = c^2 * 0.5 (P + P^T) with c = 1 / s^2 (or 1 with the spectral option); cscale = c.
__global__ void finish_local_kernel(Geometry G, int sub0, int spec, const double* diag_s, SubTables st,
                                    double* cscale, const double* SCi, double* Sloc) {
  const int b = blockIdx.x, sub = sub0 + b;
  const double s = diag_s[sub];
  const double c = spec ? 1.0 : 1.0 / (s * s);
  if (threadIdx.x == 0) cscale[sub] = c;
  const int n = G.nc_pad;
  const int* cc = st.con_coarse + (long long)sub * n;
  const double* pp = SCi + (long long)b * n * n;
  double* out = Sloc + (long long)sub * n * n;
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int i = idx % n, j = idx / n;
    double v = 0.0;
    if (cc[i] >= 0 && cc[j] >= 0) v = 0.5 * (pp[i + j * n] + pp[j + i * n]) - (i == j ? s : 0.0);
    out[idx] = (c * c) * v;
  }
}

}  // namespace

size_t local_setup_workspace(const Geometry& g, int chunk) {
  const size_t E = 2 * (size_t)g.nI_pad * g.nG_pad + 2 * (size_t)g.nblk * g.m_pad * g.m_pad;
  const size_t SG = (size_t)g.nG_pad * g.nG_pad;
  const size_t X = (size_t)g.nG_pad * g.nc_pad;
  const size_t SC = (size_t)g.nc_pad * g.nc_pad;
  return (size_t)chunk * (E + SG + 2 * X + 3 * SC);
}

void local_setup(Ctx& c, double* ws, size_t ws_doubles) {
  const Geometry& G = c.geo;
  cudaStream_t s = c.stream;
  const size_t per = local_setup_workspace(G, 1);
  int chunk = (int)std::min<size_t>(G.s_hi - G.s_lo, ws_doubles / per);
  if (chunk <= 0) throw CudaError("local setup workspace too small");
  const long long mm = (long long)G.m_pad * G.m_pad;
  const long long wS = (long long)G.nblk * mm;
  const long long lsS = (long long)G.nG_pad * G.nG_pad;
  const long long phS = (long long)G.nG_pad * G.nc_pad;
  const long long scS = (long long)G.nc_pad * G.nc_pad;
  const long long eS = (long long)G.nI_pad * G.nG_pad;
  const int btchol_smem = 4 * G.m_pad * (G.m_pad + 1) * (int)sizeof(double);
  BDDC_CUDA(cudaFuncSetAttribute(btchol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, btchol_smem));

  for (int sub0 = G.s_lo; sub0 < G.s_hi; sub0 += chunk) {  // this rank's subdomains
    const int cnt = std::min(chunk, G.s_hi - sub0);
    double* E = ws;                             // A_IG, then E - Lo E (in place)
    double* E2 = E + (size_t)chunk * eS;        // E = L_I^{-1} A_IG
    double* Wd = E2 + (size_t)chunk * eS;       // T_j -> Linv_j (dense)
    double* Wo = Wd + (size_t)chunk * wS;       // B_j -> Lo_j (dense)
    double* X = Wo + (size_t)chunk * wS;      // G = L^{-1} C^T, then V = L^{-T} Q
    double* SC = X + (size_t)chunk * phS;     // S_C -> L_C
    double* P = SC + (size_t)chunk * scS;     // L_C^{-1} (blocked path only)
    double* LIv = P + (size_t)chunk * scS;    // L_S^{-1}
    double* Y = LIv + (size_t)chunk * lsS;    // Q = G L_C^{-T}
    double* SCi = Y + (size_t)chunk * phS;    // S_C^{-1}
    double* LS = c.LS + sub0 * lsS;
    double* PH = c.Phi + sub0 * phS;
    const bool fused2d = G.nblk > 0 && schur2d_supported(G);
    const bool fused3d = G.nblk > 0 && !fused2d && schur3d_supported(G);
    if (!fused2d && !fused3d) {  // the fused kernels generate T_j, B_j and A_IG from the stencil
      BDDC_CUDA(cudaMemsetAsync(Wd, 0, sizeof(double) * 2 * (size_t)chunk * wS, s));
      BDDC_CUDA(cudaMemsetAsync(E, 0, sizeof(double) * cnt * eS, s));
    }
    if (!fused3d && !fused2d) BDDC_CUDA(cudaMemsetAsync(LS, 0, sizeof(double) * cnt * lsS, s));  // fused: every entry written
    BMat LSb{LS, lsS, G.nG_pad};
    if (fused3d) {
      // 3D: W recursion + per-chunk R_j / H_j, then S_G = A_GG - R~^T H~ as one staircase
      // GEMM (beta = 0, both triangles); A_GG is added by the assembly below
      PhaseScope ps(c.prof, "setup.schur", s);
      int klo[16];
      schur3d(c, sub0, cnt, E, E2, eS, klo, s);
      BMat Rb{E, eS, G.nI_pad}, Hb{E2, eS, G.nI_pad};
      gemm_batched(true, false, G.nG_pad, G.nG_pad, G.nI_pad, -1.0, Rb, Hb, 0.0, LSb, cnt, s, true, 0, true, klo);
    }
    // host-buffer path: alpha arrives in slabs; the 2D on-chip elimination of slab k starts as
    // soon as its cells have landed (assembly + W recursion + Schur kernels per slab)
    if (fused2d && c.alpha_nslab > 0 && sub0 == G.s_lo && cnt == G.s_hi - G.s_lo) {
      PhaseScope ps(c.prof, "setup.schur", s);
      for (int k = 0; k < c.alpha_nslab; ++k) {
        const int sa = std::max(sub0, c.alpha_slab_sub[k]), sb = std::min(sub0 + cnt, c.alpha_slab_sub[k + 1]);
        BDDC_CUDA(cudaStreamWaitEvent(s, c.alpha_ev[k], 0));
        if (sa >= sb) continue;
        { assemble_local_kernel<2, false, false, false><<<sb - sa, 256, 0, s>>>(G, c.alpha, c.lt, sa, Wd, Wo, E, c.LS, c.diag_s); BDDC_COUNT(); }
        BDDC_LAUNCH_CHECK();
        if (!schur2d(c, sa, sb - sa, Wd, Wo, E, s)) throw CudaError("schur2d: unsupported geometry");
      }
    } else {
    // 1. assembly
    c.prof.begin("setup.assemble", s);
    if (fused3d)
      { assemble_local_kernel<3, false, true><<<cnt, 256, 0, s>>>(G, c.alpha, c.lt, sub0, Wd, Wo, E, c.LS, c.diag_s); BDDC_COUNT(); }
    else if (G.dim == 2 && fused2d)
      { assemble_local_kernel<2, false, false, false><<<cnt, 256, 0, s>>>(G, c.alpha, c.lt, sub0, Wd, Wo, E, c.LS, c.diag_s); BDDC_COUNT(); }
    else if (G.dim == 2)
      { assemble_local_kernel<2, true><<<cnt, 256, 0, s>>>(G, c.alpha, c.lt, sub0, Wd, Wo, E, c.LS, c.diag_s); BDDC_COUNT(); }
    else
      { assemble_local_kernel<3, true><<<cnt, 256, 0, s>>>(G, c.alpha, c.lt, sub0, Wd, Wo, E, c.LS, c.diag_s); BDDC_COUNT(); }
    BDDC_LAUNCH_CHECK();
    c.prof.end("setup.assemble", s);
    // 2-3. fused on-chip interior elimination (2D) or the generic batched path
    bool fused = fused3d;
    if (fused2d) {
      c.prof.begin("setup.schur", s);
      fused = schur2d(c, sub0, cnt, Wd, Wo, E, s);
      c.prof.end("setup.schur", s);
    }
    if (!fused) {
    // 2. interior block-tridiagonal Cholesky (+ inverses of the diagonal blocks)
    c.prof.begin("setup.btchol", s);
    if (G.nblk > 0) {
      { btchol_kernel<<<cnt, 128, btchol_smem, s>>>(G, sub0, Wd, Wo, c.LI, c.info); BDDC_COUNT(); }
      BDDC_LAUNCH_CHECK();
    }
    c.prof.end("setup.btchol", s);
    // 3. E = L_I^{-1} A_IG:  E2_j = Linv_j (E_j - Lo_j E2_{j-1})
    c.prof.begin("setup.E", s);
    for (int j = 0; j < G.nblk; ++j) {
      BMat Ej{E + (long long)j * G.m_pad, eS, G.nI_pad};
      BMat E2j{E2 + (long long)j * G.m_pad, eS, G.nI_pad};
      if (j > 0) {
        BMat Lo{Wo + j * mm, wS, G.m_pad};
        BMat E2p{E2 + (long long)(j - 1) * G.m_pad, eS, G.nI_pad};
        gemm_batched(false, false, G.m_pad, G.nG_pad, G.m_pad, -1.0, Lo, E2p, 1.0, Ej, cnt, s);
      }
      BMat Li{Wd + j * mm, wS, G.m_pad};
      gemm_batched(false, false, G.m_pad, G.nG_pad, G.m_pad, 1.0, Li, Ej, 0.0, E2j, cnt, s);
    }
    c.prof.end("setup.E", s);
    // S_Gamma = A_GG - E^T E  (in LS)
    c.prof.begin("setup.SG", s);
    BMat Eb{E2, eS, G.nI_pad};
    gemm_batched(true, false, G.nG_pad, G.nG_pad, G.nI_pad, -1.0, Eb, Eb, 1.0, LSb, cnt, s);
    c.prof.end("setup.SG", s);
    }
    }  // alpha slabs
    // 4. S_K = S_Gamma + s C^T C; Cholesky
    c.prof.begin("setup.SK", s);
    { add_ctc_kernel<<<cnt, 128, 0, s>>>(G, sub0, c.st, c.diag_s, c.LS); BDDC_COUNT(); }
    BDDC_LAUNCH_CHECK();
    potrf_batched(LSb, G.nG_pad, G.nG_pad, cnt, c.info_k + sub0, c.tinv, s);
    c.prof.end("setup.SK", s);
    BMat LIb{LIv, lsS, G.nG_pad};
    {
      // 5a. L_S^{-1} (the diagonal-tile inverses are left in c.tinv by the factorization)
      PhaseScope pli(c.prof, "setup.Linv", s);
      if (!trtri_from_tiles(LSb, G.nG_pad, LIb, cnt, c.tinv, s)) {
        { identity_kernel<<<cnt, 256, 0, s>>>(LIv, G.nG_pad, lsS); BDDC_COUNT(); }
        BDDC_LAUNCH_CHECK();
        trsm_batched(TRSM_LLN, LSb, G.nG_pad, LIb, G.nG_pad, cnt, c.tinv, s, true);
      }
    }
    BMat Xb{X, phS, G.nG_pad};
    // T deferred into the dataflow coarse factorization (all subdomains in one chunk)
    const bool defer_t = c.lt_fusable && c.fp.n_coarse > 0 && sub0 == G.s_lo && cnt == G.s_hi - G.s_lo;
    c.lt_defer = LtArgs{};
    if (G.nc_pad > 0) {
      // 5b/7 through Z = S_K^{-1}: S_C = G^T G with G = L^{-1} C^T (a Gram matrix: stays SPD
      // at 1e12 coefficient contrast, where C Z C^T does not), W = Z C^T (a gather, no GEMM),
      // Phi = W S_C^{-1}, T = Z - Phi W^T (= S_K^{-1} - Phi S_C Phi^T). Z and then T in LS.
      BMat PHb{PH, phS, G.nG_pad};
      BMat SCb{SC, scS, G.nc_pad};
      BMat SCib{SCi, scS, G.nc_pad};
      {
        PhaseScope pphi(c.prof, "setup.Phi", s);
        BMat Yb{Y, phS, G.nG_pad};
        const bool gathered = g_gather(G, sub0, cnt, c.st, LIv, lsS, Y, phS, s, true);  // G
        if (!gathered) {
          BDDC_CUDA(cudaMemsetAsync(PH, 0, sizeof(double) * cnt * phS, s));
          { build_ct_kernel<<<cnt, 128, 0, s>>>(G, sub0, c.st, c.Phi); BDDC_COUNT(); }  // C^T
          BDDC_LAUNCH_CHECK();
          gemm_batched(false, false, G.nG_pad, G.nc_pad, G.nG_pad, 1.0, LIb, PHb, 0.0, Yb, cnt, s, false, 1);
        }
        gemm_batched(true, false, G.nc_pad, G.nc_pad, G.nG_pad, 1.0, Yb, Yb, 0.0, SCb, cnt, s);  // S_C
        { sc_pad_kernel<<<cnt, 128, 0, s>>>(G, sub0, c.st, SC); BDDC_COUNT(); }
        BDDC_LAUNCH_CHECK();
        gemm_batched(true, false, G.nG_pad, G.nG_pad, G.nG_pad, 1.0, LIb, LIb, 0.0, LSb, cnt, s, true, 2, true);  // Z
        if (gathered) g_gather(G, sub0, cnt, c.st, LS, lsS, X, phS, s, false);  // W = Z C^T
        else gemm_batched(false, false, G.nG_pad, G.nc_pad, G.nG_pad, 1.0, LSb, PHb, 0.0, Xb, cnt, s);
        potrf_batched(SCb, G.nc_pad, G.nc_pad, cnt, nullptr, c.tinv, s);
        const int ncb = ceil_div(G.nc_pad, kTile);
        BMat LCi{c.tinv, (long long)ncb * kTileInvStride, kTile};  // L_C^{-1} (one tile)
        if (ncb > 1) {  // L_C^{-1} in full: the S_C^{-1} product reads both triangles' blocks
          LCi = BMat{P, scS, G.nc_pad};
          BDDC_CUDA(cudaMemsetAsync(P, 0, sizeof(double) * cnt * scS, s));
          if (!trtri_from_tiles(SCb, G.nc_pad, LCi, cnt, c.tinv, s)) throw CudaError("S_C too large");
        }
        gemm_batched(true, false, G.nc_pad, G.nc_pad, G.nc_pad, 1.0, LCi, LCi, 0.0, SCib, cnt, s);  // S_C^{-1}
        gemm_batched(false, false, G.nG_pad, G.nc_pad, G.nc_pad, 1.0, Xb, SCib, 0.0, PHb, cnt, s);   // Phi
        // 6. local coarse block P = Phi^T S_Gamma Phi = S_C^{-1} - s I
        { finish_local_kernel<<<cnt, 256, 0, s>>>(G, sub0, c.coarse_scaling, c.diag_s, c.st, c.cscale, SCi,
                                                c.Sloc); BDDC_COUNT(); }
        BDDC_LAUNCH_CHECK();
      }
      // 7. T -= Phi W^T: deferred into the dataflow coarse factorization when all subdomains are
      //    one chunk (its schedule runs the tiles on the CTAs the critical path leaves idle)
      if (defer_t) {
        c.lt_defer = LtArgs{PH, X, c.LS, lsS, phS, G.nG_pad, G.nc_pad, sub0, 1, 1};
        continue;
      }
      PhaseScope pt(c.prof, "setup.T", s);
      gemm_batched(false, true, G.nG_pad, G.nG_pad, G.nc_pad, -1.0, PHb, Xb, 1.0, LSb, cnt, s, true, 0,
                   !t_lower_only(G));
      continue;
    }
    // no constraints: T = S_K^{-1} = L^{-T} L^{-1}
    if (defer_t) {
      c.lt_defer = LtArgs{LIv, X, c.LS, lsS, phS, G.nG_pad, 0, sub0, 1, 0};
      continue;
    }
    {
      PhaseScope pt(c.prof, "setup.T", s);
      gemm_batched(true, false, G.nG_pad, G.nG_pad, G.nG_pad, 1.0, LIb, LIb, 0.0, LSb, cnt, s, true, 2,
                   !t_lower_only(G));
    }
  }
}

}  // namespace bddc
