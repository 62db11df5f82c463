// Preconditioner apply z = B r (BddcOperator.apply, bddc.py:336-390), reduced form.
//
// The reference does three interior sweeps and two global SpMVs. Because interior dofs
// only couple inside their subdomain, (r - A u1)_I = 0 and (r - A(u1+u2))_I = 0, so
//   rp_Gamma = r_Gamma - (A u1)_Gamma,          u1_I = A_II^{-1} r_I
//   z_Gamma  = g = sum_i D_i R_i (w_i),          w_i = v_i + Psi_i c
//   z_I      = A_II^{-1} (r - A g_ext)_I
// which equals apply() to round-off. The local constrained Neumann
// solve restricted to Gamma is v = (I - Phi C) S_K^{-1} rho, so
//   w = u + Phi (c_i * c_loc - C u),  u = S_K^{-1} rho,  coarse rhs += c_i Phi^T rho.
#include "stencil.cuh"

namespace bddc {

namespace {

template <int DIM, bool EDGE>
__global__ void __launch_bounds__(256, (EDGE || DIM == 2) ? 3 : 1) spmv_kernel(Geometry G, const double* __restrict__ alpha,
                                                   const double* __restrict__ x, double* __restrict__ y) {
  stencil_sweep<DIM, EDGE>(G, alpha, x, [&](long long f, double v, double) { y[f] = v; });
}

// y = r - A x (all free dofs)
template <int DIM, bool EDGE>
__global__ void __launch_bounds__(256, (EDGE || DIM == 2) ? 3 : 1) residual_kernel(Geometry G, const double* __restrict__ alpha,
                                                       const double* __restrict__ r, const double* __restrict__ x,
                                                       double* __restrict__ y) {
  stencil_sweep<DIM, EDGE>(G, alpha, x, [&](long long f, double v, double) { y[f] = r[f] - v; });
}

// launch K<DIM, EDGE> over the sweep's work items (columns x row chunks of the active rows)
#define BDDC_SWEEP_LAUNCH(K, G, s, ...)                                                            \
  do {                                                                                             \
    const int th_ = 256, gr_ = grid_for(sweep_items(G), th_);                                      \
    const bool e_ = stencil_edge_only(G);                                                          \
    if (G.dim == 2) { if (e_) K<2, true><<<gr_, th_, 0, s>>>(G, __VA_ARGS__); else K<2, false><<<gr_, th_, 0, s>>>(G, __VA_ARGS__); } \
    else { if (e_) K<3, true><<<gr_, th_, 0, s>>>(G, __VA_ARGS__); else K<3, false><<<gr_, th_, 0, s>>>(G, __VA_ARGS__); } \
    BDDC_COUNT();                                                                                  \
    BDDC_LAUNCH_CHECK();                                                                           \
  } while (0)

// rpg[g] = r - (A u1) at interface dofs
template <int DIM>
__global__ void gamma_residual_kernel(Geometry G, const long long* __restrict__ gdof,
                                      const double* __restrict__ alpha, const double* __restrict__ r,
                                      const double* __restrict__ u1, double* __restrict__ rpg) {
  const int g = G.g_lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G.g_hi) return;
  const long long f = gdof[g];
  int g0, g1, g2;
  free_coords(G, f, g0, g1, g2);
  rpg[g] = r[f] - stencil_row<DIM>(G, alpha, u1, g0, g1, g2);
}

// Block-tridiagonal interior solve x_I = A_II^{-1} b_I, one warp per subdomain, with the
// factor stored as packed symmetric Schur-complement inverses W_j = S_j^{-1} plus the
// sparse coupling stencil B_j to the previous plane (block LDL^T):
//   forward   h_j = W_j (b_j - B_j h_{j-1})
//   backward  x_j = h_j - W_j (B_{j+1}^T x_{j+1})
// Each lane owns rows r = lane + 32 i (i < R). A plane's packed W and its coupling rows are
// staged by cp.async (double-buffered: plane j -+ 1 streams in while plane j is used); the
// GEMV reads the packed column-major lower triangle in shared memory with running offsets
// and the vector by broadcast. Each W_j is read from HBM once per pass.
constexpr int kBtWarps = 4;
constexpr int kBtStages = 2;  // planes in flight per warp: current + 1 ahead

struct BtSmem {  // per-warp layout (doubles)
  int nI, tm_pad, bc_pad, M2;
  __device__ __host__ int stage() const { return tm_pad + bc_pad; }
  __device__ __host__ int per_warp() const { return nI + kBtStages * stage() + M2; }
};

__device__ __host__ inline BtSmem bt_smem(const Geometry& G) {
  BtSmem b;
  b.nI = G.nI_pad;
  b.tm_pad = (G.Tm + 1) & ~1;
  b.bc_pad = (G.m_pad * G.nbo + 1) & ~1;
  b.M2 = (G.m_pad + 1) & ~1;
  return b;
}

// out[r] = sum_k W[r][k] v[k]; W packed lower, column k at ck = k M - k(k-1)/2 (rows k..M-1):
//   k <= r: W[r][k] = pk[ck + r - k]   (offset a1, advances by M - 1 - k per column)
//   k >  r: W[r][k] = pk[cr + k - r]   (offset a2 + k, a2 = cr - r)
template <int R>
__device__ __forceinline__ void bt_gemv(const double* __restrict__ pk, const double* __restrict__ v, int M,
                                        double (&out)[R], int lane) {
  int a1[R], a2[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int r = min(lane + 32 * i, M - 1);  // lanes past M repeat row M-1 (result unused)
    out[i] = 0.0;
    a1[i] = r;
    a2[i] = r * M - r * (r - 1) / 2 - r;
  }
  int d = M - 1;
#pragma unroll 4
  for (int k = 0; k < M; ++k) {
    const double vk = v[k];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int r = min(lane + 32 * i, M - 1);
      const double w = pk[k <= r ? a1[i] : a2[i] + k];
      out[i] = fma(w, vk, out[i]);
      a1[i] += d;
    }
    --d;
  }
}

template <int R>
__global__ void __launch_bounds__(32 * kBtWarps) bt_solve_kernel(Geometry G, LocalTables lt,
                                                                 const double* __restrict__ LI,
                                                                 const double* __restrict__ in,
                                                                 double* __restrict__ out) {
  extern __shared__ __align__(16) double sm[];
  const BtSmem L = bt_smem(G);
  const int M = G.m_pad, Tm = G.Tm, nbo = G.nbo, nblk = G.nblk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = G.s_lo + blockIdx.x * kBtWarps + warp;
  double* y = sm + warp * L.per_warp();        // nI_pad
  double* stg = y + L.nI;                      // kBtStages x [W packed | coupling rows]
  double* tv = stg + kBtStages * L.stage();    // M: the GEMV input vector

  if (sub >= G.s_hi) return;
  int p[3];
  sub_coords(G, sub, p);
  const double* li = LI + (long long)sub * G.li_stride;
  const double* bc = li + (long long)nblk * Tm;
  const int mb = M * nbo;
  // stage st <- W_jw and the coupling rows of plane jb (jb < 0: none)
  auto prefetch = [&](int jw, int jb, int st) {
    double* dst = stg + st * L.stage();
    const double* src = li + (long long)jw * Tm;
    for (int e = 2 * lane; e < Tm; e += 64) cp_async16(dst + e, src + e, min(2, Tm - e) * 8);
    if (jb >= 0) {
      const double* sb = bc + (long long)jb * mb;
      for (int e = 2 * lane; e < mb; e += 64) cp_async16(dst + L.tm_pad + e, sb + e, min(2, mb - e) * 8);
    }
    cp_async_commit();
  };
  // lane rows: in-plane coordinates and the coupling neighbours (clamped; the coefficient
  // of a structurally absent neighbour is zero)
  const int px = G.blk[0] - 1;
  int fwd_q[R][9], bwd_q[R][9];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int r = lane + 32 * i, x = r % px, yy = r / px;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      if (k < nbo) {
        const int qf = (x + G.bo_dx[k]) + (yy + G.bo_dy[k]) * px;
        const int qb = (x - G.bo_dx[k]) + (yy - G.bo_dy[k]) * px;
        fwd_q[i][k] = min(max(qf, 0), M - 1);
        bwd_q[i][k] = (qb >= 0 && qb < M && r < M) ? qb : -1;
      }
    }
  }
  if (nblk > 0) prefetch(0, 0, 0);
  for (int rr = lane; rr < G.nI_pad; rr += 32) {
    const int node = lt.irow_node[rr];
    double v = 0.0;
    if (node >= 0) {
      int a[3];
      local_coords(G, node, a);
      v = in[local_to_free(G, p, a)];
    }
    y[rr] = v;
  }
  double hv[R];
  // ---- forward: h_j = W_j (b_j - B_j h_{j-1}) ----
  for (int j = 0; j < nblk; ++j) {
    const int st = j & 1;
    if (j + 1 < nblk) {
      prefetch(j + 1, j + 1, st ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const double* pk = stg + st * L.stage();
    const double* bj = pk + L.tm_pad;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int r = lane + 32 * i;
      if (r < M) {
        double acc = y[j * M + r];
        if (j > 0) {
          const double* hp = y + (j - 1) * M;
#pragma unroll
          for (int k = 0; k < 9; ++k)
            if (k < nbo) acc -= bj[r * nbo + k] * hp[fwd_q[i][k]];
        }
        tv[r] = acc;
      }
    }
    __syncwarp();
    bt_gemv<R>(pk, tv, M, hv, lane);
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (lane + 32 * i < M) y[j * M + lane + 32 * i] = hv[i];
    __syncwarp();
  }
  // ---- backward: x_j = h_j - W_j (B_{j+1}^T x_{j+1}) ----
  if (nblk > 1) prefetch(nblk - 2, nblk - 1, 0);
  for (int j = nblk - 2, it = 0; j >= 0; --j, ++it) {
    const int st = it & 1;
    if (j > 0) {
      prefetch(j - 1, j, st ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const double* pk = stg + st * L.stage();
    const double* bn = pk + L.tm_pad;  // coupling rows of plane j + 1
    const double* xn = y + (j + 1) * M;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int r = lane + 32 * i;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < 9; ++k)
        if (k < nbo && bwd_q[i][k] >= 0) acc += bn[bwd_q[i][k] * nbo + k] * xn[bwd_q[i][k]];
      if (r < M) tv[r] = acc;
    }
    __syncwarp();
    bt_gemv<R>(pk, tv, M, hv, lane);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int r = lane + 32 * i;
      if (r < M) y[j * M + r] -= hv[i];
    }
    __syncwarp();
  }
  for (int rr = lane; rr < G.nI_pad; rr += 32) {
    const int node = lt.irow_node[rr];
    if (node >= 0) {
      int a[3];
      local_coords(G, node, a);
      out[local_to_free(G, p, a)] = y[rr];
    }
  }
}

// ---- specialised interior solve: compile-time plane rows M and stencil width NBO ----
// Each plane (packed W_j + its coupling rows) arrives by TMA bulk copy (cp.async.bulk,
// issued by one lane, completing on a per-stage mbarrier); the GEMV is fully unrolled with
// the packed-column offsets as immediates; the interior dofs of a subdomain are an affine
// map of its base dof (irow_rel), so gather / scatter need no index arithmetic.
template <int M>
__host__ __device__ constexpr int bt_cs(int k) { return k * M - k * (k - 1) / 2; }

template <int M, int NBO>
struct BtT {
  static constexpr int R = (M + 31) / 32;
  static constexpr int TM = M * (M + 1) / 2;
  static constexpr int MB = M * NBO;
  static constexpr int STAGE = TM + MB;  // both even (M % 8 == 0): 16-byte aligned stages
  // planes in flight per warp (NS) and warps per CTA (W): deeper prefetch for the small 2D
  // planes, more warps (latency hiding) for the large 3D ones; both fill the shared memory
  static constexpr int NS = M <= 32 ? 3 : 2;
  static constexpr int W = M <= 32 ? 5 : 7;
  static constexpr int NB = (NS + 1) & ~1;  // mbarrier slots (keeps the stages 16-byte aligned)
  static __host__ __device__ int per_warp(int nI) { return NB + NS * STAGE + nI + M; }
};

template <int M, int R>
__device__ __forceinline__ void bt_gemv_t(const double* __restrict__ pk, const double* __restrict__ v,
                                          double (&out)[R], int lane) {
  const double* b1[R];
  const double* b2[R];
  int r[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    r[i] = min(lane + 32 * i, M - 1);  // lanes past M repeat row M-1 (result unused)
    b1[i] = pk + r[i];                          // k <= r: pk[cs(k) - k + r]
    b2[i] = pk + (r[i] * M - r[i] * (r[i] - 1) / 2) - r[i];  // k > r: pk[cs(r) - r + k]
    out[i] = 0.0;
  }
#pragma unroll
  for (int k = 0; k < M; ++k) {
    const double vk = v[k];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const double w = k <= r[i] ? b1[i][bt_cs<M>(k) - k] : b2[i][k];
      out[i] = fma(w, vk, out[i]);
    }
  }
}

template <int M, int NBO>
__global__ void __launch_bounds__(32 * BtT<M, NBO>::W) bt_solve_t_kernel(Geometry G, LocalTables lt,
                                                                   const double* __restrict__ LI,
                                                                   const double* __restrict__ in,
                                                                   double* __restrict__ out) {
  using T = BtT<M, NBO>;
  constexpr int R = T::R, NS = T::NS;
  extern __shared__ __align__(16) double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nI = G.nI_pad, nblk = G.nblk;
  double* wb = sm + warp * T::per_warp(nI);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(wb);
  double* stg = wb + T::NB;
  double* y = stg + NS * T::STAGE;
  double* tv = y + nI;
  const int sub = G.s_lo + blockIdx.x * T::W + warp;
  if (sub >= G.s_hi) return;
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NS; ++q) mbar_init(&bar[q], 1);
    mbar_fence_init();
  }
  __syncwarp();
  const double* li = LI + (long long)sub * G.li_stride;
  const double* bc = li + (long long)nblk * T::TM;
  unsigned ph = 0;  // parity bit per stage
  auto issue = [&](int jw, int jb, int st) {  // plane jw's W (+ coupling rows of plane jb)
    if (lane == 0) {
      double* dst = stg + st * T::STAGE;
      mbar_expect_tx(&bar[st], (unsigned)(T::TM * 8 + (jb >= 0 ? T::MB * 8 : 0)));
      bulk_g2s(dst, li + (long long)jw * T::TM, T::TM * 8, &bar[st]);
      if (jb >= 0) bulk_g2s(dst + T::TM, bc + (long long)jb * T::MB, T::MB * 8, &bar[st]);
    }
  };
  auto wait = [&](int st) {
    mbar_wait(&bar[st], (ph >> st) & 1u);
    ph ^= 1u << st;
  };
#pragma unroll
  for (int q = 0; q < NS - 1; ++q)
    if (q < nblk) issue(q, q > 0 ? q : -1, q);
  // gather: free dof of interior row rr = base + rel[rr]
  int p[3];
  sub_coords(G, sub, p);
  long long base = (long long)(p[0] * G.blk[0] - 1) + (long long)G.nfree[0] * (p[1] * G.blk[1] - 1);
  if (G.dim == 3) base += (long long)G.nfree[0] * G.nfree[1] * (p[2] * G.blk[2] - 1);
  for (int rr = lane; rr < nI; rr += 128) {
    int rel[4];
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) rel[u] = rr + 32 * u < nI ? lt.irow_rel[rr + 32 * u] : -1;
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = rel[u] >= 0 ? in[base + rel[u]] : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (rr + 32 * u < nI) y[rr + 32 * u] = v[u];
  }
  // lane rows: coupling neighbours (clamped; absent neighbours have zero coefficients)
  const int px = G.blk[0] - 1;
  int fwd_q[R][NBO], bwd_q[R][NBO];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int r = lane + 32 * i, x = r % px, yy = r / px;
#pragma unroll
    for (int k = 0; k < NBO; ++k) {
      const int qf = (x + G.bo_dx[k]) + (yy + G.bo_dy[k]) * px;
      const int qb = (x - G.bo_dx[k]) + (yy - G.bo_dy[k]) * px;
      fwd_q[i][k] = min(max(qf, 0), M - 1);
      bwd_q[i][k] = (qb >= 0 && qb < M && r < M) ? qb : -1;
    }
  }
  __syncwarp();
  double hv[R];
  // ---- forward: h_j = W_j (b_j - B_j h_{j-1}) ----
  for (int j = 0; j < nblk; ++j) {
    const int st = j % NS;
    if (j + NS - 1 < nblk) issue(j + NS - 1, j + NS - 1, (j + NS - 1) % NS);
    wait(st);
    const double* pk = stg + st * T::STAGE;
    const double* bj = pk + T::TM;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int r = lane + 32 * i;
      if (r < M) {
        double acc = y[j * M + r];
        if (j > 0) {
          const double* hp = y + (j - 1) * M;
#pragma unroll
          for (int k = 0; k < NBO; ++k) acc -= bj[r * NBO + k] * hp[fwd_q[i][k]];
        }
        tv[r] = acc;
      }
    }
    __syncwarp();
    bt_gemv_t<M, R>(pk, tv, hv, lane);
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (lane + 32 * i < M) y[j * M + lane + 32 * i] = hv[i];
    __syncwarp();
  }
  // ---- backward: x_j = h_j - W_j (B_{j+1}^T x_{j+1}) ----
#pragma unroll
  for (int q = 0; q < NS - 1; ++q)
    if (nblk - 2 - q >= 0) issue(nblk - 2 - q, nblk - 1 - q, q);
  for (int j = nblk - 2, it = 0; j >= 0; --j, ++it) {
    const int st = it % NS;
    if (j - (NS - 1) >= 0) issue(j - (NS - 1), j - (NS - 2), (it + NS - 1) % NS);
    wait(st);
    const double* pk = stg + st * T::STAGE;
    const double* bn = pk + T::TM;  // coupling rows of plane j + 1
    const double* xn = y + (j + 1) * M;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int r = lane + 32 * i;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < NBO; ++k)
        if (bwd_q[i][k] >= 0) acc += bn[bwd_q[i][k] * NBO + k] * xn[bwd_q[i][k]];
      if (r < M) tv[r] = acc;
    }
    __syncwarp();
    bt_gemv_t<M, R>(pk, tv, hv, lane);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int r = lane + 32 * i;
      if (r < M) y[j * M + r] -= hv[i];
    }
    __syncwarp();
  }
  for (int rr = lane; rr < nI; rr += 32) {
    const int rel = lt.irow_rel[rr];
    if (rel >= 0) out[base + rel] = y[rr];
  }
}

template <int M, int NBO>
bool launch_bt_t(const Geometry& G, const LocalTables& lt, const double* LI, const double* in, double* out,
                 cudaStream_t s) {
  if (G.m_pad != M || G.nbo != NBO || G.Tm != BtT<M, NBO>::TM) return false;
  const size_t smem = sizeof(double) * BtT<M, NBO>::per_warp(G.nI_pad) * BtT<M, NBO>::W;
  if (smem > 227 * 1024) return false;
  static SmemAttr attr;
  if (attr.needs(smem)) {
    BDDC_CUDA(cudaFuncSetAttribute(bt_solve_t_kernel<M, NBO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr.set(smem);
  }
  const int grid = ceil_div(G.s_hi - G.s_lo, BtT<M, NBO>::W);
  bt_solve_t_kernel<M, NBO><<<grid, 32 * BtT<M, NBO>::W, smem, s>>>(G, lt, LI, in, out);
  BDDC_COUNT();
  BDDC_LAUNCH_CHECK();
  return true;
}

template <int NBO>
bool launch_bt_nbo(const Geometry& G, const LocalTables& lt, const double* LI, const double* in, double* out,
                   cudaStream_t s) {
  switch (G.m_pad) {
    case 8: return launch_bt_t<8, NBO>(G, lt, LI, in, out, s);
    case 16: return launch_bt_t<16, NBO>(G, lt, LI, in, out, s);
    case 32: return launch_bt_t<32, NBO>(G, lt, LI, in, out, s);
    case 56: return launch_bt_t<56, NBO>(G, lt, LI, in, out, s);
    case 64: return launch_bt_t<64, NBO>(G, lt, LI, in, out, s);
    default: return false;
  }
}

__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  return s;
}

// Per subdomain: rho = D rp_Gamma;  q = c Phi^T rho (coarse rhs);  v = T rho, with the
// explicit interface operator T = (I - Phi C) S_K^{-1} (the constrained Neumann solve on
// Gamma, bddc.py:357; symmetric, built in setup).
// WITH_T = false: the coarse solve computes v = T rho (TvArgs); rho is stored in vloc.
template <bool WITH_T>
__global__ void __launch_bounds__(128) local_gamma1_kernel(Geometry G, SubTables st,
                                                           const double* __restrict__ T,
                                                           const double* __restrict__ Phi,
                                                           const double* __restrict__ cscale,
                                                           const double* __restrict__ rpg,
                                                           double* qloc, double* vloc) {
  extern __shared__ double sm[];
  const int n = G.nG_pad, nc = G.nc_pad;
  double* rho = sm;  // n
  const int sub = G.s_lo + blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const long long so = (long long)sub * n;
  for (int s = tid; s < n; s += nt) {
    const int g = st.slot_gamma[so + s];
    rho[s] = g >= 0 ? st.slot_w[so + s] * rpg[g] : 0.0;
    if (!WITH_T) vloc[so + s] = rho[s];
  }
  __syncthreads();
  const double c = cscale[sub];
  const double* ph = Phi + (long long)sub * n * nc;
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int k = warp; k < nc; k += nw) {
    double acc = 0.0;
    for (int s = lane; s < n; s += 32) acc += ph[s + (long long)k * n] * rho[s];
    acc = warp_sum(acc);
    if (lane == 0) qloc[(long long)sub * nc + k] = c * acc;
  }
  if (!WITH_T) return;
  const double* Ts = T + (long long)sub * n * n;
  for (int i = tid; i < n; i += nt) {
    double a0 = 0.0, a1 = 0.0;
    int k = 0;
    for (; k + 1 < n; k += 2) {
      a0 += Ts[i + (long long)k * n] * rho[k];
      a1 += Ts[i + (long long)(k + 1) * n] * rho[k + 1];
    }
    if (k < n) a0 += Ts[i + (long long)k * n] * rho[k];
    vloc[so + i] = a0 + a1;
  }
}

// local_gamma1 with T stored as its lower triangle (t_lower_only): rho = D rp, q = c Phi^T rho,
// v = T rho reading every stored entry once. Warp per 32-column block J (snake order over
// the warps): each 32x32 block (I >= J) gives the direct part T_IJ rho_J (rows of I) and,
// accumulated in registers down the block column, the transposed part T_IJ^T rho_I (rows of
// J, one shared-memory transpose-sum per column). Partials are summed in a fixed order.
constexpr int kG1LThreads = 256;
size_t gamma1_lower_smem(int n) {
  const int nb = (n + 31) / 32;
  return sizeof(double) * ((size_t)nb * 32 * 2 + (size_t)nb * 32 * nb - 16 * nb * (nb - 1) +
                           (kG1LThreads / 32) * 32 * 33);
}

__global__ void __launch_bounds__(kG1LThreads, 2) local_gamma1_lower_kernel(
    Geometry G, SubTables st, const double* __restrict__ T, const double* __restrict__ Phi,
    const double* __restrict__ cscale, const double* __restrict__ rpg, double* qloc, double* vloc) {
  extern __shared__ double sm[];
  const int n = G.nG_pad, nc = G.nc_pad, nb = (n + 31) / 32, nr = nb * 32;
  constexpr int NW = kG1LThreads / 32;
  double* rho = sm;                       // nr
  double* pt = rho + nr;                  // nr transposed partials
  double* tb = pt + nr;                   // per warp 32 x 33: lane's transposed accumulators
  double* pd = tb + NW * 32 * 33;         // direct partials of block column J: rows >= 32 J
  auto pdo = [&](int J) { return (size_t)J * nr - 16 * J * (J - 1) - 32 * J; };
  const int sub = G.s_lo + blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const long long so = (long long)sub * n;
  for (int s = tid; s < nr; s += kG1LThreads) {
    const int g = s < n ? st.slot_gamma[so + s] : -1;
    rho[s] = g >= 0 ? st.slot_w[so + s] * rpg[g] : 0.0;
  }
  __syncthreads();
  const double c = cscale[sub];
  const double* ph = Phi + (long long)sub * n * nc;
  for (int k = warp; k < nc; k += NW) {  // all of a column's loads in flight at once
    double a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int s = lane + 32 * i;
      a[i] = s < n ? ph[s + (long long)k * n] : 0.0;
    }
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) acc += a[i] * rho[min(lane + 32 * i, nr - 1)];
    acc = warp_sum(acc);
    if (lane == 0) qloc[(long long)sub * nc + k] = c * acc;
  }
  const double* Ts = T + (long long)sub * n * n;
  double* mtb = tb + warp * 32 * 33 + lane * 33;
  for (int round = 0; round * NW < nb; ++round) {
    const int J = round * NW + ((round & 1) ? NW - 1 - warp : warp);
    if (J >= nb) continue;
#pragma unroll
    for (int k = 0; k < 32; ++k) mtb[k] = 0.0;
    for (int I = J; I < nb; ++I) {
      const int r = 32 * I + lane;
      double t[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int col = 32 * J + k;
        t[k] = (r < n && col < n) ? Ts[r + (long long)col * n] : 0.0;
      }
      const double rr = rho[r];
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const double td = (I > J || k <= lane) ? t[k] : 0.0;  // diagonal block: lower incl.
        const double tt = (I > J || k < lane) ? t[k] : 0.0;   // strictly lower
        if (k & 1) d1 += td * rho[32 * J + k];
        else d0 += td * rho[32 * J + k];
        mtb[k] += tt * rr;
      }
      pd[pdo(J) + r] = d0 + d1;
    }
    __syncwarp();
    double sum = 0.0;
    const double* col = tb + warp * 32 * 33 + lane;
#pragma unroll 8
    for (int i = 0; i < 32; ++i) sum += col[i * 33];
    pt[32 * J + lane] = sum;
    __syncwarp();
  }
  __syncthreads();
  for (int r = tid; r < n; r += kG1LThreads) {
    double y = pt[r];
    for (int J = 0; J <= r / 32; ++J) y += pd[pdo(J) + r];
    vloc[so + r] = y;
  }
}

// Per subdomain: w = D (v + c Phi csol[coarse])
__global__ void __launch_bounds__(128) local_gamma2_kernel(Geometry G, SubTables st,
                                                           const double* __restrict__ Phi,
                                                           const double* __restrict__ cscale,
                                                           const double* __restrict__ csol,
                                                           const double* __restrict__ vloc,
                                                           double* wloc) {
  __shared__ double e[1024];
  const int n = G.nG_pad, nc = G.nc_pad;
  const int sub = G.s_lo + blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const double c = cscale[sub];
  for (int k = tid; k < nc; k += nt) {
    const int j = st.con_coarse[(long long)sub * nc + k];
    e[k] = j >= 0 ? c * csol[j] : 0.0;
  }
  __syncthreads();
  const double* ph = Phi + (long long)sub * n * nc;
  const long long so = (long long)sub * n;
  for (int s = tid; s < n; s += nt) {
    double acc = vloc[so + s];
    for (int k = 0; k < nc; ++k) acc += ph[s + (long long)k * n] * e[k];
    wloc[so + s] = st.slot_w[so + s] * acc;
  }
}

// z[gamma dof] = sum over owner slots (ascending subdomain = reference summation order)
__global__ void gamma_gather_kernel(int g_lo, int g_hi, int W, const long long* __restrict__ gdof,
                                    const int* __restrict__ gslots, const double* __restrict__ wloc,
                                    double* __restrict__ z, long long nslots, long long n) {
  const int g = g_lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= g_hi) return;
  double acc = 0.0;
  for (int w = 0; w < W; ++w) {
    const int s = gslots[(long long)g * W + w];
    BDDC_CHECK(s < nslots);
    if (s >= 0) acc += wloc[s];
  }
  BDDC_CHECK(gdof[g] >= 0 && gdof[g] < n);
  z[gdof[g]] = acc;
}

__global__ void coarse_gather_kernel(int n_coarse, int W, const int* __restrict__ cslots,
                                     const double* __restrict__ qloc, double* __restrict__ crhs) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_coarse) return;
  double acc = 0.0;
  for (int w = 0; w < W; ++w) {
    const int s = cslots[(long long)j * W + w];
    if (s >= 0) acc += qloc[s];
  }
  crhs[j] = acc;
}

int grid_for(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  return (int)std::min<long long>(b, 148LL * 32);
}

}  // namespace

void spmv(Ctx& c, const double* x, double* y, cudaStream_t s) {
  const Geometry& G = c.geo;
  BDDC_SWEEP_LAUNCH(spmv_kernel, G, s, c.alpha, x, y);
}

static void bt_solve(Ctx& c, const double* in, double* out, cudaStream_t s) {
  const Geometry& G = c.geo;
  PhaseScope ps(c.prof, "apply.bt_solve", s);
  if (G.s_hi <= G.s_lo) return;
  bool done = false;
  if (G.nbo == 1) done = launch_bt_nbo<1>(G, c.lt, c.LI, in, out, s);
  else if (G.nbo == 3) done = launch_bt_nbo<3>(G, c.lt, c.LI, in, out, s);
  else if (G.nbo == 9) done = launch_bt_nbo<9>(G, c.lt, c.LI, in, out, s);
  if (done) return;
  const size_t smem = sizeof(double) * bt_smem(G).per_warp() * kBtWarps;
  static SmemAttr attr;
  if (attr.needs(smem)) {
    BDDC_CUDA(cudaFuncSetAttribute(bt_solve_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    BDDC_CUDA(cudaFuncSetAttribute(bt_solve_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr.set(smem);
  }
  const int grid = ceil_div(G.s_hi - G.s_lo, kBtWarps);
  if (G.m_pad <= 32) { bt_solve_kernel<1><<<grid, 32 * kBtWarps, smem, s>>>(G, c.lt, c.LI, in, out); BDDC_COUNT(); }
  else { bt_solve_kernel<2><<<grid, 32 * kBtWarps, smem, s>>>(G, c.lt, c.LI, in, out); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
}

// out holds g on Gamma and 0 on interiors; c.v1 must be zero.
void harmonic_interior(Ctx& c, double* out, cudaStream_t s) {
  const Geometry& G = c.geo;
  BDDC_SWEEP_LAUNCH(residual_kernel, G, s, c.alpha, c.v1, out, c.v2);
  bt_solve(c, c.v2, out, s);
}

void apply_bddc(Ctx& c, const double* r, double* z, cudaStream_t s) {
  const Geometry& G = c.geo;
  const int th = 256;
  const int ng = G.g_hi - G.g_lo, nl = G.s_hi - G.s_lo;
  // u1 = A_II^{-1} r_I (zero on Gamma: set once at setup, never written there)
  bt_solve(c, r, c.v1, s);
  if (c.n_gamma > 0) {
    exchange_dof_halo(c, c.v1, s);  // sharded: u1 on the rows next to the cut lines
    if (ng > 0) {
      if (G.dim == 2)
        { gamma_residual_kernel<2><<<ceil_div(ng, th), th, 0, s>>>(G, c.gamma_dof, c.alpha, r, c.v1, c.rpg); BDDC_COUNT(); }
      else
        { gamma_residual_kernel<3><<<ceil_div(ng, th), th, 0, s>>>(G, c.gamma_dof, c.alpha, r, c.v1, c.rpg); BDDC_COUNT(); }
      BDDC_LAUNCH_CHECK();
    }
    const size_t smem1 = sizeof(double) * G.nG_pad;
    // v = T rho inside the coarse solve when its schedule holds those tasks (rho parked in wloc)
    const bool tv_fused = c.fp.n_coarse > 0 && c.sched.n_tv > 0 && !c.coarse_cb;
    c.prof.begin("apply.gamma1", s);
    if (tv_fused) { local_gamma1_kernel<false><<<nl, 128, smem1, s>>>(G, c.st, c.LS, c.Phi, c.cscale, c.rpg, c.qloc, c.wloc); BDDC_COUNT(); }
    else if (t_lower_only(G)) {
      static std::atomic<unsigned long long> attr{0};
      const size_t sm = gamma1_lower_smem(G.nG_pad);
      if (first_on_device(attr))
        BDDC_CUDA(cudaFuncSetAttribute(local_gamma1_lower_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gamma1_lower_smem(512)));
      local_gamma1_lower_kernel<<<nl, kG1LThreads, sm, s>>>(G, c.st, c.LS, c.Phi, c.cscale, c.rpg, c.qloc, c.uloc);
      BDDC_COUNT();
    }
    else { local_gamma1_kernel<true><<<nl, 128, smem1, s>>>(G, c.st, c.LS, c.Phi, c.cscale, c.rpg, c.qloc, c.uloc); BDDC_COUNT(); }
    BDDC_LAUNCH_CHECK();
    c.prof.end("apply.gamma1", s);
    if (c.fp.n_coarse > 0) {
      PhaseScope pc(c.prof, "apply.coarse", s);
      allgather_subs(c, c.qloc, G.nc_pad, s);  // sharded: every rank's local coarse rhs
      { coarse_gather_kernel<<<ceil_div(c.fp.n_coarse, th), th, 0, s>>>(c.fp.n_coarse, c.fp.W,
                                                                     c.fp.coarse_slots, c.qloc, c.crhs); BDDC_COUNT(); }
      BDDC_LAUNCH_CHECK();
      const TvArgs tv{c.LS, c.wloc, c.uloc, G.nG_pad};
      if (c.coarse_cb) {  // inexact coarse solve of a multilevel method, on this stream
        if (c.coarse_cb(c.coarse_cb_user, c.crhs, c.csol, c.fp.n_coarse, (void*)s) != 0)
          throw CudaError("coarse solver callback failed");
      } else {
        if (!c.coarse_factor_valid)
          throw CudaError("no exact coarse factor: the last refactor ran under the coarse-solver hook (refactor again)");
        coarse_solve(c, c.crhs, c.csol, s, tv_fused ? &tv : nullptr);
      }
    }
    c.prof.begin("apply.gamma2", s);
    { local_gamma2_kernel<<<nl, 128, 0, s>>>(G, c.st, c.Phi, c.cscale, c.csol, c.uloc,
                                           c.wloc); BDDC_COUNT(); }
    BDDC_LAUNCH_CHECK();
    c.prof.end("apply.gamma2", s);
    exchange_boundary_rows(c, c.wloc, G.nG_pad, s);  // sharded: w of the neighbours' cut rows
  }
  BDDC_CUDA(cudaMemsetAsync(z, 0, sizeof(double) * G.n, s));
  if (ng > 0) {
    { gamma_gather_kernel<<<ceil_div(ng, th), th, 0, s>>>(G.g_lo, G.g_hi, G.npe,
                                                        c.gamma_dof, c.gamma_slots, c.wloc, z,
                                                        (long long)G.nsub * G.nG_pad, G.n); BDDC_COUNT(); }
    BDDC_LAUNCH_CHECK();
  }
  // z_I = A_II^{-1} (r - A z_Gamma)_I
  BDDC_SWEEP_LAUNCH(residual_kernel, G, s, c.alpha, r, z, c.v2);
  bt_solve(c, c.v2, z, s);
}

}  // namespace bddc
