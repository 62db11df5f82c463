// Fused interior elimination for 2D subdomains (block rows of M <= 32, interface <= NGP):
// one CTA per subdomain runs the whole plane recursion on chip
//   Lo_j = B_j Linv_{j-1}^T ;  L_j = chol(T_j - Lo_j Lo_j^T) ;  Linv_j = L_j^{-1}
//   E_j  = Linv_j (A_IG,j - Lo_j E_{j-1})
//   S_G  = A_GG - sum_j E_j^T E_j            (lower 8x8 tiles held in registers)
// with every product on the FP64 tensor pipe (mma.sync m8n8k4 -> DMMA.8x8x4). It replaces
// btchol_kernel + 2 nblk batched GEMM launches + the S_G GEMM of the generic path, and
// writes the same outputs: packed Linv_j + coupling stencil (LI) and S_G (LS, full).
#include "stencil.cuh"

namespace bddc {

namespace {

constexpr int kSchurThreads = 256;

// C(8x8 tile) += A(8 x K) B(K x 8); A(r,k) = A[r*ars + k*acs], B(k,c) = B[k*brs + c*bcs]
__device__ __forceinline__ void mma_acc(double& c0, double& c1, const double* A, int ars, int acs,
                                        const double* B, int brs, int bcs, int K, int lane) {
  const int g = lane >> 2, t = lane & 3;
  for (int k = 0; k < K; k += 4) {
    const double a = A[g * ars + (k + t) * acs];
    const double b = B[(k + t) * brs + g * bcs];
    dmma884(c0, c1, a, b);
  }
}

template <int M, int NGP>
__global__ void __launch_bounds__(kSchurThreads) schur2d_kernel(Geometry G, int sub0,
                                                                const double* __restrict__ Wd,
                                                                const double* __restrict__ Wo,
                                                                const double* __restrict__ Eg,
                                                                double* __restrict__ LI,
                                                                double* __restrict__ LS,
                                                                int* __restrict__ info) {
  constexpr int P = M + 1;       // pitch of M x M blocks (col-major X[r + c*P])
  constexpr int EP = NGP + 4;    // pitch of E blocks, row-major E[k*EP + col]
  constexpr int NT = NGP / 8;    // interface tiles per dimension
  constexpr int NLT = NT * (NT + 1) / 2;
  constexpr int NW = kSchurThreads / 32;
  constexpr int SYRK_PER_WARP = (NLT + NW - 1) / NW;
  constexpr int ET = (M / 8) * NT;  // tiles of an M x NGP block
  constexpr int ET_PER_WARP = (ET + NW - 1) / NW;
  extern __shared__ __align__(16) double sm[];
  double* Ea = sm;                 // M x EP
  double* Eb = Ea + M * EP;        // M x EP
  double* Lp = Eb + M * EP;        // Linv_{j-1}
  double* Lc = Lp + M * P;         // Linv_j
  double* Lo = Lc + M * P;
  double* Sw = Lo + M * P;         // T_j -> S_j -> L_j
  double* Bw = Sw + M * P;         // B_j
  double* col = Bw + M * P;        // 2 x M column buffers
  __shared__ int failed;
  const int b = blockIdx.x, sub = sub0 + b;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const long long mm = (long long)G.m_pad * G.m_pad;
  const double* wd = Wd + (long long)b * G.nblk * mm;
  const double* wo = Wo + (long long)b * G.nblk * mm;
  const double* eg = Eg + (long long)b * G.nI_pad * G.nG_pad;
  double* li = LI + (long long)sub * G.li_stride;
  double* bcg = li + (long long)G.nblk * G.Tm;
  const int px = G.blk[0] - 1;
  if (tid == 0) failed = -1;

  double acc[SYRK_PER_WARP][2];
#pragma unroll
  for (int q = 0; q < SYRK_PER_WARP; ++q) acc[q][0] = acc[q][1] = 0.0;

  double* Eprev = Ea;  // E_{j-1}
  double* Ecur = Eb;   // A_IG,j -> R_j
  for (int j = 0; j < G.nblk; ++j) {
    // ---- load T_j, B_j, A_IG rows of plane j ----
    for (int idx = tid; idx < M * M; idx += kSchurThreads) {
      const int r = idx % M, c = idx / M;
      Sw[r + c * P] = wd[j * mm + idx];
      Bw[r + c * P] = j > 0 ? wo[j * mm + idx] : 0.0;
    }
    for (int idx = tid; idx < M * NGP; idx += kSchurThreads) {
      const int r = idx % M, cc = idx / M;
      Ecur[r * EP + cc] = eg[(j * M + r) + (long long)cc * G.nI_pad];
    }
    __syncthreads();
    // coupling stencil Bc_j for the apply (only structurally nonzero offsets)
    for (int idx = tid; idx < M * G.nbo; idx += kSchurThreads) {
      const int r = idx / G.nbo, k = idx % G.nbo;
      double v = 0.0;
      if (j > 0 && r < G.m) {
        const int x = r % px + G.bo_dx[k], y = r / px + G.bo_dy[k];
        if (x >= 0 && x < px && y == 0) v = Bw[r + x * P];
      }
      bcg[((long long)j * M + r) * G.nbo + k] = v;
    }
    if (j > 0) {
      // ---- Lo = B_j Linv_{j-1}^T ----
      for (int tt = warp; tt < (M / 8) * (M / 8); tt += NW) {
        const int ti = tt % (M / 8), tj = tt / (M / 8);
        double c0 = 0.0, c1 = 0.0;
        mma_acc(c0, c1, Bw + ti * 8, 1, P, Lp + tj * 8, P, 1, M, lane);
        Lo[(ti * 8 + g) + (tj * 8 + 2 * t4) * P] = c0;
        Lo[(ti * 8 + g) + (tj * 8 + 2 * t4 + 1) * P] = c1;
      }
      __syncthreads();
      // ---- S_j = T_j - Lo Lo^T (lower tiles) ----
      for (int tt = warp; tt < (M / 8) * (M / 8); tt += NW) {
        const int ti = tt % (M / 8), tj = tt / (M / 8);
        if (tj > ti) continue;
        double c0 = 0.0, c1 = 0.0;
        mma_acc(c0, c1, Lo + ti * 8, 1, P, Lo + tj * 8, P, 1, M, lane);
        Sw[(ti * 8 + g) + (tj * 8 + 2 * t4) * P] -= c0;
        Sw[(ti * 8 + g) + (tj * 8 + 2 * t4 + 1) * P] -= c1;
      }
      __syncthreads();
    }
    // ---- Cholesky of S_j in place: one barrier per column (ping-pong column buffers) ----
    for (int c = 0; c < M; ++c) {
      double* cb = col + (c & 1) * M;
      double d = Sw[c + c * P];
      if (!(d > 0.0)) {
        if (tid == 0 && failed < 0) failed = j * M + c;
        d = 1.0;
      }
      const double sd = sqrt(d), id = 1.0 / d;
      if (c > 0) {  // finalize column c-1 from its buffer
        const double* pb = col + ((c - 1) & 1) * M;
        for (int i = c - 1 + tid; i < M; i += kSchurThreads) Sw[i + (c - 1) * P] = pb[i];
      }
      for (int i = c + tid; i < M; i += kSchurThreads) cb[i] = i == c ? sd : Sw[i + c * P] / sd;
      const int r = M - c - 1;
      for (int idx = tid; idx < r * r; idx += kSchurThreads) {
        const int ii = c + 1 + idx % r, kk = c + 1 + idx / r;
        if (ii >= kk) Sw[ii + kk * P] -= Sw[ii + c * P] * Sw[kk + c * P] * id;
      }
      __syncthreads();
    }
    {
      const double* pb = col + ((M - 1) & 1) * M;
      if (tid == 0) Sw[(M - 1) + (M - 1) * P] = pb[M - 1];
    }
    __syncthreads();
    // ---- Linv_j: thread per column, forward substitution (lockstep broadcasts) ----
    if (tid < M) {
      const int c = tid;
      for (int i = 0; i < M; ++i) {
        double a = (i == c) ? 1.0 : 0.0;
        for (int k = 0; k < i; ++k) a -= Sw[i + k * P] * Lc[k + c * P];
        Lc[i + c * P] = (c <= i) ? a / Sw[i + i * P] : 0.0;
      }
    }
    __syncthreads();
    // packed Linv_j for the apply (column-major lower)
    for (int c = 0; c < M; ++c) {
      const int cs = c * M - c * (c - 1) / 2;
      for (int r = c + tid; r < M; r += kSchurThreads) li[(long long)j * G.Tm + cs + (r - c)] = Lc[r + c * P];
    }
    // ---- R_j = A_IG,j - Lo E_{j-1} (in Ecur) ----
    if (j > 0) {
      for (int q = 0; q < ET_PER_WARP; ++q) {
        const int tt = warp + q * NW;
        if (tt >= ET) break;
        const int ti = tt % (M / 8), tj = tt / (M / 8);
        double c0 = 0.0, c1 = 0.0;
        mma_acc(c0, c1, Lo + ti * 8, 1, P, Eprev + tj * 8, EP, 1, M, lane);
        Ecur[(ti * 8 + g) * EP + tj * 8 + 2 * t4] -= c0;
        Ecur[(ti * 8 + g) * EP + tj * 8 + 2 * t4 + 1] -= c1;
      }
      __syncthreads();
    }
    // ---- E_j = Linv_j R_j (into Eprev) ----
    for (int q = 0; q < ET_PER_WARP; ++q) {
      const int tt = warp + q * NW;
      if (tt >= ET) break;
      const int ti = tt % (M / 8), tj = tt / (M / 8);
      double c0 = 0.0, c1 = 0.0;
      mma_acc(c0, c1, Lc + ti * 8, 1, P, Ecur + tj * 8, EP, 1, (ti + 1) * 8, lane);
      Eprev[(ti * 8 + g) * EP + tj * 8 + 2 * t4] = c0;
      Eprev[(ti * 8 + g) * EP + tj * 8 + 2 * t4 + 1] = c1;
    }
    __syncthreads();
    // ---- S_acc += E_j^T E_j (lower interface tiles) ----
#pragma unroll
    for (int q = 0; q < SYRK_PER_WARP; ++q) {
      const int tt = warp + q * NW;
      if (tt < NLT) {
        // tile (I, J) with I >= J from the linear lower-tile index tt
        int I = 0;
        while ((I + 1) * (I + 2) / 2 <= tt) ++I;
        const int J = tt - I * (I + 1) / 2;
        mma_acc(acc[q][0], acc[q][1], Eprev + I * 8, 1, EP, Eprev + J * 8, EP, 1, M, lane);
      }
    }
    // Lp <- Lc for the next plane (pointer swap needs a barrier first)
    __syncthreads();
    { double* tmp = Lp; Lp = Lc; Lc = tmp; }
  }
  // ---- S_G = A_GG - S_acc, mirrored to a full symmetric matrix ----
  double* ls = LS + (long long)sub * G.nG_pad * G.nG_pad;
  const int ld = G.nG_pad;
#pragma unroll
  for (int q = 0; q < SYRK_PER_WARP; ++q) {
    const int tt = warp + q * NW;
    if (tt >= NLT) continue;
    int I = 0;
    while ((I + 1) * (I + 2) / 2 <= tt) ++I;
    const int J = tt - I * (I + 1) / 2;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int r = I * 8 + g, c = J * 8 + 2 * t4 + e;
      if (r >= c) {
        const double v = ls[r + (long long)c * ld] - acc[q][e];
        ls[r + (long long)c * ld] = v;
        if (r != c) ls[c + (long long)r * ld] = v;
      }
    }
  }
  if (tid == 0 && failed >= 0) atomicMin(info + sub, failed);
}

template <int M, int NGP>
size_t schur2d_smem() {
  return sizeof(double) * (2 * M * (NGP + 4) + 5 * M * (M + 1) + 2 * M);
}

template <int M, int NGP>
void launch_schur2d(const Ctx& c, int sub0, int cnt, const double* Wd, const double* Wo,
                    const double* E, cudaStream_t s) {
  const size_t smem = schur2d_smem<M, NGP>();
  static bool attr = false;
  if (!attr) {
    BDDC_CUDA(cudaFuncSetAttribute(schur2d_kernel<M, NGP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    attr = true;
  }
  { schur2d_kernel<M, NGP><<<cnt, kSchurThreads, smem, s>>>(c.geo, sub0, Wd, Wo, E, c.LI, c.LS, c.info); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
}

}  // namespace

// Returns false if the geometry is not covered by a compiled instance.
bool schur2d(const Ctx& c, int sub0, int cnt, const double* Wd, const double* Wo, const double* E,
             cudaStream_t s) {
  const Geometry& G = c.geo;
  if (G.dim != 2 || G.nbo != 1 || G.bo_dx[0] != 0) return false;
  if (G.m_pad == 32 && G.nG_pad == 128) launch_schur2d<32, 128>(c, sub0, cnt, Wd, Wo, E, s);
  else if (G.m_pad == 16 && G.nG_pad == 64) launch_schur2d<16, 64>(c, sub0, cnt, Wd, Wo, E, s);
  else if (G.m_pad == 8 && G.nG_pad == 32) launch_schur2d<8, 32>(c, sub0, cnt, Wd, Wo, E, s);
  else return false;
  return true;
}

}  // namespace bddc
