// Fused interior elimination for 2D subdomains (block rows of M <= 32, interface <= NGP):
// one CTA per subdomain runs the whole plane recursion on chip as a block LDL^T with
// explicit Schur-complement inverses (B_j = coupling stencil of plane j to plane j-1):
//   S_j = T_j - B_j W_{j-1} B_j^T ;  W_j = S_j^{-1}  (Gauss-Jordan sweep, one barrier/pivot)
//   R_j = A_IG,j - B_j H_{j-1}    ;  H_j = W_j R_j  (DMMA)
//   S_G = A_GG - sum_j R_j^T H_j                    (lower 8x8 tiles in registers, DMMA)
// The B_j products are stencil operations (1 coefficient per row for P1, 3 for Q1). It
// replaces btchol_kernel + 2 nblk batched GEMM launches + the S_G GEMM of the generic
// path and writes packed W_j + the coupling stencil (LI) and S_G (LS, full).
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
  constexpr int EP = NGP + 4;    // pitch of M x NGP blocks, row-major E[k*EP + col]
  constexpr int NT = NGP / 8;    // interface tiles per dimension
  constexpr int NLT = NT * (NT + 1) / 2;
  constexpr int NW = kSchurThreads / 32;
  constexpr int SYRK_PER_WARP = (NLT + NW - 1) / NW;
  constexpr int ET = (M / 8) * NT;  // 8x8 tiles of an M x NGP block
  extern __shared__ __align__(16) double sm[];
  double* Ha = sm;                 // H_{j-1} / H_j   (M x EP)
  double* Rb = Ha + M * EP;        // A_IG,j -> R_j   (M x EP)
  double* Ww = Rb + M * EP;        // T_j -> S_j -> W_j = S_j^{-1}
  double* Wp = Ww + M * P;         // W_{j-1}
  double* Xs = Wp + M * P;         // B_j W_{j-1} (general stencils)
  double* bcs = Xs + M * P;        // B_j stencil [M][nbo]
  double* rb = bcs + M * 9;        // Gauss-Jordan row / column buffers, 2 parities
  double* cb = rb + 2 * M;
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
  const int nbo = G.nbo;
  if (tid == 0) failed = -1;

  double acc[SYRK_PER_WARP][2];
#pragma unroll
  for (int q = 0; q < SYRK_PER_WARP; ++q) acc[q][0] = acc[q][1] = 0.0;

  for (int j = 0; j < G.nblk; ++j) {
    // ---- load T_j, the B_j stencil, A_IG rows of plane j ----
    for (int idx = tid; idx < M * M; idx += kSchurThreads) Ww[idx % M + (idx / M) * P] = wd[j * mm + idx];
    for (int idx = tid; idx < M * nbo; idx += kSchurThreads) {
      const int r = idx / nbo, k = idx % nbo;
      double v = 0.0;
      if (j > 0 && r < G.m) {
        const int x = r % px + G.bo_dx[k];
        if (x >= 0 && x < px) v = wo[j * mm + r + (long long)x * M];
      }
      bcs[r * 9 + k] = v;
      bcg[((long long)j * M + r) * nbo + k] = v;
    }
    for (int idx = tid; idx < M * NGP; idx += kSchurThreads) {
      const int r = idx % M, cc = idx / M;
      Rb[r * EP + cc] = eg[(j * M + r) + (long long)cc * G.nI_pad];
    }
    __syncthreads();
    if (j > 0) {
      // ---- S_j = T_j - B_j W_{j-1} B_j^T ;  R_j = A_IG,j - B_j H_{j-1} (stencil ops) ----
      for (int idx = tid; idx < M * M; idx += kSchurThreads) {  // X = B W
        const int r = idx % M, c = idx / M;
        double a = 0.0;
        for (int k = 0; k < nbo; ++k) {
          const double cf = bcs[r * 9 + k];
          if (cf != 0.0) a += cf * Wp[(r % px + G.bo_dx[k]) + c * P];
        }
        Xs[r + c * P] = a;
      }
      for (int idx = tid; idx < M * NGP; idx += kSchurThreads) {
        const int r = idx / NGP, cc = idx % NGP;
        double a = 0.0;
        for (int k = 0; k < nbo; ++k) {
          const double cf = bcs[r * 9 + k];
          if (cf != 0.0) a += cf * Ha[(r % px + G.bo_dx[k]) * EP + cc];
        }
        Rb[r * EP + cc] -= a;
      }
      __syncthreads();
      for (int idx = tid; idx < M * M; idx += kSchurThreads) {  // S -= X B^T
        const int r = idx % M, c = idx / M;
        double a = 0.0;
        for (int k = 0; k < nbo; ++k) {
          const double cf = bcs[c * 9 + k];
          if (cf != 0.0) a += Xs[r + (c % px + G.bo_dx[k]) * P] * cf;
        }
        Ww[r + c * P] -= a;
      }
      __syncthreads();
    }
    // ---- W_j = S_j^{-1}: in-place Gauss-Jordan sweep, one barrier per pivot ----
    for (int idx = tid; idx < M; idx += kSchurThreads) {
      rb[idx] = Ww[0 + idx * P];
      cb[idx] = Ww[idx + 0 * P];
    }
    __syncthreads();
    for (int c = 0; c < M; ++c) {
      const int pa = c & 1;
      const double* rc = rb + pa * M;
      const double* cc = cb + pa * M;
      double* rn = rb + (pa ^ 1) * M;
      double* cn = cb + (pa ^ 1) * M;
      double piv = rc[c];
      if (!(piv > 0.0)) {
        if (tid == 0 && failed < 0) failed = j * M + c;
        piv = 1.0;
      }
      const double ip = 1.0 / piv;
      for (int idx = tid; idx < M * M; idx += kSchurThreads) {
        const int i = idx % M, k = idx / M;
        double v;
        if (i == c && k == c) v = ip;
        else if (i == c) v = rc[k] * ip;
        else if (k == c) v = -cc[i] * ip;
        else v = Ww[i + k * P] - cc[i] * rc[k] * ip;
        Ww[i + k * P] = v;
        if (i == c + 1) rn[k] = v;
        if (k == c + 1) cn[i] = v;
      }
      __syncthreads();
    }
    // packed W_j (lower, column-major) for the apply
    for (int idx = tid; idx < M * M; idx += kSchurThreads) {
      const int r = idx % M, c = idx / M;
      if (r >= c) li[(long long)j * G.Tm + c * M - c * (c - 1) / 2 + (r - c)] = Ww[r + c * P];
    }
    // ---- H_j = W_j R_j (into Ha) ----
    for (int tt = warp; tt < ET; tt += NW) {
      const int ti = tt % (M / 8), tj = tt / (M / 8);
      double c0 = 0.0, c1 = 0.0;
      mma_acc(c0, c1, Ww + ti * 8, 1, P, Rb + tj * 8, EP, 1, M, lane);
      Ha[(ti * 8 + g) * EP + tj * 8 + 2 * t4] = c0;
      Ha[(ti * 8 + g) * EP + tj * 8 + 2 * t4 + 1] = c1;
    }
    __syncthreads();
    // ---- S_acc += R_j^T H_j (lower interface tiles; = R^T W R, symmetric) ----
#pragma unroll
    for (int q = 0; q < SYRK_PER_WARP; ++q) {
      const int tt = warp + q * NW;
      if (tt < NLT) {
        int I = 0;
        while ((I + 1) * (I + 2) / 2 <= tt) ++I;
        const int J = tt - I * (I + 1) / 2;
        mma_acc(acc[q][0], acc[q][1], Rb + I * 8, 1, EP, Ha + J * 8, EP, 1, M, lane);
      }
    }
    { double* tmp = Wp; Wp = Ww; Ww = tmp; }
    __syncthreads();
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
  return sizeof(double) * (2 * M * (NGP + 4) + 3 * M * (M + 1) + 9 * M + 4 * M);
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
  if (G.dim != 2) return false;
  if (G.m_pad == 32 && G.nG_pad == 128) launch_schur2d<32, 128>(c, sub0, cnt, Wd, Wo, E, s);
  else if (G.m_pad == 16 && G.nG_pad == 64) launch_schur2d<16, 64>(c, sub0, cnt, Wd, Wo, E, s);
  else if (G.m_pad == 8 && G.nG_pad == 32) launch_schur2d<8, 32>(c, sub0, cnt, Wd, Wo, E, s);
  else return false;
  return true;
}

}  // namespace bddc
