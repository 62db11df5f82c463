// Fused interior elimination for 2D subdomains (plane rows M <= 32, interface <= NGP), as a
// block LDL^T with explicit Schur-complement inverses (B_j = coupling stencil plane j -> j-1):
//   S_j = T_j - B_j W_{j-1} B_j^T ;  W_j = S_j^{-1}
//   R_j = A_IG,j - B_j H_{j-1}    ;  H_j = W_j R_j
//   S_G = A_GG - sum_j R_j^T H_j
// Two kernels:
//  * wfactor2d: the W recursion, one warp per subdomain (Gauss-Jordan sweep with lane =
//    column, __syncwarp only), writes packed W_j + the stencil (the apply's interior factor);
//  * schur2d: one CTA per subdomain, R_j / H_j / S_G on the FP64 tensor pipe
//    (mma.sync m8n8k4 -> DMMA.8x8x4), restricted to the active interface prefix of plane j
//    (in the lexicographic slot order, R_j and H_j vanish beyond slot nact[j]).
// Replaces btchol_kernel + 2 nblk batched GEMMs + the S_G GEMM of the generic path.
#include "stencil.cuh"

namespace bddc {

namespace {

constexpr int kWarpsW = 4;         // subdomains per CTA in wfactor2d
constexpr int kSchurThreads = 256;

// C(8x8 tile) += A(8 x K) B(K x 8); A(r,k) = A[r*ars + k*acs], B(k,c) = B[k*brs + c*bcs]
__device__ __forceinline__ void mma_acc(double& c0, double& c1, const double* A, int ars, int acs,
                                        const double* B, int brs, int bcs, int K, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll 4
  for (int k = 0; k < K; k += 4) {
    const double a = A[g * ars + (k + t) * acs];
    const double b = B[(k + t) * brs + g * bcs];
    dmma884(c0, c1, a, b);
  }
}

// C(8x8 tile) += A(8 x K) B(K x 8) with compile-time K and strides (immediate offsets)
template <int K, int ARS, int ACS, int BRS, int BCS>
__device__ __forceinline__ void mma_acc_t(double& c0, double& c1, const double* A, const double* B, int lane) {
  const int g = lane >> 2, t = lane & 3;
  const double* a = A + g * ARS + t * ACS;
  const double* b = B + t * BRS + g * BCS;
#pragma unroll
  for (int k = 0; k < K; k += 4) dmma884(c0, c1, a[k * ACS], b[k * BRS]);
}

// C(8x8 tile) += W(rows r0.., all K) B(K x 8) with W symmetric and only its lower triangle
// (row >= col, column-major, pitch P) stored: entries above the diagonal are read at their
// transposed position (a half-warp then touches t + 4g instead of g + 4t: still conflict-free)
template <int K, int P, int BRS>
__device__ __forceinline__ void mma_symlower(double& c0, double& c1, const double* W, int r0, const double* B, int lane) {
  const int g = lane >> 2, t = lane & 3, row = r0 + g;
  const double* b = B + t * BRS + g;
#pragma unroll
  for (int k = 0; k < K; k += 4) {
    const int kk = k + t;
    dmma884(c0, c1, W[row >= kk ? row + kk * P : kk + row * P], b[k * BRS]);
  }
}

// Pitch (doubles) of a square operand read as DMMA fragments A(r, k) = X[r + k P]: a half-warp
// (g, t in 0..3) touches g + t P, conflict-free iff P = 4 or 12 mod 16 (M + 1 gives 2-4 way
// conflicts: the dominant stall of schur2d / rh3d in the ncu source counters)
constexpr int frag_pitch(int M) {
  int p = M + 1;
  while (p % 16 != 4 && p % 16 != 12) ++p;
  return p;
}

// Store a DMMA.8x8 accumulator (lane holds C[g][2t], C[g][2t+1]) into a row-major tile of
// pitch = 4 mod 16 doubles: odd rows store their second element first, so each of the two
// 64-bit store instructions hits 16 distinct bank pairs per half-warp (no 2-way conflict)
__device__ __forceinline__ void store_frag_rowmajor(double* C, int ldc, double c0, double c1, int lane) {
  const int g = lane >> 2, t = lane & 3, odd = g & 1;
  double* p = C + g * ldc + 2 * t;
  p[odd] = odd ? c1 : c0;
  p[odd ^ 1] = odd ? c0 : c1;
}

// lower-triangular 8x8 tile coordinates (I, J) of tile index tt = I(I+1)/2 + J (NGP <= 128)
__constant__ int2 c_lower_tiles[16 * 17 / 2];

// ---- W recursion (one warp per subdomain) ----
// W pitch = 4 mod 16 doubles: conflict-free 8x8x4 DMMA fragments; pivot-inverse pitch 20
template <int M>
constexpr int wpitch() { return M <= 16 ? 20 : (M <= 32 ? 36 : 68); }
constexpr int kDP = 20;
template <int M, bool DIAGB>
constexpr int wf_warp_doubles() { return (DIAGB ? 1 : 2) * M * wpitch<M>() + 8 * kDP; }

// C(8x8) -= / += A B from shared memory (A(r,k) = A[r*ars + k*acs], B(k,c) = B[k*brs + c*bcs])
__device__ __forceinline__ void mma8x8(double& c0, double& c1, const double* A, int ars, int acs,
                                       const double* B, int brs, int bcs, int lane) {
  const int g = lane >> 2, t = lane & 3;
  dmma884(c0, c1, A[g * ars + t * acs], B[t * brs + g * bcs]);
  dmma884(c0, c1, A[g * ars + (t + 4) * acs], B[(t + 4) * brs + g * bcs]);
}

// In-place inverse of the SPD M x M block W (column-major, pitch P) by blocked Gauss-Jordan
// over 8x8 blocks: the pivot block is inverted in registers (lanes 0..7 own its columns), the
// row / column / trailing block updates are DMMA.8x8x4 tiles. Returns the first bad pivot.
template <int M>
__device__ __forceinline__ int gj_inverse_blocked(double* W, double* Dm, int lane) {
  constexpr int P = wpitch<M>(), NB = M / 8;
  const int g = lane >> 2, t = lane & 3;
  int bad = -1;
#pragma unroll 1
  for (int kb = 0; kb < NB; ++kb) {
    const int K = kb * 8;
    // (1) Dinv = inverse of the pivot block (scalar Gauss-Jordan on 8 lanes, registers)
    {
      double col[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) col[i] = lane < 8 ? W[(K + i) + (K + lane) * P] : 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        double piv = __shfl_sync(0xffffffffu, col[c], c);
        if (!(piv > 0.0)) {
          if (bad < 0) bad = K + c;
          piv = 1.0;
        }
        const double ip = rcp_pos(piv);
        const double rk = col[c] * ip;  // row c of this lane's column, scaled
        double nc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double ci = __shfl_sync(0xffffffffu, col[i], c);
          if (i == c) nc[i] = lane == c ? ip : rk;
          else if (lane == c) nc[i] = -ci * ip;
          else nc[i] = fma(-ci, rk, col[i]);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) col[i] = nc[i];
      }
      if (lane < 8) {
#pragma unroll
        for (int i = 0; i < 8; ++i) Dm[i + lane * kDP] = col[i];
      }
    }
    __syncwarp();
    // (2) pivot row blocks: W[K][J] = Dinv W[K][J]
#pragma unroll
    for (int jb = 0; jb < NB; ++jb) {
      if (jb == kb) continue;
      const int J = jb * 8;
      double c0 = 0.0, c1 = 0.0;
      mma8x8(c0, c1, Dm, 1, kDP, W + K + J * P, 1, P, lane);
      __syncwarp();
      W[(K + g) + (J + 2 * t) * P] = c0;
      W[(K + g) + (J + 2 * t + 1) * P] = c1;
    }
    __syncwarp();
    // (3) trailing blocks: W[I][J] -= W[I][K] W[K][J]   (I, J != K; old column, new row)
#pragma unroll
    for (int ib = 0; ib < NB; ++ib) {
      if (ib == kb) continue;
      const int I = ib * 8;
#pragma unroll
      for (int jb = 0; jb < NB; ++jb) {
        if (jb == kb) continue;
        const int J = jb * 8;
        double d0 = 0.0, d1 = 0.0;
        mma8x8(d0, d1, W + I + K * P, 1, P, W + K + J * P, 1, P, lane);
        W[(I + g) + (J + 2 * t) * P] -= d0;
        W[(I + g) + (J + 2 * t + 1) * P] -= d1;
      }
    }
    __syncwarp();
    // (4) pivot column blocks: W[I][K] = -W[I][K] Dinv ; (5) W[K][K] = Dinv
#pragma unroll
    for (int ib = 0; ib < NB; ++ib) {
      if (ib == kb) continue;
      const int I = ib * 8;
      double d0 = 0.0, d1 = 0.0;
      mma8x8(d0, d1, W + I + K * P, 1, P, Dm, 1, kDP, lane);
      __syncwarp();
      W[(I + g) + (K + 2 * t) * P] = -d0;
      W[(I + g) + (K + 2 * t + 1) * P] = -d1;
    }
    for (int e = lane; e < 64; e += 32) W[(K + (e & 7)) + (K + (e >> 3)) * P] = Dm[(e & 7) + (e >> 3) * kDP];
    __syncwarp();
  }
  return bad;
}

template <int M, bool DIAGB>
__global__ void __launch_bounds__(32 * kWarpsW) wfactor2d_kernel(Geometry G, int sub0, int cnt,
                                                                 const double* __restrict__ alpha,
                                                                 LocalTables lt,
                                                                 double* __restrict__ LI,
                                                                 int* __restrict__ info) {
  constexpr int P = wpitch<M>();
  extern __shared__ __align__(16) double smw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * kWarpsW + warp;
  if (b >= cnt) return;
  const int sub = sub0 + b;
  // per warp: W_j (in place), pivot-block inverse, [X scratch for general stencils]
  double* W = smw + warp * wf_warp_doubles<M, DIAGB>();
  double* Dm = W + M * P;
  double* X = Dm + 8 * kDP;
  int p[3];
  sub_coords(G, sub, p);
  double* li = LI + (long long)sub * G.li_stride;
  double* bcg = li + (long long)G.nblk * G.Tm;
  const int px = G.blk[0] - 1;
  const int nbo = G.nbo;
  const int k = lane;  // owned column (general stencil path) / owned row (elsewhere)
  int failed = -1;
  for (int j = 0; j < G.nblk; ++j) {
    // this lane's row of plane j from the element stencil: T_j (in-plane, x-1 / x / x+1)
    // and the coupling B_j to plane j-1 (bc[k] for the nbo offsets)
    double t_m1 = 0.0, t_0 = 1.0, t_p1 = 0.0;  // identity on padding rows
    double cf[3] = {0.0, 0.0, 0.0};
    if (lane < G.m) {
      int a[3];
      local_coords(G, lt.irow_node[j * M + lane], a);
      const int d0[3] = {0, 0, 0}, dm[3] = {-1, 0, 0}, dp[3] = {1, 0, 0};
      t_0 = local_coef<2>(G, alpha, p, a, d0);
      if (lane > 0) t_m1 = local_coef<2>(G, alpha, p, a, dm);
      if (lane + 1 < G.m) t_p1 = local_coef<2>(G, alpha, p, a, dp);
      if (j > 0) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          if (q >= nbo) break;
          const int x = lane + G.bo_dx[q];
          const int dq[3] = {G.bo_dx[q], -1, 0};
          if (x >= 0 && x < px) cf[q] = local_coef<2>(G, alpha, p, a, dq);
        }
      }
    }
    // T_j[i][k] seen from row i = lane (tk) or, by symmetry, from column k = lane (ti)
    auto tk = [&](int kk) { return kk == lane ? t_0 : (kk == lane - 1 ? t_m1 : (kk == lane + 1 ? t_p1 : 0.0)); };
    if (lane < M) {
#pragma unroll
      for (int q = 0; q < 3; ++q)
        if (q < nbo) bcg[((long long)j * M + lane) * nbo + q] = cf[q];
    }
    if (j > 0 && DIAGB) {
      // B_j diagonal (P1): S_j[i][k] = T_j[i][k] - b_i W_{j-1}[i][k] b_k (lane = row i)
      if (lane < M) {
        const double bi = cf[0];
#pragma unroll 8
        for (int kk = 0; kk < M; ++kk) {
          const double bk = __shfl_sync(0xffffffffu >> (32 - M), cf[0], kk);
          W[lane + kk * P] = tk(kk) - bi * W[lane + kk * P] * bk;
        }
      }
    } else if (j > 0) {
      // X = B_j W_{j-1}: X[i][k] = sum_q cf_i[q] W[i + dx_q][k]  (cf of row i via shuffles)
      for (int i = 0; i < M; ++i) {
        double a = 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          if (q >= nbo) break;
          const double ci = __shfl_sync(0xffffffffu, cf[q], i);
          const int ii = i + G.bo_dx[q];
          if (ci != 0.0 && ii >= 0 && ii < M && k < M) a += ci * W[ii + k * P];
        }
        if (k < M) X[i + k * P] = a;
      }
      __syncwarp();
      // S_j = T_j - X B_j^T: S[i][k] = T[i][k] - sum_q X[i][k + dx_q] cf_k[q]
      for (int i = 0; i < M; ++i) {
        double a = 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          if (q >= nbo) break;
          const int kk = k + G.bo_dx[q];
          if (cf[q] != 0.0 && kk >= 0 && kk < M) a += X[i + kk * P] * cf[q];
        }
        if (k < M) W[i + k * P] = tk(i) - a;  // T symmetric: T[i][k] = T[k][i], k = lane
      }
    } else if (lane < M) {
      for (int kk = 0; kk < M; ++kk) W[lane + kk * P] = tk(kk);
    }
    __syncwarp();
    const int bad = gj_inverse_blocked<M>(W, Dm, lane);
    if (bad >= 0 && failed < 0) failed = j * M + bad;
    // packed W_j (column-major lower), lane = row i: coalesced per column
    if (lane < M) {
      double* lj = li + (long long)j * G.Tm;
      int cs = 0;
#pragma unroll 4
      for (int kk = 0; kk < M; ++kk) {
        if (kk <= lane) lj[cs + (lane - kk)] = W[lane + kk * P];
        cs += M - kk;
      }
    }
    __syncwarp();
  }
  if (lane == 0 && failed >= 0) atomicMin(info + sub, failed);
}

// ---- R_j / H_j / S_G with DMMA, W_j streamed back from the packed factor ----
template <int M, int NGP, int NBO>
__global__ void __launch_bounds__(kSchurThreads, 2) schur2d_kernel(Geometry G, int sub0,
                                                                const double* __restrict__ alpha,
                                                                LocalTables lt,
                                                                const double* __restrict__ LI,
                                                                double* __restrict__ LS) {
  constexpr int P = frag_pitch(M);
  constexpr int EP = NGP + 4;
  constexpr int NT = NGP / 8;
  constexpr int NLT = NT * (NT + 1) / 2;
  constexpr int NW = kSchurThreads / 32;
  constexpr int SYRK_PER_WARP = (NLT + NW - 1) / NW;
  constexpr int O_H = 0;               // H_{j-1} / H_j   (M x EP)
  constexpr int O_R = O_H + M * EP;    // A_IG,j -> R_j   (M x EP)
  constexpr int O_W = O_R + M * EP;    // W_j (square)
  constexpr int O_BC = O_W + M * P;    // stencil [M][3]
  constexpr int O_SL = O_BC + 3 * M;   // surface slot -> local node | Dirichlet bit (ints)
  extern __shared__ __align__(16) double sm[];
  int* slot_sm = reinterpret_cast<int*>(sm + O_SL);
  const int b = blockIdx.x, sub = sub0 + b;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  int p[3];
  sub_coords(G, sub, p);
  const double* li = LI + (long long)sub * G.li_stride;
  const double* bcg = li + (long long)G.nblk * G.Tm;
  const int nbo = G.nbo;
  int bdx[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) bdx[q] = q < nbo ? G.bo_dx[q] : 0;

  double acc[SYRK_PER_WARP][2];
#pragma unroll
  for (int q = 0; q < SYRK_PER_WARP; ++q) acc[q][0] = acc[q][1] = 0.0;
  for (int k = tid; k < G.nG; k += kSchurThreads) {
    const int node = lt.slot_node[k];
    int a[3];
    local_coords(G, node, a);
    slot_sm[k] = node | (local_to_free(G, p, a) < 0 ? (1 << 30) : 0);
  }
  int nprev = 0;
  for (int j = 0; j < G.nblk; ++j) {
    const int na = G.nact[j];           // active columns (multiple of 8)
    const int nat = na / 8;
    // W_j (unpack) and the coupling stencil: every global load of the plane is issued before
    // the first shared-memory store; A_IG rows (active columns) come from the element stencil
    {
      constexpr int TM = M * (M + 1) / 2;
      constexpr int NWL = (TM + kSchurThreads - 1) / kSchurThreads;
      double wv[NWL];
#pragma unroll
      for (int u = 0; u < NWL; ++u) {
        const int e = tid + u * kSchurThreads;
        wv[u] = e < TM ? li[(long long)j * G.Tm + e] : 0.0;
      }
      const double bv = tid < M * nbo ? bcg[(long long)j * M * nbo + tid] : 0.0;
      for (int r = warp; r < M; r += NW)
        for (int cc = lane; cc < na; cc += 32) sm[O_R + r * EP + cc] = 0.0;
#pragma unroll
      for (int u = 0; u < NWL; ++u) {
        const int e = tid + u * kSchurThreads;
        if (e < TM) {
          // column c of packed entry e: cs(c) = c M - c(c-1)/2 <= e < cs(c+1)
          const double q = 2.0 * M + 1.0;
          int c = (int)((q - sqrt(q * q - 8.0 * e)) * 0.5);
          if ((c + 1) * M - (c + 1) * c / 2 <= e) ++c;
          if (c * M - c * (c - 1) / 2 > e) --c;
          const int r = c + (e - (c * M - c * (c - 1) / 2));
          sm[O_W + r + c * P] = wv[u];  // lower triangle only (mma_symlower)
        }
      }
      if (tid < M * nbo) sm[O_BC + (tid / nbo) * 3 + tid % nbo] = bv;
      __syncthreads();
      // A_IG: row r of plane j couples to the (non-Dirichlet) surface slots among its 8
      // stencil neighbours
      for (int idx = tid; idx < G.m * 8; idx += kSchurThreads) {
        const int r = idx >> 3, o = idx & 7, oo = o < 4 ? o : o + 1;  // skip the centre
        int a[3];
        local_coords(G, lt.irow_node[j * M + r], a);
        const int d[3] = {oo % 3 - 1, oo / 3 - 1, 0};
        const int bn[3] = {a[0] + d[0], a[1] + d[1], 0};
        const int code = lt.node_code[bn[0] + (G.blk[0] + 1) * bn[1]];
        if (code >= 0) continue;
        const int slot = -code - 1;
        if (slot >= na || local_to_free(G, p, bn) < 0) continue;
        sm[O_R + r * EP + slot] = local_coef<2>(G, alpha, p, a, d);
      }
    }
    __syncthreads();
    if (j > 0) {  // R_j -= B_j H_{j-1} on the previously active columns (warp = row)
      for (int r = warp; r < M; r += NW) {
        double cf[NBO];
        int ro[NBO];
#pragma unroll
        for (int q = 0; q < NBO; ++q) {
          cf[q] = q < nbo ? sm[O_BC + r * 3 + q] : 0.0;
          ro[q] = min(max(r + bdx[q], 0), M - 1) * EP;  // absent neighbours have cf = 0
        }
        for (int cc = lane; cc < nprev; cc += 32) {
          double a = 0.0;
#pragma unroll
          for (int q = 0; q < NBO; ++q) a += cf[q] * sm[O_H + ro[q] + cc];
          sm[O_R + r * EP + cc] -= a;
        }
      }
      __syncthreads();
    }
    // H_j = W_j R_j (active column tiles)
    for (int tt = warp; tt < (M / 8) * nat; tt += NW) {
      const int ti = tt % (M / 8), tj = tt / (M / 8);
      double c0 = 0.0, c1 = 0.0;
      mma_symlower<M, P, EP>(c0, c1, sm + O_W, ti * 8, sm + O_R + tj * 8, lane);
      store_frag_rowmajor(sm + O_H + (ti * 8) * EP + tj * 8, EP, c0, c1, lane);
    }
    __syncthreads();
    // S_acc += R_j^T H_j on active lower tiles (I, J < nat)
    const int nlt_act = nat * (nat + 1) / 2;
#pragma unroll
    for (int q = 0; q < SYRK_PER_WARP; ++q) {
      const int tt = warp + q * NW;
      if (tt < nlt_act) {
        const int2 ij = c_lower_tiles[tt];
        mma_acc_t<M, 1, EP, EP, 1>(acc[q][0], acc[q][1], sm + O_R + ij.x * 8, sm + O_H + ij.y * 8, lane);
      }
    }
    nprev = na;
    __syncthreads();
  }
  // S_G = A_GG - S_acc (full symmetric). A_GG from the element stencil (the local Neumann
  // coupling of two surface slots, as assemble_local_kernel writes it: local_coef at the row
  // slot's node toward the column slot's node; identity on Dirichlet and padding slots)
  double* ls = LS + (long long)sub * G.nG_pad * G.nG_pad;
  const int ld = G.nG_pad;
  const int nx1 = G.blk[0] + 1;
  auto agg = [&](int r, int c) -> double {
    if (r >= G.nG || c >= G.nG) return r == c ? 1.0 : 0.0;
    const int sr = slot_sm[r], sc = slot_sm[c];
    const int nr = sr & ((1 << 30) - 1), nc = sc & ((1 << 30) - 1);
    const int a[3] = {nr % nx1, nr / nx1, 0};
    const int d[3] = {nc % nx1 - a[0], nc / nx1 - a[1], 0};
    if (d[0] < -1 || d[0] > 1 || d[1] < -1 || d[1] > 1) return 0.0;
    if ((sr | sc) >> 30) return r == c ? 1.0 : 0.0;
    return local_coef<2>(G, alpha, p, a, d);
  };
#pragma unroll
  for (int q = 0; q < SYRK_PER_WARP; ++q) {
    const int tt = warp + q * NW;
    if (tt >= NLT) continue;
    const int I = c_lower_tiles[tt].x, J = c_lower_tiles[tt].y;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int r = I * 8 + g, c = J * 8 + 2 * t4 + e;
      if (r >= c) {
        const double v = agg(r, c) - acc[q][e];
        ls[r + (long long)c * ld] = v;
        if (r != c) ls[c + (long long)r * ld] = v;
      }
    }
  }
}

template <int M, int NGP, int NBO>
void launch_schur2d(const Ctx& c, int sub0, int cnt, const double* Wd, const double* Wo,
                    const double* E, cudaStream_t s) {
  const bool diagb = c.geo.nbo == 1 && c.geo.bo_dx[0] == 0;
  const size_t smem_w = sizeof(double) * kWarpsW * (diagb ? wf_warp_doubles<M, true>() : wf_warp_doubles<M, false>());
  const size_t smem_s = sizeof(double) * (2 * M * (NGP + 4) + M * frag_pitch(M) + 3 * M + NGP / 2);
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    int2 tiles[16 * 17 / 2];
    for (int I = 0, t = 0; I < 16; ++I)
      for (int J = 0; J <= I; ++J) tiles[t++] = make_int2(I, J);
    BDDC_CUDA(cudaMemcpyToSymbol(c_lower_tiles, tiles, sizeof(tiles)));
    BDDC_CUDA(cudaFuncSetAttribute(wfactor2d_kernel<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(sizeof(double) * kWarpsW * wf_warp_doubles<M, true>())));
    BDDC_CUDA(cudaFuncSetAttribute(wfactor2d_kernel<M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(sizeof(double) * kWarpsW * wf_warp_doubles<M, false>())));
    BDDC_CUDA(cudaFuncSetAttribute(schur2d_kernel<M, NGP, NBO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_s));
  }
  if (diagb) { wfactor2d_kernel<M, true><<<ceil_div(cnt, kWarpsW), 32 * kWarpsW, smem_w, s>>>(c.geo, sub0, cnt, c.alpha, c.lt, c.LI, c.info); BDDC_COUNT(); }
  else { wfactor2d_kernel<M, false><<<ceil_div(cnt, kWarpsW), 32 * kWarpsW, smem_w, s>>>(c.geo, sub0, cnt, c.alpha, c.lt, c.LI, c.info); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
  { schur2d_kernel<M, NGP, NBO><<<cnt, kSchurThreads, smem_s, s>>>(c.geo, sub0, c.alpha, c.lt, c.LI, c.LS); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
}


// ---- 3D (planes of m = (b-1)^2 rows, P1: diagonal coupling B_j to the plane below) ----
// wfactor3d: the W recursion S_j = T_j - B_j W_{j-1} B_j, W_j = S_j^{-1}, one warp per
// subdomain (lane owns rows lane, lane + 32); T_j comes from the in-plane element stencil.
constexpr int kWarps3 = 3;
template <int M>
constexpr int wf3_warp_doubles() { return M * wpitch<M>() + 8 * kDP + M; }

template <int M>
__global__ void __launch_bounds__(32 * kWarps3) wfactor3d_kernel(Geometry G, int sub0, int cnt,
                                                                 const double* __restrict__ alpha,
                                                                 LocalTables lt,
                                                                 double* __restrict__ LI,
                                                                 int* __restrict__ info) {
  constexpr int P = wpitch<M>();
  constexpr int RPL = (M + 31) / 32;
  extern __shared__ __align__(16) double smw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * kWarps3 + warp;
  if (b >= cnt) return;
  const int sub = sub0 + b;
  double* W = smw + warp * wf3_warp_doubles<M>();
  double* Dm = W + M * P;
  double* bsh = Dm + 8 * kDP;
  int p[3];
  sub_coords(G, sub, p);
  double* li = LI + (long long)sub * G.li_stride;
  double* bcg = li + (long long)G.nblk * G.Tm;
  const int px = G.blk[0] - 1, py = G.blk[1] - 1;
  int failed = -1;
  for (int j = 0; j < G.nblk; ++j) {
    double tc[RPL][9], bi[RPL];
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int r = lane + 32 * q;
      bi[q] = 0.0;
#pragma unroll
      for (int o = 0; o < 9; ++o) tc[q][o] = 0.0;
      if (r < G.m) {
        int a[3];
        local_coords(G, lt.irow_node[j * M + r], a);
#pragma unroll
        for (int o = 0; o < 9; ++o) {
          const int dx = o % 3 - 1, dy = o / 3 - 1;
          const int x = r % px + dx, y = r / px + dy;
          if (x < 0 || x >= px || y < 0 || y >= py) continue;
          const int d[3] = {dx, dy, 0};
          tc[q][o] = local_coef<3>(G, alpha, p, a, d);
        }
        if (j > 0) {
          const int d[3] = {0, 0, -1};
          bi[q] = local_coef<3>(G, alpha, p, a, d);
        }
      } else if (r < M) {
        tc[q][4] = 1.0;  // identity on padding rows
      }
      if (r < M) {
        bcg[(long long)j * M + r] = bi[q];
        bsh[r] = bi[q];
      }
    }
    __syncwarp();
    // S_j = T_j - diag(b) W_{j-1} diag(b)  (rows owned by this lane)
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int i = lane + 32 * q;
      if (i >= M) continue;
      if (j > 0) {
        const double bq = bi[q];
#pragma unroll 8
        for (int k = 0; k < M; ++k) W[i + k * P] = -bq * W[i + k * P] * bsh[k];
      } else {
#pragma unroll 8
        for (int k = 0; k < M; ++k) W[i + k * P] = 0.0;
      }
#pragma unroll
      for (int o = 0; o < 9; ++o)
        if (tc[q][o] != 0.0) W[i + (i + (o % 3 - 1) + (o / 3 - 1) * px) * P] += tc[q][o];
    }
    __syncwarp();
    const int bad = gj_inverse_blocked<M>(W, Dm, lane);
    if (bad >= 0 && failed < 0) failed = j * M + bad;
    // packed W_j (column-major lower), lane = row i: coalesced per column
    double* lj = li + (long long)j * G.Tm;
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int i = lane + 32 * q;
      if (i >= M) continue;
      int cs = 0;
#pragma unroll 4
      for (int kk = 0; kk <= i; ++kk) {
        lj[cs + (i - kk)] = W[i + kk * P];
        cs += M - kk;
      }
    }
    __syncwarp();
  }
  if (lane == 0 && failed >= 0) atomicMin(info + sub, failed);
}

// rh3d: R_j = A_IG,j - B_j H_{j-1}, H_j = W_j R_j for one 64-column chunk of the interface
// (columns evolve independently), all planes; R~ / H~ (plane-stacked, nI_pad x nG_pad,
// column-major) feed S_G = A_GG - R~^T H~ (one staircase GEMM). Planes whose active prefix
// ends before the chunk are skipped; the rows a 16-aligned GEMM k-slice reads below the
// chunk's first active plane are zeroed.
constexpr int kRh3Threads = 256;
template <int M>
__global__ void __launch_bounds__(kRh3Threads, 2) rh3d_kernel(Geometry G, int sub0,
                                                            const double* __restrict__ alpha,
                                                            LocalTables lt,
                                                            const double* __restrict__ LI,
                                                            double* __restrict__ Rt,
                                                            double* __restrict__ Ht, long long sE) {
  constexpr int P = frag_pitch(M);
  constexpr int CW = 64, EP = CW + 4;
  constexpr int NW = kRh3Threads / 32;
  extern __shared__ __align__(16) double sm[];
  double* Wsm = sm;               // M x P
  double* R = Wsm + M * P;        // M x EP (row-major)
  double* H = R + M * EP;         // M x EP
  double* bsh = H + M * EP;       // M
  const int c0 = blockIdx.x * CW;
  const int w = min(CW, G.nG_pad - c0);
  const int b = blockIdx.y, sub = sub0 + b;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  int p[3];
  sub_coords(G, sub, p);
  const double* li = LI + (long long)sub * G.li_stride;
  const double* bcg = li + (long long)G.nblk * G.Tm;
  double* rt = Rt + b * sE;
  double* ht = Ht + b * sE;
  const int ld = G.nI_pad;
  const int n0 = G.blk[0] + 1, n1 = G.blk[1] + 1;
  for (int idx = tid; idx < M * EP; idx += kRh3Threads) H[idx] = 0.0;
  int jmin = 0;
  while (jmin < G.nblk && G.nact[jmin] <= c0) ++jmin;
  {  // zero the k-slice rows below the first active plane (see above)
    const int r1 = jmin * M, r0 = r1 & ~15;
    for (int idx = tid; idx < (r1 - r0) * w; idx += kRh3Threads) {
      const int r = r0 + idx % (r1 - r0), c = c0 + idx / (r1 - r0);
      rt[r + (long long)c * ld] = 0.0;
      ht[r + (long long)c * ld] = 0.0;
    }
  }
  for (int j = jmin; j < G.nblk; ++j) {
    {  // W_j unpacked (symmetric) and the coupling to plane j-1; R_j <- 0
      // 4 threads per column c walk its packed entries (column start c M - c (c - 1) / 2)
      if (tid < 4 * M) {
        const int c = tid >> 2, q = tid & 3;
        const double* col = li + (long long)j * G.Tm + (c * M - c * (c - 1) / 2) - c;
        for (int r = c + q; r < M; r += 4) {
          Wsm[r + c * P] = col[r];  // lower triangle only (mma_symlower)
        }
      }
      // R_j <- -B_j H_{j-1} (B_j diagonal; zero on the chunk's first active plane)
      for (int r = warp; r < M; r += NW) {
        const double br = j > jmin ? bcg[(long long)j * M + r] : 0.0;
        for (int c = lane; c < w; c += 32) R[r * EP + c] = -br * H[r * EP + c];
      }
    }
    __syncthreads();
    // R_j += A_IG,j on the chunk: row r couples to the non-Dirichlet surface slots among its
    // 6 face neighbours (P1: schur3d_supported)
    for (int idx = tid; idx < G.m * 6; idx += kRh3Threads) {
      const int r = idx / 6, o = G.nb_code[idx % 6];
      int a[3];
      local_coords(G, lt.irow_node[j * M + r], a);
      const int d[3] = {o % 3 - 1, (o / 3) % 3 - 1, o / 9 - 1};
      const int bn[3] = {a[0] + d[0], a[1] + d[1], a[2] + d[2]};
      const int code = lt.node_code[bn[0] + n0 * (bn[1] + n1 * bn[2])];
      if (code >= 0) continue;
      const int slot = -code - 1 - c0;
      if (slot < 0 || slot >= w || local_to_free(G, p, bn) < 0) continue;
      R[r * EP + slot] += local_coef<3>(G, alpha, p, a, d);
    }
    __syncthreads();
    // H_j = W_j R_j
    for (int tt = warp; tt < (M / 8) * (w / 8); tt += NW) {
      const int ti = tt % (M / 8), tj = tt / (M / 8);
      double d0 = 0.0, d1 = 0.0;
      mma_symlower<M, P, EP>(d0, d1, Wsm, ti * 8, R + tj * 8, lane);
      store_frag_rowmajor(H + (ti * 8) * EP + tj * 8, EP, d0, d1, lane);
    }
    __syncthreads();
    for (int idx = tid; idx < M * w; idx += kRh3Threads) {
      const int r = idx % M, c = idx / M;
      const long long o = (long long)(j * M + r) + (long long)(c0 + c) * ld;
      rt[o] = R[r * EP + c];
      ht[o] = H[r * EP + c];
    }
    __syncthreads();
  }
}
}  // namespace

bool schur2d_supported(const Geometry& G) {
  if (G.dim != 2 || G.nbo > 3) return false;
  return (G.m_pad == 32 && G.nG_pad == 128) || (G.m_pad == 16 && G.nG_pad == 64) ||
         (G.m_pad == 8 && G.nG_pad == 32);
}

// Returns false if the geometry is not covered by a compiled instance.
bool schur2d(const Ctx& c, int sub0, int cnt, const double* Wd, const double* Wo, const double* E,
             cudaStream_t s) {
  const Geometry& G = c.geo;
  if (G.dim != 2 || G.nbo > 3) return false;
  const bool one = G.nbo == 1;
  if (G.m_pad == 32 && G.nG_pad == 128) {
    if (one) launch_schur2d<32, 128, 1>(c, sub0, cnt, Wd, Wo, E, s);
    else launch_schur2d<32, 128, 3>(c, sub0, cnt, Wd, Wo, E, s);
  } else if (G.m_pad == 16 && G.nG_pad == 64) {
    if (one) launch_schur2d<16, 64, 1>(c, sub0, cnt, Wd, Wo, E, s);
    else launch_schur2d<16, 64, 3>(c, sub0, cnt, Wd, Wo, E, s);
  } else if (G.m_pad == 8 && G.nG_pad == 32) {
    if (one) launch_schur2d<8, 32, 1>(c, sub0, cnt, Wd, Wo, E, s);
    else launch_schur2d<8, 32, 3>(c, sub0, cnt, Wd, Wo, E, s);
  } else {
    return false;
  }
  return true;
}


bool schur3d_supported(const Geometry& G) {
  return G.dim == 3 && G.nbo == 1 && G.bo_dx[0] == 0 && G.bo_dy[0] == 0 && G.nnb == 6 &&
         G.m_pad == 56 && G.nG_pad <= 1024;
}

// 3D interior elimination: packed W_j into LI (the apply's interior factor), R~ / H~ into
// Rt / Ht (cnt x sE doubles each), and the staircase K table of S_G = A_GG - R~^T H~.
void schur3d(const Ctx& c, int sub0, int cnt, double* Rt, double* Ht, long long sE, int* klo,
             cudaStream_t s) {
  const Geometry& G = c.geo;
  constexpr int M = 56;
  const size_t smem_w = sizeof(double) * kWarps3 * wf3_warp_doubles<M>();
  const size_t smem_r = sizeof(double) * (M * frag_pitch(M) + 2 * M * 68 + M);
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    BDDC_CUDA(cudaFuncSetAttribute(wfactor3d_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_w));
    BDDC_CUDA(cudaFuncSetAttribute(rh3d_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_r));
  }
  { wfactor3d_kernel<M><<<ceil_div(cnt, kWarps3), 32 * kWarps3, smem_w, s>>>(G, sub0, cnt, c.alpha, c.lt, c.LI, c.info); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
  dim3 grid(ceil_div(G.nG_pad, 64), cnt);
  { rh3d_kernel<M><<<grid, kRh3Threads, smem_r, s>>>(G, sub0, c.alpha, c.lt, c.LI, Rt, Ht, sE); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
  for (int i = 0; i < ceil_div(G.nG_pad, 64); ++i) {
    int j = 0;
    while (j < G.nblk && G.nact[j] <= 64 * i) ++j;
    klo[i] = j * M;
  }
}

}  // namespace bddc
