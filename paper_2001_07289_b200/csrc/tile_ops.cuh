// Device-side tile building blocks shared by the batched kernels (dense_f64.cu) and the
// cooperative coarse engine (coarse_coop.cu).
#pragma once
#include <climits>

#include "dense_f64.cuh"

#ifdef BDDC_TILE_PROF
__device__ long long g_tile_marks[16];
#define TILE_MARK(i) \
  do { if (blockIdx.x == 0 && threadIdx.x == 0) g_tile_marks[i] = clock64(); } while (0)
#else
#define TILE_MARK(i) do { } while (0)
#endif

namespace bddc {
namespace tile {

constexpr int BM = 64, BN = 64, BK = 16;
constexpr int LDW = BM + 4;  // pitch of [k][m] / [k][n] tiles (m or n contiguous)
constexpr int LDK = BK + 4;  // pitch of [m][k] / [n][k] tiles (k contiguous)
constexpr int TILE_A = BK * LDW > BM * LDK ? BK * LDW : BM * LDK;
constexpr int TILE_B = TILE_A;

// Copy a pair of consecutive doubles (valid = 0, 1 or 2 of them) into shared memory.
__device__ __forceinline__ void copy_pair(double* dst, const double* src, int valid, bool al16) {
  if (al16) {
    cp_async16(dst, src, valid * 8);
  } else {
    cp_async8(dst, src, valid > 0 ? 8 : 0);
    cp_async8(dst + 1, valid > 1 ? src + 1 : src, valid > 1 ? 8 : 0);
  }
}

// Load a BM x BKT slice of op(A) (rows m0.., k0..) into shared memory.
//   !TA: A(m,k) = A[m + k*lda]  -> sm[k*LDW + m]
//    TA: A(m,k) = A[k + m*lda]  -> sm[m*(BKT+4) + k]
template <bool TA, int BKT = BK>
__device__ __forceinline__ void load_a(double* sm, const double* A, int lda, int M, int K, int m0,
                                       int k0, int tid, bool al) {
  constexpr int LDKT = BKT + 4, HK = BKT / 2;
#pragma unroll
  for (int it = 0; it < BKT / 4; ++it) {
    int c = tid + it * 128;
    if (!TA) {
      int k = c >> 5, m = (c & 31) * 2;
      int gm = m0 + m, gk = k0 + k;
      int valid = (gk < K) ? max(0, min(2, M - gm)) : 0;
      const double* src = valid ? A + gm + (long long)gk * lda : A;
      copy_pair(sm + k * LDW + m, src, valid, al);
    } else {
      int m = c / HK, k = (c % HK) * 2;
      int gm = m0 + m, gk = k0 + k;
      int valid = (gm < M) ? max(0, min(2, K - gk)) : 0;
      const double* src = valid ? A + gk + (long long)gm * lda : A;
      copy_pair(sm + m * LDKT + k, src, valid, al);
    }
  }
}

// Load a BKT x BN slice of op(B) (k0.., cols n0..).
//   !TB: B(k,n) = B[k + n*ldb]  -> sm[n*(BKT+4) + k]
//    TB: B(k,n) = B[n + k*ldb]  -> sm[k*LDW + n]
template <bool TB, int BKT = BK>
__device__ __forceinline__ void load_b(double* sm, const double* B, int ldb, int N, int K, int n0,
                                       int k0, int tid, bool al) {
  constexpr int LDKT = BKT + 4, HK = BKT / 2;
#pragma unroll
  for (int it = 0; it < BKT / 4; ++it) {
    int c = tid + it * 128;
    if (!TB) {
      int n = c / HK, k = (c % HK) * 2;
      int gn = n0 + n, gk = k0 + k;
      int valid = (gn < N) ? max(0, min(2, K - gk)) : 0;
      const double* src = valid ? B + gk + (long long)gn * ldb : B;
      copy_pair(sm + n * LDKT + k, src, valid, al);
    } else {
      int k = c >> 5, n = (c & 31) * 2;
      int gn = n0 + n, gk = k0 + k;
      int valid = (gk < K) ? max(0, min(2, N - gn)) : 0;
      const double* src = valid ? B + gn + (long long)gk * ldb : B;
      copy_pair(sm + k * LDW + n, src, valid, al);
    }
  }
}

template <int BKT>
constexpr int tile_doubles() { return BKT * LDW > BM * (BKT + 4) ? BKT * LDW : BM * (BKT + 4); }

constexpr int kGemmSmemDoubles = 4 * TILE_A;  // As[2] + Bs[2]
template <int NS, int BKT = BK>
constexpr int gemm_smem_doubles() { return 2 * NS * tile_doubles<BKT>(); }

// The DMMAs of one k-slice for the first NI x NJ accumulator blocks of a warp tile.
template <int NI, int NJ, bool TA, bool TB, int BKT>
__device__ __forceinline__ void mma_slice(double (&acc)[4][4][2], const double* as, const double* bs,
                                          int wm, int wn, int g, int q) {
  constexpr int LDKT = BKT + 4;
#pragma unroll
  for (int kk = 0; kk < BKT; kk += 4) {
    double af[NI], bf[NJ];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      int m = wm * 32 + i * 8 + g;
      af[i] = TA ? as[m * LDKT + kk + q] : as[(kk + q) * LDW + m];
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      int n = wn * 32 + j * 8 + g;
      bf[j] = TB ? bs[(kk + q) * LDW + n] : bs[n * LDKT + kk + q];
    }
#pragma unroll
    for (int i = 0; i < NI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
}

// One 64x64 output tile (rows m0.., cols n0..) of C = alpha op(A) op(B) + beta C over the
// full K range; 128 threads (4 warps, 2x2), DMMA.8x8x4 accumulators, NS-stage cp.async
// pipeline (NS - 1 k-slices in flight ahead of the one being multiplied).
// lower: only entries with row >= col are written.
// k_lo / k_hi (multiples of BK or K): the nonzero K range of this tile (triangular operands);
// mirror (with lower): also write C(c, r) = C(r, c) (symmetric result).
// PRED: a warp only issues the DMMAs of its 8-row / 8-column accumulator blocks that reach
// below row M / column N (ragged sizes: 392 = 6.125 tiles), and none for a warp tile entirely
// above the diagonal of a lower result.
template <bool TA, bool TB, int NS = 2, int BKT = BK, bool PRED = false>
__device__ __forceinline__ void gemm_tile(const double* A, int lda, const double* B, int ldb,
                                          double* C, int ldc, int M, int N, int K, int m0, int n0,
                                          double alpha, double beta, bool lower, double* smem,
                                          int k_lo = 0, int k_hi = -1, bool mirror = false) {
  static_assert(NS >= 2, "at least double buffering");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int g = lane >> 2, q = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // PRED: number of this warp's 8-row / 8-column accumulator blocks that are written
  int ni = 4, nj = 4;
  if (PRED) {
    ni = max(0, min(4, (M - m0 - wm * 32 + 7) >> 3));
    nj = max(0, min(4, (N - n0 - wn * 32 + 7) >> 3));
    if (lower && n0 + wn * 32 > m0 + wm * 32 + 31) ni = 0;  // warp tile above the diagonal
    if (ni == 0 || nj == 0) ni = nj = 0;
  }
  constexpr int TILE = tile_doubles<BKT>();
  const int kb0 = k_lo / BKT;
  const int nk = ((k_hi < 0 ? K : min(K, k_hi)) + BKT - 1) / BKT - kb0;
  const bool al_a = ((((unsigned long long)A) & 15) == 0) && ((lda & 1) == 0);
  const bool al_b = ((((unsigned long long)B) & 15) == 0) && ((ldb & 1) == 0);
  auto As = [&](int st) { return smem + st * TILE; };
  auto Bs = [&](int st) { return smem + (NS + st) * TILE; };
  // prologue: slices 0 .. NS-2
#pragma unroll
  for (int p = 0; p < NS - 1; ++p) {
    if (p < nk) {
      load_a<TA, BKT>(As(p), A, lda, M, K, m0, (kb0 + p) * BKT, tid, al_a);
      load_b<TB, BKT>(Bs(p), B, ldb, N, K, n0, (kb0 + p) * BKT, tid, al_b);
    }
    cp_async_commit();  // empty groups keep the group count uniform
  }
  for (int kt = 0; kt < nk; ++kt) {
    const int st = kt % NS;
    const int pf = kt + NS - 1;  // slice to prefetch into the stage freed last iteration
    // (one barrier per slice, with the prefetch issued after it, measured 1-5% slower on the
    // local GEMM phases and equal on the coarse engine: profiles/r02/ab/one_barrier)
    if (pf < nk) {
      load_a<TA, BKT>(As(pf % NS), A, lda, M, K, m0, (kb0 + pf) * BKT, tid, al_a);
      load_b<TB, BKT>(Bs(pf % NS), B, ldb, N, K, n0, (kb0 + pf) * BKT, tid, al_b);
    }
    cp_async_commit();
    cp_async_wait<NS - 1>();  // slice kt has landed
    __syncthreads();
    const double* as = As(st);
    const double* bs = Bs(st);
    if (!PRED) {
      mma_slice<4, 4, TA, TB, BKT>(acc, as, bs, wm, wn, g, q);
    } else {
      switch (ni * 4 + nj - 5) {  // warp-uniform; every case keeps static accumulator indices
#define BDDC_MMA_CASE(I, J) case (I) * 4 + (J) - 5: mma_slice<I, J, TA, TB, BKT>(acc, as, bs, wm, wn, g, q); break;
        BDDC_MMA_CASE(1, 1) BDDC_MMA_CASE(1, 2) BDDC_MMA_CASE(1, 3) BDDC_MMA_CASE(1, 4)
        BDDC_MMA_CASE(2, 1) BDDC_MMA_CASE(2, 2) BDDC_MMA_CASE(2, 3) BDDC_MMA_CASE(2, 4)
        BDDC_MMA_CASE(3, 1) BDDC_MMA_CASE(3, 2) BDDC_MMA_CASE(3, 3) BDDC_MMA_CASE(3, 4)
        BDDC_MMA_CASE(4, 1) BDDC_MMA_CASE(4, 2) BDDC_MMA_CASE(4, 3) BDDC_MMA_CASE(4, 4)
#undef BDDC_MMA_CASE
        default: break;  // nothing of this warp's tile is written
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  // epilogue in two halves of the warp tile (accumulator block rows 0-1, then 2-3): the C reads
  // of a half are all issued before its stores (no serial read-modify-write chain) while only
  // 32 registers hold C values next to the 64 accumulator registers
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    double cv[2][4][2];
    if (beta != 0.0) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int row = m0 + wm * 32 + (2 * h + i) * 8 + g;
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = n0 + wn * 32 + j * 8 + 2 * q + e;
            const bool ok = row < M && col < N && !(lower && col > row);
            cv[i][j][e] = ok ? __ldcg(C + row + (long long)col * ldc) : 0.0;
          }
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int row = m0 + wm * 32 + (2 * h + i) * 8 + g;
      if (row >= M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = n0 + wn * 32 + j * 8 + 2 * q + e;
          if (col >= N || (lower && col > row)) continue;
          double v = alpha * acc[2 * h + i][j][e];
          if (beta != 0.0) v += beta * cv[i][j][e];
          C[row + (long long)col * ldc] = v;
          if (mirror && row != col) C[col + (long long)row * ldc] = v;
        }
      }
    }
  }
}

// ---- blocked 64x64 Cholesky + inverse with 8x8 sub-blocks (128 threads) ----
// Shared layout: S 64 x 64 (pitch SP, col-major), X 64 x 64 (pitch SP) for L^{-1},
// per-warp 8x8 scratch. The 8x8 diagonal blocks are factored / inverted in registers by one
// warp with shuffles; panel solves, trailing updates and the inverse recursion are DMMA.8x8x4.
constexpr int SP = kTile + 4;  // pitch = 4 mod 16 doubles: conflict-free 8x8x4 fragments
// S (factor in the lower triangle, off-diagonal blocks of the inverse X transposed in the
// upper triangle), Xd (X's 8 diagonal 8x8 blocks), 2 Dv, 8 warp tmps: 43 KB, 5 tiles per SM
constexpr int kFactSmemDoubles = kTile * SP + 8 * 64 + 128 + 8 * 64;

// C(8x8) (+)= A(8x8) B(8x8) from shared memory; A(r,k)=A[r*ars+k*acs], B(k,c)=B[k*brs+c*bcs]
__device__ __forceinline__ void mma8(double& c0, double& c1, const double* A, int ars, int acs,
                                     const double* B, int brs, int bcs, int lane) {
  const int g = lane >> 2, t = lane & 3;
  dmma884(c0, c1, A[g * ars + t * acs], B[t * brs + g * bcs]);
  dmma884(c0, c1, A[g * ars + (t + 4) * acs], B[(t + 4) * brs + g * bcs]);
}

// FACTOR: factor the n x n lower tile L (ld, n <= 64) in place, then write L^{-1} to inv
// (64 x 64, ld 64, zero upper / padding). !FACTOR: L is already a factor; only invert.
// Returns the first failing local pivot or -1.
// Warp-level Cholesky + inverse of the 8x8 diagonal block at k0 (lanes 0..7 = rows), in
// registers: one rsqrt per pivot gives both the scaling and 1/L[c][c] for the inverse.
// Writes the factor into S (FACTOR), the inverse into Xd's block k0 / 8 and Dv (pitch 8).
template <bool FACTOR>
__device__ __forceinline__ void diag8(double* S, double* Xd, double* Dv, int k0, int lane,
                                      int* failed) {
  double row[8], rinv[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) row[c] = lane < 8 ? S[(k0 + lane) + (k0 + c) * SP] : 0.0;
  if (FACTOR) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      double d = __shfl_sync(0xffffffffu, row[c], c);
      if (!(d > 0.0)) {
        if (lane == 0 && *failed < 0) *failed = k0 + c;
        d = 1.0;
      }
      const double ri = rsqrt_pos(d);  // d > 0 here
      rinv[c] = ri;
      const double l = lane > c ? row[c] * ri : (lane == c ? d * ri : 0.0);
      row[c] = l;
#pragma unroll
      for (int k = c + 1; k < 8; ++k) {
        const double lk = __shfl_sync(0xffffffffu, l, k);
        if (lane >= k) row[k] -= l * lk;
      }
    }
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c) rinv[c] = 1.0 / __shfl_sync(0xffffffffu, row[c], c);
  }
  // lane c = column c of the inverse: x[r] = (delta_rc - sum_{m<r} L[r][m] x[m]) / L[r][r]
  double x[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    double acc = (r == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int m = 0; m < r; ++m) acc -= __shfl_sync(0xffffffffu, row[m], r) * x[m];
    x[r] = acc * rinv[r];
  }
  if (lane < 8) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (FACTOR) S[(k0 + lane) + (k0 + c) * SP] = c <= lane ? row[c] : 0.0;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      Dv[r + lane * 8] = r >= lane ? x[r] : 0.0;
      Xd[k0 * 8 + r + lane * 8] = r >= lane ? x[r] : 0.0;
    }
  }
}

// Cholesky + inverse of an n x n (n <= 64) SPD tile held in shared memory, blocked by 8x8
// DMMA blocks with one-block lookahead: while warps 1.. run the trailing update of step kb,
// warp 0 updates and factors diagonal block kb+1.
template <bool FACTOR = true>
__device__ __forceinline__ int potrf_trtri_tile(double* L, int ld, int n, double* inv, double* smem) {
  double* S = smem;                  // factor (lower) | X^T off-diagonal blocks (upper)
  double* Xd = smem + kTile * SP;    // X's diagonal 8x8 blocks (pitch 8)
  double* Dv = Xd + 8 * 64;          // 2 x (8x8) inverses of diagonal blocks (pitch 8)
  __shared__ int failed;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nw = nt >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int nb8 = (n + 7) >> 3, np = nb8 * 8;
  if (tid == 0) failed = -1;
  TILE_MARK(0);
  // 64x64 region, 16 independent loads in flight per thread per batch (identity padding)
#pragma unroll 1
  for (int u0 = 0; u0 < kTile * kTile; u0 += 16 * 128) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int idx = u0 + u * nt + tid, i = idx & 63, j = idx >> 6;
      v[u] = (i < n && j < n && i >= j) ? __ldcg(L + i + (long long)j * ld) : (i == j && i >= n ? 1.0 : 0.0);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int idx = u0 + u * nt + tid, i = idx & 63, j = idx >> 6;
      if (i < np && j < np) S[i + j * SP] = v[u];
    }
  }
  __syncthreads();
  TILE_MARK(1);
  if (warp == 0) diag8<FACTOR>(S, Xd, Dv, 0, lane, &failed);
  __syncthreads();
  TILE_MARK(2);
  for (int kb = 0; kb < nb8; ++kb) {
    const int k0 = kb * 8;
    if (!FACTOR) {
      if (kb + 1 < nb8) {
        if (warp == 0) diag8<FACTOR>(S, Xd, Dv, k0 + 8, lane, &failed);
        __syncthreads();
      }
      continue;
    }
    const double* Dcur = Dv + (kb & 1) * 64;
    // (2) panel below: L[ib][kb] = S[ib][kb] Dinv^T
    for (int ib = kb + 1 + warp; ib < nb8; ib += nw) {
      double c0 = 0.0, c1 = 0.0;
      mma8(c0, c1, S + ib * 8 + k0 * SP, 1, SP, Dcur, 8, 1, lane);  // B(k,c) = Dinv[c][k]
      __syncwarp();
      S[(ib * 8 + g) + (k0 + 2 * t4) * SP] = c0;
      S[(ib * 8 + g) + (k0 + 2 * t4 + 1) * SP] = c1;
    }
    __syncthreads();
    // (3) trailing update S[ib][jb] -= L[ib][kb] L[jb][kb]^T  (kb < jb <= ib); task 0 is the
    // next diagonal block, done by warp 0 followed by its factorization (lookahead).
    const int nr = nb8 - kb - 1;
    const int ntask = nr * (nr + 1) / 2;
    if (warp == 0 && nr > 0) {
      const int I = kb + 1;
      double c0 = 0.0, c1 = 0.0;
      mma8(c0, c1, S + I * 8 + k0 * SP, 1, SP, S + I * 8 + k0 * SP, SP, 1, lane);
      S[(I * 8 + g) + (I * 8 + 2 * t4) * SP] -= c0;
      S[(I * 8 + g) + (I * 8 + 2 * t4 + 1) * SP] -= c1;
      __syncwarp();
      diag8<FACTOR>(S, Xd, Dv + ((kb + 1) & 1) * 64, I * 8, lane, &failed);
    }
    const int w0 = nw > 1 ? 1 : 0, ws = nw > 1 ? nw - 1 : 1;
    if (warp >= w0) {
      for (int q = 1 + (warp - w0); q < ntask; q += ws) {
        int ib = 0;
        while ((ib + 1) * (ib + 2) / 2 <= q) ++ib;
        const int jb = q - ib * (ib + 1) / 2;
        const int I = kb + 1 + ib, J = kb + 1 + jb;
        double c0 = 0.0, c1 = 0.0;
        mma8(c0, c1, S + I * 8 + k0 * SP, 1, SP, S + J * 8 + k0 * SP, SP, 1, lane);
        S[(I * 8 + g) + (J * 8 + 2 * t4) * SP] -= c0;
        S[(I * 8 + g) + (J * 8 + 2 * t4 + 1) * SP] -= c1;
      }
    }
    __syncthreads();
  }
  TILE_MARK(3);
  // inverse recursion by block rows: X[i][k] = -X[i][i] sum_{m=k}^{i-1} L[i][m] X[m][k];
  // X block (m, k), m > k, lives transposed in S's (free) upper triangle: X[m8+r][k8+c] at
  // S[(k8 + c) + (m8 + r) SP]
  double* tmp = Dv + 128 + warp * 64;  // per-warp 8x8 scratch
  for (int ib = 1; ib < nb8; ++ib) {
    for (int kb = warp; kb < ib; kb += nt >> 5) {
      double c0 = 0.0, c1 = 0.0;
      mma8(c0, c1, S + ib * 8 + kb * 8 * SP, 1, SP, Xd + kb * 64, 1, 8, lane);
      for (int m = kb + 1; m < ib; ++m)
        mma8(c0, c1, S + ib * 8 + m * 8 * SP, 1, SP, S + kb * 8 + m * 8 * SP, SP, 1, lane);
      tmp[g + (2 * t4) * 8] = c0;
      tmp[g + (2 * t4 + 1) * 8] = c1;
      __syncwarp();
      double d0 = 0.0, d1 = 0.0;
      mma8(d0, d1, Xd + ib * 64, 1, 8, tmp, 1, 8, lane);
      S[(kb * 8 + 2 * t4) + (ib * 8 + g) * SP] = -d0;
      S[(kb * 8 + 2 * t4 + 1) + (ib * 8 + g) * SP] = -d1;
      __syncwarp();
    }
    __syncthreads();
  }
  TILE_MARK(4);
  if (FACTOR) {
    for (int idx = tid; idx < kTile * kTile; idx += nt) {
      const int i = idx & 63, j = idx >> 6;
      if (i < n && j < n && i >= j) L[i + (long long)j * ld] = S[i + j * SP];
    }
  }
  if (inv) {
    for (int idx = tid; idx < kTile * kTile; idx += nt) {
      const int i = idx & 63, j = idx >> 6;
      double v = 0.0;
      if (i < n && j < n && i >= j)
        v = (i >> 3) == (j >> 3) ? Xd[(i >> 3) * 64 + (i & 7) + 8 * (j & 7)] : S[j + i * SP];
      inv[idx] = v;
    }
  }
  __syncthreads();
  TILE_MARK(5);
  return failed;
}

// ---- 64x64 SPD inverse by blocked Gauss-Jordan (128 threads) ----
// D = M^{-1} for the n x n (n <= 64) SPD tile whose lower triangle is M (ld); D is 64 x 64
// (ld 64), zero outside n x n. 8x8 pivot blocks are inverted in registers by warp 0; the row,
// trailing and column block updates are DMMA.8x8x4 tiles over all warps. No square roots and
// no separate inverse recursion: the critical path is 8 register 8x8 inverses.
constexpr int kGjDP = 20;  // pitch of the 8x8 pivot inverse (4 mod 16)
constexpr int kGjSmemDoubles = kTile * SP + 8 * kGjDP + 8;

__device__ __forceinline__ int gj_tile_inverse(const double* M, int ld, int n, double* D, double* smem) {
  double* W = smem;              // 64 x 64, pitch SP
  double* Dm = smem + kTile * SP;
  __shared__ int failed;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  if (tid == 0) failed = -1;
  TILE_MARK(12);
  // full symmetric tile from the lower triangle (identity padding), 16 loads in flight
#pragma unroll 1
  for (int u0 = 0; u0 < kTile * kTile; u0 += 16 * 128) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int idx = u0 + u * nt + tid, i = idx & 63, j = idx >> 6;
      const int r = i >= j ? i : j, c = i >= j ? j : i;
      v[u] = (r < n) ? M[r + (long long)c * ld] : (i == j ? 1.0 : 0.0);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int idx = u0 + u * nt + tid, i = idx & 63, j = idx >> 6;
      W[i + j * SP] = v[u];
    }
  }
  __syncthreads();
  TILE_MARK(6);
#pragma unroll 1
  for (int kb = 0; kb < 8; ++kb) {
    const int K = kb * 8;
    if (kb == 1) TILE_MARK(7);
    if (warp == 0) {  // (1) Dinv = inverse of the 8x8 pivot block (lanes 0..7 own columns)
      double col[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) col[i] = lane < 8 ? W[(K + i) + (K + lane) * SP] : 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        double piv = __shfl_sync(0xffffffffu, col[c], c);
        if (!(piv > 0.0)) {
          if (lane == 0 && failed < 0) failed = K + c;
          piv = 1.0;
        }
        const double ip = rcp_pos(piv);
        const double rk = col[c] * ip;
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
        for (int i = 0; i < 8; ++i) Dm[i + lane * kGjDP] = col[i];
      }
    }
    __syncthreads();
    if (kb == 1) TILE_MARK(8);
    // (2) pivot row blocks: W[K][J] = Dinv W[K][J]   (J != K)
    for (int jb = warp; jb < 8; jb += nw) {
      if (jb == kb) continue;
      const int J = jb * 8;
      double c0 = 0.0, c1 = 0.0;
      mma8(c0, c1, Dm, 1, kGjDP, W + K + J * SP, 1, SP, lane);
      __syncwarp();
      W[(K + g) + (J + 2 * t4) * SP] = c0;
      W[(K + g) + (J + 2 * t4 + 1) * SP] = c1;
    }
    __syncthreads();
    if (kb == 1) TILE_MARK(9);
    // (3) trailing blocks: W[I][J] -= W[I][K] W[K][J]   (I, J != K)
    for (int q = warp; q < 64; q += nw) {
      const int ib = q >> 3, jb = q & 7;
      if (ib == kb || jb == kb) continue;
      const int I = ib * 8, J = jb * 8;
      double d0 = 0.0, d1 = 0.0;
      mma8(d0, d1, W + I + K * SP, 1, SP, W + K + J * SP, 1, SP, lane);
      W[(I + g) + (J + 2 * t4) * SP] -= d0;
      W[(I + g) + (J + 2 * t4 + 1) * SP] -= d1;
    }
    __syncthreads();
    if (kb == 1) TILE_MARK(10);
    // (4) pivot column blocks: W[I][K] = -W[I][K] Dinv ; W[K][K] = Dinv
    for (int ib = warp; ib < 8; ib += nw) {
      if (ib == kb) continue;
      const int I = ib * 8;
      double d0 = 0.0, d1 = 0.0;
      mma8(d0, d1, W + I + K * SP, 1, SP, Dm, 1, kGjDP, lane);
      __syncwarp();
      W[(I + g) + (K + 2 * t4) * SP] = -d0;
      W[(I + g) + (K + 2 * t4 + 1) * SP] = -d1;
    }
    if (tid < 64) W[(K + (tid & 7)) + (K + (tid >> 3)) * SP] = Dm[(tid & 7) + (tid >> 3) * kGjDP];
    __syncthreads();
  }
  TILE_MARK(11);
  for (int idx = tid; idx < kTile * kTile; idx += nt) {
    const int i = idx & 63, j = idx >> 6;
    D[idx] = (i < n && j < n) ? W[i + j * SP] : 0.0;
  }
  __syncthreads();
  return failed;
}

}  // namespace tile
}  // namespace bddc
