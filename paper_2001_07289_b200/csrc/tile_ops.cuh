// Device-side tile building blocks shared by the batched kernels (dense_f64.cu) and the
// cooperative coarse engine (coarse_coop.cu).
#pragma once
#include <climits>

#include "dense_f64.cuh"

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

// Load a BM x BK slice of op(A) (rows m0.., k0..) into shared memory.
//   !TA: A(m,k) = A[m + k*lda]  -> sm[k*LDW + m]
//    TA: A(m,k) = A[k + m*lda]  -> sm[m*LDK + k]
template <bool TA>
__device__ __forceinline__ void load_a(double* sm, const double* A, int lda, int M, int K, int m0,
                                       int k0, int tid, bool al) {
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    int c = tid + it * 128;
    if (!TA) {
      int k = c >> 5, m = (c & 31) * 2;
      int gm = m0 + m, gk = k0 + k;
      int valid = (gk < K) ? max(0, min(2, M - gm)) : 0;
      const double* src = valid ? A + gm + (long long)gk * lda : A;
      copy_pair(sm + k * LDW + m, src, valid, al);
    } else {
      int m = c >> 3, k = (c & 7) * 2;
      int gm = m0 + m, gk = k0 + k;
      int valid = (gm < M) ? max(0, min(2, K - gk)) : 0;
      const double* src = valid ? A + gk + (long long)gm * lda : A;
      copy_pair(sm + m * LDK + k, src, valid, al);
    }
  }
}

// Load a BK x BN slice of op(B) (k0.., cols n0..).
//   !TB: B(k,n) = B[k + n*ldb]  -> sm[n*LDK + k]
//    TB: B(k,n) = B[n + k*ldb]  -> sm[k*LDW + n]
template <bool TB>
__device__ __forceinline__ void load_b(double* sm, const double* B, int ldb, int N, int K, int n0,
                                       int k0, int tid, bool al) {
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    int c = tid + it * 128;
    if (!TB) {
      int n = c >> 3, k = (c & 7) * 2;
      int gn = n0 + n, gk = k0 + k;
      int valid = (gn < N) ? max(0, min(2, K - gk)) : 0;
      const double* src = valid ? B + gk + (long long)gn * ldb : B;
      copy_pair(sm + n * LDK + k, src, valid, al);
    } else {
      int k = c >> 5, n = (c & 31) * 2;
      int gn = n0 + n, gk = k0 + k;
      int valid = (gk < K) ? max(0, min(2, N - gn)) : 0;
      const double* src = valid ? B + gn + (long long)gk * ldb : B;
      copy_pair(sm + k * LDW + n, src, valid, al);
    }
  }
}


constexpr int kGemmSmemDoubles = 4 * TILE_A;  // As[2] + Bs[2]

// One 64x64 output tile (rows m0.., cols n0..) of C = alpha op(A) op(B) + beta C over the
// full K range; 128 threads (4 warps, 2x2), DMMA.8x8x4 accumulators, cp.async staging.
// lower: only entries with row >= col are written.
template <bool TA, bool TB>
__device__ __forceinline__ void gemm_tile(const double* A, int lda, const double* B, int ldb,
                                          double* C, int ldc, int M, int N, int K, int m0, int n0,
                                          double alpha, double beta, bool lower, double* smem) {
  double* As[2] = {smem, smem + TILE_A};
  double* Bs[2] = {smem + 2 * TILE_A, smem + 3 * TILE_A};
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int g = lane >> 2, q = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nk = (K + BK - 1) / BK;
  const bool al_a = ((((unsigned long long)A) & 15) == 0) && ((lda & 1) == 0);
  const bool al_b = ((((unsigned long long)B) & 15) == 0) && ((ldb & 1) == 0);
  if (nk > 0) {
    load_a<TA>(As[0], A, lda, M, K, m0, 0, tid, al_a);
    load_b<TB>(Bs[0], B, ldb, N, K, n0, 0, tid, al_b);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    const int st = kt & 1;
    if (kt + 1 < nk) {
      load_a<TA>(As[st ^ 1], A, lda, M, K, m0, (kt + 1) * BK, tid, al_a);
      load_b<TB>(Bs[st ^ 1], B, ldb, N, K, n0, (kt + 1) * BK, tid, al_b);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* as = As[st];
    const double* bs = Bs[st];
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int m = wm * 32 + i * 8 + g;
        af[i] = TA ? as[m * LDK + kk + q] : as[(kk + q) * LDW + m];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int n = wn * 32 + j * 8 + g;
        bf[j] = TB ? bs[(kk + q) * LDW + n] : bs[n * LDK + kk + q];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
  // epilogue: all C reads issued before any store (no serial read-modify-write chain)
  double cv[4][4][2];
  if (beta != 0.0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = m0 + wm * 32 + i * 8 + g;
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
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm * 32 + i * 8 + g;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = n0 + wn * 32 + j * 8 + 2 * q + e;
        if (col >= N || (lower && col > row)) continue;
        double v = alpha * acc[i][j][e];
        if (beta != 0.0) v += beta * cv[i][j][e];
        C[row + (long long)col * ldc] = v;
      }
    }
  }
}

// ---- blocked 64x64 Cholesky + inverse with 8x8 sub-blocks (128 threads) ----
// Shared layout: S 64 x 64 (pitch SP, col-major), X 64 x 64 (pitch SP) for L^{-1},
// per-warp 8x8 scratch. The 8x8 diagonal blocks are factored / inverted in registers by one
// warp with shuffles; panel solves, trailing updates and the inverse recursion are DMMA.8x8x4.
constexpr int SP = kTile + 4;  // pitch = 4 mod 16 doubles: conflict-free 8x8x4 fragments
constexpr int kFactSmemDoubles = 2 * kTile * SP + 128 + 8 * 64;  // S, X, 2 Dv, 8 warp tmps

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
// Writes the factor into S (FACTOR), the inverse into X's diagonal block and Dv (pitch 8).
template <bool FACTOR>
__device__ __forceinline__ void diag8(double* S, double* X, double* Dv, int k0, int lane,
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
      const double ri = rsqrt(d);
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
      X[(k0 + r) + (k0 + lane) * SP] = r >= lane ? x[r] : 0.0;
    }
  }
}

// Cholesky + inverse of an n x n (n <= 64) SPD tile held in shared memory, blocked by 8x8
// DMMA blocks with one-block lookahead: while warps 1.. run the trailing update of step kb,
// warp 0 updates and factors diagonal block kb+1.
template <bool FACTOR = true>
__device__ __forceinline__ int potrf_trtri_tile(double* L, int ld, int n, double* inv, double* smem) {
  double* S = smem;                  // factor
  double* X = smem + kTile * SP;     // inverse
  double* Dv = X + kTile * SP;       // 2 x (8x8) inverses of diagonal blocks (pitch 8)
  __shared__ int failed;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nw = nt >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int nb8 = (n + 7) >> 3, np = nb8 * 8;
  if (tid == 0) failed = -1;
  for (int j = warp; j < np; j += nw) {
    for (int i = lane; i < np; i += 32) {
      double v = 0.0;
      if (i < n && j < n) v = i >= j ? L[i + (long long)j * ld] : 0.0;
      else if (i == j) v = 1.0;  // identity padding
      S[i + j * SP] = v;
      X[i + j * SP] = 0.0;
    }
  }
  __syncthreads();
  if (warp == 0) diag8<FACTOR>(S, X, Dv, 0, lane, &failed);
  __syncthreads();
  for (int kb = 0; kb < nb8; ++kb) {
    const int k0 = kb * 8;
    if (!FACTOR) {
      if (kb + 1 < nb8) {
        if (warp == 0) diag8<FACTOR>(S, X, Dv, k0 + 8, lane, &failed);
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
      diag8<FACTOR>(S, X, Dv + ((kb + 1) & 1) * 64, I * 8, lane, &failed);
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
  // inverse recursion by block rows: X[i][k] = -X[i][i] sum_{m=k}^{i-1} L[i][m] X[m][k]
  double* tmp = Dv + 128 + warp * 64;  // per-warp 8x8 scratch
  for (int ib = 1; ib < nb8; ++ib) {
    for (int kb = warp; kb < ib; kb += nt >> 5) {
      double c0 = 0.0, c1 = 0.0;
      for (int m = kb; m < ib; ++m)
        mma8(c0, c1, S + ib * 8 + m * 8 * SP, 1, SP, X + m * 8 + kb * 8 * SP, 1, SP, lane);
      tmp[g + (2 * t4) * 8] = c0;
      tmp[g + (2 * t4 + 1) * 8] = c1;
      __syncwarp();
      double d0 = 0.0, d1 = 0.0;
      mma8(d0, d1, X + ib * 8 + ib * 8 * SP, 1, SP, tmp, 1, 8, lane);
      X[(ib * 8 + g) + (kb * 8 + 2 * t4) * SP] = -d0;
      X[(ib * 8 + g) + (kb * 8 + 2 * t4 + 1) * SP] = -d1;
      __syncwarp();
    }
    __syncthreads();
  }
  if (FACTOR) {
    for (int idx = tid; idx < n * n; idx += nt) {
      const int i = idx % n, j = idx / n;
      if (i >= j) L[i + (long long)j * ld] = S[i + j * SP];
    }
  }
  if (inv) {
    for (int idx = tid; idx < kTile * kTile; idx += nt) {
      const int i = idx % kTile, j = idx / kTile;
      inv[idx] = (i < n && j < n) ? X[i + j * SP] : 0.0;
    }
  }
  __syncthreads();
  return failed;
}

}  // namespace tile
}  // namespace bddc
