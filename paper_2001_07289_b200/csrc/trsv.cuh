// CTA-level blocked triangular solves with a column-major lower panel L (nrows x ncols,
// nrows >= ncols) and the vector x in shared memory:
//   forward:  solves L[0:nc,0:nc] x[0:nc] = x[0:nc], then x[nc:nr] -= L[nc:nr,0:nc] x[0:nc]
//   backward: solves L[0:nc,0:nc]^T x[0:nc] = x[0:nc] - L[nc:nr,0:nc]^T x[nc:nr]
// 64-row diagonal blocks are staged in shared memory and solved by warp 0 with shuffles;
// the off-diagonal parts are coalesced GEMVs over all threads.
#pragma once
#include "common.cuh"

namespace bddc {

constexpr int kTrsvB = 64;
constexpr int kTrsvP = kTrsvB + 1;

// dblk: shared scratch of kTrsvB * kTrsvP doubles.
__device__ inline void cta_trsv_fwd(const double* __restrict__ L, long long ld, int nr, int nc,
                                    double* x, double* dblk) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
  for (int kb = 0; kb < nc; kb += kTrsvB) {
    const int nb = min(kTrsvB, nc - kb);
    for (int idx = tid; idx < nb * nb; idx += nt) {
      const int i = idx % nb, k = idx / nb;
      dblk[i + k * kTrsvP] = i >= k ? L[(kb + i) + (kb + k) * ld] : 0.0;
    }
    __syncthreads();
    if (tid < 32) {
      double x0 = lane < nb ? x[kb + lane] : 0.0;
      double x1 = lane + 32 < nb ? x[kb + lane + 32] : 0.0;
      for (int k = 0; k < nb; ++k) {
        const double mine = k < 32 ? x0 : x1;
        double xk = __shfl_sync(0xffffffffu, mine, k & 31) / dblk[k + k * kTrsvP];
        if (lane == (k & 31)) {
          if (k < 32) x0 = xk; else x1 = xk;
        }
        if (lane > k) x0 -= dblk[lane + k * kTrsvP] * xk;
        if (lane + 32 > k && lane + 32 < nb) x1 -= dblk[lane + 32 + k * kTrsvP] * xk;
      }
      if (lane < nb) x[kb + lane] = x0;
      if (lane + 32 < nb) x[kb + lane + 32] = x1;
    }
    __syncthreads();
    for (int i = kb + nb + tid; i < nr; i += nt) {
      double s0 = 0.0, s1 = 0.0;
      int k = 0;
      for (; k + 1 < nb; k += 2) {
        s0 += L[i + (kb + k) * ld] * x[kb + k];
        s1 += L[i + (kb + k + 1) * ld] * x[kb + k + 1];
      }
      if (k < nb) s0 += L[i + (kb + k) * ld] * x[kb + k];
      x[i] -= s0 + s1;
    }
    __syncthreads();
  }
}

__device__ inline void cta_trsv_bwd(const double* __restrict__ L, long long ld, int nr, int nc,
                                    double* x, double* dblk) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int nblk = (nc + kTrsvB - 1) / kTrsvB;
  for (int b = nblk - 1; b >= 0; --b) {
    const int kb = b * kTrsvB, nb = min(kTrsvB, nc - kb);
    // x_blk -= L[below, blk]^T x_below  (warp per column, lanes over rows)
    for (int k = warp; k < nb; k += nw) {
      const double* col = L + (kb + k) * ld;
      double acc = 0.0;
      for (int i = kb + nb + lane; i < nr; i += 32) acc += col[i] * x[i];
      acc = warp_sum(acc);
      if (lane == 0) x[kb + k] -= acc;
    }
    for (int idx = tid; idx < nb * nb; idx += nt) {
      const int i = idx % nb, k = idx / nb;
      dblk[i + k * kTrsvP] = i >= k ? L[(kb + i) + (kb + k) * ld] : 0.0;
    }
    __syncthreads();
    if (tid < 32) {
      double x0 = lane < nb ? x[kb + lane] : 0.0;
      double x1 = lane + 32 < nb ? x[kb + lane + 32] : 0.0;
      for (int k = nb - 1; k >= 0; --k) {
        const double mine = k < 32 ? x0 : x1;
        double xk = __shfl_sync(0xffffffffu, mine, k & 31) / dblk[k + k * kTrsvP];
        if (lane == (k & 31)) {
          if (k < 32) x0 = xk; else x1 = xk;
        }
        // rows i < k: x_i -= L[k][i] x_k
        if (lane < k) x0 -= dblk[k + lane * kTrsvP] * xk;
        if (lane + 32 < k) x1 -= dblk[k + (lane + 32) * kTrsvP] * xk;
      }
      if (lane < nb) x[kb + lane] = x0;
      if (lane + 32 < nb) x[kb + lane + 32] = x1;
    }
    __syncthreads();
  }
}

}  // namespace bddc
