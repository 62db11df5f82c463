// Batched FP64 dense kernels (sm_100a). See dense_f64.cuh.
//
// GEMM: 64x64x16 CTA tile, 4 warps (2x2), 32x32 warp tile = 4x4 DMMA.8x8x4 accumulators,
// cp.async double-buffered shared-memory staging. Shared-memory pitches are chosen so the
// 64-bit fragment reads are bank-conflict free (pitch ≡ 4 mod 16 doubles).
#include <climits>

#include "dense_f64.cuh"
#include "tile_ops.cuh"

namespace bddc {

namespace {

using namespace tile;

struct TaskView {
  const double* A;
  const double* B;
  double* C;
  int M, N, K, lda, ldb, ldc;
};

__device__ __forceinline__ TaskView gemm_task(const GemmArgs& a, int b) {
  if (a.tasks) {
    const GemmTask& t = a.tasks[b];
    return TaskView{t.A, t.B, t.C, t.M, t.N, t.K, t.lda, t.ldb, t.ldc};
  }
  return TaskView{a.A + b * a.sA, a.B + b * a.sB, a.C + b * a.sC, a.M, a.N, a.K,
                  a.lda,          a.ldb,          a.ldc};
}

#ifndef BDDC_GEMM_STAGES
#define BDDC_GEMM_STAGES 2
#endif
#ifndef BDDC_GEMM_PRED
#define BDDC_GEMM_PRED 1
#endif
constexpr int kGemmStages = BDDC_GEMM_STAGES;
constexpr bool kGemmPred = BDDC_GEMM_PRED != 0;

// 4 CTAs per SM (128 registers; the two-half epilogue of gemm_tile keeps the kernel spill-free):
// cfg3 setup 70.24 -> 68.60 ms, cfg5 1547 -> 1535 ms against 3 CTAs (profiles/r02/ab/ctas4)
#ifndef BDDC_GEMM_CTAS
#define BDDC_GEMM_CTAS 4
#endif
template <bool TA, bool TB>
__global__ void __launch_bounds__(128, BDDC_GEMM_CTAS) gemm_f64_kernel(GemmArgs args) {
  extern __shared__ __align__(16) double smem[];
  const TaskView t = gemm_task(args, blockIdx.y);
  const int tiles_m = (t.M + BM - 1) / BM;
  const int tiles_n = (t.N + BN - 1) / BN;
  if ((int)blockIdx.x >= tiles_m * tiles_n) return;
  const int tm = blockIdx.x % tiles_m, tn = blockIdx.x / tiles_m;
  const int m0 = tm * BM, n0 = tn * BN;
  if (args.lower && n0 > m0 + BM - 1) return;  // tile strictly above the diagonal
  int k_lo = 0, k_hi = t.K;  // nonzero K range of the tile for triangular operands
  switch (args.tri) {
    case 1: k_hi = min(t.K, m0 + BM); break;  // op(A)(m, k) = 0 for k > m
    case 2: k_lo = m0; break;                  // op(A)(m, k) = 0 for k < m
    case 3: k_lo = n0; break;                  // op(B)(k, n) = 0 for k < n
    case 4: k_hi = min(t.K, n0 + BN); break;   // op(B)(k, n) = 0 for k > n
    default: break;
  }
  if (args.klo_on) k_lo = max(k_lo, args.klo[tm]);
  gemm_tile<TA, TB, kGemmStages, BK, kGemmPred>(t.A, t.lda, t.B, t.ldb, t.C, t.ldc, t.M, t.N, t.K, m0, n0, args.alpha,
                                 args.beta, args.lower != 0, smem, k_lo, k_hi, args.mirror != 0);
}

// ---------------------------------------------------------------------------------------
// tile kernels (n <= 64)
// ---------------------------------------------------------------------------------------
constexpr int TP = kTile + 1;  // odd pitch: conflict-free per-thread vectors

struct TileView {
  double* L;
  double* B;
  int n, ldl, ldb, nvec, id, offset;
  double* inv;
};

__device__ __forceinline__ TileView tile_task(const TileArgs& a, int b) {
  if (a.tasks) {
    const TileTask& t = a.tasks[b];
    return TileView{t.L, t.B, t.n, t.ldl, t.ldb, t.nvec, t.id, t.offset, t.inv};
  }
  return TileView{a.L + b * a.sL, a.B ? a.B + b * a.sB : nullptr, a.n, a.ldl, a.ldb, a.nvec, b,
                  a.offset, a.inv ? a.inv + b * a.sInv : nullptr};
}

// X = L^{-1} for a lower n x n tile (n <= 64), blocked 8x8 with DMMA (tile_ops.cuh).
__global__ void __launch_bounds__(128) trtri_tile_kernel(TileArgs args) {
  extern __shared__ __align__(16) double fsm[];
  const TileView t = tile_task(args, blockIdx.x);
  if (t.n <= 0 || !t.inv) return;
  potrf_trtri_tile<false>(t.L, t.ldl, t.n, t.inv, fsm);
}

// Cholesky of 64x64 diagonal tiles (blocked 8x8, DMMA) + their inverses (if args.inv).
__global__ void __launch_bounds__(128) potrf_tile_kernel(TileArgs args) {
  extern __shared__ __align__(16) double fsm[];
  const TileView t = tile_task(args, blockIdx.x);
  if (t.n <= 0) return;
  const int bad = potrf_trtri_tile(t.L, t.ldl, t.n, t.inv, fsm);
  if (threadIdx.x == 0 && bad >= 0 && args.info) atomicMin(&args.info[t.id], t.offset + bad);
}

// Each thread owns one right-hand-side vector (a row of B for right-side solves, a column
// for left-side solves); vectors are staged through shared memory with coalesced loads.
//   FORWARD  (LLN, RLT): x_j = (b_j - sum_{k<j} L[j][k] x_k) / L[j][j]
//   BACKWARD (LLT, RLN): x_j = (b_j - sum_{k>j} L[k][j] x_k) / L[j][j]
template <bool RIGHT, bool FORWARD>
__global__ void __launch_bounds__(64) trsm_tile_kernel(TileArgs args) {
  extern __shared__ double smem[];
  double* Ls = smem;              // kTile * TP
  double* V = smem + kTile * TP;  // 64 vectors * TP
  const TileView t = tile_task(args, blockIdx.y);
  const int n = t.n, tid = threadIdx.x;
  const int v0 = blockIdx.x * 64;
  if (v0 >= t.nvec || n <= 0) return;
  const int nv = min(64, t.nvec - v0);
  for (int idx = tid; idx < n * n; idx += 64) {
    int i = idx % n, j = idx / n;
    if (i >= j) Ls[i + j * TP] = t.L[i + (long long)j * t.ldl];
  }
  if (RIGHT) {  // B is nvec x n: vector r = row r
    for (int idx = tid; idx < 64 * n; idx += 64) {
      int r = idx % 64, k = idx / 64;
      if (r < nv) V[r * TP + k] = t.B[(v0 + r) + (long long)k * t.ldb];
    }
  } else {  // B is n x nvec: vector c = column c
    for (int idx = tid; idx < 64 * n; idx += 64) {
      int k = idx % n, c = idx / n;
      if (c < nv) V[c * TP + k] = t.B[k + (long long)(v0 + c) * t.ldb];
    }
  }
  __syncthreads();
  if (tid < nv) {
    double* x = V + tid * TP;
    if (FORWARD) {
      for (int j = 0; j < n; ++j) {
        double s0 = x[j], s1 = 0.0;
        int k = 0;
        for (; k + 1 < j; k += 2) {
          s0 -= Ls[j + k * TP] * x[k];
          s1 -= Ls[j + (k + 1) * TP] * x[k + 1];
        }
        if (k < j) s0 -= Ls[j + k * TP] * x[k];
        x[j] = (s0 + s1) / Ls[j + j * TP];
      }
    } else {
      for (int j = n - 1; j >= 0; --j) {
        double s0 = x[j], s1 = 0.0;
        int k = j + 1;
        for (; k + 1 < n; k += 2) {
          s0 -= Ls[k + j * TP] * x[k];
          s1 -= Ls[k + 1 + j * TP] * x[k + 1];
        }
        if (k < n) s0 -= Ls[k + j * TP] * x[k];
        x[j] = (s0 + s1) / Ls[j + j * TP];
      }
    }
  }
  __syncthreads();
  if (RIGHT) {
    for (int idx = tid; idx < 64 * n; idx += 64) {
      int r = idx % 64, k = idx / 64;
      if (r < nv) t.B[(v0 + r) + (long long)k * t.ldb] = V[r * TP + k];
    }
  } else {
    for (int idx = tid; idx < 64 * n; idx += 64) {
      int k = idx % n, c = idx / n;
      if (c < nv) t.B[k + (long long)(v0 + c) * t.ldb] = V[c * TP + k];
    }
  }
}

constexpr int kTrsmSmem = 2 * kTile * TP * (int)sizeof(double);

template <bool R, bool F>
void launch_trsm(const TileArgs& a, cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    BDDC_CUDA(cudaFuncSetAttribute(trsm_tile_kernel<R, F>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, kTrsmSmem));
  }
  int nvec = a.tasks ? a.max_nvec : a.nvec;
  if (nvec <= 0 || a.count <= 0) return;
  dim3 grid(ceil_div(nvec, 64), a.count);
  { trsm_tile_kernel<R, F><<<grid, 64, kTrsmSmem, s>>>(a); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
}

}  // namespace

void gemm(const GemmArgs& a, bool tA, bool tB, cudaStream_t s) {
  int M = a.tasks ? a.max_M : a.M, N = a.tasks ? a.max_N : a.N;
  if (M <= 0 || N <= 0 || a.count <= 0) return;
  dim3 grid(ceil_div(M, BM) * ceil_div(N, BN), a.count);
  constexpr int smem = gemm_smem_doubles<kGemmStages>() * (int)sizeof(double);
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    BDDC_CUDA(cudaFuncSetAttribute(gemm_f64_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    BDDC_CUDA(cudaFuncSetAttribute(gemm_f64_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    BDDC_CUDA(cudaFuncSetAttribute(gemm_f64_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    BDDC_CUDA(cudaFuncSetAttribute(gemm_f64_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  }
  if (!tA && !tB) { gemm_f64_kernel<false, false><<<grid, 128, smem, s>>>(a); BDDC_COUNT(); }
  else if (!tA && tB) { gemm_f64_kernel<false, true><<<grid, 128, smem, s>>>(a); BDDC_COUNT(); }
  else if (tA && !tB) { gemm_f64_kernel<true, false><<<grid, 128, smem, s>>>(a); BDDC_COUNT(); }
  else { gemm_f64_kernel<true, true><<<grid, 128, smem, s>>>(a); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
}

void potrf_tile(const TileArgs& a, cudaStream_t s) {
  if (a.count <= 0) return;
  constexpr int smem = kFactSmemDoubles * (int)sizeof(double);
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    BDDC_CUDA(cudaFuncSetAttribute(potrf_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  }
  { potrf_tile_kernel<<<a.count, 128, smem, s>>>(a); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
}

void trtri_tile(const TileArgs& a, cudaStream_t s) {
  if (a.count <= 0) return;
  constexpr int smem = kFactSmemDoubles * (int)sizeof(double);
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    BDDC_CUDA(cudaFuncSetAttribute(trtri_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  }
  { trtri_tile_kernel<<<a.count, 128, smem, s>>>(a); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
}

void trsm_tile(const TileArgs& a, TrsmKind kind, cudaStream_t s) {
  switch (kind) {
    case TRSM_LLN: launch_trsm<false, true>(a, s); break;
    case TRSM_LLT: launch_trsm<false, false>(a, s); break;
    case TRSM_RLT: launch_trsm<true, true>(a, s); break;
    case TRSM_RLN: launch_trsm<true, false>(a, s); break;
  }
}

void gemm_batched(bool tA, bool tB, int M, int N, int K, double alpha, BMat A, BMat B,
                  double beta, BMat C, int count, cudaStream_t s, bool lower, int tri, bool mirror,
                  const int* klo) {
  if (M <= 0 || N <= 0) return;
  GemmArgs g;
  if (klo) {
    if (ceil_div(M, BM) > 16) throw CudaError("gemm_batched: klo table covers 16 row tiles");
    g.klo_on = 1;
    for (int i = 0; i < ceil_div(M, BM); ++i) g.klo[i] = klo[i];
  }
  g.A = A.p; g.sA = A.stride; g.lda = A.ld;
  g.B = B.p; g.sB = B.stride; g.ldb = B.ld;
  g.C = C.p; g.sC = C.stride; g.ldc = C.ld;
  g.M = M; g.N = N; g.K = K; g.count = count;
  g.alpha = alpha; g.beta = beta; g.lower = lower ? 1 : 0;
  g.tri = tri; g.mirror = mirror ? 1 : 0;
  if (K <= 0) {
    if (beta == 1.0) return;
  }
  gemm(g, tA, tB, s);
}

// In-place tile solve with an explicit 64 x 64 inverse tile Vinv (ld 64), as a DMMA GEMM:
//   LLN: X = Vinv B   LLT: X = Vinv^T B   (B: nb x nother; one 64-row tile -> in place)
//   RLT: X = B Vinv^T RLN: X = B Vinv      (B: nother x nb; one 64-col tile -> in place)
static void tile_solve_gemm(TrsmKind kind, BMat Vinv, int nb, BMat B, int nother, int count,
                            cudaStream_t s) {
  switch (kind) {
    case TRSM_LLN: gemm_batched(false, false, nb, nother, nb, 1.0, Vinv, B, 0.0, B, count, s); break;
    case TRSM_LLT: gemm_batched(true, false, nb, nother, nb, 1.0, Vinv, B, 0.0, B, count, s); break;
    case TRSM_RLT: gemm_batched(false, true, nother, nb, nb, 1.0, B, Vinv, 0.0, B, count, s); break;
    case TRSM_RLN: gemm_batched(false, false, nother, nb, nb, 1.0, B, Vinv, 0.0, B, count, s); break;
  }
}

void potrf_batched(BMat A, int n, int npiv, int count, int* info, double* scratch, cudaStream_t s) {
  // the inverse of diagonal tile kb stays in scratch slot kb (trsm_batched's layout)
  const long long sInv = (long long)ceil_div(npiv, kTile) * kTileInvStride;
  if (npiv == n) {
    // left-looking: block column k is updated once with all earlier panels (one GEMM of
    // inner dimension k instead of k / 64 rank-64 read-modify-writes of the trailing matrix)
    for (int k = 0; k < n; k += kTile) {
      const int nb = std::min(kTile, n - k);
      double* inv = scratch + (k / kTile) * kTileInvStride;
      if (k > 0)  // A[k:, k:k+nb] -= L[k:, 0:k] L[k:k+nb, 0:k]^T (lower part of the diagonal tile)
        gemm_batched(false, true, n - k, nb, k, -1.0, A.at(k, 0), A.at(k, 0), 1.0, A.at(k, k), count, s, true);
      TileArgs t;
      t.L = A.p + k + (long long)k * A.ld; t.sL = A.stride; t.ldl = A.ld;
      t.n = nb; t.count = count; t.offset = k; t.info = info;
      t.inv = inv; t.sInv = sInv;
      potrf_tile(t, s);
      const int rest = n - k - nb;
      if (rest > 0) tile_solve_gemm(TRSM_RLT, BMat{inv, sInv, kTile}, nb, A.at(k + nb, k), rest, count, s);
    }
    return;
  }
  for (int k = 0; k < npiv; k += kTile) {
    const int nb = std::min(kTile, npiv - k);
    double* inv = scratch + (k / kTile) * kTileInvStride;
    TileArgs t;
    t.L = A.p + k + (long long)k * A.ld; t.sL = A.stride; t.ldl = A.ld;
    t.n = nb; t.count = count; t.offset = k; t.info = info;
    t.inv = inv; t.sInv = sInv;
    potrf_tile(t, s);
    const int rest = n - k - nb;
    if (rest <= 0) continue;
    BMat L21 = A.at(k + nb, k);
    tile_solve_gemm(TRSM_RLT, BMat{inv, sInv, kTile}, nb, L21, rest, count, s);
    // trailing update A22 -= L21 L21^T (lower tiles only)
    BMat A22 = A.at(k + nb, k + nb);
    gemm_batched(false, true, rest, rest, nb, -1.0, L21, L21, 1.0, A22, count, s, true);
  }
}

namespace {
// Linv diagonal blocks <- the kept tile inverses (64 x 64, ld 64, zero upper part). The
// blocks above the diagonal are left unwritten: every consumer skips them (triangular K
// ranges, the column gather starts at the column's diagonal block).
__global__ void place_diag_inv_kernel(const double* __restrict__ scr, long long sInv, int n, double* Linv,
                                      long long sL, int ldl) {
  const int b = blockIdx.x;
  const double* inv = scr + b * sInv;
  double* L = Linv + b * sL;
  const int nb = (n + kTile - 1) / kTile;
  for (int idx = threadIdx.x; idx < nb * kTile * kTile; idx += blockDim.x) {
    const int bi = idx / (kTile * kTile), e = idx % (kTile * kTile);
    const int i = bi * kTile + e % kTile, j = bi * kTile + e / kTile;
    if (i < n && j < n) L[i + (long long)j * ldl] = inv[bi * kTileInvStride + e];
  }
}
}  // namespace

bool trtri_from_tiles(BMat L, int n, BMat Linv, int count, const double* scratch, cudaStream_t s) {
  if (n > 16 * kTile || n <= 0) return false;
  const int nb = ceil_div(n, kTile);
  const long long sInv = (long long)nb * kTileInvStride;
  place_diag_inv_kernel<<<count, 256, 0, s>>>(scratch, sInv, n, Linv.p, Linv.stride, Linv.ld);
  BDDC_COUNT();
  BDDC_LAUNCH_CHECK();
  // block row i: X[i, 0:i] = -D_i (L[i, 0:i] X[0:i, 0:i]); X[0:i, 0:i] (block lower
  // triangular, done by the earlier rows) is the structurally lower B operand
  for (int i = 1; i < nb; ++i) {
    const int r0 = i * kTile, ni = std::min(kTile, n - r0);
    BMat Di{(double*)scratch + i * kTileInvStride, sInv, kTile};
    gemm_batched(false, false, ni, r0, r0, 1.0, L.at(r0, 0), Linv, 0.0, Linv.at(r0, 0), count, s,
                 false, 3);  // B(k, n) = 0 for k < n
    // in place over rows: one 64-row tile, each CTA reads only its own column block
    gemm_batched(false, false, ni, r0, ni, -1.0, Di, Linv.at(r0, 0), 0.0, Linv.at(r0, 0), count, s,
                 false, 1);  // D_i lower: k <= m
  }
  return true;
}

size_t trsm_scratch_doubles(int n, int count) {
  return (size_t)count * ceil_div(n, kTile) * kTileInvStride;
}

void trsm_batched(TrsmKind kind, BMat L, int n, BMat B, int nother, int count, double* scratch,
                  cudaStream_t s, bool have_inv) {
  const int nblk = ceil_div(n, kTile);
  const long long sInv = (long long)nblk * kTileInvStride;  // per batch entry
  for (int kb = 0; kb < nblk && !have_inv; ++kb) {
    const int k = kb * kTile;
    TileArgs t;
    t.L = L.p + k + (long long)k * L.ld; t.sL = L.stride; t.ldl = L.ld;
    t.n = std::min(kTile, n - k); t.count = count;
    t.inv = scratch + kb * kTileInvStride; t.sInv = sInv;
    trtri_tile(t, s);
  }
  auto inv = [&](int kb) { return BMat{scratch + kb * kTileInvStride, sInv, kTile}; };
  if (kind == TRSM_LLN) {  // forward over row blocks
    for (int kb = 0; kb < nblk; ++kb) {
      const int k = kb * kTile, nb = std::min(kTile, n - k), rest = n - k - nb;
      tile_solve_gemm(kind, inv(kb), nb, B.at(k, 0), nother, count, s);
      if (rest > 0)
        gemm_batched(false, false, rest, nother, nb, -1.0, L.at(k + nb, k), B.at(k, 0), 1.0,
                     B.at(k + nb, 0), count, s);
    }
  } else if (kind == TRSM_LLT) {  // backward over row blocks
    for (int kb = nblk - 1; kb >= 0; --kb) {
      const int k = kb * kTile, nb = std::min(kTile, n - k);
      tile_solve_gemm(kind, inv(kb), nb, B.at(k, 0), nother, count, s);
      if (k > 0)  // B[0:k] -= L[k:k+nb, 0:k]^T X_k
        gemm_batched(true, false, k, nother, nb, -1.0, L.at(k, 0), B.at(k, 0), 1.0, B.at(0, 0),
                     count, s);
    }
  } else if (kind == TRSM_RLT) {  // forward over column blocks: X L^T = B
    for (int kb = 0; kb < nblk; ++kb) {
      const int k = kb * kTile, nb = std::min(kTile, n - k), rest = n - k - nb;
      tile_solve_gemm(kind, inv(kb), nb, B.at(0, k), nother, count, s);
      if (rest > 0)  // B[:, k+nb:] -= X_k L[k+nb:, k]^T
        gemm_batched(false, true, nother, rest, nb, -1.0, B.at(0, k), L.at(k + nb, k), 1.0,
                     B.at(0, k + nb), count, s);
    }
  } else {  // RLN: backward over column blocks: X L = B
    for (int kb = nblk - 1; kb >= 0; --kb) {
      const int k = kb * kTile, nb = std::min(kTile, n - k);
      tile_solve_gemm(kind, inv(kb), nb, B.at(0, k), nother, count, s);
      if (k > 0)  // B[:, 0:k] -= X_k L[k:k+nb, 0:k]
        gemm_batched(false, false, nother, k, nb, -1.0, B.at(0, k), L.at(k, 0), 1.0, B.at(0, 0),
                     count, s);
    }
  }
}

// Batched y = alpha A^T x + beta y for column-major k x n operands (lda >= k, even): every
// output entry is a dot product over one contiguous column of A, i.e. over one row of the
// row-major n x k matrix a torch tensor holds. HBM-bound: each entry of A is read once with
// 16-byte loads (lda even, 16-byte aligned bases), x of the batch entry sits in shared memory,
// one warp per output entry, kGemvRows entries per CTA, fixed summation order.
namespace {
constexpr int kGemvWarps = 8, kGemvRows = 32;
__global__ void __launch_bounds__(32 * kGemvWarps) gemv_t_kernel(int k, int n, double alpha,
                                                                 const double* __restrict__ A, int lda,
                                                                 long long sA, const double* __restrict__ x,
                                                                 long long sx, double beta,
                                                                 double* __restrict__ y, long long sy) {
  extern __shared__ double xs[];
  const int b = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* xb = x + (long long)b * sx;
  for (int i = tid; i < k; i += blockDim.x) xs[i] = xb[i];
  if (tid == 0 && (k & 1)) xs[k] = 0.0;
  __syncthreads();
  const double* Ab = A + (long long)b * sA;
  double* yb = y + (long long)b * sy;
  const int j0 = blockIdx.x * kGemvRows;
  const int k2 = (k + 1) >> 1;  // pairs; a column's padding element (lda even) meets xs[k] = 0
  for (int jj = warp; jj < kGemvRows; jj += kGemvWarps) {
    const int j = j0 + jj;
    if (j >= n) break;
    const double2* col = reinterpret_cast<const double2*>(Ab + (long long)j * lda);
    double a0 = 0.0, a1 = 0.0;
    int p = lane;
    for (; p + 32 < k2; p += 64) {
      const double2 u = __ldcs(col + p), v = __ldcs(col + p + 32);
      a0 += u.x * xs[2 * p] + u.y * xs[2 * p + 1];
      a1 += v.x * xs[2 * p + 64] + v.y * xs[2 * p + 65];
    }
    if (p < k2) {
      const double2 u = __ldcs(col + p);
      const double ux = u.x, uy = (2 * p + 1 < k) ? u.y : 0.0;
      a0 += ux * xs[2 * p] + uy * xs[2 * p + 1];
    }
    double acc = a0 + a1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) yb[j] = beta == 0.0 ? alpha * acc : alpha * acc + beta * yb[j];
  }
}
}  // namespace

void gemv_t_batched(int k, int n, double alpha, BMat A, const double* x, long long sx, double beta, double* y,
                    long long sy, int count, cudaStream_t s) {
  if (n <= 0 || count <= 0) return;
  const size_t smem = sizeof(double) * (size_t)(k + 2);
  if (smem > 200 * 1024) throw CudaError("gemv_t_batched: x does not fit shared memory");
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr))
    BDDC_CUDA(cudaFuncSetAttribute(gemv_t_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  dim3 grid(ceil_div(n, kGemvRows), count);
  gemv_t_kernel<<<grid, 32 * kGemvWarps, smem, s>>>(k, n, alpha, A.p, A.ld, A.stride, x, sx, beta, y, sy);
  BDDC_LAUNCH_CHECK();
  BDDC_COUNT();
}

}  // namespace bddc
