// Batched FP64 dense kernels for sm_100a: DMMA (mma.sync m8n8k4 f64) grouped GEMM,
// tile Cholesky and tile triangular solves, plus blocked host drivers.
//
// All matrices are column-major. A batch is either strided (base + b*stride, uniform
// sizes) or an explicit device task array (variable sizes: multifrontal fronts).
#pragma once
#include "common.cuh"

namespace bddc {

constexpr long long kTileInvStride = 64 * 64;

struct GemmTask {
  const double* A;
  const double* B;
  double* C;
  int M, N, K, lda, ldb, ldc;
};

// C = alpha * op(A) op(B) + beta * C; lower != 0 writes only C(i,j) with i >= j.
struct GemmArgs {
  const double* A = nullptr;
  const double* B = nullptr;
  double* C = nullptr;
  long long sA = 0, sB = 0, sC = 0;
  int M = 0, N = 0, K = 0, lda = 0, ldb = 0, ldc = 0;
  int count = 0;
  const GemmTask* tasks = nullptr;  // device array; overrides the strided fields
  int max_M = 0, max_N = 0;         // grid sizing when tasks != nullptr
  double alpha = 1.0, beta = 1.0;
  int lower = 0;
  int tri = 0;     // structural zeros: 1 op(A) lower, 2 op(A) upper, 3 op(B) lower, 4 op(B) upper
  int mirror = 0;  // with lower: also write the upper triangle (symmetric result)
  // staircase operands: rows (op(A)) of 64-tile i have no nonzero K below klo[i] (klo_on)
  int klo_on = 0;
  int klo[16] = {};
};

struct TileTask {
  double* L;    // n x n lower tile
  double* B;    // right-hand sides (see kernels)
  int n, ldl, ldb, nvec;  // nvec: rows (right side) or columns (left side) of B
  int id, offset;         // batch entry id and global index of the tile's first row
  double* inv;  // 64 x 64 scratch receiving L^{-1} (trtri_tile)
};

struct TileArgs {
  double* L = nullptr;
  double* B = nullptr;
  long long sL = 0, sB = 0;
  int n = 0, ldl = 0, ldb = 0, nvec = 0;
  int count = 0;
  const TileTask* tasks = nullptr;
  int max_nvec = 0;
  int offset = 0;      // global index of first row (pivot reporting)
  int* info = nullptr; // per batch entry: first failing pivot (INT_MAX if none)
  double* inv = nullptr;  // strided: inverse scratch, 64 x 64 per entry (sInv apart)
  long long sInv = kTileInvStride;
};

enum TrsmKind {
  // side, uplo=lower always
  TRSM_LLN = 0,  // X = L^{-1} B      (left, no-trans)
  TRSM_LLT = 1,  // X = L^{-T} B      (left, trans)
  TRSM_RLT = 2,  // X = B L^{-T}      (right, trans)
  TRSM_RLN = 3,  // X = B L^{-1}      (right, no-trans)
};

void gemm(const GemmArgs& a, bool transA, bool transB, cudaStream_t s);
void potrf_tile(const TileArgs& a, cudaStream_t s);
// inverse of n x n lower tiles (n <= 64) into 64 x 64 scratch (lower, zero upper)
void trtri_tile(const TileArgs& a, cudaStream_t s);
void trsm_tile(const TileArgs& a, TrsmKind kind, cudaStream_t s);

// Strided uniform batch view of n x n (or rows x cols) matrices.
struct BMat {
  double* p;
  long long stride;
  int ld;
  BMat at(int i, int j) const { return BMat{p + i + (long long)j * ld, stride, ld}; }
};

// Blocked in-place lower Cholesky of `count` n x n matrices; factors the leading npiv
// columns only (npiv < n: partial factorization, trailing block becomes the Schur complement).
// scratch: count * ceil(npiv/64) * 64 * 64 doubles; on return slot kb holds the inverse of
// diagonal tile kb (the layout trsm_batched(..., have_inv = true) consumes).
void potrf_batched(BMat A, int n, int npiv, int count, int* info, double* scratch, cudaStream_t s);
// Blocked triangular solves with a batch of n x n lower factors L:
//   left kinds: B is n x ncol; right kinds: B is nrow x n.
// scratch: count * ceil(n/64) * 64 * 64 doubles. Diagonal tiles are inverted once (trtri)
// and every tile solve is an in-place DMMA GEMM with the inverse. have_inv: scratch already
// holds the inverses (left by potrf_batched on the same factor).
void trsm_batched(TrsmKind kind, BMat L, int n, BMat B, int nother, int count, double* scratch,
                  cudaStream_t s, bool have_inv = false);
size_t trsm_scratch_doubles(int n, int count);
// C = alpha op(A) op(B) + beta C over a strided batch.
// klo (optional, ceil(M/64) <= 16 entries): first nonzero K of op(A)'s 64-row tile i.
// y = alpha A^T x + beta y, A column-major k x n per batch entry (dot products over contiguous columns)
void gemv_t_batched(int k, int n, double alpha, BMat A, const double* x, long long sx, double beta, double* y,
                    long long sy, int count, cudaStream_t s);
void gemm_batched(bool tA, bool tB, int M, int N, int K, double alpha, BMat A, BMat B,
                  double beta, BMat C, int count, cudaStream_t s, bool lower = false, int tri = 0,
                  bool mirror = false, const int* klo = nullptr);
// L^{-1} of a batch of n x n lower factors (n <= 1024) from the diagonal-tile inverses left in
// scratch by potrf_batched (blocked, one block row at a time). Written: the lower block
// triangle (diagonal tiles with zero upper parts); the blocks above the diagonal are not.
bool trtri_from_tiles(BMat L, int n, BMat Linv, int count, const double* scratch, cudaStream_t s);

constexpr int kTile = 64;

}  // namespace bddc
