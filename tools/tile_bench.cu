// Pure kernel timing of tile::potrf_trtri_tile (64x64) and tile::gemm_tile.
#define BDDC_TILE_PROF 1
#include <cstdio>
#include <vector>
#include "../paper_2001_07289_b200/csrc/tile_ops.cuh"
using namespace bddc;
__global__ void __launch_bounds__(128) k_chol(double* A, double* inv, int reps) {
  extern __shared__ __align__(16) double sm[];
  double* a = A + (long long)blockIdx.x * 64 * 64;
  for (int r = 0; r < reps; ++r) tile::potrf_trtri_tile<true>(a, 64, 64, inv + (long long)blockIdx.x * 4096, sm);
}
__global__ void __launch_bounds__(128) k_gj(double* A, double* inv, int reps) {
  extern __shared__ __align__(16) double sm[];
  double* a = A + (long long)blockIdx.x * 64 * 64;
  for (int r = 0; r < reps; ++r) tile::gj_tile_inverse(a, 64, 64, inv + (long long)blockIdx.x * 4096, sm);
}
__global__ void __launch_bounds__(128) k_gemm(const double* A, double* C, int reps) {
  extern __shared__ __align__(16) double sm[];
  const double* a = A + (long long)blockIdx.x * 64 * 64;
  double* c = C + (long long)blockIdx.x * 64 * 64;
  for (int r = 0; r < reps; ++r) tile::gemm_tile<false, true>(a, 64, a, 64, c, 64, 64, 64, 64, 0, 0, -1.0, 1.0, true, sm);
}
int main() {
  const int nb = 148;
  std::vector<double> h(64 * 64 * nb);
  for (int b = 0; b < nb; ++b)
    for (int j = 0; j < 64; ++j)
      for (int i = 0; i < 64; ++i) h[b * 4096 + i + j * 64] = (i == j) ? 64.0 + i : 1.0 / (1 + i + j);
  double *A, *I, *Cc;
  cudaMalloc(&A, h.size() * 8); cudaMalloc(&I, h.size() * 8); cudaMalloc(&Cc, h.size() * 8);
  cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  const int smem = tile::kFactSmemDoubles * 8;
  cudaFuncSetAttribute(k_chol, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int reps : {1, 10}) {
    cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    k_chol<<<nb, 128, smem>>>(A, I, reps);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("chol+inv tile: %d reps: %.1f us per tile (%s)\n", reps, 1000 * ms / reps, cudaGetErrorString(cudaGetLastError()));
  }
  {
    long long m[16];
    cudaMemcpyFromSymbol(m, g_tile_marks, sizeof(m));
    const char* nm[6] = {"start", "loaded", "diag0", "factor loop", "inverse", "stored"};
    for (int i = 1; i < 6; ++i) printf("  %-12s +%lld cycles\n", nm[i], m[i] - m[i - 1]);
  }
  cudaFuncSetAttribute(k_gj, cudaFuncAttributeMaxDynamicSharedMemorySize, tile::kGjSmemDoubles * 8);
  for (int reps : {1, 10}) {
    cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    k_gj<<<nb, 128, tile::kGjSmemDoubles * 8>>>(A, I, reps);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("gj inverse tile: %d reps: %.1f us per tile (%s)\n", reps, 1000 * ms / reps, cudaGetErrorString(cudaGetLastError()));
  }
  {
    long long m[16];
    cudaMemcpyFromSymbol(m, g_tile_marks, sizeof(m));
    printf("  gj: load %lld | kb0 %lld | kb1: pivot %lld, row %lld, trailing %lld, col+rest %lld | total loop %lld\n",
           m[6] - m[12], m[7] - m[6], m[8] - m[7], m[9] - m[8], m[10] - m[9], m[11] - m[10], m[11] - m[6]);
  }
  cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, tile::kGemmSmemDoubles * 8);
  for (int reps : {1, 10}) {
    cudaEventRecord(e0);
    k_gemm<<<nb, 128, tile::kGemmSmemDoubles * 8>>>(A, Cc, reps);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("gemm tile 64x64x64: %d reps: %.2f us per tile\n", reps, 1000 * ms / reps);
  }
  return 0;
}
