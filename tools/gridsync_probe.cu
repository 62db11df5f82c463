// grid.sync() cost vs grid size (cooperative launch), for the coarse engine design.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, int* x) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
  if (threadIdx.x == 0) x[blockIdx.x] = 1;
}
int main() {
  int* d; cudaMalloc(&d, 1 << 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int blocks : {148, 296, 444, 592}) {
    for (int th : {128, 256}) {
      int iters = 1000;
      void* args[] = {&iters, &d};
      cudaLaunchCooperativeKernel((void*)k, blocks, th, args, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k, blocks, th, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("grid %4d x %3d: %.2f us per grid.sync (%s)\n", blocks, th, 1000.f * ms / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
