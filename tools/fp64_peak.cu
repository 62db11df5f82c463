// FP64 throughput probe: DMMA m8n8k4 (mma.sync) vs scalar DFMA, per-SM issue-bound loops.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int i = 0; i < 8; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}
__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[16];
  for (int i = 0; i < 16; i++) c[i] = i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) c[i] = fma(a, c[i], b);
  }
  double s = 0;
  for (int i = 0; i < 16; i++) s += c[i];
  if (s == 12345.0) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps = 4; warps <= 32; warps *= 2) {
    int blocks = p.multiProcessorCount * 2, iters = 4000;
    dmma_loop<<<blocks, warps * 32>>>(d, 10);
    cudaEventRecord(e0); dmma_loop<<<blocks, warps * 32>>>(d, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * warps;
    printf("DMMA warps/blk %2d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
    dfma_loop<<<blocks, warps * 32>>>(d, 10);
    cudaEventRecord(e0); dfma_loop<<<blocks, warps * 32>>>(d, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * (double)iters * blocks * warps * 32;
    printf("DFMA warps/blk %2d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  return 0;
}
