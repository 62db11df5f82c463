// Cost of CUDA VMM calls vs mapping granularity (front_vmm.cu design probe).
// usage: vmm_probe <total GB> <page MB> <mode>  mode 0: one access call over the range,
// 1: access per mapping as it is created
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { printf("%s failed %d\n", #x, (int)r); exit(1); } } while (0)
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main(int argc, char** argv) {
  double gb = atof(argv[1]); size_t pmb = atol(argv[2]); int mode = atoi(argv[3]);
  cudaFree(0);
  CUmemAllocationProp prop{}; prop.type = CU_MEM_ALLOCATION_TYPE_PINNED; prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE; prop.location.id = 0;
  size_t PB = pmb << 20; size_t n = (size_t)(gb * (1 << 30)) / PB;
  CUdeviceptr va; CK(cuMemAddressReserve(&va, n * PB, PB, 0, 0));
  CUmemAccessDesc acc{}; acc.location = prop.location; acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  std::vector<CUmemGenericAllocationHandle> h(n);
  double t0 = now();
  for (size_t i = 0; i < n; ++i) CK(cuMemCreate(&h[i], PB, &prop, 0));
  double t1 = now();
  if (mode >= 2) {  // mode threads, each maps + sets access on its share
    CUcontext ctx; cuCtxGetCurrent(&ctx);
    std::vector<std::thread> th;
    for (int t = 0; t < mode; ++t) th.emplace_back([&, t] {
      cuCtxSetCurrent(ctx);
      for (size_t i = t; i < n; i += mode) { CK(cuMemMap(va + i * PB, PB, 0, h[i], 0)); CK(cuMemSetAccess(va + i * PB, PB, &acc, 1)); }
    });
    for (auto& x : th) x.join();
  } else {
    for (size_t i = 0; i < n; ++i) { CK(cuMemMap(va + i * PB, PB, 0, h[i], 0)); if (mode == 1) CK(cuMemSetAccess(va + i * PB, PB, &acc, 1)); }
  }
  double t2 = now();
  if (mode == 0) CK(cuMemSetAccess(va, n * PB, &acc, 1));
  double t3 = now();
  CK(cuMemsetD8(va, 0, n * PB)); cuCtxSynchronize();
  double t4 = now();
  printf("total %.1f GB page %zu MB n %zu mode %d: create %.3f s map %.3f s access %.3f s memset %.3f s\n", gb, pmb, n, mode, t1 - t0, t2 - t1, t3 - t2, t4 - t3);
  for (size_t i = 0; i < n; ++i) cuMemUnmap(va + i * PB, PB);
  for (auto x : h) cuMemRelease(x);
  cuMemAddressFree(va, n * PB);
  return 0;
}
