// Shared helpers for the BDDC-SO sm_100a kernels.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace bddc {

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& s) : std::runtime_error(s) {}
};

#define BDDC_CUDA(call)                                                                   \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess)                                                                \
      throw ::bddc::CudaError(std::string(#call) + ": " + cudaGetErrorString(_e) + " at " + \
                              __FILE__ + ":" + std::to_string(__LINE__));                 \
  } while (0)

#define BDDC_LAUNCH_CHECK() BDDC_CUDA(cudaGetLastError())

// Device-side bounds checks of the index-driven gathers / scatters (extend-add maps, coarse
// assembly positions, interface gathers, the coarse solve's gathers). Compiled in only for the
// checked build (make check -> libbddcso_b200_check.so, -DBDDC_CHECKS): a failed check prints
// its location and traps, so the launch fails loudly instead of corrupting memory. This is the
// bounds evidence in place of compute-sanitizer, which is closed on this GPU pool.
#ifdef BDDC_CHECKS
#define BDDC_CHECK(cond)                                                                      \
  do {                                                                                        \
    if (!(cond)) {                                                                            \
      printf("BDDC_CHECK failed at %s:%d: %s (block %d, thread %d)\n", __FILE__, __LINE__, #cond, \
             (int)blockIdx.x, (int)threadIdx.x);                                              \
      __trap();                                                                               \
    }                                                                                         \
  } while (0)
#else
#define BDDC_CHECK(cond) \
  do {                   \
  } while (0)
#endif

// Number of kernels this library has launched (reported by bench.py as gpu_launches).
inline std::atomic<long long>& launch_counter() {
  static std::atomic<long long> c{0};
  return c;
}
#define BDDC_COUNT() (::bddc::launch_counter().fetch_add(1, std::memory_order_relaxed))

// Per-device one-time initialisation (function attributes, __constant__ tables): true the
// first time it is called on the current device for this flag word. Function attributes and
// constant memory are per device, so a process that drives several GPUs needs one init each.
inline bool first_on_device(std::atomic<unsigned long long>& mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  const unsigned long long bit = 1ULL << (dev & 63);
  return !(mask.fetch_or(bit) & bit);
}
// Largest dynamic shared memory already granted to a kernel on the current device.
struct SmemAttr {
  std::atomic<size_t> v[64] = {};
  bool needs(size_t bytes) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    return bytes > v[dev & 63].load();
  }
  void set(size_t bytes) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    v[dev & 63].store(bytes);
  }
};

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }
inline long long round_up(long long a, long long b) { return (a + b - 1) / b * b; }

// ---- device helpers ------------------------------------------------------------------

// D = A(8x4, row) * B(4x8, col) + C, FP64 tensor core (SASS: DMMA.8x8x4).
// Fragment ownership (lane = 4*g + t): a = A[g][t], b = B[t][g], c = C[g][2t..2t+1].
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// 16-byte async copy global->shared with zero fill of the bytes past src_bytes.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
// 8-byte variant (operands that are only 8-byte aligned).
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- TMA bulk copies (cp.async.bulk) completing on shared-memory mbarriers ----
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
// make mbarrier initialisation visible to the async (TMA) proxy
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// arrive (count 1) and announce `bytes` of transactions for the current phase
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// global -> shared bulk copy (16-byte aligned addresses, size multiple of 16)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 1/x and 1/sqrt(x) for x > 0: hardware approximation (MUFU.RCP64H / RSQ64H) + 2 Newton
// steps in double (full precision for the SPD pivots they are used on; no special cases)
__device__ __forceinline__ double rcp_pos(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-x, r, 2.0);
  return r * fma(-x, r, 2.0);
}
__device__ __forceinline__ double rsqrt_pos(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-0.5 * x * r, r, 1.5);
  return r * fma(-0.5 * x * r, r, 1.5);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace bddc
