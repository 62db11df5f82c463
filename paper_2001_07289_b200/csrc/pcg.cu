// Device PCG (krylov.py:31-92): x0 = 0, recurrence residual, stop at ||r|| <= tol ||b||.
// SpMV is fused with <p, Ap>; the x / r update is fused with ||r||^2; every reduction is one
// launch (block partials over a fixed grid, summed in fixed order by the last block to
// finish), hence deterministic; rz <- rz_new rides on the p update. One host synchronisation per
// iteration reads {rz, pAp, rr} for the stopping test, the SPD guards and the Lanczos
// coefficients (alpha_k, beta_k).
#include "stencil.cuh"

namespace bddc {

namespace {

constexpr int kRedBlocks = 592;  // 4 x 148 SMs
constexpr int kRedThreads = 256;

__device__ __forceinline__ void block_partial(double v, double* partial) {
  __shared__ double red[kRedThreads / 32];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < kRedThreads / 32; ++i) s += red[i];
    partial[blockIdx.x] = s;
  }
}

// The block partials of a grid reduction, then the grid total written by the LAST block to
// finish (arrival counter, reset by that block): partial i summed by thread i mod 256 in index
// order, then a fixed warp / block tree (deterministic), without a separate final launch.
__device__ __forceinline__ void grid_total(double v, double* partial, unsigned* cnt, double* out) {
  block_partial(v, partial);
  __shared__ bool last;
  __shared__ double red2[kRedThreads / 32];
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(cnt, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double acc = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) acc += __ldcg(partial + i);
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red2[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < kRedThreads / 32; ++i) t += red2[i];
    *out = t;
    *cnt = 0u;
  }
}

__global__ void __launch_bounds__(kRedThreads) dot_partial_kernel(const double* __restrict__ a,
                                                                  const double* __restrict__ b,
                                                                  long long n, double* partial, unsigned* cnt,
                                                                  double* out) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    acc += a[i] * b[i];
  grid_total(acc, partial, cnt, out);
}

// one resident wave: every thread loops over the same number of sweep items (+-1)
template <int DIM, bool EDGE>
__global__ void __launch_bounds__(kRedThreads, (EDGE || DIM == 2) ? 3 : 1) spmv_dot_kernel(Geometry G, const double* __restrict__ alpha,
                                                               const double* __restrict__ p,
                                                               double* __restrict__ Ap, double* partial,
                                                               unsigned* cnt, double* out) {
  double acc = 0.0;
  stencil_sweep<DIM, EDGE>(G, alpha, p, [&](long long f, double v, double pc) {
    Ap[f] = v;
    if (f >= G.fo_lo) acc += pc * v;  // dot over owned rows (fo_hi == f_hi)
  });
  grid_total(acc, partial, cnt, out);
}

// alpha = rz / pAp; x += alpha p; r -= alpha Ap; partial ||r||^2
__global__ void __launch_bounds__(kRedThreads) update_xr_kernel(double* __restrict__ x, double* __restrict__ r,
                                                                const double* __restrict__ p,
                                                                const double* __restrict__ Ap,
                                                                const double* __restrict__ scal,
                                                                long long lo, long long hi, long long own_lo,
                                                                double* partial, unsigned* cnt, double* out) {
  const double a = scal[0] / scal[1];
  double acc = 0.0;
  for (long long i = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < hi;
       i += (long long)gridDim.x * blockDim.x) {
    x[i] += a * p[i];
    const double ri = r[i] - a * Ap[i];
    r[i] = ri;
    if (i >= own_lo) acc += ri * ri;
  }
  grid_total(acc, partial, cnt, out);
}

// beta = rz_new / rz; p = z + beta p; then (last block) rz <- rz_new for the next iteration
__global__ void xpay_kernel(double* __restrict__ p, const double* __restrict__ z, double* scal, long long lo,
                            long long n, unsigned* cnt) {
  const double b = scal[3] / scal[0];  // every block reads both before the last one rewrites scal[0]
  for (long long i = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = z[i] + b * p[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(cnt, 1u) == gridDim.x - 1) {
      scal[0] = scal[3];
      *cnt = 0u;
    }
  }
}

}  // namespace

// dots run over the rank's owned rows (all rows when unsharded) and are summed over ranks
double dot(Ctx& c, const double* a, const double* b, long long n, cudaStream_t s) {
  const Geometry& G = c.geo;
  (void)n;
  { dot_partial_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(a + G.fo_lo, b + G.fo_lo, G.fo_hi - G.fo_lo, c.red, c.redc,
                                                          c.scal + 7); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
  allreduce_scalars(c, c.scal + 7, 1, s);
  BDDC_CUDA(cudaMemcpyAsync(c.h_scal + 7, c.scal + 7, sizeof(double), cudaMemcpyDeviceToHost, s));
  BDDC_CUDA(cudaStreamSynchronize(s));
  return c.h_scal[7];
}

static void dot_to(Ctx& c, const double* a, const double* b, long long n, double* out, cudaStream_t s) {
  const Geometry& G = c.geo;
  (void)n;
  { dot_partial_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(a + G.fo_lo, b + G.fo_lo, G.fo_hi - G.fo_lo, c.red, c.redc,
                                                          out); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
}

static PcgResult pcg_run(Ctx& c, const double* b, double* x, double tol, int max_iters, double* alphas,
                         double* betas, double* resid) {
  const Geometry& G = c.geo;
  cudaStream_t s = c.stream;
  const long long n = G.n;
  PcgResult res{0, 0, 0, 0.0, 0};
  double* sc = c.scal;
  double* hs = c.h_scal;
  BDDC_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
  BDDC_CUDA(cudaMemcpyAsync(c.r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  dot_to(c, c.r, c.r, n, sc + 4, s);
  apply_bddc(c, c.r, c.z, s);
  dot_to(c, c.r, c.z, n, sc + 0, s);
  allreduce_scalars(c, sc, 5, s);  // sharded: sum over ranks (sc[1..3] are rewritten before use)
  BDDC_CUDA(cudaMemcpyAsync(hs, sc, sizeof(double) * 8, cudaMemcpyDeviceToHost, s));
  BDDC_CUDA(cudaStreamSynchronize(s));
  const double norm0 = sqrt(hs[4]);
  resid[0] = norm0;
  if (norm0 == 0.0) {
    res.converged = 1;
    return res;
  }
  double rz = hs[0];
  if (!(rz > 0.0)) {
    res.status = 5; res.bad_value = rz; res.bad_kind = 0;
    return res;
  }
  BDDC_CUDA(cudaMemcpyAsync(c.p, c.z, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  int nbeta = 0;
  // the SpMV + dot kernel of this operator and a grid of exactly one resident wave
  const bool edge = stencil_edge_only(G);
  auto sd_kernel = G.dim == 2 ? (edge ? spmv_dot_kernel<2, true> : spmv_dot_kernel<2, false>)
                              : (edge ? spmv_dot_kernel<3, true> : spmv_dot_kernel<3, false>);
  int sd_per_sm = 1, sms = 148;
  BDDC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&sd_per_sm, sd_kernel, kRedThreads, 0));
  BDDC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
  const int sd_blocks = std::max(1, std::min(4096, sd_per_sm * sms));
  auto sd_launch = [&](int grid, int threads, size_t smem, cudaStream_t st, auto... args) {
    sd_kernel<<<grid, threads, smem, st>>>(args...);
  };
  for (int it = 0; it < max_iters; ++it) {
    exchange_dof_halo(c, c.p, s);  // sharded: p on the rows next to the cut lines
    c.prof.begin("pcg.spmv_dot", s);
    sd_launch(sd_blocks, kRedThreads, 0, s, G, c.alpha, c.p, c.Ap, c.red, c.redc, sc + 1);
    BDDC_COUNT();
    c.prof.end("pcg.spmv_dot", s);
    allreduce_scalars(c, sc + 1, 1, s);
    { update_xr_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(x, c.r, c.p, c.Ap, sc, G.f_lo, G.f_hi, G.fo_lo, c.red,
                                                         c.redc, sc + 2); BDDC_COUNT(); }
    BDDC_LAUNCH_CHECK();
    allreduce_scalars(c, sc + 2, 1, s);
    BDDC_CUDA(cudaMemcpyAsync(hs, sc, sizeof(double) * 4, cudaMemcpyDeviceToHost, s));
    BDDC_CUDA(cudaStreamSynchronize(s));
    if (it > 0) {  // rz_new of the previous iteration is now in hs[0]
      const double rz_new = hs[0];
      if (!(rz_new > 0.0)) {
        res.status = 5; res.bad_value = rz_new; res.bad_kind = 2;
        res.iterations = it;
        return res;
      }
      betas[nbeta++] = rz_new / rz;
      rz = rz_new;
    }
    const double pAp = hs[1];
    if (!(pAp > 0.0)) {
      res.status = 5; res.bad_value = pAp; res.bad_kind = 1;
      res.iterations = it;
      return res;
    }
    alphas[it] = hs[0] / pAp;
    const double rn = sqrt(hs[2]);
    resid[it + 1] = rn;
    res.iterations = it + 1;
    if (rn <= tol * norm0) {
      res.converged = 1;
      break;
    }
    if (it + 1 == max_iters) {
      // the reference computes one more B-apply and beta that the Lanczos step ignores
      apply_bddc(c, c.r, c.z, s);
      dot_to(c, c.r, c.z, n, sc + 3, s);
      allreduce_scalars(c, sc + 3, 1, s);
      BDDC_CUDA(cudaMemcpyAsync(hs + 3, sc + 3, sizeof(double), cudaMemcpyDeviceToHost, s));
      BDDC_CUDA(cudaStreamSynchronize(s));
      if (!(hs[3] > 0.0)) {
        res.status = 5; res.bad_value = hs[3]; res.bad_kind = 2;
      }
      break;
    }
    apply_bddc(c, c.r, c.z, s);
    dot_to(c, c.r, c.z, n, sc + 3, s);
    allreduce_scalars(c, sc + 3, 1, s);
    { xpay_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(c.p, c.z, sc, G.f_lo, G.f_hi, c.redc); BDDC_COUNT(); }
    BDDC_LAUNCH_CHECK();
  }
  return res;
}

PcgResult pcg_solve(Ctx& c, const double* b, double* x, double tol, int max_iters, double* alphas,
                    double* betas, double* resid) {
  const PcgResult res = pcg_run(c, b, x, tol, max_iters, alphas, betas, resid);
  // a coarse-solve dependency timeout poisons z with NaN: report it as what it is, not as a
  // non-SPD preconditioner
  if (coarse_solve_error(c)) throw CudaError("coarse dataflow solve: dependency wait timed out");
  return res;
}

}  // namespace bddc
