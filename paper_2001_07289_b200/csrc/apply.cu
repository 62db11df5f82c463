// Preconditioner apply z = B r (BddcOperator.apply, bddc.py:336-390), reduced form.
//
// The reference does three interior sweeps and two global SpMVs. Because interior dofs
// only couple inside their subdomain, (r - A u1)_I = 0 and (r - A(u1+u2))_I = 0, so
//   rp_Gamma = r_Gamma - (A u1)_Gamma,          u1_I = A_II^{-1} r_I
//   z_Gamma  = g = sum_i D_i R_i (w_i),          w_i = v_i + Psi_i c
//   z_I      = A_II^{-1} (r - A g_ext)_I
// which equals apply() to round-off. The local constrained Neumann
// solve restricted to Gamma is v = (I - Phi C) S_K^{-1} rho, so
//   w = u + Phi (c_i * c_loc - C u),  u = S_K^{-1} rho,  coarse rhs += c_i Phi^T rho.
#include "stencil.cuh"

namespace bddc {

namespace {

template <int DIM>
__global__ void spmv_kernel(Geometry G, const double* __restrict__ alpha, const double* __restrict__ x,
                            double* __restrict__ y) {
  for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < G.n;
       f += (long long)gridDim.x * blockDim.x) {
    int g0, g1, g2;
    free_coords(G, f, g0, g1, g2);
    y[f] = stencil_row<DIM>(G, alpha, x, g0, g1, g2);
  }
}

// y = r - A x (all free dofs)
template <int DIM>
__global__ void residual_kernel(Geometry G, const double* __restrict__ alpha, const double* __restrict__ r,
                                const double* __restrict__ x, double* __restrict__ y) {
  for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < G.n;
       f += (long long)gridDim.x * blockDim.x) {
    int g0, g1, g2;
    free_coords(G, f, g0, g1, g2);
    y[f] = r[f] - stencil_row<DIM>(G, alpha, x, g0, g1, g2);
  }
}

// rpg[g] = r - (A u1) at interface dofs
template <int DIM>
__global__ void gamma_residual_kernel(Geometry G, int n_gamma, const long long* __restrict__ gdof,
                                      const double* __restrict__ alpha, const double* __restrict__ r,
                                      const double* __restrict__ u1, double* __restrict__ rpg) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_gamma) return;
  const long long f = gdof[g];
  int g0, g1, g2;
  free_coords(G, f, g0, g1, g2);
  rpg[g] = r[f] - stencil_row<DIM>(G, alpha, u1, g0, g1, g2);
}

// Block-tridiagonal interior solve x_I = A_II^{-1} b_I per subdomain (forward + backward).
template <int DIM>
__global__ void bt_solve_kernel(Geometry G, LocalTables lt, const double* __restrict__ LI,
                                const double* __restrict__ in, double* __restrict__ out) {
  extern __shared__ double sm[];
  const int M = G.m_pad;
  const long long mm = (long long)M * M;
  double* y = sm;             // nI_pad
  double* Ld = sm + G.nI_pad; // M*M
  double* Lo = Ld + mm;       // M*M
  const int sub = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  int p[3];
  sub_coords(G, sub, p);
  const double* li = LI + (long long)sub * G.nblk * 2 * mm;
  for (int rr = tid; rr < G.nI_pad; rr += nt) {
    const int node = lt.irow_node[rr];
    double v = 0.0;
    if (node >= 0) {
      int a[3];
      local_coords(G, node, a);
      v = in[local_to_free(G, p, a)];
    }
    y[rr] = v;
  }
  // forward: y_j = Ld_j^{-1} (b_j - Lo_j y_{j-1})
  for (int j = 0; j < G.nblk; ++j) {
    for (int idx = tid; idx < mm; idx += nt) Ld[idx] = li[2LL * j * mm + idx];
    if (j > 0)
      for (int idx = tid; idx < mm; idx += nt) Lo[idx] = li[(2LL * j + 1) * mm + idx];
    __syncthreads();
    double* yj = y + j * M;
    if (j > 0 && tid < M) {
      const double* yp = y + (j - 1) * M;
      double s0 = 0.0, s1 = 0.0;
      int k = 0;
      for (; k + 1 < M; k += 2) {
        s0 += Lo[tid + k * M] * yp[k];
        s1 += Lo[tid + (k + 1) * M] * yp[k + 1];
      }
      if (k < M) s0 += Lo[tid + k * M] * yp[k];
      yj[tid] -= s0 + s1;
    }
    __syncthreads();
    for (int k = 0; k < M; ++k) {
      if (tid == k) yj[k] /= Ld[k + k * M];
      __syncthreads();
      if (tid > k && tid < M) yj[tid] -= Ld[tid + k * M] * yj[k];
    }
    __syncthreads();
  }
  // backward: x_j = Ld_j^{-T} (y_j - Lo_{j+1}^T x_{j+1})
  for (int j = G.nblk - 1; j >= 0; --j) {
    for (int idx = tid; idx < mm; idx += nt) Ld[idx] = li[2LL * j * mm + idx];
    if (j + 1 < G.nblk)
      for (int idx = tid; idx < mm; idx += nt) Lo[idx] = li[(2LL * (j + 1) + 1) * mm + idx];
    __syncthreads();
    double* yj = y + j * M;
    if (j + 1 < G.nblk && tid < M) {
      const double* xn = y + (j + 1) * M;
      double s0 = 0.0, s1 = 0.0;
      int k = 0;
      for (; k + 1 < M; k += 2) {
        s0 += Lo[k + tid * M] * xn[k];
        s1 += Lo[k + 1 + tid * M] * xn[k + 1];
      }
      if (k < M) s0 += Lo[k + tid * M] * xn[k];
      yj[tid] -= s0 + s1;
    }
    __syncthreads();
    for (int k = M - 1; k >= 0; --k) {
      if (tid == k) yj[k] /= Ld[k + k * M];
      __syncthreads();
      if (tid < k) yj[tid] -= Ld[k + tid * M] * yj[k];
    }
    __syncthreads();
  }
  for (int rr = tid; rr < G.nI_pad; rr += nt) {
    const int node = lt.irow_node[rr];
    if (node >= 0) {
      int a[3];
      local_coords(G, node, a);
      out[local_to_free(G, p, a)] = y[rr];
    }
  }
}

__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  return s;
}

// Per subdomain: rho = D rp_Gamma; q = c Phi^T rho; u = S_K^{-1} rho; t = C u.
__global__ void __launch_bounds__(128) local_gamma1_kernel(Geometry G, SubTables st,
                                                           const double* __restrict__ LS,
                                                           const double* __restrict__ Phi,
                                                           const double* __restrict__ cscale,
                                                           const double* __restrict__ rpg,
                                                           double* qloc, double* uloc,
                                                           double* tloc) {
  extern __shared__ double sm[];
  const int n = G.nG_pad, nc = G.nc_pad;
  double* u = sm;          // n
  double* rho = sm + n;    // n
  __shared__ double red[32];
  const int sub = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const long long so = (long long)sub * n;
  for (int s = tid; s < n; s += nt) {
    const int g = st.slot_gamma[so + s];
    const double v = g >= 0 ? st.slot_w[so + s] * rpg[g] : 0.0;
    rho[s] = v;
    u[s] = v;
  }
  __syncthreads();
  const double c = cscale[sub];
  const double* ph = Phi + (long long)sub * n * nc;
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int k = warp; k < nc; k += nw) {
    double acc = 0.0;
    for (int s = lane; s < n; s += 32) acc += ph[s + (long long)k * n] * rho[s];
    acc = warp_sum(acc);
    if (lane == 0) qloc[(long long)sub * nc + k] = c * acc;
  }
  // forward: L u = rho (column oriented)
  const double* L = LS + (long long)sub * n * n;
  for (int k = 0; k < n; ++k) {
    if (tid == 0) u[k] /= L[k + (long long)k * n];
    __syncthreads();
    const double uk = u[k];
    for (int i = k + 1 + tid; i < n; i += nt) u[i] -= L[i + (long long)k * n] * uk;
    __syncthreads();
  }
  // backward: L^T u = y (dot form over column k)
  for (int k = n - 1; k >= 0; --k) {
    double part = 0.0;
    for (int i = k + 1 + tid; i < n; i += nt) part += L[i + (long long)k * n] * u[i];
    const double tot = block_sum(part, red);
    if (tid == 0) u[k] = (u[k] - tot) / L[k + (long long)k * n];
    __syncthreads();
  }
  for (int s = tid; s < n; s += nt) uloc[so + s] = u[s];
  for (int k = tid; k < nc; k += nt) {
    double acc = 0.0;
    for (int s = 0; s < n; ++s)
      if (st.slot_con[so + s] == k) acc += st.slot_coef[so + s] * u[s];
    tloc[(long long)sub * nc + k] = acc;
  }
}

// Per subdomain: e = c * csol[coarse] - t;  w = D (u + Phi e)
__global__ void __launch_bounds__(128) local_gamma2_kernel(Geometry G, SubTables st,
                                                           const double* __restrict__ Phi,
                                                           const double* __restrict__ cscale,
                                                           const double* __restrict__ csol,
                                                           const double* __restrict__ uloc,
                                                           const double* __restrict__ tloc,
                                                           double* wloc) {
  __shared__ double e[1024];
  const int n = G.nG_pad, nc = G.nc_pad;
  const int sub = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const double c = cscale[sub];
  for (int k = tid; k < nc; k += nt) {
    const int j = st.con_coarse[(long long)sub * nc + k];
    e[k] = j >= 0 ? c * csol[j] - tloc[(long long)sub * nc + k] : 0.0;
  }
  __syncthreads();
  const double* ph = Phi + (long long)sub * n * nc;
  const long long so = (long long)sub * n;
  for (int s = tid; s < n; s += nt) {
    double acc = uloc[so + s];
    for (int k = 0; k < nc; ++k) acc += ph[s + (long long)k * n] * e[k];
    wloc[so + s] = st.slot_w[so + s] * acc;
  }
}

// z[gamma dof] = sum over owner slots (ascending subdomain = reference summation order)
__global__ void gamma_gather_kernel(int n_gamma, int W, const long long* __restrict__ gdof,
                                    const int* __restrict__ gslots, const double* __restrict__ wloc,
                                    double* __restrict__ z) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_gamma) return;
  double acc = 0.0;
  for (int w = 0; w < W; ++w) {
    const int s = gslots[(long long)g * W + w];
    if (s >= 0) acc += wloc[s];
  }
  z[gdof[g]] = acc;
}

__global__ void coarse_gather_kernel(int n_coarse, int W, const int* __restrict__ cslots,
                                     const double* __restrict__ qloc, double* __restrict__ crhs) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_coarse) return;
  double acc = 0.0;
  for (int w = 0; w < W; ++w) {
    const int s = cslots[(long long)j * W + w];
    if (s >= 0) acc += qloc[s];
  }
  crhs[j] = acc;
}

int grid_for(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  return (int)std::min<long long>(b, 148LL * 32);
}

}  // namespace

void spmv(Ctx& c, const double* x, double* y, cudaStream_t s) {
  const Geometry& G = c.geo;
  const int th = 256, gr = grid_for(G.n, th);
  if (G.dim == 2) { spmv_kernel<2><<<gr, th, 0, s>>>(G, c.alpha, x, y); BDDC_COUNT(); }
  else { spmv_kernel<3><<<gr, th, 0, s>>>(G, c.alpha, x, y); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
}

static void bt_solve(Ctx& c, const double* in, double* out, cudaStream_t s) {
  const Geometry& G = c.geo;
  PhaseScope ps(c.prof, "apply.bt_solve", s);
  const int th = G.m_pad <= 32 ? 32 : 64;
  const size_t smem = sizeof(double) * (G.nI_pad + 2LL * G.m_pad * G.m_pad);
  static size_t attr = 0;
  if (smem > attr) {
    BDDC_CUDA(cudaFuncSetAttribute(bt_solve_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    BDDC_CUDA(cudaFuncSetAttribute(bt_solve_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  if (G.dim == 2) { bt_solve_kernel<2><<<G.nsub, th, smem, s>>>(G, c.lt, c.LI, in, out); BDDC_COUNT(); }
  else { bt_solve_kernel<3><<<G.nsub, th, smem, s>>>(G, c.lt, c.LI, in, out); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
}

// out holds g on Gamma and 0 on interiors; c.v1 must be zero.
void harmonic_interior(Ctx& c, double* out, cudaStream_t s) {
  const Geometry& G = c.geo;
  const int th = 256, gr = grid_for(G.n, th);
  if (G.dim == 2) { residual_kernel<2><<<gr, th, 0, s>>>(G, c.alpha, c.v1, out, c.v2); BDDC_COUNT(); }
  else { residual_kernel<3><<<gr, th, 0, s>>>(G, c.alpha, c.v1, out, c.v2); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
  bt_solve(c, c.v2, out, s);
}

void apply_bddc(Ctx& c, const double* r, double* z, cudaStream_t s) {
  const Geometry& G = c.geo;
  const int th = 256;
  // u1 = A_II^{-1} r_I (zero on Gamma)
  BDDC_CUDA(cudaMemsetAsync(c.v1, 0, sizeof(double) * G.n, s));
  bt_solve(c, r, c.v1, s);
  if (c.n_gamma > 0) {
    if (G.dim == 2)
      { gamma_residual_kernel<2><<<ceil_div(c.n_gamma, th), th, 0, s>>>(G, c.n_gamma, c.gamma_dof, c.alpha, r, c.v1, c.rpg); BDDC_COUNT(); }
    else
      { gamma_residual_kernel<3><<<ceil_div(c.n_gamma, th), th, 0, s>>>(G, c.n_gamma, c.gamma_dof, c.alpha, r, c.v1, c.rpg); BDDC_COUNT(); }
    BDDC_LAUNCH_CHECK();
    const size_t smem1 = sizeof(double) * 2 * G.nG_pad;
    c.prof.begin("apply.gamma1", s);
    { local_gamma1_kernel<<<G.nsub, 128, smem1, s>>>(G, c.st, c.LS, c.Phi, c.cscale, c.rpg, c.qloc,
                                                   c.uloc, c.tloc); BDDC_COUNT(); }
    BDDC_LAUNCH_CHECK();
    c.prof.end("apply.gamma1", s);
    if (c.fp.n_coarse > 0) {
      PhaseScope pc(c.prof, "apply.coarse", s);
      { coarse_gather_kernel<<<ceil_div(c.fp.n_coarse, th), th, 0, s>>>(c.fp.n_coarse, c.fp.W,
                                                                     c.fp.coarse_slots, c.qloc, c.crhs); BDDC_COUNT(); }
      BDDC_LAUNCH_CHECK();
      coarse_solve(c, c.crhs, c.csol, s);
    }
    c.prof.begin("apply.gamma2", s);
    { local_gamma2_kernel<<<G.nsub, 128, 0, s>>>(G, c.st, c.Phi, c.cscale, c.csol, c.uloc, c.tloc,
                                               c.wloc); BDDC_COUNT(); }
    BDDC_LAUNCH_CHECK();
    c.prof.end("apply.gamma2", s);
  }
  BDDC_CUDA(cudaMemsetAsync(z, 0, sizeof(double) * G.n, s));
  if (c.n_gamma > 0) {
    { gamma_gather_kernel<<<ceil_div(c.n_gamma, th), th, 0, s>>>(c.n_gamma, G.npe,
                                                               c.gamma_dof, c.gamma_slots, c.wloc, z); BDDC_COUNT(); }
    BDDC_LAUNCH_CHECK();
  }
  // z_I = A_II^{-1} (r - A z_Gamma)_I
  const int gr = grid_for(G.n, th);
  if (G.dim == 2) { residual_kernel<2><<<gr, th, 0, s>>>(G, c.alpha, r, z, c.v2); BDDC_COUNT(); }
  else { residual_kernel<3><<<gr, th, 0, s>>>(G, c.alpha, r, z, c.v2); BDDC_COUNT(); }
  BDDC_LAUNCH_CHECK();
  bt_solve(c, c.v2, z, s);
}

}  // namespace bddc
