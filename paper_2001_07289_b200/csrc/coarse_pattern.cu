// Device construction of the coarse assembly pattern (cold start): the lower CSR
// of S_0 in elimination order, its segmented contribution lists and the CSR -> front positions,
// from the per-subdomain constraint -> coarse index table alone. Same arrays as the host
// statements (symbolic.coarse_csr, numpy; bddc_coarse_pattern, host C++), which stay as the
// checkers (tests/test_host_plan.py, tests/test_gpu_scale.py).
//
// Reference: the coarse COO -> CSR assembly of build_bddc (bddc.py:494-505): entry (r, c) sums
// the local coarse blocks of the subdomains owning both constraints, in ascending-subdomain
// order (the COO duplicate order the device segmented sum reproduces).
//
//   1. count: m_p (m_p + 1) / 2 pairs per subdomain, exclusive scan -> offsets
//   2. gen: pair {k >= l} of subdomain p -> key (max e, min e) = row * n + col, value = the
//      local block index of (row constraint, column constraint); written in subdomain order
//   3. stable radix sort by key (subdomain order kept inside each entry)
//   4. segment starts (key changes) -> seg_ptr, nnz; per entry: front, front row / column
#include <cub/cub.cuh>

#include "bddc_internal.cuh"

namespace bddc {
namespace {

__global__ void pair_count_kernel(int nsub, int nc_pad, const int* __restrict__ con_coarse, long long* cnt) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nsub) return;
  int m = 0;
  while (m < nc_pad && con_coarse[(long long)p * nc_pad + m] >= 0) ++m;
  cnt[p] = (long long)m * (m + 1) / 2;
}

// one warp per subdomain
__global__ void pair_gen_kernel(int nsub, int nc_pad, long long n, const int* __restrict__ con_coarse,
                                const long long* __restrict__ off, unsigned long long* key, int* val) {
  const int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= nsub) return;
  const int* e = con_coarse + (long long)p * nc_pad;
  int m = 0;
  while (m < nc_pad && e[m] >= 0) ++m;
  const long long base = (long long)p * nc_pad * nc_pad;
  const long long o = off[p];
  const long long npair = (long long)m * (m + 1) / 2;
  for (long long q = lane; q < npair; q += 32) {
    // q = k (k + 1) / 2 + l, l <= k
    int k = (int)((sqrt(8.0 * (double)q + 1.0) - 1.0) * 0.5);
    while ((long long)(k + 1) * (k + 2) / 2 <= q) ++k;
    while ((long long)k * (k + 1) / 2 > q) --k;
    const int l = (int)(q - (long long)k * (k + 1) / 2);
    const long long ek = e[k], el = e[l];
    long long r, c, idx;
    if (ek >= el) {
      r = ek; c = el; idx = base + k + (long long)l * nc_pad;
    } else {
      r = el; c = ek; idx = base + l + (long long)k * nc_pad;
    }
    key[o + q] = (unsigned long long)(r * n + c);
    val[o + q] = (int)idx;
  }
}

__global__ void newkey_kernel(long long m, const unsigned long long* __restrict__ key, int* flag) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < m) flag[i] = i == 0 || key[i] != key[i - 1];
}

__global__ void node_of_kernel(int nnodes, const int* __restrict__ sep_start, const int* __restrict__ sep_size,
                               int* node_of) {
  const int nd = blockIdx.x;
  for (int q = threadIdx.x; q < sep_size[nd]; q += blockDim.x) node_of[sep_start[nd] + q] = nd;
}

__global__ void entry_kernel(long long nnz, long long n, const unsigned long long* __restrict__ key,
                             const long long* __restrict__ start, FrontDev fd, const int* __restrict__ node_of,
                             long long* pos, int* row_out, int* col_out, int* bad) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  const unsigned long long k = key[start[e]];
  const long long r = (long long)(k / (unsigned long long)n), c = (long long)(k % (unsigned long long)n);
  row_out[e] = (int)r;
  col_out[e] = (int)c;
  const int nd = node_of[c];
  const long long s0 = fd.sep_start[nd], ss = fd.sep_size[nd];
  const long long fcol = c - s0;
  long long frow;
  if (r < s0 + ss) {
    frow = r - s0;
  } else {  // position of r among the front's boundary dofs (ascending)
    int lo = fd.bnd_ptr[nd], hi = fd.bnd_ptr[nd + 1];
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (fd.bnd_idx[mid] < r) lo = mid + 1; else hi = mid;
    }
    if (lo == fd.bnd_ptr[nd + 1] || fd.bnd_idx[lo] != r) atomicExch(bad, 1);
    frow = ss + (lo - fd.bnd_ptr[nd]);
  }
  if (fcol < 0 || fcol >= ss) atomicExch(bad, 1);
  pos[e] = fd.front_off[nd] + frow + fcol * fd.ld[nd];
}

__global__ void seg_kernel(long long nnz, long long m, const long long* __restrict__ start, long long* seg) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e < nnz) seg[e] = start[e];
  if (e == 0) seg[nnz] = m;
}

struct TmpBufs {  // scratch of the pattern build, freed on return
  std::vector<void*> p;
  template <class T>
  T* get(long long k) {
    void* q = nullptr;
    BDDC_CUDA(cudaMalloc(&q, sizeof(T) * (size_t)std::max(k, 1LL)));
    p.push_back(q);
    return (T*)q;
  }
  ~TmpBufs() {
    for (void* q : p) cudaFree(q);
  }
};

inline int grid_of(long long n, int b = 256) { return (int)std::max(1LL, (n + b - 1) / b); }

}  // namespace

// Fills fp.nnz, csr_front_pos, seg_ptr, ncontrib, contrib, csr_val, csr_row_dev / csr_col_dev.
void device_coarse_pattern(Ctx& c, const int* con_coarse_host) {
  FrontPlan& fp = c.fp;
  const Geometry& G = c.geo;
  cudaStream_t st = c.stream;
  const int nsub = (int)G.nsub, nc_pad = G.nc_pad;
  const long long n = fp.n_coarse;
  TmpBufs T;
  int* cc = T.get<int>((long long)nsub * nc_pad);
  BDDC_CUDA(cudaMemcpyAsync(cc, con_coarse_host, sizeof(int) * (size_t)nsub * nc_pad, cudaMemcpyHostToDevice, st));
  long long* cnt = T.get<long long>(nsub + 1);
  long long* off = T.get<long long>(nsub + 1);
  BDDC_CUDA(cudaMemsetAsync(cnt + nsub, 0, sizeof(long long), st));
  pair_count_kernel<<<grid_of(nsub), 256, 0, st>>>(nsub, nc_pad, cc, cnt);
  BDDC_LAUNCH_CHECK();
  BDDC_COUNT();
  size_t tb = 0;
  BDDC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, nsub + 1, st));
  void* tmp = T.get<char>((long long)tb);
  BDDC_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, nsub + 1, st));
  long long m = 0;
  BDDC_CUDA(cudaMemcpyAsync(&m, off + nsub, sizeof(long long), cudaMemcpyDeviceToHost, st));
  BDDC_CUDA(cudaStreamSynchronize(st));
  if ((long long)nsub * nc_pad * nc_pad >= (1LL << 31)) throw CudaError("coarse pattern: local block index exceeds int32");
  unsigned long long* key[2] = {T.get<unsigned long long>(m), T.get<unsigned long long>(m)};
  int* val[2] = {T.get<int>(m), nullptr};
  fp.contrib = c.alloc<int>(std::max(m, 1LL));  // the sorted values land here
  val[1] = fp.contrib;
  pair_gen_kernel<<<grid_of((long long)nsub * 32), 256, 0, st>>>(nsub, nc_pad, n, cc, off, key[0], val[0]);
  BDDC_LAUNCH_CHECK();
  BDDC_COUNT();
  int bits = 1;
  while (bits < 64 && (1ULL << bits) <= (unsigned long long)(n * n)) ++bits;
  size_t tb2 = 0;
  BDDC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb2, key[0], key[1], val[0], val[1], m, 0, bits, st));
  void* tmp2 = T.get<char>((long long)tb2);
  BDDC_CUDA(cub::DeviceRadixSort::SortPairs(tmp2, tb2, key[0], key[1], val[0], val[1], m, 0, bits, st));
  unsigned long long* sk = key[1];
  int* flag = T.get<int>(m);
  newkey_kernel<<<grid_of(m), 256, 0, st>>>(m, sk, flag);
  BDDC_LAUNCH_CHECK();
  BDDC_COUNT();
  long long* start = T.get<long long>(m);
  long long* nsel = T.get<long long>(1);
  size_t tb3 = 0;
  cub::CountingInputIterator<long long> it(0);
  BDDC_CUDA(cub::DeviceSelect::Flagged(nullptr, tb3, it, flag, start, nsel, m, st));
  void* tmp3 = T.get<char>((long long)tb3);
  BDDC_CUDA(cub::DeviceSelect::Flagged(tmp3, tb3, it, flag, start, nsel, m, st));
  long long nnz = 0;
  BDDC_CUDA(cudaMemcpyAsync(&nnz, nsel, sizeof(long long), cudaMemcpyDeviceToHost, st));
  BDDC_CUDA(cudaStreamSynchronize(st));
  fp.nnz = nnz;
  fp.ncontrib = m;
  fp.seg_ptr = c.alloc<long long>(nnz + 1);
  fp.csr_front_pos = c.alloc<long long>(std::max(nnz, 1LL));
  fp.csr_row_dev = c.alloc<int>(std::max(nnz, 1LL));
  fp.csr_col_dev = c.alloc<int>(std::max(nnz, 1LL));
  fp.csr_val = c.alloc<double>(std::max(nnz, 1LL));
  int* node_of = T.get<int>(n);
  int* bad = T.get<int>(1);
  BDDC_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  node_of_kernel<<<fp.nnodes, 256, 0, st>>>(fp.nnodes, fp.d.sep_start, fp.d.sep_size, node_of);
  BDDC_LAUNCH_CHECK();
  BDDC_COUNT();
  seg_kernel<<<grid_of(nnz + 1), 256, 0, st>>>(nnz, m, start, fp.seg_ptr);
  BDDC_LAUNCH_CHECK();
  BDDC_COUNT();
  entry_kernel<<<grid_of(nnz), 256, 0, st>>>(nnz, n, sk, start, fp.d, node_of, fp.csr_front_pos, fp.csr_row_dev,
                                             fp.csr_col_dev, bad);
  BDDC_LAUNCH_CHECK();
  BDDC_COUNT();
  int hbad = 0;
  BDDC_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  BDDC_CUDA(cudaStreamSynchronize(st));
  if (hbad) throw CudaError("coarse pattern: an entry falls outside its front");
}

}  // namespace bddc
