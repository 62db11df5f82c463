// Device index-set pipeline: membership, interface objects and their per-owner weights of a
// partition pair, bit-exact with the reference's host code:
//   membership      partition.py:117-131  (sorted distinct labels of the cells at each dof)
//   Γ / Γ̂           partition.py:79-83    (dofs with >= 2 subdomain / subsubdomain labels)
//   objects          partition.py:223-250  (Γ dofs grouped by Θ̂ signature, Python tuple order,
//                                           dofs ascending; kind; owners = sorted parents)
//   weights          bddc.py:108-145       (counting 1/|owners|, cardinality #hats in Ω_i / #hats)
//
// Pipeline (one stream, one sync at the end):
//   1. member_kernel: per free dof, the 2^d cell labels sorted in registers -> Γ / Γ̂ flags
//   2. cub::DeviceSelect::Flagged: ascending Γ (and Γ̂) dof lists
//   3. sig_kernel: the −1 padded Θ̂ signature row of every Γ dof
//   4. LSD radix sort of the rows: the columns packed into 64-bit keys (as many labels per key
//      as the label width allows), stable cub::DeviceRadixSort::SortPairs from the last column
//      group to the first, starting from ascending dofs -> Python tuple order with −1 (= the
//      end of a shorter tuple) below every label, dofs ascending inside a signature
//   5. object starts (row differs from its predecessor) by a flag + inclusive scan
//   6. obj_kernel: signature, kind, owners, weights per object; dof_kernel: dof lists
// The coefficient weighting (exact rationals of α, bddc.py:137-142) stays on the host.
#include <cub/cub.cuh>

#include <cstring>
#include <type_traits>
#include <string>
#include <vector>

#include "bddc_internal.cuh"

namespace bddc {
namespace {

constexpr int kMaxW = 8;

struct IxGeom {
  int dim, W;
  int nf[3];      // free nodes per axis (cells - 1)
  long long cs[3];  // cell strides (x fastest)
};

template <int W>
__device__ __forceinline__ void sort_small(int (&v)[W]) {
#pragma unroll
  for (int i = 1; i < W; ++i)
#pragma unroll
    for (int j = i; j > 0; --j)
      if (v[j] < v[j - 1]) {
        const int t = v[j];
        v[j] = v[j - 1];
        v[j - 1] = t;
      }
}

// labels of the 2^d cells around free dof f; corner c has bit d <-> -1 on axis d of the node
template <int W>
__device__ __forceinline__ void cell_labels(const IxGeom& g, long long f, const int* __restrict__ hat, int (&v)[W]) {
  long long rem = f;
  long long node[3] = {0, 0, 0};
  for (int d = 0; d < g.dim; ++d) {
    node[d] = rem % g.nf[d] + 1;
    rem /= g.nf[d];
  }
#pragma unroll
  for (int c = 0; c < W; ++c) {
    long long cid = 0;
    for (int d = 0; d < g.dim; ++d) cid += (node[d] - ((c >> d) & 1)) * g.cs[d];
    v[c] = __ldg(hat + cid);
  }
}

// distinct sorted values in place (front), count returned; the rest set to -1
template <int W>
__device__ __forceinline__ int distinct_sorted(int (&v)[W]) {
  sort_small<W>(v);
  int n = 1;
#pragma unroll
  for (int i = 1; i < W; ++i)
    if (v[i] != v[n - 1]) v[n++] = v[i];
#pragma unroll
  for (int i = 0; i < W; ++i)
    if (i >= n) v[i] = -1;
  return n;
}

template <int W>
__global__ void member_kernel(IxGeom g, long long n_free, const int* __restrict__ hat, const int* __restrict__ parent,
                              unsigned char* gflag, unsigned char* hflag) {
  const long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (f >= n_free) return;
  int v[W];
  cell_labels<W>(g, f, hat, v);
  const int nh = distinct_sorted<W>(v);
  int p[W];
#pragma unroll
  for (int i = 0; i < W; ++i) p[i] = i < nh ? __ldg(parent + v[i]) : 0x7fffffff;
  sort_small<W>(p);
  int np = 1;
#pragma unroll
  for (int i = 1; i < W; ++i)
    if (i < nh && p[i] != p[i - 1]) ++np;
  gflag[f] = np >= 2;
  hflag[f] = nh >= 2;
}

template <int W>
__global__ void sig_kernel(IxGeom g, int n_gamma, const int* __restrict__ gamma, const int* __restrict__ hat,
                           int* rows, int* lens) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_gamma) return;
  int v[W];
  cell_labels<W>(g, gamma[i], hat, v);
  lens[i] = distinct_sorted<W>(v);
#pragma unroll
  for (int k = 0; k < W; ++k) rows[(long long)i * W + k] = v[k];
}

// key of columns [c0, c1) of row perm[i]: (label + 1) per column, the first column most significant
__global__ void key_kernel(int n, int W, const int* __restrict__ rows, const int* __restrict__ perm, int c0, int c1,
                           int bits, unsigned long long* key) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int* r = rows + (long long)perm[i] * W;
  unsigned long long k = 0;
  for (int c = c0; c < c1; ++c) k = (k << bits) | (unsigned long long)(unsigned)(r[c] + 1);
  key[i] = k;
}

__global__ void iota_kernel(int n, int* a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}

__global__ void newobj_kernel(int n, int W, const int* __restrict__ rows, const int* __restrict__ perm, int* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int f = i == 0;
  if (!f) {
    const int* a = rows + (long long)perm[i] * W;
    const int* b = rows + (long long)perm[i - 1] * W;
    for (int k = 0; k < W; ++k) f |= a[k] != b[k];
  }
  flag[i] = f;
}

// per object: signature / kind / owners / weights (counting and cardinality)
template <int W>
__global__ void obj_kernel(int n_obj, int n_gamma, int dim, const int* __restrict__ starts, const int* __restrict__ rows,
                           const int* __restrict__ lens, const int* __restrict__ perm, const int* __restrict__ parent,
                           int* sig, int* sig_len, int* owners, int* owner_len, signed char* kind, double* w_count,
                           double* w_card, int* card_cnt) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= n_obj) return;
  const int s = starts[o], e = o + 1 < n_obj ? starts[o + 1] : n_gamma;
  const int src = perm[s];
  const int L = lens[src];
  int v[W], p[W];
#pragma unroll
  for (int k = 0; k < W; ++k) {
    v[k] = rows[(long long)src * W + k];
    sig[(long long)o * W + k] = v[k];
    p[k] = k < L ? __ldg(parent + v[k]) : 0x7fffffff;
  }
  sig_len[o] = L;
  const int nd = e - s;
  kind[o] = nd == 1 ? 0 : (L == 2 ? (dim == 3 ? 2 : 1) : 1);
  int q[W];
#pragma unroll
  for (int k = 0; k < W; ++k) q[k] = p[k];
  sort_small<W>(q);
  int no = 0;
#pragma unroll
  for (int k = 0; k < W; ++k)
    if (q[k] != 0x7fffffff && (no == 0 || q[k] != q[no - 1])) q[no++] = q[k];
  owner_len[o] = no;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const long long at = (long long)o * W + k;
    if (k < no) {
      int cnt = 0;
#pragma unroll
      for (int h = 0; h < W; ++h) cnt += p[h] == q[k];
      owners[at] = q[k];
      card_cnt[at] = cnt;
      w_count[at] = 1.0 / (double)no;
      w_card[at] = (double)cnt / (double)L;
    } else {
      owners[at] = -1;
      card_cnt[at] = 0;
      w_count[at] = 0.0;
      w_card[at] = 0.0;
    }
  }
}

__global__ void dof_kernel(int n, const int* __restrict__ gamma, const int* __restrict__ perm,
                           const int* __restrict__ incl, int* obj_dofs, int* dof_obj) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int d = gamma[perm[i]];
  obj_dofs[i] = d;
  dof_obj[d] = incl[i] - 1;
}

struct DevBuf {
  std::vector<void*> ptrs;
  template <class T>
  T* get(long long n) {
    void* p = nullptr;
    BDDC_CUDA(cudaMalloc(&p, sizeof(T) * (size_t)std::max(n, 1LL)));
    ptrs.push_back(p);
    return (T*)p;
  }
  ~DevBuf() {
    for (void* p : ptrs) cudaFree(p);
  }
};

inline int grid_of(long long n, int b = 256) { return (int)std::max(1LL, (n + b - 1) / b); }

}  // namespace

// Host copies of the results (the caller copies them out by name).
struct IndexResult {
  int dim = 0, W = 0;
  long long n_free = 0, n_gamma = 0, n_gamma_hat = 0, n_obj = 0;
  std::vector<int> gamma, gamma_hat, sig, sig_len, owners, owner_len, obj_ptr, obj_dofs, dof_obj, card_cnt;
  std::vector<signed char> kind;
  std::vector<double> w_count, w_card;
};

template <int W>
static void run_index(IndexResult& R, int device, int dim, const int* cells, const int* theta_hat_h,
                      const int* parent_h, int n_hat) {
  BDDC_CUDA(cudaSetDevice(device));
  cudaStream_t st;
  BDDC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{st};
  IxGeom g{};
  g.dim = dim;
  g.W = W;
  long long ncell = 1, n_free = 1, stride = 1;
  for (int d = 0; d < dim; ++d) {
    g.nf[d] = cells[d] - 1;
    g.cs[d] = stride;
    stride *= cells[d];
    ncell *= cells[d];
    n_free *= cells[d] - 1;
  }
  R.dim = dim;
  R.W = W;
  R.n_free = n_free;
  if (n_free <= 0) return;
  if (n_free > (1LL << 31) - 1) throw CudaError("index sets: more than 2^31 free dofs");
  DevBuf B;
  int* hat = B.get<int>(ncell);
  int* par = B.get<int>(n_hat);
  BDDC_CUDA(cudaMemcpyAsync(hat, theta_hat_h, sizeof(int) * ncell, cudaMemcpyHostToDevice, st));
  BDDC_CUDA(cudaMemcpyAsync(par, parent_h, sizeof(int) * n_hat, cudaMemcpyHostToDevice, st));
  unsigned char* gflag = B.get<unsigned char>(n_free);
  unsigned char* hflag = B.get<unsigned char>(n_free);
  member_kernel<W><<<grid_of(n_free), 256, 0, st>>>(g, n_free, hat, par, gflag, hflag);
  BDDC_LAUNCH_CHECK();
  BDDC_COUNT();
  // Γ / Γ̂ lists (ascending)
  int* gamma = B.get<int>(n_free);
  int* gamma_hat = B.get<int>(n_free);
  int* cnt = B.get<int>(2);
  size_t tmp_bytes = 0, t2 = 0;
  cub::CountingInputIterator<int> it(0);
  BDDC_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp_bytes, it, gflag, gamma, cnt, (int)n_free, st));
  void* tmp = B.get<char>((long long)tmp_bytes);
  BDDC_CUDA(cub::DeviceSelect::Flagged(tmp, tmp_bytes, it, gflag, gamma, cnt, (int)n_free, st));
  BDDC_CUDA(cub::DeviceSelect::Flagged(tmp, tmp_bytes, it, hflag, gamma_hat, cnt + 1, (int)n_free, st));
  int hc[2];
  BDDC_CUDA(cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, st));
  BDDC_CUDA(cudaStreamSynchronize(st));
  const int ng = hc[0];
  R.n_gamma = ng;
  R.n_gamma_hat = hc[1];
  R.gamma.resize(ng);
  R.gamma_hat.resize(hc[1]);
  BDDC_CUDA(cudaMemcpyAsync(R.gamma.data(), gamma, sizeof(int) * ng, cudaMemcpyDeviceToHost, st));
  BDDC_CUDA(cudaMemcpyAsync(R.gamma_hat.data(), gamma_hat, sizeof(int) * hc[1], cudaMemcpyDeviceToHost, st));
  R.dof_obj.assign(n_free, -1);
  if (ng == 0) {
    R.obj_ptr.assign(1, 0);
    BDDC_CUDA(cudaStreamSynchronize(st));
    return;
  }
  // signatures and their lexicographic (Python tuple) order
  int* rows = B.get<int>((long long)ng * W);
  int* lens = B.get<int>(ng);
  sig_kernel<W><<<grid_of(ng), 256, 0, st>>>(g, ng, gamma, hat, rows, lens);
  BDDC_LAUNCH_CHECK();
  BDDC_COUNT();
  int bits = 1;
  while ((1LL << bits) <= (long long)n_hat) ++bits;  // label + 1 in [0, n_hat]
  const int per = std::max(1, std::min(W, 64 / bits));
  int* perm[2] = {B.get<int>(ng), B.get<int>(ng)};
  unsigned long long* key[2] = {B.get<unsigned long long>(ng), B.get<unsigned long long>(ng)};
  iota_kernel<<<grid_of(ng), 256, 0, st>>>(ng, perm[0]);
  BDDC_LAUNCH_CHECK();
  BDDC_COUNT();
  BDDC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t2, key[0], key[1], perm[0], perm[1], ng, 0, 64, st));
  void* tmp2 = B.get<char>((long long)t2);
  int cur = 0;
  for (int c1 = W; c1 > 0; c1 -= per) {
    const int c0 = std::max(0, c1 - per);
    key_kernel<<<grid_of(ng), 256, 0, st>>>(ng, W, rows, perm[cur], c0, c1, bits, key[0]);
    BDDC_LAUNCH_CHECK();
    BDDC_COUNT();
    size_t tb = t2;
    BDDC_CUDA(cub::DeviceRadixSort::SortPairs(tmp2, tb, key[0], key[1], perm[cur], perm[cur ^ 1], ng, 0,
                                              bits * (c1 - c0), st));
    cur ^= 1;
  }
  int* P = perm[cur];
  // object starts
  int* flag = B.get<int>(ng);
  int* incl = B.get<int>(ng);
  newobj_kernel<<<grid_of(ng), 256, 0, st>>>(ng, W, rows, P, flag);
  BDDC_LAUNCH_CHECK();
  BDDC_COUNT();
  size_t t3 = 0;
  BDDC_CUDA(cub::DeviceScan::InclusiveSum(nullptr, t3, flag, incl, ng, st));
  void* tmp3 = B.get<char>((long long)t3);
  BDDC_CUDA(cub::DeviceScan::InclusiveSum(tmp3, t3, flag, incl, ng, st));
  int* starts = B.get<int>(ng);
  size_t t4 = 0;
  BDDC_CUDA(cub::DeviceSelect::Flagged(nullptr, t4, it, flag, starts, cnt, ng, st));
  void* tmp4 = B.get<char>((long long)t4);
  BDDC_CUDA(cub::DeviceSelect::Flagged(tmp4, t4, it, flag, starts, cnt, ng, st));
  int nobj = 0;
  BDDC_CUDA(cudaMemcpyAsync(&nobj, cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
  BDDC_CUDA(cudaStreamSynchronize(st));
  R.n_obj = nobj;
  int* sig = B.get<int>((long long)nobj * W);
  int* sig_len = B.get<int>(nobj);
  int* owners = B.get<int>((long long)nobj * W);
  int* owner_len = B.get<int>(nobj);
  signed char* kind = B.get<signed char>(nobj);
  double* w_count = B.get<double>((long long)nobj * W);
  double* w_card = B.get<double>((long long)nobj * W);
  int* card_cnt = B.get<int>((long long)nobj * W);
  obj_kernel<W><<<grid_of(nobj, 128), 128, 0, st>>>(nobj, ng, dim, starts, rows, lens, P, par, sig, sig_len, owners,
                                                owner_len, kind, w_count, w_card, card_cnt);
  BDDC_LAUNCH_CHECK();
  BDDC_COUNT();
  int* obj_dofs = B.get<int>(ng);
  int* dof_obj = B.get<int>(n_free);
  BDDC_CUDA(cudaMemsetAsync(dof_obj, 0xff, sizeof(int) * n_free, st));
  dof_kernel<<<grid_of(ng), 256, 0, st>>>(ng, gamma, P, incl, obj_dofs, dof_obj);
  BDDC_LAUNCH_CHECK();
  BDDC_COUNT();
  auto d2h = [&](auto& v, const auto* src, long long n) {
    v.resize(n);
    BDDC_CUDA(cudaMemcpyAsync(v.data(), src, sizeof(v[0]) * n, cudaMemcpyDeviceToHost, st));
  };
  d2h(R.sig, sig, (long long)nobj * W);
  d2h(R.sig_len, sig_len, nobj);
  d2h(R.owners, owners, (long long)nobj * W);
  d2h(R.owner_len, owner_len, nobj);
  d2h(R.kind, kind, nobj);
  d2h(R.w_count, w_count, (long long)nobj * W);
  d2h(R.w_card, w_card, (long long)nobj * W);
  d2h(R.card_cnt, card_cnt, (long long)nobj * W);
  d2h(R.obj_dofs, obj_dofs, ng);
  d2h(R.dof_obj, dof_obj, n_free);
  std::vector<int> st_h;
  d2h(st_h, starts, nobj);
  BDDC_CUDA(cudaStreamSynchronize(st));
  R.obj_ptr.resize(nobj + 1);
  for (int o = 0; o < nobj; ++o) R.obj_ptr[o] = st_h[o];
  R.obj_ptr[nobj] = ng;
}

// ---- per-subdomain slot tables of the device operator (layout.py, bddc.py:420-490) ----
namespace {

struct LayGeom {
  int dim, nsub, nG, nG_pad, W, nloc;
  int subs[3], blk[3], cells[3], nf[3];
};

// one thread per (subdomain p, surface slot j): global free dof, interface position, local
// constraint (binary search in p's ascending constraint list), coefficient, weight
__global__ void slot_kernel(LayGeom g, const int* __restrict__ slot_coords, const int* __restrict__ gidx,
                            const int* __restrict__ con_of, const double* __restrict__ coef_of,
                            const int* __restrict__ dof_obj, const int* __restrict__ owners,
                            const double* __restrict__ obj_w, const long long* __restrict__ sub_con_ptr,
                            const int* __restrict__ sub_con, int* slot_gamma, int* slot_con, double* slot_coef,
                            double* slot_w) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)g.nsub * g.nG_pad) return;
  const int p = (int)(idx / g.nG_pad), j = (int)(idx % g.nG_pad);
  int sg = -1, sc = -1;
  double co = 0.0, w = 0.0;
  if (j < g.nG) {
    int rem = p;
    long long fid = 0, st = 1;
    bool dir = false;
    for (int d = 0; d < g.dim; ++d) {
      const int pc = rem % g.subs[d];
      rem /= g.subs[d];
      const int gc = pc * g.blk[d] + slot_coords[j * g.dim + d];
      dir |= gc == 0 || gc == g.cells[d];
      fid += (long long)(gc - 1) * st;
      st *= g.nf[d];
    }
    if (!dir) {
      sg = gidx[fid];
      const int cn = con_of[fid];
      if (cn >= 0) {
        long long lo = sub_con_ptr[p], hi = sub_con_ptr[p + 1];
        const long long a0 = lo;
        while (lo < hi) {
          const long long mid = (lo + hi) >> 1;
          if (sub_con[mid] < cn) lo = mid + 1; else hi = mid;
        }
        sc = (int)(lo - a0);
        co = coef_of[fid];
      }
      const int o = dof_obj[fid];
      for (int k = 0; k < g.W; ++k)
        if (owners[(long long)o * g.W + k] == p) w += obj_w[(long long)o * g.W + k];
    }
  }
  slot_gamma[idx] = sg;
  slot_con[idx] = sc;
  slot_coef[idx] = co;
  slot_w[idx] = w;
}

__global__ void gidx_kernel(int n, const int* __restrict__ gam, int* gidx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) gidx[gam[i]] = i;
}

// one thread per (interface dof, owner k): the owner's slot of the dof, -1 padded
__global__ void gamma_slot_kernel(LayGeom g, int n_gamma, const int* __restrict__ gamma, const int* __restrict__ dof_obj,
                                  const int* __restrict__ owners, const int* __restrict__ slot_of_node, int* out) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)n_gamma * g.W) return;
  const int gi = (int)(idx / g.W), k = (int)(idx % g.W);
  const int dof = gamma[gi];
  const int p = owners[(long long)dof_obj[dof] * g.W + k];
  int v = -1;
  if (p >= 0) {
    int rem = dof, prem = p;
    long long ln = 0, st = 1;
    for (int d = 0; d < g.dim; ++d) {
      const int gc = rem % g.nf[d] + 1;
      rem /= g.nf[d];
      const int pc = prem % g.subs[d];
      prem /= g.subs[d];
      ln += (long long)(gc - pc * g.blk[d]) * st;
      st *= g.blk[d] + 1;
    }
    const int sl = (ln >= 0 && ln < g.nloc) ? slot_of_node[ln] : -1;
    v = sl >= 0 ? p * g.nG_pad + sl : -2;  // -2: the dof is not a surface slot of its owner
  }
  out[idx] = v;
}

}  // namespace
}  // namespace bddc

extern "C" int bddc_layout_tables(int device, int dim, const int* cells, const int* subs, int nG, int nG_pad, int nloc,
                                  const int* slot_coords, const int* slot_of_node, long long n_free,
                                  const int* gamma, int n_gamma, const int* con_of, const double* coef_of,
                                  const int* dof_obj, int n_obj, const int* owners, const double* obj_w,
                                  const long long* sub_con_ptr, const int* sub_con, int* slot_gamma, int* slot_con,
                                  double* slot_coef, double* slot_w, int* gamma_slots, char* err, size_t errlen) {
  using namespace bddc;
  try {
    BDDC_CUDA(cudaSetDevice(device));
    LayGeom g{};
    g.dim = dim;
    g.W = 1 << dim;
    g.nG = nG;
    g.nG_pad = nG_pad;
    g.nloc = nloc;
    g.nsub = 1;
    for (int d = 0; d < dim; ++d) {
      g.subs[d] = subs[d];
      g.cells[d] = cells[d];
      g.blk[d] = cells[d] / subs[d];
      g.nf[d] = cells[d] - 1;
      g.nsub *= subs[d];
    }
    cudaStream_t st;
    BDDC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct SG {
      cudaStream_t s;
      ~SG() { cudaStreamDestroy(s); }
    } sgd{st};
    DevBuf B;
    auto up = [&](const auto* h, long long n) {
      using T = std::remove_cv_t<std::remove_pointer_t<decltype(h)>>;
      T* d = B.get<T>(n);
      if (n) BDDC_CUDA(cudaMemcpyAsync(d, h, sizeof(T) * n, cudaMemcpyHostToDevice, st));
      return d;
    };
    const long long nslots = (long long)g.nsub * nG_pad;
    const long long ncon_pairs = sub_con_ptr[g.nsub];
    int* d_sc = up(slot_coords, (long long)nG * dim);
    int* d_son = up(slot_of_node, nloc);
    int* d_gamma = up(gamma, n_gamma);
    int* d_con = up(con_of, n_free);
    double* d_coef = up(coef_of, n_free);
    int* d_dobj = up(dof_obj, n_free);
    int* d_own = up(owners, (long long)n_obj * g.W);
    double* d_w = up(obj_w, (long long)n_obj * g.W);
    long long* d_ptr = up(sub_con_ptr, g.nsub + 1);
    int* d_scon = up(sub_con, ncon_pairs);
    // interface position of every free dof
    int* d_gidx = B.get<int>(n_free);
    BDDC_CUDA(cudaMemsetAsync(d_gidx, 0xff, sizeof(int) * n_free, st));
    if (n_gamma) {  // gidx[gamma[i]] = i
      gidx_kernel<<<grid_of(n_gamma), 256, 0, st>>>(n_gamma, d_gamma, d_gidx);
      BDDC_LAUNCH_CHECK();
      BDDC_COUNT();
    }
    int* o_sg = B.get<int>(nslots);
    int* o_sc = B.get<int>(nslots);
    double* o_co = B.get<double>(nslots);
    double* o_w = B.get<double>(nslots);
    int* o_gs = B.get<int>((long long)n_gamma * g.W);
    slot_kernel<<<grid_of(nslots), 256, 0, st>>>(g, d_sc, d_gidx, d_con, d_coef, d_dobj, d_own, d_w, d_ptr, d_scon,
                                                 o_sg, o_sc, o_co, o_w);
    BDDC_LAUNCH_CHECK();
    BDDC_COUNT();
    if (n_gamma) {
      gamma_slot_kernel<<<grid_of((long long)n_gamma * g.W), 256, 0, st>>>(g, n_gamma, d_gamma, d_dobj, d_own, d_son,
                                                                          o_gs);
      BDDC_LAUNCH_CHECK();
      BDDC_COUNT();
    }
    BDDC_CUDA(cudaMemcpyAsync(slot_gamma, o_sg, sizeof(int) * nslots, cudaMemcpyDeviceToHost, st));
    BDDC_CUDA(cudaMemcpyAsync(slot_con, o_sc, sizeof(int) * nslots, cudaMemcpyDeviceToHost, st));
    BDDC_CUDA(cudaMemcpyAsync(slot_coef, o_co, sizeof(double) * nslots, cudaMemcpyDeviceToHost, st));
    BDDC_CUDA(cudaMemcpyAsync(slot_w, o_w, sizeof(double) * nslots, cudaMemcpyDeviceToHost, st));
    if (n_gamma)
      BDDC_CUDA(cudaMemcpyAsync(gamma_slots, o_gs, sizeof(int) * n_gamma * g.W, cudaMemcpyDeviceToHost, st));
    BDDC_CUDA(cudaStreamSynchronize(st));
  } catch (const std::exception& e) {
    if (err && errlen) {
      const std::string m = e.what();
      const size_t n = std::min(errlen - 1, m.size());
      memcpy(err, m.data(), n);
      err[n] = 0;
    }
    return 6;
  }
  return 0;
}

struct bddc_index {
  bddc::IndexResult r;
};

extern "C" {

int bddc_index_build(int device, int dim, const int* cells, const int* theta_hat, const int* parent, int n_hat,
                     bddc_index** out, char* err, size_t errlen) {
  auto set = [&](const std::string& m) {
    if (err && errlen) {
      const size_t n = std::min(errlen - 1, m.size());
      memcpy(err, m.data(), n);
      err[n] = 0;
    }
  };
  if (!out || !cells || !theta_hat || !parent || (dim != 2 && dim != 3) || n_hat < 1) {
    set("invalid argument");
    return 1;
  }
  *out = nullptr;
  for (int d = 0; d < dim; ++d)
    if (cells[d] < 1) {
      set("cells must be positive");
      return 1;
    }
  bddc_index* ix = new bddc_index;
  try {
    if (dim == 2)
      bddc::run_index<4>(ix->r, device, dim, cells, theta_hat, parent, n_hat);
    else
      bddc::run_index<8>(ix->r, device, dim, cells, theta_hat, parent, n_hat);
  } catch (const std::exception& e) {
    delete ix;
    set(e.what());
    return 6;
  }
  *out = ix;
  return 0;
}

long long bddc_index_size(const bddc_index* ix, const char* what) {
  if (!ix || !what) return -1;
  const auto& r = ix->r;
  const std::string w(what);
  if (w == "n_free") return r.n_free;
  if (w == "n_gamma") return r.n_gamma;
  if (w == "n_gamma_hat") return r.n_gamma_hat;
  if (w == "n_obj") return r.n_obj;
  if (w == "width") return r.W;
  return -1;
}

// int arrays are widened to int64, kind is int8, weights float64; count must match
int bddc_index_copy(const bddc_index* ix, const char* name, void* host, long long count) {
  if (!ix || !name || (!host && count)) return 1;
  const auto& r = ix->r;
  const std::string n(name);
  auto wide = [&](const std::vector<int>& v) {
    if ((long long)v.size() != count) return 1;
    long long* o = (long long*)host;
    for (long long i = 0; i < count; ++i) o[i] = v[i];
    return 0;
  };
  if (n == "gamma_dofs") return wide(r.gamma);
  if (n == "gamma_hat_dofs") return wide(r.gamma_hat);
  if (n == "signature") return wide(r.sig);
  if (n == "sig_len") return wide(r.sig_len);
  if (n == "owners") return wide(r.owners);
  if (n == "owner_len") return wide(r.owner_len);
  if (n == "dof_ptr") return wide(r.obj_ptr);
  if (n == "dof_list") return wide(r.obj_dofs);
  if (n == "dof_obj") return wide(r.dof_obj);
  if (n == "card_counts") return wide(r.card_cnt);
  if (n == "kind") {
    if ((long long)r.kind.size() != count) return 1;
    memcpy(host, r.kind.data(), count);
    return 0;
  }
  if (n == "w_counting" || n == "w_cardinality") {
    const auto& v = n == "w_counting" ? r.w_count : r.w_card;
    if ((long long)v.size() != count) return 1;
    memcpy(host, v.data(), sizeof(double) * count);
    return 0;
  }
  return 1;
}

void bddc_index_free(bddc_index* ix) { delete ix; }

}  // extern "C"
