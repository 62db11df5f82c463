// Multi-GPU sharding of the operator: one rank per GPU, each owning a slab
// of the subdomain lattice along the last axis.
//
// Every rank keeps global-length vectors and the global index tables (small) but factors,
// stores and applies only its own subdomains. A slab's subdomains are a contiguous id range
// and its node rows a contiguous free-dof range (x-fastest numbering, mesh.py:88-102), so
// every exchange is a contiguous block:
//   * dof halo: the node row (plane) next to each cut line, for the stencil at cut rows
//     (u1 before the interface residual; p before the PCG SpMV);
//   * boundary subdomain rows: the per-slot interface values w of the neighbour's subdomains
//     touching the cut, so the interface gather sums every owner slot in the single-GPU order;
//   * allgather of per-subdomain blocks: local coarse blocks (setup) and local coarse
//     right-hand sides (apply), so the replicated coarse problem is assembled in the
//     single-GPU order on every rank (bit-identical coarse factor and solution);
//   * sum-allreduce of the PCG scalars (dots over owned rows).
// Exchanges happen between kernel launches on the operator stream; no kernel waits on
// another rank. Transports: NCCL (dlopen'd: the process may already hold torch's NCCL) and a
// host callback (tests with ranks sharing one GPU, staged through pinned host buffers).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>

#include "bddc_internal.cuh"

namespace bddc {

void slab_partition(Geometry& G, Slab& sl, int rank, int world, const long long* gamma_dof, int n_gamma) {
  const int ax = G.dim - 1;
  const int R = G.subs[ax];
  if (world < 1 || rank < 0 || rank >= world) throw std::runtime_error("invalid rank / world size");
  if (world > R)
    throw std::runtime_error("more ranks (" + std::to_string(world) + ") than subdomain rows along the last axis (" +
                             std::to_string(R) + ")");
  if (world > 1 && G.blk[ax] < 2) throw std::runtime_error("sharding needs >= 2 cells per subdomain along the last axis");
  const int r_lo = (int)((long long)rank * R / world), r_hi = (int)((long long)(rank + 1) * R / world);
  sl = Slab{};
  sl.sub_row = G.nsub / R;
  G.s_lo = r_lo * sl.sub_row;
  G.s_hi = r_hi * sl.sub_row;
  sl.row_len = G.n / G.nfree[ax];
  const int H = G.blk[ax];
  const int cut_lo = r_lo * H, cut_hi = r_hi * H;
  const int y_lo = std::max(cut_lo, 1), y_hi = std::min(cut_hi, G.cells[ax] - 1);  // active rows
  G.f_lo = (long long)(y_lo - 1) * sl.row_len;
  G.f_hi = (long long)y_hi * sl.row_len;
  G.fo_lo = rank == 0 ? G.f_lo : (long long)cut_lo * sl.row_len;
  G.fo_hi = G.f_hi;
  if (rank > 0) {
    sl.lo_recv = (long long)(cut_lo - 2) * sl.row_len;  // row cut_lo - 1
    sl.lo_send = (long long)cut_lo * sl.row_len;        // row cut_lo + 1
    sl.lo_rows_send = G.s_lo;
    sl.lo_rows_recv = G.s_lo - sl.sub_row;
  }
  if (rank < world - 1) {
    sl.hi_recv = (long long)cut_hi * sl.row_len;        // row cut_hi + 1
    sl.hi_send = (long long)(cut_hi - 2) * sl.row_len;  // row cut_hi - 1
    sl.hi_rows_send = G.s_hi - sl.sub_row;
    sl.hi_rows_recv = G.s_hi;
  }
  sl.sub_off.resize(world);
  sl.sub_cnt.resize(world);
  for (int r = 0; r < world; ++r) {
    const long long a = (long long)r * R / world, b = (long long)(r + 1) * R / world;
    sl.sub_off[r] = a * sl.sub_row;
    sl.sub_cnt[r] = (b - a) * sl.sub_row;
  }
  G.g_lo = (int)(std::lower_bound(gamma_dof, gamma_dof + n_gamma, G.f_lo) - gamma_dof);
  G.g_hi = (int)(std::lower_bound(gamma_dof, gamma_dof + n_gamma, G.f_hi) - gamma_dof);
}

void exchange_dof_halo(Ctx& c, double* v, cudaStream_t s) {
  if (!c.tp) return;
  const Slab& sl = c.slab;
  const bool lo = sl.lo_send >= 0, hi = sl.hi_send >= 0;
  c.tp->neighbors(lo ? v + sl.lo_send : nullptr, lo ? v + sl.lo_recv : nullptr, lo ? sl.row_len : 0,
                  hi ? v + sl.hi_send : nullptr, hi ? v + sl.hi_recv : nullptr, hi ? sl.row_len : 0, s);
}

void exchange_boundary_rows(Ctx& c, double* per_sub, int stride, cudaStream_t s) {
  if (!c.tp) return;
  const Slab& sl = c.slab;
  const long long n = (long long)sl.sub_row * stride;
  const bool lo = sl.lo_rows_send >= 0, hi = sl.hi_rows_send >= 0;
  c.tp->neighbors(lo ? per_sub + (long long)sl.lo_rows_send * stride : nullptr,
                  lo ? per_sub + (long long)sl.lo_rows_recv * stride : nullptr, lo ? n : 0,
                  hi ? per_sub + (long long)sl.hi_rows_send * stride : nullptr,
                  hi ? per_sub + (long long)sl.hi_rows_recv * stride : nullptr, hi ? n : 0, s);
}

void allgather_subs(Ctx& c, double* per_sub, long long stride, cudaStream_t s) {
  if (!c.tp) return;
  const Slab& sl = c.slab;
  std::vector<long long> off(sl.sub_off.size()), cnt(sl.sub_cnt.size());
  for (size_t r = 0; r < off.size(); ++r) {
    off[r] = sl.sub_off[r] * stride;
    cnt[r] = sl.sub_cnt[r] * stride;
  }
  c.tp->allgatherv(per_sub, off.data(), cnt.data(), s);
}

namespace {
// packed lower triangle of a b x b block (column j: rows j..b-1) <-> contiguous stage
__global__ void lower_pack_kernel(double* blk, int b, int ld, double* packed, int dir) {
  const long long tot = (long long)b * (b + 1) / 2;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < tot; q += (long long)gridDim.x * blockDim.x) {
    // column j with off(j) = j b - j (j - 1) / 2 <= q
    long long j = (long long)((2.0 * b + 1.0 - sqrt((2.0 * b + 1.0) * (2.0 * b + 1.0) - 8.0 * (double)q)) * 0.5);
    if (j < 0) j = 0;
    while (j > 0 && j * b - j * (j - 1) / 2 > q) --j;
    while ((j + 1) * b - (j + 1) * j / 2 <= q) ++j;
    const long long i = j + (q - (j * b - j * (j - 1) / 2));
    double* e = blk + i + j * ld;
    if (dir == 0) packed[q] = *e;
    else *e = packed[q];
  }
}
}  // namespace

void allgather_segments(Ctx& c, const std::vector<ExSeg>& segs, cudaStream_t s) {
  if (!c.tp || segs.empty()) return;
  const int world = c.tp->world, rank = c.tp->rank;
  std::vector<long long> len(segs.size()), off(world, 0), cnt(world, 0), pos(segs.size());
  for (size_t k = 0; k < segs.size(); ++k) {
    const ExSeg& g = segs[k];
    len[k] = g.kind ? (long long)g.b * (g.b + 1) / 2 : g.n;
    cnt[g.owner] += len[k];
  }
  for (int r = 1; r < world; ++r) off[r] = off[r - 1] + cnt[r - 1];
  const long long tot = off[world - 1] + cnt[world - 1];
  if (tot > c.dist.stage_len) {
    if (c.dist.stage) cudaFree(c.dist.stage);
    c.dist.stage = nullptr;
    BDDC_CUDA(cudaMalloc(&c.dist.stage, sizeof(double) * std::max(tot, 1LL)));
    c.dist.stage_len = tot;
  }
  double* st = c.dist.stage;
  std::vector<long long> fill(off);
  for (size_t k = 0; k < segs.size(); ++k) pos[k] = fill[segs[k].owner], fill[segs[k].owner] += len[k];
  auto move = [&](size_t k, int dir) {  // dir 0: segment -> stage, 1: stage -> segment
    const ExSeg& g = segs[k];
    if (len[k] == 0) return;
    if (g.kind == 0) {
      if (dir == 0) BDDC_CUDA(cudaMemcpyAsync(st + pos[k], g.ptr, sizeof(double) * g.n, cudaMemcpyDeviceToDevice, s));
      else BDDC_CUDA(cudaMemcpyAsync(g.ptr, st + pos[k], sizeof(double) * g.n, cudaMemcpyDeviceToDevice, s));
    } else {
      const int grid = (int)std::min<long long>((len[k] + 255) / 256, 148 * 8);
      lower_pack_kernel<<<grid, 256, 0, s>>>(g.ptr, g.b, g.ld, st + pos[k], dir);
      BDDC_LAUNCH_CHECK();
      BDDC_COUNT();
    }
  };
  for (size_t k = 0; k < segs.size(); ++k)
    if (segs[k].owner == rank) move(k, 0);
  c.tp->allgatherv(st, off.data(), cnt.data(), s);
  for (size_t k = 0; k < segs.size(); ++k)
    if (segs[k].owner != rank) move(k, 1);
}

void allreduce_scalars(Ctx& c, double* d, int n, cudaStream_t s) {
  if (c.tp) c.tp->allreduce_sum(d, n, s);
}

// ---------------------------------------------------------------------------------------
// NCCL transport
// ---------------------------------------------------------------------------------------
namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {
  static NcclApi a;
  static bool tried = false;
  if (!tried) {
    tried = true;
    // RTLD_NOLOAD first: reuse the NCCL the process already has (torch's), else load one
    a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!a.h) a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.h) a.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (a.h) {
#define BDDC_SYM(f) a.f = reinterpret_cast<decltype(a.f)>(dlsym(a.h, "nccl" #f))
      BDDC_SYM(GetUniqueId);
      BDDC_SYM(CommInitRank);
      BDDC_SYM(CommDestroy);
      BDDC_SYM(GroupStart);
      BDDC_SYM(GroupEnd);
      BDDC_SYM(Send);
      BDDC_SYM(Recv);
      BDDC_SYM(Broadcast);
      BDDC_SYM(AllReduce);
      BDDC_SYM(GetErrorString);
#undef BDDC_SYM
    }
  }
  if (!a.h || !a.CommInitRank || !a.AllReduce || !a.Send || !a.Recv || !a.Broadcast)
    throw std::runtime_error("NCCL (libnccl.so.2) not available");
  return a;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* m = nccl_api().GetErrorString ? nccl_api().GetErrorString(r) : "?";
    throw std::runtime_error(std::string("NCCL ") + what + ": " + m);
  }
}

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  int* d_int = nullptr;
  cudaStream_t st = nullptr;  // the failure-code reduction's own stream (not the legacy stream)
  NcclTransport(int r, int w, const void* id) {
    rank = r;
    world = w;
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    nccl_check(nccl_api().CommInitRank(&comm, w, uid, r), "CommInitRank");
    BDDC_CUDA(cudaMalloc(&d_int, sizeof(int)));
    BDDC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  }
  ~NcclTransport() override {
    if (comm) nccl_api().CommDestroy(comm);
    if (d_int) cudaFree(d_int);
    if (st) cudaStreamDestroy(st);
  }
  void neighbors(const double* lo_send, double* lo_recv, long long lo_n, const double* hi_send, double* hi_recv,
                 long long hi_n, cudaStream_t s) override {
    NcclApi& a = nccl_api();
    nccl_check(a.GroupStart(), "GroupStart");
    if (lo_n > 0) {
      nccl_check(a.Send(lo_send, lo_n, ncclDouble, rank - 1, comm, s), "Send");
      nccl_check(a.Recv(lo_recv, lo_n, ncclDouble, rank - 1, comm, s), "Recv");
    }
    if (hi_n > 0) {
      nccl_check(a.Send(hi_send, hi_n, ncclDouble, rank + 1, comm, s), "Send");
      nccl_check(a.Recv(hi_recv, hi_n, ncclDouble, rank + 1, comm, s), "Recv");
    }
    nccl_check(a.GroupEnd(), "GroupEnd");
  }
  void allgatherv(double* buf, const long long* off, const long long* cnt, cudaStream_t s) override {
    NcclApi& a = nccl_api();
    nccl_check(a.GroupStart(), "GroupStart");
    for (int r = 0; r < world; ++r)
      if (cnt[r] > 0) nccl_check(a.Broadcast(buf + off[r], buf + off[r], cnt[r], ncclDouble, r, comm, s), "Broadcast");
    nccl_check(a.GroupEnd(), "GroupEnd");
  }
  void allreduce_sum(double* buf, int n, cudaStream_t s) override {
    nccl_check(nccl_api().AllReduce(buf, buf, n, ncclDouble, ncclSum, comm, s), "AllReduce");
  }
  int allreduce_max_host(int v) override {
    BDDC_CUDA(cudaMemcpyAsync(d_int, &v, sizeof(int), cudaMemcpyHostToDevice, st));
    nccl_check(nccl_api().AllReduce(d_int, d_int, 1, ncclInt32, ncclMax, comm, st), "AllReduce");
    BDDC_CUDA(cudaMemcpyAsync(&v, d_int, sizeof(int), cudaMemcpyDeviceToHost, st));
    BDDC_CUDA(cudaStreamSynchronize(st));
    return v;
  }
};

// ---------------------------------------------------------------------------------------
// host-callback transport: ops 1 sendrecv(a -> peer, b <- peer), 2 broadcast(a, root = peer),
// 3 sum-allreduce(a), 4 max-allreduce(a); all on host buffers of n doubles
// ---------------------------------------------------------------------------------------
struct HostTransport : Transport {
  bddc_host_exchange_fn fn;
  void* user;
  std::vector<double> ha, hb;
  HostTransport(int r, int w, bddc_host_exchange_fn f, void* u) : fn(f), user(u) {
    rank = r;
    world = w;
  }
  void call(int op, double* a, double* b, long long n, int peer) {
    if (fn(user, op, a, b, n, peer) != 0) throw std::runtime_error("host exchange callback failed");
  }
  void pair(const double* send, double* recv, long long n, int peer, cudaStream_t s) {
    ha.resize(n);
    hb.resize(n);
    BDDC_CUDA(cudaMemcpyAsync(ha.data(), send, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    BDDC_CUDA(cudaStreamSynchronize(s));
    call(1, ha.data(), hb.data(), n, peer);
    BDDC_CUDA(cudaMemcpyAsync(recv, hb.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
    BDDC_CUDA(cudaStreamSynchronize(s));
  }
  void neighbors(const double* lo_send, double* lo_recv, long long lo_n, const double* hi_send, double* hi_recv,
                 long long hi_n, cudaStream_t s) override {
    // lower pair first: rank r pairs with r-1, then r+1 (a chain, no cycle)
    if (lo_n > 0) pair(lo_send, lo_recv, lo_n, rank - 1, s);
    if (hi_n > 0) pair(hi_send, hi_recv, hi_n, rank + 1, s);
  }
  void allgatherv(double* buf, const long long* off, const long long* cnt, cudaStream_t s) override {
    for (int r = 0; r < world; ++r) {
      if (cnt[r] <= 0) continue;
      ha.resize(cnt[r]);
      if (r == rank) {
        BDDC_CUDA(cudaMemcpyAsync(ha.data(), buf + off[r], cnt[r] * sizeof(double), cudaMemcpyDeviceToHost, s));
        BDDC_CUDA(cudaStreamSynchronize(s));
      }
      call(2, ha.data(), nullptr, cnt[r], r);
      if (r != rank) {
        BDDC_CUDA(cudaMemcpyAsync(buf + off[r], ha.data(), cnt[r] * sizeof(double), cudaMemcpyHostToDevice, s));
        BDDC_CUDA(cudaStreamSynchronize(s));
      }
    }
  }
  void allreduce_sum(double* buf, int n, cudaStream_t s) override {
    ha.resize(n);
    BDDC_CUDA(cudaMemcpyAsync(ha.data(), buf, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    BDDC_CUDA(cudaStreamSynchronize(s));
    call(3, ha.data(), nullptr, n, -1);
    BDDC_CUDA(cudaMemcpyAsync(buf, ha.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
    BDDC_CUDA(cudaStreamSynchronize(s));
  }
  int allreduce_max_host(int v) override {
    double d = v;
    call(4, &d, nullptr, 1, -1);
    return (int)d;
  }
};

}  // namespace

Transport* make_nccl_transport(int rank, int world, const void* unique_id) {
  return new NcclTransport(rank, world, unique_id);
}

Transport* make_host_transport(int rank, int world, bddc_host_exchange_fn fn, void* user) {
  return new HostTransport(rank, world, fn, user);
}

// One-rank self-test of the NCCL binding on the current device: every symbol the transport
// uses runs once on a communicator of world size 1 (sum-allreduce, max-allreduce, the grouped
// broadcast of allgatherv, and a grouped send/recv to self standing in for the neighbour
// exchange). Returns 0 when every result is the expected one.
int nccl_selftest() {
  ncclUniqueId id;
  NcclApi& a = nccl_api();
  if (!a.GetUniqueId || !a.GroupStart || !a.GroupEnd) throw std::runtime_error("NCCL symbols missing");
  nccl_check(a.GetUniqueId(&id), "GetUniqueId");
  NcclTransport t(0, 1, &id);
  cudaStream_t s;
  BDDC_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const int n = 1024;
  std::vector<double> h(2 * n);
  for (int i = 0; i < n; ++i) h[i] = 0.5 * i + 1.0;
  double* d = nullptr;
  BDDC_CUDA(cudaMalloc(&d, sizeof(double) * 2 * n));
  BDDC_CUDA(cudaMemcpyAsync(d, h.data(), sizeof(double) * 2 * n, cudaMemcpyHostToDevice, s));
  t.allreduce_sum(d, n, s);
  const long long off[1] = {0}, cnt[1] = {n};
  t.allgatherv(d, off, cnt, s);
  nccl_check(a.GroupStart(), "GroupStart");  // self send/recv: [0, n) -> [n, 2n)
  nccl_check(a.Send(d, n, ncclDouble, 0, t.comm, s), "Send");
  nccl_check(a.Recv(d + n, n, ncclDouble, 0, t.comm, s), "Recv");
  nccl_check(a.GroupEnd(), "GroupEnd");
  BDDC_CUDA(cudaMemcpyAsync(h.data(), d, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, s));
  BDDC_CUDA(cudaStreamSynchronize(s));
  const int mx = t.allreduce_max_host(7);
  cudaFree(d);
  cudaStreamDestroy(s);
  int bad = mx != 7;
  for (int i = 0; i < n; ++i) bad |= (h[i] != 0.5 * i + 1.0) || (h[n + i] != h[i]);
  return bad;
}

void nccl_unique_id(void* out) {
  ncclUniqueId id;
  NcclApi& a = nccl_api();
  if (!a.GetUniqueId) throw std::runtime_error("ncclGetUniqueId missing");
  nccl_check(a.GetUniqueId(&id), "GetUniqueId");
  memcpy(out, &id, sizeof(id));
}

}  // namespace bddc
