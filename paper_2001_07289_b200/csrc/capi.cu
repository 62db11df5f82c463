// C ABI (include/bddcso_b200.h): context, setup upload, numeric factorization, apply, PCG.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <climits>
#include <cstring>
#include <map>
#include <numeric>
#include <string>

#include "../../include/bddcso_b200.h"
#include "bddc_internal.cuh"
#include "stencil.cuh"

using namespace bddc;

namespace bddc {
void coop_release(const Ctx& c);
}

struct bddc_ctx {
  Ctx c;
  cudaEvent_t ev[8] = {};
  double* ws = nullptr;
  size_t ws_doubles = 0;
  double* alpha_host_shadow = nullptr;
  long long ncells = 0;
};

namespace {

constexpr int kNoFail = 0x7f7f7f7f;


void set_err(char* err, size_t len, const std::string& msg) {
  if (!err || len == 0) return;
  size_t n = std::min(len - 1, msg.size());
  memcpy(err, msg.data(), n);
  err[n] = 0;
}

struct ApiError {
  int code;
  std::string msg;
};

template <class F>
int guarded(char* err, size_t len, F&& f) {
  try {
    f();
    return 0;
  } catch (const ApiError& e) {
    set_err(err, len, e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_err(err, len, e.what());
    return 6;
  }
}

__global__ void scatter_gamma_kernel(int n_gamma, const long long* gdof, const double* g, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_gamma) out[gdof[i]] = g[i];
}

// numeric setup: local batched factorizations + coarse assembly / multifrontal factor
void numeric_setup(bddc_ctx* h) {
  Ctx& c = h->c;
  cudaStream_t s = c.stream;
  cudaEvent_t e0, e1, e2;
  BDDC_CUDA(cudaEventCreate(&e0));
  BDDC_CUDA(cudaEventCreate(&e1));
  BDDC_CUDA(cudaEventCreate(&e2));
  BDDC_CUDA(cudaMemsetAsync(c.info, 0x7f, sizeof(int) * c.geo.nsub, s));
  BDDC_CUDA(cudaMemsetAsync(c.info_k, 0x7f, sizeof(int) * c.geo.nsub, s));
  if (c.fp.nnodes) BDDC_CUDA(cudaMemsetAsync(c.fp.info, 0x7f, sizeof(int) * c.fp.nnodes, s));
  BDDC_CUDA(cudaEventRecord(e0, s));
  local_setup(c, h->ws, h->ws_doubles);
  // sharded: every rank assembles the replicated coarse matrix from all local blocks
  allgather_subs(c, c.Sloc, (long long)c.geo.nc_pad * c.geo.nc_pad, s);
  BDDC_CUDA(cudaEventRecord(e1, s));
  // three-level hook installed (bddc_set_coarse_solver): the exact coarse factor is never used,
  // so a re-setup skips its assembly and factorization, unless the local T tiles are
  // deferred into that engine (lt_defer: the 2D path)
  c.coarse_factor_valid = !(c.coarse_lean || (c.coarse_cb && !c.lt_defer.on && c.setup_done));
  if (c.coarse_factor_valid) coarse_assemble_and_factor(c);
  BDDC_CUDA(cudaEventRecord(e2, s));
  BDDC_CUDA(cudaEventSynchronize(e2));
  BDDC_CUDA(cudaEventElapsedTime(&c.t_local_ms, e0, e1));
  BDDC_CUDA(cudaEventElapsedTime(&c.t_coarse_ms, e1, e2));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  const int nsub = c.geo.nsub;
  std::vector<int> info(nsub), info_k(nsub);
  BDDC_CUDA(cudaMemcpy(info.data(), c.info, sizeof(int) * nsub, cudaMemcpyDeviceToHost));
  BDDC_CUDA(cudaMemcpy(info_k.data(), c.info_k, sizeof(int) * nsub, cudaMemcpyDeviceToHost));
  int bad_sub = -1, code = 0;
  for (int i = c.geo.s_lo; i < c.geo.s_hi && !code; ++i)
    if (info[i] != kNoFail) { code = 2; bad_sub = i; }
  for (int i = c.geo.s_lo; i < c.geo.s_hi && !code; ++i)
    if (info_k[i] != kNoFail) { code = 3; bad_sub = i; }
  // all ranks agree on failure (a rank that failed alone would leave the others waiting)
  const int any = c.tp ? c.tp->allreduce_max_host(code) : code;
  if (code == 2)
    throw ApiError{2, "subdomain " + std::to_string(bad_sub) +
                          ": matrix not SPD: nonpositive pivot at index " + std::to_string(info[bad_sub])};
  if (code == 3)
    throw ApiError{3, "subdomain " + std::to_string(bad_sub) +
                          ": saddle system numerically singular (floating subdomain "
                          "underconstrained or rank-deficient constraints)"};
  if (any) throw ApiError{any, "setup failed on another rank"};
  if (c.fp.nnodes) {
    std::vector<int> fi(c.fp.nnodes);
    BDDC_CUDA(cudaMemcpy(fi.data(), c.fp.info, sizeof(int) * c.fp.nnodes, cudaMemcpyDeviceToHost));
    int bad = kNoFail;
    for (int v : fi) bad = std::min(bad, v);
    // distributed coarse factorization: a pivot failure in another rank's subtree
    const int any4 = c.dist.on ? c.tp->allreduce_max_host(bad != kNoFail ? 4 : 0) : 0;
    if (bad != kNoFail)
      throw ApiError{4, "matrix not SPD: nonpositive pivot at index " + std::to_string(bad)};
    if (any4) throw ApiError{4, "matrix not SPD (coarse pivot failure on another rank)"};
  }
  c.setup_done = true;
}

// Distributed coarse factorization of a sharded operator: the ND subtrees
// rooted at the first depth with at least `world` nodes are dealt round-robin to the ranks;
// the fronts above are replicated. BDDC_DIST_COARSE=0 keeps the replicated coarse problem.
void build_dist(Ctx& c) {
  DistCoarse& D = c.dist;
  if (D.stage) cudaFree(D.stage);
  D = DistCoarse{};
  const FrontPlan& fp = c.fp;
  const char* e = getenv("BDDC_DIST_COARSE");
  if (!c.tp || c.tp->world < 2 || fp.nnodes == 0 || (e && atoi(e) == 0)) return;
  const int N = fp.nnodes, world = c.tp->world, rank = c.tp->rank;
  std::vector<int> depth(N, 0), size(N, 1);
  for (int v = N - 1; v >= 0; --v) depth[v] = fp.parent[v] < 0 ? 0 : depth[fp.parent[v]] + 1;  // parents after children
  for (int v = 0; v < N; ++v)
    if (fp.parent[v] >= 0) size[fp.parent[v]] += size[v];
  int maxd = 0;
  for (int v = 0; v < N; ++v) maxd = std::max(maxd, depth[v]);
  std::vector<int> cnt(maxd + 1, 0);
  for (int v = 0; v < N; ++v) cnt[depth[v]]++;
  int d = -1;
  for (int k = 0; k <= maxd && d < 0; ++k)
    if (cnt[k] >= world) d = k;
  if (d < 0) return;  // tree too small to deal out: replicated
  D.depth = d;
  D.phase.assign(N, 1);
  for (int v = 0; v < N; ++v)
    if (depth[v] == d) {
      const int owner = (int)D.roots.size() % world;
      D.roots.push_back(v);
      D.root_owner.push_back(owner);
      D.sub_lo.push_back(v - size[v] + 1);  // postorder: a subtree is a contiguous node range
      D.sub_hi.push_back(v);
      for (int u = v - size[v] + 1; u <= v; ++u) {
        int a = u;  // postorder check: u lies in v's subtree
        while (a >= 0 && a != v) a = fp.parent[a];
        if (a != v) throw CudaError("distributed coarse plan: subtree is not a contiguous node range");
        D.phase[u] = owner == rank ? 0 : -1;
      }
    }
  D.on = true;
}

void build_plan(Ctx& c, const bddc_setup_desc* d) {
  FrontPlan& fp = c.fp;
  fp.n_coarse = d->n_coarse;
  fp.nnodes = d->nnodes;
  fp.W = c.geo.npe;
  if (fp.n_coarse == 0) return;
  // three-level operators (hook installed before the setup): the coarse problem is never
  // factored, so no front memory, schedules or assembly pattern are built; the apply only
  // needs the gather of the coarse right-hand side
  c.coarse_lean = c.coarse_cb != nullptr;
  if (c.coarse_lean) {
    if (c.tp) throw ApiError{1, "three-level operators are single-rank"};
    fp.nnodes = 0;
    fp.nlevels = 0;
    c.lt_fusable = false;
    c.sched = LevelSchedule{};
    fp.coarse_slots = c.upload(d->coarse_slots, (size_t)d->n_coarse * fp.W);
    return;
  }
  const int N = fp.nnodes;
  fp.sep_start.assign(d->node_sep_start, d->node_sep_start + N);
  fp.sep_size.assign(d->node_sep_size, d->node_sep_size + N);
  fp.parent.assign(d->node_parent, d->node_parent + N);
  fp.bnd_ptr.assign(d->bnd_ptr, d->bnd_ptr + N + 1);
  fp.bnd_size.resize(N);
  fp.ld.resize(N);
  fp.front_off.resize(N);
  fp.upd_off.resize(N);
  int nlev = 0;
  for (int i = 0; i < N; ++i) nlev = std::max(nlev, d->node_level[i] + 1);
  fp.nlevels = nlev;
  long long off = 0, uoff = 0;
  fp.max_front = 0;
  for (int i = 0; i < N; ++i) {
    fp.bnd_size[i] = fp.bnd_ptr[i + 1] - fp.bnd_ptr[i];
    const int f = fp.sep_size[i] + fp.bnd_size[i];
    fp.ld[i] = (int)round_up(std::max(f, 2), 2);
    fp.front_off[i] = off;
    off += (long long)fp.ld[i] * f;
    off = round_up(off, 2);
    fp.upd_off[i] = uoff;
    uoff += fp.bnd_size[i];
    fp.max_front = std::max(fp.max_front, f);
  }
  fp.front_pool = off;
  fp.upd_pool = uoff;
  fp.alias = false;
  fp.ualias.assign(N, 0);
  // children CSR (in node order) and level lists
  fp.child_ptr.assign(N + 1, 0);
  for (int i = 0; i < N; ++i)
    if (fp.parent[i] >= 0) fp.child_ptr[fp.parent[i] + 1]++;
  for (int i = 0; i < N; ++i) fp.child_ptr[i + 1] += fp.child_ptr[i];
  fp.child_list.assign(fp.child_ptr[N], 0);
  {
    std::vector<int> fill(fp.child_ptr.begin(), fp.child_ptr.end() - 1);
    for (int i = 0; i < N; ++i)
      if (fp.parent[i] >= 0) fp.child_list[fill[fp.parent[i]]++] = i;
  }
  fp.level_ptr.assign(nlev + 1, 0);
  for (int i = 0; i < N; ++i) fp.level_ptr[d->node_level[i] + 1]++;
  for (int l = 0; l < nlev; ++l) fp.level_ptr[l + 1] += fp.level_ptr[l];
  fp.level_list.assign(N, 0);
  {
    std::vector<int> fill(fp.level_ptr.begin(), fp.level_ptr.end() - 1);
    for (int i = 0; i < N; ++i) fp.level_list[fill[d->node_level[i]]++] = i;
  }
  // device copies
  FrontDev& fd = fp.d;
  // multifrontal update blocks share pages when the resident fronts would not fit (front_vmm.cu)
  HostTimer ht0;
  ht0.mark("plan: tree tables");
  if (!front_alias_layout(c)) fd.fronts = c.alloc<double>(fp.front_pool);
  ht0.mark("plan: front memory / aliasing");
  fd.ualias = c.upload(fp.ualias.data(), N);
  fd.upd = c.alloc<double>(std::max<long long>(fp.upd_pool, 1));
  fd.sep_start = c.upload(fp.sep_start.data(), N);
  fd.sep_size = c.upload(fp.sep_size.data(), N);
  fd.bnd_size = c.upload(fp.bnd_size.data(), N);
  fd.ld = c.upload(fp.ld.data(), N);
  fd.front_off = c.upload(fp.front_off.data(), N);
  fd.upd_off = c.upload(fp.upd_off.data(), N);
  fd.child_ptr = c.upload(fp.child_ptr.data(), N + 1);
  fd.child_list = c.upload(fp.child_list.data(), fp.child_list.size());
  fd.bnd_ptr = c.upload(fp.bnd_ptr.data(), N + 1);
  fd.bnd_idx = c.upload(d->bnd_idx, fp.bnd_ptr[N]);
  fd.rmap = c.upload(d->rmap, fp.bnd_ptr[N]);
  fp.rmap_host.assign(d->rmap, d->rmap + fp.bnd_ptr[N]);
  fd.rmap_ptr = fd.bnd_ptr;
  fp.info = c.alloc<int>(N);
  if (!d->contrib) {
    // no host pattern in the descriptor: build it on the device (coarse_pattern.cu)
    if (!d->con_coarse) throw ApiError{1, "coarse pattern: con_coarse is required"};
    device_coarse_pattern(c, d->con_coarse);
    ht0.mark("plan: uploads + device CSR pattern");
  } else {
    // CSR -> front positions
    fp.nnz = d->nnz;
    std::vector<long long> pos(d->nnz);
    for (long long e = 0; e < d->nnz; ++e) {
      const int nd = d->csr_node[e];
      if (d->csr_col[e] >= fp.sep_size[nd]) throw ApiError{1, "coarse CSR entry outside its front's panel"};
      pos[e] = fp.front_off[nd] + d->csr_row[e] + (long long)d->csr_col[e] * fp.ld[nd];
    }
    ht0.mark("plan: uploads + CSR positions");
    fp.csr_front_pos = c.upload(pos.data(), pos.size());
    fp.seg_ptr = c.upload(d->seg_ptr, d->nnz + 1);
    fp.ncontrib = d->ncontrib;
    fp.contrib = c.upload(d->contrib, d->ncontrib);
    fp.csr_val = c.alloc<double>(d->nnz);
  }
  fp.coarse_slots = c.upload(d->coarse_slots, (size_t)d->n_coarse * fp.W);
  build_dist(c);
  HostTimer ht;
  build_level_schedule(c);
  ht.mark("solve + factor schedules");
}

void do_setup(bddc_ctx* h, const bddc_setup_desc* d) {
  Ctx& c = h->c;
  if (!d) throw ApiError{1, "null descriptor"};
  if (d->dim != 2 && d->dim != 3) throw ApiError{1, "dim must be 2 or 3"};
  c.free_all();
  c.setup_done = false;
  Geometry& G = c.geo;
  G = Geometry{};
  G.dim = d->dim;
  G.npe = 1 << d->dim;
  long long ncells = 1, n = 1;
  G.nsub = 1;
  for (int a = 0; a < 3; ++a) {
    const bool used = a < d->dim;
    G.cells[a] = used ? d->cells[a] : 1;
    G.subs[a] = used ? d->subs[a] : 1;
    if (used && (G.subs[a] < 1 || G.cells[a] % G.subs[a]))
      throw ApiError{1, "subdomains must divide the cell grid"};
    G.blk[a] = G.cells[a] / G.subs[a];
    G.nfree[a] = used ? G.cells[a] - 1 : 1;
    ncells *= G.cells[a];
    if (used) n *= G.nfree[a];
    G.nsub *= G.subs[a];
  }
  G.n = n;
  G.nloc_nodes = d->nloc_nodes;
  G.nG = d->nG;
  G.nG_pad = d->nG_pad;
  G.m = d->m;
  G.m_pad = d->m_pad;
  G.nblk = d->nblk;
  G.nI_pad = d->nI_pad;
  G.nc_pad = d->nc_pad;
  if (G.m_pad > 64 || G.m_pad % 8 || G.nI_pad != G.m_pad * G.nblk || G.nblk > 64)
    throw ApiError{1, "interior planes must fit one 64-row tile (m_pad <= 64, multiple of 8)"};
  if (G.nG_pad > 1024 || G.nG_pad % 8 || G.nc_pad > 1024 || G.nc_pad % 8)
    throw ApiError{1, "interface / constraint padding out of range"};
  for (int i = 0; i < G.npe * G.npe; ++i) G.K[i] = d->elem_K[i];
  // structurally nonzero neighbour offsets: some corner pair (s, t) of an element with
  // K[s][t] != 0 and t - s = the offset
  G.nnb = 0;
  for (int o = 0; o < 27; ++o) {
    const int dd[3] = {o % 3 - 1, (o / 3) % 3 - 1, o / 9 - 1};
    if (o == 13 || (G.dim == 2 && dd[2] != 0)) continue;
    bool used = false;
    for (int s0 = 0; s0 < G.npe && !used; ++s0)
      for (int t0 = 0; t0 < G.npe && !used; ++t0) {
        if (G.K[s0 * G.npe + t0] == 0.0) continue;
        bool match = true;
        for (int ax = 0; ax < G.dim; ++ax)
          if (((t0 >> ax) & 1) - ((s0 >> ax) & 1) != dd[ax]) match = false;
        used = match;
      }
    if (used) G.nb_code[G.nnb++] = o;
  }
  // structurally nonzero couplings from a plane to the previous one (last axis -1)
  G.nbo = 0;
  for (int dy = -1; dy <= 1; ++dy)
    for (int dx = -1; dx <= 1; ++dx) {
      if (G.dim == 2 && dy != 0) continue;
      bool used = false;
      for (int s0 = 0; s0 < G.npe && !used; ++s0)
        for (int t0 = 0; t0 < G.npe && !used; ++t0) {
          if (G.K[s0 * G.npe + t0] == 0.0) continue;
          int d[3];
          for (int ax = 0; ax < G.dim; ++ax) d[ax] = ((t0 >> ax) & 1) - ((s0 >> ax) & 1);
          const int last = d[G.dim - 1];
          const int ddx = d[0], ddy = G.dim == 3 ? d[1] : 0;
          if (last == -1 && ddx == dx && ddy == dy) used = true;
        }
      if (used) {
        G.bo_dx[G.nbo] = dx;
        G.bo_dy[G.nbo] = dy;
        G.nbo++;
      }
    }
  G.Tm = G.m_pad * (G.m_pad + 1) / 2;
  // active interface prefix per plane: the largest slot coupled to planes <= j (A_IG)
  {
    std::vector<int> code(d->node_code, d->node_code + G.nloc_nodes);
    std::vector<int> act(std::max(G.nblk, 1), 0);
    const int n0 = G.blk[0] + 1, n1 = G.blk[1] + 1;
    for (int node = 0; node < G.nloc_nodes; ++node) {
      if (code[node] < 0) continue;  // interior nodes only
      const int plane = code[node] / G.m_pad;
      const int a0 = node % n0, a1 = (node / n0) % n1, a2 = G.dim == 3 ? node / (n0 * n1) : 0;
      for (int o = 0; o < (G.dim == 3 ? 27 : 9); ++o) {
        const int b0 = a0 + o % 3 - 1, b1 = a1 + (o / 3) % 3 - 1, b2 = a2 + (G.dim == 3 ? o / 9 - 1 : 0);
        if (b0 < 0 || b1 < 0 || b2 < 0 || b0 >= n0 || b1 >= n1) continue;
        if (G.dim == 3 && b2 > G.blk[2]) continue;
        const int nb = b0 + n0 * (b1 + n1 * b2);
        if (code[nb] < 0) act[plane] = std::max(act[plane], -code[nb]);  // slot + 1
      }
    }
    for (int j = 1; j < G.nblk; ++j) act[j] = std::max(act[j], act[j - 1]);
    for (int j = 0; j < 64; ++j) {
      const int a = j < G.nblk ? act[j] : G.nG_pad;
      G.nact[j] = std::min<int>(G.nG_pad, (int)round_up(std::max(a, 8), 8));
    }
  }
  G.li_stride = round_up((long long)G.nblk * G.Tm + (long long)G.nblk * G.m_pad * G.nbo, 2);
  if (d->n_gamma && !d->gamma_dof) throw ApiError{1, "gamma_dof missing"};
  for (int g = 1; g < d->n_gamma; ++g)
    if (d->gamma_dof[g] <= d->gamma_dof[g - 1]) throw ApiError{1, "gamma_dof must be ascending"};
  try {
    slab_partition(G, c.slab, c.tp ? c.tp->rank : 0, c.tp ? c.tp->world : 1, d->gamma_dof, d->n_gamma);
  } catch (const std::runtime_error& e) {
    throw ApiError{1, e.what()};
  }
  c.element = d->element;
  c.coarse_scaling = d->coarse_scaling;
  h->ncells = ncells;

  cudaEvent_t e0, e1;
  BDDC_CUDA(cudaEventCreate(&e0));
  BDDC_CUDA(cudaEventCreate(&e1));
  BDDC_CUDA(cudaEventRecord(e0, c.stream));
  c.alpha = c.upload(d->alpha, ncells);
  c.lt.node_code = c.upload(d->node_code, G.nloc_nodes);
  c.lt.slot_node = c.upload(d->slot_node, G.nG);
  c.lt.irow_node = c.upload(d->irow_node, G.nI_pad);
  {
    // interior rows: free dof = base(subdomain) + rel (the numbering is affine inside a box)
    std::vector<int> rel(G.nI_pad, -1);
    const long long nf0 = G.nfree[0], nf1 = G.nfree[1];
    for (int rr = 0; rr < G.nI_pad; ++rr) {
      const int node = d->irow_node[rr];
      if (node < 0) continue;
      const int a0 = node % (G.blk[0] + 1), a1 = (node / (G.blk[0] + 1)) % (G.blk[1] + 1);
      const int a2 = G.dim == 3 ? node / ((G.blk[0] + 1) * (G.blk[1] + 1)) : 0;
      rel[rr] = (int)(a0 + nf0 * (a1 + nf1 * a2));
    }
    c.lt.irow_rel = c.upload(rel.data(), G.nI_pad);
  }
  const size_t ns = (size_t)G.nsub * G.nG_pad, nc = (size_t)G.nsub * G.nc_pad;
  c.st.slot_gamma = c.upload(d->slot_gamma, ns);
  c.st.slot_w = c.upload(d->slot_w, ns);
  c.st.slot_con = c.upload(d->slot_con, ns);
  c.st.slot_coef = c.upload(d->slot_coef, ns);
  c.st.con_coarse = c.upload(d->con_coarse, nc);
  c.n_gamma = d->n_gamma;
  c.gamma_dof = c.upload(d->gamma_dof, d->n_gamma);
  c.gamma_slots = c.upload(d->gamma_slots, (size_t)d->n_gamma * G.npe);
  HostTimer ht;
  build_plan(c, d);
  ht.mark("coarse plan (total)");
  BDDC_CUDA(cudaEventRecord(e1, c.stream));
  BDDC_CUDA(cudaEventSynchronize(e1));
  BDDC_CUDA(cudaEventElapsedTime(&c.t_upload_ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);

  // persistent factors (this rank's subdomains; the base pointers are shifted so kernels
  // index them with global subdomain ids) and workspaces
  const size_t nl = (size_t)(G.s_hi - G.s_lo);
  const long long lsS = (long long)G.nG_pad * G.nG_pad, phS = (long long)G.nG_pad * G.nc_pad;
  c.LI = c.alloc<double>(nl * G.li_stride) - (long long)G.s_lo * G.li_stride;
  c.LS = c.alloc<double>(nl * lsS) - (long long)G.s_lo * lsS;
  c.Phi = c.alloc<double>(nl * phS) - (long long)G.s_lo * phS;
  c.Sloc = c.alloc<double>((size_t)G.nsub * G.nc_pad * G.nc_pad);
  c.cscale = c.alloc<double>(G.nsub);
  c.diag_s = c.alloc<double>(G.nsub);
  c.info = c.alloc<int>(G.nsub);
  c.info_k = c.alloc<int>(G.nsub);
  c.v1 = c.alloc<double>(G.n);
  // u1 scratch: zero once; the interior solve only ever writes interior entries, so its
  // Gamma entries stay zero (no memset per apply)
  BDDC_CUDA(cudaMemsetAsync(c.v1, 0, sizeof(double) * G.n, c.stream));
  c.v2 = c.alloc<double>(G.n);
  c.rpg = c.alloc<double>(std::max(c.n_gamma, 1));
  c.qloc = c.alloc<double>(nc);
  c.tloc = c.alloc<double>(nc);
  c.uloc = c.alloc<double>(ns);
  c.wloc = c.alloc<double>(ns);
  c.crhs = c.alloc<double>(std::max(c.fp.n_coarse, 1));
  c.csol = c.alloc<double>(std::max(c.fp.n_coarse, 1));
  c.r = c.alloc<double>(G.n);
  c.z = c.alloc<double>(G.n);
  c.p = c.alloc<double>(G.n);
  c.Ap = c.alloc<double>(G.n);
  c.bbuf = c.alloc<double>(G.n);
  c.xbuf = c.alloc<double>(G.n);
  c.red = c.alloc<double>(4096);
  c.redc = c.alloc<unsigned>(1);
  BDDC_CUDA(cudaMemsetAsync(c.redc, 0, sizeof(unsigned), c.stream));
  c.scal = c.alloc<double>(16);
  BDDC_CUDA(cudaMemsetAsync(c.scal, 0, 16 * sizeof(double), c.stream));
  // setup workspace: all subdomains at once if it fits in ~60% of the free memory
  size_t free_b = 0, total_b = 0;
  BDDC_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const size_t per = local_setup_workspace(G, 1);
  size_t want = per * nl;
  // three-level operators leave the memory to the level 2 (chunks of 4,096 subdomains run the
  // local chain at the same rate: cfg3 is one such chunk)
  if (c.coarse_lean) want = std::min(want, per * (size_t)4096);
  size_t cap = (size_t)(0.6 * free_b) / sizeof(double);
  size_t use = std::min(want, std::max(cap - cap % per, per));
  h->ws = c.alloc<double>(use);
  h->ws_doubles = use;
  const int chunk = (int)std::min<size_t>(nl, use / per);
  c.tinv_doubles = std::max(trsm_scratch_doubles(G.nG_pad, chunk), trsm_scratch_doubles(G.nc_pad, chunk));
  c.tinv = c.alloc<double>(c.tinv_doubles);
  ht.mark("factor / workspace allocation");
  numeric_setup(h);
  ht.mark("first numeric setup");
}

// Run f on the caller's stream (NULL = legacy default stream), ordered after pending work
// of the context stream and before later context-stream work (shared workspaces).
template <class F>
void on_stream(bddc_ctx* h, void* stream, F&& f) {
  cudaStream_t s = (cudaStream_t)stream;
  if (s == h->c.stream) {
    f(s);
    return;
  }
  cudaEvent_t e;
  BDDC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  BDDC_CUDA(cudaEventRecord(e, h->c.stream));
  BDDC_CUDA(cudaStreamWaitEvent(s, e, 0));
  f(s);
  BDDC_CUDA(cudaEventRecord(e, s));
  BDDC_CUDA(cudaStreamWaitEvent(h->c.stream, e, 0));
  BDDC_CUDA(cudaEventDestroy(e));
}

}  // namespace

namespace bddc {
bool schur2d_supported(const Geometry& G);
}

extern "C" {

int bddc_create(int device, bddc_ctx** out) {
  if (!out) return 1;
  try {
    BDDC_CUDA(cudaSetDevice(device));
    auto* h = new bddc_ctx();
    h->c.device = device;
    BDDC_CUDA(cudaStreamCreateWithFlags(&h->c.stream, cudaStreamNonBlocking));
    BDDC_CUDA(cudaMallocHost(&h->c.h_scal, 16 * sizeof(double)));
    *out = h;
    return 0;
  } catch (const std::exception&) {
    return 6;
  }
}

void bddc_destroy(bddc_ctx* h) {
  if (!h) return;
  bddc::coop_release(h->c);
  cudaSetDevice(h->c.device);
  cudaStreamSynchronize(h->c.stream);
  h->c.free_all();
  delete h->c.tp;
  h->c.tp = nullptr;
  if (h->c.h_scal) cudaFreeHost(h->c.h_scal);
  if (h->c.copy_stream) {
    cudaStreamSynchronize(h->c.copy_stream);
    for (int k = 0; k < Ctx::kMaxSlabs; ++k) cudaEventDestroy(h->c.alpha_ev[k]);
    cudaEventDestroy(h->c.b_ev);
    cudaStreamDestroy(h->c.copy_stream);
  }
  cudaStreamDestroy(h->c.stream);
  delete h;
}

int bddc_setup(bddc_ctx* h, const bddc_setup_desc* d, char* err, size_t errlen) {
  if (!h) return 1;
  return guarded(err, errlen, [&] {
    BDDC_CUDA(cudaSetDevice(h->c.device));
    do_setup(h, d);
  });
}

int bddc_refactor(bddc_ctx* h, const double* alpha_host, char* err, size_t errlen) {
  if (!h) return 1;
  return guarded(err, errlen, [&] {
    if (!h->c.alpha) throw ApiError{1, "bddc_refactor before bddc_setup"};
    BDDC_CUDA(cudaSetDevice(h->c.device));
    if (alpha_host)
      BDDC_CUDA(cudaMemcpyAsync(h->c.alpha, alpha_host, sizeof(double) * h->ncells,
                                cudaMemcpyHostToDevice, h->c.stream));
    numeric_setup(h);
  });
}

int bddc_apply(bddc_ctx* h, const double* r, double* z, void* stream) {
  if (!h || !h->c.setup_done) return 1;
  return guarded(nullptr, 0, [&] {
    BDDC_CUDA(cudaSetDevice(h->c.device));
    on_stream(h, stream, [&](cudaStream_t s) { apply_bddc(h->c, r, z, s); });
  });
}

int bddc_harmonic(bddc_ctx* h, const double* g, double* out, void* stream) {
  if (!h || !h->c.setup_done) return 1;
  return guarded(nullptr, 0, [&] {
    BDDC_CUDA(cudaSetDevice(h->c.device));
    on_stream(h, stream, [&](cudaStream_t s) {
    Ctx& c = h->c;
    const Geometry& G = c.geo;
    // out_Gamma = g; out_I = A_II^{-1} (0 - A g_ext)_I
    BDDC_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * G.n, s));
    BDDC_CUDA(cudaMemsetAsync(c.v1, 0, sizeof(double) * G.n, s));
    const int ng = G.g_hi - G.g_lo;
    if (ng > 0)
      { scatter_gamma_kernel<<<ceil_div(ng, 256), 256, 0, s>>>(ng, c.gamma_dof + G.g_lo, g + G.g_lo, out); BDDC_COUNT(); }
    BDDC_LAUNCH_CHECK();
    harmonic_interior(c, out, s);
    });
  });
}

int bddc_spmv(bddc_ctx* h, const double* x, double* y, void* stream) {
  if (!h || !h->c.alpha) return 1;
  return guarded(nullptr, 0, [&] {
    BDDC_CUDA(cudaSetDevice(h->c.device));
    on_stream(h, stream, [&](cudaStream_t s) { spmv(h->c, x, y, s); });
  });
}

int bddc_pcg(bddc_ctx* h, const double* b, double* x, double tol, int max_iters, double* alphas,
             double* betas, double* resid, bddc_pcg_report* rep, char* err, size_t errlen) {
  if (!h || !h->c.setup_done) return 1;
  return guarded(err, errlen, [&] {
    BDDC_CUDA(cudaSetDevice(h->c.device));
    PcgResult r = pcg_solve(h->c, b, x, tol, max_iters, alphas, betas, resid);
    if (rep) {
      rep->iterations = r.iterations;
      rep->converged = r.converged;
      rep->bad_value = r.bad_value;
      rep->bad_kind = r.bad_kind;
    }
    if (r.status == 5) {
      char buf[128];
      snprintf(buf, sizeof buf, r.bad_kind == 1 ? "operator not SPD: <p, Ap> = %.17g"
                                                : "preconditioner not SPD: <r, Br> = %.17g",
               r.bad_value);
      throw ApiError{5, buf};
    }
  });
}

// Setup + solve with host buffers (the reference's build_bddc + pcg pair, experiments.py
// run): alpha goes up in slabs of subdomain rows on a copy stream and the 2D elimination of
// slab k starts when its cells land; b goes up behind alpha while the setup runs; x comes
// back after the solve. Same results as bddc_refactor + bddc_pcg_host.
int bddc_solve_host(bddc_ctx* h, const double* alpha_host, const double* b_host, double* x_host,
                    double tol, int max_iters, double* alphas, double* betas, double* resid,
                    bddc_pcg_report* rep, char* err, size_t errlen) {
  if (!h || !h->c.setup_done) return 1;
  int code = guarded(err, errlen, [&] {
    Ctx& c = h->c;
    const Geometry& G = c.geo;
    BDDC_CUDA(cudaSetDevice(c.device));
    if (!c.copy_stream) {
      BDDC_CUDA(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
      for (int k = 0; k < Ctx::kMaxSlabs; ++k)
        BDDC_CUDA(cudaEventCreateWithFlags(&c.alpha_ev[k], cudaEventDisableTiming));
      BDDC_CUDA(cudaEventCreateWithFlags(&c.b_ev, cudaEventDisableTiming));
    }
    // the copy stream must not overwrite buffers the context stream may still read
    BDDC_CUDA(cudaEventRecord(c.b_ev, c.stream));
    BDDC_CUDA(cudaStreamWaitEvent(c.copy_stream, c.b_ev, 0));
    const int last = G.dim - 1;
    const int rows = G.subs[last];
    long long row_cells = G.blk[last];
    for (int a = 0; a < last; ++a) row_cells *= G.cells[a];
    const int per_row = G.nsub / rows;
    c.alpha_nslab = 0;
    if (alpha_host) {
      const bool slab = bddc::schur2d_supported(G) && G.nblk > 0;
      // two halves: the second lands while the first is eliminated (measured on cfg2: 4 or 8
      // slabs, or a smaller first slab, cost more in kernel tails than they hide)
      const double first = 0.5;
      const int ns = slab && rows >= 4 && first > 0.0 && first < 1.0 ? 2 : 1;
      const int rsplit = std::max(1, (int)(rows * first));
      for (int k = 0; k < ns; ++k) {
        const int r0 = k == 0 ? 0 : rsplit, r1 = (ns == 1 || k == 1) ? rows : rsplit;
        const long long c0 = r0 * row_cells, c1 = r1 * row_cells;
        BDDC_CUDA(cudaMemcpyAsync(c.alpha + c0, alpha_host + c0, sizeof(double) * (c1 - c0),
                                  cudaMemcpyHostToDevice, c.copy_stream));
        BDDC_CUDA(cudaEventRecord(c.alpha_ev[k], c.copy_stream));
        c.alpha_slab_sub[k] = r0 * per_row;
        c.alpha_slab_sub[k + 1] = r1 * per_row;
      }
      if (slab) c.alpha_nslab = ns;
      else BDDC_CUDA(cudaStreamWaitEvent(c.stream, c.alpha_ev[0], 0));
    }
    BDDC_CUDA(cudaMemcpyAsync(c.bbuf + G.f_lo, b_host + G.f_lo, sizeof(double) * (G.f_hi - G.f_lo),
                              cudaMemcpyHostToDevice, c.copy_stream));
    BDDC_CUDA(cudaEventRecord(c.b_ev, c.copy_stream));
    try {
      numeric_setup(h);
    } catch (...) {
      c.alpha_nslab = 0;
      BDDC_CUDA(cudaStreamWaitEvent(c.stream, c.b_ev, 0));
      throw;
    }
    c.alpha_nslab = 0;
    BDDC_CUDA(cudaStreamWaitEvent(c.stream, c.b_ev, 0));
  });
  if (code) return code;
  code = bddc_pcg(h, h->c.bbuf, h->c.xbuf, tol, max_iters, alphas, betas, resid, rep, err, errlen);
  int code2 = guarded(err, code ? 0 : errlen, [&] {
    const Geometry& G = h->c.geo;
    BDDC_CUDA(cudaMemcpyAsync(x_host + G.fo_lo, h->c.xbuf + G.fo_lo, sizeof(double) * (G.fo_hi - G.fo_lo),
                              cudaMemcpyDeviceToHost, h->c.stream));
    BDDC_CUDA(cudaStreamSynchronize(h->c.stream));
  });
  return code ? code : code2;
}

int bddc_pcg_host(bddc_ctx* h, const double* b_host, double* x_host, double tol, int max_iters,
                  double* alphas, double* betas, double* resid, bddc_pcg_report* rep, char* err,
                  size_t errlen) {
  if (!h || !h->c.setup_done) return 1;
  int code = 0;
  code = guarded(err, errlen, [&] {
    Ctx& c = h->c;
    BDDC_CUDA(cudaSetDevice(c.device));
    const Geometry& G = c.geo;  // sharded: this rank's active rows in, owned rows out
    BDDC_CUDA(cudaMemcpyAsync(c.bbuf + G.f_lo, b_host + G.f_lo, sizeof(double) * (G.f_hi - G.f_lo),
                              cudaMemcpyHostToDevice, c.stream));
  });
  if (code) return code;
  code = bddc_pcg(h, h->c.bbuf, h->c.xbuf, tol, max_iters, alphas, betas, resid, rep, err, errlen);
  int code2 = guarded(err, code ? 0 : errlen, [&] {
    const Geometry& G = h->c.geo;
    BDDC_CUDA(cudaMemcpyAsync(x_host + G.fo_lo, h->c.xbuf + G.fo_lo, sizeof(double) * (G.fo_hi - G.fo_lo),
                              cudaMemcpyDeviceToHost, h->c.stream));
    BDDC_CUDA(cudaStreamSynchronize(h->c.stream));
  });
  return code ? code : code2;
}

int bddc_nccl_unique_id(void* out) {
  if (!out) return 1;
  try {
    nccl_unique_id(out);
    return 0;
  } catch (const std::exception&) {
    return 6;
  }
}

int bddc_nccl_selftest(int device) {
  try {
    BDDC_CUDA(cudaSetDevice(device));
    return nccl_selftest() ? 2 : 0;
  } catch (const std::exception& e) {
    fprintf(stderr, "bddc_nccl_selftest: %s\n", e.what());
    return 6;
  }
}

int bddc_comm_init_nccl(bddc_ctx* h, int rank, int world, const void* id) {
  if (!h || !id || world < 1 || rank < 0 || rank >= world) return 1;
  try {
    BDDC_CUDA(cudaSetDevice(h->c.device));
    delete h->c.tp;
    h->c.tp = world > 1 ? make_nccl_transport(rank, world, id) : nullptr;
    return 0;
  } catch (const std::exception&) {
    return 6;
  }
}

int bddc_comm_init_host(bddc_ctx* h, int rank, int world, bddc_host_exchange_fn fn, void* user) {
  if (!h || !fn || world < 1 || rank < 0 || rank >= world) return 1;
  delete h->c.tp;
  h->c.tp = world > 1 ? make_host_transport(rank, world, fn, user) : nullptr;
  return 0;
}

int bddc_partition_info(int dim, const int* cells, const int* subs, int rank, int world, long long* out) {
  if ((dim != 2 && dim != 3) || !cells || !subs || !out) return 1;
  Geometry G{};
  G.dim = dim;
  G.n = 1;
  G.nsub = 1;
  for (int a = 0; a < 3; ++a) {
    const bool used = a < dim;
    G.cells[a] = used ? cells[a] : 1;
    G.subs[a] = used ? subs[a] : 1;
    if (used && (G.subs[a] < 1 || G.cells[a] % G.subs[a])) return 1;
    G.blk[a] = G.cells[a] / G.subs[a];
    G.nfree[a] = used ? G.cells[a] - 1 : 1;
    if (used) G.n *= G.nfree[a];
    G.nsub *= G.subs[a];
  }
  Slab sl;
  try {
    slab_partition(G, sl, rank, world, nullptr, 0);
  } catch (const std::exception&) {
    return 1;
  }
  const long long v[10] = {G.s_lo, G.s_hi, G.f_lo, G.f_hi, G.fo_lo, G.fo_hi,
                           sl.lo_send, sl.lo_recv, sl.hi_send, sl.hi_recv};
  for (int i = 0; i < 10; ++i) out[i] = v[i];
  return 0;
}

int bddc_get_stats(bddc_ctx* h, bddc_stats* o) {
  if (!h || !o) return 1;
  const Ctx& c = h->c;
  const Geometry& G = c.geo;
  memset(o, 0, sizeof(*o));
  o->t_upload_ms = c.t_upload_ms;
  o->t_local_ms = c.t_local_ms;
  o->t_coarse_ms = c.t_coarse_ms;
  o->n = G.n;
  o->n_gamma = c.n_gamma;
  o->n_coarse = c.fp.n_coarse;
  o->nsub = G.nsub;
  o->factor_bytes = 8LL * (G.s_hi - G.s_lo) * (G.li_stride + (long long)G.nG_pad * G.nG_pad +
                                    (long long)G.nG_pad * G.nc_pad);
  o->front_bytes = c.fp.alias ? c.fp.alias_resident_bytes : 8LL * c.fp.front_pool;
  o->workspace_bytes = 8LL * h->ws_doubles;
  o->nG_pad = G.nG_pad;
  o->nI_pad = G.nI_pad;
  o->m_pad = G.m_pad;
  o->nblk = G.nblk;
  o->nc_pad = G.nc_pad;
  o->nlevels = c.fp.nlevels;
  o->max_front = c.fp.max_front;
  o->t_in_coarse_factor = c.lt_defer.on;
  o->tv_in_coarse_solve = c.fp.n_coarse > 0 && c.sched.n_tv > 0;
  return 0;
}

int bddc_update_weights(bddc_ctx* h, const double* slot_w_host, char* err, size_t errlen) {
  if (!h || !slot_w_host) return 1;
  return guarded(err, errlen, [&] {
    Ctx& c = h->c;
    if (!c.st.slot_w) throw ApiError{1, "bddc_update_weights before bddc_setup"};
    BDDC_CUDA(cudaSetDevice(c.device));
    BDDC_CUDA(cudaMemcpyAsync(c.st.slot_w, slot_w_host, sizeof(double) * (size_t)c.geo.nsub * c.geo.nG_pad,
                              cudaMemcpyHostToDevice, c.stream));
    BDDC_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int bddc_coarse_solve(bddc_ctx* h, const double* rhs, double* sol, void* stream) {
  if (!h || !h->c.setup_done || !rhs || !sol) return 1;
  return guarded(nullptr, 0, [&] {
    BDDC_CUDA(cudaSetDevice(h->c.device));
    if (h->c.fp.n_coarse == 0) return;
    if (!h->c.coarse_factor_valid) throw ApiError{1, "the exact coarse factor was skipped under the coarse-solver hook"};
    on_stream(h, stream, [&](cudaStream_t s) { coarse_solve(h->c, rhs, sol, s, nullptr); });
  });
}

int bddc_set_coarse_solver(bddc_ctx* h, bddc_coarse_solver_fn fn, void* user) {
  if (!h) return 1;
  if (fn && h->c.tp) return 1;  // single-rank operators only
  h->c.coarse_cb = fn;
  h->c.coarse_cb_user = user;
  return 0;
}

int bddc_check(bddc_ctx* h, char* err, size_t errlen) {
  if (!h) return 1;
  return guarded(err, errlen, [&] {
    BDDC_CUDA(cudaSetDevice(h->c.device));
    BDDC_CUDA(cudaStreamSynchronize(h->c.stream));
    if (h->c.setup_done && coarse_solve_error(h->c))
      throw CudaError("coarse dataflow solve: dependency wait timed out (the last apply's result is invalid)");
  });
}

int bddc_sync(bddc_ctx* h) {
  if (!h) return 1;
  if (cudaSetDevice(h->c.device) != cudaSuccess) return 6;
  return cudaStreamSynchronize(h->c.stream) == cudaSuccess ? 0 : 6;
}

int bddc_kernel_launches_per_apply(bddc_ctx* h) {
  if (!h) return -1;
  const Ctx& c = h->c;
  // bt_solve x2, gamma residual, local_gamma1, coarse gather, fwd/bwd per level,
  // local_gamma2, gamma gather, residual (memsets are copy-engine ops, not kernels)
  int n = 2 + 1 + 1 + 1 + 1 + 1;
  if (c.fp.n_coarse) n += 1 + 2 * c.fp.nlevels;
  return n;
}

long long bddc_launch_count(void) { return launch_counter().load(); }

int bddc_event_record(bddc_ctx* h, int slot) {
  if (!h || slot < 0 || slot >= 8) return 1;
  if (cudaSetDevice(h->c.device) != cudaSuccess) return 6;
  if (!h->ev[slot] && cudaEventCreate(&h->ev[slot]) != cudaSuccess) return 6;
  return cudaEventRecord(h->ev[slot], h->c.stream) == cudaSuccess ? 0 : 6;
}

double bddc_event_elapsed_ms(bddc_ctx* h, int a, int b) {
  if (!h || a < 0 || b < 0 || a >= 8 || b >= 8 || !h->ev[a] || !h->ev[b]) return -1.0;
  float ms = 0.f;
  if (cudaEventSynchronize(h->ev[b]) != cudaSuccess) return -1.0;
  if (cudaEventElapsedTime(&ms, h->ev[a], h->ev[b]) != cudaSuccess) return -1.0;
  return ms;
}

int bddc_profile(bddc_ctx* h, int enable) {
  if (!h) return 1;
  if (cudaSetDevice(h->c.device) != cudaSuccess) return 6;
  cudaStreamSynchronize(h->c.stream);
  h->c.prof.on = enable != 0;
  h->c.prof.reset();
  return 0;
}

double bddc_profile_read(bddc_ctx* h, const char* phase, long long* count) {
  if (!h || !phase || !count) return -1.0;
  return h->c.prof.read(phase, count);
}

long long bddc_coarse_csr(bddc_ctx* h, long long* row, long long* col, long long* seg_ptr, int* contrib,
                          long long cap_nnz, long long cap_contrib) {
  if (!h) return -1;
  const FrontPlan& fp = h->c.fp;
  if (!fp.csr_row_dev && fp.nnz > 0) return -1;  // pattern came from the host descriptor
  if (!row && !col && !seg_ptr && !contrib) return fp.nnz;
  if (cap_nnz < fp.nnz || (contrib && cap_contrib < fp.ncontrib)) return -1;
  if (cudaSetDevice(h->c.device) != cudaSuccess || cudaStreamSynchronize(h->c.stream) != cudaSuccess) return -1;
  std::vector<int> tmp(std::max(fp.nnz, 1LL));
  for (int which = 0; which < 2; ++which) {
    long long* out = which ? col : row;
    if (!out) continue;
    if (fp.nnz && cudaMemcpy(tmp.data(), which ? fp.csr_col_dev : fp.csr_row_dev, sizeof(int) * fp.nnz,
                             cudaMemcpyDeviceToHost) != cudaSuccess)
      return -1;
    for (long long e = 0; e < fp.nnz; ++e) out[e] = tmp[e];
  }
  if (seg_ptr && cudaMemcpy(seg_ptr, fp.seg_ptr, sizeof(long long) * (fp.nnz + 1), cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  if (contrib && fp.ncontrib &&
      cudaMemcpy(contrib, fp.contrib, sizeof(int) * fp.ncontrib, cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  return fp.nnz;
}

const double* bddc_coarse_elements(bddc_ctx* h, long long* count) {
  if (!h || !h->c.setup_done || !h->c.Sloc) return nullptr;
  if (cudaSetDevice(h->c.device) != cudaSuccess || cudaStreamSynchronize(h->c.stream) != cudaSuccess) return nullptr;
  if (count) *count = (long long)h->c.geo.nsub * h->c.geo.nc_pad * h->c.geo.nc_pad;
  return h->c.Sloc;
}

long long bddc_read_buffer(bddc_ctx* h, const char* name, long long offset, long long count, double* host) {
  if (!h || !name) return -1;
  const Ctx& c = h->c;
  const Geometry& G = c.geo;
  const double* src = nullptr;
  long long n = 0;
  std::string nm(name);
  const long long nl = G.s_hi - G.s_lo;  // this rank's subdomains (all of them when unsharded)
  if (nm == "LI") { src = c.LI + (long long)G.s_lo * G.li_stride; n = nl * G.li_stride; }
  else if (nm == "LS") { src = c.LS + (long long)G.s_lo * G.nG_pad * G.nG_pad; n = nl * G.nG_pad * G.nG_pad; }
  else if (nm == "Phi") { src = c.Phi + (long long)G.s_lo * G.nG_pad * G.nc_pad; n = nl * G.nG_pad * G.nc_pad; }
  else if (nm == "Sloc") { src = c.Sloc; n = (long long)G.nsub * G.nc_pad * G.nc_pad; }
  else if (nm == "cscale") { src = c.cscale; n = G.nsub; }
  else if (nm == "diag_s") { src = c.diag_s; n = G.nsub; }
  else if (nm == "csr_val") { src = c.fp.csr_val; n = c.fp.nnz; }
  else if (nm == "fronts") { src = c.fp.d.fronts; n = c.fp.front_pool; }
  else if (nm == "v1") { src = c.v1; n = G.n; }
  else if (nm == "v2") { src = c.v2; n = G.n; }
  else if (nm == "rpg") { src = c.rpg; n = c.n_gamma; }
  else if (nm == "qloc") { src = c.qloc; n = (long long)G.nsub * G.nc_pad; }
  else if (nm == "tloc") { src = c.tloc; n = (long long)G.nsub * G.nc_pad; }
  else if (nm == "uloc") { src = c.uloc; n = (long long)G.nsub * G.nG_pad; }
  else if (nm == "wloc") { src = c.wloc; n = (long long)G.nsub * G.nG_pad; }
  else if (nm == "crhs") { src = c.crhs; n = c.fp.n_coarse; }
  else if (nm == "csol") { src = c.csol; n = c.fp.n_coarse; }
  else return -1;
  if (!host) return n;
  if (!src || offset < 0 || count < 0 || offset + count > n) return -1;
  if (cudaSetDevice(c.device) != cudaSuccess) return -1;
  if (cudaStreamSynchronize(c.stream) != cudaSuccess) return -1;
  if (count && cudaMemcpy(host, src + offset, sizeof(double) * count, cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  return count;
}

long long bddc_debug_copy(bddc_ctx* h, const char* name, double* host, long long cap) {
  const long long n = bddc_read_buffer(h, name, 0, 0, nullptr);
  if (n < 0 || !host) return n;
  if (cap < n) return -1;
  return bddc_read_buffer(h, name, 0, n, host);
}

int bddc_dense_potrf(double* A, int n, int lda, long long stride, int count, int* info_host,
                     void* stream) {
  if (!A || n <= 0 || lda < n || (lda & 1) || count <= 0) return 1;
  return guarded(nullptr, 0, [&] {
    cudaStream_t s = (cudaStream_t)stream;
    int* info = nullptr;
    BDDC_CUDA(cudaMallocAsync((void**)&info, sizeof(int) * count, s));
    BDDC_CUDA(cudaMemsetAsync(info, 0x7f, sizeof(int) * count, s));
    double* scr = nullptr;
    BDDC_CUDA(cudaMallocAsync((void**)&scr, sizeof(double) * trsm_scratch_doubles(n, count), s));
    potrf_batched(BMat{A, stride, lda}, n, n, count, info, scr, s);
    BDDC_CUDA(cudaFreeAsync(scr, s));
    if (info_host) {
      BDDC_CUDA(cudaMemcpyAsync(info_host, info, sizeof(int) * count, cudaMemcpyDeviceToHost, s));
      BDDC_CUDA(cudaStreamSynchronize(s));
      for (int i = 0; i < count; ++i)
        if (info_host[i] == kNoFail) info_host[i] = -1;
    }
    BDDC_CUDA(cudaFreeAsync(info, s));
  });
}

int bddc_dense_trsm(int kind, const double* L, int n, int ldl, long long sL, double* B, int nother,
                    int ldb, long long sB, int count, void* stream) {
  if (!L || !B || kind < 0 || kind > 3 || (ldl & 1) || (ldb & 1)) return 1;
  return guarded(nullptr, 0, [&] {
    cudaStream_t s = (cudaStream_t)stream;
    double* scr = nullptr;
    BDDC_CUDA(cudaMallocAsync((void**)&scr, sizeof(double) * trsm_scratch_doubles(n, count), s));
    trsm_batched((TrsmKind)kind, BMat{(double*)L, sL, ldl}, n, BMat{B, sB, ldb}, nother, count,
                 scr, s);
    BDDC_CUDA(cudaFreeAsync(scr, s));
  });
}

int bddc_dense_gemm(int tA, int tB, int M, int N, int K, double alpha, const double* A, int lda,
                    long long sA, const double* B, int ldb, long long sB, double beta, double* C,
                    int ldc, long long sC, int count, void* stream) {
  if ((lda & 1) || (ldb & 1)) return 1;
  return guarded(nullptr, 0, [&] {
    gemm_batched(tA != 0, tB != 0, M, N, K, alpha, BMat{(double*)A, sA, lda}, BMat{(double*)B, sB, ldb},
                 beta, BMat{C, sC, ldc}, count, (cudaStream_t)stream);
  });
}

int bddc_dense_gemv_t(int k, int n, double alpha, const double* A, int lda, long long sA, const double* x,
                      long long sx, double beta, double* y, long long sy, int count, void* stream) {
  if (!A || !x || !y || k <= 0 || lda < k || (lda & 1) || (sA & 1) || ((uintptr_t)A & 15)) return 1;
  return guarded(nullptr, 0, [&] {
    gemv_t_batched(k, n, alpha, BMat{(double*)A, sA, lda}, x, sx, beta, y, sy, count, (cudaStream_t)stream);
  });
}

}  // extern "C"
