// Internal structures of the BDDC-SO device operator.
//
// Local layout of every subdomain (all subdomains of a uniform box partition share it):
//   * interior nodes: (b0-1)(b1-1)[(b2-1)] in x-fastest order, grouped in nblk "planes"
//     along the slowest axis, each plane padded to m_pad rows -> block-tridiagonal A_II;
//   * surface slots: the box-surface nodes in x-fastest order (= ascending global dof,
//     the reference's gamma_local order, bddc.py:429-433), padded to nG_pad; Dirichlet
//     surface nodes keep their slot as a decoupled identity row.
#pragma once
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "../../include/bddcso_b200.h"
#include "common.cuh"
#include "dense_f64.cuh"

namespace bddc {

// BDDC_HOST_TIMING=1: wall time of the host phases of bddc_setup on stderr (cold start)
struct HostTimer {
  bool on;
  std::chrono::steady_clock::time_point t;
  HostTimer() : on(getenv("BDDC_HOST_TIMING") != nullptr), t(std::chrono::steady_clock::now()) {}
  void mark(const char* what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "bddc_setup host: %-28s %9.3f s\n", what, std::chrono::duration<double>(n - t).count());
    t = n;
  }
};

struct Geometry {
  int dim;
  int cells[3];
  int subs[3];
  int blk[3];
  int nfree[3];  // free nodes per axis = cells - 1
  long long n;   // free dofs
  int nsub;
  int nloc_nodes;  // prod(blk+1)
  int m, m_pad, nblk, nI_pad;
  int nG, nG_pad;
  int nc_pad;
  int npe;      // nodes per element = 2^dim
  double K[64]; // reference element matrix (alpha = 1), row-major npe x npe
  // interior factor storage per subdomain: nblk packed lower-triangular inverses of the
  // diagonal Cholesky blocks (Tm = m_pad(m_pad+1)/2 doubles each), then the coupling
  // stencil to the previous plane, Bc[j][r][k] for the nbo structurally nonzero offsets
  int Tm;
  int nact[64];  // 2D: active interface columns (prefix) of R_j / H_j at plane j
  int nbo;
  // structurally nonzero neighbour offsets of the assembled stencil (excluding the node
  // itself): code = (dx+1) + 3 (dy+1) + 9 (dz+1); P1: 4 (2D) / 6 (3D), Q1: 8 / 26
  int nnb;
  int nb_code[26];
  int bo_dx[9], bo_dy[9];
  long long li_stride;
  // this rank's slab of the subdomain lattice (last axis); world = 1: everything
  int s_lo, s_hi;          // subdomains [s_lo, s_hi) (global ids)
  long long f_lo, f_hi;    // active free dofs: node rows from the lower to the upper cut line
  long long fo_lo, fo_hi;  // owned free dofs (a cut line belongs to the lower rank): dots
  int g_lo, g_hi;          // active interface dofs (indices into the ascending Gamma list)
};

// Rank-to-rank exchanges of the sharded operator (multigpu.cu). All pointers are device
// pointers on the operator's stream; implementations: NCCL (one rank per GPU) and a host
// callback transport (tests: ranks sharing one GPU, exchanges staged through the host).
struct Transport {
  int rank = 0, world = 1;
  virtual ~Transport() {}
  // send [lo_send, +lo_n) to rank-1 and receive [lo_recv, +lo_n) from it; same with rank+1
  virtual void neighbors(const double* lo_send, double* lo_recv, long long lo_n, const double* hi_send,
                         double* hi_recv, long long hi_n, cudaStream_t s) = 0;
  // in place: block r ([off[r], off[r] + cnt[r])) comes from rank r
  virtual void allgatherv(double* buf, const long long* off, const long long* cnt, cudaStream_t s) = 0;
  virtual void allreduce_sum(double* buf, int n, cudaStream_t s) = 0;
  // host value, max over ranks (error agreement)
  virtual int allreduce_max_host(int v) = 0;
};

// Distributed coarse factorization (sharded operators): the ND subtrees rooted
// at depth `depth` are dealt to the ranks (root i -> rank i % world); each rank factors and
// solves its subtrees only, the fronts above (`top`) are replicated. phase[nd]: 0 this
// rank's subtrees, 1 top, -1 another rank's subtree.
struct DistCoarse {
  bool on = false;
  int depth = 0;
  std::vector<int> phase;      // per node
  std::vector<int> roots;      // subtree roots (depth == depth), node order
  std::vector<int> root_owner;
  std::vector<int> sub_lo, sub_hi;  // per root: its subtree's node range [lo, hi] (postorder)
  double* stage = nullptr;     // exchange staging (device)
  long long stage_len = 0;
};

// one block of an exchange: `n` doubles at `ptr` (kind 0), or the lower triangle of the b x b
// block at `ptr` with leading dimension ld (kind 1, packed column by column); owner's copy wins
struct ExSeg {
  double* ptr;
  long long n;
  int owner, kind, b, ld;
};

// Slab bookkeeping derived from the geometry (host).
struct Slab {
  long long row_len = 0;  // free dofs per node row (2D) / plane (3D) of the last axis
  // halo rows of dof vectors (u1, p): offsets in free-dof index, -1 if no neighbour
  long long lo_send = -1, lo_recv = -1, hi_send = -1, hi_recv = -1;
  // boundary subdomain rows for the interface gather (w values, nG_pad per subdomain)
  int sub_row = 0;  // subdomains per lattice row (last axis)
  int lo_rows_send = -1, lo_rows_recv = -1, hi_rows_send = -1, hi_rows_recv = -1;  // first sub
  std::vector<long long> sub_off, sub_cnt;  // per rank: [s_lo, s_hi) in subdomains
};

// Decoded local node information (host-built tables, device copies).
struct LocalTables {
  int* node_code = nullptr;  // [nloc_nodes]: >=0 interior row (j*m_pad+r); <0: -(slot+1)
  int* slot_node = nullptr;  // [nG]
  int* irow_node = nullptr;  // [nI_pad] local node of interior row, -1 for pad rows
  int* irow_rel = nullptr;   // [nI_pad] free-dof offset of the row from the subdomain base, -1 pad
};

// Per-subdomain index data (device), shapes [nsub x nG_pad] / [nsub x nc_pad].
struct SubTables {
  int* slot_gamma = nullptr;    // global interface index, -1 (Dirichlet / pad)
  double* slot_w = nullptr;     // weight delta_i(xi)
  int* slot_con = nullptr;      // local constraint index or -1
  double* slot_coef = nullptr;  // constraint coefficient (1 or 1/|obj|)
  int* con_coarse = nullptr;    // coarse index (elimination order) or -1
};

// Device view of the multifrontal plan (POD: passed by value to kernels).
struct FrontDev {
  double* fronts = nullptr;
  double* upd = nullptr;        // per-node update vectors (solve)
  int* sep_start = nullptr;
  int* sep_size = nullptr;
  int* bnd_size = nullptr;
  int* ld = nullptr;
  long long* front_off = nullptr;
  long long* upd_off = nullptr;
  int* child_ptr = nullptr;
  int* child_list = nullptr;
  int* rmap = nullptr;          // per node: positions of its boundary dofs in the parent front
  int* rmap_ptr = nullptr;
  int* bnd_idx = nullptr;       // per node: boundary dofs (elimination order)
  int* bnd_ptr = nullptr;
  unsigned char* ualias = nullptr;  // per node: update columns on shared pool pages (front_vmm.cu)
  int* grp = nullptr;               // per node: panels per group of the dataflow factorization
};

// Coarse multifrontal plan (device data + host schedule).
struct FrontPlan {
  int n_coarse = 0;
  int nnodes = 0;
  int nlevels = 0;
  // host copies
  std::vector<int> level_ptr;     // nodes sorted by level: [level_ptr[l], level_ptr[l+1])
  std::vector<int> sep_start, sep_size, bnd_size, ld;
  std::vector<long long> front_off, upd_off;
  std::vector<int> child_ptr, child_list;  // CSR children per node
  std::vector<int> rmap_off;               // offset of node's rmap into its parent's front
  std::vector<int> bnd_ptr;                // CSR offsets into bnd_idx
  std::vector<int> parent;
  long long front_pool = 0, upd_pool = 0;
  int max_front = 0;
  bool alias = false;                  // update blocks aliased through the page pool (front_vmm.cu)
  long long alias_resident_bytes = 0;  // physical bytes behind the fronts when aliased
  std::vector<unsigned char> ualias;
  FrontDev d;  // device pointers (POD, passed to kernels)
  // CSR of the assembled coarse operator (elimination order, lower triangle) + maps
  long long nnz = 0;
  long long* csr_front_pos = nullptr;  // [nnz] offset into the front pool
  long long ncontrib = 0;
  long long* seg_ptr = nullptr;        // [nnz+1] contributions of each CSR entry
  int* contrib = nullptr;              // [ncontrib] index into local coarse blocks
  double* csr_val = nullptr;           // [nnz]
  int* csr_row_dev = nullptr;          // [nnz] elimination positions (device-built pattern only)
  int* csr_col_dev = nullptr;
  int* coarse_slots = nullptr;         // [n_coarse x W] (sub*nc_pad + k), -1 pad
  int W = 0;
  std::vector<int> level_list;         // nodes sorted by level (see level_ptr)
  std::vector<int> rmap_host;          // aligned with bnd_idx
  int* info = nullptr;                 // per node pivot failure (global coarse index)
};

// Coarse-solve plan: per level, GEMV tasks over the partitioned-inverse fronts. Every task
// carries its front's metadata (no dependent loads before its first front read).
struct CsTask {
  long long front_off;  // front base in the pool
  long long w_off;      // W21 = L21 X (fronts with s <= the W limit) offset in the scratch pool
  long long gat_base;   // node's offset into gat_ptr (child-update gathers per position)
  long long upd_off;    // node's update-vector offset
  int node, r0, c0;
  int s, f, ld, s0;     // separator size, front size, leading dimension, first coarse index
  int part;             // partial slot (np > 1)
  int red;              // global reduction index (arrival counter), -1 = none
  int np;               // tasks contributing to this task's reduction (1: write directly)
  int mode;             // forward: 0 = rows of [X; W21] (64 x cw), 1 = s <= 64 (256 rows x all s),
                        // 4 = L21 rows x y_s (64 x cw); backward: 2 = -L21^T x_bnd into t,
                        // 3 = rows of [X; W21]^T (y + t, -x_bnd); W21 fronts: ldw > 0
  int ldw;              // leading dimension of W21 (dataflow)
  int span;             // forward mode 0/4: columns per task; backward: rows per task (256 or 64)
  int rend;             // end of the task's rows (chunks never straddle the separator / boundary split)
};
// Dataflow coarse solve task: forward tasks (bottom-up) then backward tasks (top-down) in one
// queue; dependencies are node counters of finalized chunks (coarse.cu builds them).
struct SdTask {
  CsTask t;
  int dir;         // 0 forward, 1 backward
  int dep, tgt;    // wait until ctr[dep] >= tgt (dep < 0: none)
  int sig0, sig1, sig2;  // counters incremented when this task finalizes its chunk
};

struct CsRed {  // reduction over the partials of one row / column chunk
  int t0, p0, np;
};

struct LevelView {  // POD view of the gather maps for kernels
  const int* gat_ptr;
  const int* gat_src;
};

struct LevelSchedule {
  // solve: per level fwd / bwd GEMV tasks and reductions
  std::vector<CsTask*> fwd_t, bwd_t;
  std::vector<CsRed*> fwd_r, bwd_r;
  std::vector<int> n_fwd_t, n_bwd_t, n_fwd_r, n_bwd_r;
  double* partial = nullptr;
  double* ybuf = nullptr;     // forward-solve values of the separator rows (n)
  double* tbuf = nullptr;     // backward: -L21^T x_bnd of the separator rows (n; 0 where b = 0)
  int* red_cnt = nullptr;     // arrival counters of the fused reductions (self-resetting)
  int* gat_ptr = nullptr;     // per node front position -> sources in the update pool
  int* gat_src = nullptr;
  // dataflow solve (default): one task queue, node counters [3 N] + queue head + error flag
  SdTask* df_tasks = nullptr;
  int n_df = 0;
  std::vector<std::pair<SdTask*, int>> queues;  // 1 queue, or 3 (distributed coarse: coarse.cu)
  int n_tv = 0;               // of which v = T rho tasks of the apply's local Gamma phase (dir 2)
  int* df_ctr = nullptr;
  int n_ctr = 0;
};

// Optional per-phase CUDA-event timers (bench.py reads them for the roofline of the
// dominant kernel; disabled by default, zero cost when off).
struct PhaseTimers {
  bool on = false;
  struct Timer {
    std::vector<cudaEvent_t> ev;  // pairs
    size_t used = 0;
  };
  std::map<std::string, Timer> t;
  void begin(const char* name, cudaStream_t s) {
    if (!on) return;
    Timer& tm = t[name];
    if (tm.used + 2 > tm.ev.size()) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      tm.ev.push_back(a);
      tm.ev.push_back(b);
    }
    cudaEventRecord(tm.ev[tm.used], s);
  }
  void end(const char* name, cudaStream_t s) {
    if (!on) return;
    Timer& tm = t[name];
    cudaEventRecord(tm.ev[tm.used + 1], s);
    tm.used += 2;
  }
  void reset() {
    for (auto& kv : t) kv.second.used = 0;
  }
  // total ms and count (synchronizes on the events)
  double read(const std::string& name, long long* count) {
    auto it = t.find(name);
    if (it == t.end()) { *count = 0; return 0.0; }
    double tot = 0.0;
    for (size_t i = 0; i + 1 < it->second.used; i += 2) {
      float ms = 0.f;
      cudaEventSynchronize(it->second.ev[i + 1]);
      cudaEventElapsedTime(&ms, it->second.ev[i], it->second.ev[i + 1]);
      tot += ms;
    }
    *count = (long long)(it->second.used / 2);
    return tot;
  }
};

struct PhaseScope {
  PhaseTimers& pt;
  const char* name;
  cudaStream_t s;
  PhaseScope(PhaseTimers& p, const char* n, cudaStream_t st) : pt(p), name(n), s(st) { pt.begin(n, s); }
  ~PhaseScope() { pt.end(name, s); }
};

// T = L^{-T} L^{-1} - V V^T of the local setup, computed by the dataflow coarse factorization
// in the time its critical path leaves CTAs idle (local_setup sets it when it defers T)
struct LtArgs {
  const double* LI;  // zmode 0: [cnt][n][n] L^{-1}; zmode 1: Phi [cnt][n][nc] (stride sV)
  const double* V;   // zmode 0: [cnt][n][nc] V; zmode 1: W = Z C^T (sub at (sub - sub0))
  double* T;         // [nsub][n][n] (absolute subdomain index)
  long long sL, sV;
  int n, nc, sub0, on;
  int zmode;         // 1: T already holds Z = S_K^{-1}; the tasks do T -= Phi W^T
};

// The explicit interface operator T is stored as its lower triangle only (the apply's GEMV
// reads each stored entry once for both triangles) when nG_pad is in (256, 512]; smaller
// interfaces run v = T rho inside the coarse solve and keep T full.
inline bool t_lower_only(const Geometry& G) { return G.nG_pad > 256 && G.nG_pad <= 512; }

struct Ctx;
struct FrontVmm;
void front_vmm_release(Ctx& c);
void front_vmm_wait(Ctx& c);  // join the background mapping of the aliased fronts (rethrows)
bool front_alias_layout(Ctx& c);
void front_memset(Ctx& c, cudaStream_t s);
void front_pool_mark_clean(Ctx& c);  // the factorization completed: the alias pool is zero

struct Ctx {
  int device = 0;
  FrontVmm* vmm = nullptr;  // aliased coarse fronts (front_vmm.cu), released by free_all
  PhaseTimers prof;
  cudaStream_t stream = nullptr;
  // host-buffer solve (bddc_solve_host): alpha arrives in slabs of subdomain rows on the copy
  // stream; the first setup kernels of slab k wait on alpha_ev[k] (alpha_nslab = 0: resident)
  cudaStream_t copy_stream = nullptr;
  static constexpr int kMaxSlabs = 8;
  cudaEvent_t alpha_ev[kMaxSlabs] = {};
  cudaEvent_t b_ev = nullptr;
  int alpha_nslab = 0;
  int alpha_slab_sub[kMaxSlabs + 1] = {};
  Geometry geo{};
  int element = 0;
  int coarse_scaling = 0;  // 0 reference (Psi = Phi / s^2), 1 spec (Psi = Phi)
  bool setup_done = false;
  // inputs (device)
  double* alpha = nullptr;  // [ncells]
  LocalTables lt;
  SubTables st;
  int n_gamma = 0;
  long long* gamma_dof = nullptr;  // [n_gamma]
  int* gamma_slots = nullptr;      // [n_gamma x W]
  // factors (device)
  double* LI = nullptr;      // [nsub x li_stride] interior factor: packed L_j^{-1} + coupling stencil
  double* LS = nullptr;      // [nsub x nG_pad^2] Cholesky of S_K = S_Gamma + rho C^T C
  double* Phi = nullptr;     // [nsub x nG_pad x nc_pad] energy-minimal coarse basis on Gamma
  double* cscale = nullptr;  // [nsub] c_i (1/s_i^2 reference, 1 spec)
  double* diag_s = nullptr;  // [nsub] s_i = mean |diag A_i|
  double* Sloc = nullptr;    // [nsub x nc_pad^2] local coarse blocks (kept for assembly)
  int* info = nullptr;       // [nsub] interior (A_II) pivot failure per subdomain
  int* info_k = nullptr;     // [nsub] S_K pivot failure (underconstrained) per subdomain
  double* tinv = nullptr;    // diagonal-tile inverse scratch for batched TRSM / POTRF
  size_t tinv_doubles = 0;
  FrontPlan fp;
  LevelSchedule sched;
  // apply workspaces (device)
  double *v1 = nullptr, *v2 = nullptr;    // [n]
  double* rpg = nullptr;                  // [n_gamma]
  double *qloc = nullptr, *tloc = nullptr;  // [nsub x nc_pad]
  double *uloc = nullptr, *wloc = nullptr;  // [nsub x nG_pad]
  double *crhs = nullptr, *csol = nullptr;  // [n_coarse]
  // pcg workspaces
  double *r = nullptr, *z = nullptr, *p = nullptr, *Ap = nullptr;
  double *bbuf = nullptr, *xbuf = nullptr;  // host-facing PCG staging
  double* red = nullptr;     // reduction partials
  unsigned* redc = nullptr;  // arrival counter of the one-launch grid reductions (pcg.cu)
  double* scal = nullptr;    // device scalars
  double* h_scal = nullptr;  // pinned host mirror
  // multi-GPU: slab of this rank and the exchange transport (null: single rank)
  Slab slab;
  Transport* tp = nullptr;
  DistCoarse dist;
  // three-level hook (bddc_set_coarse_solver): replaces the exact coarse solve of the apply
  bddc_coarse_solver_fn coarse_cb = nullptr;
  void* coarse_cb_user = nullptr;
  bool coarse_lean = false;          // set up under the hook: no coarse plan, fronts or factor exist
  bool coarse_factor_valid = true;  // false after a re-setup under the hook skipped the factorization
  // timing of the last setup (ms) per phase
  float t_local_ms = 0, t_coarse_ms = 0, t_upload_ms = 0;
  std::vector<void*> allocations;

  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    BDDC_CUDA(cudaMalloc(&p, count * sizeof(T)));
    allocations.push_back(p);
    return (T*)p;
  }
  template <class T>
  T* upload(const T* host, size_t count) {
    T* d = alloc<T>(count);
    if (count && host) BDDC_CUDA(cudaMemcpyAsync(d, host, count * sizeof(T), cudaMemcpyHostToDevice, stream));
    return d;
  }
  void free_all() {
    front_vmm_release(*this);
    for (void* p : allocations) cudaFree(p);
    allocations.clear();
    if (dist.stage) cudaFree(dist.stage);
    dist = DistCoarse{};
  }
  LtArgs lt_defer{};      // local T deferred into the coarse factorization (on = 1)
  bool lt_fusable = false;  // the coarse factor program holds the T tasks
};

// local_setup.cu
void local_setup(Ctx& c, double* workspace, size_t ws_doubles);
size_t local_setup_workspace(const Geometry& g, int chunk);
// coarse_coop.cu: dataflow coarse factorization and its per-front scratch layout (inverse slots, Y partials, W21 = L21 X kept for the solve)
int coarse_w21_max_sep();
long long coarse_df_layout(const FrontPlan& fp, std::vector<long long>& inv, std::vector<long long>& Y,
                           std::vector<long long>& W, std::vector<int>& ldw);
// coarse.cu
void build_level_schedule(Ctx& c);
void coarse_assemble_and_factor(Ctx& c);
// v_i = T_i rho_i for the local subdomains, run by the dataflow coarse solve in the time its
// top-of-tree chain leaves CTAs idle (apply.cu passes it when the schedule holds those tasks)
struct TvArgs {
  const double* T;    // [nsub][n][n] explicit interface operators
  const double* rho;  // [nsub][n]
  double* v;          // [nsub][n]
  int n;
};
int coarse_solve_error(Ctx& c);  // 1 if the last coarse solve hit a dependency timeout (syncs)
// coarse assembly pattern built on the device from the con_coarse table (coarse_pattern.cu)
void device_coarse_pattern(Ctx& c, const int* con_coarse_host);
void coarse_solve(Ctx& c, const double* rhs, double* sol, cudaStream_t s, const TvArgs* tv = nullptr);
// apply.cu
void apply_bddc(Ctx& c, const double* r, double* z, cudaStream_t s);
void spmv(Ctx& c, const double* x, double* y, cudaStream_t s);
void harmonic_interior(Ctx& c, double* out, cudaStream_t s);
// pcg.cu
struct PcgResult {
  int iterations;
  int converged;
  int status;  // 0 ok, 5 not SPD operator
  double bad_value;
  int bad_kind;  // 0 <r,Br> (initial), 1 <p,Ap>, 2 <r,Br>
};
PcgResult pcg_solve(Ctx& c, const double* b, double* x, double tol, int max_iters, double* alphas,
                    double* betas, double* resid);
double dot(Ctx& c, const double* a, const double* b, long long n, cudaStream_t s);
// multigpu.cu
void slab_partition(Geometry& G, Slab& sl, int rank, int world, const long long* gamma_dof, int n_gamma);
void exchange_dof_halo(Ctx& c, double* v, cudaStream_t s);        // rows next to the cut lines
void exchange_boundary_rows(Ctx& c, double* per_sub, int stride, cudaStream_t s);  // nG_pad / sub
void allgather_subs(Ctx& c, double* per_sub, long long stride, cudaStream_t s);   // [nsub x stride]
// every rank gets every segment from its owner (staged in c.dist.stage, allgatherv)
void allgather_segments(Ctx& c, const std::vector<ExSeg>& segs, cudaStream_t s);
void allreduce_scalars(Ctx& c, double* d, int n, cudaStream_t s);
Transport* make_nccl_transport(int rank, int world, const void* unique_id);
Transport* make_host_transport(int rank, int world, bddc_host_exchange_fn fn, void* user);
void nccl_unique_id(void* out);
int nccl_selftest();  // world-1 run of every NCCL symbol the transport binds (0 = ok)

}  // namespace bddc
