/* C ABI of the B200-native BDDC-SO operator (libbddcso_b200.so).
 *
 * The reference (arXiv 2001.07289 package `bddcso`, pure Python) has no native FFI; its
 * operator interface for this path is the set of Python callables below. Each entry
 * point here replaces one of them; the ctypes binding that a maintainer adds on the
 * reference side is shown in INTEGRATION.md (and lives in paper_2001_07289_b200/_capi.py).
 *
 *   bddc_setup     <- build_bddc(system, pair, objects, recipe, weights)  bddc.py:393-523
 *   bddc_refactor  <- build_bddc numeric phase on resident inputs         bddc.py:419-511
 *   bddc_apply     <- BddcOperator.apply(r) / apply_bddc(bddc, r)          bddc.py:336-380, 526
 *   bddc_harmonic  <- harmonic_extension(bddc, g) / BddcOperator._harmonic bddc.py:382-390, 530
 *   bddc_spmv      <- SparseSym.matvec / `A @ v` in run()                   linalg.py:79, experiments.py:232
 *   bddc_pcg       <- pcg(lambda v: A @ v, op.apply, b, tol, max_iters)    krylov.py:31-92
 *   bddc_solve_host<- build_bddc numeric phase + pcg from host arrays, as   experiments.py:207, 231
 *                     run() calls them (uploads overlapped with the setup)
 *   bddc_dense_*   <- spd_factor / saddle_factor / their solves            linalg.py:117-212
 *
 * Streams: `stream` is a cudaStream_t (NULL = the legacy default stream); work is ordered
 * after earlier calls on the context and before later ones.
 * Conventions: plain pointers and sizes only; all vectors are float64 over free dofs in
 * the reference's numbering (mesh.py:97-102). Device pointers where marked; host arrays
 * in bddc_setup_desc are read during the call only. Return codes:
 *   0 ok, 1 invalid argument, 2 not SPD (NotSpdError), 3 underconstrained
 *   (UnderconstrainedError), 4 coarse matrix not SPD (NotSpdError), 5 operator / preconditioner
 *   not SPD inside PCG (NotSpdOperatorError), 6 CUDA error.
 * The message buffer `err` (may be NULL) receives the reference-style text.
 */
#ifndef BDDCSO_B200_H
#define BDDCSO_B200_H
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bddc_ctx bddc_ctx;

typedef struct {
  /* geometry (uniform box partition of the unit box, mesh.py:73 + partition.py:134) */
  int dim;
  int cells[3];
  int subs[3];
  int element;        /* 0 Q1, 1 P1-Kuhn (informational; elem_K carries the numbers) */
  int coarse_scaling; /* 0 "reference" (Psi = Phi / s_i^2), 1 "spec" (Psi = Phi) */
  const double* alpha;  /* [prod(cells)] coefficient per cell */
  const double* elem_K; /* [2^dim * 2^dim] row-major element matrix for alpha = 1 */
  /* local layout (identical for all subdomains) */
  int nloc_nodes, nG, nG_pad, m, m_pad, nblk, nI_pad, nc_pad;
  const int* node_code; /* [nloc_nodes] >=0 interior row, <0 -(slot+1) */
  const int* slot_node; /* [nG] */
  const int* irow_node; /* [nI_pad] -1 on padding rows */
  /* per-subdomain slots [nsub * nG_pad] and constraints [nsub * nc_pad] */
  const int* slot_gamma;
  const double* slot_w;
  const int* slot_con;
  const double* slot_coef;
  const int* con_coarse; /* coarse index in elimination order, -1 on padding */
  /* interface: global position -> free dof, owner slots (ascending subdomain) */
  int n_gamma;
  const long long* gamma_dof;
  const int* gamma_slots; /* [n_gamma * 2^dim] sub*nG_pad + slot, -1 pad */
  /* coarse problem */
  int n_coarse;
  const int* coarse_slots; /* [n_coarse * 2^dim] sub*nc_pad + k (elimination order), -1 pad */
  int nnodes;              /* nested-dissection fronts, children before parents */
  const int* node_sep_start;
  const int* node_sep_size;
  const int* node_level;
  const int* node_parent; /* -1 for roots */
  const int* bnd_ptr;     /* [nnodes + 1] */
  const int* bnd_idx;     /* boundary dofs of each front (elimination order, ascending) */
  const int* rmap;        /* aligned with bnd_idx: position in the parent front */
  /* coarse assembly pattern: contrib = NULL lets the setup build it on the device from
     con_coarse (coarse_pattern.cu); otherwise the host statement's arrays: */
  long long nnz;          /* lower-triangular coarse CSR entries */
  const int* csr_node;    /* front receiving each entry */
  const int* csr_row;     /* row position in that front */
  const int* csr_col;     /* column position in that front */
  const long long* seg_ptr; /* [nnz + 1] contributions per entry */
  long long ncontrib;
  const int* contrib; /* index into the local coarse blocks [nsub * nc_pad * nc_pad] */
} bddc_setup_desc;

typedef struct {
  int iterations;
  int converged;
  double bad_value; /* offending inner product when the return code is 5 */
  int bad_kind;     /* 0 <r,Br> initial, 1 <p,Ap>, 2 <r,Br> */
} bddc_pcg_report;

typedef struct {
  double t_upload_ms, t_local_ms, t_coarse_ms; /* last setup, CUDA events */
  long long n, n_gamma, n_coarse, nsub;
  long long factor_bytes, front_bytes, workspace_bytes;
  int nG_pad, nI_pad, m_pad, nblk, nc_pad, nlevels, max_front;
  int t_in_coarse_factor; /* the local T tiles run inside the coarse factorization */
  int tv_in_coarse_solve; /* the apply's v = T rho runs inside the coarse solve */
} bddc_stats;

int bddc_create(int device, bddc_ctx** out);
void bddc_destroy(bddc_ctx* ctx);
int bddc_setup(bddc_ctx* ctx, const bddc_setup_desc* desc, char* err, size_t errlen);
int bddc_refactor(bddc_ctx* ctx, const double* alpha_host, char* err, size_t errlen);
int bddc_apply(bddc_ctx* ctx, const double* r_dev, double* z_dev, void* stream);
int bddc_harmonic(bddc_ctx* ctx, const double* gamma_dev, double* out_dev, void* stream);
int bddc_spmv(bddc_ctx* ctx, const double* x_dev, double* y_dev, void* stream);
int bddc_pcg(bddc_ctx* ctx, const double* b_dev, double* x_dev, double tol, int max_iters,
             double* alphas, double* betas, double* resid, bddc_pcg_report* rep, char* err,
             size_t errlen);
/* setup (alpha_host, NULL: keep the resident alpha) + PCG with host buffers: replaces
   build_bddc's numeric phase + pcg (bddc.py:393-523, krylov.py:31-92) as experiments.py:207,231
   run() calls them; alpha / b uploads overlap the setup, x is downloaded at the end */
int bddc_solve_host(bddc_ctx* ctx, const double* alpha_host, const double* b_host, double* x_host,
                    double tol, int max_iters, double* alphas, double* betas, double* resid,
                    bddc_pcg_report* rep, char* err, size_t errlen);
int bddc_pcg_host(bddc_ctx* ctx, const double* b_host, double* x_host, double tol, int max_iters,
                  double* alphas, double* betas, double* resid, bddc_pcg_report* rep, char* err,
                  size_t errlen);
int bddc_get_stats(bddc_ctx* ctx, bddc_stats* out);
int bddc_sync(bddc_ctx* ctx);
/* synchronize the context stream and report an asynchronous failure of the last apply (a
   coarse-solve dependency timeout poisons its result): 0 ok, 6 + message */
int bddc_check(bddc_ctx* ctx, char* err, size_t errlen);
/* new interface weights slot_w [nsub * nG_pad] (host), e.g. coefficient weights recomputed for
   a new alpha before bddc_refactor (compute_weights, bddc.py:108-145) */
int bddc_update_weights(bddc_ctx* ctx, const double* slot_w_host, char* err, size_t errlen);
/* coarse solve S_0 x = rhs with the device factor (coarse_factor.solve, bddc.py:362-364);
   device vectors of n_coarse in the ELIMINATION order of the descriptor */
int bddc_coarse_solve(bddc_ctx* ctx, const double* rhs_dev, double* sol_dev, void* stream);
/* multilevel hook (the paper's outlook; not in the reference):
   when set, bddc_apply / bddc_pcg call fn in place of the exact coarse solve, with device
   vectors of n_coarse in elimination order and the stream the apply runs on (fn must order
   its work on that stream); fn returns 0 on success. NULL restores the direct solve.
   Single-rank operators only. While the hook is installed, bddc_refactor skips the coarse
   assembly and factorization (3D path; the 2D path keeps it: its local T tiles run inside that
   engine); after such a refactor and NULL, applies fail until the next bddc_refactor.
   Installed BEFORE bddc_setup, the setup builds no coarse plan at all (no front memory, no
   schedules, no factorization): such a context can only apply through the hook. */
typedef int (*bddc_coarse_solver_fn)(void* user, const double* rhs_dev, double* sol_dev, long long n_coarse,
                                     void* stream);
int bddc_set_coarse_solver(bddc_ctx* ctx, bddc_coarse_solver_fn fn, void* user);
/* device pointer to the coarse element matrices S_0i = Psi_i^T A_i Psi_i of the last setup
   (nsub blocks of nc_pad x nc_pad, symmetric; bddc.py:494-505 sums them into S_0); valid until
   the next setup / refactor / destroy. The stream is synchronized first. */
const double* bddc_coarse_elements(bddc_ctx* ctx, long long* count);
int bddc_kernel_launches_per_apply(bddc_ctx* ctx);
/* measurement: kernels launched by this library so far (process-wide); CUDA events on the
   context stream (slots 0..7); optional per-phase event timers ("apply.bt_solve",
   "apply.gamma1", "apply.coarse", "apply.gamma2", "setup.assemble", "setup.btchol",
   "setup.E", "setup.SG", "setup.SK", "setup.Phi", "setup.coarse", "pcg.spmv_dot") */
long long bddc_launch_count(void);
int bddc_event_record(bddc_ctx* ctx, int slot);
double bddc_event_elapsed_ms(bddc_ctx* ctx, int slot_a, int slot_b);
int bddc_profile(bddc_ctx* ctx, int enable);
double bddc_profile_read(bddc_ctx* ctx, const char* phase, long long* count);
/* diagnostics: copy an internal buffer ("LI", "LS", "Phi", "Sloc", "cscale", "diag_s",
   "csr_val", "fronts") to host; returns the element count (or -1) */
long long bddc_debug_copy(bddc_ctx* ctx, const char* name, double* host, long long capacity);
/* the same buffers, elements [offset, offset + count) (count 0 / host NULL: total length);
   backs the operator's lazy host views (.subdomains[i].coarse_basis, .coarse_matrix) */
long long bddc_read_buffer(bddc_ctx* ctx, const char* name, long long offset, long long count, double* host);

/* the coarse assembly pattern the setup built on the device (descriptor with contrib = NULL):
   lower CSR of S_0 in elimination order (row, col), seg_ptr [nnz + 1] and contrib (local block
   index per contribution, ascending subdomain inside an entry); all pointers NULL: returns nnz.
   -1 if the pattern came from the descriptor or a capacity is too small. */
long long bddc_coarse_csr(bddc_ctx* ctx, long long* row, long long* col, long long* seg_ptr, int* contrib,
                          long long cap_nnz, long long cap_contrib);

/* multi-GPU: one rank per GPU, each owning a slab of the subdomain lattice
   along the last axis (rows [r*R/world, (r+1)*R/world) of the R subdomain rows). Call one
   of the comm_init functions before bddc_setup; every rank passes the same global
   descriptor. Vectors stay global-length on every rank: inputs must be valid on the rank's
   active rows (both cut lines included), outputs are valid on its owned rows (a cut line
   belongs to the lower rank). The reference is single-process; this replaces its
   per-subdomain loop (bddc.py:419-511) across GPUs.
   host exchange callback ops (host buffers of n doubles):
     1 sendrecv(a -> peer, b <- peer), 2 broadcast(a from root = peer),
     3 sum-allreduce(a), 4 max-allreduce(a); return 0 on success */
typedef int (*bddc_host_exchange_fn)(void* user, int op, double* a, double* b, long long n, int peer);
int bddc_nccl_unique_id(void* out128);
int bddc_comm_init_nccl(bddc_ctx* ctx, int rank, int world, const void* unique_id128);
/* one-GPU self-test of the NCCL binding on `device`: a world-1 communicator runs every NCCL
   call the transport makes (allreduce sum / max, grouped broadcast, grouped send/recv to
   self). 0 ok, 2 wrong result, 6 NCCL / CUDA error (message on stderr) */
int bddc_nccl_selftest(int device);
int bddc_comm_init_host(bddc_ctx* ctx, int rank, int world, bddc_host_exchange_fn fn, void* user);
/* host-only: slab of `rank` for a dim/cells/subs box; out[10] = s_lo, s_hi, f_lo, f_hi, fo_lo,
   fo_hi, halo_lo_send, halo_lo_recv, halo_hi_send, halo_hi_recv (free-dof offsets, -1 none) */
int bddc_partition_info(int dim, const int* cells, const int* subs, int rank, int world, long long* out);

/* host-only symbolic work (no GPU): the lower CSR pattern of the coarse matrix in elimination
   order, its segmented contribution lists (ascending subdomain per entry, the reference's COO
   duplicate order, bddc.py:494-505) and the CSR -> front positions; output arrays hold up to the
   number of lower contributions (incl. the diagonal). Returns nnz, -1 if an entry falls outside
   its front. Same result as the numpy statement symbolic.coarse_csr. */
long long bddc_coarse_pattern(int nsub, const long long* sub_con_ptr, const long long* sub_con_ids,
                              const long long* iperm, long long n, int nc_pad, int nnodes,
                              const long long* sep_start, const long long* sep_size, const long long* bnd_ptr,
                              const long long* bnd_idx, long long* csr_row, long long* csr_col,
                              long long* csr_node, long long* frow, long long* fcol, long long* seg_ptr,
                              int* contrib);

/* device index sets: membership, interface objects and counting /
   cardinality weights of a partition pair on GPU `device`, bit-exact with the reference's
   host code it replaces:
     partition.py:117-131 (_node_membership), :75-83 (gamma dofs), :223-250 (classify_objects),
     bddc.py:108-145 (compute_weights, counting and cardinality modes).
   theta_hat [prod(cells)] subsubdomain per cell, parent [n_hat] subdomain per subsubdomain.
   Results are held by the handle: sizes by name ("n_free", "n_gamma", "n_gamma_hat",
   "n_obj", "width" = 2^dim), arrays copied out by name: "gamma_dofs", "gamma_hat_dofs",
   "signature", "sig_len", "owners", "owner_len", "dof_ptr", "dof_list", "dof_obj",
   "card_counts" (int64), "kind" (int8: 0 vertex, 1 edge, 2 face), "w_counting",
   "w_cardinality" (float64, [n_obj * width]); count must equal the array length. */
typedef struct bddc_index bddc_index;
int bddc_index_build(int device, int dim, const int* cells, const int* theta_hat, const int* parent,
                     int n_hat, bddc_index** out, char* err, size_t errlen);
long long bddc_index_size(const bddc_index* ix, const char* what);
int bddc_index_copy(const bddc_index* ix, const char* name, void* host, long long count);
void bddc_index_free(bddc_index* ix);

/* host-only symbolic analysis of the coarse problem (no GPU): the nested-dissection tree over
   the subdomain lattice, the elimination order, every front's boundary and the extend-add maps
   (the numpy statement symbolic.analyze is the checker). owners [n * W] -1 padded owner
   subdomains per coarse dof, sub_coords [nsub * dim], subs [dim], sub_con_ptr / sub_con_ids:
   subdomain -> coarse ids. Sizes by name ("nnodes", "nbnd", "n"); int64 arrays by name
   ("perm", "sep_start", "sep_size", "level", "parent", "bnd_ptr", "bnd_idx", "rmap"). */
typedef struct bddc_nd bddc_nd;
int bddc_nd_build(long long n, int W, const int* owners, int nsub, int dim, const int* sub_coords, const int* subs,
                  const long long* sub_con_ptr, const long long* sub_con_ids, bddc_nd** out, char* err, size_t errlen);
long long bddc_nd_size(const bddc_nd* h, const char* what);
int bddc_nd_copy(const bddc_nd* h, const char* name, long long* host, long long count);
void bddc_nd_free(bddc_nd* h);

/* device per-subdomain slot tables of the operator (layout.py; bddc.py:420-490): for every
   (subdomain, surface slot) the interface position, local constraint, coefficient and weight
   [nsub * nG_pad], and for every interface dof its owners' slots [n_gamma * 2^dim]; inputs
   are host arrays (slot coordinates of the local layout, per-free-dof constraint / coefficient
   / object, object owners and weights, subdomain -> ascending constraint lists). */
int bddc_layout_tables(int device, int dim, const int* cells, const int* subs, int nG, int nG_pad, int nloc,
                       const int* slot_coords, const int* slot_of_node, long long n_free, const int* gamma,
                       int n_gamma, const int* con_of, const double* coef_of, const int* dof_obj, int n_obj,
                       const int* owners, const double* obj_w, const long long* sub_con_ptr, const int* sub_con,
                       int* slot_gamma, int* slot_con, double* slot_coef, double* slot_w, int* gamma_slots,
                       char* err, size_t errlen);

/* dense FP64 batched kernels (column-major, even leading dimensions, device pointers) */
int bddc_dense_potrf(double* A, int n, int lda, long long stride, int count, int* info_host,
                     void* stream);
int bddc_dense_trsm(int kind, const double* L, int n, int ldl, long long sL, double* B,
                    int nother, int ldb, long long sB, int count, void* stream);
int bddc_dense_gemm(int transA, int transB, int M, int N, int K, double alpha, const double* A,
                    int lda, long long sA, const double* B, int ldb, long long sB, double beta,
                    double* C, int ldc, long long sC, int count, void* stream);

/* batched y = alpha A^T x + beta y: A column-major k x n (lda >= k even, 16-byte aligned, even
   stride, finite padding), x of k and y of n doubles per batch entry; equivalently the row-major n x k matrix
   times x. HBM-bound (each entry of A read once). Used by the three-level prototype's apply. */
int bddc_dense_gemv_t(int k, int n, double alpha, const double* A, int lda, long long sA, const double* x,
                      long long sx, double beta, double* y, long long sy, int count, void* stream);

#ifdef __cplusplus
}
#endif
#endif
