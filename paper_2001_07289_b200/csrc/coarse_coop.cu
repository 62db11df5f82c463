// Coarse engine: the multifrontal factorization and the coarse solve, each ONE persistent
// cooperative launch running a host-built dataflow program.
//
// The factorization program is a list of tile tasks in a topological order; CTAs pull
// tasks from a global queue, wait (bounded) on dependency counters and signal counters
// when done, so the tree's levels overlap and no grid barrier is needed. Per front:
//   EA(k)     extend-add child k's update block into the front
//   per 64-column panel p:
//     PT      potrf + trtri of the diagonal tile (inverse -> scratch)
//     TS      L21 tile <- A21 tile inv^T
//     SY      trailing tile -= L21 L21^T (lower)            [+ lookahead PT of panel p+1]
//     X1/X2   X = L11^{-1} accumulated left-looking (X written in place over L11)
//   W         W21 = L21 X  (kept in the scratch pool for the solve)
// so each front ends as the partitioned inverse [X; W21] (both coarse triangular solves are
// GEMVs). The solve program: forward GEMV tasks bottom-up, backward top-down, chunk partials
// reduced in fixed order (deterministic).
#include <cooperative_groups.h>

#include <algorithm>
#include <queue>
#include <cstdio>
#include <cstdlib>
#include <map>

#include "bddc_internal.cuh"
#include "tile_ops.cuh"

namespace cg = cooperative_groups;

namespace bddc {

#ifndef BDDC_X1_CHUNK
#define BDDC_X1_CHUNK 256
#endif
// K width of one X1 task (a multiple of 64): X[p, c] = -inv_pp sum_m L[p, m] X[m, c] is split
// into chunks of kX1Chunk / 64 panel blocks m; X2 sums the chunk partials (fewer, longer X1
// tasks: 4x less partial traffic than one panel block per task)
constexpr int kX1Chunk = BDDC_X1_CHUNK;
constexpr int kX1Blocks = kX1Chunk / 64;
constexpr int kCoopStages = 2;  // cp.async depth of the engine GEMM tiles: 41 KB smem leaves more L1 (measured: 3 stages are slower)

enum CoopType : int {
  CT_EA = 0, CT_PT = 1, CT_TS = 2, CT_X1 = 3, CT_SY = 4, CT_X2 = 5, CT_W = 6,
  CT_LT = 7,   // local interface operator tile T_IJ of subdomain (node) (the local setup's T)
  CT_SYG = 8,  // trailing tile -= L21 L21^T over a whole panel group (K = kGroup panels)
  CT_NTYPES = 9
};

// Panels are factored in groups of kGroup (a 512-column block column): inside the group the
// right-looking SY updates touch only the block column (K = 64); the trailing matrix beyond
// it is updated ONCE per group (CT_SYG, K = kGroup * 64 = 512), so every trailing tile is read
// and written 1/kGroup as often as with per-panel updates (the DRAM traffic of the large
// fronts), and the program has half the tasks of groups of 4 (cfg5: 1.31 -> 1.25 s, measured
// with groups of 4 / 6 / 8 / 12 / 16: tools/gpu_ab_group.sh, tools/gpu_ab2.sh).
#ifndef BDDC_KGROUP
#define BDDC_KGROUP 8
#endif
constexpr int kGroup = BDDC_KGROUP;
#ifndef BDDC_SYG_BK
#define BDDC_SYG_BK 16
#endif
constexpr int kSygBK = BDDC_SYG_BK;  // K-slice width of the group trailing-update tiles
// group size per front (FrontDev::grp): kGroup panels, or 1 (the per-panel right-looking update
// with lookahead) for separators below BDDC_GROUP_MIN_SEP (default 0: groups everywhere; 512 /
// 1024 / 2048 / 4096 measured slower on cfg5, cfg3 and cfg2 L=h, 4% faster on cfg2 L=4h only:
// tools/gpu_ab8.sh)
__host__ __device__ __forceinline__ int group_k0(int g, int G) { return g * G * kTile; }
__host__ __device__ __forceinline__ int group_k1(int g, int G, int s) { return min(s, (g + 1) * G * kTile); }

struct CoopTask {
  int type, node, a, b, arg;
};

struct CoopScratch {  // per-node offsets (doubles) into the scratch pool
  long long* inv;  // one 64 x 64 inverse slot per panel
  long long* Y;    // X1 partials, two sets by panel parity
  long long* W;    // W21 = L21 X (read by the solve)
  int* ldw;        // leading dimension of W (even)
};

struct CoopProgram {
  CoopScratch sc;
  double* pool;
  LtArgs lt;  // deferred local T (CT_LT tasks; no-ops when lt.on == 0)
};

// Dataflow program: tasks in a topological order, each with up to kDeps dependencies
// (counter >= target) and up to 3 counters it increments when done.
constexpr int kDeps = 6;
constexpr int kSigs = 6;
// 4 CTAs per SM (128 registers) since the GEMM tile epilogue handles the C tile in two halves
// (56 bytes of spills; the one-pass epilogue spilled 680): cfg5 coarse 1220.8 -> 1186.8 ms, cfg3
// 30.07 -> 30.40 ms against 3 CTAs on the same box (profiles/r02/ab/ctas4)
#ifndef BDDC_DF_CTAS
#define BDDC_DF_CTAS 4
#endif
constexpr int kDfCtasPerSm = BDDC_DF_CTAS;  // dataflow: no grid barrier, more CTAs hide tile latency
struct DfTask {
  CoopTask t;
  int dep[kDeps], tgt[kDeps];
  int sig[kSigs];
  unsigned char sw[8];  // increment of each signal (a group update counts as its panels)
};

namespace {

using namespace tile;

__device__ void run_task(const CoopTask& t, const FrontDev& fd, const CoopProgram& pg, int* info,
                         double* smem) {
  if (t.type == CT_LT) {  // (node = subdomain) T_IJ = sum_{k >= I} LI_kI^T LI_kJ - V_I V_J^T
    const LtArgs& a = pg.lt;
    if (!a.on) return;
    const int sub = t.node, m0 = t.a * kTile, n0 = t.b * kTile;
    double* T = a.T + (long long)sub * a.sL;
    if (a.zmode) {  // T = Z - Phi W^T (lower tile, mirrored)
      const double* Ph = a.LI + (long long)(sub - a.sub0) * a.sV;
      const double* W = a.V + (long long)(sub - a.sub0) * a.sV;
      gemm_tile<false, true, kCoopStages>(Ph, a.n, W, a.n, T, a.n, a.n, a.n, a.nc, m0, n0, -1.0, 1.0, true, smem, 0,
                                          -1, true);
      return;
    }
    const double* LI = a.LI + (long long)(sub - a.sub0) * a.sL;
    gemm_tile<true, false, kCoopStages>(LI, a.n, LI, a.n, T, a.n, a.n, a.n, a.n, m0, n0, 1.0, 0.0, true, smem,
                                        m0, -1, a.nc == 0);
    if (a.nc > 0) {
      __syncthreads();
      const double* V = a.V + (long long)(sub - a.sub0) * a.sV;
      gemm_tile<false, true, kCoopStages>(V, a.n, V, a.n, T, a.n, a.n, a.n, a.nc, m0, n0, -1.0, 1.0, true, smem, 0,
                                          -1, true);
    }
    return;
  }
  const int node = t.node;
  const int s = fd.sep_size[node], f = s + fd.bnd_size[node], ld = fd.ld[node];
  double* F = fd.fronts + fd.front_off[node];
  double* X = F;  // L11^{-1} is written in place over L11
  const int ldx = ld;
  switch (t.type) {
    case CT_EA: {  // child #arg of node, columns [a, a + b) of its lower update block
      const int c0 = fd.child_ptr[node];
      const int ch = fd.child_list[c0 + t.arg];
      const int bc = fd.bnd_size[ch], sc = fd.sep_size[ch], lc = fd.ld[ch];
      double* U = fd.fronts + fd.front_off[ch] + sc + (long long)sc * lc;
      const bool zu = fd.ualias[ch];  // pool pages: leave them zero for the next block
      const int* rm = fd.rmap + fd.rmap_ptr[ch];
      // columns [a, a + cb) in batches of 16; thread owns rows i = a + tid + 128 m, loads
      // rm[i] once and issues 16 independent read-modify-writes per batch
      const int je = min(bc, t.a + t.b);
      for (int j0 = t.a; j0 < je; j0 += 16) {
        long long cof[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) cof[c] = j0 + c < je ? (long long)rm[j0 + c] * ld : 0;
        for (int i = j0 + threadIdx.x; i < bc; i += blockDim.x) {
          const long long r = rm[i];
          BDDC_CHECK(r >= 0 && r < f);  // extend-add row inside the parent front
          double u[16], fv[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const bool ok = j0 + c < je && i >= j0 + c;
            u[c] = ok ? __ldcg(U + i + (long long)(j0 + c) * lc) : 0.0;
            fv[c] = ok ? __ldcg(F + r + cof[c]) : 0.0;
          }
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (j0 + c < je && i >= j0 + c) {
              F[r + cof[c]] = fv[c] + u[c];
              if (zu) U[i + (long long)(j0 + c) * lc] = 0.0;
            }
        }
      }
      break;
    }
    case CT_PT: {  // factor + invert diagonal tile of panel arg
      const int k = t.arg * kTile, nb = min(kTile, s - k);
      double* inv = pg.pool + pg.sc.inv[node] + t.arg * kTileInvStride;
      const int bad = potrf_trtri_tile(F + k + (long long)k * ld, ld, nb, inv, smem);
      if (threadIdx.x == 0 && bad >= 0) atomicMin(info + node, fd.sep_start[node] + k + bad);
      break;
    }
    case CT_TS: {  // rows (k+nb) + 64a.. of the panel: L21 <- A21 inv^T (in place)
      const int k = t.arg * kTile, nb = min(kTile, s - k), rest = f - k - nb;
      double* A21 = F + (k + nb) + (long long)k * ld;
      const double* inv = pg.pool + pg.sc.inv[node] + t.arg * kTileInvStride;
      gemm_tile<false, true, kCoopStages>(A21, ld, inv, kTile, A21, ld, rest, nb, nb, t.a * kTile, 0, 1.0, 0.0,
                             false, smem);
      break;
    }
    case CT_X1: {  // Y_q[:, c] = L[k.., c*64 + kq ..) X[.., c]  over K chunk q (c = a, q = b)
      const int k = t.arg * kTile, nb = min(kTile, s - k), c = t.a * kTile;
      const int kq0 = c + t.b * kX1Chunk, kq1 = min(k, kq0 + kX1Chunk);
      // dataflow: panel-parity Y partial sets (X1 of panel p + 2 waits for X2 of panel p)
      const long long ysz = (long long)kTile * s * ((s + kX1Chunk - 1) / kX1Chunk);
      double* Y = pg.pool + pg.sc.Y[node] + (t.arg & 1) * ysz + (long long)t.b * kTile * s;
      gemm_tile<false, false, kCoopStages>(F + k + (long long)kq0 * ld, ld, X + kq0 + (long long)c * ldx, ldx,
                              Y + (long long)c * kTile, kTile, nb, min(kTile, k - c), kq1 - kq0, 0, 0,
                              1.0, 0.0, false, smem);
      break;
    }
    case CT_SY: {  // tile (a, b) of the panel's trailing matrix INSIDE its group's block column
      // (columns < group_k1) -= L21 L21^T; tile (0,0) + lookahead:
      const int k = t.arg * kTile, nb = min(kTile, s - k), rest = f - k - nb;
      const int G = fd.grp[node];
      const int ncols = group_k1(t.arg / G, G, s) - (k + nb);
      double* L21 = F + (k + nb) + (long long)k * ld;
      double* A22 = F + (k + nb) + (long long)(k + nb) * ld;
      gemm_tile<false, true, kCoopStages>(L21, ld, L21, ld, A22, ld, rest, ncols, nb, t.a * kTile, t.b * kTile,
                             -1.0, 1.0, true, smem);
      if (t.a == 0 && t.b == 0 && k + nb < s) {  // factor the next panel's diagonal tile now
        __syncthreads();
        const int k1 = k + nb, nb1 = min(kTile, s - k1);
        double* inv1 = pg.pool + pg.sc.inv[node] + (t.arg + 1) * kTileInvStride;
        const int bad = potrf_trtri_tile(F + k1 + (long long)k1 * ld, ld, nb1, inv1, smem);
        if (threadIdx.x == 0 && bad >= 0) atomicMin(info + node, fd.sep_start[node] + k1 + bad);
      }
      break;
    }
    case CT_SYG: {  // trailing tile (a, b) beyond group arg's block column -= L21 L21^T, K = group
      const int G = fd.grp[node];
      const int k0 = group_k0(t.arg, G), k1 = group_k1(t.arg, G, s), rest = f - k1;
      const double* L21 = F + k1 + (long long)k0 * ld;
      double* A22 = F + k1 + (long long)k1 * ld;
      gemm_tile<false, true, kCoopStages, kSygBK>(L21, ld, L21, ld, A22, ld, rest, rest, k1 - k0, t.a * kTile,
                                                  t.b * kTile, -1.0, 1.0, true, smem);
      if (t.a == 0 && t.b == 0 && k1 < s) {  // the next group's first diagonal tile is final: factor it
        __syncthreads();
        const int p1 = k1 / kTile, nb1 = min(kTile, s - k1);
        double* inv1 = pg.pool + pg.sc.inv[node] + p1 * kTileInvStride;
        const int bad = potrf_trtri_tile(F + k1 + (long long)k1 * ld, ld, nb1, inv1, smem);
        if (threadIdx.x == 0 && bad >= 0) atomicMin(info + node, fd.sep_start[node] + k1 + bad);
      }
      break;
    }
    case CT_X2: {  // X[k.., c] = -inv Y[:, c] (c < panel) or X[k.., k..] = inv
      const int k = t.arg * kTile, nb = min(kTile, s - k), c = t.a * kTile;
      const double* inv = pg.pool + pg.sc.inv[node] + t.arg * kTileInvStride;
      if (c < k) {  // X[k, c] = -inv sum_q Y_q[:, c]: sum the partials into Y_0, one GEMM
        const int nq = (k - c + kX1Chunk - 1) / kX1Chunk;
        const long long ysz = (long long)kTile * s * ((s + kX1Chunk - 1) / kX1Chunk);
        double* Y0 = pg.pool + pg.sc.Y[node] + (t.arg & 1) * ysz + (long long)c * kTile;
        if (nq > 1) {
          const long long qs = (long long)kTile * s;  // stride between partials
          constexpr int PER = kTile * kTile / 128;     // elements per thread (128 threads)
          double acc[PER];  // one partial = PER independent loads in flight per thread
#pragma unroll
          for (int u = 0; u < PER; ++u) acc[u] = __ldcg(Y0 + threadIdx.x + 128 * u);
          for (int qq = 1; qq < nq; ++qq) {
            const double* Yq = Y0 + qq * qs;
#pragma unroll
            for (int u = 0; u < PER; ++u) acc[u] += __ldcg(Yq + threadIdx.x + 128 * u);
          }
#pragma unroll
          for (int u = 0; u < PER; ++u) Y0[threadIdx.x + 128 * u] = acc[u];
          __threadfence();
          __syncthreads();
        }
        gemm_tile<false, false, kCoopStages>(inv, kTile, Y0, kTile, X + k + (long long)c * ldx, ldx, nb, kTile,
                                             nb, 0, 0, -1.0, 0.0, false, smem);
      } else {
        for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
          const int i = idx % nb, j = idx / nb;
          X[(k + i) + (long long)(k + j) * ldx] = __ldcg(inv + i + j * kTile);
        }
      }
      break;
    }
    case CT_W: {  // W21 tile (a, c) = L21[a, c*64..s) X[c*64..s, c]
      const int b = f - s, c = t.b * kTile;
      double* W = pg.pool + pg.sc.W[node];
      const int ldw = pg.sc.ldw[node];
      gemm_tile<false, false, kCoopStages>(F + s + (long long)c * ld, ld, X + c + (long long)c * ldx, ldx,
                              W + (long long)c * ldw, ldw, b, min(kTile, s - c), s - c, t.a * kTile, 0,
                              1.0, 0.0, false, smem);
      break;
    }
  }
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Dataflow factorization: CTAs pull tasks in the program's topological order from a global
// counter; a task's first thread waits (bounded) until each dependency counter reaches its
// target, the task runs, and its counters are incremented after a fence. A task only waits
// on earlier tasks and all CTAs are co-resident (cooperative launch), so the queue always
// progresses; a wait that exceeds the bound sets *err (the host raises) instead of hanging.
__global__ void __launch_bounds__(128, kDfCtasPerSm) coop_factor_df_kernel(FrontDev fd, CoopProgram pg,
                                                             const DfTask* __restrict__ tasks, int ntasks,
                                                             int* ctr, int* qhead, int* info, int* err,
                                                             unsigned long long* prof,
                                                             unsigned long long* trace) {
  extern __shared__ __align__(16) double smem[];
  constexpr int kWords = (int)(sizeof(DfTask) / sizeof(int));
  static_assert(kWords <= 32 && sizeof(DfTask) % sizeof(int) == 0, "task descriptor must fit one warp");
  __shared__ int ti_s[2];
  __shared__ DfTask tsh[2];  // current / next task (the next one is claimed and loaded ahead)
  const int tid = threadIdx.x;
  if (tid == 0) ti_s[0] = atomicAdd(qhead, 1);
  __syncthreads();
  if (tid < kWords && ti_s[0] < ntasks) reinterpret_cast<int*>(&tsh[0])[tid] = reinterpret_cast<const int*>(tasks + ti_s[0])[tid];
  __syncthreads();
  for (int buf = 0;; buf ^= 1) {
    const int ti = ti_s[buf];
    if (ti >= ntasks) break;
    const DfTask& t = tsh[buf];
    // claim the next task now: the queue atomic's latency hides behind this task
    if (tid == 0) ti_s[buf ^ 1] = atomicAdd(qhead, 1);
    long long c0 = 0, c1 = 0;
    if (prof && tid == 0) c0 = clock64();
    if (trace && tid == 0) trace[4 * ti + 0] = gtimer();
    if (tid < kDeps) {  // one thread per dependency
      const int cix = t.dep[tid];
      if (cix >= 0) {
        const int tg = t.tgt[tid];
        long long spins = 0;
        while (*(volatile int*)(ctr + cix) < tg) {
          __nanosleep(32);
          if (++spins > (1LL << 25) || *(volatile int*)err) {  // bounded; after one timeout, none
            atomicExch(err, 1);
            break;
          }
        }
      }
      __threadfence();
    }
    __syncthreads();
    if (prof && tid == 0) c1 = clock64();
    if (trace && tid == 0) trace[4 * ti + 1] = gtimer();
    const int tn = ti_s[buf ^ 1];
    int nw = 0;  // next descriptor word, loaded before the task and parked in shared memory after it
    if (tid < kWords && tn < ntasks) nw = __ldg(reinterpret_cast<const int*>(tasks + tn) + tid);
    run_task(t.t, fd, pg, info, smem);
    __syncthreads();
    if (tid < kSigs) {  // one thread per signal, each after its own release fence
      __threadfence();
      if (t.sig[tid] >= 0) atomicAdd(ctr + t.sig[tid], (int)t.sw[tid]);
    }
    if (tid == 0) {
      if (trace) {
        trace[4 * ti + 2] = gtimer();
        trace[4 * ti + 3] = blockIdx.x;
      }
      if (prof) {  // per task type: waiting cycles, running cycles, count
        const long long c2 = clock64();
        atomicAdd(prof + 3 * t.t.type + 0, (unsigned long long)(c1 - c0));
        atomicAdd(prof + 3 * t.t.type + 1, (unsigned long long)(c2 - c1));
        atomicAdd(prof + 3 * t.t.type + 2, 1ULL);
      }
    }
    if (tid < kWords && tn < ntasks) reinterpret_cast<int*>(&tsh[buf ^ 1])[tid] = nw;
    __syncthreads();
  }
}

// ---- cooperative coarse solve ----
struct SolveProgram {
  const CsTask* ft;
  const CsTask* bt;
  const CsRed* fr;
  const CsRed* br;
  const int* ft_off;  // [L+1]
  const int* bt_off;
  const int* fr_off;
  const int* br_off;
  int nlevels;
  int nfr;  // number of forward reductions (offset of the backward counters)
  const double* wpool;  // W21 rows (r >= s) of the W21 fronts (CsTask w_off / ldw)
  double* tbuf;         // backward: t = -L21^T x_bnd per separator row of the L21 fronts
  int n;                // coarse size
};

struct SolveShared {
  double vs[512];
  double red[4][64];
  int last;
};

// Static part of one gather (child-update sources of one front position), loaded before the
// dependency wait; value() then only reads the update entries (same summation order).
struct GatherPre {
  int q0, q1, i0, i1;
  __device__ __forceinline__ void load(const LevelView& lv, long long gbase, int pos, bool on) {
    q0 = q1 = 0;
    i0 = i1 = -1;
    if (!on) return;
    const int* gp = lv.gat_ptr + gbase;
    q0 = gp[pos];
    q1 = gp[pos + 1];
    if (q1 > q0) i0 = lv.gat_src[q0];
    if (q1 > q0 + 1) i1 = lv.gat_src[q0 + 1];
    BDDC_CHECK(q1 >= q0 && i0 >= -1 && i1 >= -1);
  }
  __device__ __forceinline__ double value(const LevelView& lv, const double* __restrict__ upd) const {
    double acc = 0.0;
    if (i0 >= 0) acc += __ldcg(upd + i0);
    if (i1 >= 0) acc += __ldcg(upd + i1);
    for (int q = q0 + 2; q < q1; ++q) acc += __ldcg(upd + lv.gat_src[q]);
    return acc;
  }
};

// sum_p partial[(p0 + p) * 64 + i] in order p = 0 .. np-1, four loads in flight
__device__ __forceinline__ double sum_partials(const double* __restrict__ partial, int p0, int np, int i) {
  double a = 0.0;
  int p = 0;
  for (; p + 4 <= np; p += 4) {
    const double v0 = __ldcg(partial + (long long)(p0 + p) * 64 + i);
    const double v1 = __ldcg(partial + (long long)(p0 + p + 1) * 64 + i);
    const double v2 = __ldcg(partial + (long long)(p0 + p + 2) * 64 + i);
    const double v3 = __ldcg(partial + (long long)(p0 + p + 3) * 64 + i);
    a += v0;
    a += v1;
    a += v2;
    a += v3;
  }
  for (; p < np; ++p) a += __ldcg(partial + (long long)(p0 + p) * 64 + i);
  return a;
}

// sum over the np partials of all 64 outputs by the whole CTA: thread (o, quarter) sums its
// quarter in order, the quarters are added in order (deterministic). Valid for tid < 64.
__device__ __forceinline__ double sum_partials_cta(const double* __restrict__ partial, int p0, int np,
                                                   SolveShared& sh) {
  const int tid = threadIdx.x, o = tid & 63, qt = tid >> 6;
  const int a = (np * qt) >> 2, b = (np * (qt + 1)) >> 2;
  double* red = &sh.red[0][0];
  red[qt * 64 + o] = sum_partials(partial, p0 + a, b - a, o);
  __syncthreads();
  return tid < 64 ? ((red[o] + red[64 + o]) + (red[128 + o] + red[192 + o])) : 0.0;
}

// Forward task (bottom-up). A front holds [X; L21] (X = L11^{-1}); fronts with s up to the W
// limit also keep W21 = L21 X in the scratch pool (t.ldw > 0). Modes:
//   0: rows of [X; W21] times v = rhs + child updates: y_s (rows < s), upd = gathered - W21 v;
//      for L21 fronts only rows < s (their chunks end at s)
//   1: s <= 64 (W21 fronts): 256 rows x all separator columns, one thread per row
//   4: L21 rows times the final y_s chunk: upd = gathered - L21 y_s
// Everything that does not depend on other tasks (front entries, gather indices) is loaded
// before wait() (the dataflow dependency wait). Returns true when this CTA wrote the chunk's
// final values (single task, or the last of the chunk's tasks to arrive, which sums the
// partials in fixed order: deterministic).
template <class Wait>
__device__ bool solve_fwd_task(const CsTask& t, const FrontDev& fd, const LevelView& lv, const SolveProgram& sp,
                               const double* __restrict__ rhs, double* __restrict__ partial,
                               double* __restrict__ ybuf, int* __restrict__ cnt_f, SolveShared& sh, Wait wait) {
  const int tid = threadIdx.x;
  const double* F = fd.fronts + t.front_off;
  const long long ld = t.ld;
  const int s = t.s;
  const bool wf = t.ldw > 0;  // W21 front
  __syncthreads();
  if (t.mode == 1) {  // s <= 64: one thread per row, all separator columns
    const int r = t.r0 + tid;
    const int ke = r < t.rend ? (r < s ? r + 1 : s) : 0;
    const bool wr = r >= s;
    const double* Fr = wr ? sp.wpool + t.w_off + (r - s) : F + r;
    const long long lr = wr ? (long long)t.ldw : ld;
    double fv[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) fv[u] = u < ke ? __ldcs(Fr + (long long)u * lr) : 0.0;
    GatherPre gv, gr;
    gv.load(lv, t.gat_base, tid, tid < s);
    gr.load(lv, t.gat_base, r, r >= s && r < t.rend);
    const double rv = tid < s ? rhs[t.s0 + tid] : 0.0;
    wait();
    if (tid < s) sh.vs[tid] = rv + gv.value(lv, fd.upd);
    const double gu = gr.value(lv, fd.upd);
    __syncthreads();
    if (r < t.rend) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k0 = 0; k0 < ke; k0 += 16) {
        if (k0 > 0) {
#pragma unroll
          for (int u = 0; u < 16; ++u) fv[u] = k0 + u < ke ? __ldcs(Fr + (long long)(k0 + u) * lr) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) acc[u & 3] += k0 + u < ke ? fv[u] * sh.vs[k0 + u] : 0.0;
      }
      const double a = (acc[0] + acc[1]) + (acc[2] + acc[3]);
      if (r < s) ybuf[t.s0 + r] = a;
      else fd.upd[t.upd_off + (r - s)] = gu - a;
    }
    return true;
  }
  const bool lrows = t.mode == 4;  // L21 rows x the final y_s
  const int rr = tid & 63, grp = tid >> 6;
  const int r = t.r0 + rr;
  const int cg = t.span >> 2;  // columns per thread group: 64, or 16 (one batch, before the wait)
  const int kb = t.c0 + grp * cg;
  int ke = r < t.rend ? min(kb + cg, s) : kb;
  if (r < s) ke = min(ke, r + 1);
  const bool wr = wf && r >= s;
  const double* Fr = wr ? sp.wpool + t.w_off + (r - s) : F + r;
  const long long lr = wr ? (long long)t.ldw : ld;
  double fv[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) fv[u] = kb + u < ke ? __ldcs(Fr + (long long)(kb + u) * lr) : 0.0;
  const int kk = t.c0 + tid;
  const int rw = t.r0 + tid;  // row finalized by this thread (tid < 64)
  GatherPre gv, gr;
  gv.load(lv, t.gat_base, kk, !lrows && kk < s && tid < t.span);
  gr.load(lv, t.gat_base, rw, tid < 64 && rw < t.rend && rw >= s);
  const double rv = (!lrows && kk < s) ? rhs[t.s0 + kk] : 0.0;
  wait();
  double vin = 0.0;
  if (kk < s && tid < t.span) vin = lrows ? __ldcg(ybuf + t.s0 + kk) : rv + gv.value(lv, fd.upd);
  sh.vs[tid] = vin;
  if (t.span > 256) {  // 512-wide tasks: the second half of the columns, gathered after the wait
    const int k2 = kk + 256;
    double v2 = 0.0;
    if (k2 < s) {
      if (lrows) {
        v2 = __ldcg(ybuf + t.s0 + k2);
      } else {
        GatherPre g2;
        g2.load(lv, t.gat_base, k2, true);
        v2 = rhs[t.s0 + k2] + g2.value(lv, fd.upd);
      }
    }
    sh.vs[256 + tid] = v2;
  }
  __syncthreads();
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k0 = kb; k0 < ke; k0 += 16) {
    if (k0 > kb) {
#pragma unroll
      for (int u = 0; u < 16; ++u) fv[u] = k0 + u < ke ? __ldcs(Fr + (long long)(k0 + u) * lr) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) acc[u & 3] += k0 + u < ke ? fv[u] * sh.vs[k0 + u - t.c0] : 0.0;
  }
  sh.red[grp][rr] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
  __syncthreads();
  auto finish = [&](double a) {
    if (rw < s) ybuf[t.s0 + rw] = a;
    else fd.upd[t.upd_off + (rw - s)] = gr.value(lv, fd.upd) - a;
  };
  if (t.np == 1) {
    if (tid < 64 && rw < t.rend) finish(sh.red[0][tid] + sh.red[1][tid] + sh.red[2][tid] + sh.red[3][tid]);
    return true;
  }
  if (tid < 64) {
    partial[(long long)t.part * 64 + tid] = sh.red[0][tid] + sh.red[1][tid] + sh.red[2][tid] + sh.red[3][tid];
    __threadfence();
  }
  __syncthreads();
  if (tid == 0) sh.last = atomicAdd(cnt_f + t.red, 1) == t.np - 1;
  __syncthreads();
  if (!sh.last) return false;
  __threadfence();
  const CsRed R = sp.fr[t.red];
  const double a = sum_partials_cta(partial, R.p0, R.np, sh);
  if (tid < 64 && rw < t.rend) finish(a);
  if (tid == 0) cnt_f[t.red] = 0;
  return true;
}

// Backward task (top-down), rw rows x 64 columns. Mode 3: rows of [X; W21]^T:
// x_s = X^T (y_s + t) - W21^T x_bnd (t = 0 and W21 rows on the W21 fronts; X rows only on the
// L21 fronts); mode 2 (L21 fronts, rows >= s): t = -L21^T x_bnd.
template <class Wait>
__device__ bool solve_bwd_task(const CsTask& t, const FrontDev& fd, const SolveProgram& sp,
                               double* __restrict__ sol, double* __restrict__ partial,
                               const double* __restrict__ ybuf, int* __restrict__ cnt_b, SolveShared& sh,
                               Wait wait) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int s = t.s;
  const long long ld = t.ld;
  const bool wf = t.ldw > 0;
  const int* bidx = fd.bnd_idx + fd.bnd_ptr[t.node];
  const double* F = fd.fronts + t.front_off;
  double* dst = t.mode == 2 ? sp.tbuf : sol;
  __syncthreads();
  // warp: 8 columns; lane: rows i = lane + 32 m; 16 loads in flight per batch
  const int kw = t.c0 + warp * 8;
  double fv[2][8];
  auto load_rows = [&](int m) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = lane + 32 * (m + h), r = t.r0 + i;
      const bool wr = wf && r >= s;
      const double* Fr = wr ? sp.wpool + t.w_off + (r - s) : F + r;
      const long long lr = wr ? (long long)t.ldw : ld;
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        const int k = kw + cc;
        const bool ok = k < s && r < t.rend && (r >= s || r >= k);
        fv[h][cc] = ok ? __ldcs(Fr + (long long)k * lr) : 0.0;
      }
    }
  };
  load_rows(0);
  const int r = t.r0 + tid;
  const bool mine = tid < t.span && r < t.rend;
  const int bi = (mine && r >= s) ? bidx[r - s] : -1;
  BDDC_CHECK(bi < sp.n);
  wait();
  sh.vs[tid] = !mine ? 0.0 : (r >= s ? -__ldcg(sol + bi) : __ldcg(ybuf + t.s0 + r) + __ldcg(sp.tbuf + t.s0 + r));
  if (t.span > 256) {  // 512-row tasks: the second half of the rows
    const int r2 = r + 256;
    const bool m2 = r2 < t.rend;
    sh.vs[256 + tid] = !m2 ? 0.0 : (r2 >= s ? -__ldcg(sol + bidx[r2 - s])
                                            : __ldcg(ybuf + t.s0 + r2) + __ldcg(sp.tbuf + t.s0 + r2));
  }
  __syncthreads();
  double acc[8];
#pragma unroll
  for (int cc = 0; cc < 8; ++cc) acc[cc] = 0.0;
  const int mend = min(t.span >> 5, (t.rend - t.r0 + 31) / 32);  // row batches that hold task rows
#pragma unroll 4
  for (int m = 0; m < 16; m += 2) {
    if (m >= mend) break;
    if (m > 0) load_rows(m);
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) acc[cc] += fv[h][cc] * sh.vs[lane + 32 * (m + h)];
  }
  if (t.np == 1) {
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const double v = warp_sum(acc[cc]);
      const int k = kw + cc;
      if (lane == 0 && k < s) dst[t.s0 + k] = v;
    }
    return true;
  }
#pragma unroll
  for (int cc = 0; cc < 8; ++cc) {
    const double v = warp_sum(acc[cc]);
    if (lane == 0) partial[(long long)t.part * 64 + warp * 8 + cc] = v;
  }
  if (lane == 0) __threadfence();
  __syncthreads();
  if (tid == 0) sh.last = atomicAdd(cnt_b + t.red, 1) == t.np - 1;
  __syncthreads();
  if (!sh.last) return false;
  __threadfence();
  const CsRed R = sp.br[t.red];
  const int k = R.t0 + tid;
  const double a = sum_partials_cta(partial, R.p0, R.np, sh);
  if (tid < 64 && k < s) dst[t.s0 + k] = a;
  if (tid == 0) cnt_b[t.red] = 0;
  return true;
}

// Dataflow solve: one queue (forward tasks bottom-up, then backward tasks top-down). A
// forward task waits until every row chunk of the node's children is final; a backward
// task until the nearest ancestor with separator columns is final (or, without one, its own
// forward sweep). Chunks finalized signal their node counters. No grid barriers.
// v = T rho for one subdomain (n <= 256): thread (row i, half h) sums k = h, h + 2, ...; the
// halves are combined in fixed order.
__device__ void solve_tv_task(int sub, const TvArgs& tv, SolveShared& sh) {
  const int tid = threadIdx.x, n = tv.n;
  const double* T = tv.T + (long long)sub * n * n;
  __syncthreads();
  if (tid < n) sh.vs[tid] = tv.rho[(long long)sub * n + tid];
  __syncthreads();
  double* part = &sh.red[0][0];  // [2][128]
  for (int i0 = 0; i0 < n; i0 += 128) {
    const int i = i0 + (tid & 127), h = tid >> 7;
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    if (i < n) {
      int k = h;
      for (; k + 14 < n; k += 16) {
        double tv8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) tv8[u] = __ldcs(T + i + (long long)(k + 2 * u) * n);
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u & 3] += tv8[u] * sh.vs[k + 2 * u];
      }
      for (; k < n; k += 2) a[0] += __ldcs(T + i + (long long)k * n) * sh.vs[k];
    }
    part[h * 128 + (tid & 127)] = (a[0] + a[1]) + (a[2] + a[3]);
    __syncthreads();
    if (tid < 128 && i0 + tid < n) tv.v[(long long)sub * n + i0 + tid] = part[tid] + part[128 + tid];
    __syncthreads();
  }
}

#ifndef BDDC_SOLVE_CTAS
#define BDDC_SOLVE_CTAS 3  // A/B compile switch: resident CTAs per SM of the coarse solve
#endif
__global__ void __launch_bounds__(256, BDDC_SOLVE_CTAS) coop_solve_df_kernel(FrontDev fd, LevelView lv, SolveProgram sp,
                                                            const SdTask* __restrict__ tasks, int ntasks,
                                                            int* ctr, int* qhead, int* err,
                                                            const double* __restrict__ rhs,
                                                            double* __restrict__ sol,
                                                            double* __restrict__ partial,
                                                            double* __restrict__ ybuf, int* __restrict__ cnt,
                                                            TvArgs tv, unsigned long long* __restrict__ trace) {
  __shared__ SolveShared sh;
  constexpr int kWords = (int)(sizeof(SdTask) / sizeof(int));
  static_assert(kWords <= 64, "solve task descriptor too large");
  __shared__ int ti_s[2];
  __shared__ SdTask tsh[2];
  const int tid = threadIdx.x;
  int* cnt_f = cnt;
  int* cnt_b = cnt + sp.nfr;
  if (tid == 0) ti_s[0] = atomicAdd(qhead, 1);
  __syncthreads();
  if (tid < kWords && ti_s[0] < ntasks)
    reinterpret_cast<int*>(&tsh[0])[tid] = reinterpret_cast<const int*>(tasks + ti_s[0])[tid];
  __syncthreads();
  for (int buf = 0;; buf ^= 1) {
    const int ti = ti_s[buf];
    if (ti >= ntasks) break;
    const SdTask& T = tsh[buf];
    if (trace && tid == 32) trace[4 * ti] = gtimer();
    int tn = ntasks, nw = 0;
    // the next task is claimed now (the result is first needed at the wait below) and its
    // descriptor loaded after the wait (parked in shared memory after this task)
    int claim = 0;
    if (tid == 0) claim = atomicAdd(qhead, 1);
    // dependency wait, after the task has issued its static loads
    auto wait = [&] {
      if (tid == 0) ti_s[buf ^ 1] = claim;
      if (tid == 32 && T.dep >= 0) {
        long long spins = 0;
        while (*(volatile int*)(ctr + T.dep) < T.tgt) {
          __nanosleep(20);
          if (++spins > (1LL << 25) || *(volatile int*)err) {
            atomicExch(err, 1);
            break;
          }
        }
        __threadfence();
      }
      if (trace && tid == 32) trace[4 * ti + 1] = gtimer();
      __syncthreads();
      tn = ti_s[buf ^ 1];
      if (tid < kWords && tn < ntasks) nw = __ldg(reinterpret_cast<const int*>(tasks + tn) + tid);
    };
    bool fin = false;
    if (T.dir == 0) fin = solve_fwd_task(T.t, fd, lv, sp, rhs, partial, ybuf, cnt_f, sh, wait);
    else if (T.dir == 1) fin = solve_bwd_task(T.t, fd, sp, sol, partial, ybuf, cnt_b, sh, wait);
    else {
      wait();
      if (tv.T) solve_tv_task(T.t.node, tv, sh);
    }
    __syncthreads();
    if (trace && tid == 0) {
      trace[4 * ti + 2] = gtimer();
      trace[4 * ti + 3] = blockIdx.x;
    }
    if (fin && tid == 0) {
      __threadfence();
      if (T.sig0 >= 0) atomicAdd(ctr + T.sig0, 1);
      if (T.sig1 >= 0) atomicAdd(ctr + T.sig1, 1);
      if (T.sig2 >= 0) atomicAdd(ctr + T.sig2, 1);
    }
    if (tid < kWords && tn < ntasks) reinterpret_cast<int*>(&tsh[buf ^ 1])[tid] = nw;
    __syncthreads();
  }
  if (*(volatile int*)err)  // a dependency wait timed out: poison the result (PCG reports it)
    for (int i = blockIdx.x * blockDim.x + tid; i < sp.n; i += gridDim.x * blockDim.x)
      sol[i] = __longlong_as_double(0x7ff8000000000000LL);
}

}  // namespace

// ---------------------------------------------------------------------------------------
// host: program construction and launches
// ---------------------------------------------------------------------------------------

struct CoopState {
  CoopProgram pg{};
  SolveProgram sp{};
  int grid_f = 0, grid_s = 0;
  size_t smem_f = 0;
  DfTask* dtasks = nullptr;  // the program of the launch in flight (one of progs)
  int ndtasks = 0;
  std::vector<std::pair<DfTask*, int>> progs;  // 1 program, or 2 (this rank's subtrees, top)
  int* ctr = nullptr;  // [nctr] dependency counters + queue head + error flag
  int nctr = 0;
  unsigned long long* prof = nullptr;  // BDDC_COOP_TIMING: per task type wait / run cycles
};

static std::map<const Ctx*, CoopState> g_coop;

// Fronts whose separator is at most this size keep W21 = L21 X for the solve (one GEMV phase
// per front and direction); larger ones (the top of the tree: 78% of the W21 flops at cfg5 in
// 15 fronts) solve with L21 in place and one more dependent GEMV phase (coarse.cu). The
// threshold trades setup for solve time: measured at 4 CTAs/SM (profiles/r02/ab/w21_ctas4), cfg5
// coarse 1183 / 1163 / 1147 ms and coarse solve 11.5 / 11.9 / 13.7 ms per apply at 2048 / 1024 /
// 512; 1024 wins below about 50 applies per setup (the BASELINE configs take 6-10).
int coarse_w21_max_sep() {  // (>= 127: L21 fronts have separators of two 64-chunks or more)
  const char* e = getenv("BDDC_W21_MAX_SEP");
  return e ? std::max(atoi(e), 127) : 1024;
}

long long coarse_df_layout(const FrontPlan& fp, std::vector<long long>& inv, std::vector<long long>& Y,
                           std::vector<long long>& W, std::vector<int>& ldw) {
  const int N = fp.nnodes;
  const int wmax = coarse_w21_max_sep();
  inv.assign(N, 0); Y.assign(N, 0); W.assign(N, 0); ldw.assign(N, 0);
  long long off = 0;  // every front its own scratch (levels overlap in the dataflow program)
  for (int l = 0; l < fp.nlevels; ++l)
    for (int i = fp.level_ptr[l]; i < fp.level_ptr[l + 1]; ++i) {
      const int nd = fp.level_list[i];
      const int s = fp.sep_size[nd], b = fp.bnd_size[nd], np = ceil_div(s, kTile);
      inv[nd] = off; off += (long long)std::max(np, 1) * kTileInvStride;
      Y[nd] = off; off += 2 * round_up((long long)kTile * std::max(s, 1), 2) * ceil_div(std::max(s, 1), kX1Chunk);
      if (s <= wmax) {  // W21 front (ldw > 0 marks it for the solve)
        ldw[nd] = (int)round_up(std::max(b, 2), 2);
        W[nd] = off; off += round_up((long long)ldw[nd] * std::max(s, 1), 2);
      }
    }
  return std::max(off, 2LL);
}

void coop_build(Ctx& c) {
  FrontPlan& fp = c.fp;
  LevelSchedule& ls = c.sched;
  CoopState& st = g_coop[&c];
  st = CoopState{};
  st.smem_f = sizeof(double) * std::max<int>(std::max(gemm_smem_doubles<kCoopStages>(), gemm_smem_doubles<kCoopStages, kSygBK>()),
                                             kFactSmemDoubles);
  BDDC_CUDA(cudaFuncSetAttribute(coop_factor_df_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)st.smem_f));
  int nsm = 0, per_f = 0, per_s = 0;
  BDDC_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c.device));
  BDDC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_s, coop_solve_df_kernel, 256, 0));
  BDDC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_f, coop_factor_df_kernel, 128, st.smem_f));
  st.grid_f = nsm * std::max(std::min(per_f, kDfCtasPerSm), 1);
  st.grid_s = nsm * std::max(std::min(per_s, 4), 1);
  const int grid_f = st.grid_f;
  const int N = fp.nnodes, L = fp.nlevels;
  std::vector<long long> inv(N, 0), Y(N, 0), W(N, 0);
  std::vector<int> ldw(N, 2);
  long long pool = 2;
  int max_children = 0;
  for (int nd = 0; nd < N; ++nd) max_children = std::max(max_children, fp.child_ptr[nd + 1] - fp.child_ptr[nd]);
  std::vector<int> grp(N, kGroup);
  {
    const char* e = getenv("BDDC_GROUP_MIN_SEP");
    const int gmin = e ? atoi(e) : 0;
    for (int nd = 0; nd < N; ++nd)
      if (fp.sep_size[nd] < gmin) grp[nd] = 1;
    c.fp.d.grp = c.upload(grp.data(), N);
  }
  // ---- dataflow factorization program ----
  HostTimer ht;
  {
    int nctr = 0;
    auto newc = [&](int n) { const int b = nctr; nctr += n; return b; };
    // per node counter bases and totals
    std::vector<int> c_ea(N), c_syall(N), c_pt(N), c_tsr(N), c_upd(N), c_x1(N), c_x2(N), c_x2row(N),
        c_x2col(N), c_x2all(N), c_tsall(N), c_w(N), c_gts(N), nT(N), nP(N), tot_sy(N, 0), tot_ts(N, 0),
        tot_w(N, 0), tot_x2(N, 0);
    std::vector<std::vector<int>> nea(N);
    for (int nd = 0; nd < N; ++nd) {
      const int s = fp.sep_size[nd], f = s + fp.bnd_size[nd];
      const int T = ceil_div(std::max(f, 1), kTile), np = ceil_div(s, kTile), ng = ceil_div(s, grp[nd] * kTile);
      nT[nd] = T; nP[nd] = np;
      c_ea[nd] = newc(std::max(1, fp.child_ptr[nd + 1] - fp.child_ptr[nd]));
      c_syall[nd] = newc(1); c_tsall[nd] = newc(1); c_w[nd] = newc(1); c_x2all[nd] = newc(1);
      c_pt[nd] = newc(std::max(np, 1));
      c_tsr[nd] = newc(std::max(np * T, 1));
      c_gts[nd] = newc(std::max(ng, 1));        // TS tasks done per panel group
      c_upd[nd] = newc(T * (T + 1) / 2);        // panels applied per (lower) absolute tile
      c_x1[nd] = newc(std::max(np, 1));         // X1 tasks done per panel row
      c_x2[nd] = newc(std::max(np * np, 1));
      c_x2row[nd] = newc(std::max(np, 1));
      c_x2col[nd] = newc(std::max(np, 1));
      nea[nd].assign(std::max(1, fp.child_ptr[nd + 1] - fp.child_ptr[nd]), 0);
    }
    auto upd = [&](int nd, int I, int J) { return c_upd[nd] + I * (I + 1) / 2 + J; };
    auto mk = [&](int type, int nd, int a, int b, int arg) {
      DfTask t;
      t.t = CoopTask{type, nd, a, b, arg};
      for (int d = 0; d < kDeps; ++d) { t.dep[d] = -1; t.tgt[d] = 0; }
      for (int q = 0; q < kSigs; ++q) t.sig[q] = -1;
      for (int q = 0; q < 8; ++q) t.sw[q] = 1;
      return t;
    };
    auto dep = [&](DfTask& t, int cix, int tgt) {
      if (tgt <= 0) return;
      for (int d = 0; d < kDeps; ++d)
        if (t.dep[d] < 0) { t.dep[d] = cix; t.tgt[d] = tgt; return; }
      throw std::runtime_error("coarse dataflow: too many dependencies");
    };
    auto sig = [&](DfTask& t, int cix, int w = 1) {
      for (int q = 0; q < kSigs; ++q)
        if (t.sig[q] < 0) { t.sig[q] = cix; t.sw[q] = (unsigned char)w; return; }
      throw std::runtime_error("coarse dataflow: too many signals");
    };
    // one program over the active nodes `act` (with_lt: also the local T tiles)
    auto gen = [&](const std::vector<char>& act, bool with_lt) {
    std::vector<DfTask> dt;
    const long long off = coarse_df_layout(fp, inv, Y, W, ldw);  // X lives in the fronts
    // the local setup's T tiles (no dependencies): the simulated schedule places them in the
    // CTA time the critical path leaves idle
    c.lt_fusable = c.geo.nG_pad > 0 && c.geo.nG_pad % kTile == 0;
    if (c.lt_fusable && with_lt) {
      const int nt = c.geo.nG_pad / kTile;
      for (int sub = c.geo.s_lo; sub < c.geo.s_hi; ++sub)
        for (int I = 0; I < nt; ++I)
          for (int J = 0; J <= I; ++J) dt.push_back(mk(CT_LT, sub, I, J, 0));
    }
    for (int l = 0; l < L; ++l) {
      std::vector<int> nodes(fp.level_list.begin() + fp.level_ptr[l], fp.level_list.begin() + fp.level_ptr[l + 1]);
      // extend-add of the children (child order per parent)
      for (int k = 0; k < max_children; ++k) {
        long long cols = 0;
        for (int nd : nodes)
          if (act[nd] && fp.child_ptr[nd + 1] - fp.child_ptr[nd] > k) cols += fp.bnd_size[fp.child_list[fp.child_ptr[nd] + k]];
        int chunk = 64;
        while (chunk > 2 && cols / chunk < 2LL * grid_f) chunk >>= 1;
        for (int nd : nodes) {
          if (!act[nd] || fp.child_ptr[nd + 1] - fp.child_ptr[nd] <= k) continue;
          const int ch = fp.child_list[fp.child_ptr[nd] + k];
          for (int q = 0; q < fp.bnd_size[ch]; q += chunk) {
            DfTask t = mk(CT_EA, nd, q, chunk, k);
            // (a child outside this program was factored before its launch: no counter)
            if (act[ch]) dep(t, c_syall[ch], tot_sy[ch]);
            // an aliased update block may share pages with grandchildren's: no write into it
            // before every child subtree is done (front_vmm.cu)
            if (fp.ualias[nd] && k == 0)
              for (int o = fp.child_ptr[nd] + 1; o < fp.child_ptr[nd + 1]; ++o)
                if (act[fp.child_list[o]]) dep(t, c_syall[fp.child_list[o]], tot_sy[fp.child_list[o]]);
            if (k > 0) dep(t, c_ea[nd] + k - 1, nea[nd][k - 1]);
            sig(t, c_ea[nd] + k);
            dt.push_back(t);
            nea[nd][k]++;
          }
        }
      }
      for (int nd : nodes) {
        const int s = fp.sep_size[nd], f = s + fp.bnd_size[nd], np = nP[nd], T = nT[nd];
        const int nch = fp.child_ptr[nd + 1] - fp.child_ptr[nd];
        if (s <= 0 || !act[nd]) continue;
        {
          DfTask t = mk(CT_PT, nd, 0, 0, 0);
          if (nch > 0) dep(t, c_ea[nd] + nch - 1, nea[nd][nch - 1]);
          sig(t, c_pt[nd] + 0);
          dt.push_back(t);
        }
        auto tiles_of = [&](int r0, int r1) {  // absolute 64-tiles overlapping rows [r0, r1)
          return std::make_pair(r0 / kTile, (std::min(r1, f) - 1) / kTile);
        };
        // tile (I, J) holds every update of the panels before p (TS / SY / SYG readiness)
        auto dep_tile = [&](DfTask& t, int r0, int c0, int p) {
          if (p <= 0) return;
          const auto ri = tiles_of(r0, r0 + kTile), ci = tiles_of(c0, c0 + kTile);
          for (int I = ri.first; I <= ri.second; ++I)
            for (int J = ci.first; J <= ci.second; ++J)
              if (I >= J) dep(t, upd(nd, I, J), p);
        };
        // ---- factorization: panels in groups of kGroup ----
        const int Gn = grp[nd];
        const int ng = ceil_div(s, Gn * kTile);
        for (int g = 0; g < ng; ++g) {
          const int k0 = group_k0(g, Gn), k1 = group_k1(g, Gn, s), p0 = k0 / kTile, p1 = ceil_div(k1, kTile);
          int gts = 0;  // TS tasks of this group
          for (int p = p0; p < p1; ++p) {
            const int k = p * kTile, nb = std::min(kTile, s - k), rest = f - k - nb, nt = ceil_div(rest, kTile);
            for (int a = 0; a < nt; ++a) {
              DfTask t = mk(CT_TS, nd, a, 0, p);
              dep(t, c_pt[nd] + p, 1);
              dep_tile(t, k + nb + a * kTile, k, p);
              sig(t, c_tsr[nd] + p * T + a);
              sig(t, c_tsall[nd]);
              sig(t, c_gts[nd] + g);
              dt.push_back(t);
              tot_ts[nd]++;
              gts++;
            }
            // right-looking updates inside the group's block column (columns [k + nb, k1))
            const int ncol = ceil_div(k1 - k - nb, kTile);
            for (int a = 0; a < nt; ++a)
              for (int bb = 0; bb <= a && bb < ncol; ++bb) {
                DfTask t = mk(CT_SY, nd, a, bb, p);
                dep(t, c_tsr[nd] + p * T + a, 1);
                if (bb != a) dep(t, c_tsr[nd] + p * T + bb, 1);
                dep_tile(t, k + nb + a * kTile, k + nb + bb * kTile, p);
                if (nb == kTile) sig(t, upd(nd, p + 1 + a, p + 1 + bb));
                sig(t, c_syall[nd]);
                if (a == 0 && bb == 0 && k + nb < s) sig(t, c_pt[nd] + p + 1);  // lookahead PT
                dt.push_back(t);
                tot_sy[nd]++;
              }
          }
          // the trailing matrix beyond the block column, once for the whole group (K = k1 - k0)
          const int ntg = ceil_div(f - k1, kTile);
          for (int a = 0; a < ntg; ++a)
            for (int bb = 0; bb <= a; ++bb) {
              DfTask t = mk(CT_SYG, nd, a, bb, g);
              dep(t, c_gts[nd] + g, gts);
              dep_tile(t, k1 + a * kTile, k1 + bb * kTile, p0);
              if (k1 < s) sig(t, upd(nd, p1 + a, p1 + bb), p1 - p0);  // (k1 aligned: full group)
              sig(t, c_syall[nd]);
              if (a == 0 && bb == 0 && k1 < s) sig(t, c_pt[nd] + p1);  // lookahead PT
              dt.push_back(t);
              tot_sy[nd]++;
            }
        }
        // ---- X = L11^{-1} in place over L11, after the whole factorization of this front
        // (every TS / SY / SYG read of L11 is then done) ----
        for (int p = 0; p < np; ++p) {
          int nx1 = 0;  // X1 tasks of row p
          for (int cc = 0; cc < p; ++cc)
            for (int qq = 0; qq * kX1Blocks < p - cc; ++qq) {  // chunk qq: panel blocks m0 .. m1 - 1
              const int m0 = cc + qq * kX1Blocks, m1 = std::min(p, m0 + kX1Blocks);
              DfTask t = mk(CT_X1, nd, cc, qq, p);
              if (kX1Blocks <= 4)
                for (int m = m0; m < m1; ++m) dep(t, c_tsr[nd] + m * T + (p - m - 1), 1);  // L[p, m] final
              else
                dep(t, c_tsall[nd], tot_ts[nd]);  // (wider chunks: every L21 panel of the front final)
              dep(t, c_x2col[nd] + cc, m1 - cc);  // X[m, cc] final for m < m1 (column cc finishes in m order)
              if (p >= 2) dep(t, c_x2row[nd] + p - 2, p - 1);
              sig(t, c_x1[nd] + p);
              dt.push_back(t);
              ++nx1;
            }
          for (int cc = 0; cc <= p; ++cc) {
            DfTask t = mk(CT_X2, nd, cc, 0, p);
            dep(t, c_pt[nd] + p, 1);
            dep(t, c_syall[nd], tot_sy[nd]);
            if (cc < p) dep(t, c_x1[nd] + p, nx1);  // every X1 of row p read L[p, .]
            sig(t, c_x2[nd] + p * np + cc);
            sig(t, c_x2row[nd] + p);
            sig(t, c_x2col[nd] + cc);
            sig(t, c_x2all[nd]);
            dt.push_back(t);
            tot_x2[nd]++;
          }
        }
        const int b = f - s;
        if (b > 0 && ldw[nd] > 0) {  // W21 = L21 X for the solve (coarse_w21_max_sep)
          for (int a = 0; a < ceil_div(b, kTile); ++a)
            for (int cc = 0; cc < np; ++cc) {
              DfTask t = mk(CT_W, nd, a, cc, 0);
              dep(t, c_tsall[nd], tot_ts[nd]);
              dep(t, c_x2col[nd] + cc, np - cc);
              sig(t, c_w[nd]);
              dt.push_back(t);
              tot_w[nd]++;
            }
        }
        // X is in place in the front over L11; L21 stays; W21 (if any) in the scratch pool
      }
    }
    pool = std::max(pool, off);
    ht.mark("factor program: tasks");
    if (ht.on) fprintf(stderr, "bddc_setup host: factor program: %zu tasks, %d counters\n", dt.size(), nctr);
    // Queue order = the start order of a simulated list schedule on grid_f CTAs: whenever a
    // CTA is free it takes the ready task of highest upward rank (its estimated cost plus the
    // longest chain of work depending on it). A task is only started after its producers
    // finished, so the order is topological (deadlock-free under any real timing), and work
    // with no successors (X, W21) fills the CTAs that would otherwise block on the serial
    // panel chains of the top fronts.
    {
      const double ovh = 1.0;  // per-task scheduling cost (us)
      auto cost_of = [&](const DfTask& t) {
        const CoopTask& q = t.t;
        const int s = fp.sep_size[q.node];
        switch (q.type) {  // measured averages at 3 CTAs per SM (tools/df_trace.py)
          case CT_EA: return 2.5 + 0.15 * q.b;
          case CT_PT: return 15.0;
          case CT_TS: return 6.5;
          case CT_X1: return 8.5 * kX1Blocks;
          case CT_SY: {
            const int k = q.arg * kTile;
            return (q.a == 0 && q.b == 0 && k + kTile < s) ? 10.7 + 15.0 : 10.7;  // + lookahead PT
          }
          case CT_SYG: {
            const int k0 = group_k0(q.arg, grp[q.node]), k1 = group_k1(q.arg, grp[q.node], s);
            const double run = 4.0 + 6.7 * (k1 - k0) / 64.0;
            return (q.a == 0 && q.b == 0 && k1 < s) ? run + 15.0 : run;
          }
          case CT_X2: return 6.9;
          case CT_W: return 9.1;
          case CT_LT: return 18.2;
          default: return 8.0;
        }
      };
      const size_t n = dt.size();
      std::vector<double> cst(n), maxc(nctr, 0.0), rank(n, 0.0);
      for (size_t i = 0; i < n; ++i) cst[i] = cost_of(dt[i]) + ovh;
      for (long long i = (long long)n - 1; i >= 0; --i) {
        const DfTask& t = dt[i];
        double succ = 0.0;
        for (int q = 0; q < kSigs; ++q)
          if (t.sig[q] >= 0) succ = std::max(succ, maxc[t.sig[q]]);
        rank[i] = cst[i] + succ;
        for (int d = 0; d < kDeps; ++d)
          if (t.dep[d] >= 0) maxc[t.dep[d]] = std::max(maxc[t.dep[d]], rank[i]);
      }
      // waiters per counter (CSR), each counter's list by target
      std::vector<int> ndep(n, 0), cval(nctr, 0), wptr(nctr + 1, 0);
      for (size_t i = 0; i < n; ++i)
        for (int d = 0; d < kDeps; ++d)
          if (dt[i].dep[d] >= 0) { wptr[dt[i].dep[d] + 1]++; ndep[i]++; }
      for (int q = 0; q < nctr; ++q) wptr[q + 1] += wptr[q];
      std::vector<std::pair<int, int>> wlist(wptr[nctr]);
      {
        std::vector<int> fill(wptr.begin(), wptr.end() - 1);
        for (size_t i = 0; i < n; ++i)
          for (int d = 0; d < kDeps; ++d)
            if (dt[i].dep[d] >= 0) wlist[fill[dt[i].dep[d]]++] = {dt[i].tgt[d], (int)i};
      }
      for (int q = 0; q < nctr; ++q)
        if (wptr[q + 1] - wptr[q] > 1) std::sort(wlist.begin() + wptr[q], wlist.begin() + wptr[q + 1]);
      std::vector<int> wpos(wptr.begin(), wptr.end() - 1);
      // max-heap on (upward rank, then lower index), the keys stored in the heap entries
      // (no indirect rank[] loads in the comparisons)
      using Rk = std::pair<double, int>;  // (rank, -index)
      std::priority_queue<Rk> ready;
      for (size_t i = 0; i < n; ++i)
        if (!ndep[i]) ready.push({rank[i], -(int)i});
      using Ev = std::pair<double, int>;  // (finish time, task)
      std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> running;
      std::vector<int> order;
      order.reserve(n);
      int free = std::max(grid_f, 1);
      double now = 0.0;
      while (order.size() < n || !running.empty()) {
        while (free > 0 && !ready.empty()) {
          const int i = -ready.top().second;
          ready.pop();
          order.push_back(i);
          running.push({now + cst[i], i});
          --free;
        }
        if (running.empty()) break;  // (cannot happen for a valid program)
        const Ev e = running.top();
        running.pop();
        now = e.first;
        ++free;
        const DfTask& t = dt[e.second];
        for (int q = 0; q < kSigs; ++q) {
          const int cix = t.sig[q];
          if (cix < 0) continue;
          cval[cix] += t.sw[q];
          int& wp = wpos[cix];
          while (wp < wptr[cix + 1] && wlist[wp].first <= cval[cix]) {
            const int j = wlist[wp++].second;
            if (--ndep[j] == 0) ready.push({rank[j], -j});
          }
        }
      }
      ht.mark("factor program: list schedule");
      if (order.size() != n) throw std::runtime_error("coarse dataflow: program is not schedulable");
      std::vector<DfTask> sorted(n);
      for (size_t i = 0; i < n; ++i) sorted[i] = dt[order[i]];
      dt.swap(sorted);

      if (getenv("BDDC_COOP_TIMING"))
        fprintf(stderr, "coarse dataflow: simulated makespan %.1f us on %d CTAs (critical path %.1f us)\n", now,
                grid_f, *std::max_element(rank.begin(), rank.end()));
    }
    return dt;
    };
    std::vector<std::vector<DfTask>> programs;
    if (c.dist.on) {  // this rank's subtrees, then the replicated top (capi.cu: build_dist)
      std::vector<char> a0(N), a1(N);
      for (int nd = 0; nd < N; ++nd) a0[nd] = c.dist.phase[nd] == 0, a1[nd] = c.dist.phase[nd] == 1;
      programs.push_back(gen(a0, true));
      programs.push_back(gen(a1, false));
    } else {
      programs.push_back(gen(std::vector<char>(N, 1), true));
    }
    for (auto& dt : programs) st.progs.push_back({c.upload(dt.data(), dt.size()), (int)dt.size()});
    st.dtasks = st.progs[0].first;
    st.ndtasks = st.progs[0].second;
    ht.mark("factor program: upload");
    st.nctr = nctr;
    st.ctr = c.alloc<int>(nctr + 2);  // + queue head + error flag
  }
  if (getenv("BDDC_COOP_TIMING")) st.prof = c.alloc<unsigned long long>(3 * CT_NTYPES);
  st.pg.sc.inv = c.upload(inv.data(), N);
  st.pg.sc.Y = c.upload(Y.data(), N);
  st.pg.sc.W = c.upload(W.data(), N);
  st.pg.sc.ldw = c.upload(ldw.data(), N);
  st.pg.pool = c.alloc<double>(pool);
  // solve program: reductions of the forward / backward chunk partials
  int nfr = 0;
  for (int l = 0; l < L; ++l) nfr += ls.n_fwd_r[l];
  st.sp.fr = ls.fwd_r[0];
  st.sp.br = ls.bwd_r[0];
  st.sp.nfr = nfr;
  st.sp.tbuf = ls.tbuf;
  st.sp.wpool = st.pg.pool;
  st.sp.n = fp.n_coarse;
}

void coop_release(const Ctx& c) { g_coop.erase(&c); }

void coop_factor(Ctx& c, cudaStream_t s, int prog) {
  CoopState& st = g_coop.at(&c);
  st.dtasks = st.progs.at(prog).first;
  st.ndtasks = st.progs.at(prog).second;
  FrontDev fd = c.fp.d;
  int* info = c.fp.info;
  BDDC_CUDA(cudaMemsetAsync(st.ctr, 0, sizeof(int) * (st.nctr + 2), s));
  int* qhead = st.ctr + st.nctr;
  int* err = st.ctr + st.nctr + 1;
  const DfTask* tasks = st.dtasks;
  int ntasks = st.ndtasks;
  unsigned long long* prof = st.prof;
  unsigned long long* trace = nullptr;
  const char* tpath = getenv("BDDC_COOP_TRACE");  // per-task timestamps (diagnostics)
  if (tpath) trace = c.alloc<unsigned long long>((size_t)ntasks * 4);
  if (prof) BDDC_CUDA(cudaMemsetAsync(prof, 0, sizeof(unsigned long long) * 3 * CT_NTYPES, s));
  st.pg.lt = c.lt_defer;
  void* dargs[] = {&fd, &st.pg, (void*)&tasks, &ntasks, &st.ctr, &qhead, &info, &err, &prof, &trace};
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (prof) {
    BDDC_CUDA(cudaEventCreate(&e0));
    BDDC_CUDA(cudaEventCreate(&e1));
    BDDC_CUDA(cudaEventRecord(e0, s));
  }
  BDDC_CUDA(cudaLaunchCooperativeKernel((void*)coop_factor_df_kernel, st.grid_f, 128, dargs, st.smem_f, s));
  BDDC_COUNT();
  int herr = 0;
  BDDC_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, s));
  BDDC_CUDA(cudaStreamSynchronize(s));
  if (herr) throw CudaError("coarse dataflow factorization: dependency wait timed out");
  if (trace) {  // binary: ntasks, then per task DfTask + 4 x u64 (dequeue, ready, end, cta)
    std::vector<DfTask> ht(ntasks);
    std::vector<unsigned long long> tr((size_t)ntasks * 4);
    BDDC_CUDA(cudaMemcpy(ht.data(), tasks, sizeof(DfTask) * ntasks, cudaMemcpyDeviceToHost));
    BDDC_CUDA(cudaMemcpy(tr.data(), trace, sizeof(unsigned long long) * tr.size(), cudaMemcpyDeviceToHost));
    if (FILE* fo = fopen(tpath, "wb")) {
      const int hdr[4] = {ntasks, (int)sizeof(DfTask), kDeps, kSigs};
      fwrite(hdr, sizeof(int), 4, fo);
      fwrite(ht.data(), sizeof(DfTask), ntasks, fo);
      fwrite(tr.data(), sizeof(unsigned long long), tr.size(), fo);
      fclose(fo);
    }
  }
  if (prof) {
    BDDC_CUDA(cudaEventRecord(e1, s));
    BDDC_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    BDDC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    fprintf(stderr, "coop factor (dataflow): %d tasks, %d counters, %.1f us\n", ntasks, st.nctr, ms * 1e3);
    unsigned long long h[3 * CT_NTYPES];
    BDDC_CUDA(cudaMemcpy(h, prof, sizeof(h), cudaMemcpyDeviceToHost));
    const char* nm[CT_NTYPES] = {"EA", "PT", "TS", "X1", "SY", "X2", "W", "LT", "SYG"};
    for (int k = 0; k < CT_NTYPES; ++k)
      if (h[3 * k + 2])
        fprintf(stderr, "  %-3s n=%7llu  wait %8.1f us/CTA  run %8.1f us/CTA  (avg wait %.2f run %.2f us)\n", nm[k],
                h[3 * k + 2], h[3 * k] / 1.9e3 / st.grid_f, h[3 * k + 1] / 1.9e3 / st.grid_f,
                h[3 * k] / 1.9e3 / h[3 * k + 2], h[3 * k + 1] / 1.9e3 / h[3 * k + 2]);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
}

int coarse_solve_error(Ctx& c) {
  if (!c.fp.n_coarse || !c.sched.df_ctr) return 0;
  int e = 0;
  BDDC_CUDA(cudaMemcpyAsync(&e, c.sched.df_ctr + c.sched.n_ctr + 1, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  BDDC_CUDA(cudaStreamSynchronize(c.stream));
  return e;
}

void coop_solve(Ctx& c, const double* rhs, double* sol, cudaStream_t s, const TvArgs* tva, int queue) {
  CoopState& st = g_coop.at(&c);
  FrontDev fd = c.fp.d;
  LevelView lv{c.sched.gat_ptr, c.sched.gat_src};
  double* partial = c.sched.partial;
  double* ybuf = c.sched.ybuf;
  int* cnt = c.sched.red_cnt;
  const LevelSchedule& ls = c.sched;
  int* ctr = ls.df_ctr;
  int* qhead = ctr + ls.n_ctr;
  int* err = qhead + 1;
  const SdTask* tasks = ls.queues.at(queue).first;
  int ntasks = ls.queues.at(queue).second;
  // counters, queue head and the error flag start at zero every launch (a timeout poisons
  // this launch's result only; pcg_solve / bddc_check report it)
  BDDC_CUDA(cudaMemsetAsync(ctr, 0, sizeof(int) * (ls.n_ctr + 2), s));
  unsigned long long* trace = nullptr;
  TvArgs tv{};
  if (tva) tv = *tva;
  void* dargs[] = {&fd, &lv, &st.sp, (void*)&tasks, &ntasks, &ctr, &qhead, &err, (void*)&rhs, (void*)&sol,
                   &partial, &ybuf, &cnt, &tv, &trace};
  BDDC_CUDA(cudaLaunchCooperativeKernel((void*)coop_solve_df_kernel, st.grid_s, 256, dargs, 0, s));
  BDDC_COUNT();
}

}  // namespace bddc
