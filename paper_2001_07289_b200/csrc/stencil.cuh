// Matrix-free element-by-element operator on the structured grid.
//
// (A x)[g] = sum over the 2^d cells c containing node g of alpha_c * sum_t K[s][t] x[c + t],
// with s = g - c the node's corner in c and x = 0 on Dirichlet nodes. This is the
// assembled operator of mesh.py:172-198 applied without storing it: 8 B of alpha per cell
// plus the x / y streams, instead of 12 B per CSR nonzero.
#pragma once
#include "bddc_internal.cuh"

namespace bddc {

__device__ __forceinline__ long long free_id(const Geometry& G, int g0, int g1, int g2) {
  return (long long)(g0 - 1) + (long long)G.nfree[0] * ((g1 - 1) + (long long)G.nfree[1] * (g2 - 1));
}

__device__ __forceinline__ long long cell_id(const Geometry& G, int c0, int c1, int c2) {
  return (long long)c0 + (long long)G.cells[0] * (c1 + (long long)G.cells[1] * c2);
}

__device__ __forceinline__ void free_coords(const Geometry& G, long long f, int& g0, int& g1,
                                            int& g2) {
  if (G.n < (1LL << 31)) {  // 32-bit division (the 64-bit one is a long software sequence)
    unsigned u = (unsigned)f;
    const unsigned q = u / (unsigned)G.nfree[0];
    g0 = (int)(u - q * (unsigned)G.nfree[0]) + 1;
    if (G.dim == 3) {
      const unsigned q2 = q / (unsigned)G.nfree[1];
      g1 = (int)(q - q2 * (unsigned)G.nfree[1]) + 1;
      g2 = (int)q2 + 1;
    } else {
      g1 = (int)q + 1;
      g2 = 0;
    }
    return;
  }
  g0 = (int)(f % G.nfree[0]) + 1;
  f /= G.nfree[0];
  if (G.dim == 3) {
    g1 = (int)(f % G.nfree[1]) + 1;
    g2 = (int)(f / G.nfree[1]) + 1;
  } else {
    g1 = (int)f + 1;
    g2 = 0;
  }
}

// Row g of A applied to x with 32-bit index arithmetic (cell and free-dof counts < 2^31):
// the neighbour offsets are compile-time after unrolling, so each load is base + constant.
template <int DIM>
__device__ __forceinline__ double stencil_row32(const Geometry& G, const double* __restrict__ alpha,
                                                const double* __restrict__ x, int g0, int g1, int g2) {
  constexpr int NPE = 1 << DIM;
  const int c0n = G.cells[0], c1n = G.cells[1], nf0 = G.nfree[0], nf1 = G.nfree[1];
  const int fg = (g0 - 1) + nf0 * ((g1 - 1) + (DIM == 3 ? nf1 * (g2 - 1) : 0));
  const int cg = g0 + c0n * (g1 + (DIM == 3 ? c1n * g2 : 0));
  double acc = 0.0;
#pragma unroll
  for (int s = 0; s < NPE; ++s) {
    const int sx = s & 1, sy = (s >> 1) & 1, sz = DIM == 3 ? (s >> 2) & 1 : 0;
    const double a = __ldg(alpha + (cg - sx - c0n * (sy + (DIM == 3 ? c1n * sz : 0))));
    double part = 0.0;
#pragma unroll
    for (int t = 0; t < NPE; ++t) {
      const double k = G.K[s * NPE + t];
      if (k == 0.0) continue;
      const int dx = (t & 1) - sx, dy = ((t >> 1) & 1) - sy, dz = DIM == 3 ? ((t >> 2) & 1) - sz : 0;
      if ((dx && (g0 + dx == 0 || g0 + dx == c0n)) || (dy && (g1 + dy == 0 || g1 + dy == c1n))) continue;
      if (DIM == 3 && dz && (g2 + dz == 0 || g2 + dz == G.cells[2])) continue;
      part += k * __ldg(x + (fg + dx + nf0 * (dy + (DIM == 3 ? nf1 * dz : 0))));
    }
    acc += a * part;
  }
  return acc;
}

// Row g of A applied to x (g is a free node).
template <int DIM>
__device__ __forceinline__ double stencil_row(const Geometry& G, const double* __restrict__ alpha,
                                              const double* __restrict__ x, int g0, int g1,
                                              int g2) {
  if (G.n < (1LL << 30)) return stencil_row32<DIM>(G, alpha, x, g0, g1, g2);
  constexpr int NPE = 1 << DIM;
  double acc = 0.0;
#pragma unroll
  for (int s = 0; s < NPE; ++s) {
    const int c0 = g0 - (s & 1), c1 = g1 - ((s >> 1) & 1), c2 = DIM == 3 ? g2 - ((s >> 2) & 1) : 0;
    const double a = __ldg(alpha + cell_id(G, c0, c1, c2));
    double part = 0.0;
#pragma unroll
    for (int t = 0; t < NPE; ++t) {
      const double k = G.K[s * NPE + t];
      if (k == 0.0) continue;
      const int n0 = c0 + (t & 1), n1 = c1 + ((t >> 1) & 1), n2 = DIM == 3 ? c2 + ((t >> 2) & 1) : 1;
      if (n0 == 0 || n0 == G.cells[0] || n1 == 0 || n1 == G.cells[1]) continue;
      if (DIM == 3 && (n2 == 0 || n2 == G.cells[2])) continue;
      part += k * __ldg(x + free_id(G, n0, n1, DIM == 3 ? n2 : 1));
    }
    acc += a * part;
  }
  return acc;
}

// ---- plane-marching sweep of the operator over the rank's active rows --------------------
// A thread owns one column of nodes (fixed g0 [, g1]) over kSweepChunk consecutive rows of the
// last axis and keeps the 3^d window of x and the 2^d cell coefficients around its node in
// registers: marching one row loads 3^(d-1) x values and 2^(d-1) coefficients (P1: only the
// axis neighbours survive) instead of the 2^d (1 + nonzeros) loads of stencil_row. The row
// value is accumulated in stencil_row's order (cells s ascending, nodes t ascending, zero
// K entries and Dirichlet neighbours contributing exact zeros), so it is the same number.
// EDGE: K(s, t) != 0 only for t = s or t an axis neighbour of s (P1 Kuhn; checked on the host).
constexpr int kSweepChunk = 16;

__host__ __device__ inline bool stencil_edge_only(const Geometry& G) {
  for (int s = 0; s < G.npe; ++s)
    for (int t = 0; t < G.npe; ++t) {
      const int d = s ^ t;
      if ((d & (d - 1)) != 0 && G.K[s * G.npe + t] != 0.0) return false;
    }
  return true;
}

// work items of a sweep over the rank's active rows
inline long long sweep_items(const Geometry& G) {
  const long long ncol = G.dim == 3 ? (long long)G.nfree[0] * G.nfree[1] : G.nfree[0];
  const long long rows = (G.f_hi - G.f_lo) / ncol;
  return ncol * ((rows + kSweepChunk - 1) / kSweepChunk);
}

// emit(f, v, xc): row f, v = (A x)[f], xc = x[f]
template <int DIM, bool EDGE, class F>
__device__ __forceinline__ void stencil_sweep(const Geometry& G, const double* __restrict__ alpha,
                                              const double* __restrict__ x, F&& emit) {
  constexpr int NPE = 1 << DIM;
  constexpr int NY = DIM == 3 ? 3 : 1;   // window extent along axis 1 for DIM == 3
  const int nf0 = G.nfree[0], c0n = G.cells[0];
  const int nf1 = DIM == 3 ? G.nfree[1] : 1, c1n = G.cells[1];
  const int ncol = nf0 * nf1;                      // nodes per row of the last axis
  const int clast = G.cells[DIM - 1];
  const int L_lo = (int)(G.f_lo / ncol), L_hi = (int)(G.f_hi / ncol);  // free rows [L_lo, L_hi)
  const int nchunk = (L_hi - L_lo + kSweepChunk - 1) / kSweepChunk;
  const long long items = (long long)ncol * nchunk;
  const long long cstride = DIM == 3 ? (long long)c0n * c1n : c0n;  // cells per layer of the last axis
  for (long long item = blockIdx.x * (long long)blockDim.x + threadIdx.x; item < items;
       item += (long long)gridDim.x * blockDim.x) {
    const int col = (int)(item % ncol), chunk = (int)(item / ncol);
    const int g0 = col % nf0 + 1, g1 = DIM == 3 ? col / nf0 + 1 : 0;
    const int za = L_lo + chunk * kSweepChunk, zb = min(za + kSweepChunk, L_hi);
    const bool xok[3] = {g0 > 1, true, g0 < c0n - 1};
    const bool yok[3] = {DIM == 3 ? g1 > 1 : true, true, DIM == 3 ? g1 < c1n - 1 : true};
    // window: w[dl][dy][dx] = x(g + (dx-1, dy-1, dl-1)); a[sl][sy][sx] = alpha(cell g - s)
    double w[3][NY][3], a[2][DIM == 3 ? 2 : 1][2];
    auto load_row = [&](double (&dst)[NY][3], int z) {  // free row z of the last axis
      const bool zok = z >= 0 && z + 1 < clast;
      const double* xb = x + ((long long)z * ncol + col);
#pragma unroll
      for (int dy = 0; dy < NY; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
          const int yy = DIM == 3 ? dy : 1;
          const bool ok = zok && xok[dx] && yok[yy];
          dst[dy][dx] = ok ? __ldg(xb + (dx - 1) + nf0 * (DIM == 3 ? dy - 1 : 0)) : 0.0;
        }
    };
    auto load_cells = [&](double (&dst)[DIM == 3 ? 2 : 1][2], int cl) {  // cell layer cl of the last axis
      const double* ab = alpha + (cl * cstride + (DIM == 3 ? (long long)g1 * c0n : 0) + g0);
#pragma unroll
      for (int sy = 0; sy < (DIM == 3 ? 2 : 1); ++sy)
#pragma unroll
        for (int sx = 0; sx < 2; ++sx) dst[sy][sx] = __ldg(ab - sx - (DIM == 3 ? sy * c0n : 0));
    };
    load_row(w[0], za - 1);
    load_row(w[1], za);
    load_cells(a[1], za);  // node coordinate = za + 1: the layer below it is cell layer za
    load_row(w[2], za + 1);
    load_cells(a[0], za + 1);
    for (int z = za; z < zb; ++z) {
      // the next row's upper neighbours and cells are requested before this row is computed
      // (one row of loads in flight per thread: the sweep is bound by memory-level parallelism)
      double nw[NY][3], na[DIM == 3 ? 2 : 1][2];
      if (z + 1 < zb) {
        load_row(nw, z + 2);
        load_cells(na, z + 2);
      }
      double acc = 0.0;
#pragma unroll
      for (int s = 0; s < NPE; ++s) {
        const int sx = s & 1, sy = DIM == 3 ? (s >> 1) & 1 : 0, sl = (s >> (DIM - 1)) & 1;
        double part = 0.0;
#pragma unroll
        for (int t = 0; t < NPE; ++t) {
          if (EDGE && ((s ^ t) & ((s ^ t) - 1)) != 0) continue;
          const int tx = t & 1, ty = DIM == 3 ? (t >> 1) & 1 : 0, tl = (t >> (DIM - 1)) & 1;
          part += G.K[s * NPE + t] * w[1 + tl - sl][DIM == 3 ? 1 + ty - sy : 0][1 + tx - sx];
        }
        acc += a[sl][sy][sx] * part;
      }
      emit((long long)z * ncol + col, acc, w[1][DIM == 3 ? 1 : 0][1]);
#pragma unroll
      for (int dy = 0; dy < NY; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
          w[0][dy][dx] = w[1][dy][dx];
          w[1][dy][dx] = w[2][dy][dx];
          w[2][dy][dx] = nw[dy][dx];
        }
#pragma unroll
      for (int sy = 0; sy < (DIM == 3 ? 2 : 1); ++sy)
#pragma unroll
        for (int sx = 0; sx < 2; ++sx) {
          a[1][sy][sx] = a[0][sy][sx];
          a[0][sy][sx] = na[sy][sx];
        }
    }
  }
}

// Coefficient A_i(a, a + d) of subdomain p's local Neumann matrix (local node coords a),
// summing only cells of the subdomain box (bddc.py:427 via assemble_cells).
template <int DIM>
__device__ __forceinline__ double local_coef(const Geometry& G, const double* __restrict__ alpha,
                                             const int p[3], const int a[3], const int d[3]) {
  constexpr int NPE = 1 << DIM;
  double acc = 0.0;
  // candidate cell offsets per axis: d=0 -> {a-1, a}; d=1 -> {a}; d=-1 -> {a-1}
#pragma unroll
  for (int s = 0; s < NPE; ++s) {
    int cc[3] = {0, 0, 0};
    bool ok = true;
#pragma unroll
    for (int ax = 0; ax < DIM; ++ax) {
      const int bit = (s >> ax) & 1;  // 1: cell below the node on this axis
      if (d[ax] == 1 && bit) ok = false;
      if (d[ax] == -1 && !bit) ok = false;
      cc[ax] = a[ax] - bit;
      if (cc[ax] < 0 || cc[ax] >= G.blk[ax]) ok = false;
    }
    if (!ok) continue;
    int ca = 0, cb = 0;
#pragma unroll
    for (int ax = 0; ax < DIM; ++ax) {
      ca |= ((s >> ax) & 1) << ax;
      cb |= (a[ax] + d[ax] - cc[ax]) << ax;
    }
    const double k = G.K[ca * NPE + cb];
    if (k == 0.0) continue;
    const long long cid = cell_id(G, p[0] * G.blk[0] + cc[0], p[1] * G.blk[1] + cc[1],
                                  DIM == 3 ? p[2] * G.blk[2] + cc[2] : 0);
    acc += __ldg(alpha + cid) * k;
  }
  return acc;
}

__device__ __forceinline__ void sub_coords(const Geometry& G, int sub, int p[3]) {
  p[0] = sub % G.subs[0];
  p[1] = (sub / G.subs[0]) % G.subs[1];
  p[2] = G.dim == 3 ? sub / (G.subs[0] * G.subs[1]) : 0;
}

__device__ __forceinline__ void local_coords(const Geometry& G, int node, int a[3]) {
  a[0] = node % (G.blk[0] + 1);
  a[1] = (node / (G.blk[0] + 1)) % (G.blk[1] + 1);
  a[2] = G.dim == 3 ? node / ((G.blk[0] + 1) * (G.blk[1] + 1)) : 0;
}

// Global free dof of local node a of subdomain p, or -1 if it is a Dirichlet node.
__device__ __forceinline__ long long local_to_free(const Geometry& G, const int p[3],
                                                   const int a[3]) {
  const int g0 = p[0] * G.blk[0] + a[0], g1 = p[1] * G.blk[1] + a[1];
  if (g0 == 0 || g0 == G.cells[0] || g1 == 0 || g1 == G.cells[1]) return -1;
  int g2 = 1;
  if (G.dim == 3) {
    g2 = p[2] * G.blk[2] + a[2];
    if (g2 == 0 || g2 == G.cells[2]) return -1;
  }
  return free_id(G, g0, g1, g2);
}

}  // namespace bddc
