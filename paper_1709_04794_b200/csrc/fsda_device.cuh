// fsda_device.cuh — sm_100a kernels of the FSDA hot path.
//
// Reference path (all under /root/reference/pkg/src/sdakit):
//   X p        SparseMatrix.matvec            sparse.py:116-121  (scipy csr_matvec)
//   X^T z      SparseMatrix.matvec_transpose  sparse.py:123-134  (scipy csc_matvec)
//   mu         labeled_mean                   sparse.py:258-265
//   X_c^T z    centered_matvec_transpose      sparse.py:274-277
//   M y        apply_smoother                 sda.py:131-140
//   rhs        fsda_solve                     sda.py:297-301 (+ apply_w sda.py:120-128)
//   shifted CG shifted_cg                     krylov.py:168-281
//   ratings    _ratings_from_projection       sda.py:265-284
//
// Arithmetic contract.  The library is compiled with
// -fmad=false, so every `a * b + c` below rounds twice exactly like numpy;
// fma() is written out where the canonical reduction wants it (dot leaves).
//   * Row sums (X p, L y, X W) are sequential in stored column order: one
//     thread per row, acc = 0.0; acc = acc + term.  Bit-identical to scipy.
//   * Every other sum uses the canonical "R256" tree: a leaf covers <= 256
//     consecutive values; lane l of a warp sums values l, l+32, ... from 0.0,
//     then a xor-butterfly 16,8,4,2,1 combines lanes.  More than 256 values:
//     R256 of the leaf partials of consecutive 256-blocks.  The tree depends
//     only on the vector length, never on the launch shape.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fsda {

constexpr unsigned FULL = 0xffffffffu;
constexpr int LEAF = 256;           // values per canonical leaf
constexpr int WARPS_PER_BLOCK = 4;  // leaf-group kernels: 4 warps = 1024 values
constexpr int LEAF_THREADS = 32 * WARPS_PER_BLOCK;

enum Status : int { ST_OK = 0, ST_BREAKDOWN = 2, ST_NONFINITE = 3 };

// Counters for the "last block finishes" pattern, one slot per kernel kind.
enum Counter : int {
  C_SMOOTH = 0, C_DOT = 1, C_UPDATE = 2, C_CLASS = 3, C_APPLYW = 4, C_INIT = 5,
  C_ORIENT = 6, C_SUM = 7, N_COUNTERS = 8
};

// Scalar state of one shifted-CG solve.  Lives in device memory; written only
// by the single "last" block of a kernel, read by later kernels.
struct CgScalars {
  double rr;          // r.r entering the iteration
  double gamma_prev;  // gamma_{i-1}   (krylov.py:202)
  double alpha;       // momentum entering the iteration (krylov.py:203)
  double gamma;       // gamma_i
  double alpha_new;   // rr_new / rr
  double b_norm;
  double thresh;
  double sum_z;       // sum(z) of the current smoother output / apply_w output
  double class_mean1; // apply_w class means (sda.py:126-127)
  double class_mean2;
  double tol;
  long long iter;     // iterations completed
  long long max_iter;
  long long fail_iter;
  int status;
  int finished;
  int n_active;
  int absolute_tol;
  long long body_runs;  // while-loop body executions (safety valve)
  unsigned counters[N_COUNTERS];
};

// Per-shift state, struct-of-arrays (n_shifts each).
struct ShiftState {
  const double* beta;
  double* zeta_prev;
  double* zeta;
  double* zeta_next;
  double* gamma_s;
  double* alpha_s;
  double* resid;
  long long* iters;
  unsigned char* conv;
  int* active;   // still iterating
  int* good;     // good this iteration (zeta_next finite and not underflowed)
  int* pending;  // deferred P update owed from the previous iteration
  int* flip;     // orientation flip (projection phase)
};

// ---------------------------------------------------------------- R256 tree

__device__ __forceinline__ double butterfly(double a) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) a = a + __shfl_xor_sync(FULL, a, off);
  return a;
}

// Butterfly restricted to aligned groups of w lanes (w power of two <= 32).
// For a column with n <= w values this equals the full-warp leaf: the lanes
// >= w of the canonical leaf hold exactly 0.0 and add nothing.
__device__ __forceinline__ double group_butterfly(double a, int w) {
  for (int off = w >> 1; off >= 1; off >>= 1) a = a + __shfl_xor_sync(FULL, a, off);
  return a;
}

// Canonical leaf over src[0..n) (n <= 256) by one warp; result in all lanes.
__device__ __forceinline__ double warp_leaf(const double* src, int n, int lane) {
  double a = 0.0;
  for (int k = lane; k < n; k += 32) a = a + __ldcg(src + k);
  return butterfly(a);
}

// R256 over m partials by one block (any multiple of 32 threads).  Requires
// m <= 65536 (two levels); the host checks vector lengths against this.
// Returns the result to every thread.  smem needs 257 doubles.
__device__ double block_reduce_partials(const double* part, long long m, double* smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (m <= LEAF) {
    if (warp == 0) {
      double r = warp_leaf(part, (int)m, lane);
      if (lane == 0) smem[256] = r;
    }
  } else {
    const int m2 = (int)((m + LEAF - 1) / LEAF);
    for (int g = warp; g < m2; g += nw) {
      long long lo = (long long)g * LEAF;
      int len = (int)min((long long)LEAF, m - lo);
      double r = warp_leaf(part + lo, len, lane);
      if (lane == 0) smem[g] = r;
    }
    __syncthreads();
    if (warp == 0) {
      double a = 0.0;
      for (int k = lane; k < m2; k += 32) a = a + smem[k];
      a = butterfly(a);
      if (lane == 0) smem[256] = a;
    }
  }
  __syncthreads();
  return smem[256];
}

// Last-block detection.  Every writer of a partial must have issued
// __threadfence() before calling this.
__device__ __forceinline__ bool arrive_last(unsigned* counter, unsigned total) {
  __shared__ int am_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned prev = atomicAdd(counter, 1u);
    am_last = (prev == total - 1);
    if (am_last) *counter = 0;  // ready for the next launch
  }
  __syncthreads();
  if (am_last) __threadfence();
  return am_last != 0;
}

__device__ __forceinline__ bool loop_idle(const CgScalars* sc) {
  return sc->finished != 0 || sc->status != ST_OK;
}

// ------------------------------------------------------------- K1: y = X p
// One thread per row, sequential sum in stored column order (scipy order).
// `guard` (nullable): skip when the solve loop is idle (host-loop mode).
__global__ void k_spmv_rows(const int* __restrict__ rowptr, const int* __restrict__ cols,
                            const double* __restrict__ p, double* __restrict__ y, int n_rows,
                            const CgScalars* guard) {
  if (guard && loop_idle(guard)) return;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rows) return;
  int lo = __ldg(rowptr + i), hi = __ldg(rowptr + i + 1);
  double acc = 0.0;
  int jj = lo;
  for (; jj + 4 <= hi; jj += 4) {
    int c0 = __ldg(cols + jj), c1 = __ldg(cols + jj + 1), c2 = __ldg(cols + jj + 2),
        c3 = __ldg(cols + jj + 3);
    double v0 = __ldg(p + c0), v1 = __ldg(p + c1), v2 = __ldg(p + c2), v3 = __ldg(p + c3);
    acc = acc + v0;
    acc = acc + v1;
    acc = acc + v2;
    acc = acc + v3;
  }
  for (; jj < hi; ++jj) acc = acc + __ldg(p + __ldg(cols + jj));
  y[i] = acc;
}

// Dense symmetric operator for fsda_shifted_cg_dense: q = A p, row-major A,
// sequential per row (the device stand-in for LinearOperator.from_dense).
__global__ void k_dense_matvec(const double* __restrict__ a, const double* __restrict__ p,
                               double* __restrict__ q, int dim, const CgScalars* guard) {
  if (guard && loop_idle(guard)) return;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= dim) return;
  const double* row = a + (long long)i * dim;
  double acc = 0.0;
  for (int j = 0; j < dim; ++j) acc = acc + row[j] * p[j];
  q[i] = acc;
}

// --------------------------------------------- K2: z = M y, plus sum(z)
// apply_smoother (sda.py:131-140): masked = y on labeled rows else 0;
//   alpha == 0 -> masked; alpha == 1 -> alpha * (L y); else
//   (1 - alpha) * masked + alpha * (L y).
// L y is sequential over the row's stored columns, the diagonal term
// diag[i] * y[i] at its sorted position, off-diagonals -y[j] (values -1).
// Warp g covers rows [256g, 256g+256) in 8 rounds so that its z values form
// one canonical leaf of sum(z).  part: n_leaf partials.  If `sum_out` is
// non-null the last block writes sum(z) there.
__global__ void k_smoother(const int* __restrict__ lrowptr, const int* __restrict__ lcols,
                           const double* __restrict__ ldiag, const signed char* __restrict__ labels,
                           const double* __restrict__ y, double* __restrict__ z, int n,
                           double alpha, int alpha_mode, double* __restrict__ part, long long n_leaf,
                           CgScalars* sc, int guarded, double* sum_out) {
  if (guarded && loop_idle(sc)) return;
  __shared__ double smem[257];
  const int lane = threadIdx.x & 31;
  const long long g = (long long)blockIdx.x * WARPS_PER_BLOCK + (threadIdx.x >> 5);
  const double one_minus = 1.0 - alpha;
  if (g < n_leaf) {
    double a = 0.0;
    for (int k = 0; k < 8; ++k) {
      long long i = g * LEAF + k * 32 + lane;
      if (i < n) {
        double yi = y[i];
        double masked = labels[i] != 0 ? yi : 0.0;
        double out;
        if (alpha_mode == 0) {
          out = masked;
        } else {
          int lo = __ldg(lrowptr + i), hi = __ldg(lrowptr + i + 1);
          double acc = 0.0;
          for (int jj = lo; jj < hi; ++jj) {
            int c = __ldg(lcols + jj);
            double t = (c == (int)i) ? __ldg(ldiag + i) * yi : -__ldg(y + c);
            acc = acc + t;
          }
          double smoothed = alpha * acc;
          out = (alpha_mode == 1) ? smoothed : one_minus * masked + smoothed;
        }
        z[i] = out;
        a = a + out;
      }
    }
    a = butterfly(a);
    if (lane == 0) { part[g] = a; __threadfence(); }
  }
  if (arrive_last(&sc->counters[C_SMOOTH], gridDim.x)) {
    double s = block_reduce_partials(part, n_leaf, smem);
    if (threadIdx.x == 0) {
      sc->sum_z = s;
      if (sum_out) *sum_out = s;
    }
  }
}

// Generic canonical sum of a vector (used for sum(w) outside the loop and by
// the parity probes).  Writes the result to *out and, if sc, to sc->sum_z.
__global__ void k_vector_sum(const double* __restrict__ v, long long n, double* __restrict__ part,
                             long long n_leaf, CgScalars* sc, double* out) {
  __shared__ double smem[257];
  const int lane = threadIdx.x & 31;
  const long long g = (long long)blockIdx.x * WARPS_PER_BLOCK + (threadIdx.x >> 5);
  if (g < n_leaf) {
    double a = 0.0;
    for (int k = 0; k < 8; ++k) {
      long long i = g * LEAF + k * 32 + lane;
      if (i < n) a = a + v[i];
    }
    a = butterfly(a);
    if (lane == 0) { part[g] = a; __threadfence(); }
  }
  if (arrive_last(&sc->counters[C_SUM], gridDim.x)) {
    double s = block_reduce_partials(part, n_leaf, smem);
    if (threadIdx.x == 0) {
      if (out) *out = s;
      sc->sum_z = s;
    }
  }
}

// ------------------------------------------------------- K3: X^T z on CSC
// Column work plan (built on the host from the CSC column pointer):
//   class w in {1,2,4,8,16}: columns with n_c <= w, 32/w columns per warp;
//   class "warp": 16 < n_c <= 256, one warp per column;
//   heavy: n_c > 256, one warp per 256-entry segment -> segment partial,
//          combined per column by k_xt_heavy.
// Finalization (mode): 0 plain X^T z; 1 centred X^T z - mu * sum_z
// (sparse.py:274-277); 2 labeled mean (X^T z) / ell (sparse.py:258-265).
struct XtPlan {
  const int* colptr;     // D+1
  const int* rows;       // nnz, ascending within each column
  const int* tiny_cols;  // columns of classes 1..16, grouped by class
  long long tiny_off[6]; // class k (w = 1<<k) occupies tiny_cols[tiny_off[k] .. tiny_off[k+1])
  const int* warp_cols;
  long long n_warp_cols;
  const int* seg_col;    // heavy segments: owning column
  const int* seg_start;  // absolute start in rows[]
  long long n_segs;
  const int* heavy_cols; // heavy columns
  const int* heavy_seg0; // first segment index of each heavy column
  const int* heavy_nseg;
  long long n_heavy;
  double* seg_part;      // n_segs partials
  long long warps_tiny[5];  // warps needed per tiny class
  long long warp_base[8];   // prefix over task kinds: 5 tiny classes, warp cols, segments, end
};

__device__ __forceinline__ double xt_finalize(double colsum, int c, int mode, const double* mu,
                                              double sum_z, double inv_scale) {
  if (mode == 1) return colsum - mu[c] * sum_z;
  if (mode == 2) return colsum / inv_scale;
  return colsum;
}

__global__ void k_xt_light(XtPlan pl, const double* __restrict__ z, double* __restrict__ q,
                           int mode, const double* __restrict__ mu, const CgScalars* sc,
                           double ell, int guarded) {
  if (guarded && loop_idle(sc)) return;
  const int lane = threadIdx.x & 31;
  const long long total = pl.warp_base[7];
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  const double sum_z = (mode == 1) ? sc->sum_z : 0.0;
  for (long long t = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < total;
       t += nwarps) {
    if (t < pl.warp_base[5]) {
      int k = 0;
      while (t >= pl.warp_base[k + 1]) ++k;  // tiny class k, w = 1 << k
      const int w = 1 << k;
      const int per = 32 / w;
      long long idx = pl.tiny_off[k] + (t - pl.warp_base[k]) * per + lane / w;
      const int tl = lane & (w - 1);
      double a = 0.0;
      int c = -1;
      if (idx < pl.tiny_off[k + 1]) {
        c = pl.tiny_cols[idx];
        int lo = __ldg(pl.colptr + c), hi = __ldg(pl.colptr + c + 1);
        if (lo + tl < hi) a = a + __ldg(z + __ldg(pl.rows + lo + tl));
      }
      a = group_butterfly(a, w);
      if (c >= 0 && tl == 0) q[c] = xt_finalize(a, c, mode, mu, sum_z, ell);
    } else if (t < pl.warp_base[6]) {
      int c = pl.warp_cols[t - pl.warp_base[5]];
      int lo = __ldg(pl.colptr + c), hi = __ldg(pl.colptr + c + 1);
      double a = 0.0;
      for (int jj = lo + lane; jj < hi; jj += 32) a = a + __ldg(z + __ldg(pl.rows + jj));
      a = butterfly(a);
      if (lane == 0) q[c] = xt_finalize(a, c, mode, mu, sum_z, ell);
    } else {
      long long s = t - pl.warp_base[6];
      int c = pl.seg_col[s];
      int lo = pl.seg_start[s];
      int hi = min(lo + LEAF, __ldg(pl.colptr + c + 1));
      double a = 0.0;
      for (int jj = lo + lane; jj < hi; jj += 32) a = a + __ldg(z + __ldg(pl.rows + jj));
      a = butterfly(a);
      if (lane == 0) pl.seg_part[s] = a;
    }
  }
}

// One block per heavy column: canonical reduction of its segment partials.
__global__ void k_xt_heavy(XtPlan pl, double* __restrict__ q, int mode,
                           const double* __restrict__ mu, const CgScalars* sc, double ell,
                           int guarded) {
  if (guarded && loop_idle(sc)) return;
  __shared__ double smem[257];
  const double sum_z = (mode == 1) ? sc->sum_z : 0.0;
  for (long long h = blockIdx.x; h < pl.n_heavy; h += gridDim.x) {
    int c = pl.heavy_cols[h];
    double s = block_reduce_partials(pl.seg_part + pl.heavy_seg0[h], pl.heavy_nseg[h], smem);
    if (threadIdx.x == 0) q[c] = xt_finalize(s, c, mode, mu, sum_z, ell);
  }
}

// ----------------------------------------- K4a: p.q and the shift scalars
// Leaf partials of p.q (fma leaves); the last block finishes the reduction and
// runs krylov.py:212-229 for every active shift.
__global__ void k_dot_pq(const double* __restrict__ p, const double* __restrict__ q, long long d,
                         double* __restrict__ part, long long n_leaf, CgScalars* sc, ShiftState ss,
                         int n_shifts) {
  if (loop_idle(sc)) return;
  __shared__ double smem[257];
  const int lane = threadIdx.x & 31;
  const long long g = (long long)blockIdx.x * WARPS_PER_BLOCK + (threadIdx.x >> 5);
  if (g < n_leaf) {
    double a = 0.0;
    for (int k = 0; k < 8; ++k) {
      long long i = g * LEAF + k * 32 + lane;
      if (i < d) a = fma(p[i], q[i], a);
    }
    a = butterfly(a);
    if (lane == 0) { part[g] = a; __threadfence(); }
  }
  if (arrive_last(&sc->counters[C_DOT], gridDim.x)) {
    double pq = block_reduce_partials(part, n_leaf, smem);
    if (threadIdx.x == 0) {
      if (!isfinite(pq)) {
        sc->status = ST_NONFINITE; sc->fail_iter = sc->iter; sc->finished = 1;
      } else if (pq == 0.0) {
        sc->status = ST_BREAKDOWN; sc->fail_iter = sc->iter; sc->finished = 1;
      } else {
        const double gamma = -sc->rr / pq;
        const double gp = sc->gamma_prev, al = sc->alpha;
        sc->gamma = gamma;
        for (int s = 0; s < n_shifts; ++s) {
          if (!ss.active[s]) { ss.good[s] = 0; continue; }
          const double zp = ss.zeta_prev[s], z = ss.zeta[s];
          const double denom = gamma * al * (zp - z) + zp * gp * (1.0 - ss.beta[s] * gamma);
          const double zn = zp * z * gp / denom;
          const int bad = !isfinite(zn) || fabs(zn) < 1e-290;
          ss.good[s] = !bad;
          if (!bad) {
            ss.zeta_next[s] = zn;
            ss.gamma_s[s] = gamma * zn / z;
          }
        }
      }
    }
  }
}

// ---------------------------------- K4b: shift updates, r update, r.r
// blockIdx.y == 0: r_next = r + gamma q, leaf partials of r_next.r_next.
// blockIdx.y == s+1: for a good shift, the deferred P update owed from the
//   previous iteration (krylov.py:241), then sols -= P * gamma_s (krylov.py:230).
// The last block runs krylov.py:233-268 (freeze / retire / roll).
__global__ void k_update(const double* __restrict__ q, double* __restrict__ r0,
                         double* __restrict__ r1, double* __restrict__ bigp,
                         double* __restrict__ sols, long long d, double* __restrict__ part,
                         long long n_leaf, CgScalars* sc, ShiftState ss, int n_shifts) {
  if (loop_idle(sc)) return;
  __shared__ double smem[257];
  const int lane = threadIdx.x & 31;
  const long long g = (long long)blockIdx.x * WARPS_PER_BLOCK + (threadIdx.x >> 5);
  // r ping-pongs between r0/r1 by iteration parity so the shift blocks can
  // read r_i while block row 0 writes r_{i+1}.
  const double* r_cur = (sc->iter & 1) ? r1 : r0;
  double* r_next = (sc->iter & 1) ? r0 : r1;
  if (blockIdx.y == 0) {
    const double gamma = sc->gamma;
    if (g < n_leaf) {
      double a = 0.0;
      for (int k = 0; k < 8; ++k) {
        long long i = g * LEAF + k * 32 + lane;
        if (i < d) {
          double rn = r_cur[i] + gamma * q[i];
          r_next[i] = rn;
          a = fma(rn, rn, a);
        }
      }
      a = butterfly(a);
      if (lane == 0) { part[g] = a; __threadfence(); }
    }
  } else {
    const int s = blockIdx.y - 1;
    if (ss.active[s] && ss.good[s] && g < n_leaf) {
      const double gs = ss.gamma_s[s];
      const int pend = ss.pending[s];
      const double zc = ss.zeta[s], as = ss.alpha_s[s];
      double* P = bigp + (long long)s * d;
      double* X = sols + (long long)s * d;
      for (int k = 0; k < 8; ++k) {
        long long i = g * LEAF + k * 32 + lane;
        if (i < d) {
          double pv = P[i];
          if (pend) {
            pv = zc * r_cur[i] + as * pv;
            P[i] = pv;
          }
          X[i] = X[i] - pv * gs;
        }
      }
    }
  }
  if (arrive_last(&sc->counters[C_UPDATE], gridDim.x * gridDim.y)) {
    double rr_new = block_reduce_partials(part, n_leaf, smem);
    if (threadIdx.x == 0) {
      const long long i = sc->iter;
      if (!isfinite(rr_new)) {
        sc->status = ST_NONFINITE; sc->fail_iter = i; sc->finished = 1;
      } else {
        const double r_norm = sqrt(rr_new);
        const double gamma = sc->gamma;
        const double alpha_new = rr_new / sc->rr;
        int n_active = 0;
        for (int s = 0; s < n_shifts; ++s) {
          if (!ss.active[s]) continue;
          if (!ss.good[s]) {  // degenerate zeta: freeze untouched (krylov.py:251-255)
            ss.iters[s] = i + 1; ss.resid[s] = __longlong_as_double(0x7ff0000000000000LL);
            ss.active[s] = 0; ss.pending[s] = 0;
            continue;
          }
          const double zn = ss.zeta_next[s], z = ss.zeta[s], gs = ss.gamma_s[s];
          ss.alpha_s[s] = alpha_new * (zn * gs) / (z * gamma);
          const double shift_res = fabs(zn) * r_norm;
          if (shift_res < sc->thresh) {  // converged: freeze (krylov.py:256-261)
            ss.iters[s] = i + 1; ss.resid[s] = shift_res; ss.conv[s] = 1;
            ss.active[s] = 0; ss.pending[s] = 0;
          } else {
            ss.zeta_prev[s] = z;
            ss.zeta[s] = zn;
            ss.pending[s] = 1;
            ++n_active;
          }
        }
        sc->gamma_prev = gamma;
        sc->alpha = alpha_new;
        sc->alpha_new = alpha_new;
        sc->rr = rr_new;
        sc->iter = i + 1;
        sc->n_active = n_active;
        if (n_active == 0 || i + 1 >= sc->max_iter) sc->finished = 1;
      }
    }
  }
}

// K4c: p = r + alpha_new p (krylov.py:239), and the while-loop condition.
__global__ void k_pupdate(const double* __restrict__ r0, const double* __restrict__ r1,
                          double* __restrict__ p, long long d, const CgScalars* sc,
                          unsigned long long cond_handle, int use_cond) {
  if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) {
    CgScalars* w = const_cast<CgScalars*>(sc);
    const long long runs = ++w->body_runs;
    unsigned keep = (sc->finished == 0 && sc->status == ST_OK) ? 1u : 0u;
    if (runs > sc->max_iter + 1) keep = 0u;  // never spin past the iteration budget
    cudaGraphSetConditional((cudaGraphConditionalHandle)cond_handle, keep);
  }
  if (sc->status != ST_OK) return;
  // When the base loop just finished the direction is never used again, but
  // computing it is harmless and keeps the kernel branch-free.
  const double a = sc->alpha_new;
  const double* r = (sc->iter & 1) ? r1 : r0;  // r_{i+1}; iter was advanced by k_update
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < d;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = r[i] + a * p[i];
}

// ------------------------------------------------------------ solve setup

// Reset scalars + per-shift state for a new solve.
__global__ void k_solve_reset(CgScalars* sc, ShiftState ss, int n_shifts, long long max_iter,
                              double tol, int absolute_tol) {
  int t = threadIdx.x;
  if (t == 0) {
    sc->rr = 0.0; sc->gamma_prev = 1.0; sc->alpha = 0.0; sc->gamma = 0.0; sc->alpha_new = 0.0;
    sc->b_norm = 0.0; sc->thresh = 0.0; sc->sum_z = 0.0;
    sc->iter = 0; sc->max_iter = max_iter; sc->fail_iter = -1; sc->status = ST_OK;
    sc->finished = 0; sc->n_active = n_shifts; sc->tol = tol; sc->absolute_tol = absolute_tol;
    sc->body_runs = 0;
    for (int k = 0; k < N_COUNTERS; ++k) sc->counters[k] = 0;
  }
  for (int s = t; s < n_shifts; s += blockDim.x) {
    ss.zeta_prev[s] = 1.0; ss.zeta[s] = 1.0; ss.zeta_next[s] = 1.0;
    ss.gamma_s[s] = 0.0; ss.alpha_s[s] = 0.0; ss.resid[s] = 0.0;
    ss.iters[s] = max_iter; ss.conv[s] = 0; ss.active[s] = 1; ss.good[s] = 0;
    ss.pending[s] = 0; ss.flip[s] = 0;
  }
}

// Indicator of labeled rows as doubles (the reference's mask_labeled.astype).
__global__ void k_indicator(const signed char* __restrict__ labels, double* __restrict__ out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = labels[i] != 0 ? 1.0 : 0.0;
}

// apply_w part 1 (sda.py:126-127): class sums of t, canonical over N with
// zeros off-class; the last block stores the class means.
__global__ void k_class_sums(const double* __restrict__ t, const signed char* __restrict__ labels,
                             long long n, double* __restrict__ part, long long n_leaf,
                             CgScalars* sc, double n1, double n2) {
  __shared__ double smem[257];
  const int lane = threadIdx.x & 31;
  const long long g = (long long)blockIdx.x * WARPS_PER_BLOCK + (threadIdx.x >> 5);
  if (g < n_leaf) {
    double a1 = 0.0, a2 = 0.0;
    for (int k = 0; k < 8; ++k) {
      long long i = g * LEAF + k * 32 + lane;
      if (i < n) {
        signed char l = labels[i];
        double v = t[i];
        a1 = a1 + (l == 1 ? v : 0.0);
        a2 = a2 + (l == -1 ? v : 0.0);
      }
    }
    a1 = butterfly(a1);
    a2 = butterfly(a2);
    if (lane == 0) { part[g] = a1; part[n_leaf + g] = a2; __threadfence(); }
  }
  if (arrive_last(&sc->counters[C_CLASS], gridDim.x)) {
    double s1 = block_reduce_partials(part, n_leaf, smem);
    double s2 = block_reduce_partials(part + n_leaf, n_leaf, smem);
    if (threadIdx.x == 0) {
      sc->class_mean1 = s1 / n1;
      sc->class_mean2 = s2 / n2;
    }
  }
}

// apply_w part 2: broadcast class means, plus sum(w) (sparse.py:277).
__global__ void k_apply_w(const signed char* __restrict__ labels, double* __restrict__ w,
                          long long n, double* __restrict__ part, long long n_leaf,
                          CgScalars* sc) {
  __shared__ double smem[257];
  const int lane = threadIdx.x & 31;
  const long long g = (long long)blockIdx.x * WARPS_PER_BLOCK + (threadIdx.x >> 5);
  const double c1 = sc->class_mean1, c2 = sc->class_mean2;
  if (g < n_leaf) {
    double a = 0.0;
    for (int k = 0; k < 8; ++k) {
      long long i = g * LEAF + k * 32 + lane;
      if (i < n) {
        signed char l = labels[i];
        double v = l == 1 ? c1 : (l == -1 ? c2 : 0.0);
        w[i] = v;
        a = a + v;
      }
    }
    a = butterfly(a);
    if (lane == 0) { part[g] = a; __threadfence(); }
  }
  if (arrive_last(&sc->counters[C_APPLYW], gridDim.x)) {
    double s = block_reduce_partials(part, n_leaf, smem);
    if (threadIdx.x == 0) sc->sum_z = s;
  }
}

// Shifted-CG initialisation (krylov.py:185-208): b_norm, threshold, rr, and
// r = p = b, P_s = b, sols = 0.  blockIdx.y == 0: r/p + b.b leaves;
// blockIdx.y == s+1: shift s.
__global__ void k_cg_init(const double* __restrict__ b, double* __restrict__ r,
                          double* __restrict__ p, double* __restrict__ bigp,
                          double* __restrict__ sols, long long d, double* __restrict__ part,
                          long long n_leaf, CgScalars* sc, ShiftState ss, int n_shifts) {
  __shared__ double smem[257];
  const int lane = threadIdx.x & 31;
  const long long g = (long long)blockIdx.x * WARPS_PER_BLOCK + (threadIdx.x >> 5);
  if (blockIdx.y == 0) {
    if (g < n_leaf) {
      double a = 0.0;
      for (int k = 0; k < 8; ++k) {
        long long i = g * LEAF + k * 32 + lane;
        if (i < d) {
          double v = b[i];
          r[i] = v;
          p[i] = v;
          a = fma(v, v, a);
        }
      }
      a = butterfly(a);
      if (lane == 0) { part[g] = a; __threadfence(); }
    }
  } else {
    const int s = blockIdx.y - 1;
    if (g < n_leaf) {
      double* P = bigp + (long long)s * d;
      double* X = sols + (long long)s * d;
      for (int k = 0; k < 8; ++k) {
        long long i = g * LEAF + k * 32 + lane;
        if (i < d) { P[i] = b[i]; X[i] = 0.0; }
      }
    }
  }
  if (arrive_last(&sc->counters[C_INIT], gridDim.x * gridDim.y)) {
    double bb = block_reduce_partials(part, n_leaf, smem);
    if (threadIdx.x == 0) {
      const double b_norm = sqrt(bb);
      sc->b_norm = b_norm;
      sc->rr = b_norm * b_norm;
      sc->thresh = sc->absolute_tol ? sc->tol : sc->tol * b_norm;
      if (b_norm == 0.0) {  // krylov.py:188-194: zero solutions, all converged
        for (int s = 0; s < n_shifts; ++s) {
          ss.iters[s] = 0; ss.resid[s] = 0.0; ss.conv[s] = 1; ss.active[s] = 0;
        }
        sc->n_active = 0;
        sc->finished = 1;
      } else if (sc->max_iter <= 0) {
        sc->finished = 1;
      }
    }
  }
}

// After the loop: shifts still active report |zeta| * sqrt(rr) (krylov.py:272-275).
__global__ void k_cg_finish(CgScalars* sc, ShiftState ss, int n_shifts) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (sc->status != ST_OK) return;
  const double rn = sqrt(sc->rr);
  for (int s = 0; s < n_shifts; ++s) {
    if (ss.active[s]) {
      ss.iters[s] = sc->max_iter;
      ss.resid[s] = fabs(ss.zeta[s]) * rn;
    }
  }
}

// ------------------------------------------------------- projection phase

// W[c * ns + s] = sols[s * D + c]: feature-major copy for the score SpMM.
__global__ void k_transpose_sols(const double* __restrict__ sols, double* __restrict__ w,
                                 long long d, int ns) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= d * ns) return;
  long long c = t / ns;
  int s = (int)(t - c * ns);
  w[t] = sols[(long long)s * d + c];
}

// scores[s * N + i] = sum over row i of W[c * ns + s], sequential in stored
// column order (what scipy does for each x.matvec(w), sda.py:279).
template <int CH>
__global__ void k_spmm_scores(const int* __restrict__ rowptr, const int* __restrict__ cols,
                              const double* __restrict__ w, double* __restrict__ scores,
                              int n_rows, int ns) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rows) return;
  int lo = __ldg(rowptr + i), hi = __ldg(rowptr + i + 1);
  for (int s0 = 0; s0 < ns; s0 += CH) {
    double acc[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) acc[k] = 0.0;
    const int m = min(CH, ns - s0);
    for (int jj = lo; jj < hi; ++jj) {
      const double* wr = w + (long long)__ldg(cols + jj) * ns + s0;
#pragma unroll
      for (int k = 0; k < CH; ++k)
        if (k < m) acc[k] = acc[k] + __ldg(wr + k);
    }
#pragma unroll
    for (int k = 0; k < CH; ++k)
      if (k < m) scores[(long long)(s0 + k) * n_rows + i] = acc[k];
  }
}

// Orientation dots y.s per shift (sda.py:280), canonical over N with fma
// leaves; blockIdx.y = shift.  The last block sets the flip flags.
__global__ void k_orient(const signed char* __restrict__ labels, const double* __restrict__ scores,
                         long long n, double* __restrict__ part, long long n_leaf, CgScalars* sc,
                         ShiftState ss, int ns) {
  __shared__ double smem[257];
  const int lane = threadIdx.x & 31;
  const long long g = (long long)blockIdx.x * WARPS_PER_BLOCK + (threadIdx.x >> 5);
  const int s = blockIdx.y;
  if (g < n_leaf) {
    const double* sv = scores + (long long)s * n;
    double a = 0.0;
    for (int k = 0; k < 8; ++k) {
      long long i = g * LEAF + k * 32 + lane;
      if (i < n) a = fma((double)labels[i], sv[i], a);
    }
    a = butterfly(a);
    if (lane == 0) { part[(long long)s * n_leaf + g] = a; __threadfence(); }
  }
  if (arrive_last(&sc->counters[C_ORIENT], gridDim.x * gridDim.y)) {
    for (int t = 0; t < ns; ++t) {
      double v = block_reduce_partials(part + (long long)t * n_leaf, n_leaf, smem);
      if (threadIdx.x == 0) ss.flip[t] = (v < 0.0) ? 1 : 0;
    }
  }
}

// Negate flipped shifts' scores and directions.
__global__ void k_flip(double* __restrict__ scores, double* __restrict__ sols, long long n,
                       long long d, ShiftState ss) {
  const int s = blockIdx.y;
  if (!ss.flip[s]) return;
  long long lim = n > d ? n : d;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < lim;
       i += (long long)gridDim.x * blockDim.x) {
    if (scores && i < n) scores[(long long)s * n + i] = -scores[(long long)s * n + i];
    if (i < d) sols[(long long)s * d + i] = -sols[(long long)s * d + i];
  }
}

// ------------------------------------------------------------ upload side

// int64 -> int32 narrowing with range validation.  err receives a non-zero
// code on the first violation.
__global__ void k_narrow_idx(const long long* __restrict__ in, int* __restrict__ out, long long n,
                             long long limit, int* err) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    long long v = in[i];
    if (v < 0 || v > limit) atomicExch(err, 1);
    out[i] = (int)v;
  }
}

// Row id of every nonzero (CSC construction input), and strict column order
// validation inside rows.
__global__ void k_row_ids(const int* __restrict__ rowptr, const int* __restrict__ cols,
                          int* __restrict__ row_of, int n_rows, int* err) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rows) return;
  int lo = rowptr[i], hi = rowptr[i + 1];
  if (hi < lo) { atomicExch(err, 2); return; }
  for (int jj = lo; jj < hi; ++jj) {
    row_of[jj] = i;
    if (jj > lo && cols[jj] <= cols[jj - 1]) atomicExch(err, 3);
  }
}

// colptr[c] = first position of column c in the column-sorted key array.
__global__ void k_colptr_from_sorted(const int* __restrict__ sorted_cols, long long nnz,
                                     int* __restrict__ colptr, int n_cols) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > n_cols) return;
  long long lo = 0, hi = nnz;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if (sorted_cols[mid] < c) lo = mid + 1; else hi = mid;
  }
  colptr[c] = (int)lo;
}

// Laplacian: extract the diagonal values and check every off-diagonal is -1.
__global__ void k_laplacian_split(const int* __restrict__ rowptr, const int* __restrict__ cols,
                                  const double* __restrict__ vals, double* __restrict__ diag,
                                  int n, int* err) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int lo = rowptr[i], hi = rowptr[i + 1];
  double dv = 0.0;
  for (int jj = lo; jj < hi; ++jj) {
    int c = cols[jj];
    if (jj > lo && c <= cols[jj - 1]) atomicExch(err, 3);
    if (c == i) dv = vals[jj];
    else if (vals[jj] != -1.0) atomicExch(err, 4);
  }
  diag[i] = dv;
}

}  // namespace fsda
