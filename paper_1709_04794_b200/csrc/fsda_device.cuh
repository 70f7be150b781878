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
//   * The projection rows s = X w (and the X v probe API) are sequential in
//     stored column order: acc = 0.0; acc = acc + term.  Bit-identical to
//     scipy's csr_matvec.
//   * Every other sum — the operator's rows X p and L y included — uses the
//     canonical "R256" tree: a leaf covers <= 256
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
  double sum_z_iter;  // sum(z) of the loop's smoother output, reduced by k_xt_coop's last CTA
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
  // snapshot of one iteration's shift scalars for k_shift_update
  int* upd_mode;    // 0 nothing, 1 sols only (froze this iteration), 3 sols and P
  double* upd_gs;   // gamma_s
  double* upd_zn;   // zeta_next
  double* upd_as;   // alpha_s
  // deferred ("basis") shift updates: P_s = sum_j coef_a[s][j] r_j and
  // sols_s = sum_j coef_c[s][j] r_j over the stored residuals r_0 .. r_K
  double* coef_a;
  double* coef_c;
  long long coef_ld;  // max_iter + 1
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
    ss.pending[s] = 0; ss.flip[s] = 0; ss.upd_mode[s] = 0;
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
template <typename V>
__global__ void k_cg_init(const double* __restrict__ b, V* __restrict__ r,
                          V* __restrict__ p, double* __restrict__ bigp,
                          double* __restrict__ sols, long long d, double* __restrict__ part,
                          long long n_leaf, CgScalars* sc, ShiftState ss, int n_shifts, int basis) {
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
          r[i] = (V)v;
          p[i] = (V)v;
          a = fma(v, v, a);
        }
      }
      a = butterfly(a);
      if (lane == 0) { part[g] = a; __threadfence(); }
    }
  } else if (basis) {
    // P_s = r_0 (= b), sols_s = 0 as coefficient rows
    const int s = blockIdx.y - 1;
    double* A = ss.coef_a + (long long)s * ss.coef_ld;
    double* Cc = ss.coef_c + (long long)s * ss.coef_ld;
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < ss.coef_ld;
         j += (long long)gridDim.x * blockDim.x) {
      A[j] = j == 0 ? 1.0 : 0.0;
      Cc[j] = 0.0;
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

// Orientation dots y.s per shift (sda.py:280), canonical over N with fma
// leaves; blockIdx.y = shift.  Leaf partials only: k_orient_final reduces
// them, one block per shift.
__global__ void k_orient(const signed char* __restrict__ labels, const double* __restrict__ scores,
                         long long n, double* __restrict__ part, long long n_leaf) {
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
    if (lane == 0) part[(long long)s * n_leaf + g] = a;
  }
}

// R256 of shift blockIdx.x's orientation leaves; sets its flip flag.
__global__ void k_orient_final(const double* __restrict__ part, long long n_leaf, ShiftState ss,
                               double* dots_out) {
  __shared__ double smem[257];
  const int s = blockIdx.x;
  const double v = block_reduce_partials(part + (long long)s * n_leaf, n_leaf, smem);
  if (threadIdx.x == 0) {
    ss.flip[s] = (v < 0.0) ? 1 : 0;
    if (dots_out) dots_out[s] = v;
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

// Encoded column indices for K1: hot columns become (slot | 0x80000000).
__global__ void k_encode_cols(const int* __restrict__ cols, const int* __restrict__ hot_slot,
                              int* __restrict__ enc, long long nnz) {
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < nnz;
       j += (long long)gridDim.x * blockDim.x) {
    const int c = cols[j];
    const int s = hot_slot[c];
    enc[j] = s >= 0 ? (int)(0x80000000u | (unsigned)s) : c;
  }
}

// Laplacian: extract the diagonal values and check every off-diagonal is -1.
__global__ void k_laplacian_split(const int* __restrict__ rowptr, const int* __restrict__ cols,
                                  const double* __restrict__ vals, double* __restrict__ diag,
                                  int n, int* err, int row_base) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int lo = rowptr[i], hi = rowptr[i + 1];
  double dv = 0.0;
  if (hi < lo) atomicExch(err, 2);
  for (int jj = lo; jj < hi; ++jj) {
    int c = cols[jj];
    if (jj > lo && c <= cols[jj - 1]) atomicExch(err, 3);
    if (c == i + row_base) dv = vals[jj];
    else if (vals[jj] != -1.0) atomicExch(err, 4);
  }
  diag[i] = dv;
}

}  // namespace fsda
