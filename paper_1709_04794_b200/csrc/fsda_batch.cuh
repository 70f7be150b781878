// fsda_batch.cuh — T FSDA sweeps on one X and one graph in a single pass per
// operator product (cfg4: the per-fold solves of
// evaluation.py:110-123 / nested_cv, which share X and L and differ only in
// their label mask and probe).
//
// Layout: every per-task vector is stored task-minor, v[i * TP + t], with
// TP = 32 * G (tasks padded to whole warps).  A warp owns 32 tasks — lane t
// is task 32 g + t — so each gathered row of P, Y or Z is one coalesced
// 256-byte load for 32 tasks instead of 32 separate 32-byte sectors.
//
// Arithmetic: each lane reproduces, for its own task, exactly the canonical
// tree of the single-task kernels (fsda_device.cuh / fsda_hot.cuh): a leaf of
// <= 256 values is accumulated in 32 registers A[l] = sum_k v[l + 32 k]
// (from 0.0, in k order; fma for dot leaves) and folded by the xor-butterfly
// order 16, 8, 4, 2, 1 (tree32).  Sums of more than 256 values are trees of
// leaf sums, as in R256.  Every task's result is therefore bit-identical to
// the single-task solve of the same label mask and probe (fsda_set_label_mask
// + fsda_solve), which tests/test_gpu_batch.py checks.
#pragma once

namespace fsda {

constexpr int BG = 32;  // tasks per group (one per lane)
#ifndef GATHER_MLP
#define GATHER_MLP 8        // row gathers in flight per lane (16: same speed, spills)
#endif
// minimum CTAs per SM (register caps) of the batch gather kernels
#ifndef KB_XROWS_MINB
#define KB_XROWS_MINB 4
#endif
#ifndef KB_LROWS_MINB
#define KB_LROWS_MINB 4
#endif
#ifndef KB_ROWS_F32_EXTRA
#define KB_ROWS_F32_EXTRA 1   // fp32 storage: the row kernels fit 5 CTAs per SM (measured 3 % faster)
#endif
#ifndef KB_COLS_MINB
#define KB_COLS_MINB 4
#endif
#ifndef F32_LS
#define F32_LS 4            // fp32 storage: lane pairs in flight per step (8 spills at 64 registers)
#endif

// Per-task scalars (index t) and per-(task, shift) state (index t * ns + s).
struct BatchState {
  // per task
  double* rr;
  double* gamma_prev;
  double* alpha;
  double* b_norm;
  double* thresh;
  double* gamma;
  double* alpha_new;
  double* mean1;
  double* mean2;
  double* ell;       // labeled count (double), n1, n2
  double* n1;
  double* n2;
  double* sum_v;     // sum(w) at setup, sum(z) in the loop
  double* pq;
  double* rr_new;
  long long* iter;
  long long* fail_iter;
  int* status;       // ST_*; ST_PAD for padding lanes
  int* finished;
  int* n_active;
  // per (task, shift)
  const double* beta;  // ns
  double* zeta_prev;
  double* zeta;
  double* alpha_s;
  double* resid;
  double* s_zn;        // this iteration's zeta_next / gamma_s / good (phase B)
  double* s_gs;
  unsigned char* s_good;
  double* upd_gs;      // shift-update snapshot (phase C)
  double* upd_zn;
  double* upd_as;
  int* upd_mode;
  long long* iters;
  unsigned char* conv;
  unsigned char* active;
  unsigned char* flip;
  int ns;
  int tp;
  long long max_iter;
};

constexpr int ST_PAD = 7;

// w / G for the (item, task group) decomposition of a warp index: a shift when
// G is a power of two (the 64-bit division costs ~50 instructions per warp).
__device__ __forceinline__ long long div_groups(long long w, int G) {
  return (G & (G - 1)) == 0 ? (w >> (31 - __clz(G))) : w / G;
}

__device__ __forceinline__ bool b_live(const BatchState& B, int t) {
  return B.status[t] == ST_OK && !B.finished[t];
}

__device__ __forceinline__ double tree32(double (&A)[32]) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
    for (int l = 0; l < off; ++l) A[l] = A[l] + A[l + off];
  return A[0];
}

// Canonical leaf of n <= 256 values val(e), e = 0..n-1, for this lane's task.
// val may use warp shuffles: control flow is uniform (n is warp-uniform).
template <typename Val>
__device__ __forceinline__ double emu_leaf(int n, Val val) {
  double A[32];
#pragma unroll
  for (int l = 0; l < 32; ++l) A[l] = 0.0;
  for (int base = 0; base < n; base += 32) {
#pragma unroll
    for (int l = 0; l < 32; ++l)
      if (base + l < n) A[l] = A[l] + val(base, l);
  }
  return tree32(A);
}

// Dot leaf: A[l] = fma(x, y, A[l]).
template <typename XY>
__device__ __forceinline__ double emu_dot_leaf(int n, XY xy) {
  double A[32];
#pragma unroll
  for (int l = 0; l < 32; ++l) A[l] = 0.0;
  for (int base = 0; base < n; base += 32) {
#pragma unroll
    for (int l = 0; l < 32; ++l)
      if (base + l < n) {
        double x, y;
        xy(base + l, x, y);
        A[l] = fma(x, y, A[l]);
      }
  }
  return tree32(A);
}

// Gathered-value terms: special(idx) marks the one index treated differently
// (the diagonal of a Laplacian row), operator()(is_special, v) maps the value.
struct TermPlain {
  static constexpr bool kSpecial = false;
  __device__ __forceinline__ bool special(int) const { return false; }
  __device__ __forceinline__ int special_row() const { return 0; }
  __device__ __forceinline__ int map(int idx) const { return idx; }
  __device__ __forceinline__ double operator()(bool, double v) const { return v; }
};
struct TermLap {  // (L y)_i terms: d_i y_i on the diagonal, -y_j off it
  static constexpr bool kSpecial = true;
  int row;
  double dg;
  __device__ __forceinline__ bool special(int idx) const { return idx == row; }
  __device__ __forceinline__ int special_row() const { return row; }
  __device__ __forceinline__ int map(int idx) const { return idx; }
  __device__ __forceinline__ double operator()(bool sp, double v) const { return sp ? dg * v : -v; }
};
// The same row sum with every term negated, so that no gather needs a select:
// off-diagonal slots add +y_j, and the diagonal's slot is pointed (by the lane
// that owns its index) at a second block of the table that holds
// -(d_i y_i), written by the producer of y.  IEEE addition is symmetric under
// negation, so the tree of negated terms is the negated tree: the caller
// negates the result and has TermLap's sum bit for bit (a sum that is exactly
// zero may differ in the sign of zero).
struct TermLapNeg {
  static constexpr bool kSpecial = false;
  int row;
  int yd_row0;  // first row of the -(d y) block in the table
  __device__ __forceinline__ bool special(int) const { return false; }
  __device__ __forceinline__ int special_row() const { return 0; }
  __device__ __forceinline__ int map(int idx) const { return idx == row ? yd_row0 + idx : idx; }
  __device__ __forceinline__ double operator()(bool, double v) const { return v; }
};

// Canonical leaf of a gathered index segment: ind[s0, s0 + len) (len <= 256)
// selects rows of src (task-minor); term maps the gathered value.
// The canonical lane accumulators A[l] = sum_k v[l + 32 k] are built in pairs
// (l, l + 16) and folded at once into B[l] = A[l] + A[l + 16] — the first
// butterfly step — so only 16 partial sums stay live (register budget: four
// 256-thread CTAs per SM).  Indices arrive 32 at a time (coalesced); the
// owning lane turns each into the element offset idx * tp once, and the
// offsets are shuffled to every lane; 2 LS values per lane are in flight.
// Slots past the segment's end gather the table's zero row (every gathered
// table carries one more row of zeros) and add (+/-)0.0, which leaves every
// partial sum unchanged bit for bit (no partial sum is ever -0.0): no bounds
// test or select per gather.
template <int LS, int NK, typename V, typename Term>
__device__ __forceinline__ double emu_gather_leaf_ls(const int* __restrict__ ind, long long s0, int len,
                                                     const V* __restrict__ src, int tp, int t,
                                                     int lane, Term term, unsigned zoff) {
  const int nk = (len + 31) >> 5;     // <= NK index chunks of 32 (NK = 1, 2 or 8: len <= 32 NK)
  // byte offset idx * tp * sizeof(V) of the gathered row (host: below 2^32);
  // slots past the segment's end point at the table's zero row (zoff)
  unsigned my[NK];
  const unsigned row_bytes = (unsigned)tp * (unsigned)sizeof(V);
#pragma unroll
  for (int k = 0; k < NK; ++k)
    my[k] = (32 * k + lane < len) ? (unsigned)term.map(__ldg(ind + s0 + 32 * k + lane)) * row_bytes : zoff;
  // this lane's column of src as an opaque address, so that a gather is one
  // 64-bit add away (the compiler otherwise rebuilds (idx * tp + t) * 8 + src
  // for every load)
  unsigned long long bp = (unsigned long long)(src + t);
  asm volatile("" : "+l"(bp));
  const unsigned sp_off = (unsigned)term.special_row() * row_bytes;
  // Steps run in the order l0 = h, h + 8 (h = 0, LS, ..) and the butterfly's
  // offset-8 step B[l] + B[l + 8] is taken as soon as both halves exist, so
  // at most 8 folded sums (and one step's 2 LS) stay live instead of 16.
  // Same additions as the plain order, only scheduled earlier.
  static_assert(LS <= 8, "a step holds at most 8 lane pairs");
  double Bp[8];
#pragma unroll
  for (int h = 0; h < 8; h += LS) {
    double Bh[2][LS];
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int l0 = h + 8 * half;
      double a1[LS], a2[LS];
#pragma unroll
      for (int q = 0; q < LS; ++q) a1[q] = a2[q] = 0.0;
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        if (NK > 2 && k >= nk) break;  // NK <= 2: a chunk past the end gathers the zero row
        V v1[LS], v2[LS];
        unsigned sp1 = 0u, sp2 = 0u;
        // the step's second half (slots l + 16) lies wholly past the end: its
        // loads would all read the zero row, so they are skipped (warp-uniform;
        // adding the zeros below is the same sum)
        const bool second = 32 * k + l0 + 16 < len;
#pragma unroll
        for (int q = 0; q < LS; ++q) {
          const int l = l0 + q;
          const unsigned o1 = __shfl_sync(FULL, my[k], l);
          v1[q] = __ldg(reinterpret_cast<const V*>(bp + o1));
          if (Term::kSpecial) sp1 |= (o1 == sp_off) ? (1u << q) : 0u;
        }
        if (second) {
#pragma unroll
          for (int q = 0; q < LS; ++q) {
            const unsigned o2 = __shfl_sync(FULL, my[k], l0 + q + 16);
            v2[q] = __ldg(reinterpret_cast<const V*>(bp + o2));
            if (Term::kSpecial) sp2 |= (o2 == sp_off) ? (1u << q) : 0u;
          }
        } else {
#pragma unroll
          for (int q = 0; q < LS; ++q) v2[q] = (V)0;
        }
#pragma unroll
        for (int q = 0; q < LS; ++q) {
          a1[q] = a1[q] + term((sp1 >> q) & 1u, (double)v1[q]);
          a2[q] = a2[q] + term((sp2 >> q) & 1u, (double)v2[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < LS; ++q) Bh[half][q] = a1[q] + a2[q];  // B[l0 + q]
    }
#pragma unroll
    for (int q = 0; q < LS; ++q) Bp[h + q] = Bh[0][q] + Bh[1][q];  // B[l] + B[l + 8]
  }
#pragma unroll
  for (int off = 4; off >= 1; off >>= 1)
#pragma unroll
    for (int l = 0; l < off; ++l) Bp[l] = Bp[l] + Bp[l + off];
  return Bp[0];
}

// LS lane pairs (2 LS gathers per lane) in flight per step.  A segment of at
// most 32 entries (a row of L, ~21 at cfg4) has a single index chunk, so its
// steps are latency rounds with little else to overlap: it takes 8 pairs per
// step (2 rounds instead of 4); longer segments keep GATHER_MLP.  Same
// accumulation order either way.
template <typename V, typename Term>
__device__ __forceinline__ double emu_gather_leaf(const int* __restrict__ ind, long long s0, int len,
                                                  const V* __restrict__ src, int tp, int t,
                                                  int lane, Term term, unsigned zoff) {
  constexpr int LS = sizeof(V) == 4 ? F32_LS : GATHER_MLP / 2;
  if (len <= 32) return emu_gather_leaf_ls<8, 1, V>(ind, s0, len, src, tp, t, lane, term, zoff);
  if (len <= 64) return emu_gather_leaf_ls<LS, 2, V>(ind, s0, len, src, tp, t, lane, term, zoff);
  return emu_gather_leaf_ls<LS, 8, V>(ind, s0, len, src, tp, t, lane, term, zoff);
}

// Segments longer than 256 entries: R256 over their leaves (two levels,
// n <= 65536).  Kept out of line: it holds a second accumulator set.
template <typename V, typename Term>
__device__ __noinline__ double emu_gather_long(const int* __restrict__ ind, long long start, int n,
                                               const V* __restrict__ src, int tp, int t,
                                               int lane, Term term, unsigned zoff) {
  const int m = (n + LEAF - 1) / LEAF;  // <= 256 (host-checked)
  double P[32];
#pragma unroll
  for (int l = 0; l < 32; ++l) P[l] = 0.0;
  for (int gb = 0; gb < m; gb += 32) {
    for (int l = 0; l < 32 && gb + l < m; ++l) {
      const int g = gb + l;
      const double v = emu_gather_leaf(ind, start + (long long)g * LEAF, min(LEAF, n - g * LEAF),
                                       src, tp, t, lane, term, zoff);
#pragma unroll
      for (int q = 0; q < 32; ++q)
        if (q == l) P[q] = P[q] + v;
    }
  }
  return tree32(P);
}

template <typename V, typename Term>
__device__ __forceinline__ double emu_segment(const int* __restrict__ ind, long long start, int n,
                                              const V* __restrict__ src, int tp, int t,
                                              int lane, Term term, unsigned zoff) {
  if (n <= LEAF) return emu_gather_leaf(ind, start, n, src, tp, t, lane, term, zoff);
  return emu_gather_long(ind, start, n, src, tp, t, lane, term, zoff);
}

// ------------------------------------------------------------ layout moves

// labels [T][N] -> lab [N][TP] (padding 0) and the labeled indicator.
__global__ void kb_labels_in(const signed char* __restrict__ in, signed char* __restrict__ lab,
                             double* __restrict__ ind, long long n, int T, int tp) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n * tp;
       k += (long long)gridDim.x * blockDim.x) {
    const long long i = k / tp;
    const int t = (int)(k - i * tp);
    const signed char l = t < T ? in[(long long)t * n + i] : 0;
    lab[k] = l;
    ind[k] = l != 0 ? 1.0 : 0.0;
  }
}

// x [T][L] -> out [L][TP] (padding 0.0).
__global__ void kb_task_minor(const double* __restrict__ in, double* __restrict__ out, long long len,
                              int T, int tp) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < len * tp;
       k += (long long)gridDim.x * blockDim.x) {
    const long long i = k / tp;
    const int t = (int)(k - i * tp);
    out[k] = t < T ? in[(long long)t * len + i] : 0.0;
  }
}

// sols [D][TP * ns] -> out [T * ns][D], negated where the orientation flips
// (sda.py:280-283): a 32 x 32 tiled transpose through shared memory, so both
// the reads (along task-shift) and the writes (along features) are coalesced.
// blockDim = (32, 8); grid = (ceil(D / 32), ceil(Q / 32)), Q = T * ns (the
// long dimension on grid.x).
__global__ void __launch_bounds__(256) kb_directions_out(const double* __restrict__ sols,
                                                         double* __restrict__ out, long long d, int T,
                                                         int tp, int ns,
                                                         const unsigned char* __restrict__ flip) {
  __shared__ double tile[32][33];
  const long long Q = (long long)T * ns, ld = (long long)tp * ns;
  const long long q0 = (long long)blockIdx.y * 32, c0 = (long long)blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const long long c = c0 + r, q = q0 + threadIdx.x;
    tile[r][threadIdx.x] = (c < d && q < Q) ? sols[c * ld + q] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const long long q = q0 + r, c = c0 + threadIdx.x;
    if (q < Q && c < d) {
      const double v = tile[threadIdx.x][r];
      out[q * d + c] = flip[q] ? -v : v;
    }
  }
}

// ------------------------------------------------------------- setup

__global__ void kb_reset(BatchState B, int T, double tol) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B.tp) return;
  B.rr[t] = 0.0; B.gamma_prev[t] = 1.0; B.alpha[t] = 0.0; B.b_norm[t] = 0.0; B.thresh[t] = 0.0;
  B.gamma[t] = 0.0; B.alpha_new[t] = 0.0; B.sum_v[t] = 0.0;
  B.iter[t] = 0; B.fail_iter[t] = -1; B.status[t] = t < T ? ST_OK : ST_PAD;
  B.finished[t] = t < T ? 0 : 1;
  B.n_active[t] = B.ns;
  for (int s = 0; s < B.ns; ++s) {
    const int k = t * B.ns + s;
    B.zeta_prev[k] = 1.0; B.zeta[k] = 1.0; B.alpha_s[k] = 0.0; B.resid[k] = 0.0;
    B.iters[k] = B.max_iter; B.conv[k] = 0; B.active[k] = 1; B.flip[k] = 0; B.upd_mode[k] = 0;
  }
  (void)tol;
}

// ------------------------------------------------------- operator products

// Row sums over a CSR pattern for every task: K1 (y = X p) and K2 (z = M y).
// One warp per (row, task group).
// YD (fp64 storage, the loop's K1 / K2 pair): K1 also writes -(d_i y_i) into
// rows yd_row0 + i of its output table, and K2 sums with TermLapNeg.
template <int KIND, typename V, bool YD = false>
__global__ void __launch_bounds__(256, (KIND == SEG_LROWS ? KB_LROWS_MINB : KB_XROWS_MINB) +
                                            (sizeof(V) == 4 ? KB_ROWS_F32_EXTRA : 0)) kb_rows(const int* __restrict__ rowptr,
                                               const int* __restrict__ cols,
                                               const V* __restrict__ src,
                                               V* __restrict__ out, long long n_rows, int G,
                                               int tp, const double* __restrict__ ldiag,
                                               const signed char* __restrict__ lab, double alpha,
                                               int alpha_mode, long long src_rows, long long yd_row0) {
  const unsigned zoff = (unsigned)(src_rows * tp * (long long)sizeof(V));  // the zero row of src
  const int lane = threadIdx.x & 31;
  const long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= n_rows * G) return;
  const long long i = div_groups(w, G);
  const int g = (int)(w - i * G);
  const int t = g * BG + lane;
  const int lo = __ldg(rowptr + i), n = __ldg(rowptr + i + 1) - lo;
  double s;
  if (KIND == SEG_LROWS) {
    if (YD) {
      s = -emu_segment(cols, lo, n, src, tp, t, lane, TermLapNeg{(int)i, (int)yd_row0}, zoff);
    } else {
      const double dg = __ldg(ldiag + i);
      s = emu_segment(cols, lo, n, src, tp, t, lane, TermLap{(int)i, dg}, zoff);
    }
    const double masked = lab[i * tp + t] != 0 ? (double)src[i * tp + t] : 0.0;
    const double smoothed = alpha * s;
    s = (alpha_mode == 1) ? smoothed : (1.0 - alpha) * masked + smoothed;
  } else {
    s = emu_segment(cols, lo, n, src, tp, t, lane, TermPlain{}, zoff);
    if (YD) out[(yd_row0 + i) * tp + t] = (V)(-(__ldg(ldiag + i) * (double)(V)s));
  }
  out[i * tp + t] = (V)s;
}

// z = masked y (apply_smoother at alpha == 0).
template <typename V>
__global__ void kb_mask(const V* __restrict__ y, const signed char* __restrict__ lab,
                        V* __restrict__ z, long long len) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < len;
       k += (long long)gridDim.x * blockDim.x)
    z[k] = lab[k] != 0 ? y[k] : (V)0;
}

// Column finish of X^T: mode 0 raw, 1 centred (s - mu * sum_v[t]), 2 / ell[t].
__device__ __forceinline__ double b_col_finish(double s, int mode, long long c, int t, int tp,
                                               const double* __restrict__ mu,
                                               const BatchState& B) {
  if (mode == 1) return s - mu[c * tp + t] * B.sum_v[t];
  if (mode == 2) return s / B.ell[t];
  return s;
}

// X^T columns with n <= 256: the class tasks of the single-task column plan
// (any class: each entry is one column segment).  One warp per (entry, group).
template <typename V>
__global__ void __launch_bounds__(256, KB_COLS_MINB) kb_cols_light(SegPlan pl, const V* __restrict__ src,
                                                     double* __restrict__ out, int G, int tp,
                                                     int mode, const double* __restrict__ mu,
                                                     BatchState B, long long src_rows) {
  const unsigned zoff = (unsigned)(src_rows * tp * (long long)sizeof(V));
  const int lane = threadIdx.x & 31;
  const long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long n_entries = pl.cls_off[6];
  if (w >= n_entries * G) return;
  const long long e = div_groups(w, G);
  const int g = (int)(w - e * G);
  const int t = g * BG + lane;
  const int4 tk = __ldg(pl.tasks + e);
  const double s = emu_gather_leaf(pl.ind, tk.y, tk.z, src, tp, t, lane, TermPlain{}, zoff);
  out[(long long)tk.x * tp + t] = b_col_finish(s, mode, tk.x, t, tp, mu, B);
}

// Leaf sums of the long columns: the heavy leaves (plan_xc heavy tasks, up to
// 4 leaves each) into hpart[slot][TP], and the blocked slices (XtDense tasks,
// one <= 256-entry leaf each) into xpart[slot][TP].
template <typename V>
__global__ void __launch_bounds__(256, KB_COLS_MINB) kb_cols_leaves(SegPlan pl, XtDense dn,
                                                      const V* __restrict__ src,
                                                      double* __restrict__ hpart,
                                                      double* __restrict__ xpart, long long n_hleaf,
                                                      long long n_xtask, int G, int tp,
                                                      long long src_rows) {
  const unsigned zoff = (unsigned)(src_rows * tp * (long long)sizeof(V));
  const int lane = threadIdx.x & 31;
  const long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= (n_hleaf + n_xtask) * G) return;
  const long long u = div_groups(w, G);
  const int g = (int)(w - u * G);
  const int t = g * BG + lane;
  // one gather call for both kinds of leaf (a single inlined copy of the loop)
  const int* ind;
  long long start;
  int len;
  double* dst;
  if (u < n_hleaf) {
    // u indexes heavy leaves in task order: task j covers leaves [4j, 4j + 4)
    const long long j = u >> 2;
    const int lf = (int)(u & 3);
    const int4 tk = __ldg(pl.tasks + pl.cls_off[6] + j);
    if (lf * LEAF >= tk.z) return;
    const int h = tk.w;
    const int slot = __ldg(pl.heavy_seg0 + h) + (tk.y - __ldg(pl.heavy_start + h)) / LEAF + lf;
    ind = pl.ind;
    start = tk.y + lf * LEAF;
    len = min(LEAF, tk.z - lf * LEAF);
    dst = hpart + (long long)slot * tp + t;
  } else {
    const int4 tk = __ldg(dn.tasks + (u - n_hleaf));
    ind = dn.rows;
    start = tk.y;
    len = tk.z;
    dst = xpart + (long long)tk.x * tp + t;
  }
  *dst = emu_gather_leaf(ind, start, len, src, tp, t, lane, TermPlain{}, zoff);
}

// Canonical leaf over len <= 256 consecutive task-minor partials.
__device__ __forceinline__ double emu_part_leaf(const double* __restrict__ part, long long k0,
                                                int len, int tp, int t) {
  double A[32];
#pragma unroll
  for (int l = 0; l < 32; ++l) A[l] = 0.0;
  for (int base = 0; base < len; base += 32) {
#pragma unroll
    for (int sub = 0; sub < 4; ++sub) {
      if (base + sub * 8 >= len) break;
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int e = base + sub * 8 + j;
        v[j] = e < len ? part[(k0 + e) * tp + t] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (base + sub * 8 + j < len) A[sub * 8 + j] = A[sub * 8 + j] + v[j];
    }
  }
  return tree32(A);
}

__device__ __noinline__ double emu_part_long(const double* __restrict__ part, long long m, int tp,
                                             int t) {
  const int m2 = (int)((m + LEAF - 1) / LEAF);
  double P[32];
#pragma unroll
  for (int l = 0; l < 32; ++l) P[l] = 0.0;
  for (int gb = 0; gb < m2; gb += 32) {
    for (int l = 0; l < 32 && gb + l < m2; ++l) {
      const long long k0 = (long long)(gb + l) * LEAF;
      const double v = emu_part_leaf(part, k0, (int)min((long long)LEAF, m - k0), tp, t);
#pragma unroll
      for (int q = 0; q < 32; ++q)
        if (q == l) P[q] = P[q] + v;
    }
  }
  return tree32(P);
}

// R256 over m partials part[k][TP] (k = 0..m-1) for this lane's task, as
// block_reduce_partials does for one task: m <= 256 one leaf; otherwise
// leaves of 256 partials, then a leaf over their sums.  One warp.
__device__ __forceinline__ double emu_partials(const double* __restrict__ part, long long m,
                                               int tp, int t) {
  if (m <= LEAF) return emu_part_leaf(part, 0, (int)m, tp, t);
  return emu_part_long(part, m, tp, t);
}

// Block-level canonical leaves over (up to) 256 task-minor rows: warp w owns
// the canonical lanes l = 4w .. 4w + 3 and builds A[l] = sum over k of row
// l + 32 k (k ascending from 0.0; fma for dot leaves) straight from global
// memory — every row is one coalesced 256-byte load per warp, eight rows in
// flight per lane.  The 32 lane sums go through 8 KB of shared memory to
// warp 0, which folds them with tree32.  sm holds 32 x 32 doubles.
constexpr int BLK_SM = 32 * 32;

template <bool DOT, typename Load>
__device__ __forceinline__ double block_leaf(int n, Load load, double* sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int l = 4 * w + j;
    double x[8], y[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x[k] = 0.0;
      y[k] = 0.0;
      if (l + 32 * k < n) load(l + 32 * k, x[k], y[k]);
    }
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (l + 32 * k < n) a = DOT ? fma(x[k], y[k], a) : a + x[k];
    sm[l * 32 + lane] = a;
  }
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    double A[32];
#pragma unroll
    for (int l = 0; l < 32; ++l) A[l] = sm[l * 32 + lane];
    r = tree32(A);
  }
  __syncthreads();
  return r;
}

// The long columns' partials, unit u: heavy segment u (hn leaf sums from h0)
// for u < n_heavy, else blocked column u - n_heavy (its poff range).
__device__ __forceinline__ const double* unit_part(const SegPlan& pl, const XtDense& dn,
                                                   const double* hpart, const double* xpart,
                                                   long long n_heavy, long long u, int tp,
                                                   long long* m) {
  if (u < n_heavy) {
    *m = __ldg(pl.heavy_nseg + u);
    return hpart + (long long)__ldg(pl.heavy_seg0 + u) * tp;
  }
  const long long b = u - n_heavy;
  const long long p0 = __ldg(dn.poff + b);
  *m = __ldg(dn.poff + b + 1) - p0;
  return xpart + p0 * tp;
}

// Level 1 of the long units (more than 256 partials — the Zipf head's
// blocked columns hold up to ~6k): one warp per (256-partial group, task
// group) writes the group's canonical leaf to gsum, so no warp walks a whole
// column alone.  chunks[k] = {unit, group}; gsoff[unit] = its first slot.
__global__ void __launch_bounds__(256) kb_part_groups(SegPlan pl, XtDense dn,
                                                      const double* __restrict__ hpart,
                                                      const double* __restrict__ xpart,
                                                      long long n_heavy, const int2* __restrict__ chunks,
                                                      long long n_chunks, const int* __restrict__ gsoff,
                                                      double* __restrict__ gsum, int G, int tp) {
  const int lane = threadIdx.x & 31;
  const long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= n_chunks * G) return;
  const long long k = div_groups(w, G);
  const int g = (int)(w - k * G);
  const int t = g * BG + lane;
  const int2 ch = __ldg(chunks + k);
  long long m;
  const double* part = unit_part(pl, dn, hpart, xpart, n_heavy, ch.x, tp, &m);
  const long long k0 = (long long)ch.y * LEAF;
  gsum[((long long)__ldg(gsoff + ch.x) + ch.y) * tp + t] =
      emu_part_leaf(part, k0, (int)min((long long)LEAF, m - k0), tp, t);
}

// Level 2 over m2 <= 256 precomputed group leaves gs[j][TP]: lane
// accumulators P[l] = sum of leaves j = l, l + 32, ... in order, then
// tree32 — the second level of emu_part_long.
__device__ __noinline__ double emu_group_level2(const double* __restrict__ gs, int m2, int tp, int t) {
  double P[32];
#pragma unroll
  for (int l = 0; l < 32; ++l) P[l] = 0.0;
  for (int gb = 0; gb < m2; gb += 32) {
#pragma unroll
    for (int l = 0; l < 32; ++l)
      if (gb + l < m2) P[l] = P[l] + gs[(long long)(gb + l) * tp + t];
  }
  return tree32(P);
}

// Combine the long columns: heavy segment h (hn[h] leaf sums from h0[h]) and
// blocked column b (poff range).  One warp per (column, group); units with
// more than 256 partials take their level-1 leaves from kb_part_groups.
__global__ void __launch_bounds__(256, 2) kb_cols_combine(SegPlan pl, XtDense dn,
                                                       const double* __restrict__ hpart,
                                                       const double* __restrict__ xpart,
                                                       long long n_heavy,
                                                       double* __restrict__ out, int G, int tp,
                                                       int mode, const double* __restrict__ mu,
                                                       BatchState B, const int* __restrict__ gsoff,
                                                       const double* __restrict__ gsum) {
  const int lane = threadIdx.x & 31;
  const long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= (n_heavy + dn.n_dense) * G) return;
  const long long u = div_groups(w, G);
  const int g = (int)(w - u * G);
  const int t = g * BG + lane;
  long long m;
  const double* part = unit_part(pl, dn, hpart, xpart, n_heavy, u, tp, &m);
  const long long col = u < n_heavy ? (long long)__ldg(pl.heavy_seg + u) : (long long)__ldg(dn.col + (u - n_heavy));
  const int go = gsoff ? __ldg(gsoff + u) : -1;
  const double s = go >= 0 ? emu_group_level2(gsum + (long long)go * tp, (int)((m + LEAF - 1) / LEAF), tp, t)
                           : emu_partials(part, m, tp, t);
  out[col * tp + t] = b_col_finish(s, mode, col, t, tp, mu, B);
}

// Leaf sums over a contiguous task-minor vector (len rows): kind 0 sum(v),
// 1 sum over class +1 (off-class 0.0), 2 class -1, 3 fma dot v . v2.
// One 256-thread block per (leaf, group).
template <typename V>
__global__ void __launch_bounds__(256) kb_vec_leaves(const V* __restrict__ v,
                                                     const V* __restrict__ v2,
                                                     const signed char* __restrict__ lab,
                                                     long long len, int kind,
                                                     double* __restrict__ part, long long n_leaf,
                                                     int G, int tp) {
  __shared__ double sm[BLK_SM];
  const long long lf = blockIdx.x / G;
  const int g = (int)(blockIdx.x - lf * G);
  const int lane = threadIdx.x & 31;
  const int t = g * BG + lane;
  const long long i0 = lf * LEAF;
  const int n = (int)min((long long)LEAF, len - i0);
  double s;
  if (kind == 3) {
    s = block_leaf<true>(n, [&](int e, double& x, double& y) {
      x = (double)v[(i0 + e) * tp + t];
      y = (double)v2[(i0 + e) * tp + t];
    }, sm);
  } else {
    s = block_leaf<false>(n, [&](int e, double& x, double&) {
      const long long k = (i0 + e) * tp + t;
      const double u = (double)v[k];
      x = kind == 1 ? (lab[k] == 1 ? u : 0.0) : (kind == 2 ? (lab[k] == -1 ? u : 0.0) : u);
    }, sm);
  }
  if (threadIdx.x < 32) part[lf * tp + t] = s;
}

// Canonical leaf over n <= 256 task-minor partials -> out[t]; one 256-thread
// block per group (the last level of every R256 reduction).  Longer partial
// lists first go through kb_vec_leaves (kind 0), which folds each run of 256
// partials exactly as the first level of R256 does.
__global__ void __launch_bounds__(256) kb_combine_leaf(const double* __restrict__ part, int n,
                                                       double* __restrict__ out, int tp) {
  __shared__ double sm[BLK_SM];
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * BG + lane;
  const double s = block_leaf<false>(n, [&](int e, double& x, double&) { x = part[(long long)e * tp + t]; }, sm);
  if (threadIdx.x < 32) out[t] = s;
}

// apply_w: class-mean broadcast; the class sums arrive in out1 / out2.
__global__ void kb_class_means(BatchState B, const double* __restrict__ s1,
                               const double* __restrict__ s2) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B.tp) return;
  B.mean1[t] = s1[t] / B.n1[t];
  B.mean2[t] = s2[t] / B.n2[t];
}

__global__ void kb_apply_w(const signed char* __restrict__ lab, double* __restrict__ w,
                           long long len, int tp, BatchState B) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < len;
       k += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(k % tp);
    const signed char l = lab[k];
    w[k] = l == 1 ? B.mean1[t] : (l == -1 ? B.mean2[t] : 0.0);
  }
}

// r = p = b; P_s = b, sols_s = 0 (krylov.py:199-208); thread j of a block
// owns (task, shift) j and walks the rows, as kb_step_c.
__global__ void kb_cg_init_vec(const double* __restrict__ b, double* __restrict__ r,
                               double* __restrict__ p, double* __restrict__ bigp,
                               double* __restrict__ sols, long long d, int tp, int ns) {
  const int tsn = tp * ns;
  for (int j = threadIdx.x; j < tsn; j += blockDim.x) {
    const int t = j / ns, s = j - t * ns;
    for (long long i = blockIdx.x; i < d; i += gridDim.x) {
      const long long k = i * tp + t;
      const double v = b[k];
      if (s == 0) {
        r[k] = v;
        p[k] = v;
      }
      const long long e = i * tsn + j;
      bigp[e] = v;
      sols[e] = 0.0;
    }
  }
}

// Deferred ("basis") shift updates for the batch (the single-solve
// k_coef_update / k_combine_basis per task): coefficient rows
// coef[(t * ns + s) * ld + j].  Init: a = e_0, c = 0.
__global__ void kb_coef_init(double* __restrict__ coef_a, double* __restrict__ coef_c,
                             long long rows, long long ld) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < rows * ld;
       e += (long long)gridDim.x * blockDim.x) {
    coef_a[e] = (e % ld) == 0 ? 1.0 : 0.0;
    coef_c[e] = 0.0;
  }
}

// r = p = b only (the deferred mode keeps no P / sols during the loop).
template <typename V>
__global__ void kb_cg_init_rp(const double* __restrict__ b, V* __restrict__ r,
                              V* __restrict__ p, long long len) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < len;
       k += (long long)gridDim.x * blockDim.x) {
    const double v = b[k];
    r[k] = (V)v;
    p[k] = (V)v;
  }
}

// The loop iteration lives on the device (*BIter::it, advanced by
// kb_loop_next), so the body's launches are identical every iteration and
// the loop can run as a captured graph with a conditional WHILE node.  The
// residual slots of iteration it: r_it / r_{it+1} of the deferred basis, or
// the ping-pong pair of the per-iteration mode.
template <typename V>
struct BIterT {
  V* rb;                 // deferred basis: slot j at rb + j * stride
  V* r0;                 // per-iteration mode: ping-pong residuals
  V* r1;
  long long stride;      // d * TP
  int basis;
  const long long* it;   // loop iteration (device)
};

using BIter = BIterT<double>;

template <typename V>
__device__ __forceinline__ void b_iter_ptrs(const BIterT<V>& bi, const V*& cur, V*& nxt) {
  const long long it = *bi.it;
  if (bi.basis) {
    cur = bi.rb + it * bi.stride;
    nxt = bi.rb + (it + 1) * bi.stride;
  } else {
    cur = (it & 1) ? bi.r1 : bi.r0;
    nxt = (it & 1) ? bi.r0 : bi.r1;
  }
}

// Coefficient updates of loop iteration it for the tasks that stepped
// (kb_step_c's shift part on coefficients).  blockIdx.y = (task, shift).
__global__ void kb_coef_update(BatchState B, const int* __restrict__ stepped, double* __restrict__ coef_a,
                               double* __restrict__ coef_c, long long ld, const long long* __restrict__ itp) {
  const long long it = *itp;
  const int k = blockIdx.y;
  const int t = k / B.ns;
  if (!stepped[t]) return;
  const int mode = B.upd_mode[k];
  if (mode == 0) return;
  const double gs = B.upd_gs[k], zn = B.upd_zn[k], as = B.upd_as[k];
  double* A = coef_a + (long long)k * ld;
  double* Cc = coef_c + (long long)k * ld;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j <= it + 1;
       j += (long long)gridDim.x * blockDim.x) {
    if (j <= it) {
      const double a = A[j];
      Cc[j] = Cc[j] - a * gs;
      if (mode == 3) A[j] = as * a;
    } else if (mode == 3 && j < ld) {
      A[j] = zn;
    }
  }
}

// p = r_next + alpha_new p for the tasks that stepped (kb_step_c without the
// shift state).
template <typename V>
__global__ void kb_step_c_p(BIterT<V> bi, V* __restrict__ p, long long len,
                            int tp, BatchState B, const int* __restrict__ stepped) {
  const V* r_cur;
  V* r_next;
  b_iter_ptrs(bi, r_cur, r_next);
  (void)r_cur;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < len;
       k += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(k % tp);
    if (stepped[t]) p[k] = (V)((double)r_next[k] + B.alpha_new[t] * (double)p[k]);
  }
}

// sols[(i * tp + t) * ns + s] = sum_{j < iter_t} c[t][s][j] * r_j[i * tp + t],
// j ascending from 0.0, one fma per term — the single solve's k_combine_basis
// per task.
template <typename V>
__global__ void __launch_bounds__(256) kb_combine_basis(const V* __restrict__ rb, long long d,
                                                        BatchState B, const double* __restrict__ coef_c,
                                                        long long ld, double* __restrict__ sols) {
  const int tp = B.tp, ns = B.ns;
  const long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= d * tp) return;
  const int t = (int)(x % tp);
  const long long J = B.status[t] == ST_OK ? B.iter[t] : 0;
  const long long stride = d * tp;
  for (int s0 = 0; s0 < ns; s0 += 8) {
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
    const double* cc = coef_c + ((long long)t * ns + s0) * ld;
    for (long long j = 0; j < J; ++j) {
      const double r = (double)__ldcs(rb + j * stride + x);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (s0 + u < ns) acc[u] = fma(__ldg(cc + (long long)u * ld + j), r, acc[u]);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (s0 + u < ns) sols[x * ns + s0 + u] = acc[u];
  }
}

// b.b arrives in bb[t] (krylov.py:185-194).
__global__ void kb_cg_init_scalars(BatchState B, const double* __restrict__ bb, double tol) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B.tp || B.status[t] == ST_PAD) return;
  const double b_norm = sqrt(bb[t]);
  B.b_norm[t] = b_norm;
  B.rr[t] = b_norm * b_norm;
  B.thresh[t] = tol * b_norm;
  if (b_norm == 0.0) {
    for (int s = 0; s < B.ns; ++s) {
      const int k = t * B.ns + s;
      B.iters[k] = 0; B.resid[k] = 0.0; B.conv[k] = 1; B.active[k] = 0;
    }
    B.n_active[t] = 0;
    B.finished[t] = 1;
  } else if (B.max_iter <= 0) {
    B.finished[t] = 1;
  }
}

// ---------------------------------------------------------------- CG step

// A: centring q -= mu * sum(z) and the p.q leaves (fma); one 256-thread
// block per (leaf, group).
template <typename V>
__global__ void __launch_bounds__(256) kb_step_a(double* __restrict__ q,
                                                 const V* __restrict__ p,
                                                 const double* __restrict__ mu, long long d,
                                                 double* __restrict__ part, long long n_leaf,
                                                 int G, BatchState B) {
  __shared__ double sm[BLK_SM];
  const long long lf = blockIdx.x / G;
  const int g = (int)(blockIdx.x - lf * G);
  const int lane = threadIdx.x & 31;
  const int tp = B.tp, t = g * BG + lane;
  if (!__any_sync(FULL, b_live(B, t))) return;  // uniform per block (same group)
  const bool live = b_live(B, t);
  const long long i0 = lf * LEAF;
  const int n = (int)min((long long)LEAF, d - i0);
  const double sz = B.sum_v[t];
  const double s = block_leaf<true>(n, [&](int e, double& x, double& y) {
    const long long k = (i0 + e) * tp + t;
    const double qc = q[k] - mu[k] * sz;
    if (live) q[k] = qc;
    x = (double)p[k];
    y = qc;
  }, sm);
  if (threadIdx.x < 32 && live) part[lf * tp + t] = s;
}

// Scalars after p.q (phase B of k_cg_step): gamma and zeta_next / gamma_s.
__global__ void kb_scalars_b(BatchState B) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B.tp || !b_live(B, t)) return;
  const double pq = B.pq[t];
  if (!isfinite(pq) || pq == 0.0) {
    B.status[t] = isfinite(pq) ? ST_BREAKDOWN : ST_NONFINITE;
    B.fail_iter[t] = B.iter[t];
    B.finished[t] = 1;
    return;
  }
  const double rr = B.rr[t], gp = B.gamma_prev[t], al = B.alpha[t];
  const double gamma = -rr / pq;
  B.gamma[t] = gamma;
  for (int s = 0; s < B.ns; ++s) {
    const int k = t * B.ns + s;
    double zn = 0.0, gs = 0.0;
    unsigned char good = 0;
    if (B.active[k]) {
      const double zp = B.zeta_prev[k], z = B.zeta[k];
      const double denom = gamma * al * (zp - z) + zp * gp * (1.0 - B.beta[s] * gamma);
      zn = zp * z * gp / denom;
      if (isfinite(zn) && !(fabs(zn) < 1e-290)) {
        good = 1;
        gs = gamma * zn / z;
      }
    }
    B.s_zn[k] = zn;
    B.s_gs[k] = gs;
    B.s_good[k] = good;
  }
}

// B: r_next = r + gamma q and the r.r leaves; one block per (leaf, group).
template <typename V>
__global__ void __launch_bounds__(256) kb_step_b(const double* __restrict__ q, BIterT<V> bi, long long d,
                                                 double* __restrict__ part, long long n_leaf,
                                                 int G, BatchState B) {
  __shared__ double sm[BLK_SM];
  const V* r_cur;
  V* r_next;
  b_iter_ptrs(bi, r_cur, r_next);
  const long long lf = blockIdx.x / G;
  const int g = (int)(blockIdx.x - lf * G);
  const int lane = threadIdx.x & 31;
  const int tp = B.tp, t = g * BG + lane;
  if (!__any_sync(FULL, b_live(B, t))) return;
  const bool live = b_live(B, t);
  const long long i0 = lf * LEAF;
  const int n = (int)min((long long)LEAF, d - i0);
  const double gamma = B.gamma[t];
  const double s = block_leaf<true>(n, [&](int e, double& x, double& y) {
    const long long k = (i0 + e) * tp + t;
    // rounded to storage once; the dot runs over the stored value
    const V st = (V)((double)r_cur[k] + gamma * q[k]);
    if (live) r_next[k] = st;
    x = (double)st;
    y = (double)st;
  }, sm);
  if (threadIdx.x < 32 && live) part[lf * tp + t] = s;
}

// Scalars after r.r (phase C of k_cg_step, block 0's bookkeeping).
__global__ void kb_scalars_c(BatchState B) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B.tp || !b_live(B, t)) return;
  const double rr_new = B.rr_new[t];
  const long long it = B.iter[t];
  for (int s = 0; s < B.ns; ++s) B.upd_mode[t * B.ns + s] = 0;
  if (!isfinite(rr_new)) {
    B.status[t] = ST_NONFINITE;
    B.fail_iter[t] = it;
    B.finished[t] = 1;
    return;
  }
  const double rr = B.rr[t], gamma = B.gamma[t];
  const double alpha_new = rr_new / rr;
  B.alpha_new[t] = alpha_new;
  const double r_norm = sqrt(rr_new);
  int n_active = 0;
  for (int s = 0; s < B.ns; ++s) {
    const int k = t * B.ns + s;
    if (!B.active[k]) continue;
    if (!B.s_good[k]) {  // degenerate zeta: freeze untouched (krylov.py:251-255)
      B.iters[k] = it + 1;
      B.resid[k] = __longlong_as_double(0x7ff0000000000000LL);
      B.active[k] = 0;
      continue;
    }
    const double zn = B.s_zn[k], z = B.zeta[k], gs = B.s_gs[k];
    const double as = alpha_new * (zn * gs) / (z * gamma);
    B.alpha_s[k] = as;
    B.upd_gs[k] = gs;
    B.upd_zn[k] = zn;
    B.upd_as[k] = as;
    const double shift_res = fabs(zn) * r_norm;
    if (shift_res < B.thresh[t]) {
      B.iters[k] = it + 1;
      B.resid[k] = shift_res;
      B.conv[k] = 1;
      B.active[k] = 0;
      B.upd_mode[k] = 1;
    } else {
      B.zeta_prev[k] = z;
      B.zeta[k] = zn;
      B.upd_mode[k] = 3;
      ++n_active;
    }
  }
  B.gamma_prev[t] = gamma;
  B.alpha[t] = alpha_new;
  B.rr[t] = rr_new;
  B.iter[t] = it + 1;
  B.n_active[t] = n_active;
  // finished is raised by kb_step_c after the last p / shift updates
}

// C: p = r_next + alpha_new p, then the shift updates of this iteration
// (krylov.py:230, 238-241).  Thread j of a block owns one (task, shift) pair
// (t = j / ns, s = j % ns: its scalars stay in registers) and walks the rows
// i = blockIdx.x, +gridDim.x, ...; for a fixed row the block's accesses to
// the (row, task, shift) shift state are contiguous.
__global__ void kb_step_c(BIter bi, double* __restrict__ p,
                          double* __restrict__ bigp, double* __restrict__ sols, long long d,
                          BatchState B, const int* __restrict__ stepped) {
  const double* r_cur;
  double* r_next;
  b_iter_ptrs(bi, r_cur, r_next);
  (void)r_cur;
  const int tp = B.tp, ns = B.ns, tsn = tp * ns;
  for (int j = threadIdx.x; j < tsn; j += blockDim.x) {
    const int t = j / ns, s = j - t * ns;
    if (!stepped[t]) continue;
    const int mode = B.upd_mode[j];
    const double an = B.alpha_new[t];
    const double gs = B.upd_gs[j], zn = B.upd_zn[j], as = B.upd_as[j];
    for (long long i = blockIdx.x; i < d; i += gridDim.x) {
      const long long k = i * tp + t;
      const double rn = r_next[k];
      if (s == 0) p[k] = rn + an * p[k];
      if (mode == 0) continue;
      const long long e = i * tsn + j;
      const double pv = bigp[e];
      sols[e] = sols[e] - pv * gs;
      if (mode == 3) bigp[e] = zn * rn + as * pv;
    }
  }
}

// Which tasks ran this iteration's updates (live after phase C), then the
// end-of-iteration flags (krylov.py:269-270 and the iteration budget).
__global__ void kb_mark_stepped(BatchState B, int* __restrict__ stepped) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B.tp) return;
  stepped[t] = b_live(B, t) ? 1 : 0;
}

__global__ void kb_end_iteration(BatchState B, const int* __restrict__ stepped,
                                 int* __restrict__ n_live) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B.tp) return;
  if (stepped[t] && (B.n_active[t] == 0 || B.iter[t] >= B.max_iter)) B.finished[t] = 1;
  if (b_live(B, t)) atomicAdd(n_live, 1);
}

// End of a loop iteration: advance the device iteration, decide whether
// another one runs (a live task and budget left) and reset the live count.
// In the captured loop the decision is the WHILE node's condition; the
// eager loop reads *keep.
__global__ void kb_loop_next(int* __restrict__ n_live, long long* __restrict__ itp, long long max_iter,
                             int* __restrict__ keep_out, unsigned long long cond_handle, int use_cond) {
  const long long it = *itp + 1;
  *itp = it;
  const int keep = (*n_live > 0 && it < max_iter) ? 1 : 0;
  *n_live = 0;
  *keep_out = keep;
  if (use_cond) cudaGraphSetConditional((cudaGraphConditionalHandle)cond_handle, (unsigned)keep);
}

// After the loop: still-active shifts report |zeta| sqrt(rr) (krylov.py:272-275).
__global__ void kb_finish(BatchState B) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B.tp || B.status[t] != ST_OK) return;
  const double rn = sqrt(B.rr[t]);
  for (int s = 0; s < B.ns; ++s) {
    const int k = t * B.ns + s;
    if (B.active[k]) {
      B.iters[k] = B.max_iter;
      B.resid[k] = fabs(B.zeta[k]) * rn;
    }
  }
}

// Projection scores of the labeled rows only (the orientation y . s needs no
// others; used when the caller does not ask for the scores).  A warp covers 32
// tasks of one row; for each labeled (row, task) among them the whole warp
// walks the row's columns in stored order — the order of k_spmm_scores and of
// scipy's csr_matvec — with lane = shift, so the W row reads are coalesced.
// lab: labels task-minor [N][TP] (TP a multiple of 32).
constexpr int SC_SH = 8;  // shifts per pass of kb_orient_leaves
__global__ void __launch_bounds__(256) kb_scores_labeled(const int* __restrict__ rowptr,
                                                         const int* __restrict__ cols,
                                                         const signed char* __restrict__ lab,
                                                         const double* __restrict__ sols,
                                                         double* __restrict__ scores, long long n,
                                                         int tp, int ns) {
  const int lane = threadIdx.x & 31;
  const long long k0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) - lane;  // warp's first (row, task)
  if (k0 >= n * tp) return;
  unsigned m = __ballot_sync(FULL, lab[k0 + lane] != 0);
  if (m == 0u) return;
  const long long i = k0 / tp;
  const int t0 = (int)(k0 - i * tp);
  const int lo = __ldg(rowptr + i), hi = __ldg(rowptr + i + 1);
  while (m) {
    const int b = __ffs(m) - 1;
    m &= m - 1;
    const int t = t0 + b;
    for (int s0 = 0; s0 < ns; s0 += 32) {
      const int sh = s0 + lane;
      double acc = 0.0;
      if (sh < ns)
        for (int j = lo; j < hi; ++j) acc = acc + sols[((long long)__ldg(cols + j) * tp + t) * ns + sh];
      if (sh < ns) scores[((long long)t * ns + sh) * n + i] = acc;
    }
  }
}

// Orientation leaves y . s per (task, shift) over N (fma, canonical lanes over
// rows) for SC_SH shifts of one task per warp pass: blockIdx.y = task *
// n_chunks + chunk.  Unlabeled rows are skipped: fma(0, s, a) == a for every
// finite s, so the leaf sums equal the single solve's k_orient bit for bit
// (a non-finite score on an unlabeled row would differ; such a task has
// already failed with ST_NONFINITE).  labt: labels task-major [T][N].
__global__ void kb_orient_leaves(const signed char* __restrict__ labt,
                                 const double* __restrict__ scores, long long n,
                                 double* __restrict__ part, long long n_leaf, int ns,
                                 int t_base) {
  const int lane = threadIdx.x & 31;
  const long long g = (long long)blockIdx.x * WARPS_PER_BLOCK + (threadIdx.x >> 5);
  const int nch = (ns + SC_SH - 1) / SC_SH;
  const int tl = blockIdx.y / nch, s0 = (blockIdx.y - tl * nch) * SC_SH;
  const int t = t_base + tl;
  if (g >= n_leaf) return;
  double a[SC_SH];
#pragma unroll
  for (int u = 0; u < SC_SH; ++u) a[u] = 0.0;
  for (int k = 0; k < 8; ++k) {
    const long long i = g * LEAF + k * 32 + lane;
    if (i >= n) continue;
    const signed char lb = labt[(long long)t * n + i];
    if (lb == 0) continue;
#pragma unroll
    for (int u = 0; u < SC_SH; ++u)
      if (s0 + u < ns) a[u] = fma((double)lb, scores[((long long)t * ns + s0 + u) * n + i], a[u]);
  }
#pragma unroll
  for (int u = 0; u < SC_SH; ++u) {
    const double v = butterfly(a[u]);
    if (lane == 0 && s0 + u < ns) part[((long long)t * ns + s0 + u) * n_leaf + g] = v;
  }
}

__global__ void kb_orient_combine(const double* __restrict__ part, long long n_leaf,
                                  BatchState B) {
  __shared__ double smem[257];
  const int ts = blockIdx.x;
  const double v = block_reduce_partials(part + (long long)ts * n_leaf, n_leaf, smem);
  if (threadIdx.x == 0) B.flip[ts] = v < 0.0 ? 1 : 0;
}

// Negate the flipped (task, shift) score vectors [T * ns][N] (the directions
// take their sign in kb_directions_out).
__global__ void kb_flip(double* __restrict__ scores, long long n, int T, BatchState B) {
  const int ts = blockIdx.y;
  const int t = ts / B.ns;
  if (t >= T || !B.flip[ts]) return;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    scores[(long long)ts * n + i] = -scores[(long long)ts * n + i];
}

}  // namespace fsda
