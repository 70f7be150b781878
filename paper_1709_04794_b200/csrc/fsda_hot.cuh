// fsda_hot.cuh — the per-iteration kernels of the FSDA sweep (included by
// fsda_device.cuh; same arithmetic contract, see the header there).
//
// One shifted-CG iteration = 5 launches:
//   k_segsum<SEG_XROWS>  y = X p                (rows, canonical tree)
//   k_segsum<SEG_LROWS>  z = M y                (rows of L, canonical tree, blend),
//                        + leaf partials of sum(z)
//   k_xt_coop            q_raw = X^T z          (columns, cooperative)
//   k_cg_step            cooperative: centring, p.q -> shift scalars -> r, r.r -> p
//   k_shift_update       sols / P for every active shift (side stream)
// k_spmv_rows (scipy's sequential row order) serves the X v probe API.
#pragma once

#include <cooperative_groups.h>

namespace fsda {

namespace cg = cooperative_groups;

constexpr int STAGE = 1024;    // column indices staged per warp and chunk
constexpr int ROW_WARPS = 8;   // warps per block in the row kernels

// Copy cols[c0, c1) into a warp's shared stage with 16-byte loads.  The copy
// starts at the 16-byte boundary below c0 (index arrays carry >= 4 ints of
// tail padding), so stage[j - base] holds cols[j].  Returns base.
__device__ __forceinline__ int stage_cols(const int* __restrict__ cols, int c0, int c1, int* st,
                                          int lane) {
  const int base = c0 & ~3;
  const int n4 = (c1 - base + 3) >> 2;
  const int4* src = reinterpret_cast<const int4*>(cols + base);
  int4* dst = reinterpret_cast<int4*>(st);
  for (int k = lane; k < n4; k += 32) dst[k] = __ldg(src + k);
  __syncwarp();
  return base;
}

// acc + v[st[j - base]] for j in [a, b), strictly in order; gathers batched 8
// deep for memory-level parallelism.
__device__ __forceinline__ double gather_sum(double acc, const int* st, int base, int a, int b,
                                             const double* __restrict__ v) {
  int j = a;
  for (; j + 8 <= b; j += 8) {
    double t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = __ldg(v + st[j + u - base]);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = acc + t[u];
  }
  for (; j < b; ++j) acc = acc + __ldg(v + st[j - base]);
  return acc;
}

// ------------------------------------------------------------- K1: y = X p
// A warp owns 32 consecutive rows (one per lane).  It streams the rows' column
// indices through shared memory with coalesced 16-byte loads, and each lane
// sums p over its own row sequentially in stored column order — the order of
// scipy's csr_matvec (sparse.py:121), so y is bit-identical to the reference.
__global__ void __launch_bounds__(256) k_spmv_rows(const int* __restrict__ rowptr,
                                                   const int* __restrict__ cols,
                                                   const double* __restrict__ p,
                                                   double* __restrict__ y, int n_rows,
                                                   const CgScalars* guard) {
  if (guard && loop_idle(guard)) return;
  __shared__ __align__(16) int stage[ROW_WARPS][STAGE + 8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long r0 = ((long long)blockIdx.x * ROW_WARPS + warp) * 32;
  if (r0 >= n_rows) return;
  const int row = (int)r0 + lane;
  const bool valid = row < n_rows;
  const int start = valid ? __ldg(rowptr + row) : 0;
  const int end = valid ? __ldg(rowptr + row + 1) : 0;
  const int last = (int)min(32LL, (long long)n_rows - r0) - 1;
  const int wlo = __shfl_sync(FULL, start, 0);
  const int whi = __shfl_sync(FULL, end, last);
  int* st = stage[warp];
  double acc = 0.0;
  for (int c0 = wlo; c0 < whi; c0 += STAGE) {
    const int c1 = min(c0 + STAGE, whi);
    const int base = stage_cols(cols, c0, c1, st, lane);
    const int a = max(start, c0), b = min(end, c1);
    if (a < b) acc = gather_sum(acc, st, base, a, b, p);
    __syncwarp();
  }
  if (valid) y[row] = acc;
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

// Canonical sum of a vector (sum(w) for the parity probes).
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

// R256 of m partials by one warp (m <= 65536); result in every lane.
__device__ __forceinline__ double warp_reduce_partials(const double* part, int m, int lane) {
  if (m <= LEAF) return warp_leaf(part, m, lane);
  const int m2 = (m + LEAF - 1) / LEAF;
  double acc = 0.0;
  for (int g = 0; g < m2; ++g) {
    const double r = warp_leaf(part + g * LEAF, min(LEAF, m - g * LEAF), lane);
    if ((g & 31) == lane) acc = acc + r;
  }
  return butterfly(acc);
}

// -------------------------------------------- segmented canonical sums
// X p (rows of X), L y (rows of L) and X^T z (columns of X) are all "sum the
// gathered terms of every segment with the canonical R256 tree".  A host-built
// plan sorts segments into classes by length:
//   class k (W = 1 << k, k = 0..5): segments with n <= 8W, 32/W per warp, one
//     W-lane group per segment, every lane holding <= 8 elements;
//   heavy: n > 256, warp tasks of <= 4 leaves; each leaf partial goes to
//     seg_part and the task that completes a segment (atomic counter,
//     self-resetting) reduces its leaves with the same tree.
// A W-lane group reproduces the canonical leaf exactly: lane t of the group
// keeps accumulator A_m = sum_k v[t + mW + 32k] (in k order, from 0.0) —
// the canonical lane t + mW — then combines A_m + A_{m+j} for j = M/2..1 and
// finishes with the butterfly over the W lanes.  Those are precisely the
// canonical xor-butterfly steps at offsets >= W and < W; accumulators that
// can only hold zeros are skipped (x + 0.0 == x).
enum SegKind : int { SEG_XROWS = 0, SEG_LROWS = 1, SEG_XCOLS = 2 };

struct SegPlan {
  const int* ind;            // index stream (X columns, L columns, or CSC rows)
  const int4* tasks;         // {segment, start, length, heavy id or -1}
  long long cls_off[7];      // class k tasks: [cls_off[k], cls_off[k+1]); heavy: [cls_off[6], ...)
  long long warp_base[9];    // warps: classes 0..5, heavy tasks (6), sum leaves (7), end (8)
  const int* heavy_seg0;     // first leaf partial of heavy segment h
  const int* heavy_nseg;     // leaves of heavy segment h
  const int* heavy_start;    // index-stream start of heavy segment h
  const int* heavy_ntask;    // warp tasks of heavy segment h
  const int* heavy_seg;      // segment id of heavy segment h
  unsigned* heavy_count;     // arrival counters
  double* seg_part;          // leaf partials
};

// V: storage type of the gathered vector src (double, or float for the
// fp32-storage mode); O: storage type of out (q stays double).  Every sum
// runs in double over the stored values; out is rounded to O once.
template <typename V, typename O>
struct SegArgsT {
  using value_type = V;
  const V* src;              // gathered vector: p, y or z
  O* out;                    // y, z or q (raw)
  // L rows: z = blend(alpha, masked y, alpha * (L y))
  const double* ldiag;
  const signed char* labels;
  double alpha;
  int alpha_mode;
  int row_base;              // global index of local row 0 (row-sharded L)
  // X^T columns: 0 raw, 1 centred (mu, *sum_ptr), 2 divided by ell
  int mode;
  const double* mu;
  const double* sum_ptr;
  double ell;
  // optional leaf partials of sum(src) (K3 in the loop: sum(z))
  double* sum_part;
  long long sum_n;
};
using SegArgs = SegArgsT<double, double>;
using SegArgs32 = SegArgsT<float, float>;     // K1 / K2 in fp32 storage
using SegArgs32D = SegArgsT<float, double>;   // K3 in fp32 storage: q in double

template <int KIND, typename A>
__device__ __forceinline__ double seg_term(const A& a, int seg, int idx, double dg) {
  const double v = (double)__ldg(a.src + idx);
  if (KIND == SEG_LROWS) return (idx == seg + a.row_base) ? dg * v : -v;
  return v;
}

// The row's own loads that seg_finish needs (L rows: the masked y_i), issued
// with the task so they do not add a round trip after the reduction.
template <int KIND, typename A>
__device__ __forceinline__ double seg_pre(const A& a, int seg) {
  if (KIND != SEG_LROWS) return 0.0;
  const signed char l = __ldg(a.labels + seg);
  const double y = (double)__ldg(a.src + seg + a.row_base);
  return l != 0 ? y : 0.0;
}

template <int KIND, typename A>
__device__ __forceinline__ void seg_finish(const A& a, int seg, double s, double masked) {
  if (KIND == SEG_XROWS) {
    a.out[seg] = s;
  } else if (KIND == SEG_LROWS) {
    const double smoothed = a.alpha * s;
    a.out[seg] = (a.alpha_mode == 1) ? smoothed : (1.0 - a.alpha) * masked + smoothed;
  } else {
    if (a.mode == 1) s = s - a.mu[seg] * (*a.sum_ptr);
    else if (a.mode == 2) s = s / a.ell;
    a.out[seg] = s;
  }
}

template <int KIND, typename A>
__device__ __forceinline__ void seg_finish(const A& a, int seg, double s) {
  seg_finish<KIND>(a, seg, s, seg_pre<KIND>(a, seg));
}

// Canonical leaf of segment elements [start, start+n) (n <= 8W) by a W-lane
// group; t = lane within the group; result in every lane of the group.
template <int W, int KIND, typename SA>
__device__ __forceinline__ double group_leaf(const SegPlan& pl, const SA& a, int seg, int start,
                                             int n, int t) {
  constexpr int M = 32 / W;
  constexpr int MA = M < 8 ? M : 8;
  constexpr int KA = W >= 8 ? W / 4 : 1;
  double dg = 0.0;
  if (KIND == SEG_LROWS && n > 0) dg = __ldg(a.ldiag + seg);
  int ix[MA * KA];
  double v[MA * KA];
#pragma unroll
  for (int m = 0; m < MA; ++m)
#pragma unroll
    for (int k = 0; k < KA; ++k) {
      const int e = t + m * W + 32 * k;
      ix[m * KA + k] = (e < n) ? __ldg(pl.ind + start + e) : 0;
    }
#pragma unroll
  for (int m = 0; m < MA; ++m)
#pragma unroll
    for (int k = 0; k < KA; ++k) {
      const int e = t + m * W + 32 * k;
      v[m * KA + k] = (e < n) ? seg_term<KIND, SA>(a, seg, ix[m * KA + k], dg) : 0.0;
    }
  double A[MA];
#pragma unroll
  for (int m = 0; m < MA; ++m) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < KA; ++k)
      if (t + m * W + 32 * k < n) acc = acc + v[m * KA + k];
    A[m] = acc;
  }
#pragma unroll
  for (int j = MA / 2; j >= 1; j >>= 1)
#pragma unroll
    for (int m = 0; m < j; ++m) A[m] = A[m] + A[m + j];
  double r = A[0];
#pragma unroll
  for (int off = W / 2; off >= 1; off >>= 1) r = r + __shfl_xor_sync(FULL, r, off);
  return r;
}

template <int W, int KIND, typename A>
__device__ __forceinline__ void seg_class_task(const SegPlan& pl, const A& a, int cls,
                                               long long tw, int lane) {
  const long long idx = pl.cls_off[cls] + (tw - pl.warp_base[cls]) * (32 / W) + lane / W;
  int4 tk = make_int4(-1, 0, 0, -1);
  if (idx < pl.cls_off[cls + 1]) tk = __ldg(pl.tasks + idx);
  const bool leader = tk.x >= 0 && (lane & (W - 1)) == 0;
  const double pre = leader ? seg_pre<KIND, A>(a, tk.x) : 0.0;
  const double s = group_leaf<W, KIND, A>(pl, a, tk.x, tk.y, tk.z, lane & (W - 1));
  if (leader) seg_finish<KIND, A>(a, tk.x, s, pre);
}

template <int KIND, typename A>
__device__ __forceinline__ void seg_heavy_task(const SegPlan& pl, const A& a, long long tw,
                                               int lane) {
  // heavy task: up to 4 consecutive leaves of one segment
  const int4 tk = __ldg(pl.tasks + pl.cls_off[6] + (tw - pl.warp_base[6]));
  const int h = tk.w;
  const int leaf0 = __ldg(pl.heavy_seg0 + h) + (tk.y - __ldg(pl.heavy_start + h)) / LEAF;
  for (int lf = 0; lf * LEAF < tk.z; ++lf) {
    const double s = group_leaf<32, KIND, A>(pl, a, tk.x, tk.y + lf * LEAF,
                                          min(LEAF, tk.z - lf * LEAF), lane);
    if (lane == 0) pl.seg_part[leaf0 + lf] = s;
  }
  int is_last = 0;
  if (lane == 0) {
    __threadfence();
    const unsigned old = atomicAdd(pl.heavy_count + h, 1u);
    is_last = (old == (unsigned)__ldg(pl.heavy_ntask + h) - 1u);
  }
  is_last = __shfl_sync(FULL, is_last, 0);
  if (is_last) {
    __threadfence();
    const double s = warp_reduce_partials(pl.seg_part + __ldg(pl.heavy_seg0 + h),
                                          __ldg(pl.heavy_nseg + h), lane);
    if (lane == 0) {
      seg_finish<KIND, A>(a, tk.x, s);
      pl.heavy_count[h] = 0u;
    }
  }
}

// Programmatic dependent launch: a kernel lets its successor's CTAs launch
// once all of its own CTAs are running (they fill the SMs its last wave
// leaves idle), and waits for its predecessor's completion and memory before
// touching the predecessor's output.  Both are no-ops without the launch
// attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <int KIND, typename A>
__global__ void __launch_bounds__(256, 6) k_segsum(SegPlan pl, A a, const CgScalars* sc,
                                                int guarded) {
  pdl_trigger();
  pdl_wait();
  if (guarded && loop_idle(sc)) return;
  const int lane = threadIdx.x & 31;
  const long long total = pl.warp_base[8];
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long tw = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); tw < total;
       tw += nwarps) {
    if (tw < pl.warp_base[6]) {
      int k = 0;
      while (tw >= pl.warp_base[k + 1]) ++k;
      switch (k) {
        case 0: seg_class_task<1, KIND, A>(pl, a, 0, tw, lane); break;
        case 1: seg_class_task<2, KIND, A>(pl, a, 1, tw, lane); break;
        case 2: seg_class_task<4, KIND, A>(pl, a, 2, tw, lane); break;
        case 3: seg_class_task<8, KIND, A>(pl, a, 3, tw, lane); break;
        case 4: seg_class_task<16, KIND, A>(pl, a, 4, tw, lane); break;
        default: seg_class_task<32, KIND, A>(pl, a, 5, tw, lane); break;
      }
      continue;
    }
    if (tw >= pl.warp_base[7]) {  // leaf partials of sum(src)
      const long long g = tw - pl.warp_base[7];
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const long long i = g * LEAF + k * 32 + lane;
        if (i < a.sum_n) s = s + (double)__ldg(a.src + i);
      }
      s = butterfly(s);
      if (lane == 0) a.sum_part[g] = s;
      continue;
    }
    seg_heavy_task<KIND, A>(pl, a, tw, lane);
  }
}

// ------------------------------------------ K3: X^T z, dense columns blocked
// Canonical column sum:
//   * n <= 256: the R256 leaf over z[rows] in row order;
//   * n > 256 and n < 8 nb (nb = ceil(N / XT_RB) row blocks): R256 over its
//     leaves of 256 entries;
//   * blocked ("dense": n > 256 and n >= 8 nb, i.e. at least 8 entries per
//     row block on average — the Zipf head): rows are cut into blocks of
//     XT_RB; the column's entries in block b are cut into leaves of 256 (an
//     empty block contributes one 0.0), and the column sum is R256 over all
//     those leaf sums in (block, leaf) order.
// The dense rule lets a CTA stage one XT_RB-row block of z in shared memory
// and serve every dense-column gather of that block from it.  Each (block,
// dense column) slice is one task of the W-class scheme (host plan per
// block), so a warp runs 32/W slices at once.  One cooperative launch:
//   phase 1  CTA per row block: stage z, run the block's slice tasks;
//            then warp tasks for the other columns (SegPlan, with the
//            leaf-combining heavy tasks) and the leaf partials of sum(z)
//   -- grid sync --
//   phase 2  one warp per dense column reduces its nb partials.
constexpr int XT_RB = 8192;             // rows per staged z block (64 KB of shared memory)
constexpr int XT_DENSE_PER_BLOCK = 8;   // blocked: n > 256 and n >= XT_DENSE_PER_BLOCK * nb
// k_xt_coop: two 24-warp CTAs per SM at <= 40 registers (measured: 1.04x / 1.06x
// cfg2 / cfg3 over one 32-warp CTA)
constexpr int XT_THREADS = 768;
constexpr int XT_CTAS_PER_SM = 2;
// phase-1b tasks claimed per ticket draw (halves the single-address atomics;
// measured 1.02x at cfg2 / cfg3 over 1, and 4 is worse at cfg2)
constexpr int XT_TICKET_CHUNK = 2;
// phase 2: dense columns with more leaf sums than this are reduced by a CTA
constexpr int XT_BIG_PARTS = 1024;

struct XtDense {
  const int* rows;        // CSC row indices
  const int4* tasks;      // {partial slot, start, length, -}, grouped by (block, class)
  const long long* boff;  // per block: 6 class starts + end; (nb + 1) * 7
  const long long* bwarp; // per block: warp prefixes of the 6 classes + total; nb * 7
  const int* col;         // dense id -> column
  const long long* poff;  // dense id -> first leaf-sum slot; n_dense + 1
  double* part;           // leaf sums, (block, leaf) order per dense column
  long long n_dense;
  int nb;
  int rb;                 // rows per block (XT_RB)
  int ticket_chunk;       // tasks claimed per ticket draw
  int splits;             // CTAs sharing one row block's slices
  const int* big;         // dense ids with more than XT_BIG_PARTS leaf sums (phase 2 by a CTA)
  long long n_big;
};

template <int W, typename V>
__device__ __forceinline__ void dense_slice_task(const XtDense& dn, const V* zs, int r0,
                                                 const long long* off, const long long* wb,
                                                 int cls, long long tw_local, int lane) {
  constexpr int M = 32 / W;
  constexpr int MA = M < 8 ? M : 8;
  constexpr int KA = W >= 8 ? W / 4 : 1;
  const long long idx = off[cls] + (tw_local - wb[cls]) * (32 / W) + lane / W;
  int4 tk = make_int4(-1, 0, 0, 0);
  if (idx < off[cls + 1]) tk = __ldg(dn.tasks + idx);
  const int t = lane & (W - 1);
  const int n = tk.z;
  int ix[MA * KA];
#pragma unroll
  for (int m = 0; m < MA; ++m)
#pragma unroll
    for (int k = 0; k < KA; ++k) {
      const int e = t + m * W + 32 * k;
      ix[m * KA + k] = (e < n) ? __ldg(dn.rows + tk.y + e) - r0 : 0;
    }
  double A[MA];
#pragma unroll
  for (int m = 0; m < MA; ++m) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < KA; ++k)
      if (t + m * W + 32 * k < n) acc = acc + (double)zs[ix[m * KA + k]];
    A[m] = acc;
  }
#pragma unroll
  for (int j = MA / 2; j >= 1; j >>= 1)
#pragma unroll
    for (int m = 0; m < j; ++m) A[m] = A[m] + A[m + j];
  double r = A[0];
#pragma unroll
  for (int off2 = W / 2; off2 >= 1; off2 >>= 1) r = r + __shfl_xor_sync(FULL, r, off2);
  if (tk.x >= 0 && t == 0) dn.part[tk.x] = r;
}

// z row block -> shared memory by one TMA bulk copy (cp.async.bulk, completion
// on an mbarrier), so staging costs one instruction and no registers.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  unsigned done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.b32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}

// Thread 0 copies src[0, n) to zs (16-byte-aligned src: the bulk part by TMA,
// an odd last element by a plain load); every thread waits for the bytes.
// The caller's __syncthreads() before the call retires the previous block's
// reads; the one after it publishes the odd element.
template <typename V>
__device__ __forceinline__ void stage_block(V* zs, const V* __restrict__ src, int n,
                                            unsigned long long* bar, unsigned phase) {
  if (threadIdx.x == 0) {
    const unsigned bytes = (unsigned)(sizeof(V) * n) & ~15u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
    if (bytes)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(zs)),
          "l"(src), "r"(bytes), "r"(smem_u32(bar))
          : "memory");
    for (int k = (int)(bytes / sizeof(V)); k < n; ++k) zs[k] = __ldg(src + k);
  }
  mbar_wait(bar, phase);
}

__device__ int g_xt_trace_on = 0;
__device__ unsigned long long g_xt_trace[5][1024];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define XT_MARK(k) \
  if (g_xt_trace_on && threadIdx.x == 0 && blockIdx.x < 1024) g_xt_trace[k][blockIdx.x] = gtimer();

template <typename A>
__global__ void __launch_bounds__(XT_THREADS, XT_CTAS_PER_SM) k_xt_coop(SegPlan pl, XtDense dn, A a,
                                                    const CgScalars* sc, int guarded, int n_rows,
                                                    unsigned long long* ticket, double* sum_out) {
  using V = typename A::value_type;
  pdl_trigger();
  pdl_wait();
  if (guarded && loop_idle(sc)) return;  // uniform across the grid
  extern __shared__ __align__(16) double zs_raw[];  // dn.rb values of z
  V* zs = reinterpret_cast<V*>(zs_raw);
  __shared__ unsigned long long zs_bar;
  __shared__ long long s_off[7], s_wb[7];  // the current row block's class starts / warp prefixes
  XT_MARK(0)
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // ---- phase 1a: (row block, split) units with their dense-column slices
  if (dn.n_dense > 0) {
    const bool tma = (reinterpret_cast<size_t>(a.src) & 15) == 0;
    if (threadIdx.x == 0) mbar_init(&zs_bar);
    unsigned phase = 0;
    const long long units = (long long)dn.nb * dn.splits;
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
      const int b = (int)(u / dn.splits), sp = (int)(u - (long long)b * dn.splits);
      const int r0 = b * dn.rb;
      const int nr = min(dn.rb, n_rows - r0);
      __syncthreads();
      if (threadIdx.x < 7) {
        s_off[threadIdx.x] = __ldg(dn.boff + (long long)b * 7 + threadIdx.x);
        s_wb[threadIdx.x] = __ldg(dn.bwarp + (long long)b * 7 + threadIdx.x);
      }
      if (tma) {
        stage_block(zs, a.src + r0, nr, &zs_bar, phase);
        phase ^= 1u;
      } else {
        for (int k = threadIdx.x; k < nr; k += blockDim.x) zs[k] = __ldg(a.src + r0 + k);
      }
      __syncthreads();
      const long long c0 = s_wb[6] * sp / dn.splits, c1 = s_wb[6] * (sp + 1) / dn.splits;
      for (long long tw = c0 + warp; tw < c1; tw += nw) {
        int k = 0;
        while (tw >= s_wb[k + 1]) ++k;
        switch (k) {
          case 0: dense_slice_task<1, V>(dn, zs, r0, s_off, s_wb, 0, tw, lane); break;
          case 1: dense_slice_task<2, V>(dn, zs, r0, s_off, s_wb, 1, tw, lane); break;
          case 2: dense_slice_task<4, V>(dn, zs, r0, s_off, s_wb, 2, tw, lane); break;
          case 3: dense_slice_task<8, V>(dn, zs, r0, s_off, s_wb, 3, tw, lane); break;
          case 4: dense_slice_task<16, V>(dn, zs, r0, s_off, s_wb, 4, tw, lane); break;
          default: dense_slice_task<32, V>(dn, zs, r0, s_off, s_wb, 5, tw, lane); break;
        }
      }
    }
  }
  __syncthreads();
  XT_MARK(1)
  // ---- phase 1b: the other columns and the sum(z) leaves; warps draw tasks
  // from a grid-wide ticket so CTAs that staged a dense block catch up.
  const long long total = pl.warp_base[8];
  const long long nheavy = pl.warp_base[7] - pl.warp_base[6];
  const int chunk = dn.ticket_chunk;
  for (;;) {
    long long base = 0;
    if (lane == 0) base = (long long)atomicAdd(ticket, (unsigned long long)chunk);
    base = __shfl_sync(FULL, base, 0);
    if (base >= total) break;
    const long long lim = min(base + chunk, total);
    for (long long nxt = base; nxt < lim; ++nxt) {
    // largest tasks first: tickets [0, nheavy) are the heavy tasks, then the
    // class tasks, then the sum(z) leaves
    const long long tw = nxt < nheavy ? pl.warp_base[6] + nxt
                                      : (nxt < pl.warp_base[7] ? nxt - nheavy : nxt);
    if (tw < pl.warp_base[6]) {
      int k = 0;
      while (tw >= pl.warp_base[k + 1]) ++k;
      switch (k) {
        case 0: seg_class_task<1, SEG_XCOLS, A>(pl, a, 0, tw, lane); break;
        case 1: seg_class_task<2, SEG_XCOLS, A>(pl, a, 1, tw, lane); break;
        case 2: seg_class_task<4, SEG_XCOLS, A>(pl, a, 2, tw, lane); break;
        case 3: seg_class_task<8, SEG_XCOLS, A>(pl, a, 3, tw, lane); break;
        case 4: seg_class_task<16, SEG_XCOLS, A>(pl, a, 4, tw, lane); break;
        default: seg_class_task<32, SEG_XCOLS, A>(pl, a, 5, tw, lane); break;
      }
    } else if (tw < pl.warp_base[7]) {
      seg_heavy_task<SEG_XCOLS, A>(pl, a, tw, lane);
    } else {
      const long long g = tw - pl.warp_base[7];
      double v = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const long long i = g * LEAF + k * 32 + lane;
        if (i < a.sum_n) v = v + (double)__ldg(a.src + i);
      }
      v = butterfly(v);
      if (lane == 0) a.sum_part[g] = v;
    }
    }
  }
  __syncthreads();
  XT_MARK(2)
  grid.sync();
  XT_MARK(3)
  if (blockIdx.x == 0 && threadIdx.x == 0) *ticket = 0ULL;  // every warp has drawn its last ticket
  const long long nwarps = (long long)gridDim.x * nw;
  // sum(z) from its leaf partials (the CG step's centring needs it): the last
  // CTA, whose warps hold the fewest dense columns, reduces it with the same
  // tree as k_cg_step's block_reduce_partials would
  if (sum_out && blockIdx.x == gridDim.x - 1) {
    const double s = block_reduce_partials(a.sum_part, (a.sum_n + LEAF - 1) / LEAF, zs_raw);
    if (threadIdx.x == 0) *sum_out = s;
  }
  // ---- phase 2: dense columns.  Columns with more than XT_BIG_PARTS leaf
  // sums (the Zipf head at large N) are reduced by a whole CTA each
  // (block_reduce_partials: the same R256 tree, leaves spread over the warps),
  // the others by one warp each.
  for (long long i = blockIdx.x; i < dn.n_big; i += gridDim.x) {
    const int h = __ldg(dn.big + i);
    const long long p0 = __ldg(dn.poff + h);
    const double v = block_reduce_partials(dn.part + p0, __ldg(dn.poff + h + 1) - p0, zs_raw);
    if (threadIdx.x == 0) seg_finish<SEG_XCOLS, A>(a, __ldg(dn.col + h), v);
  }
  const long long gw = (long long)blockIdx.x * nw + warp;
  for (long long h = gw; h < dn.n_dense; h += nwarps) {
    const long long p0 = __ldg(dn.poff + h);
    const int m = (int)(__ldg(dn.poff + h + 1) - p0);
    if (m > XT_BIG_PARTS) continue;
    const double v = warp_reduce_partials(dn.part + p0, m, lane);
    if (lane == 0) seg_finish<SEG_XCOLS, A>(a, __ldg(dn.col + h), v);
  }
  __syncthreads();
  XT_MARK(4)
}

// bptr[h * (nb + 1) + b] = first position in column dense_col[h] whose row is
// >= b * XT_RB (b = nb gives the column end).
__global__ void k_heavy_bptr(const int* __restrict__ colptr, const int* __restrict__ rows,
                             const int* __restrict__ heavy_col, int* __restrict__ bptr,
                             long long n_heavy, int nb, int rb) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_heavy * (nb + 1)) return;
  const long long h = t / (nb + 1);
  const int b = (int)(t - h * (nb + 1));
  const int c = heavy_col[h];
  int lo = colptr[c], hi = colptr[c + 1];
  if (b == nb) { bptr[t] = hi; return; }
  const int target = b * rb;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (rows[mid] < target) lo = mid + 1; else hi = mid;
  }
  bptr[t] = lo;
}

// z = masked y (apply_smoother at alpha == 0: no Laplacian term, sda.py:135-136).
template <typename V>
__global__ void k_mask_labeled(const V* __restrict__ y, const signed char* __restrict__ labels,
                               V* __restrict__ z, int n, const CgScalars* sc, int guarded,
                               int row_base) {
  if (guarded && loop_idle(sc)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) z[i] = labels[i] != 0 ? y[i + row_base] : (V)0;
}

// q[i] = q[i] - mu[i] * q[d]  (centring of an all-reduced [X^T z | sum z]),
// or q[i] = q[i] / scale when mu is null (labeled mean).
__global__ void k_center(const double* __restrict__ mu, double* __restrict__ q, long long d,
                         double scale) {
  const double s = mu ? q[d] : 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < d;
       i += (long long)gridDim.x * blockDim.x)
    q[i] = mu ? q[i] - mu[i] * s : q[i] / scale;
}

// -------------------------------------------- K4: one cooperative CG step
// krylov.py:211-268 for the base system in one launch with two grid-wide
// barriers.  Warp w owns 256-element leaf w (plus leaves w + total_warps, ...
// when d is larger than the grid covers); the first leaf's p, q, r and the
// centring coefficient are loaded into registers at entry, together with the
// shift state, so each phase waits on one round of loads (its partials):
//   A  sum(z) (leaf partials from K2/K3), centring of q, leaf partials of p.q
//   -- grid sync --
//   B  every block finishes p.q (identical tree, identical result), derives
//      gamma and the per-shift zeta_next / gamma_s / good flags; r_next = r +
//      gamma q with leaf partials of r_next.r_next
//   -- grid sync --
//   C  every block finishes r.r and alpha_new; p = r_next + alpha_new p from
//      registers; block 0 retires converged / degenerate shifts, rolls zeta,
//      writes the shift-update snapshot for k_shift_update, advances the
//      iteration, and sets the while-loop condition.
// Scalars needed after block 0 starts writing them are read into registers
// at kernel entry, so no block reads state that block 0 modifies.
constexpr int STEP_THREADS = 256;

// V: storage of p and the residual slots (double, or float in the fp32-storage
// mode: every update is computed in double and rounded once when stored; the
// dots run over the stored values).
template <typename V>
__global__ void __launch_bounds__(STEP_THREADS) k_cg_step(
    double* __restrict__ q, V* __restrict__ p, V* __restrict__ rbuf, int nslots,
    double* __restrict__ bigp, double* __restrict__ sols, long long d,
    double* __restrict__ part_pq, double* __restrict__ part_rr, long long n_leaf, CgScalars* sc,
    ShiftState ss, int ns, unsigned long long cond_handle, int use_cond,
    const double* __restrict__ mu, const double* __restrict__ part_z, long long n_leaf_z,
    const signed char* __restrict__ labels, double ell, const double* sum_ready) {
  extern __shared__ double dyn[];  // zn[ns], gs[ns], good[ns] (as double)
  __shared__ double smem[257];
  __shared__ int s_flag;
  double* s_zn = dyn;
  double* s_gs = dyn + ns;
  double* s_good = dyn + 2 * ns;
  cg::grid_group grid = cg::this_grid();
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;

  if (leader && use_cond) ++sc->body_runs;
  const int idle = loop_idle(sc);
  const long long it = sc->iter;
  const double rr = sc->rr, gp = sc->gamma_prev, al = sc->alpha, thresh = sc->thresh;
  const long long max_iter = sc->max_iter;
  const long long runs = sc->body_runs;
  if (idle) {
    if (leader && use_cond) cudaGraphSetConditional((cudaGraphConditionalHandle)cond_handle, 0u);
    return;
  }

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + warp;
  const long long tw = (long long)gridDim.x * (blockDim.x >> 5);
  // residual slots: ping-pong (nslots 2) or the stored basis r_0 .. r_K
  const V* r_cur = rbuf + (it % nslots) * d;
  V* r_next = rbuf + ((it + 1) % nslots) * d;
  const bool center = part_z != nullptr;
  const bool own = gw < n_leaf;  // this warp's register-cached leaf

  // ---- entry loads: the cached leaf and this thread's first shift
  double pr[8], qr[8], rv[8], cr[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const long long i = gw * LEAF + k * 32 + lane;
    const bool in = own && i < d;
    pr[k] = in ? (double)p[i] : 0.0;
    rv[k] = in ? (double)r_cur[i] : 0.0;
    cr[k] = (in && center) ? (mu ? mu[i] : (labels[i] != 0 ? 1.0 : 0.0)) : 0.0;
  }
  // everything above is this step's own state; q and the sum(z) leaves come
  // from the X^T kernel, which may still be finishing (programmatic launch)
  pdl_wait();
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const long long i = gw * LEAF + k * 32 + lane;
    qr[k] = (own && i < d) ? q[i] : 0.0;
  }
  const int s0 = threadIdx.x;
  int act0 = 0;
  double zp0 = 0.0, z0 = 0.0, b0 = 0.0;
  if (s0 < ns) {
    act0 = ss.active[s0];
    zp0 = ss.zeta_prev[s0];
    z0 = ss.zeta[s0];
    b0 = ss.beta[s0];
  }

  // ---- A: centring q = X^T z - mu sum(z) (sparse.py:277) or, for SA-SDA,
  // M z - 1_l (sum(M z) / l) (sda.py:155-157); then the p.q leaves
  double sz = 0.0;
  if (center) {
    const double sum_z = sum_ready ? *sum_ready : block_reduce_partials(part_z, n_leaf_z, smem);
    sz = mu ? sum_z : sum_z / ell;
  }
  if (own) {
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (gw * LEAF + k * 32 + lane < d) {
        if (center) qr[k] = qr[k] - cr[k] * sz;
        a = fma(pr[k], qr[k], a);
      }
    }
    a = butterfly(a);
    if (lane == 0) part_pq[gw] = a;
  }
  for (long long g = gw + tw; g < n_leaf; g += tw) {
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const long long i = g * LEAF + k * 32 + lane;
      if (i < d) {
        double qi = q[i];
        if (center) {
          qi = qi - (mu ? mu[i] : (labels[i] != 0 ? 1.0 : 0.0)) * sz;
          q[i] = qi;
        }
        a = fma((double)p[i], qi, a);
      }
    }
    a = butterfly(a);
    if (lane == 0) part_pq[g] = a;
  }
  grid.sync();

  // ---- B: scalars, then r_next = r + gamma q and its r.r leaves (krylov.py:232-233)
  const double pq = block_reduce_partials(part_pq, n_leaf, smem);
  if (!isfinite(pq) || pq == 0.0) {
    if (leader) {
      sc->status = isfinite(pq) ? ST_BREAKDOWN : ST_NONFINITE;
      sc->fail_iter = it;
      sc->finished = 1;
      if (use_cond) cudaGraphSetConditional((cudaGraphConditionalHandle)cond_handle, 0u);
    }
    return;  // uniform: every block computed the same pq
  }
  const double gamma = -rr / pq;
  for (int s = threadIdx.x; s < ns; s += blockDim.x) {
    const bool first = s == s0;
    double zn = 0.0, gs = 0.0, good = 0.0;
    if (first ? act0 : ss.active[s]) {
      const double zp = first ? zp0 : ss.zeta_prev[s], z = first ? z0 : ss.zeta[s];
      const double beta = first ? b0 : ss.beta[s];
      const double denom = gamma * al * (zp - z) + zp * gp * (1.0 - beta * gamma);
      zn = zp * z * gp / denom;
      if (isfinite(zn) && !(fabs(zn) < 1e-290)) {
        good = 1.0;
        gs = gamma * zn / z;
      }
    }
    s_zn[s] = zn;
    s_gs[s] = gs;
    s_good[s] = good;
  }
  if (own) {
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const long long i = gw * LEAF + k * 32 + lane;
      if (i < d) {
        const V st = (V)(rv[k] + gamma * qr[k]);
        r_next[i] = st;
        rv[k] = (double)st;
        a = fma(rv[k], rv[k], a);
      }
    }
    a = butterfly(a);
    if (lane == 0) part_rr[gw] = a;
  }
  for (long long g = gw + tw; g < n_leaf; g += tw) {
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const long long i = g * LEAF + k * 32 + lane;
      if (i < d) {
        const V st = (V)((double)r_cur[i] + gamma * q[i]);
        r_next[i] = st;
        const double rn = (double)st;
        a = fma(rn, rn, a);
      }
    }
    a = butterfly(a);
    if (lane == 0) part_rr[g] = a;
  }
  grid.sync();

  // ---- C: r.r, alpha_new, p, bookkeeping
  const double rr_new = block_reduce_partials(part_rr, n_leaf, smem);
  if (!isfinite(rr_new)) {
    if (leader) {
      sc->status = ST_NONFINITE;
      sc->fail_iter = it;
      sc->finished = 1;
      if (use_cond) cudaGraphSetConditional((cudaGraphConditionalHandle)cond_handle, 0u);
    }
    return;
  }
  const double alpha_new = rr_new / rr;
  if (own) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const long long i = gw * LEAF + k * 32 + lane;
      if (i < d) p[i] = (V)(rv[k] + alpha_new * pr[k]);
    }
  }
  for (long long g = gw + tw; g < n_leaf; g += tw) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const long long i = g * LEAF + k * 32 + lane;
      if (i < d) p[i] = (V)((double)r_next[i] + alpha_new * (double)p[i]);  // this thread wrote r_next[i] in B
    }
  }
  if (blockIdx.x != 0) return;
  if (threadIdx.x == 0) s_flag = 0;
  __syncthreads();
  const double r_norm = sqrt(rr_new);
  for (int s = threadIdx.x; s < ns; s += blockDim.x) {
    const bool first = s == s0;
    ss.upd_mode[s] = 0;
    if (!(first ? act0 : ss.active[s])) continue;
    if (s_good[s] == 0.0) {  // degenerate zeta: freeze untouched (krylov.py:251-255)
      ss.iters[s] = it + 1;
      ss.resid[s] = __longlong_as_double(0x7ff0000000000000LL);
      ss.active[s] = 0;
      continue;
    }
    const double zn = s_zn[s], z = first ? z0 : ss.zeta[s], gs = s_gs[s];
    const double as = alpha_new * (zn * gs) / (z * gamma);
    ss.alpha_s[s] = as;
    ss.upd_gs[s] = gs;
    ss.upd_zn[s] = zn;
    ss.upd_as[s] = as;
    const double shift_res = fabs(zn) * r_norm;
    if (shift_res < thresh) {  // converged: freeze after its last sols update (krylov.py:256-261)
      ss.iters[s] = it + 1;
      ss.resid[s] = shift_res;
      ss.conv[s] = 1;
      ss.active[s] = 0;
      ss.upd_mode[s] = 1;
    } else {
      ss.zeta_prev[s] = z;
      ss.zeta[s] = zn;
      ss.upd_mode[s] = 3;
      atomicAdd(&s_flag, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int n_active = s_flag;
    sc->gamma_prev = gamma;
    sc->alpha = alpha_new;
    sc->alpha_new = alpha_new;
    sc->gamma = gamma;
    sc->rr = rr_new;
    sc->iter = it + 1;
    sc->n_active = n_active;
    const int fin = (n_active == 0 || it + 1 >= max_iter) ? 1 : 0;
    if (fin) sc->finished = 1;
    if (use_cond) {
      unsigned keep = fin ? 0u : 1u;
      if (runs > max_iter + 1) keep = 0u;  // never spin past the iteration budget
      cudaGraphSetConditional((cudaGraphConditionalHandle)cond_handle, keep);
    }
  }
}

// The shift updates of the iteration whose snapshot k_cg_step wrote
// (krylov.py:230, 240-241): sols_s -= gamma_s P_s, then P_s = zeta_next r +
// alpha_s P_s for shifts still active.  r is the current residual r_{i+1}.
// A block covers SU_ELEMS * 256 rows for SU_SHIFTS shifts, so r is read once
// per SU_SHIFTS shifts and every thread keeps 2 * SU_ELEMS loads in flight.
// Launched on a second stream beside the next iteration's sparse kernels
// (guarded: skipped once the loop is idle) and once more, unguarded, after the
// loop for the final iteration.
constexpr int SU_ELEMS = 4;
constexpr int SU_SHIFTS = 4;

__global__ void __launch_bounds__(256) k_shift_update(const double* __restrict__ rbuf, int nslots,
                                                      double* __restrict__ bigp,
                                                      double* __restrict__ sols, long long d,
                                                      ShiftState ss, const CgScalars* sc,
                                                      int ns, int guarded) {
  if (guarded && loop_idle(sc)) return;
  const double* r = rbuf + (sc->iter % nslots) * d;
  const long long base = (long long)blockIdx.x * (256 * SU_ELEMS) + threadIdx.x;
  double rv[SU_ELEMS];
#pragma unroll
  for (int e = 0; e < SU_ELEMS; ++e) {
    const long long i = base + e * 256;
    rv[e] = i < d ? __ldcg(r + i) : 0.0;
  }
  for (int sj = 0; sj < SU_SHIFTS; ++sj) {
    const int s = blockIdx.y * SU_SHIFTS + sj;
    if (s >= ns) break;
    const int mode = ss.upd_mode[s];
    if (mode == 0) continue;
    const double gs = ss.upd_gs[s], zn = ss.upd_zn[s], as = ss.upd_as[s];
    double* P = bigp + (long long)s * d;
    double* X = sols + (long long)s * d;
    double pv[SU_ELEMS], xv[SU_ELEMS];
#pragma unroll
    for (int e = 0; e < SU_ELEMS; ++e) {
      const long long i = base + e * 256;
      pv[e] = i < d ? P[i] : 0.0;
      xv[e] = i < d ? X[i] : 0.0;
    }
#pragma unroll
    for (int e = 0; e < SU_ELEMS; ++e) {
      const long long i = base + e * 256;
      if (i < d) {
        X[i] = xv[e] - pv[e] * gs;
        if (mode == 3) P[i] = zn * rv[e] + as * pv[e];
      }
    }
  }
}

// Deferred ("basis") shift updates.  With every residual r_0 .. r_K kept,
// P_s and sols_s are linear combinations of them, so an iteration only
// updates the coefficient rows (krylov.py:230, 240-241 on coefficients):
//   sols_s -= gamma_s P_s   ->  c_s[j] = c_s[j] - a_s[j] * gamma_s   (j <= i)
//   P_s = zeta_next r_{i+1} + alpha_s P_s
//                           ->  a_s[j] = alpha_s * a_s[j] (j <= i), a_s[i+1] = zeta_next
// and the directions are formed once, after the loop (k_combine_basis).  The
// per-iteration shift traffic (32 D n_s bytes) becomes O(n_s K) scalars.
// blockIdx.y = shift; threads over j.  Same guard / snapshot contract as
// k_shift_update.
__global__ void __launch_bounds__(256) k_coef_update(ShiftState ss, const CgScalars* sc, int ns,
                                                     int guarded) {
  if (guarded && loop_idle(sc)) return;
  const int s = blockIdx.y;
  const int mode = ss.upd_mode[s];
  if (mode == 0) return;
  const long long i = sc->iter - 1;  // the iteration the snapshot belongs to
  const double gs = ss.upd_gs[s], zn = ss.upd_zn[s], as = ss.upd_as[s];
  double* A = ss.coef_a + (long long)s * ss.coef_ld;
  double* Cc = ss.coef_c + (long long)s * ss.coef_ld;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j <= i + 1;
       j += (long long)gridDim.x * blockDim.x) {
    if (j <= i) {
      const double a = A[j];
      Cc[j] = Cc[j] - a * gs;
      if (mode == 3) A[j] = as * a;
    } else if (mode == 3 && j < ss.coef_ld) {
      A[j] = zn;
    }
  }
}

// sols[s][k] = sum_{j < J} c_s[j] * r_j[k], j ascending from 0.0 with one
// fused multiply-add per term, J = iterations run.  A thread owns
// one feature k for SH shifts; r_j[k] loads are coalesced and the
// coefficient tile sits in shared memory (broadcast reads).
constexpr int CB_SH = 16;    // shifts per thread
constexpr int CB_JT = 128;   // coefficient columns per shared tile
template <typename V>
__global__ void __launch_bounds__(256) k_combine_basis(const V* __restrict__ rbuf, long long d,
                                                       ShiftState ss, const CgScalars* sc, int ns,
                                                       double* __restrict__ sols) {
  __shared__ double ct[CB_SH][CB_JT];
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int s0 = blockIdx.y * CB_SH;
  const int nsh = min(CB_SH, ns - s0);
  const long long J = sc->status == ST_OK ? sc->iter : 0;
  double acc[CB_SH];
#pragma unroll
  for (int t = 0; t < CB_SH; ++t) acc[t] = 0.0;
  for (long long j0 = 0; j0 < J; j0 += CB_JT) {
    const int jn = (int)min((long long)CB_JT, J - j0);
    __syncthreads();
    for (int e = threadIdx.x; e < CB_SH * CB_JT; e += blockDim.x) {
      const int t = e / CB_JT, jj = e - t * CB_JT;
      ct[t][jj] = (t < nsh && jj < jn) ? ss.coef_c[(long long)(s0 + t) * ss.coef_ld + j0 + jj] : 0.0;
    }
    __syncthreads();
    if (k < d) {
      for (int jj = 0; jj < jn; ++jj) {
        const double r = (double)__ldcs(rbuf + (j0 + jj) * d + k);
#pragma unroll
        for (int t = 0; t < CB_SH; ++t) acc[t] = fma(ct[t][jj], r, acc[t]);
      }
    }
  }
  if (k < d) {
#pragma unroll
    for (int t = 0; t < CB_SH; ++t)
      if (t < nsh) sols[(long long)(s0 + t) * d + k] = acc[t];
  }
}

// ------------------------------------------------------- projection SpMM
// scores[s * N + i] = sum over row i of W[c * ns + s] (W = directions,
// feature-major).  A warp owns a row; lane s owns shift s and adds W[c, s]
// for the row's columns in stored order — what scipy does for each
// x.matvec(w) (sda.py:279), so scores == X @ w bit for bit.  A row's column
// indices are read once per 32 shifts; the W row gathers are coalesced.
__global__ void __launch_bounds__(256) k_spmm_scores(const int* __restrict__ rowptr,
                                                     const int* __restrict__ cols,
                                                     const double* __restrict__ w,
                                                     double* __restrict__ scores, int n_rows,
                                                     int ns) {
  const int lane = threadIdx.x & 31;
  const long long row = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= n_rows) return;
  const int lo = __ldg(rowptr + row), hi = __ldg(rowptr + row + 1);
  for (int s0 = 0; s0 < ns; s0 += 32) {
    const int s = s0 + lane;
    const bool on = s < ns;
    double acc = 0.0;
    for (int j0 = lo; j0 < hi; j0 += 32) {
      const int cnt = min(32, hi - j0);
      const int mycol = (lane < cnt) ? __ldg(cols + j0 + lane) : 0;
      int u = 0;
      for (; u + 8 <= cnt; u += 8) {
        double t[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int c = __shfl_sync(FULL, mycol, u + k);
          t[k] = on ? __ldg(w + (long long)c * ns + s) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc = acc + t[k];
      }
      for (; u < cnt; ++u) {
        const int c = __shfl_sync(FULL, mycol, u);
        acc = acc + (on ? __ldg(w + (long long)c * ns + s) : 0.0);
      }
    }
    if (on) scores[(long long)s * n_rows + row] = acc;
  }
}

}  // namespace fsda
