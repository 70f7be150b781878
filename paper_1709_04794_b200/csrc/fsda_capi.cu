// fsda_capi.cu — context, uploads, solve orchestration and the C ABI declared
// in include/fsda_b200.h.
//
// One solve = one CUDA graph: setup kernels (labeled mean, rhs, CG init), a
// conditional WHILE node whose body is one shifted-CG iteration (7 kernels),
// and the projection kernels.  The body's last kernel sets the loop condition
// from the device-side "finished" flag, so the graph runs exactly as many
// iterations as the reference's Python loop (krylov.py:210-270) without any
// host round trip.  The eager path (same kernels, host loop) serves the
// per-kernel profiler and is the fallback when conditional nodes are absent.
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>

#if defined(__x86_64__)
#include <immintrin.h>
#endif
#include <omp.h>
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fsda_b200.h"
#include "fsda_device.cuh"
#include "fsda_hot.cuh"
#include "fsda_batch.cuh"
#include "graph_knn.cuh"
#include "graph_gemm.cuh"

#include <cub/device/device_select.cuh>

using namespace fsda;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

// FSDA_B200_TRACE=1 prints host-visible phase times of the upload / solve
// calls to stderr (the e2e breakdown; tools/time_e2e.py).
struct Trace {
  bool on = std::getenv("FSDA_B200_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[fsda trace] %-24s %8.3f ms\n", what,
            std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// Host threads of the upload passes: two fewer than the machine has (unless
// OMP_NUM_THREADS or FSDA_B200_HOST_THREADS says otherwise).  The CUDA driver's
// own threads, the calling thread's copies and the Python side need cores too:
// with every core in the OpenMP team, one drop-in call in ten took 20-50 ms
// longer on a 16-vCPU box (mean 120-125 ms against 114-115 ms with 14 threads).
int host_threads() {
  static const int v = [] {
    if (const char* e = std::getenv("FSDA_B200_HOST_THREADS")) return std::max(1, std::atoi(e));
    if (std::getenv("OMP_NUM_THREADS")) return std::max(1, omp_get_max_threads());
    const int procs = omp_get_num_procs();
    return std::max(1, std::min(omp_get_max_threads(), procs > 4 ? procs - 2 : procs));
  }();
  return v;
}

struct CudaError {
  cudaError_t err;
  const char* what;
  int line;
};

#define CK(call)                                                         \
  do {                                                                   \
    cudaError_t e_ = (call);                                             \
    if (e_ != cudaSuccess) throw CudaError{e_, #call, __LINE__};         \
  } while (0)
#define CKL() CK(cudaGetLastError())

// Bumped on every device (re)allocation; part of the graph cache key so a
// cached graph never holds a stale buffer pointer.
std::atomic<unsigned long long> g_alloc_gen{0};  // bumped from any thread / context

template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t cap = 0;  // elements
  void ensure(size_t n) {
    if (n <= cap && ptr) return;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    size_t alloc = std::max<size_t>(n, 1);
    CK(cudaMalloc(&ptr, alloc * sizeof(T)));
    cap = alloc;
    ++g_alloc_gen;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
  }
};

// Page-locked host staging for the upload plans (async H2D; reused across
// uploads, which synchronise before returning).
struct PinnedBuf {
  void* ptr = nullptr;
  size_t cap = 0;  // bytes
  void* ensure(size_t bytes) {
    if (bytes <= cap && ptr) return ptr;
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    cap = 0;
    const size_t alloc = std::max<size_t>(bytes + bytes / 4, 4096);
    CK(cudaHostAlloc(&ptr, alloc, cudaHostAllocDefault));
    cap = alloc;
    return ptr;
  }
  void release() {
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    cap = 0;
  }
};

inline long long cdiv(long long a, long long b) { return (a + b - 1) / b; }
inline long long n_leaves(long long n) { return cdiv(n, LEAF); }
constexpr long long MAX_REDUCE = 65536LL * LEAF;  // two-level R256 limit

// One kernel launch seen by the profiler.
struct Launch {
  const char* name;
  double bytes;
};

// Device side of one segmented-sum plan (see SegPlan in fsda_hot.cuh).
struct HostPlan {
  DevBuf<int4> tasks;
  DevBuf<int> h0, hn, hs, ht, hseg;
  DevBuf<unsigned> hc;
  DevBuf<double> part;
  PinnedBuf stage;
  long long n_heavy = 0, n_heavy_leaves = 0;  // heavy segments and their leaves
  SegPlan pl{};
  void release() {
    tasks.release(); h0.release(); hn.release(); hs.release(); ht.release(); hseg.release();
    hc.release();
    part.release(); stage.release();
  }
};

}  // namespace

// Device buffers of the multi-task batch (fsda_solve_batch), task-minor.
struct BatchBufs {
  DevBuf<signed char> lab, labt;
  DevBuf<double> ind, P, Q, R0, R1, MU, Bv, PR, Y, Z, BIGP, SOLS, SCORES, OUT;
  DevBuf<double> RB, CA, CC;  // deferred mode: residual slots, coefficient rows
  DevBuf<int2> gchunks;       // long X^T units: {unit, 256-partial group}
  DevBuf<int> gsoff;          // per unit: first group-leaf slot, or -1
  DevBuf<double> gsum;        // group leaves [slot][TP]
  DevBuf<double> partD, partN, part2, hpart, xpart, opart, scal;
  DevBuf<long long> lscal;
  DevBuf<int> iscal;
  DevBuf<double> sh_d;
  DevBuf<long long> sh_l;
  DevBuf<unsigned char> sh_u;
  DevBuf<int> sh_i;
  DevBuf<double> betas;
  DevBuf<char> raw;
  void release() {
    lab.release(); labt.release(); ind.release(); P.release(); Q.release(); R0.release(); R1.release();
    MU.release(); Bv.release(); PR.release(); Y.release(); Z.release(); BIGP.release();
    SOLS.release(); SCORES.release(); OUT.release(); partD.release(); partN.release();
    RB.release(); CA.release(); CC.release();
    gchunks.release(); gsoff.release(); gsum.release();
    hpart.release(); xpart.release(); opart.release(); scal.release(); lscal.release();
    part2.release();
    iscal.release(); sh_d.release(); sh_l.release(); sh_u.release(); sh_i.release();
    betas.release(); raw.release();
  }
};

// Tanimoto k-NN graph build (graph_knn.cuh) and its last result.
struct GraphBufs {
  DevBuf<int> head_of, cand, ncand, nbr, rsize, tsize;
  DevBuf<signed char> A;
  DevBuf<HeadCount> C;
  DevBuf<unsigned long long> keys, keys2;
  DevBuf<unsigned char> temp;
  DevBuf<long long> offs, cols, count;
  long long n = 0, nnz = 0;
  double tail_avg = 0.0;  // tail-column occurrences per row of the last build
  CUtensorMap amap{};            // TMA descriptor of A (re-encoded per build)
  long long block_rows = 0;      // rows per GEMM / scan block of the current build
  bool gemm_attr = false;        // k_head_gemm's shared-memory opt-in done
  void release() {
    head_of.release(); cand.release(); ncand.release(); nbr.release(); rsize.release(); tsize.release(); A.release();
    C.release();
    keys.release(); keys2.release(); temp.release(); offs.release(); cols.release(); count.release();
  }
};

struct fsda_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::mutex mu;
  int num_sms = 148;

  // X: CSR + CSC (int32 indices, value-free)
  long long n = 0, d = 0, nnz = 0;
  bool has_x = false;
  DevBuf<int> x_rowptr, x_cols, csc_colptr, csc_rows;
  // upload scratch (persistent so that repeated uploads of same-size data do
  // not reallocate and the cached solve graph stays valid)
  DevBuf<long long> scratch_i64, scratch_l64;  // raw int64 indices of X / of L
  DevBuf<double> scratch_f64;
  DevBuf<int> scratch_row_of, scratch_keys;
  DevBuf<unsigned char> scratch_sort;
  // segmented-sum plans: rows of X, rows of L, light columns of X
  HostPlan plan_xr, plan_lr, plan_xc;
  // dense columns of X (blocked by rows, see k_xt_coop)
  DevBuf<int> xh_col, xh_bptr, xh_big;
  DevBuf<int4> xh_tasks;
  DevBuf<long long> xh_boff, xh_bwarp, xh_poff;
  long long xh_ntasks = 0, xh_nslots = 0;
  BatchBufs batch;
  GraphBufs knn;
  PinnedBuf xh_stage;
  DevBuf<double> xh_part;
  XtDense xh{};
  int xt_blocks = 0;
  DevBuf<unsigned long long> xt_ticket;  // phase-1b work ticket (reset by the kernel)
  int step_blocks = 0;  // cooperative grid of k_cg_step
  bool batch_attrs_set = false;  // kb_* dynamic shared-memory opt-in done on this device

  // L: CSR with diagonal entries in place, diag values split out.  Row-sharded
  // contexts hold rows [row_base, row_base + n) of an n_global-row L.
  long long row_base = 0, n_global = 0;
  bool has_l = false;
  long long l_nnz = 0;
  DevBuf<int> l_rowptr, l_cols;
  DevBuf<double> l_diag;

  // labels
  bool has_labels = false;
  DevBuf<signed char> labels;
  long long n1 = 0, n2 = 0, ell = 0;

  // work vectors
  DevBuf<double> y, z, q, p, mu_v, t, wv, b, ind, probe, part_n, part_d, part_d2, part_o;
  // residual slots: 2 (ping-pong, per-iteration shift updates) or max_iter + 1
  // (the stored basis r_0 .. r_K of the deferred shift updates)
  DevBuf<double> rbuf;
  int nslots = 2;
  // shift-update mode: requested (0 auto, 1 per-iteration, 2 deferred basis)
  // and the one the current solve uses (1 or 2)
  int su_req = 0, su_mode = 1;
  // storage of the FSDA solve's vectors (p, y, z, r slots): 64, or 32 = fp32
  // storage with fp64 reductions (BASELINE cfg5); q, mu, b and all scalars
  // stay double.  fp32 storage always runs with the deferred basis.
  int store_bits = 64;
  DevBuf<double> coef_a, coef_c;
  long long coef_ld = 1;
  DevBuf<double> bigp, sols, wT, scores, dense_a;
  // per-shift state
  DevBuf<double> beta, zeta_prev, zeta, zeta_next, gamma_s, alpha_s, resid;
  DevBuf<long long> iters;
  DevBuf<unsigned char> conv;
  DevBuf<int> active, good, pending, flip, err, upd_mode;
  DevBuf<double> upd_gs, upd_zn, upd_as;
  // side stream (low priority) + events for the shift update forked beside
  // the sparse kernels inside the solve graph
  cudaStream_t side = nullptr;
  cudaEvent_t ev_lfork = nullptr, ev_lcopy = nullptr;  // combined upload: L's copies on `side`
  PinnedBuf ldiag_stage;  // combined upload: L's diagonal, split out on the host
  // bounce ring for host -> device copies from pageable memory (h2d)
  PinnedBuf h2d_ring;
  cudaEvent_t h2d_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  unsigned h2d_next = 0;
  int l_host_err = 0;     // the host split's validation result (check_err_flag codes)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  CgScalars* sc = nullptr;

  // graph cache for the solve
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  std::string graph_key;
  bool cond_supported = true;
  // launch the solve's kernels one by one from the host instead of the
  // captured graph (FSDA_B200_EAGER=1 at creation, or fsda_set_eager): ncu
  // cannot profile kernel nodes of graphs that contain conditional nodes
  bool eager = false;

  long long graph_fixed = 0, graph_body = 0;  // launches in the cached graph
  // which operator the solve graph runs: 0 FSDA (sda.py:162-174), 1 the
  // regression operator X^T X (sda.py:177-179) on a caller-supplied rhs
  int solve_kind = 0;
  int solve_abs_tol = 0;

  // resident-solve parameters
  double r_alpha = 0.0, r_tol = 0.0;
  int r_ns = 0;
  long long r_max_iter = 0;
  bool r_prepared = false;
  long long last_launch_count = 0;

  // row-sharded solve (fsda_shard_init, fsda_shard.cuh): this context holds
  // one contiguous row block of X and L of a problem split over `world` ranks
  int world = 1, rank = 0;
  long long maxc = 0;          // rows of the largest shard: the y all-gather slot
  long long shard_n_global = 0;
  void* nccl = nullptr;        // ncclComm_t (one process per GPU), or null (local ranks)
  DevBuf<double> ypad, qpart, qrecv, qown, spart, sall;
  cudaEvent_t ev_x = nullptr, ev_y = nullptr;  // local-rank exchanges

  ShiftState shifts() {
    ShiftState s;
    s.beta = beta.ptr; s.zeta_prev = zeta_prev.ptr; s.zeta = zeta.ptr;
    s.zeta_next = zeta_next.ptr; s.gamma_s = gamma_s.ptr; s.alpha_s = alpha_s.ptr;
    s.resid = resid.ptr; s.iters = iters.ptr; s.conv = conv.ptr; s.active = active.ptr;
    s.good = good.ptr; s.pending = pending.ptr; s.flip = flip.ptr;
    s.upd_mode = upd_mode.ptr; s.upd_gs = upd_gs.ptr; s.upd_zn = upd_zn.ptr; s.upd_as = upd_as.ptr;
    s.coef_a = su_mode == 2 ? coef_a.ptr : nullptr;
    s.coef_c = su_mode == 2 ? coef_c.ptr : nullptr;
    s.coef_ld = coef_ld;
    return s;
  }

  void invalidate_graph() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr;
    graph = nullptr;
    graph_key.clear();
  }
};

namespace {

// ---------------------------------------------------------------- helpers

struct Recorder {
  // Eager profiling: events around each launch.
  std::vector<std::pair<const char*, double>> names;  // name, bytes
  std::vector<cudaEvent_t> ev;
  cudaStream_t stream = nullptr;
  void before(const char* name, double bytes) {
    cudaEvent_t e0;
    CK(cudaEventCreate(&e0));
    CK(cudaEventRecord(e0, stream));
    ev.push_back(e0);
    names.emplace_back(name, bytes);
  }
  void after() {
    cudaEvent_t e1;
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e1, stream));
    ev.push_back(e1);
  }
  ~Recorder() {
    for (auto e : ev) cudaEventDestroy(e);
  }
};

struct Enq {
  fsda_ctx* c;
  Recorder* rec = nullptr;
  long long count = 0;
  template <typename F>
  void go(const char* name, double bytes, F&& f) {
    if (rec) rec->before(name, bytes);
    f();
    CKL();
    if (rec) rec->after();
    ++count;
  }
};

void ensure_vectors(fsda_ctx* c, int ns) {
  const long long n = std::max<long long>(c->n, 1), d = std::max<long long>(c->d, 1);
  c->y.ensure(n); c->z.ensure(n); c->t.ensure(n); c->wv.ensure(n); c->ind.ensure(n);
  c->q.ensure(d); c->p.ensure(d); c->mu_v.ensure(d);
  c->b.ensure(d); c->probe.ensure(d);
  c->part_n.ensure(2 * n_leaves(n) + 2);
  c->part_d.ensure(n_leaves(d) + 1);
  c->part_d2.ensure(n_leaves(d) + 1);
  const int nsx = std::max(ns, 1);
  c->part_o.ensure((size_t)nsx * n_leaves(n) + 1);
  c->sols.ensure((size_t)nsx * d);
  if (c->su_mode == 2) {
    c->bigp.ensure(1);
    c->rbuf.ensure((size_t)c->nslots * d);
    c->coef_a.ensure((size_t)nsx * c->coef_ld);
    c->coef_c.ensure((size_t)nsx * c->coef_ld);
  } else {
    c->bigp.ensure((size_t)nsx * d);
    c->rbuf.ensure((size_t)2 * d);
  }
  c->wT.ensure((size_t)nsx * d); c->scores.ensure((size_t)nsx * n);
  c->beta.ensure(nsx); c->zeta_prev.ensure(nsx); c->zeta.ensure(nsx); c->zeta_next.ensure(nsx);
  c->gamma_s.ensure(nsx); c->alpha_s.ensure(nsx); c->resid.ensure(nsx); c->iters.ensure(nsx);
  c->conv.ensure(nsx); c->active.ensure(nsx); c->good.ensure(nsx); c->pending.ensure(nsx);
  c->flip.ensure(nsx);
  c->upd_mode.ensure(nsx); c->upd_gs.ensure(nsx); c->upd_zn.ensure(nsx); c->upd_as.ensure(nsx);
}

int grid_for(long long n, int block) { return (int)std::max<long long>(1, cdiv(n, block)); }

// ---- segmented sums (K1 / K2 / K3)
// Programmatic dependent launch inside an iteration (bit mask; default all,
// FSDA_B200_PDL=0 turns it off): 1 K2 after K1, 2 X^T after K2, 4 CG step
// after X^T.  Measured at cfg2: 88.6 -> 93.5 solves/s.
int pdl_mode() {
  static const int v = std::getenv("FSDA_B200_PDL") ? std::atoi(std::getenv("FSDA_B200_PDL")) : 7;
  return v;
}

// fp32 storage applies to the FSDA solve's loop vectors
inline bool f32(const fsda_ctx* c) { return c->store_bits == 32 && c->solve_kind == 0; }

template <int KIND, typename A>
void launch_segsum(fsda_ctx* c, const HostPlan& hp, const A& a, int guarded,
                   long long sum_leaves) {
  SegPlan pl = hp.pl;
  pl.warp_base[8] = pl.warp_base[7] + sum_leaves;
  const long long warps = pl.warp_base[8];
  if (warps == 0) return;
  const int blocks = (int)std::max<long long>(
      1, std::min<long long>(cdiv(warps, 8), (long long)c->num_sms * 16));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  // K2 (L rows) follows K1 directly on the stream: let it launch early
  cfg.numAttrs = (pdl_mode() & 1) && KIND == SEG_LROWS ? 1 : 0;
  cfg.attrs = at;
  const CgScalars* sc = c->sc;
  CK(cudaLaunchKernelEx(&cfg, k_segsum<KIND, A>, pl, a, sc, guarded));
}

template <typename A = SegArgs>
A seg_args(const void* src, void* out) {
  A a;
  memset(&a, 0, sizeof(a));
  a.src = static_cast<const typename A::value_type*>(src);
  a.out = static_cast<decltype(a.out)>(out);
  return a;
}

// X^T z: mode 0 raw (+ optional sum(z) leaves), 1 centred with *sum_ptr, 2 / ell.
// zf32: z is stored as float (the fp32-storage loop); out (q) is double.
template <typename A>
void enq_xt_t(Enq& e, const void* zsrc, double* out, int mode, const double* sum_ptr, int guarded,
              double* sum_part, double* sum_out) {
  fsda_ctx* c = e.c;
  const double vb = sizeof(typename A::value_type);
  const double bytes = 4.0 * (c->d + 1) + 4.0 * c->nnz + vb * c->n + 8.0 * c->d +
                       (mode == 1 ? 8.0 * c->d : 0.0);
  A a = seg_args<A>(zsrc, out);
  a.mode = mode;
  a.mu = c->mu_v.ptr;
  a.sum_ptr = sum_ptr;
  a.ell = (double)c->ell;
  a.sum_part = sum_part;
  a.sum_n = sum_part ? c->n : 0;
  e.go("xt", bytes, [&] {
    SegPlan pl = c->plan_xc.pl;
    pl.warp_base[8] = pl.warp_base[7] + (sum_part ? n_leaves(c->n) : 0);
    XtDense xh = c->xh;
    const CgScalars* sc = c->sc;
    int n_rows = (int)c->n;
    unsigned long long* ticket = c->xt_ticket.ptr;

    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c->xt_blocks);
    cfg.blockDim = dim3(XT_THREADS);
    cfg.dynamicSmemBytes = sizeof(typename A::value_type) * xh.rb;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = (pdl_mode() & 2) ? 2 : 1;
    cfg.attrs = at;
    CK(cudaLaunchKernelEx(&cfg, k_xt_coop<A>, pl, xh, a, sc, guarded, n_rows, ticket, sum_out));
  });
}

void enq_xt(Enq& e, const double* zsrc, double* out, int mode, const double* sum_ptr, int guarded,
            double* sum_part, double* sum_out = nullptr, bool zf32 = false) {
  if (zf32) enq_xt_t<SegArgs32D>(e, zsrc, out, mode, sum_ptr, guarded, sum_part, sum_out);
  else enq_xt_t<SegArgs>(e, zsrc, out, mode, sum_ptr, guarded, sum_part, sum_out);
}

// y = X v in the canonical row order (vf32: v and y stored as float).
void enq_xrows(Enq& e, const void* v, void* out, int guarded, bool vf32 = false) {
  fsda_ctx* c = e.c;
  const double vb = vf32 ? 4.0 : 8.0;
  const double bytes = 4.0 * (c->n + 1) + 4.0 * c->nnz + vb * c->d + vb * c->n;
  if (vf32) {
    SegArgs32 a = seg_args<SegArgs32>(v, out);
    e.go("spmv_rows", bytes, [&] { launch_segsum<SEG_XROWS>(c, c->plan_xr, a, guarded, 0); });
  } else {
    SegArgs a = seg_args<SegArgs>(v, out);
    e.go("spmv_rows", bytes, [&] { launch_segsum<SEG_XROWS>(c, c->plan_xr, a, guarded, 0); });
  }
}

int alpha_mode_of(double alpha) { return alpha == 0.0 ? 0 : (alpha == 1.0 ? 1 : 2); }

// z = M y (apply_smoother, sda.py:131-140); vf32: y and z stored as float.
template <typename A>
void enq_smoother_t(Enq& e, double alpha, const void* y, void* z, int guarded) {
  fsda_ctx* c = e.c;
  using V = typename A::value_type;
  const double vb = sizeof(V);
  const int amode = alpha_mode_of(alpha);
  if (amode == 0) {
    e.go("smoother", (2.0 * vb + 1.0) * c->n, [&] {
      k_mask_labeled<V><<<grid_for(c->n, 256), 256, 0, c->stream>>>(
          static_cast<const V*>(y), c->labels.ptr, static_cast<V*>(z), (int)c->n, c->sc, guarded,
          (int)c->row_base);
    });
    return;
  }
  A a = seg_args<A>(y, z);
  a.ldiag = c->l_diag.ptr;
  a.labels = c->labels.ptr;
  a.alpha = alpha;
  a.alpha_mode = amode;
  a.row_base = (int)c->row_base;
  const double bytes = 4.0 * (c->n + 1) + 4.0 * c->l_nnz + vb * c->n + 1.0 * c->n + 8.0 * c->n + vb * c->n;
  e.go("smoother", bytes, [&] { launch_segsum<SEG_LROWS>(c, c->plan_lr, a, guarded, 0); });
}

void enq_smoother(Enq& e, double alpha, const void* y, void* z, int guarded, bool vf32 = false) {
  if (vf32) enq_smoother_t<SegArgs32>(e, alpha, y, z, guarded);
  else enq_smoother_t<SegArgs>(e, alpha, y, z, guarded);
}

size_t step_smem(int ns) { return sizeof(double) * 3 * (size_t)std::max(ns, 1); }

// Cooperative launch of k_cg_step (capturable into graphs).
// center: 0 none, 1 FSDA (q - mu sum z), 2 SA-SDA (q - 1_l sum z / l)
void launch_cg_step(fsda_ctx* c, int ns, long long d, unsigned long long cond, int use_cond,
                    int center, const double* sum_ready = nullptr) {
  ShiftState ss = c->shifts();
  const long long nlD = n_leaves(d);
  double* q = c->q.ptr;
  double* p = c->p.ptr;
  void* rb = c->rbuf.ptr;
  int nsl = c->nslots;
  double* bigp = c->bigp.ptr;
  double* sols = c->sols.ptr;
  double* pp = c->part_d.ptr;
  double* pr = c->part_d2.ptr;
  CgScalars* sc = c->sc;
  const double* mu = center == 1 ? c->mu_v.ptr : nullptr;
  const double* pz = center ? c->part_n.ptr : nullptr;
  const long long nlz = center ? n_leaves(c->n) : 0;
  const signed char* lab = c->labels.ptr;
  double ell = (double)c->ell;

  const size_t smem = step_smem(ns);
  // One warp per 256-element leaf (the leaf's p, q, r stay in registers across
  // the two grid barriers); warps loop over further leaves only when d exceeds
  // what a co-resident grid covers.
  if (c->step_blocks == 0) {
    int nb = 0, nb32 = 0;
    CK(cudaFuncSetAttribute(k_cg_step<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_cg_step<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_cg_step<double>, STEP_THREADS,
                                                     step_smem(4096)));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb32, k_cg_step<float>, STEP_THREADS,
                                                     step_smem(4096)));
    c->step_blocks = std::max(1, std::min(nb, nb32)) * c->num_sms;
  }
  const long long want = (nlD + STEP_THREADS / 32 - 1) / (STEP_THREADS / 32);
  const int blocks = (int)std::max(1LL, std::min<long long>(want, c->step_blocks));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(STEP_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.numAttrs = (pdl_mode() & 4) ? 2 : 1;
  cfg.attrs = at;
  if (f32(c))
    CK(cudaLaunchKernelEx(&cfg, k_cg_step<float>, q, (float*)p, (float*)rb, nsl, bigp, sols, d, pp, pr,
                          nlD, sc, ss, ns, cond, use_cond, mu, pz, nlz, lab, ell, sum_ready));
  else
    CK(cudaLaunchKernelEx(&cfg, k_cg_step<double>, q, p, (double*)rb, nsl, bigp, sols, d, pp, pr, nlD,
                          sc, ss, ns, cond, use_cond, mu, pz, nlz, lab, ell, sum_ready));
}

// The shift-state update of the last base step on `stream`: sols / P
// streamed (k_shift_update), or, in the deferred mode, the coefficient rows
// (k_coef_update).
void launch_shift_update(fsda_ctx* c, int ns, long long d, cudaStream_t stream, int guarded) {
  ShiftState ss = c->shifts();
  if (c->su_mode == 2) {
    dim3 g((unsigned)grid_for(c->coef_ld, 256), (unsigned)ns);
    k_coef_update<<<g, 256, 0, stream>>>(ss, c->sc, ns, guarded);
    CKL();
    return;
  }
  dim3 g((unsigned)((d + 256 * SU_ELEMS - 1) / (256 * SU_ELEMS)),
         (unsigned)((ns + SU_SHIFTS - 1) / SU_SHIFTS));
  k_shift_update<<<g, 256, 0, stream>>>(c->rbuf.ptr, c->nslots, c->bigp.ptr, c->sols.ptr, d, ss,
                                        c->sc, ns, guarded);
  CKL();
}

// Shift-update mode of a solve with these sizes: the deferred basis needs
// (max_iter + 1) residuals of d doubles plus two n_s x (max_iter + 1)
// coefficient tables; it is used when they fit a quarter of the free device
// memory (FSDA_B200_SHIFT_MODE=1/2 or fsda_set_shift_update_mode force one).
void resolve_shift_mode(fsda_ctx* c, int ns, long long max_iter, long long d) {
  int req = c->su_req;
  if (req == 0 && std::getenv("FSDA_B200_SHIFT_MODE")) req = std::atoi(std::getenv("FSDA_B200_SHIFT_MODE"));
  int mode = 1;
  const long long slots = std::max<long long>(max_iter, 0) + 1;
  const double need = 8.0 * (double)slots * (double)std::max<long long>(d, 1) +
                      16.0 * (double)std::max(ns, 1) * (double)slots;
  if (req == 2) {
    mode = 2;
  } else if (req == 0) {
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    const double have = 8.0 * (double)c->rbuf.cap + 8.0 * (double)(c->coef_a.cap + c->coef_c.cap);
    mode = need <= 0.25 * (double)free_b + have ? 2 : 1;
  }
  if (c->store_bits == 32 && c->solve_kind == 0) mode = 2;
  c->su_mode = mode;
  c->nslots = mode == 2 ? (int)std::min<long long>(slots, INT32_MAX) : 2;
  c->coef_ld = mode == 2 ? slots : 1;
}

// r_0 = p = b, P_s = b / coefficient rows, sols = 0, b.b (krylov.py:185-208)
void launch_cg_init(fsda_ctx* c, const double* bsrc, long long d, int ns) {
  ShiftState ss = c->shifts();
  const long long nlD = n_leaves(d);
  dim3 g(grid_for(nlD, WARPS_PER_BLOCK), 1 + ns);
  if (f32(c))
    k_cg_init<float><<<g, LEAF_THREADS, 0, c->stream>>>(bsrc, (float*)c->rbuf.ptr, (float*)c->p.ptr,
                                                        c->bigp.ptr, c->sols.ptr, d, c->part_d.ptr, nlD,
                                                        c->sc, ss, ns, 1);
  else
    k_cg_init<double><<<g, LEAF_THREADS, 0, c->stream>>>(bsrc, c->rbuf.ptr, c->p.ptr, c->bigp.ptr,
                                                         c->sols.ptr, d, c->part_d.ptr, nlD, c->sc, ss,
                                                         ns, c->su_mode == 2 ? 1 : 0);
  CKL();
}

// The last iteration's shift update, and in the deferred mode the
// directions formed from the stored residuals.
void launch_final_shift(fsda_ctx* c, int ns, long long d) {
  launch_shift_update(c, ns, d, c->stream, 0);
  if (c->su_mode == 2 && d > 0) {
    ShiftState ss = c->shifts();
    dim3 g((unsigned)grid_for(d, 256), (unsigned)((ns + CB_SH - 1) / CB_SH));
    if (f32(c))
      k_combine_basis<float><<<g, 256, 0, c->stream>>>((const float*)c->rbuf.ptr, d, ss, c->sc, ns,
                                                       c->sols.ptr);
    else
      k_combine_basis<double><<<g, 256, 0, c->stream>>>(c->rbuf.ptr, d, ss, c->sc, ns, c->sols.ptr);
    CKL();
  }
}

// One iteration = sparse products `sparse` (K1..K3 or the operator's
// equivalent) + the cooperative base step.  In the graph body the previous
// iteration's shift update is forked onto the side stream, beside the sparse
// kernels (it reads r_i and writes sols / P, which they never touch); eagerly
// it follows the base step on the same stream.
template <typename Sparse>
void enq_iteration_body(Enq& e, int ns, long long d, int center, unsigned long long cond,
                        int use_cond, double step_bytes, Sparse&& sparse,
                        const double* sum_ready = nullptr) {
  fsda_ctx* c = e.c;
  const double su_bytes = c->su_mode == 2 ? 32.0 * ns * (double)c->coef_ld : 32.0 * d * ns + 8.0 * d;
  static const bool inline_su = std::getenv("FSDA_B200_SU_INLINE") != nullptr;
  // timing experiment only (results wrong): no per-iteration shift update
  const bool skip_su = std::getenv("FSDA_B200_EXP_SKIP_SU") != nullptr;
  if (skip_su) {
    sparse();
    e.go("cg_step", step_bytes, [&] { launch_cg_step(c, ns, d, cond, use_cond, center, sum_ready); });
    return;
  }
  if (use_cond && !inline_su) {
    CK(cudaEventRecord(c->ev_fork, c->stream));
    CK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    e.go("shift_update", su_bytes, [&] { launch_shift_update(c, ns, d, c->side, 1); });
    CK(cudaEventRecord(c->ev_join, c->side));
    sparse();
    CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    e.go("cg_step", step_bytes, [&] { launch_cg_step(c, ns, d, cond, use_cond, center, sum_ready); });
  } else {
    sparse();
    e.go("cg_step", step_bytes, [&] { launch_cg_step(c, ns, d, cond, use_cond, center, sum_ready); });
    e.go("shift_update", su_bytes, [&] { launch_shift_update(c, ns, d, c->stream, 1); });
  }
}

// One shifted-CG iteration for the FSDA operator (graph body).
void enq_fsda_iteration(Enq& e, double alpha, int ns, unsigned long long cond, int use_cond) {
  fsda_ctx* c = e.c;
  const long long d = c->d;
  // k_xt_coop's last CTA reduces sum(z) for the CG step's centring
  // (FSDA_B200_K3_SUM=0: the CG step reduces it)
  static const bool k3_sum = !std::getenv("FSDA_B200_K3_SUM") || std::atoi(std::getenv("FSDA_B200_K3_SUM"));
  double* sum_out = k3_sum ? &c->sc->sum_z_iter : nullptr;
  const bool v32 = f32(c);
  enq_iteration_body(e, ns, d, 1, cond, use_cond, 8.0 * c->n + 24.0 * d + 24.0 * d + 24.0 * d, [&] {
    enq_xrows(e, c->p.ptr, c->y.ptr, 1, v32);
    enq_smoother(e, alpha, c->y.ptr, c->z.ptr, 1, v32);
    enq_xt(e, c->z.ptr, c->q.ptr, 0, nullptr, 1, c->part_n.ptr, sum_out, v32);
  }, sum_out);
}

// Setup (labeled mean, rhs, CG init) — sda.py:297-301, krylov.py:185-208.
void enq_fsda_setup(Enq& e, int ns, long long max_iter, double tol) {
  fsda_ctx* c = e.c;
  const long long n = c->n, d = c->d, nlN = n_leaves(n), nlD = n_leaves(d);
  ShiftState ss = c->shifts();
  e.go("solve_reset", 0.0, [&] {
    k_solve_reset<<<1, 256, 0, c->stream>>>(c->sc, ss, ns, max_iter, tol, 0);
  });
  e.go("indicator", 9.0 * n, [&] {
    k_indicator<<<grid_for(n, 256), 256, 0, c->stream>>>(c->labels.ptr, c->ind.ptr, (int)n);
  });
  enq_xt(e, c->ind.ptr, c->mu_v.ptr, 2, nullptr, 0, nullptr);
  enq_xrows(e, c->probe.ptr, c->t.ptr, 0);
  e.go("class_sums", 9.0 * n, [&] {
    k_class_sums<<<grid_for(nlN, WARPS_PER_BLOCK), LEAF_THREADS, 0, c->stream>>>(
        c->t.ptr, c->labels.ptr, n, c->part_n.ptr, nlN, c->sc, (double)c->n1, (double)c->n2);
  });
  e.go("apply_w", 9.0 * n, [&] {
    k_apply_w<<<grid_for(nlN, WARPS_PER_BLOCK), LEAF_THREADS, 0, c->stream>>>(
        c->labels.ptr, c->wv.ptr, n, c->part_n.ptr, nlN, c->sc);
  });
  enq_xt(e, c->wv.ptr, c->b.ptr, 1, &c->sc->sum_z, 0, nullptr);
  e.go("cg_init", 8.0 * d * 3 + 16.0 * d * ns, [&] { launch_cg_init(c, c->b.ptr, d, ns); });
}

// Projection (sda.py:265-284) and the still-active residuals.
void enq_fsda_tail(Enq& e, int ns) {
  fsda_ctx* c = e.c;
  const long long n = c->n, d = c->d, nlN = n_leaves(n);
  ShiftState ss = c->shifts();
  e.go(c->su_mode == 2 ? "combine_basis" : "shift_update", c->su_mode == 2 ? 8.0 * d * (double)c->coef_ld + 8.0 * d * ns : 32.0 * d * ns,
       [&] { launch_final_shift(c, ns, d); });
  e.go("cg_finish", 0.0, [&] { k_cg_finish<<<1, 32, 0, c->stream>>>(c->sc, ss, ns); });
  e.go("transpose_sols", 16.0 * d * ns, [&] {
    k_transpose_sols<<<grid_for(d * ns, 256), 256, 0, c->stream>>>(c->sols.ptr, c->wT.ptr, d, ns);
  });
  e.go("spmm_scores", 4.0 * (n + 1) + 4.0 * c->nnz + 8.0 * d * ns + 8.0 * n * ns, [&] {
    k_spmm_scores<<<grid_for(n, 8), 256, 0, c->stream>>>(c->x_rowptr.ptr, c->x_cols.ptr, c->wT.ptr,
                                                         c->scores.ptr, (int)n, ns);
  });
  e.go("orient", 8.0 * n * ns + 1.0 * n, [&] {
    dim3 g(grid_for(nlN, WARPS_PER_BLOCK), ns);
    k_orient<<<g, LEAF_THREADS, 0, c->stream>>>(c->labels.ptr, c->scores.ptr, n, c->part_o.ptr, nlN);
    k_orient_final<<<ns, 256, 0, c->stream>>>(c->part_o.ptr, nlN, ss, nullptr);
  });
  e.go("flip", 0.0, [&] {
    dim3 g((unsigned)std::min<long long>(grid_for(std::max(n, d), 256), 1024), ns);
    k_flip<<<g, 256, 0, c->stream>>>(c->scores.ptr, c->sols.ptr, n, d, ss);
  });
}

// Regression-phase shifted solve (shifted_cg(regression_operator(p), b),
// sda.py:177-179, 339, 439-442; evaluation.py:288-291): w -> X^T (X w).
void enq_reg_setup(Enq& e, int ns, long long max_iter, double tol, int abs_tol) {
  fsda_ctx* c = e.c;
  const long long d = c->d, nlD = n_leaves(d);
  ShiftState ss = c->shifts();
  e.go("solve_reset", 0.0, [&] {
    k_solve_reset<<<1, 256, 0, c->stream>>>(c->sc, ss, ns, max_iter, tol, abs_tol);
  });
  e.go("cg_init", 8.0 * d * 3 + 16.0 * d * ns, [&] { launch_cg_init(c, c->b.ptr, d, ns); });
}

void enq_reg_iteration(Enq& e, int ns, unsigned long long cond, int use_cond) {
  fsda_ctx* c = e.c;
  const long long d = c->d;
  enq_iteration_body(e, ns, d, 0, cond, use_cond, 24.0 * d + 24.0 * d + 24.0 * d, [&] {
    enq_xrows(e, c->p.ptr, c->y.ptr, 1);
    enq_xt(e, c->y.ptr, c->q.ptr, 0, nullptr, 1, nullptr);
  });
}

void enq_reg_tail(Enq& e, int ns) {
  fsda_ctx* c = e.c;
  ShiftState ss = c->shifts();
  e.go(c->su_mode == 2 ? "combine_basis" : "shift_update", 32.0 * c->d * ns, [&] { launch_final_shift(c, ns, c->d); });
  e.go("cg_finish", 0.0, [&] { k_cg_finish<<<1, 32, 0, c->stream>>>(c->sc, ss, ns); });
}

// SA-SDA (sda.py:360-396): shifted CG in sample space on the centred spectral
// operator z -> M z - 1_l (sum(M z) / l) (sda.py:148-159); the vectors of the
// recurrence have N entries (the context's d is N while it runs).  The rhs is
// apply_w of the orthogonalized probe (uploaded into t), sda.py:287-290, 373.
void enq_sa_setup(Enq& e, int ns, long long max_iter, double tol) {
  fsda_ctx* c = e.c;
  const long long n = c->n, nlN = n_leaves(n);
  ShiftState ss = c->shifts();
  e.go("solve_reset", 0.0, [&] {
    k_solve_reset<<<1, 256, 0, c->stream>>>(c->sc, ss, ns, max_iter, tol, 0);
  });
  e.go("class_sums", 9.0 * n, [&] {
    k_class_sums<<<grid_for(nlN, WARPS_PER_BLOCK), LEAF_THREADS, 0, c->stream>>>(
        c->t.ptr, c->labels.ptr, n, c->part_n.ptr, nlN, c->sc, (double)c->n1, (double)c->n2);
  });
  e.go("apply_w", 9.0 * n, [&] {
    k_apply_w<<<grid_for(nlN, WARPS_PER_BLOCK), LEAF_THREADS, 0, c->stream>>>(
        c->labels.ptr, c->wv.ptr, n, c->part_n.ptr, nlN, c->sc);
  });
  e.go("cg_init", 8.0 * n * 3 + 16.0 * n * ns, [&] { launch_cg_init(c, c->wv.ptr, n, ns); });
}

void enq_sa_iteration(Enq& e, double alpha, int ns, unsigned long long cond, int use_cond) {
  fsda_ctx* c = e.c;
  const long long n = c->n, nlN = n_leaves(n);
  enq_iteration_body(e, ns, n, 2, cond, use_cond, 8.0 * n + 48.0 * n + 24.0 * n, [&] {
    enq_smoother(e, alpha, c->p.ptr, c->q.ptr, 1);
    e.go("vector_sum", 8.0 * n, [&] {
      k_vector_sum<<<grid_for(nlN, WARPS_PER_BLOCK), LEAF_THREADS, 0, c->stream>>>(
          c->q.ptr, n, c->part_n.ptr, nlN, c->sc, nullptr);
    });
  });
}

void enq_sa_tail(Enq& e, int ns) {
  fsda_ctx* c = e.c;
  const long long n = c->n, nlN = n_leaves(n);
  ShiftState ss = c->shifts();
  e.go(c->su_mode == 2 ? "combine_basis" : "shift_update", 32.0 * n * ns, [&] { launch_final_shift(c, ns, n); });
  e.go("cg_finish", 0.0, [&] { k_cg_finish<<<1, 32, 0, c->stream>>>(c->sc, ss, ns); });
  e.go("orient", 8.0 * n * ns + 1.0 * n, [&] {  // _oriented, sda.py:256-262
    dim3 g(grid_for(nlN, WARPS_PER_BLOCK), ns);
    k_orient<<<g, LEAF_THREADS, 0, c->stream>>>(c->labels.ptr, c->sols.ptr, n, c->part_o.ptr, nlN);
    k_orient_final<<<ns, 256, 0, c->stream>>>(c->part_o.ptr, nlN, ss, nullptr);
  });
  e.go("flip", 0.0, [&] {
    dim3 g((unsigned)std::min<long long>(grid_for(n, 256), 1024), ns);
    k_flip<<<g, 256, 0, c->stream>>>(nullptr, c->sols.ptr, 0, n, ss);
  });
}

void enq_setup_k(Enq& e, int ns, long long max_iter, double tol) {
  if (e.c->solve_kind == 1) enq_reg_setup(e, ns, max_iter, tol, e.c->solve_abs_tol);
  else if (e.c->solve_kind == 2) enq_sa_setup(e, ns, max_iter, tol);
  else enq_fsda_setup(e, ns, max_iter, tol);
}

void enq_iteration_k(Enq& e, double alpha, int ns, unsigned long long cond, int use_cond) {
  if (e.c->solve_kind == 1) enq_reg_iteration(e, ns, cond, use_cond);
  else if (e.c->solve_kind == 2) enq_sa_iteration(e, alpha, ns, cond, use_cond);
  else enq_fsda_iteration(e, alpha, ns, cond, use_cond);
}

void enq_tail_k(Enq& e, int ns) {
  if (e.c->solve_kind == 1) enq_reg_tail(e, ns);
  else if (e.c->solve_kind == 2) enq_sa_tail(e, ns);
  else enq_fsda_tail(e, ns);
}

// Build (or reuse) the whole-solve graph with a conditional WHILE node.
bool build_solve_graph(fsda_ctx* c, double alpha, int ns, long long max_iter, double tol,
                       long long* launches_fixed, long long* launches_body) {
  // The key covers everything baked into the graph's kernel arguments:
  // scalars, buffer generation (pointers), and the plan structs by value.
  unsigned long long h = 1469598103934665603ULL;
  auto mix = [&](const void* p, size_t n) {
    const unsigned char* b = (const unsigned char*)p;
    for (size_t k = 0; k < n; ++k) h = (h ^ b[k]) * 1099511628211ULL;
  };
  mix(&c->plan_xr.pl, sizeof(SegPlan));
  mix(&c->plan_lr.pl, sizeof(SegPlan));
  mix(&c->plan_xc.pl, sizeof(SegPlan));
  mix(&c->xh, sizeof(XtDense));
  mix(&c->ell, sizeof(c->ell));
  mix(&c->n1, sizeof(c->n1));
  mix(&c->n2, sizeof(c->n2));
  char key[320];
  snprintf(key, sizeof(key), "%d|%d|%a|%d|%lld|%a|%lld|%lld|%lld|%llu|%llx|%d|%d", c->solve_kind,
           c->solve_abs_tol, alpha, ns, max_iter, tol, c->n, c->d, c->nnz, g_alloc_gen.load(), h,
           c->su_mode, c->nslots * (c->store_bits == 32 ? -1 : 1));
  if (c->exec && c->graph_key == key) {
    *launches_fixed = c->graph_fixed;
    *launches_body = c->graph_body;
    return true;
  }
  c->invalidate_graph();
  cudaStream_t s = c->stream;
  cudaGraph_t graph;
  CK(cudaGraphCreate(&graph, 0));
  CK(cudaStreamBeginCaptureToGraph(s, graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  Enq e{c};
  try {
    enq_setup_k(e, ns, max_iter, tol);
  } catch (...) {
    cudaGraph_t g2;
    cudaStreamEndCapture(s, &g2);
    cudaGraphDestroy(graph);
    throw;
  }
  long long fixed = e.count;
  cudaStreamCaptureStatus st;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  cudaGraph_t cap_graph;
  CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &cap_graph, &deps, &ndeps));
  cudaGraphConditionalHandle handle;
  CK(cudaGraphConditionalHandleCreate(&handle, cap_graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cond_node;
  CK(cudaGraphAddNode(&cond_node, cap_graph, deps, ndeps, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CK(cudaStreamUpdateCaptureDependencies(s, &cond_node, 1, cudaStreamSetCaptureDependencies));
  // capture the body on a side stream
  cudaStream_t s2;
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  CK(cudaStreamBeginCaptureToGraph(s2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  Enq eb{c};
  cudaStream_t saved = c->stream;
  c->stream = s2;
  enq_iteration_k(eb, alpha, ns, (unsigned long long)handle, 1);
  c->stream = saved;
  cudaGraph_t body_out;
  CK(cudaStreamEndCapture(s2, &body_out));
  CK(cudaStreamDestroy(s2));
  enq_tail_k(e, ns);
  cudaGraph_t out;
  CK(cudaStreamEndCapture(s, &out));
  c->graph = out;
  CK(cudaGraphInstantiate(&c->exec, out, 0));
  c->graph_key = key;
  *launches_fixed = c->graph_fixed = e.count;  // setup + tail
  *launches_body = c->graph_body = eb.count;  // per iteration
  (void)fixed;
  return true;
}

struct SolveOut {
  double* directions;
  double* scores;
  double* residuals;
  int64_t* iterations;
  uint8_t* converged;
  int64_t* n_applies;
  int64_t* fail_iter;
};

int check_solve_args(fsda_ctx* c, double alpha, const double* betas, int ns, double tol) {
  if (!c->has_x) return fail(FSDA_EINVAL, "fsda_solve: X has not been uploaded");
  if (!c->has_l) return fail(FSDA_EINVAL, "fsda_solve: Laplacian has not been uploaded");
  if (!c->has_labels) return fail(FSDA_EINVAL, "fsda_solve: labels have not been set");
  if (c->ell == 0) return fail(FSDA_ELABEL, "centering requires at least one labeled sample");
  if (c->n1 == 0 || c->n2 == 0)
    return fail(FSDA_EINVAL, "both classes need at least one labeled sample");
  if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(FSDA_EINVAL, "alpha must lie in [0, 1], got %g", alpha);
  if (ns <= 0) return fail(FSDA_EINVAL, "shift grid must be a non-empty 1-d array");
  if (ns > FSDA_MAX_SHIFTS) return fail(FSDA_EINVAL, "at most 4096 shifts per solve");
  for (int s = 0; s < ns; ++s) {
    if (!std::isfinite(betas[s])) return fail(FSDA_EINVAL, "shifts must be finite");
    if (s == 0 && betas[s] < 0) return fail(FSDA_EINVAL, "shifts must be non-negative");
    if (s > 0 && !(betas[s] > betas[s - 1])) return fail(FSDA_EINVAL, "shifts must be strictly ascending");
  }
  if (!(tol > 0)) return fail(FSDA_EINVAL, "tol must be positive");
  if (c->d <= 0) return fail(FSDA_EINVAL, "operator dimension must be positive");
  return FSDA_OK;
}

void upload_solve_params(fsda_ctx* c, const double* betas, int ns, const double* probe,
                         long long max_iter) {
  resolve_shift_mode(c, ns, max_iter, c->d);
  ensure_vectors(c, ns);
  CK(cudaMemcpyAsync(c->beta.ptr, betas, sizeof(double) * ns, cudaMemcpyHostToDevice, c->stream));
  if (probe)
    CK(cudaMemcpyAsync(c->probe.ptr, probe, sizeof(double) * c->d, cudaMemcpyHostToDevice, c->stream));
}

// Launch one complete solve (graph, or eager when rec != null or no graph).
long long launch_solve(fsda_ctx* c, double alpha, int ns, long long max_iter, double tol,
                       Recorder* rec) {
  if (!rec && c->cond_supported && !c->eager) {
    long long fixed = 0, body = 0;
    try {
      build_solve_graph(c, alpha, ns, max_iter, tol, &fixed, &body);
      CK(cudaGraphLaunch(c->exec, c->stream));
      // launches = fixed + body * iterations; iterations known after sync
      c->last_launch_count = -(fixed * 1000000LL + body);  // decoded by fetch
      return 0;
    } catch (CudaError& ce) {
      c->invalidate_graph();
      // only "conditional nodes unsupported" switches to the eager loop; any
      // other error (OOM, a fault from an earlier launch) is reported
      if (ce.err != cudaErrorNotSupported && ce.err != cudaErrorCallRequiresNewerDriver) throw;
      cudaGetLastError();
      c->cond_supported = false;  // fall through to eager
    }
  }
  Enq e{c, rec};
  enq_setup_k(e, ns, max_iter, tol);
  for (long long it = 0; it < max_iter; ++it) enq_iteration_k(e, alpha, ns, 0, 0);
  enq_tail_k(e, ns);
  c->last_launch_count = e.count;
  return e.count;
}

int read_results(fsda_ctx* c, int ns, const SolveOut& o, int64_t* launches) {
  CgScalars h;
  CK(cudaMemcpyAsync(&h, c->sc, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  std::vector<long long> it(ns);
  std::vector<unsigned char> cv(ns);
  if (o.directions)
    CK(cudaMemcpyAsync(o.directions, c->sols.ptr, sizeof(double) * ns * c->d, cudaMemcpyDeviceToHost, c->stream));
  if (o.scores)
    CK(cudaMemcpyAsync(o.scores, c->scores.ptr, sizeof(double) * ns * c->n, cudaMemcpyDeviceToHost, c->stream));
  if (o.residuals)
    CK(cudaMemcpyAsync(o.residuals, c->resid.ptr, sizeof(double) * ns, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(it.data(), c->iters.ptr, sizeof(long long) * ns, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(cv.data(), c->conv.ptr, ns, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (o.iterations)
    for (int s = 0; s < ns; ++s) o.iterations[s] = it[s];
  if (o.converged)
    for (int s = 0; s < ns; ++s) o.converged[s] = cv[s];
  if (o.n_applies) *o.n_applies = h.iter;
  if (o.fail_iter) *o.fail_iter = h.fail_iter;
  if (launches) {
    long long lc = c->last_launch_count;
    if (lc < 0) {
      long long enc = -lc, fixed = enc / 1000000LL, body = enc % 1000000LL;
      // every captured iteration launches its kernels (guarded ones exit at
      // once after the loop finished): body_runs counts the CG-step launches
      lc = fixed + body * std::max<long long>(h.body_runs, 1);
    }
    *launches = lc;
  }
  if (h.status == ST_BREAKDOWN)
    return fail(FSDA_EBREAKDOWN, "singular direction: <p, Bp> = 0 at iteration %lld", h.fail_iter);
  if (h.status == ST_NONFINITE)
    return fail(FSDA_ENONFINITE, "non-finite <p, Bp> or residual at iteration %lld", h.fail_iter);
  return FSDA_OK;
}

// Build a segmented-sum plan from host segment offsets (S+1 entries) over the
// device index stream `ind`.  Classes: W = 1 << k for segments with n <= 8W,
// heavy tasks of <= 4 leaves for n > 256.
inline int seg_class(long long n) {
  int k = 0;
  while (8LL * (1 << k) < n) ++k;
  return k;
}

// Two passes over the host offsets (count, then fill a pinned staging buffer),
// each split into chunks of segments run by OpenMP threads (the chunk prefix
// sums keep the plan identical to a sequential build), and asynchronous copies
// on `stream`; the caller synchronises before the plan is used or the staging
// buffer is reused.
template <typename OffT>
void build_seg_plan(HostPlan& hp, cudaStream_t stream, const OffT* offs, long long S,
                    const int* ind, std::vector<int>* dense_out = nullptr,
                    long long dense_min = 0) {
  struct Count {
    long long cls[6] = {0, 0, 0, 0, 0, 0};
    long long heavy = 0, htask = 0, leaves = 0;
    std::vector<int> dense;
  };
  const int nch = (int)std::max<long long>(1, std::min<long long>(64, S / 8192));
  std::vector<Count> cc(nch);
#pragma omp parallel for schedule(dynamic, 1) num_threads(host_threads())
  for (int ch = 0; ch < nch; ++ch) {
    Count& q = cc[ch];
    for (long long sgi = S * ch / nch; sgi < S * (ch + 1) / nch; ++sgi) {
      const long long n = (long long)(offs[sgi + 1] - offs[sgi]);
      if (n <= LEAF) {
        ++q.cls[seg_class(n)];
      } else if (dense_out && n >= dense_min) {
        q.dense.push_back((int)sgi);
      } else {
        ++q.heavy;
        q.htask += cdiv(n, 4 * LEAF);
        q.leaves += cdiv(n, LEAF);
      }
    }
  }
  long long cnt[6] = {0, 0, 0, 0, 0, 0}, n_heavy = 0, n_htask = 0, leaves = 0;
  for (const Count& q : cc) {
    for (int k = 0; k < 6; ++k) cnt[k] += q.cls[k];
    n_heavy += q.heavy;
    n_htask += q.htask;
    leaves += q.leaves;
    if (dense_out) dense_out->insert(dense_out->end(), q.dense.begin(), q.dense.end());
  }
  SegPlan& pl = hp.pl;
  memset(&pl, 0, sizeof(pl));
  long long wb = 0, t = 0;
  for (int k = 0; k < 6; ++k) {
    pl.cls_off[k] = t;
    t += cnt[k];
    pl.warp_base[k] = wb;
    wb += cdiv(cnt[k], 32 >> k);
  }
  pl.cls_off[6] = t;
  pl.warp_base[6] = wb;
  wb += n_htask;
  pl.warp_base[7] = wb;
  pl.warp_base[8] = wb;
  const long long n_tasks = t + n_htask;
  char* st = (char*)hp.stage.ensure(sizeof(int4) * n_tasks + 5 * sizeof(int) * n_heavy + 16);
  int4* tasks = (int4*)st;
  int* h0 = (int*)(tasks + n_tasks);
  int* hn = h0 + n_heavy;
  int* hs = hn + n_heavy;
  int* ht = hs + n_heavy;
  int* hg = ht + n_heavy;
  // per-chunk start positions: class tasks, heavy tasks, heavy ids, leaves
  std::vector<std::array<long long, 9>> start(nch);
  {
    std::array<long long, 9> run{};
    for (int k = 0; k < 6; ++k) run[k] = pl.cls_off[k];
    run[6] = pl.cls_off[6];
    for (int ch = 0; ch < nch; ++ch) {
      start[ch] = run;
      for (int k = 0; k < 6; ++k) run[k] += cc[ch].cls[k];
      run[6] += cc[ch].htask;
      run[7] += cc[ch].heavy;
      run[8] += cc[ch].leaves;
    }
  }
#pragma omp parallel for schedule(dynamic, 1) num_threads(host_threads())
  for (int ch = 0; ch < nch; ++ch) {
    std::array<long long, 9> pos = start[ch];
    for (long long sgi = S * ch / nch; sgi < S * (ch + 1) / nch; ++sgi) {
      const int lo = (int)offs[sgi], n = (int)(offs[sgi + 1] - offs[sgi]);
      if (n <= LEAF) {
        tasks[pos[seg_class(n)]++] = make_int4((int)sgi, lo, n, -1);
      } else if (dense_out && n >= dense_min) {
        continue;
      } else {
        const int nseg = (int)cdiv(n, LEAF), ntask = (int)cdiv(n, 4 * LEAF);
        const long long h = pos[7]++;
        h0[h] = (int)pos[8];
        hg[h] = (int)sgi;
        hn[h] = nseg;
        hs[h] = lo;
        ht[h] = ntask;
        for (int j = 0; j < ntask; ++j)
          tasks[pos[6]++] = make_int4((int)sgi, lo + j * 4 * LEAF, std::min(4 * LEAF, n - j * 4 * LEAF), (int)h);
        pos[8] += nseg;
      }
    }
  }
  hp.tasks.ensure(n_tasks);
  if (n_tasks) CK(cudaMemcpyAsync(hp.tasks.ptr, tasks, sizeof(int4) * n_tasks, cudaMemcpyHostToDevice, stream));
  DevBuf<int>* dsts[5] = {&hp.h0, &hp.hn, &hp.hs, &hp.ht, &hp.hseg};
  int* srcs[5] = {h0, hn, hs, ht, hg};
  for (int k = 0; k < 5; ++k) {
    dsts[k]->ensure(n_heavy);
    if (n_heavy)
      CK(cudaMemcpyAsync(dsts[k]->ptr, srcs[k], sizeof(int) * n_heavy, cudaMemcpyHostToDevice, stream));
  }
  hp.hc.ensure(n_heavy);
  CK(cudaMemsetAsync(hp.hc.ptr, 0, sizeof(unsigned) * std::max<long long>(n_heavy, 1), stream));
  hp.part.ensure(leaves);
  hp.n_heavy = n_heavy;
  hp.n_heavy_leaves = leaves;
  pl.ind = ind;
  pl.tasks = hp.tasks.ptr;
  pl.heavy_seg0 = hp.h0.ptr;
  pl.heavy_nseg = hp.hn.ptr;
  pl.heavy_start = hp.hs.ptr;
  pl.heavy_ntask = hp.ht.ptr;
  pl.heavy_seg = hp.hseg.ptr;
  pl.heavy_count = hp.hc.ptr;
  pl.seg_part = hp.part.ptr;
}

// Per-row-block slice tasks for the dense columns (k_xt_coop phase 1a).
// Rows per staged z block; the oracle's XT_RB must match.
int xt_rb() { return XT_RB; }

void build_dense_plan(fsda_ctx* c, const std::vector<int>& dense) {
  const long long nh = (long long)dense.size();
  const int rb = xt_rb();
  const int nb = (int)std::max<long long>(1, cdiv(c->n, rb));
  c->xh_col.ensure(nh);
  c->xh_bptr.ensure(nh * (nb + 1));
  Trace tr;
  std::vector<int> bptr;
  if (nh) {
    // stream-ordered: a plain cudaMemcpy would also wait for L's copies queued
    // on the side stream by fsda_upload_problem
    CK(cudaMemcpyAsync(c->xh_col.ptr, dense.data(), sizeof(int) * nh, cudaMemcpyHostToDevice, c->stream));
    k_heavy_bptr<<<grid_for(nh * (nb + 1), 256), 256, 0, c->stream>>>(
        c->csc_colptr.ptr, c->csc_rows.ptr, c->xh_col.ptr, c->xh_bptr.ptr, nh, nb, rb);
    CKL();
    bptr.resize(nh * (nb + 1));
    CK(cudaMemcpyAsync(bptr.data(), c->xh_bptr.ptr, sizeof(int) * bptr.size(), cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  tr.mark("  blocked: bptr");
  // pass 1 (parallel over columns): leaf-sum slots — column h owns
  // max(1, ceil(n_hb / 256)) slots per block b — and each (h, b)'s first slot
  std::vector<long long> poff0((size_t)nh + 1, 0);
  std::vector<int> slot0((size_t)nh * nb);
#pragma omp parallel for schedule(dynamic, 64) num_threads(host_threads())
  for (long long h = 0; h < nh; ++h) {
    long long m = 0;
    const int* bp = bptr.data() + h * (nb + 1);
    for (int b = 0; b < nb; ++b) {
      slot0[(size_t)h * nb + b] = (int)m;
      m += std::max<long long>(1, cdiv(bp[b + 1] - bp[b], LEAF));
    }
    poff0[h + 1] = m;
  }
  std::vector<std::pair<long long, int>> bigs;
  for (long long h = 0; h < nh; ++h)
    if (poff0[h + 1] > XT_BIG_PARTS) bigs.push_back({-poff0[h + 1], (int)h});
  std::sort(bigs.begin(), bigs.end());  // most leaf sums first
  std::vector<int> big_ids;
  for (auto& pr : bigs) big_ids.push_back(pr.second);
  c->xh_big.ensure(std::max<size_t>(1, big_ids.size()));
  if (!big_ids.empty())
    CK(cudaMemcpyAsync(c->xh_big.ptr, big_ids.data(), sizeof(int) * big_ids.size(),
                       cudaMemcpyHostToDevice, c->stream));
  for (long long h = 0; h < nh; ++h) poff0[h + 1] += poff0[h];
  // poff[nh] <= nnz / XT_DENSE_PER_BLOCK + nnz / LEAF < 2^31: int slots suffice
  // pass 2 (parallel over blocks): task counts per (block, class)
  std::vector<long long> cnt((size_t)nb * 6, 0);
#pragma omp parallel for schedule(dynamic, 1) num_threads(host_threads())
  for (int b = 0; b < nb; ++b)
    for (long long h = 0; h < nh; ++h) {
      const long long n = bptr[h * (nb + 1) + b + 1] - bptr[h * (nb + 1) + b];
      for (long long c0 = 0; c0 < n; c0 += LEAF) ++cnt[(size_t)b * 6 + seg_class(std::min<long long>(LEAF, n - c0))];
    }
  long long n_tasks = 0;
  for (long long v : cnt) n_tasks += v;
  const size_t n_boff = (size_t)(nb + 1) * 7, n_bwarp = (size_t)nb * 7, n_poff = (size_t)nh + 1;
  char* st = (char*)c->xh_stage.ensure(sizeof(int4) * n_tasks +
                                       sizeof(long long) * (n_boff + n_bwarp + n_poff));
  int4* tasks = (int4*)st;
  long long* boff = (long long*)(tasks + n_tasks);
  long long* bwarp = boff + n_boff;
  long long* poff = bwarp + n_bwarp;
  std::copy(poff0.begin(), poff0.end(), poff);
  std::vector<long long> pos((size_t)nb * 6);
  long long t = 0;
  for (int b = 0; b < nb; ++b) {
    long long wb = 0;
    for (int k = 0; k < 6; ++k) {
      boff[(size_t)b * 7 + k] = t;
      bwarp[(size_t)b * 7 + k] = wb;
      pos[(size_t)b * 6 + k] = t;
      t += cnt[(size_t)b * 6 + k];
      wb += cdiv(cnt[(size_t)b * 6 + k], 32 >> k);
    }
    bwarp[(size_t)b * 7 + 6] = wb;
    boff[(size_t)b * 7 + 6] = t;
  }
  for (int k = 0; k < 7; ++k) boff[(size_t)nb * 7 + k] = t;
  // pass 3 (parallel over blocks): tasks by block, class, column (an empty
  // block's slot stays 0.0, see below)
#pragma omp parallel for schedule(dynamic, 1) num_threads(host_threads())
  for (int b = 0; b < nb; ++b) {
    long long* pb = pos.data() + (size_t)b * 6;
    for (long long h = 0; h < nh; ++h) {
      const int lo = bptr[h * (nb + 1) + b], n = bptr[h * (nb + 1) + b + 1] - lo;
      long long slot = poff[h] + slot0[(size_t)h * nb + b];
      for (int c0 = 0; c0 < n; c0 += LEAF) {
        const int len = std::min(LEAF, n - c0);
        tasks[pb[seg_class(len)]++] = make_int4((int)slot++, lo + c0, len, 0);
      }
    }
  }
  tr.mark("  blocked: host passes");
  c->xh_tasks.ensure(n_tasks);
  c->xh_boff.ensure(n_boff);
  c->xh_bwarp.ensure(n_bwarp);
  c->xh_poff.ensure(n_poff);
  c->xh_part.ensure(std::max<long long>(1, poff[nh]));
  if (n_tasks)
    CK(cudaMemcpyAsync(c->xh_tasks.ptr, tasks, sizeof(int4) * n_tasks, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->xh_boff.ptr, boff, sizeof(long long) * n_boff, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->xh_bwarp.ptr, bwarp, sizeof(long long) * n_bwarp, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->xh_poff.ptr, poff, sizeof(long long) * n_poff, cudaMemcpyHostToDevice, c->stream));
  // empty blocks never get a task: their slots must read 0.0
  if (poff[nh]) CK(cudaMemsetAsync(c->xh_part.ptr, 0, sizeof(double) * poff[nh], c->stream));
  CK(cudaStreamSynchronize(c->stream));  // the staging buffer is reused by the next upload
  tr.mark("  blocked: h2d");
  if (c->xt_blocks == 0) {
    int per_sm = 0;
    // the fp32-storage instance needs half the shared memory: the fp64 grid
    // is co-resident for both
    CK(cudaFuncSetAttribute(k_xt_coop<SegArgs>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(sizeof(double) * rb)));
    CK(cudaFuncSetAttribute(k_xt_coop<SegArgs32D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(sizeof(double) * rb)));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_xt_coop<SegArgs>, XT_THREADS,
                                                     sizeof(double) * rb));
    c->xt_blocks = std::max(1, std::min(per_sm, XT_CTAS_PER_SM)) * c->num_sms;
  }
  XtDense& xh = c->xh;
  xh.rows = c->csc_rows.ptr;
  xh.tasks = c->xh_tasks.ptr;
  xh.boff = c->xh_boff.ptr;
  xh.bwarp = c->xh_bwarp.ptr;
  xh.col = c->xh_col.ptr;
  xh.part = c->xh_part.ptr;
  xh.poff = c->xh_poff.ptr;
  xh.n_dense = nh;
  c->xh_ntasks = n_tasks;
  c->xh_nslots = poff[nh];
  xh.nb = nb;
  xh.rb = rb;
  xh.ticket_chunk = XT_TICKET_CHUNK;
  xh.splits = (int)std::max<long long>(1, c->xt_blocks / nb);
  xh.big = c->xh_big.ptr;
  xh.n_big = (long long)big_ids.size();
  if (!c->xt_ticket.ptr) {
    c->xt_ticket.ensure(1);
    CK(cudaMemset(c->xt_ticket.ptr, 0, sizeof(unsigned long long)));
  }
}

int check_err_flag(fsda_ctx* c, const char* what) {
  int h = 0;
  CK(cudaMemcpy(&h, c->err.ptr, sizeof(int), cudaMemcpyDeviceToHost));
  if (h == 1) return fail(FSDA_EINVAL, "%s: index out of range", what);
  if (h == 2) return fail(FSDA_EINVAL, "%s: row_offsets must be non-decreasing", what);
  if (h == 3) return fail(FSDA_EINVAL, "%s: column indices must be strictly increasing within each row", what);
  if (h == 4)
    return fail(FSDA_EINVAL, "%s: only unit-weight graphs are supported (off-diagonal values must be -1)", what);
  return FSDA_OK;
}

// Upload an int64 index array and narrow it to int32 on the device.
// int64 host indices -> int32 device indices (range-checked into c->err).
// Asynchronous: tmp must stay allocated until the stream has passed it.
// int64 indices already on the device (tmp) -> int32 `out`, range-checked.
void narrow_async(fsda_ctx* c, const long long* tmp, long long n, long long limit, DevBuf<int>& out) {
  out.ensure(n + 8);  // tail padding: the row kernels stage indices with 16-byte loads
  CK(cudaMemsetAsync(out.ptr + n, 0, 8 * sizeof(int), c->stream));
  if (n == 0) return;
  int g = (int)std::min<long long>(cdiv(n, 256), (long long)c->num_sms * 32);
  k_narrow_idx<<<g, 256, 0, c->stream>>>(tmp, out.ptr, n, limit, c->err.ptr);
  CKL();
}

// Host -> device copy of an input array.  Page-locked sources go straight to
// the DMA engine.  Pageable ones (a plain numpy array, as sdakit callers pass
// them) would go through the driver's single-threaded bounce buffer at a
// fraction of the link's speed; instead they stream through a 4-slot pinned
// ring: all host threads copy a 16 MB chunk into a free slot, the DMA drains
// it, and the next chunk fills the next slot meanwhile.
bool host_page_locked(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void h2d(fsda_ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  constexpr size_t CH = (size_t)16 << 20;
  constexpr int SLOTS = 4;
  if (bytes == 0) return;
  if (bytes < CH || host_page_locked(src)) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    return;
  }
  char* ring = static_cast<char*>(c->h2d_ring.ensure(CH * SLOTS));
  for (size_t off = 0; off < bytes; off += CH) {
    const size_t len = std::min(CH, bytes - off);
    const int slot = (int)(c->h2d_next++ % SLOTS);
    CK(cudaEventSynchronize(c->h2d_ev[slot]));  // the DMA out of this slot is done
    char* stage = ring + (size_t)slot * CH;
    const char* from = static_cast<const char*>(src) + off;
    const long long parts = (long long)((len + (1 << 20) - 1) >> 20);
#pragma omp parallel for schedule(dynamic, 1) num_threads(host_threads())
    for (long long k = 0; k < parts; ++k) {
      const size_t a = (size_t)k << 20, b = std::min(len, a + ((size_t)1 << 20));
      memcpy(stage + a, from + a, b - a);
    }
    CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, stage, len, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(c->h2d_ev[slot], st));
  }
}

// One block of the host narrowing: int64 -> int32 with the range check, AVX2
// when the CPU has it (8 indices per step, non-temporal stores: the staged
// int32s are read next by the DMA engine, not by this core, so they need not
// displace the cache or cost a read-for-ownership), scalar otherwise.
// Returns 1 when an index lies outside [0, limit].
int narrow_block_scalar(const int64_t* from, int* stage, long long len, long long limit) {
  int bad = 0;
  for (long long k = 0; k < len; ++k) {
    const long long v = from[k];
    bad |= (v < 0 || v > limit) ? 1 : 0;
    stage[k] = (int)v;
  }
  return bad;
}

#if defined(__x86_64__) && defined(__GNUC__)
__attribute__((target("avx2"))) int narrow_block_avx2(const int64_t* from, int* stage, long long len,
                                                      long long limit) {
  long long k = 0;
  int bad = 0;
  // scalar head up to a 32-byte boundary of the stage (stream stores need it)
  while (k < len && (reinterpret_cast<uintptr_t>(stage + k) & 31u)) {
    const long long v = from[k];
    bad |= (v < 0 || v > limit) ? 1 : 0;
    stage[k] = (int)v;
    ++k;
  }
  const __m256i lim = _mm256_set1_epi64x(limit), zero = _mm256_setzero_si256();
  const __m256i even = _mm256_setr_epi32(0, 2, 4, 6, 0, 2, 4, 6);
  __m256i badv = zero;
  for (; k + 8 <= len; k += 8) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(from + k));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(from + k + 4));
    badv = _mm256_or_si256(badv, _mm256_or_si256(_mm256_cmpgt_epi64(a, lim), _mm256_cmpgt_epi64(zero, a)));
    badv = _mm256_or_si256(badv, _mm256_or_si256(_mm256_cmpgt_epi64(b, lim), _mm256_cmpgt_epi64(zero, b)));
    const __m256i a32 = _mm256_permutevar8x32_epi32(a, even);  // low dwords of a in lanes 0..3
    const __m256i b32 = _mm256_permutevar8x32_epi32(b, even);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(stage + k), _mm256_permute2x128_si256(a32, b32, 0x20));
  }
  bad |= _mm256_testz_si256(badv, badv) ? 0 : 1;
  for (; k < len; ++k) {
    const long long v = from[k];
    bad |= (v < 0 || v > limit) ? 1 : 0;
    stage[k] = (int)v;
  }
  _mm_sfence();
  return bad;
}
#endif

int narrow_block(const int64_t* from, int* stage, long long len, long long limit) {
#if defined(__x86_64__) && defined(__GNUC__)
  static const bool avx2 = __builtin_cpu_supports("avx2") &&
                           !(std::getenv("FSDA_B200_NARROW_SCALAR") && std::atoi(std::getenv("FSDA_B200_NARROW_SCALAR")));
  if (avx2) return narrow_block_avx2(from, stage, len, limit);
#endif
  return narrow_block_scalar(from, stage, len, limit);
}

// int64 host indices -> int32 device indices, narrowed (and range-checked)
// on the host by all threads into the pinned ring, so only half the bytes
// cross the link.  Returns 1 when an index lies outside [0, limit] (the
// check k_narrow_idx makes on the device).
int h2d_narrow(fsda_ctx* c, DevBuf<int>& out, const int64_t* src, long long n, long long limit,
               cudaStream_t st) {
  constexpr size_t CH = (size_t)16 << 20;  // bytes of int32 per ring slot
  constexpr int SLOTS = 4;
  out.ensure(n + 8);  // tail padding: the row kernels stage indices with 16-byte loads
  CK(cudaMemsetAsync(out.ptr + n, 0, 8 * sizeof(int), st));
  if (n == 0) return 0;
  char* ring = static_cast<char*>(c->h2d_ring.ensure(CH * SLOTS));
  const long long che = (long long)(CH / sizeof(int));
  int bad = 0;
  for (long long off = 0; off < n; off += che) {
    const long long len = std::min(che, n - off);
    const int slot = (int)(c->h2d_next++ % SLOTS);
    CK(cudaEventSynchronize(c->h2d_ev[slot]));
    int* stage = reinterpret_cast<int*>(ring + (size_t)slot * CH);
    const int64_t* from = src + off;
    constexpr long long NB = 1 << 16;  // indices per block: a few blocks per thread and chunk
    const long long nblk = (len + NB - 1) / NB;
#pragma omp parallel for schedule(dynamic, 1) reduction(max : bad) num_threads(host_threads())
    for (long long bk = 0; bk < nblk; ++bk) {
      const long long k0 = bk * NB;
      bad = std::max(bad, narrow_block(from + k0, stage + k0, std::min(NB, len - k0), limit));
    }
    CK(cudaMemcpyAsync(out.ptr + off, stage, sizeof(int) * len, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(c->h2d_ev[slot], st));
  }
  return bad;
}

// FSDA_B200_DEVICE_NARROW=1: copy the int64 indices and narrow them on the
// device (the round-1 path) instead of h2d_narrow.
bool device_narrow() {
  static const bool v = std::getenv("FSDA_B200_DEVICE_NARROW") && std::atoi(std::getenv("FSDA_B200_DEVICE_NARROW"));
  return v;
}

// Returns 1 when the host narrowing already saw an index out of range (the
// device flag is raised too); 0 otherwise, or when the device narrows.
int upload_narrow_async(fsda_ctx* c, const int64_t* host, long long n, long long limit,
                        DevBuf<int>& out, long long* tmp) {
  if (!device_narrow()) {
    static const int k_out_of_range = 1;  // check_err_flag's "index out of range"
    const int bad = h2d_narrow(c, out, host, n, limit, c->stream);
    if (bad) CK(cudaMemcpyAsync(c->err.ptr, &k_out_of_range, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    return bad;
  }
  if (n > 0) h2d(c, tmp, host, sizeof(long long) * n, c->stream);
  narrow_async(c, tmp, n, limit, out);
  return 0;
}


#define API_BEGIN(ctx)                                   \
  if (!(ctx)) return fail(FSDA_EINVAL, "null context"); \
  std::lock_guard<std::mutex> lock_((ctx)->mu);          \
  try {                                                  \
    CK(cudaSetDevice((ctx)->device));
#define API_END                                                                     \
  }                                                                                 \
  catch (CudaError & e) {                                                           \
    return fail(FSDA_ECUDA, "CUDA error %s at %s (line %d)", cudaGetErrorString(e.err), e.what, \
                e.line);                                                            \
  }

}  // namespace

// ===================================================================== C ABI

extern "C" {

int fsda_abi_version(void) { return 2; }

int fsda_set_shift_update_mode(fsda_ctx* c, int mode) {
  API_BEGIN(c)
  if (mode < 0 || mode > 2) return fail(FSDA_EINVAL, "shift-update mode must be 0 (auto), 1 or 2");
  c->su_req = mode;
  c->invalidate_graph();
  return FSDA_OK;
  API_END
}

int fsda_last_shift_update_mode(fsda_ctx* c) {
  if (!c) return fail(FSDA_EINVAL, "null context");
  return c->su_mode;
}

int fsda_set_eager(fsda_ctx* c, int eager) {
  API_BEGIN(c)
  c->eager = eager != 0;
  return FSDA_OK;
  API_END
}

int fsda_set_storage(fsda_ctx* c, int bits) {
  API_BEGIN(c)
  if (bits != 32 && bits != 64) return fail(FSDA_EINVAL, "storage must be 32 or 64 bits, got %d", bits);
  c->store_bits = bits;
  c->invalidate_graph();
  return FSDA_OK;
  API_END
}

const char* fsda_last_error(void) { return g_last_error.c_str(); }

int fsda_values_all_ones(const double* values, int64_t n) {
  if (n <= 0) return 1;
  if (!values) return 0;
  int ok = 1;
#pragma omp parallel for schedule(static) reduction(min : ok) if (n > 65536) num_threads(host_threads())
  for (int64_t k = 0; k < n; ++k) ok = std::min(ok, values[k] == 1.0 ? 1 : 0);
  return ok;
}

int fsda_ctx_create(fsda_ctx** out, int device, void* stream) {
  if (!out) return fail(FSDA_EINVAL, "null output pointer");
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(FSDA_ECUDA, "no CUDA device available (%s)", cudaGetErrorString(e));
  if (device < 0 || device >= ndev) return fail(FSDA_EINVAL, "device %d out of range", device);
  fsda_ctx* c = new fsda_ctx();
  c->device = device;
  c->eager = getenv("FSDA_B200_EAGER") && getenv("FSDA_B200_EAGER")[0] == '1';
  try {
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      throw CudaError{cudaErrorInvalidDevice, "this library is built for sm_100a (B200)", __LINE__};
    c->num_sms = prop.multiProcessorCount;
    if (stream) {
      c->stream = (cudaStream_t)stream;
    } else {
      CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    CK(cudaMalloc(&c->sc, sizeof(CgScalars)));
    CK(cudaMemset(c->sc, 0, sizeof(CgScalars)));
    int lo_prio = 0, hi_prio = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    CK(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, lo_prio));
    CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_lfork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_lcopy, cudaEventDisableTiming));
    for (cudaEvent_t& e : c->h2d_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->err.ensure(1);
    CK(cudaMemset(c->err.ptr, 0, sizeof(int)));
  } catch (CudaError& ce) {
    delete c;
    return fail(FSDA_ECUDA, "CUDA error %s at %s", cudaGetErrorString(ce.err), ce.what);
  }
  *out = c;
  return FSDA_OK;
}

void shard_release_comm(fsda_ctx* c);  // fsda_shard.cuh

int fsda_ctx_destroy(fsda_ctx* c) {
  if (!c) return FSDA_OK;
  {
    std::lock_guard<std::mutex> lock(c->mu);
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    c->invalidate_graph();
    DevBuf<int>* ib[] = {&c->x_rowptr, &c->x_cols, &c->csc_colptr, &c->csc_rows, &c->l_rowptr,
                         &c->l_cols, &c->active, &c->good, &c->pending, &c->flip, &c->err};
    c->scratch_i64.release();
    c->scratch_l64.release();
    c->scratch_f64.release();
    c->scratch_row_of.release();
    c->scratch_keys.release();
    c->scratch_sort.release();
    c->xt_ticket.release();
    c->xh_col.release();
    c->xh_bptr.release();
    c->xh_big.release();
    c->xh_tasks.release();
    c->xh_boff.release();
    c->xh_bwarp.release();
    c->xh_part.release();
    c->xh_poff.release();
    c->xh_stage.release();
    c->ldiag_stage.release();
    c->h2d_ring.release();
    c->batch.release();
    c->knn.release();
    c->plan_xr.release();
    c->plan_lr.release();
    c->plan_xc.release();
    for (auto b : ib) b->release();
    c->rbuf.release(); c->coef_a.release(); c->coef_c.release();
    DevBuf<double>* db[] = {&c->l_diag, &c->y, &c->z, &c->q, &c->p,
                            &c->mu_v, &c->t, &c->wv, &c->b, &c->ind, &c->probe, &c->part_n,
                            &c->part_d, &c->part_d2, &c->part_o, &c->bigp, &c->sols, &c->wT, &c->scores,
                            &c->dense_a, &c->beta, &c->zeta_prev, &c->zeta, &c->zeta_next,
                            &c->gamma_s, &c->alpha_s, &c->resid};
    for (auto b : db) b->release();
    c->iters.release();
    c->conv.release();
    c->labels.release();
    if (c->sc) cudaFree(c->sc);
    c->upd_mode.release(); c->upd_gs.release(); c->upd_zn.release(); c->upd_as.release();
    if (c->side) cudaStreamDestroy(c->side);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->ev_lfork) cudaEventDestroy(c->ev_lfork);
    if (c->ev_lcopy) cudaEventDestroy(c->ev_lcopy);
    for (cudaEvent_t e : c->h2d_ev)
      if (e) cudaEventDestroy(e);
    if (c->ev_x) cudaEventDestroy(c->ev_x);
    if (c->ev_y) cudaEventDestroy(c->ev_y);
    c->ypad.release(); c->qpart.release(); c->qrecv.release(); c->qown.release();
    c->spart.release(); c->sall.release();
    shard_release_comm(c);
    if (c->own_stream) cudaStreamDestroy(c->stream);
  }
  delete c;
  return FSDA_OK;
}

int fsda_ctx_set_stream(fsda_ctx* c, void* stream) {
  API_BEGIN(c)
  CK(cudaStreamSynchronize(c->stream));
  if (c->own_stream) CK(cudaStreamDestroy(c->stream));
  c->own_stream = false;
  if (stream) {
    c->stream = (cudaStream_t)stream;
  } else {
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  c->invalidate_graph();
  return FSDA_OK;
  API_END
}

// X upload; `after_h2d` (optional) runs once X's copies are enqueued — the
// combined upload uses it to start the Laplacian's copies behind them.
static int upload_x_impl(fsda_ctx* c, int64_t n_rows, int64_t n_cols, const int64_t* row_offsets,
                         const int64_t* col_indices, void (*after_h2d)(void*), void* hook_arg) {
  if (n_rows < 0 || n_cols < 0) return fail(FSDA_EINVAL, "matrix shape must be non-negative");
  if (!row_offsets) return fail(FSDA_EINVAL, "row_offsets is null");
  const long long nnz = row_offsets[n_rows];
  if (row_offsets[0] != 0 || nnz < 0) return fail(FSDA_EINVAL, "row_offsets must be non-decreasing from 0 to nnz");
  if (nnz > 0 && !col_indices) return fail(FSDA_EINVAL, "col_indices is null");
  if (nnz >= (1LL << 31) - 1 || n_rows >= (1LL << 31) - 1 || n_cols >= (1LL << 31) - 1)
    return fail(FSDA_EINVAL, "X too large for int32 device indices (nnz=%lld)", nnz);
  if (n_rows > MAX_REDUCE || n_cols > MAX_REDUCE)
    return fail(FSDA_EINVAL, "vector length above the two-level reduction limit (%lld)", MAX_REDUCE);
  c->has_x = false;
  if (n_rows != c->n) {
    // the Laplacian and the labels on the device are sized for the old N
    c->has_l = false;
    c->has_labels = false;
    c->n1 = c->n2 = c->ell = 0;
  }
  CK(cudaMemset(c->err.ptr, 0, sizeof(int)));
  c->n = n_rows;
  c->d = n_cols;
  c->nnz = nnz;
  Trace tr;
  // H2D + narrowing run on the stream while the host builds the row plan
  // (it needs only the host offsets).
  c->scratch_i64.ensure(std::max<long long>(n_rows + 1 + nnz, 1));
  int bad_x = upload_narrow_async(c, row_offsets, n_rows + 1, nnz, c->x_rowptr, c->scratch_i64.ptr);
  bad_x |= upload_narrow_async(c, col_indices, nnz, n_cols - 1, c->x_cols, c->scratch_i64.ptr + n_rows + 1);
  // the hook's copies (the Laplacian, on the side stream) queue behind X's
  // copies only, not behind the CSC build enqueued next
  if (after_h2d) CK(cudaEventRecord(c->ev_lfork, c->stream));
  // Row ids (with the in-row order check) and the CSC: a stable radix sort of
  // (column, row) pairs, rows stay ascending.  Enqueued without host syncs.
  DevBuf<int>& row_of = c->scratch_row_of;
  DevBuf<int>& keys_out = c->scratch_keys;
  auto enqueue_csc = [&] {
    row_of.ensure(nnz);
    c->csc_rows.ensure(nnz);
    c->csc_colptr.ensure(n_cols + 1);
    keys_out.ensure(nnz);
    if (n_rows > 0) {
      k_row_ids<<<grid_for(n_rows, 256), 256, 0, c->stream>>>(c->x_rowptr.ptr, c->x_cols.ptr,
                                                              row_of.ptr, (int)n_rows, c->err.ptr);
      CKL();
    }
    if (nnz > 0) {
      int end_bit = 1;
      while ((1LL << end_bit) < n_cols) ++end_bit;
      size_t temp_bytes = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, c->x_cols.ptr, keys_out.ptr, row_of.ptr,
                                         c->csc_rows.ptr, (int)nnz, 0, end_bit, c->stream));
      c->scratch_sort.ensure(temp_bytes);
      void* temp = c->scratch_sort.ptr;
      CK(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, c->x_cols.ptr, keys_out.ptr, row_of.ptr,
                                         c->csc_rows.ptr, (int)nnz, 0, end_bit, c->stream));
    }
    k_colptr_from_sorted<<<grid_for(n_cols + 1, 256), 256, 0, c->stream>>>(keys_out.ptr, nnz,
                                                                            c->csc_colptr.ptr, (int)n_cols);
    CKL();
  };
  // With the indices range-checked on the host, the device builds the CSC
  // while the host runs the hook (the Laplacian's pass) and the row plan;
  // otherwise it waits for the device-side range check first.
  const bool early = !bad_x && !device_narrow();
  if (early) enqueue_csc();
  if (after_h2d) after_h2d(hook_arg);
  build_seg_plan(c->plan_xr, c->stream, row_offsets, n_rows, c->x_cols.ptr);
  tr.mark("x: row plan (host)");
  CK(cudaStreamSynchronize(c->stream));
  int rc = check_err_flag(c, "X");
  if (rc) return rc;
  tr.mark("x: h2d + narrow");
  if (!early) {
    enqueue_csc();
    CK(cudaStreamSynchronize(c->stream));
    rc = check_err_flag(c, "X");
    if (rc) return rc;
  }
  tr.mark("x: csc sort");
  {
    std::vector<int> colptr(n_cols + 1);
    CK(cudaMemcpy(colptr.data(), c->csc_colptr.ptr, sizeof(int) * (n_cols + 1), cudaMemcpyDeviceToHost));
    tr.mark("x: colptr d2h");
    std::vector<int> dense;
    const long long dpb = XT_DENSE_PER_BLOCK;
    const long long dense_min =
        std::max<long long>(LEAF + 1, dpb * std::max<long long>(1, cdiv(n_rows, xt_rb())));
    build_seg_plan(c->plan_xc, c->stream, colptr.data(), n_cols, c->csc_rows.ptr, &dense, dense_min);
    tr.mark("x: column plan");
    build_dense_plan(c, dense);
    tr.mark("x: blocked plan");
  }

  c->has_x = true;
  return FSDA_OK;
}

int fsda_upload_x(fsda_ctx* c, int64_t n_rows, int64_t n_cols, const int64_t* row_offsets,
                  const int64_t* col_indices) {
  API_BEGIN(c)
  return upload_x_impl(c, n_rows, n_cols, row_offsets, col_indices, nullptr, nullptr);
  API_END
}

static int upload_laplacian_rows(fsda_ctx* c, int64_t n, int64_t n_global, int64_t row_base,
                                 const int64_t* row_offsets, const int64_t* col_indices,
                                 const double* values, bool prefetched = false) {
  if (!c->has_x) return fail(FSDA_EINVAL, "upload X before the Laplacian");
  if (n != c->n) return fail(FSDA_EINVAL, "laplacian must be square with one row per sample");
  if (row_base < 0 || row_base + n > n_global)
    return fail(FSDA_EINVAL, "laplacian row block outside [0, n_global)");
  if (!row_offsets) return fail(FSDA_EINVAL, "row_offsets is null");
  const long long nnz = row_offsets[n];
  if (row_offsets[0] != 0 || nnz < 0) return fail(FSDA_EINVAL, "row_offsets must be non-decreasing from 0 to nnz");
  if (nnz >= (1LL << 31) - 1 || n_global >= (1LL << 31) - 1)
    return fail(FSDA_EINVAL, "Laplacian too large for int32 indices");
  c->has_l = false;
  CK(cudaMemset(c->err.ptr, 0, sizeof(int)));
  c->l_nnz = nnz;
  c->row_base = row_base;
  c->n_global = n_global;
  Trace tr;
  // H2D, narrowing and the diagonal split run on the stream while the host
  // builds the row plan.
  if (prefetched) {
    // the raw arrays were copied on the side stream (l_prefetch)
    CK(cudaStreamWaitEvent(c->stream, c->ev_lcopy, 0));
    if (device_narrow()) {
      narrow_async(c, c->scratch_l64.ptr, n + 1, nnz, c->l_rowptr);
      narrow_async(c, c->scratch_l64.ptr + n + 1, nnz, n_global - 1, c->l_cols);
    }
  } else {
    c->scratch_l64.ensure(std::max<long long>(n + 1 + nnz, 1));
    upload_narrow_async(c, row_offsets, n + 1, nnz, c->l_rowptr, c->scratch_l64.ptr);
    upload_narrow_async(c, col_indices, nnz, n_global - 1, c->l_cols, c->scratch_l64.ptr + n + 1);
  }
  c->l_diag.ensure(n);
  if (prefetched) {
    // values checked and the diagonal split on the host by l_prefetch
    if (c->l_host_err) {
      CK(cudaStreamSynchronize(c->stream));
      const int e = c->l_host_err;
      c->l_host_err = 0;
      CK(cudaMemcpy(c->err.ptr, &e, sizeof(int), cudaMemcpyHostToDevice));
      return check_err_flag(c, "laplacian");
    }
  } else if (n > 0) {
    c->scratch_f64.ensure(std::max<long long>(nnz, 1));
    double* dvals = c->scratch_f64.ptr;
    if (nnz > 0)
      h2d(c, dvals, values, sizeof(double) * nnz, c->stream);
    k_laplacian_split<<<grid_for(n, 256), 256, 0, c->stream>>>(c->l_rowptr.ptr, c->l_cols.ptr, dvals,
                                                               c->l_diag.ptr, (int)n, c->err.ptr,
                                                               (int)row_base);
    CKL();
  }
  build_seg_plan(c->plan_lr, c->stream, row_offsets, n, c->l_cols.ptr);
  tr.mark("L: row plan (host)");
  CK(cudaStreamSynchronize(c->stream));
  int rc = check_err_flag(c, "laplacian");
  if (rc) return rc;
  tr.mark("L: h2d + split");
  c->has_l = true;
  return FSDA_OK;
}

int fsda_upload_laplacian(fsda_ctx* c, int64_t n, const int64_t* row_offsets,
                          const int64_t* col_indices, const double* values) {
  API_BEGIN(c)
  return upload_laplacian_rows(c, n, n, 0, row_offsets, col_indices, values);
  API_END
}

namespace {
struct LPrefetch {
  fsda_ctx* c;
  long long n, nnz;
  const int64_t* offs;
  const int64_t* cols;
  const double* vals;
};

// The Laplacian's raw arrays to device scratch on the side stream, queued
// behind X's copies, so they cross the link while X's CSC and plans build.
// The Laplacian's columns in one host pass (offsets already checked):
// narrowed to int32 into the pinned ring and copied on the side stream, and in
// the same sweep the order check, the unit-weight check and the diagonal
// split — cols is read once instead of twice.  Entries go ring chunk by ring
// chunk; the rows overlapping a chunk are found by binary search in offs and
// shared out over the host threads.  Returns the validation code (0, 3 or 4);
// *range_bad = 1 when a column lies outside [0, n).
int l_cols_fused(fsda_ctx* c, const LPrefetch* a, double* diag, int* range_bad) {
  constexpr size_t CH = (size_t)16 << 20;  // bytes of int32 per ring slot (as h2d_narrow)
  constexpr int SLOTS = 4;
  const long long n = a->n, nnz = a->nnz;
  const int64_t* offs = a->offs;
  const int64_t* cols = a->cols;
  const double* vals = a->vals;
  cudaStream_t st = c->side;
  c->l_cols.ensure(nnz + 8);  // tail padding: the row kernels stage indices with 16-byte loads
  CK(cudaMemsetAsync(c->l_cols.ptr + nnz, 0, 8 * sizeof(int), st));
#pragma omp parallel for schedule(static) num_threads(host_threads())
  for (long long i = 0; i < n; ++i) diag[i] = 0.0;
  char* ring = static_cast<char*>(c->h2d_ring.ensure(CH * SLOTS));
  const long long che = (long long)(CH / sizeof(int));
  int err = 0, bad = 0;
  for (long long off = 0; off < nnz; off += che) {
    const long long len = std::min(che, nnz - off), end = off + len;
    const int slot = (int)(c->h2d_next++ % SLOTS);
    CK(cudaEventSynchronize(c->h2d_ev[slot]));
    int* stage = reinterpret_cast<int*>(ring + (size_t)slot * CH);
    // rows with entries in [off, end): from the last row starting at or before off
    const long long r0 = std::max<long long>(0, (std::upper_bound(offs, offs + n + 1, (int64_t)off) - offs) - 1);
    const long long r1 = std::min<long long>(n, std::lower_bound(offs, offs + n + 1, (int64_t)end) - offs);
#pragma omp parallel for schedule(dynamic, 2048) reduction(max : err, bad) num_threads(host_threads())
    for (long long i = r0; i < r1; ++i) {
      const long long lo = offs[i], hi = offs[i + 1];
      const long long jb = std::max(lo, off), je = std::min(hi, end);
      for (long long jj = jb; jj < je; ++jj) {
        const long long cc = cols[jj];
        if (cc < 0 || cc > n - 1) bad = 1;
        stage[jj - off] = (int)cc;
        if (jj > lo && cc <= cols[jj - 1]) err = std::max(err, 3);
        if (cc == i) diag[i] = vals[jj];
        else if (vals[jj] != -1.0) err = std::max(err, 4);
      }
    }
    CK(cudaMemcpyAsync(c->l_cols.ptr + off, stage, sizeof(int) * len, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(c->h2d_ev[slot], st));
  }
  *range_bad = bad;
  return err;
}

void l_prefetch(void* arg) {
  LPrefetch* a = static_cast<LPrefetch*>(arg);
  fsda_ctx* c = a->c;
  CK(cudaStreamWaitEvent(c->side, c->ev_lfork, 0));  // recorded behind X's copies by upload_x_impl
  int range_err = 0;
  if (device_narrow()) {
    c->scratch_l64.ensure(std::max<long long>(a->n + 1 + a->nnz, 1));
    h2d(c, c->scratch_l64.ptr, a->offs, sizeof(long long) * (a->n + 1), c->side);
    if (a->nnz > 0) h2d(c, c->scratch_l64.ptr + a->n + 1, a->cols, sizeof(long long) * a->nnz, c->side);
  } else {
    range_err |= h2d_narrow(c, c->l_rowptr, a->offs, a->n + 1, a->nnz, c->side);
    // offsets that walk the entries exactly once let the columns go in one fused pass
    static const bool fuse = !std::getenv("FSDA_B200_L_FUSED") || std::atoi(std::getenv("FSDA_B200_L_FUSED"));
    int off_ok = fuse && !range_err && a->nnz > 0 && a->n > 0 && a->offs[0] == 0 && a->offs[a->n] == a->nnz;
    if (off_ok) {
      const int64_t* o = a->offs;
      const long long nn = a->n;
#pragma omp parallel for schedule(static) reduction(min : off_ok) num_threads(host_threads())
      for (long long i = 0; i < nn; ++i) off_ok = std::min(off_ok, o[i + 1] >= o[i] ? 1 : 0);
    }
    if (off_ok) {
      double* dg = static_cast<double*>(c->ldiag_stage.ensure(sizeof(double) * std::max<long long>(a->n, 1)));
      int bad = 0;
      const int err = l_cols_fused(c, a, dg, &bad);
      c->l_host_err = bad ? 1 : err;
      c->l_diag.ensure(std::max<long long>(a->n, 1));
      CK(cudaMemcpyAsync(c->l_diag.ptr, dg, sizeof(double) * a->n, cudaMemcpyHostToDevice, c->side));
      CK(cudaEventRecord(c->ev_lcopy, c->side));
      return;
    }
    range_err |= h2d_narrow(c, c->l_cols, a->cols, a->nnz, a->n - 1, c->side);
  }
  // L's values never cross the link: off-diagonals must be -1 (a unit-weight
  // graph, graph.py:191-195) and the diagonal is the degree, so the host
  // checks them and splits the diagonal out (what k_laplacian_split does on
  // the device) while the index copies are in flight — 12 MB instead of the
  // values' 8 bytes per entry.
  const long long n = a->n, nnz = a->nnz;
  const int64_t* offs = a->offs;
  const int64_t* cols = a->cols;
  const double* vals = a->vals;
  double* diag = static_cast<double*>(c->ldiag_stage.ensure(sizeof(double) * std::max<long long>(n, 1)));
  int err = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(max : err) num_threads(host_threads())
  for (long long i = 0; i < n; ++i) {
    const long long lo = offs[i], hi = offs[i + 1];
    double dv = 0.0;
    if (lo < 0 || hi < lo || hi > nnz) {
      err = std::max(err, 2);
    } else {
      for (long long jj = lo; jj < hi; ++jj) {
        const long long cc = cols[jj];
        if (jj > lo && cc <= cols[jj - 1]) err = std::max(err, 3);
        if (cc == i) dv = vals[jj];
        else if (vals[jj] != -1.0) err = std::max(err, 4);
      }
    }
    diag[i] = dv;
  }
  c->l_host_err = range_err ? 1 : err;
  c->l_diag.ensure(std::max<long long>(n, 1));
  if (n > 0) CK(cudaMemcpyAsync(c->l_diag.ptr, diag, sizeof(double) * n, cudaMemcpyHostToDevice, c->side));
  CK(cudaEventRecord(c->ev_lcopy, c->side));
}
}  // namespace

static int set_labels_impl(fsda_ctx* c, const int8_t* labels, bool require_first);

// Host-side label checks (values in {+1, -1, 0}; labeled rows first when
// required); counts the classes.
static int check_labels(const int8_t* labels, long long n, bool require_first, long long* n1_out,
                        long long* n2_out) {
  // one pass over host threads: class counts, value check, and the position of
  // the first unlabeled / last labeled row (labeled-first <=> last < first)
  long long n1 = 0, n2 = 0, first_unlabeled = n, last_labeled = -1;
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : n1, n2) reduction(max : bad, last_labeled) num_threads(host_threads()) \
    reduction(min : first_unlabeled) if (n > 65536)
  for (long long i = 0; i < n; ++i) {
    const int8_t l = labels[i];
    if (l != 0 && l != 1 && l != -1) bad = 1;
    n1 += l == 1;
    n2 += l == -1;
    if (l == 0) first_unlabeled = std::min(first_unlabeled, i);
    else last_labeled = std::max(last_labeled, i);
  }
  if (bad) return fail(FSDA_ELABEL, "labels must take values in {+1, -1, 0}");
  const bool labeled_first = last_labeled < first_unlabeled;
  if (require_first && !labeled_first)
    return fail(FSDA_EINVAL,
                "labeled samples must occupy the first rows; use arrange_labeled_first to permute the problem");
  *n1_out = n1;
  *n2_out = n2;
  return FSDA_OK;
}

int fsda_upload_problem(fsda_ctx* c, int64_t n_rows, int64_t n_cols, const int64_t* x_offsets,
                        const int64_t* x_cols, const int64_t* l_offsets, const int64_t* l_cols,
                        const double* l_values, const int8_t* labels) {
  API_BEGIN(c)
  if (!l_offsets || !labels) return fail(FSDA_EINVAL, "laplacian row_offsets / labels are null");
  if (n_rows < 0) return fail(FSDA_EINVAL, "matrix shape must be non-negative");
  const long long l_nnz = l_offsets[n_rows];
  if (l_offsets[0] != 0 || l_nnz < 0) return fail(FSDA_EINVAL, "row_offsets must be non-decreasing from 0 to nnz");
  if (l_nnz >= (1LL << 31) - 1) return fail(FSDA_EINVAL, "Laplacian too large for int32 indices");
  if (l_nnz > 0 && (!l_cols || !l_values)) return fail(FSDA_EINVAL, "laplacian arrays are null");
  {
    // the labels are checked before anything on the device is replaced
    long long n1 = 0, n2 = 0;
    int lrc = check_labels(labels, n_rows, true, &n1, &n2);
    if (lrc) return lrc;
  }
  LPrefetch pf{c, n_rows, l_nnz, l_offsets, l_cols, l_values};
  int rc = upload_x_impl(c, n_rows, n_cols, x_offsets, x_cols, l_prefetch, &pf);
  if (rc) {
    CK(cudaStreamSynchronize(c->side));  // the prefetch (if issued) reads host memory of this call
    return rc;
  }
  rc = upload_laplacian_rows(c, n_rows, n_rows, 0, l_offsets, l_cols, l_values, true);
  if (rc) return rc;
  return set_labels_impl(c, labels, true);
  API_END
}

int fsda_upload_laplacian_rows(fsda_ctx* c, int64_t n_local, int64_t n_global, int64_t row_base,
                               const int64_t* row_offsets, const int64_t* col_indices,
                               const double* values) {
  API_BEGIN(c)
  return upload_laplacian_rows(c, n_local, n_global, row_base, row_offsets, col_indices, values);
  API_END
}

static int set_labels_impl(fsda_ctx* c, const int8_t* labels, bool require_first) {
  if (!c->has_x) return fail(FSDA_EINVAL, "upload X before the labels");
  long long n1 = 0, n2 = 0;
  int rc = check_labels(labels, c->n, require_first, &n1, &n2);
  if (rc) return rc;
  c->has_labels = false;
  c->labels.ensure(std::max<long long>(c->n, 1));
  if (c->n > 0)
    CK(cudaMemcpyAsync(c->labels.ptr, labels, c->n, cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->n1 = n1;
  c->n2 = n2;
  c->ell = n1 + n2;
  c->has_labels = true;
  return FSDA_OK;
}

int fsda_set_labels(fsda_ctx* c, const int8_t* labels) {
  API_BEGIN(c)
  return set_labels_impl(c, labels, true);
  API_END
}

int fsda_set_label_mask(fsda_ctx* c, const int8_t* labels) {
  API_BEGIN(c)
  return set_labels_impl(c, labels, false);
  API_END
}

// ---- parity probes ---------------------------------------------------------

int fsda_matvec(fsda_ctx* c, const double* v, double* yout) {
  API_BEGIN(c)
  if (!c->has_x) return fail(FSDA_EINVAL, "X has not been uploaded");
  ensure_vectors(c, 1);
  CK(cudaMemcpyAsync(c->p.ptr, v, sizeof(double) * c->d, cudaMemcpyHostToDevice, c->stream));
  if (c->n > 0) {
    k_spmv_rows<<<grid_for(c->n, 256), 256, 0, c->stream>>>(c->x_rowptr.ptr, c->x_cols.ptr, c->p.ptr,
                                                            c->y.ptr, (int)c->n, nullptr);
    CKL();
  }
  CK(cudaMemcpyAsync(yout, c->y.ptr, sizeof(double) * c->n, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return FSDA_OK;
  API_END
}

static int xt_probe(fsda_ctx* c, const double* mu, const double* w, double* out, int mode) {
  ensure_vectors(c, 1);
  CK(cudaMemcpyAsync(c->z.ptr, w, sizeof(double) * c->n, cudaMemcpyHostToDevice, c->stream));
  if (mode == 1) {
    CK(cudaMemcpyAsync(c->mu_v.ptr, mu, sizeof(double) * c->d, cudaMemcpyHostToDevice, c->stream));
    long long nl = n_leaves(c->n);
    k_vector_sum<<<grid_for(nl, WARPS_PER_BLOCK), LEAF_THREADS, 0, c->stream>>>(
        c->z.ptr, c->n, c->part_n.ptr, nl, c->sc, nullptr);
    CKL();
  }
  Enq e{c};
  enq_xt(e, c->z.ptr, c->q.ptr, mode, &c->sc->sum_z, 0, nullptr);
  CK(cudaMemcpyAsync(out, c->q.ptr, sizeof(double) * c->d, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return FSDA_OK;
}

int fsda_matvec_transpose(fsda_ctx* c, const double* w, double* u) {
  API_BEGIN(c)
  if (!c->has_x) return fail(FSDA_EINVAL, "X has not been uploaded");
  return xt_probe(c, nullptr, w, u, 0);
  API_END
}

int fsda_centered_matvec_transpose(fsda_ctx* c, const double* mu, const double* w, double* u) {
  API_BEGIN(c)
  if (!c->has_x) return fail(FSDA_EINVAL, "X has not been uploaded");
  return xt_probe(c, mu, w, u, 1);
  API_END
}

int fsda_labeled_mean(fsda_ctx* c, double* mu) {
  API_BEGIN(c)
  if (!c->has_x || !c->has_labels) return fail(FSDA_EINVAL, "X and labels must be uploaded");
  if (c->ell == 0) return fail(FSDA_ELABEL, "centering requires at least one labeled sample");
  ensure_vectors(c, 1);
  k_indicator<<<grid_for(c->n, 256), 256, 0, c->stream>>>(c->labels.ptr, c->ind.ptr, (int)c->n);
  CKL();
  Enq e{c};
  enq_xt(e, c->ind.ptr, c->mu_v.ptr, 2, nullptr, 0, nullptr);
  CK(cudaMemcpyAsync(mu, c->mu_v.ptr, sizeof(double) * c->d, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return FSDA_OK;
  API_END
}

int fsda_apply_smoother(fsda_ctx* c, double alpha, const double* yin, double* zout) {
  API_BEGIN(c)
  if (!c->has_l || !c->has_labels) return fail(FSDA_EINVAL, "Laplacian and labels must be uploaded");
  if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(FSDA_EINVAL, "alpha must lie in [0, 1], got %g", alpha);
  ensure_vectors(c, 1);
  CK(cudaMemcpyAsync(c->y.ptr, yin, sizeof(double) * c->n, cudaMemcpyHostToDevice, c->stream));
  Enq e{c};
  enq_smoother(e, alpha, c->y.ptr, c->z.ptr, 0);
  CK(cudaMemcpyAsync(zout, c->z.ptr, sizeof(double) * c->n, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return FSDA_OK;
  API_END
}

int fsda_operator_apply(fsda_ctx* c, double alpha, const double* w, double* qout) {
  API_BEGIN(c)
  if (!c->has_x || !c->has_l || !c->has_labels)
    return fail(FSDA_EINVAL, "X, Laplacian and labels must be uploaded");
  if (c->ell == 0) return fail(FSDA_ELABEL, "centering requires at least one labeled sample");
  ensure_vectors(c, 1);
  // mu
  k_indicator<<<grid_for(c->n, 256), 256, 0, c->stream>>>(c->labels.ptr, c->ind.ptr, (int)c->n);
  CKL();
  Enq e{c};
  enq_xt(e, c->ind.ptr, c->mu_v.ptr, 2, nullptr, 0, nullptr);
  CK(cudaMemcpyAsync(c->p.ptr, w, sizeof(double) * c->d, cudaMemcpyHostToDevice, c->stream));
  enq_xrows(e, c->p.ptr, c->y.ptr, 0);
  enq_smoother(e, alpha, c->y.ptr, c->z.ptr, 0);
  long long nl = n_leaves(c->n);
  k_vector_sum<<<grid_for(nl, WARPS_PER_BLOCK), LEAF_THREADS, 0, c->stream>>>(
      c->z.ptr, c->n, c->part_n.ptr, nl, c->sc, nullptr);
  CKL();
  enq_xt(e, c->z.ptr, c->q.ptr, 1, &c->sc->sum_z, 0, nullptr);
  CK(cudaMemcpyAsync(qout, c->q.ptr, sizeof(double) * c->d, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return FSDA_OK;
  API_END
}

// ---- the hot path -----------------------------------------------------------

int fsda_solve(fsda_ctx* c, double alpha, const double* betas, int ns, double tol,
               int64_t max_iter, const double* probe, double* directions, double* scores,
               double* residuals, int64_t* iterations, uint8_t* converged, int64_t* n_applies,
               int64_t* fail_iter) {
  API_BEGIN(c)
  int rc = check_solve_args(c, alpha, betas, ns, tol);
  if (rc) return rc;
  if (!probe) return fail(FSDA_EINVAL, "probe is null");
  c->solve_kind = 0;
  c->solve_abs_tol = 0;
  Trace tr;
  upload_solve_params(c, betas, ns, probe, max_iter);
  launch_solve(c, alpha, ns, max_iter, tol, nullptr);
  if (tr.on) {
    CK(cudaStreamSynchronize(c->stream));
    tr.mark("solve: device");
  }
  SolveOut o{directions, scores, residuals, iterations, converged, n_applies, fail_iter};
  rc = read_results(c, ns, o, nullptr);
  tr.mark("solve: d2h results");
  return rc;
  API_END
}

int fsda_prepare_resident(fsda_ctx* c, double alpha, const double* betas, int ns, double tol,
                          int64_t max_iter, const double* probe) {
  API_BEGIN(c)
  int rc = check_solve_args(c, alpha, betas, ns, tol);
  if (rc) return rc;
  c->solve_kind = 0;
  c->solve_abs_tol = 0;
  upload_solve_params(c, betas, ns, probe, max_iter);
  CK(cudaStreamSynchronize(c->stream));
  c->r_alpha = alpha;
  c->r_ns = ns;
  c->r_tol = tol;
  c->r_max_iter = max_iter;
  c->r_prepared = true;
  return FSDA_OK;
  API_END
}

int fsda_solve_async(fsda_ctx* c) {
  API_BEGIN(c)
  if (!c->r_prepared) return fail(FSDA_EINVAL, "call fsda_prepare_resident first");
  c->solve_kind = 0;
  resolve_shift_mode(c, c->r_ns, c->r_max_iter, c->d);
  ensure_vectors(c, c->r_ns);
  launch_solve(c, c->r_alpha, c->r_ns, c->r_max_iter, c->r_tol, nullptr);
  return FSDA_OK;
  API_END
}

int fsda_fetch_results(fsda_ctx* c, double* directions, double* scores, double* residuals,
                       int64_t* iterations, uint8_t* converged, int64_t* n_applies,
                       int64_t* fail_iter, int64_t* launches) {
  API_BEGIN(c)
  if (!c->r_prepared) return fail(FSDA_EINVAL, "call fsda_prepare_resident first");
  SolveOut o{directions, scores, residuals, iterations, converged, n_applies, fail_iter};
  return read_results(c, c->r_ns, o, launches);
  API_END
}

int fsda_profile_kernels(fsda_ctx* c, int max_kernels, int* n_kernels, const char** names,
                         double* ms_per_launch, double* bytes_per_launch,
                         int64_t* launches_per_solve) {
  API_BEGIN(c)
  if (!c->r_prepared) return fail(FSDA_EINVAL, "call fsda_prepare_resident first");
  Recorder rec;
  rec.stream = c->stream;
  c->solve_kind = 0;
  resolve_shift_mode(c, c->r_ns, c->r_max_iter, c->d);
  ensure_vectors(c, c->r_ns);
  launch_solve(c, c->r_alpha, c->r_ns, c->r_max_iter, c->r_tol, &rec);
  CK(cudaStreamSynchronize(c->stream));
  // accumulate per name, skipping launches after the loop finished is not
  // needed: for the measured configurations every iteration runs.
  std::vector<std::string> order;
  std::map<std::string, double> ms, bytes;
  std::map<std::string, long long> cnt;
  for (size_t k = 0; k < rec.names.size(); ++k) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, rec.ev[2 * k], rec.ev[2 * k + 1]));
    std::string nm = rec.names[k].first;
    if (!cnt.count(nm)) order.push_back(nm);
    ms[nm] += t;
    bytes[nm] = rec.names[k].second;
    cnt[nm] += 1;
  }
  static thread_local std::vector<std::string> keep;
  keep = order;
  int k = 0;
  for (auto& nm : keep) {
    if (k >= max_kernels) break;
    names[k] = nm.c_str();
    ms_per_launch[k] = ms[nm] / (double)cnt[nm];
    bytes_per_launch[k] = bytes[nm];
    launches_per_solve[k] = cnt[nm];
    ++k;
  }
  *n_kernels = k;
  return FSDA_OK;
  API_END
}

int fsda_shifted_cg_dense(fsda_ctx* c, int64_t dim, const double* a, const double* bvec,
                          const double* betas, int ns, double tol, int64_t max_iter,
                          int absolute_tol, double* solutions, double* residuals,
                          int64_t* iterations, uint8_t* converged, int64_t* n_applies,
                          int64_t* fail_iter) {
  API_BEGIN(c)
  if (dim <= 0) return fail(FSDA_EINVAL, "operator dimension must be positive");
  if (dim > MAX_REDUCE) return fail(FSDA_EINVAL, "dimension above the reduction limit");
  if (ns <= 0) return fail(FSDA_EINVAL, "shift grid must be a non-empty 1-d array");
  if (ns > FSDA_MAX_SHIFTS) return fail(FSDA_EINVAL, "at most 4096 shifts per solve");
  for (int s = 0; s < ns; ++s) {
    if (!std::isfinite(betas[s])) return fail(FSDA_EINVAL, "shifts must be finite");
    if (s == 0 && betas[s] < 0) return fail(FSDA_EINVAL, "shifts must be non-negative");
    if (s > 0 && !(betas[s] > betas[s - 1])) return fail(FSDA_EINVAL, "shifts must be strictly ascending");
  }
  if (!(tol > 0)) return fail(FSDA_EINVAL, "tol must be positive");
  // Borrow the solve buffers with d = dim; restore the problem shape on exit.
  struct ShapeGuard {
    fsda_ctx* c;
    long long n, d;
    ~ShapeGuard() { c->n = n; c->d = d; c->invalidate_graph(); }
  } guard{c, c->n, c->d};
  c->d = dim;
  c->n = std::max<long long>(c->n, 1);
  resolve_shift_mode(c, ns, max_iter, dim);
  ensure_vectors(c, ns);
  c->dense_a.ensure((size_t)dim * dim);
  CK(cudaMemcpyAsync(c->dense_a.ptr, a, sizeof(double) * dim * dim, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->b.ptr, bvec, sizeof(double) * dim, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->beta.ptr, betas, sizeof(double) * ns, cudaMemcpyHostToDevice, c->stream));
  ShiftState ss = c->shifts();
  k_solve_reset<<<1, 256, 0, c->stream>>>(c->sc, ss, ns, max_iter, tol, absolute_tol);
  CKL();
  launch_cg_init(c, c->b.ptr, dim, ns);
  for (long long it = 0; it < max_iter; ++it) {
    k_dense_matvec<<<grid_for(dim, 128), 128, 0, c->stream>>>(c->dense_a.ptr, c->p.ptr, c->q.ptr,
                                                              (int)dim, c->sc);
    CKL();
    launch_cg_step(c, ns, dim, 0, 0, 0);
    launch_shift_update(c, ns, dim, c->stream, 1);
    if ((it & 15) == 15) {  // stop launching once every shift froze
      CgScalars h;
      CK(cudaMemcpyAsync(&h, c->sc, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      if (h.finished || h.status) break;
    }
  }
  launch_final_shift(c, ns, dim);
  k_cg_finish<<<1, 32, 0, c->stream>>>(c->sc, ss, ns);
  CKL();
  SolveOut o{solutions, nullptr, residuals, iterations, converged, n_applies, fail_iter};
  return read_results(c, ns, o, nullptr);
  API_END
}

// ---- row-sharded building blocks -------------------------------------------

int fsda_dev_xrows(fsda_ctx* c, const double* d_v, double* d_y) {
  API_BEGIN(c)
  if (!c->has_x) return fail(FSDA_EINVAL, "X has not been uploaded");
  ensure_vectors(c, 1);
  Enq e{c};
  enq_xrows(e, d_v, d_y, 0);
  return FSDA_OK;
  API_END
}

int fsda_dev_smoother(fsda_ctx* c, double alpha, const double* d_y_full, double* d_z) {
  API_BEGIN(c)
  if (!c->has_l || !c->has_labels) return fail(FSDA_EINVAL, "Laplacian and labels must be uploaded");
  if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(FSDA_EINVAL, "alpha must lie in [0, 1], got %g", alpha);
  ensure_vectors(c, 1);
  Enq e{c};
  enq_smoother(e, alpha, d_y_full, d_z, 0);
  return FSDA_OK;
  API_END
}

int fsda_dev_xt_partial(fsda_ctx* c, const double* d_z, double* d_out) {
  API_BEGIN(c)
  if (!c->has_x) return fail(FSDA_EINVAL, "X has not been uploaded");
  ensure_vectors(c, 1);
  Enq e{c};
  enq_xt(e, d_z, d_out, 0, nullptr, 0, nullptr);
  const long long nl = n_leaves(c->n);
  k_vector_sum<<<grid_for(nl, WARPS_PER_BLOCK), LEAF_THREADS, 0, c->stream>>>(
      d_z, c->n, c->part_n.ptr, nl, c->sc, d_out + c->d);
  CKL();
  return FSDA_OK;
  API_END
}

int fsda_dev_class_sums(fsda_ctx* c, const double* d_t, double* d_out) {
  API_BEGIN(c)
  if (!c->has_labels) return fail(FSDA_EINVAL, "labels have not been set");
  ensure_vectors(c, 1);
  const long long nl = n_leaves(c->n);
  k_class_sums<<<grid_for(nl, WARPS_PER_BLOCK), LEAF_THREADS, 0, c->stream>>>(
      d_t, c->labels.ptr, c->n, c->part_n.ptr, nl, c->sc, 1.0, 1.0);
  CKL();
  CK(cudaMemcpyAsync(d_out, &c->sc->class_mean1, 2 * sizeof(double), cudaMemcpyDeviceToDevice,
                     c->stream));
  return FSDA_OK;
  API_END
}

int fsda_dev_apply_w(fsda_ctx* c, double c1, double c2, double* d_w) {
  API_BEGIN(c)
  if (!c->has_labels) return fail(FSDA_EINVAL, "labels have not been set");
  ensure_vectors(c, 1);
  const double cm[2] = {c1, c2};
  CK(cudaMemcpyAsync(&c->sc->class_mean1, cm, 2 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  const long long nl = n_leaves(c->n);
  k_apply_w<<<grid_for(nl, WARPS_PER_BLOCK), LEAF_THREADS, 0, c->stream>>>(
      c->labels.ptr, d_w, c->n, c->part_n.ptr, nl, c->sc);
  CKL();
  CK(cudaStreamSynchronize(c->stream));  // cm lives on this stack frame
  return FSDA_OK;
  API_END
}

int fsda_dev_center(fsda_ctx* c, const double* d_mu, double* d_q, double scale) {
  API_BEGIN(c)
  k_center<<<grid_for(c->d, 256), 256, 0, c->stream>>>(d_mu, d_q, c->d, scale);
  CKL();
  return FSDA_OK;
  API_END
}

int fsda_dev_cg_begin(fsda_ctx* c, const double* betas, int ns, double tol, int64_t max_iter,
                      const double* d_b) {
  API_BEGIN(c)
  if (c->d <= 0) return fail(FSDA_EINVAL, "operator dimension must be positive");
  if (ns <= 0) return fail(FSDA_EINVAL, "shift grid must be a non-empty 1-d array");
  if (ns > FSDA_MAX_SHIFTS) return fail(FSDA_EINVAL, "at most 4096 shifts per solve");
  for (int s = 0; s < ns; ++s) {
    if (!std::isfinite(betas[s])) return fail(FSDA_EINVAL, "shifts must be finite");
    if (s == 0 && betas[s] < 0) return fail(FSDA_EINVAL, "shifts must be non-negative");
    if (s > 0 && !(betas[s] > betas[s - 1])) return fail(FSDA_EINVAL, "shifts must be strictly ascending");
  }
  if (!(tol > 0)) return fail(FSDA_EINVAL, "tol must be positive");
  upload_solve_params(c, betas, ns, nullptr, max_iter);
  ShiftState ss = c->shifts();
  const long long d = c->d;
  k_solve_reset<<<1, 256, 0, c->stream>>>(c->sc, ss, ns, max_iter, tol, 0);
  CKL();
  launch_cg_init(c, d_b, d, ns);
  c->r_ns = ns;
  CK(cudaStreamSynchronize(c->stream));  // betas were read from host memory
  return FSDA_OK;
  API_END
}

int fsda_dev_cg_step(fsda_ctx* c, const double* d_q) {
  API_BEGIN(c)
  if (c->r_ns <= 0) return fail(FSDA_EINVAL, "call fsda_dev_cg_begin first");
  if (d_q != c->q.ptr)
    CK(cudaMemcpyAsync(c->q.ptr, d_q, sizeof(double) * c->d, cudaMemcpyDeviceToDevice, c->stream));
  launch_cg_step(c, c->r_ns, c->d, 0, 0, 0);
  launch_shift_update(c, c->r_ns, c->d, c->stream, 1);
  return FSDA_OK;
  API_END
}

int fsda_dev_cg_direction(fsda_ctx* c, const double** d_p) {
  API_BEGIN(c)
  ensure_vectors(c, 1);
  *d_p = c->p.ptr;
  return FSDA_OK;
  API_END
}

int fsda_dev_cg_status(fsda_ctx* c, int* finished, int64_t* iterations, int* status) {
  API_BEGIN(c)
  CgScalars h;
  CK(cudaMemcpyAsync(&h, c->sc, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (finished) *finished = h.finished;
  if (iterations) *iterations = h.iter;
  if (status) *status = h.status;
  return FSDA_OK;
  API_END
}

int fsda_dev_project(fsda_ctx* c, double* d_scores, double* d_orient) {
  API_BEGIN(c)
  const int ns = c->r_ns;
  if (ns <= 0) return fail(FSDA_EINVAL, "call fsda_dev_cg_begin first");
  const long long n = c->n, d = c->d, nlN = n_leaves(n);
  ShiftState ss = c->shifts();
  launch_final_shift(c, ns, d);
  k_cg_finish<<<1, 32, 0, c->stream>>>(c->sc, ss, ns);
  k_transpose_sols<<<grid_for(d * ns, 256), 256, 0, c->stream>>>(c->sols.ptr, c->wT.ptr, d, ns);
  if (n > 0)
    k_spmm_scores<<<grid_for(n, 8), 256, 0, c->stream>>>(c->x_rowptr.ptr, c->x_cols.ptr, c->wT.ptr,
                                                         d_scores, (int)n, ns);
  dim3 g(grid_for(nlN, WARPS_PER_BLOCK), ns);
  k_orient<<<g, LEAF_THREADS, 0, c->stream>>>(c->labels.ptr, d_scores, n, c->part_o.ptr, nlN);
  k_orient_final<<<ns, 256, 0, c->stream>>>(c->part_o.ptr, nlN, ss, d_orient);
  CKL();
  return FSDA_OK;
  API_END
}

int fsda_dev_finish(fsda_ctx* c, const uint8_t* flip, double* d_scores, double* directions,
                    double* residuals, int64_t* iterations, uint8_t* converged, int64_t* n_applies,
                    int64_t* fail_iter) {
  API_BEGIN(c)
  const int ns = c->r_ns;
  if (ns <= 0) return fail(FSDA_EINVAL, "call fsda_dev_cg_begin first");
  std::vector<int> fl(ns);
  for (int s = 0; s < ns; ++s) fl[s] = flip[s] ? 1 : 0;
  CK(cudaMemcpyAsync(c->flip.ptr, fl.data(), sizeof(int) * ns, cudaMemcpyHostToDevice, c->stream));
  ShiftState ss = c->shifts();
  dim3 g((unsigned)std::min<long long>(grid_for(std::max(c->n, c->d), 256), 1024), ns);
  k_flip<<<g, 256, 0, c->stream>>>(d_scores, c->sols.ptr, c->n, c->d, ss);
  CKL();
  SolveOut o{directions, nullptr, residuals, iterations, converged, n_applies, fail_iter};
  return read_results(c, ns, o, nullptr);
  API_END
}

int fsda_regression_shifted_cg(fsda_ctx* c, const double* rhs, const double* betas, int ns,
                                double tol, int64_t max_iter, int absolute_tol, double* solutions,
                                double* residuals, int64_t* iterations, uint8_t* converged,
                                int64_t* n_applies, int64_t* fail_iter) {
  API_BEGIN(c)
  if (!c->has_x) return fail(FSDA_EINVAL, "X has not been uploaded");
  if (c->d <= 0) return fail(FSDA_EINVAL, "operator dimension must be positive");
  if (ns <= 0) return fail(FSDA_EINVAL, "shift grid must be a non-empty 1-d array");
  if (ns > FSDA_MAX_SHIFTS) return fail(FSDA_EINVAL, "at most 4096 shifts per solve");
  for (int s = 0; s < ns; ++s) {
    if (!std::isfinite(betas[s])) return fail(FSDA_EINVAL, "shifts must be finite");
    if (s == 0 && betas[s] < 0) return fail(FSDA_EINVAL, "shifts must be non-negative");
    if (s > 0 && !(betas[s] > betas[s - 1])) return fail(FSDA_EINVAL, "shifts must be strictly ascending");
  }
  if (!(tol > 0)) return fail(FSDA_EINVAL, "tol must be positive");
  upload_solve_params(c, betas, ns, nullptr, max_iter);
  CK(cudaMemcpyAsync(c->b.ptr, rhs, sizeof(double) * c->d, cudaMemcpyHostToDevice, c->stream));
  c->solve_kind = 1;
  c->solve_abs_tol = absolute_tol ? 1 : 0;
  launch_solve(c, 0.0, ns, max_iter, tol, nullptr);
  SolveOut o{solutions, nullptr, residuals, iterations, converged, n_applies, fail_iter};
  const int rc = read_results(c, ns, o, nullptr);
  c->solve_kind = 0;
  return rc;
  API_END
}

int fsda_sa_solve(fsda_ctx* c, double alpha, const double* betas, int ns, double tol,
                  int64_t max_iter, const double* probe, double* solutions, double* residuals,
                  int64_t* iterations, uint8_t* converged, int64_t* n_applies, int64_t* fail_iter) {
  API_BEGIN(c)
  if (!c->has_l || !c->has_labels) return fail(FSDA_EINVAL, "Laplacian and labels must be uploaded");
  if (alpha == 0.0)
    return fail(FSDA_EINVAL, "sa-sda requires alpha != 0: without the Laplacian term the spectral "
                             "system never propagates ratings to unlabeled samples");
  if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(FSDA_EINVAL, "alpha must lie in [0, 1], got %g", alpha);
  if (c->ell == 0) return fail(FSDA_ELABEL, "centering requires at least one labeled sample");
  if (c->n1 == 0 || c->n2 == 0) return fail(FSDA_EINVAL, "both classes need at least one labeled sample");
  if (ns <= 0) return fail(FSDA_EINVAL, "shift grid must be a non-empty 1-d array");
  if (ns > FSDA_MAX_SHIFTS) return fail(FSDA_EINVAL, "at most 4096 shifts per solve");
  for (int s = 0; s < ns; ++s) {
    if (!std::isfinite(betas[s])) return fail(FSDA_EINVAL, "shifts must be finite");
    if (s == 0 && betas[s] < 0) return fail(FSDA_EINVAL, "shifts must be non-negative");
    if (s > 0 && !(betas[s] > betas[s - 1])) return fail(FSDA_EINVAL, "shifts must be strictly ascending");
  }
  if (!(tol > 0)) return fail(FSDA_EINVAL, "tol must be positive");
  if (c->n > MAX_REDUCE) return fail(FSDA_EINVAL, "N above the reduction limit");
  // the recurrence runs over N-vectors: borrow the D-space buffers with d = N
  struct DimGuard {
    fsda_ctx* c;
    long long d;
    ~DimGuard() { c->d = d; c->solve_kind = 0; }
  } guard{c, c->d};
  c->d = c->n;
  c->solve_kind = 2;
  c->solve_abs_tol = 0;
  ensure_vectors(c, ns);
  upload_solve_params(c, betas, ns, nullptr, max_iter);
  CK(cudaMemcpyAsync(c->t.ptr, probe, sizeof(double) * c->n, cudaMemcpyHostToDevice, c->stream));
  launch_solve(c, alpha, ns, max_iter, tol, nullptr);
  SolveOut o{solutions, nullptr, residuals, iterations, converged, n_applies, fail_iter};
  return read_results(c, ns, o, nullptr);
  API_END
}


// ---- multi-task batch (fsda_batch.cuh) -----------------------------------

extern "C++" {
// V: storage type of the loop vectors P, Y, Z and the residual slots (double,
// or float after fsda_set_storage(32): sums, dots and scalars stay double —
// the single solve's fp32-storage mode per task).
template <typename V>
static int batch_solve_t(fsda_ctx* c, int T, const int8_t* labels, double alpha,
                            const double* betas, int ns, double tol, int64_t max_iter,
                            const double* probes, double* directions, double* scores,
                            double* residuals, int64_t* iterations, uint8_t* converged,
                            int64_t* n_applies, int64_t* fail_iter, int* status) {
  if (!c->has_x) return fail(FSDA_EINVAL, "fsda_solve_batch: X has not been uploaded");
  if (!c->has_l) return fail(FSDA_EINVAL, "fsda_solve_batch: Laplacian has not been uploaded");
  if (T <= 0) return fail(FSDA_EINVAL, "fsda_solve_batch: need at least one task");
  if (!labels || !probes || !betas) return fail(FSDA_EINVAL, "fsda_solve_batch: null input");
  if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(FSDA_EINVAL, "alpha must lie in [0, 1], got %g", alpha);
  if (ns <= 0) return fail(FSDA_EINVAL, "shift grid must be a non-empty 1-d array");
  if (ns > FSDA_MAX_SHIFTS) return fail(FSDA_EINVAL, "at most 4096 shifts per solve");
  for (int s = 0; s < ns; ++s) {
    if (!std::isfinite(betas[s])) return fail(FSDA_EINVAL, "shifts must be finite");
    if (s == 0 && betas[s] < 0) return fail(FSDA_EINVAL, "shifts must be non-negative");
    if (s > 0 && !(betas[s] > betas[s - 1])) return fail(FSDA_EINVAL, "shifts must be strictly ascending");
  }
  if (!(tol > 0)) return fail(FSDA_EINVAL, "tol must be positive");
  if (c->row_base != 0 || c->n_global != c->n)
    return fail(FSDA_EINVAL, "fsda_solve_batch: needs the whole Laplacian (not a row shard)");
  const long long n = c->n, d = c->d;
  Trace tr;
  const int G = (T + BG - 1) / BG, tp = G * BG;
  if ((std::max(n, d) + 1) * (long long)tp * 8 >= (1LL << 32))  // the setup products gather doubles in either storage
    return fail(FSDA_EINVAL, "fsda_solve_batch: a task-minor vector must stay below 4 GiB (32-bit gather offsets)");
  std::vector<double> ell(tp, 1.0), n1v(tp, 1.0), n2v(tp, 1.0);
  std::vector<int> bad(T, 0);
#pragma omp parallel for schedule(static) num_threads(host_threads())
  for (int t = 0; t < T; ++t) {
    long long a = 0, b = 0;
    int other = 0;
    const int8_t* l = labels + (long long)t * n;
    for (long long i = 0; i < n; ++i) {
      other |= (l[i] != 0 && l[i] != 1 && l[i] != -1);
      a += l[i] == 1;
      b += l[i] == -1;
    }
    bad[t] = other ? 1 : (a + b == 0 ? 2 : ((a == 0 || b == 0) ? 3 : 0));
    ell[t] = (double)(a + b);
    n1v[t] = (double)a;
    n2v[t] = (double)b;
  }
  for (int t = 0; t < T; ++t) {
    if (bad[t] == 1) return fail(FSDA_ELABEL, "task %d: labels must take values in {+1, -1, 0}", t);
    if (bad[t] == 2) return fail(FSDA_ELABEL, "task %d: centering requires at least one labeled sample", t);
    if (bad[t] == 3) return fail(FSDA_EINVAL, "task %d: both classes need at least one labeled sample", t);
  }
  tr.mark("batch: validate labels");
  BatchBufs& bb = c->batch;
  cudaStream_t st = c->stream;
  const long long nlN = n_leaves(n), nlD = n_leaves(d);
  const long long ND = (long long)tp;
  // shift-update mode (as resolve_shift_mode, for T tasks): the deferred basis
  // keeps max_iter + 1 task-minor residuals
  int bmode = c->su_req;
  if (bmode == 0 && std::getenv("FSDA_B200_SHIFT_MODE")) bmode = std::atoi(std::getenv("FSDA_B200_SHIFT_MODE"));
  const long long bslots = std::max<long long>(max_iter, 0) + 1;
  if (bmode == 0) {
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    const double need = 8.0 * (double)bslots * (double)std::max<long long>(d, 1) * (double)tp +
                        16.0 * (double)tp * ns * (double)bslots;
    const double have = 8.0 * (double)(c->batch.RB.cap + c->batch.CA.cap + c->batch.CC.cap);
    bmode = need <= 0.4 * (double)free_b + have ? 2 : 1;
  }
  constexpr bool V32 = sizeof(V) == 4;
  if (V32) bmode = 2;  // as the single solve: fp32 storage keeps the residual basis
  if ((long long)tp * ns > 65535) {  // kb_coef_update's grid.y is one (task, shift)
    if (V32) return fail(FSDA_EINVAL, "fsda_solve_batch: fp32 storage supports at most 65535 (task, shift) pairs");
    bmode = 1;
  }
  c->su_mode = bmode;
  const bool basis = bmode == 2;
  bb.lab.ensure(n * ND);
  // every gathered table (ind, PR, P over features; Y, Z over samples) carries
  // one more row of zeros: the gathers' out-of-range slots read it
  bb.ind.ensure((n + 1) * ND);
  for (DevBuf<double>* v : {&bb.P, &bb.Q, &bb.MU, &bb.Bv, &bb.PR}) v->ensure(std::max(1LL, (d + 1) * ND));
  if (basis) {
    bb.RB.ensure(std::max(1LL, V32 ? cdiv(bslots * d * ND, 2) : bslots * d * ND));
    bb.CA.ensure(std::max(1LL, bslots * ND * ns));
    bb.CC.ensure(std::max(1LL, bslots * ND * ns));
  } else {
    bb.R0.ensure(std::max(1LL, d * ND));
    bb.R1.ensure(std::max(1LL, d * ND));
  }
  // fp64 storage: Y also holds -(d_i y_i) in rows n + 1 .. 2n + 1, the block the
  // loop's K2 reads for its diagonal slot (TermLapNeg), when the 32-bit gather
  // offsets reach it
  const bool use_yd = !V32 && (2 * n + 2) * (long long)tp * 8 < (1LL << 32) &&
                      !(std::getenv("FSDA_B200_BATCH_YD") && !std::atoi(std::getenv("FSDA_B200_BATCH_YD")));
  bb.Y.ensure(std::max(1LL, (use_yd ? 2 * n + 2 : n + 1) * ND));
  bb.Z.ensure(std::max(1LL, (n + 1) * ND));
  bb.BIGP.ensure(basis ? 1LL : std::max(1LL, d * ND * ns));
  bb.SOLS.ensure(std::max(1LL, d * ND * ns));
  bb.SCORES.ensure(std::max(1LL, n * ND * ns));
  bb.OUT.ensure(std::max(1LL, (long long)T * ns * d));
  bb.partD.ensure(std::max(1LL, nlD * ND));
  bb.partN.ensure(std::max(1LL, nlN * ND));
  bb.part2.ensure(std::max(1LL, cdiv(std::max(nlN, nlD), LEAF) * ND));
  bb.hpart.ensure(std::max(1LL, c->plan_xc.n_heavy_leaves * ND));
  bb.xpart.ensure(std::max(1LL, c->xh_nslots * ND));
  bb.opart.ensure(std::max(1LL, nlN * ND * ns));
  bb.scal.ensure(15 * ND);
  bb.lscal.ensure(2 * ND + 1);
  bb.iscal.ensure(5 * ND + 2);
  bb.sh_d.ensure(9 * ND * ns);
  bb.sh_l.ensure(ND * ns);
  bb.sh_u.ensure(4 * ND * ns);
  bb.sh_i.ensure(ND * ns);
  bb.betas.ensure(ns);
  // inputs
  bb.raw.ensure((long long)T * d * 8);
  bb.labt.ensure(std::max<long long>((long long)T * n, 1));  // task-major labels, kept for the orientation
  h2d(c, bb.labt.ptr, labels, (size_t)T * n, st);
  kb_labels_in<<<(unsigned)std::min<long long>(cdiv(n * ND, 256), 65535LL * 4), 256, 0, st>>>(
      bb.labt.ptr, bb.lab.ptr, bb.ind.ptr, n, T, tp);
  CKL();
  h2d(c, bb.raw.ptr, probes, sizeof(double) * T * d, st);
  kb_task_minor<<<(unsigned)std::min<long long>(cdiv(d * ND, 256), 65535LL * 4), 256, 0, st>>>(
      (const double*)bb.raw.ptr, bb.PR.ptr, d, T, tp);
  CKL();
  CK(cudaMemcpyAsync(bb.betas.ptr, betas, sizeof(double) * ns, cudaMemcpyHostToDevice, st));
  // loop vectors in storage type (the setup products use Y / Z as doubles)
  V* const Pv = reinterpret_cast<V*>(bb.P.ptr);
  V* const Yv = reinterpret_cast<V*>(bb.Y.ptr);
  V* const Zv = reinterpret_cast<V*>(bb.Z.ptr);
  V* const RBv = reinterpret_cast<V*>(bb.RB.ptr);
  auto zero_row = [&](auto* table, long long rows) {
    CK(cudaMemsetAsync(table + rows * ND, 0, sizeof(*table) * ND, st));
  };
  zero_row(bb.ind.ptr, n);   // the setup products gather doubles
  zero_row(bb.PR.ptr, d);
  zero_row(bb.Y.ptr, n);
  zero_row(bb.Z.ptr, n);
  BatchState B;
  double* sd = bb.scal.ptr;
  B.rr = sd; B.gamma_prev = sd + ND; B.alpha = sd + 2 * ND; B.b_norm = sd + 3 * ND;
  B.thresh = sd + 4 * ND; B.gamma = sd + 5 * ND; B.alpha_new = sd + 6 * ND; B.mean1 = sd + 7 * ND;
  B.mean2 = sd + 8 * ND; B.ell = sd + 9 * ND; B.n1 = sd + 10 * ND; B.n2 = sd + 11 * ND;
  B.sum_v = sd + 12 * ND; B.pq = sd + 13 * ND; B.rr_new = sd + 14 * ND;
  B.iter = bb.lscal.ptr; B.fail_iter = bb.lscal.ptr + ND;
  B.status = bb.iscal.ptr; B.finished = bb.iscal.ptr + ND; B.n_active = bb.iscal.ptr + 2 * ND;
  int* stepped = bb.iscal.ptr + 3 * ND;
  int* n_live = bb.iscal.ptr + 5 * ND;
  const long long NS = ND * ns;
  double* hd = bb.sh_d.ptr;
  B.zeta_prev = hd; B.zeta = hd + NS; B.alpha_s = hd + 2 * NS; B.resid = hd + 3 * NS;
  B.s_zn = hd + 4 * NS; B.s_gs = hd + 5 * NS; B.upd_gs = hd + 6 * NS; B.upd_zn = hd + 7 * NS;
  B.upd_as = hd + 8 * NS;
  B.iters = bb.sh_l.ptr;
  B.s_good = bb.sh_u.ptr; B.conv = bb.sh_u.ptr + NS; B.active = bb.sh_u.ptr + 2 * NS;
  B.flip = bb.sh_u.ptr + 3 * NS;
  B.upd_mode = bb.sh_i.ptr;
  B.beta = bb.betas.ptr;
  B.ns = ns;
  B.tp = tp;
  B.max_iter = max_iter;
  CK(cudaMemcpyAsync(B.ell, ell.data(), sizeof(double) * ND, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(B.n1, n1v.data(), sizeof(double) * ND, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(B.n2, n2v.data(), sizeof(double) * ND, cudaMemcpyHostToDevice, st));
  const int tb = (int)cdiv(ND, 128);
  kb_reset<<<tb, 128, 0, st>>>(B, T, tol);
  CKL();
  if (tr.on) {
    CK(cudaStreamSynchronize(st));
    tr.mark("batch: alloc + inputs h2d");
  }
  if (c->xh_nslots) CK(cudaMemsetAsync(bb.xpart.ptr, 0, sizeof(double) * c->xh_nslots * ND, st));

  auto grid_w = [](long long warps) { return (unsigned)std::max<long long>(1, cdiv(warps, 8)); };
  auto rows_x = [&](auto* src, auto* out) {
    using U = std::remove_cv_t<std::remove_pointer_t<decltype(out)>>;
    kb_rows<SEG_XROWS, U><<<grid_w(n * G), 256, 0, st>>>(c->x_rowptr.ptr, c->x_cols.ptr, (const U*)src, out,
                                                        n, G, tp, nullptr, nullptr, 0.0, 0, d, 0);
    CKL();
  };
  // the loop's K1 / K2 in fp64 storage: y and -(d y) out of K1, K2 without the diagonal select
  auto rows_x_yd = [&](const double* src, double* out) {
    kb_rows<SEG_XROWS, double, true><<<grid_w(n * G), 256, 0, st>>>(
        c->x_rowptr.ptr, c->x_cols.ptr, src, out, n, G, tp, c->l_diag.ptr, nullptr, 0.0, 0, d, n + 1);
    CKL();
  };
  auto smoother_yd = [&](const double* y, double* z) {
    kb_rows<SEG_LROWS, double, true><<<grid_w(n * G), 256, 0, st>>>(
        c->l_rowptr.ptr, c->l_cols.ptr, y, z, n, G, tp, c->l_diag.ptr, bb.lab.ptr, alpha, alpha_mode_of(alpha), n,
        n + 1);
    CKL();
  };
  auto smoother = [&](auto* y, auto* z) {
    using U = std::remove_cv_t<std::remove_pointer_t<decltype(z)>>;
    const int amode = alpha_mode_of(alpha);
    if (amode == 0)
      kb_mask<U><<<(unsigned)std::min<long long>(cdiv(n * ND, 256), 65535LL * 4), 256, 0, st>>>(
          (const U*)y, bb.lab.ptr, z, n * ND);
    else
      kb_rows<SEG_LROWS, U><<<grid_w(n * G), 256, 0, st>>>(c->l_rowptr.ptr, c->l_cols.ptr, (const U*)y, z, n,
                                                          G, tp, c->l_diag.ptr, bb.lab.ptr, alpha, amode, n, 0);
    CKL();
  };
  const SegPlan& pxc = c->plan_xc.pl;
  const long long n_light = pxc.cls_off[6];
  const long long n_htask = pxc.warp_base[7] - pxc.warp_base[6];
  const long long n_heavy = c->plan_xc.n_heavy;
  // units (heavy segments, blocked columns) with more than 256 leaf partials:
  // their level-1 group leaves go to kb_part_groups, spread over warps
  long long n_gchunks = 0;
  {
    const long long nu = n_heavy + c->xh.n_dense;
    std::vector<int> hn((size_t)std::max<long long>(n_heavy, 1));
    std::vector<long long> poff((size_t)c->xh.n_dense + 1, 0);
    if (n_heavy) CK(cudaMemcpy(hn.data(), pxc.heavy_nseg, sizeof(int) * n_heavy, cudaMemcpyDeviceToHost));
    if (c->xh.n_dense)
      CK(cudaMemcpy(poff.data(), c->xh.poff, sizeof(long long) * (c->xh.n_dense + 1), cudaMemcpyDeviceToHost));
    std::vector<int> gso((size_t)std::max<long long>(nu, 1), -1);
    std::vector<int2> chunks;
    long long slots = 0;
    for (long long u = 0; u < nu; ++u) {
      const long long m = u < n_heavy ? hn[u] : poff[u - n_heavy + 1] - poff[u - n_heavy];
      if (m <= LEAF) continue;
      const long long m2 = cdiv(m, LEAF);
      gso[u] = (int)slots;
      for (long long j = 0; j < m2; ++j) chunks.push_back(make_int2((int)u, (int)j));
      slots += m2;
    }
    n_gchunks = (long long)chunks.size();
    bb.gsoff.ensure(std::max<long long>(nu, 1));
    bb.gchunks.ensure(std::max<long long>(n_gchunks, 1));
    bb.gsum.ensure(std::max<long long>(slots * ND, 1));
    if (nu) CK(cudaMemcpyAsync(bb.gsoff.ptr, gso.data(), sizeof(int) * nu, cudaMemcpyHostToDevice, st));
    if (n_gchunks)
      CK(cudaMemcpyAsync(bb.gchunks.ptr, chunks.data(), sizeof(int2) * n_gchunks, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));  // the host vectors go out of scope
  }
  auto xt = [&](auto* src_any, double* out, int mode) {
    using U = std::remove_cv_t<std::remove_pointer_t<decltype(src_any)>>;
    const U* src = src_any;
    if (n_light)
      kb_cols_light<U><<<grid_w(n_light * G), 256, 0, st>>>(pxc, src, out, G, tp, mode, bb.MU.ptr, B, n);
    CKL();
    if (n_htask || c->xh_ntasks) {
      kb_cols_leaves<U><<<grid_w((4 * n_htask + c->xh_ntasks) * G), 256, 0, st>>>(
          pxc, c->xh, src, bb.hpart.ptr, bb.xpart.ptr, 4 * n_htask, c->xh_ntasks, G, tp, n);
      CKL();
      if (n_gchunks) {
        kb_part_groups<<<grid_w(n_gchunks * G), 256, 0, st>>>(pxc, c->xh, bb.hpart.ptr, bb.xpart.ptr, n_heavy,
                                                              bb.gchunks.ptr, n_gchunks, bb.gsoff.ptr,
                                                              bb.gsum.ptr, G, tp);
        CKL();
      }
      kb_cols_combine<<<grid_w((n_heavy + c->xh.n_dense) * G), 256, 0, st>>>(
          pxc, c->xh, bb.hpart.ptr, bb.xpart.ptr, n_heavy, out, G, tp, mode, bb.MU.ptr, B,
          n_gchunks ? bb.gsoff.ptr : nullptr, bb.gsum.ptr);
      CKL();
    }
  };
  // the block-level leaves use 8 KB of static shared memory
  const size_t sm_dot = 0, sm_sum = 0;
  auto combine = [&](const double* part, long long nl, double* out) {
    // R256 over nl <= 65536 partials: level 1 (runs of 256) by kb_vec_leaves,
    // the last level by kb_combine_leaf
    if (nl > LEAF) {
      const long long m2 = cdiv(nl, LEAF);
      kb_vec_leaves<double><<<(unsigned)(m2 * G), 256, sm_sum, st>>>(part, nullptr, nullptr, nl, 0,
                                                                     bb.part2.ptr, m2, G, tp);
      CKL();
      part = bb.part2.ptr;
      nl = m2;
    }
    kb_combine_leaf<<<G, 256, sm_sum, st>>>(part, (int)nl, out, tp);
    CKL();
  };
  auto vec_sum = [&](auto* v_any, decltype(v_any) v2, int kind, long long len, double* part,
                     double* out) {
    using U = std::remove_cv_t<std::remove_pointer_t<decltype(v_any)>>;
    const U* v = v_any;
    const long long nl = n_leaves(len);
    if (nl == 0) {
      CK(cudaMemsetAsync(out, 0, sizeof(double) * ND, st));
      return;
    }
    kb_vec_leaves<U><<<(unsigned)(nl * G), 256, kind == 3 ? sm_dot : sm_sum, st>>>(
        v, (const U*)v2, bb.lab.ptr, len, kind, part, nl, G, tp);
    CKL();
    combine(part, nl, out);
  };

  // ---- setup (sda.py:297-301, krylov.py:185-208), per task
  xt(bb.ind.ptr, bb.MU.ptr, 2);                       // mu = X^T 1_l / l
  rows_x(bb.PR.ptr, bb.Y.ptr);                        // t = X r
  vec_sum(bb.Y.ptr, (double*)nullptr, 1, n, bb.partN.ptr, B.pq);
  vec_sum(bb.Y.ptr, (double*)nullptr, 2, n, bb.partN.ptr, B.rr_new);
  kb_class_means<<<tb, 128, 0, st>>>(B, B.pq, B.rr_new);
  CKL();
  kb_apply_w<<<(unsigned)std::min<long long>(cdiv(n * ND, 256), 65535LL * 4), 256, 0, st>>>(
      bb.lab.ptr, bb.Z.ptr, n * ND, tp, B);
  CKL();
  vec_sum(bb.Z.ptr, (double*)nullptr, 0, n, bb.partN.ptr, B.sum_v);   // sum(w)
  xt(bb.Z.ptr, bb.Bv.ptr, 1);                                // b = X^T w - mu sum(w)
  // threads per block: the (task, shift) pairs split evenly over <= 1024 threads
  const long long tsn = ND * ns, passes = cdiv(tsn, 1024);
  const int sblk = (int)(cdiv(cdiv(tsn, passes), 32) * 32);
  const unsigned srows = (unsigned)std::max<long long>(1, std::min<long long>(d, (long long)c->num_sms * 8));
  const unsigned vblocks = (unsigned)std::max<long long>(1, std::min<long long>(cdiv(d * ND, 256), (long long)c->num_sms * 16));
  if (basis) {
    kb_cg_init_rp<V><<<vblocks, 256, 0, st>>>(bb.Bv.ptr, RBv, Pv, d * ND);
    CKL();
    kb_coef_init<<<(unsigned)std::min<long long>(cdiv(bslots * ND * ns, 256), 4096), 256, 0, st>>>(
        bb.CA.ptr, bb.CC.ptr, ND * ns, bslots);
    CKL();
  } else {
    kb_cg_init_vec<<<srows, sblk, 0, st>>>(
        bb.Bv.ptr, bb.R0.ptr, bb.P.ptr, bb.BIGP.ptr, bb.SOLS.ptr, d, tp, ns);
    CKL();
  }
  vec_sum(bb.Bv.ptr, bb.Bv.ptr, 3, d, bb.partD.ptr, B.pq);   // b.b
  kb_cg_init_scalars<<<tb, 128, 0, st>>>(B, B.pq, tol);
  CKL();
  if (tr.on) {
    CK(cudaStreamSynchronize(st));
    tr.mark("batch: setup");
  }

  // the loop vectors' zero rows, in storage type (the setup used Y / Z as doubles)
  zero_row(Pv, d);
  zero_row(Yv, n);
  zero_row(Zv, n);
  // ---- the shifted-CG loop (krylov.py:210-270), all live tasks in step.
  // The iteration index lives on the device (kb_loop_next), so the body is
  // the same launches every time: it runs as a CUDA graph whose conditional
  // WHILE node repeats it until no task is live or max_iter is reached (no
  // host round trip per iteration), or eagerly from a host loop
  // (FSDA_B200_EAGER=1 / fsda_set_eager, or no conditional-node support).
  long long* loop_it = bb.lscal.ptr + 2 * ND;
  int* keep = n_live + 1;
  BIterT<V> bi{RBv, reinterpret_cast<V*>(bb.R0.ptr), reinterpret_cast<V*>(bb.R1.ptr), d * ND, basis ? 1 : 0,
               loop_it};
  CK(cudaMemsetAsync(loop_it, 0, sizeof(long long), st));
  CK(cudaMemsetAsync(n_live, 0, sizeof(int), st));
  auto body = [&](unsigned long long handle, int use_cond) {
    if constexpr (!V32) {
      if (use_yd && alpha_mode_of(alpha) != 0) {
        rows_x_yd(bb.P.ptr, bb.Y.ptr);                         // K1  y = X p and -(d y)
        smoother_yd(bb.Y.ptr, bb.Z.ptr);                       // K2  z = M y
      } else {
        rows_x(Pv, Yv);
        smoother(Yv, Zv);
      }
    } else {
      rows_x(Pv, Yv);                                          // K1  y = X p
      smoother(Yv, Zv);                                        // K2  z = M y
    }
    xt(Zv, bb.Q.ptr, 0);                                       // K3  q = X^T z
    vec_sum(Zv, (V*)nullptr, 0, n, bb.partN.ptr, B.sum_v);     //     sum(z)
    if (nlD) {
      kb_step_a<V><<<(unsigned)(nlD * G), 256, sm_dot, st>>>(bb.Q.ptr, Pv, bb.MU.ptr, d, bb.partD.ptr,
                                                             nlD, G, B);
      CKL();
      combine(bb.partD.ptr, nlD, B.pq);
    } else {
      CK(cudaMemsetAsync(B.pq, 0, sizeof(double) * ND, st));
    }
    kb_scalars_b<<<tb, 128, 0, st>>>(B);
    CKL();
    if (nlD) {
      kb_step_b<V><<<(unsigned)(nlD * G), 256, sm_dot, st>>>(bb.Q.ptr, bi, d, bb.partD.ptr, nlD, G, B);
      CKL();
      combine(bb.partD.ptr, nlD, B.rr_new);
    } else {
      CK(cudaMemsetAsync(B.rr_new, 0, sizeof(double) * ND, st));
    }
    kb_scalars_c<<<tb, 128, 0, st>>>(B);
    CKL();
    kb_mark_stepped<<<tb, 128, 0, st>>>(B, stepped);
    CKL();
    if (basis) {
      kb_step_c_p<V><<<vblocks, 256, 0, st>>>(bi, Pv, d * ND, tp, B, stepped);
      CKL();
      kb_coef_update<<<dim3((unsigned)cdiv(bslots + 1, 256), (unsigned)(ND * ns)), 256, 0, st>>>(
          B, stepped, bb.CA.ptr, bb.CC.ptr, bslots, loop_it);
      CKL();
    } else {
      if constexpr (!V32) {
        kb_step_c<<<srows, sblk, 0, st>>>(bi, bb.P.ptr, bb.BIGP.ptr, bb.SOLS.ptr, d, B, stepped);
        CKL();
      }
    }
    kb_end_iteration<<<tb, 128, 0, st>>>(B, stepped, n_live);
    CKL();
    kb_loop_next<<<1, 1, 0, st>>>(n_live, loop_it, max_iter, keep, handle, use_cond);
    CKL();
  };
  cudaGraphExec_t loop_exec = nullptr;
  cudaGraph_t loop_graph = nullptr;
  bool looped = max_iter <= 0;
  if (!looped && c->cond_supported && !c->eager) {
    try {
      CK(cudaGraphCreate(&loop_graph, 0));
      cudaGraphConditionalHandle handle;
      CK(cudaGraphConditionalHandleCreate(&handle, loop_graph, 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = handle;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t cond_node;
      CK(cudaGraphAddNode(&cond_node, loop_graph, nullptr, 0, &cp));
      CK(cudaStreamBeginCaptureToGraph(st, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                       cudaStreamCaptureModeThreadLocal));
      try {
        body((unsigned long long)handle, 1);
      } catch (...) {
        cudaGraph_t g2;
        cudaStreamEndCapture(st, &g2);
        throw;
      }
      cudaGraph_t body_out;
      CK(cudaStreamEndCapture(st, &body_out));
      CK(cudaGraphInstantiate(&loop_exec, loop_graph, 0));
      CK(cudaGraphLaunch(loop_exec, st));
      looped = true;
    } catch (CudaError& ce) {
      if (loop_exec) cudaGraphExecDestroy(loop_exec);
      if (loop_graph) cudaGraphDestroy(loop_graph);
      loop_exec = nullptr;
      loop_graph = nullptr;
      if (ce.err != cudaErrorNotSupported && ce.err != cudaErrorCallRequiresNewerDriver) throw;
      cudaGetLastError();
      c->cond_supported = false;  // the eager loop below
    }
  }
  if (!looped) {
    for (long long it = 0; it < max_iter; ++it) {
      body(0ULL, 0);
      int h_keep = 0;
      CK(cudaMemcpyAsync(&h_keep, keep, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (!h_keep) break;
    }
  }
  struct LoopGraphGuard {
    cudaGraphExec_t& e;
    cudaGraph_t& g;
    cudaStream_t s;
    ~LoopGraphGuard() {
      if (e || g) cudaStreamSynchronize(s);
      if (e) cudaGraphExecDestroy(e);
      if (g) cudaGraphDestroy(g);
    }
  } loop_guard{loop_exec, loop_graph, st};
  if (tr.on) CK(cudaStreamSynchronize(st));
  if (tr.on) tr.mark("batch: iterations");
  // ---- tail: directions (deferred mode), residuals, projections, orientation
  // (sda.py:265-284)
  if (basis && d > 0) {
    kb_combine_basis<V><<<(unsigned)cdiv(d * ND, 256), 256, 0, st>>>(RBv, d, B, bb.CC.ptr, bslots,
                                                                     bb.SOLS.ptr);
    CKL();
  }
  kb_finish<<<tb, 128, 0, st>>>(B);
  CKL();
  const int nsp = tp * ns;
  if (scores) {
    k_spmm_scores<<<grid_for(n, 8), 256, 0, st>>>(c->x_rowptr.ptr, c->x_cols.ptr, bb.SOLS.ptr,
                                                  bb.SCORES.ptr, (int)n, nsp);
  } else if (n > 0) {
    // the caller wants no scores: the orientation needs the labeled rows' only
    kb_scores_labeled<<<(unsigned)cdiv(n * ND, 256), 256, 0, st>>>(c->x_rowptr.ptr, c->x_cols.ptr, bb.lab.ptr,
                                                                  bb.SOLS.ptr, bb.SCORES.ptr, n, tp, ns);
  }
  CKL();
  if (nlN) {
    const int nch = (int)cdiv(ns, SC_SH), t_per = std::max(1, 65535 / nch);  // grid.y <= 65535
    for (int tb0 = 0; tb0 < T; tb0 += t_per) {
      dim3 g((unsigned)grid_for(nlN, WARPS_PER_BLOCK), (unsigned)(std::min(t_per, T - tb0) * nch));
      kb_orient_leaves<<<g, LEAF_THREADS, 0, st>>>(bb.labt.ptr, bb.SCORES.ptr, n, bb.opart.ptr, nlN, ns, tb0);
      CKL();
    }
    kb_orient_combine<<<T * ns, 256, 0, st>>>(bb.opart.ptr, nlN, B);
    CKL();
  }
  if (scores && n > 0) {
    dim3 g((unsigned)std::min<long long>(grid_for(n, 256), 1024), (unsigned)(T * ns));
    kb_flip<<<g, 256, 0, st>>>(bb.SCORES.ptr, n, T, B);
    CKL();
  }
  if (d > 0) {
    dim3 g((unsigned)cdiv(d, 32), (unsigned)cdiv((long long)T * ns, 32));
    kb_directions_out<<<g, dim3(32, 8), 0, st>>>(bb.SOLS.ptr, bb.OUT.ptr, d, T, tp, ns, B.flip);
    CKL();
  }
  if (tr.on) {
    CK(cudaStreamSynchronize(st));
    tr.mark("batch: projections + orientation");
  }
  // ---- results
  const long long TS = (long long)T * ns;
  if (directions && d > 0)
    CK(cudaMemcpyAsync(directions, bb.OUT.ptr, sizeof(double) * TS * d, cudaMemcpyDeviceToHost, st));
  if (scores && n > 0)
    CK(cudaMemcpyAsync(scores, bb.SCORES.ptr, sizeof(double) * TS * n, cudaMemcpyDeviceToHost, st));
  if (residuals) CK(cudaMemcpyAsync(residuals, B.resid, sizeof(double) * TS, cudaMemcpyDeviceToHost, st));
  std::vector<long long> its(TS), itr(T), fit(T);
  std::vector<unsigned char> cv(TS);
  std::vector<int> stt(T);
  CK(cudaMemcpyAsync(its.data(), B.iters, sizeof(long long) * TS, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(cv.data(), B.conv, TS, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(itr.data(), B.iter, sizeof(long long) * T, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(fit.data(), B.fail_iter, sizeof(long long) * T, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(stt.data(), B.status, sizeof(int) * T, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (long long k = 0; k < TS; ++k) {
    if (iterations) iterations[k] = its[k];
    if (converged) converged[k] = cv[k];
  }
  tr.mark("batch: results d2h");
  for (int t = 0; t < T; ++t) {
    if (n_applies) n_applies[t] = itr[t];
    if (fail_iter) fail_iter[t] = fit[t];
    if (status) status[t] = stt[t] == ST_BREAKDOWN ? FSDA_EBREAKDOWN : (stt[t] == ST_NONFINITE ? FSDA_ENONFINITE : FSDA_OK);
  }
  return FSDA_OK;
}

}  // extern "C++"

static int batch_solve_impl(fsda_ctx* c, int T, const int8_t* labels, double alpha,
                            const double* betas, int ns, double tol, int64_t max_iter,
                            const double* probes, double* directions, double* scores,
                            double* residuals, int64_t* iterations, uint8_t* converged,
                            int64_t* n_applies, int64_t* fail_iter, int* status) {
  if (c->store_bits == 32)
    return batch_solve_t<float>(c, T, labels, alpha, betas, ns, tol, max_iter, probes, directions, scores,
                                residuals, iterations, converged, n_applies, fail_iter, status);
  return batch_solve_t<double>(c, T, labels, alpha, betas, ns, tol, max_iter, probes, directions, scores,
                               residuals, iterations, converged, n_applies, fail_iter, status);
}

int fsda_solve_batch(fsda_ctx* c, int n_tasks, const int8_t* labels, double alpha,
                     const double* betas, int ns, double tol, int64_t max_iter,
                     const double* probes, double* directions, double* scores,
                     double* residuals, int64_t* iterations, uint8_t* converged,
                     int64_t* n_applies, int64_t* fail_iter, int* status) {
  API_BEGIN(c)
  return batch_solve_impl(c, n_tasks, labels, alpha, betas, ns, tol, max_iter, probes, directions,
                          scores, residuals, iterations, converged, n_applies, fail_iter, status);
  API_END
}

}  // extern "C"

#include "fsda_shard.cuh"

// debug: per-CTA phase timestamps of the last k_xt_coop launch (globaltimer ns)
extern "C" int fsda_debug_xt_trace(int on, unsigned long long* out) {
  if (out) return cudaMemcpyFromSymbol(out, g_xt_trace, sizeof(unsigned long long) * 5 * 1024) == cudaSuccess ? 0 : 4;
  return cudaMemcpyToSymbol(g_xt_trace_on, &on, sizeof(int)) == cudaSuccess ? 0 : 4;
}

// ---------------------------------------------------------------- k-NN graph
// graph.py:152-166 knn_graph on the context's X (fsda_upload_x first).
namespace {


}  // namespace

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link
// dependency on libcuda).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

const char* encode_head_map(CUtensorMap* map, const signed char* A, int H, long long rows) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      return "cuTensorMapEncodeTiled unavailable";
    fn = (EncodeTiledFn)p;
  }
  // A: rows x H bytes, row-major; boxes of 128 bytes x 128 rows, 128-byte swizzle
  const cuuint64_t dims[2] = {(cuuint64_t)H, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)H};
  const cuuint32_t box[2] = {(cuuint32_t)HG_BK, (cuuint32_t)HG_BM};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)A, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? nullptr : "cuTensorMapEncodeTiled failed";
}

#define CK_HG(x)                                                    \
  do {                                                              \
    const char* e_ = (x);                                           \
    if (e_) return fail(FSDA_ECUDA, "head-count GEMM: %s", e_);     \
  } while (0)

bool head_gemm_pairs();

// C block (nb16 x n16) of head counts for rows [r0, r0 + nb16): k_head_gemm on
// one persistent CTA per SM (at most one per tile).
void launch_head_gemm(fsda_ctx* c, GraphBufs& g, int r0, int nb16, int n16, int H) {
  const int n_tiles = (n16 + HG_BN - 1) / HG_BN;
  if (!head_gemm_pairs()) {
    const int m_tiles = (nb16 + HG_BM - 1) / HG_BM;
    const int grid = std::max(1, std::min(m_tiles * n_tiles, c->num_sms));
    k_head_gemm<<<grid, HG_THREADS, HG_SMEM, c->stream>>>(g.amap, r0, nb16, n16, H / HG_BK, g.C.ptr,
                                                          (long long)n16, m_tiles, n_tiles);
    CKL();
    return;
  }
  // CTA pairs on 256 x 256 tiles: one cluster of two per TPC
  const int m_tiles = (nb16 + 255) / 256;
  const int grid = 2 * std::max(1, std::min(m_tiles * n_tiles, c->num_sms / 2));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(HG_THREADS);
  cfg.dynamicSmemBytes = HG2_SMEM;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k_head_gemm2, g.amap, r0, nb16, n16, H / HG_BK, g.C.ptr, (long long)n16, m_tiles,
                        n_tiles));
}

// k_head_gemm2 (CTA pairs, cta_group::2) unless FSDA_B200_HEAD_GEMM=1sm
bool head_gemm_pairs() {
  const char* v = std::getenv("FSDA_B200_HEAD_GEMM");  // read per build: tests switch it
  return !(v && std::string(v) == "1sm");
}

// Rows per block of the graph builds: as many as a 16 GiB (at most a quarter
// of free memory) block of 16-bit head counts allows, a multiple of 16.  The
// scans run one warp per row of the block, so small blocks starve the GPU at
// large N (r01's 2^30-element cap gave 715-row blocks at cfg3).
long long graph_block_rows(GraphBufs& g, long long n16) {
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  const double budget = std::min(16.0 * (1LL << 30), 0.25 * (double)free_b);
  long long b = (long long)(budget / (sizeof(HeadCount) * (double)std::max<long long>(n16, 1))) & ~15LL;
  if (const char* f = std::getenv("FSDA_B200_GRAPH_BLOCK_ROWS"))  // tests: many blocks on small inputs
    b = std::atoll(f) & ~15LL;
  b = std::max<long long>(16, std::min<long long>(n16, b));
  g.block_rows = b;
  return b;
}

// Shared by the k-NN and threshold builds: head selection, the int8 head
// matrix, then per row block the head-count GEMM followed by `per_block`.
template <typename F>
int graph_blocks(fsda_ctx* c, GraphBufs& g, F per_block) {
  const long long n = c->n, d = c->d;
  // head = the most frequent columns with at least two entries (ties: lower index)
  std::vector<int> colptr((size_t)d + 1);
  CK(cudaMemcpy(colptr.data(), c->csc_colptr.ptr, sizeof(int) * (d + 1), cudaMemcpyDeviceToHost));
  std::vector<int> order;
  for (long long col = 0; col < d; ++col)
    if (colptr[col + 1] - colptr[col] >= 2) order.push_back((int)col);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return colptr[a + 1] - colptr[a] > colptr[b + 1] - colptr[b];
  });
  // Head width: the int8 GEMM costs 2 N^2 H ops (~4e15/s measured); every
  // tail occurrence costs ~0.4-0.6 ns in the sorted-runs path, ~6 ns once a
  // row's occurrences overflow the shared-memory sort.  Pick the cheapest.
  std::vector<double> sq(order.size() + 1, 0.0);  // sq[h] = sum over ranks >= h of n_c^2
  for (long long h = (long long)order.size() - 1; h >= 0; --h) {
    const double nc = (double)(colptr[order[h] + 1] - colptr[order[h]]);
    sq[h] = sq[h + 1] + nc * nc;
  }
  int nh = 0;
  double best = 1e300;
  for (int cand : {256, 512, 1024, 2048, 4096, 8192, 16384}) {
    const int hc = (int)std::min<size_t>(order.size(), (size_t)cand);
    const double occ = sq[hc], avg = n > 0 ? occ / (double)n : 0.0;
    const double per = avg <= KNN_TAIL_CAP_BIG / 2 ? (avg <= KNN_TAIL_CAP / 2 ? 0.4e-9 : 0.6e-9) : 6e-9;
    const double est = 2.0 * (double)n * (double)n * hc / 4e15 + occ * per;
    if (est < best) {
      best = est;
      nh = hc;
    }
    if ((size_t)cand >= order.size()) break;
  }
  if (const char* f = std::getenv("FSDA_B200_GRAPH_HEAD"))  // experiments: force the head width
    nh = (int)std::min<size_t>(order.size(), (size_t)std::max(0, std::atoi(f)));
  g.tail_avg = n > 0 ? sq[nh] / (double)n : 0.0;
  const int H = nh > 0 ? (nh + HG_BK - 1) / HG_BK * HG_BK : 0;  // GEMM depth padded to 128 (zero columns)
  std::vector<int> head_of((size_t)std::max<long long>(d, 1), -1);
  for (int h = 0; h < nh; ++h) head_of[order[h]] = h;
  g.head_of.ensure(std::max<long long>(d, 1));
  CK(cudaMemcpyAsync(g.head_of.ptr, head_of.data(), sizeof(int) * std::max<long long>(d, 1),
                     cudaMemcpyHostToDevice, c->stream));
  // int8 tensor-core GEMM shapes: rows of A and C's leading dimension padded
  // to 16 (zero rows); blocks of g.block_rows rows (graph_block_rows)
  const long long n16 = (n + 15) & ~15LL;
  const long long B = g.block_rows;
  g.rsize.ensure(n16);
  CK(cudaMemsetAsync(g.rsize.ptr, 0, sizeof(int) * n16, c->stream));
  k_knn_rsize<<<grid_for(n, 256), 256, 0, c->stream>>>(c->x_rowptr.ptr, g.rsize.ptr, (int)n);
  CKL();
  g.tsize.ensure(n16);
  CK(cudaMemsetAsync(g.tsize.ptr, 0, sizeof(int) * n16, c->stream));
  k_knn_tsize<<<grid_for(n, 256), 256, 0, c->stream>>>(c->x_rowptr.ptr, c->x_cols.ptr, g.head_of.ptr,
                                                      g.tsize.ptr, (int)n);
  CKL();
  {
    const int big = (int)(sizeof(int) * KNN_TAIL_CAP_BIG * KNN_REFINE_WARPS_BIG);
    CK(cudaFuncSetAttribute(k_knn_refine<KNN_TAIL_CAP_BIG, KNN_REFINE_WARPS_BIG>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CK(cudaFuncSetAttribute(k_graph_threshold<KNN_TAIL_CAP_BIG, KNN_REFINE_WARPS_BIG>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, big));
  }
  if (H > 0) {
    g.A.ensure(n16 * H);
    g.C.ensure(B * n16);
    CK(cudaMemsetAsync(g.A.ptr, 0, (size_t)n16 * H, c->stream));
    k_knn_head_dense<<<grid_for(n, 256), 256, 0, c->stream>>>(c->x_rowptr.ptr, c->x_cols.ptr, g.head_of.ptr,
                                                             g.A.ptr, (int)n, H);
    CKL();
    CK_HG(encode_head_map(&g.amap, g.A.ptr, H, n16));
    if (!g.gemm_attr) {
      CK(cudaFuncSetAttribute(k_head_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, HG_SMEM));
      CK(cudaFuncSetAttribute(k_head_gemm2, cudaFuncAttributeMaxDynamicSharedMemorySize, HG2_SMEM));
      g.gemm_attr = true;
    }
  }
  for (long long r0 = 0; r0 < n; r0 += B) {
    const long long nb = std::min(B, n - r0);
    if (H > 0) {
      const long long nb16 = (nb + 15) & ~15LL;
      // C (nb16 x n16, row-major) = A_blk . A^T: row b = head counts of row
      // r0 + b against every row
      launch_head_gemm(c, g, (int)r0, (int)nb16, (int)n16, H);
    }
    per_block(r0, nb, n16, H > 0 ? g.C.ptr : nullptr);
  }
  return FSDA_OK;
}

// Sorted, de-duplicated keys[0, m2) -> the context's CSR adjacency.
void graph_csr(fsda_ctx* c, GraphBufs& g, long long m2) {
  const long long n = c->n;
  g.keys2.ensure(std::max<long long>(m2, 1));
  g.count.ensure(1);
  int bits = 1;
  while (bits < 64 && ((unsigned long long)n * (unsigned long long)n) >> bits) ++bits;
  size_t tb_sort = 0, tb_uniq = 0;
  CK(cub::DeviceRadixSort::SortKeys(nullptr, tb_sort, g.keys.ptr, g.keys2.ptr, (int)m2, 0, bits, c->stream));
  CK(cub::DeviceSelect::Unique(nullptr, tb_uniq, g.keys2.ptr, g.keys.ptr, g.count.ptr, (int)m2, c->stream));
  g.temp.ensure(std::max<size_t>(std::max(tb_sort, tb_uniq), 1));
  long long m = 0;
  if (m2 > 0) {
    CK(cub::DeviceRadixSort::SortKeys(g.temp.ptr, tb_sort, g.keys.ptr, g.keys2.ptr, (int)m2, 0, bits, c->stream));
    CK(cub::DeviceSelect::Unique(g.temp.ptr, tb_uniq, g.keys2.ptr, g.keys.ptr, g.count.ptr, (int)m2, c->stream));
    CK(cudaMemcpyAsync(&m, g.count.ptr, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  g.offs.ensure(n + 1);
  g.cols.ensure(std::max<long long>(m, 1));
  k_knn_csr<<<grid_for(std::max(m, n + 1), 256), 256, 0, c->stream>>>(g.keys.ptr, m, n, g.offs.ptr, g.cols.ptr);
  CKL();
  CK(cudaStreamSynchronize(c->stream));
  g.n = n;
  g.nnz = m;
}

extern "C" int fsda_graph_knn(fsda_ctx* c, int32_t k, int64_t* nnz_out) {
  API_BEGIN(c)
  if (!c->has_x) return fail(FSDA_EINVAL, "upload X before building its graph");
  const long long n = c->n;
  if (!(k > 0 && (long long)k < n))
    return fail(FSDA_EINVAL, "k must satisfy 0 < k < n_samples, got k=%d, n=%lld", (int)k, n);
  if (k > KNN_MAX_K) return fail(FSDA_EINVAL, "k=%d above the device limit %d", (int)k, KNN_MAX_K);
  if (n * (long long)k * 2 >= (1LL << 31)) return fail(FSDA_EINVAL, "graph too large (n*k)");
  GraphBufs& g = c->knn;
  Trace tr;
  const long long n16 = (n + 15) & ~15LL;
  const long long B = graph_block_rows(g, n16);
  g.cand.ensure(B * k);
  g.ncand.ensure(B);
  g.nbr.ensure(n * k);
  int rc = graph_blocks(c, g, [&](long long r0, long long nb, long long ldc, const HeadCount* C) {
    if (C) {
      k_knn_scan<<<(unsigned)cdiv(nb, KNN_WARPS), KNN_WARPS * 32, 0, c->stream>>>(
          C, (int)r0, (int)nb, (int)n, (int)ldc, g.rsize.ptr, k, g.cand.ptr, g.ncand.ptr);
      CKL();
    } else {
      CK(cudaMemsetAsync(g.ncand.ptr, 0, sizeof(int) * nb, c->stream));
    }
    if (g.tail_avg <= KNN_TAIL_CAP / 2) {
      k_knn_refine<KNN_TAIL_CAP, KNN_REFINE_WARPS>
          <<<(unsigned)cdiv(nb, KNN_REFINE_WARPS), KNN_REFINE_WARPS * 32,
             sizeof(int) * KNN_TAIL_CAP * KNN_REFINE_WARPS, c->stream>>>(
              C, (int)ldc, (int)r0, (int)nb, (int)n, c->x_rowptr.ptr, c->x_cols.ptr, c->csc_colptr.ptr,
              c->csc_rows.ptr, g.head_of.ptr, k, g.cand.ptr, g.ncand.ptr, g.nbr.ptr);
    } else {
      k_knn_refine<KNN_TAIL_CAP_BIG, KNN_REFINE_WARPS_BIG>
          <<<(unsigned)cdiv(nb, KNN_REFINE_WARPS_BIG), KNN_REFINE_WARPS_BIG * 32,
             sizeof(int) * KNN_TAIL_CAP_BIG * KNN_REFINE_WARPS_BIG, c->stream>>>(
              C, (int)ldc, (int)r0, (int)nb, (int)n, c->x_rowptr.ptr, c->x_cols.ptr, c->csc_colptr.ptr,
              c->csc_rows.ptr, g.head_of.ptr, k, g.cand.ptr, g.ncand.ptr, g.nbr.ptr);
    }
    CKL();
  });
  if (rc) return rc;
  tr.mark("knn: head counts, scan, refine");
  // union symmetrization: both directions, sorted, duplicates dropped
  const long long m2 = 2 * n * k;
  g.keys.ensure(m2);
  k_knn_keys<<<grid_for(n * k, 256), 256, 0, c->stream>>>(g.nbr.ptr, n, k, g.keys.ptr);
  CKL();
  graph_csr(c, g, m2);
  tr.mark("knn: symmetrize");
  if (nnz_out) *nnz_out = g.nnz;
  return FSDA_OK;
  API_END
}

extern "C" int fsda_graph_threshold(fsda_ctx* c, double theta, int64_t* nnz_out) {
  API_BEGIN(c)
  if (!c->has_x) return fail(FSDA_EINVAL, "upload X before building its graph");
  if (!(theta > 0.0 && theta <= 1.0)) return fail(FSDA_EINVAL, "theta must lie in (0, 1], got %g", theta);
  const long long n = c->n;
  GraphBufs& g = c->knn;
  Trace tr;
  g.count.ensure(1);
  unsigned long long cap = (unsigned long long)std::max<long long>(1LL << 20, 16 * n);
  unsigned long long hits = 0;
  graph_block_rows(g, (n + 15) & ~15LL);
  for (int attempt = 0; attempt < 2; ++attempt) {
    g.keys.ensure((long long)cap);
    CK(cudaMemsetAsync(g.count.ptr, 0, sizeof(long long), c->stream));
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(g.count.ptr);
    int rc = graph_blocks(c, g, [&](long long r0, long long nb, long long ldc, const HeadCount* C) {
      if (g.tail_avg <= KNN_TAIL_CAP / 2) {
        k_graph_threshold<KNN_TAIL_CAP, KNN_REFINE_WARPS>
            <<<(unsigned)cdiv(nb, KNN_REFINE_WARPS), KNN_REFINE_WARPS * 32,
               sizeof(int) * KNN_TAIL_CAP * KNN_REFINE_WARPS, c->stream>>>(
                C, (int)ldc, (int)r0, (int)nb, (int)n, g.rsize.ptr, c->x_rowptr.ptr, c->x_cols.ptr,
                c->csc_colptr.ptr, c->csc_rows.ptr, g.head_of.ptr, g.tsize.ptr, theta, g.keys.ptr, cnt, cap);
      } else {
        k_graph_threshold<KNN_TAIL_CAP_BIG, KNN_REFINE_WARPS_BIG>
            <<<(unsigned)cdiv(nb, KNN_REFINE_WARPS_BIG), KNN_REFINE_WARPS_BIG * 32,
               sizeof(int) * KNN_TAIL_CAP_BIG * KNN_REFINE_WARPS_BIG, c->stream>>>(
                C, (int)ldc, (int)r0, (int)nb, (int)n, g.rsize.ptr, c->x_rowptr.ptr, c->x_cols.ptr,
                c->csc_colptr.ptr, c->csc_rows.ptr, g.head_of.ptr, g.tsize.ptr, theta, g.keys.ptr, cnt, cap);
      }
      CKL();
    });
    if (rc) return rc;
    CK(cudaMemcpyAsync(&hits, cnt, sizeof(hits), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (hits <= cap) break;
    cap = hits;  // the first pass counted every hit: rerun with room for all
  }
  if (hits >= (1ULL << 31)) return fail(FSDA_EINVAL, "threshold graph too large (%llu pairs)", hits);
  tr.mark("threshold: head counts, scan");
  graph_csr(c, g, (long long)hits);
  tr.mark("threshold: csr");
  if (nnz_out) *nnz_out = g.nnz;
  return FSDA_OK;
  API_END
}

extern "C" int fsda_head_counts(fsda_ctx* c, int64_t n_rows, int32_t h, const int8_t* a, int64_t r0,
                                int64_t nb, int32_t* counts) {
  API_BEGIN(c)
  if (n_rows <= 0 || h <= 0 || !a || !counts) return fail(FSDA_EINVAL, "fsda_head_counts: empty input");
  if (r0 < 0 || nb <= 0 || r0 + nb > n_rows) return fail(FSDA_EINVAL, "fsda_head_counts: bad row block");
  if (h > 65535) return fail(FSDA_EINVAL, "fsda_head_counts: counts are 16-bit (h <= 65535)");
  if (n_rows * (long long)nb >= (1LL << 31)) return fail(FSDA_EINVAL, "fsda_head_counts: block too large");
  GraphBufs& g = c->knn;
  const long long n16 = (n_rows + 15) & ~15LL, nb16 = (nb + 15) & ~15LL;
  const int H = (h + HG_BK - 1) / HG_BK * HG_BK;
  g.A.ensure(n16 * H);
  g.C.ensure(nb16 * n16);
  CK(cudaMemsetAsync(g.A.ptr, 0, (size_t)n16 * H, c->stream));
  CK(cudaMemcpy2DAsync(g.A.ptr, H, a, h, h, n_rows, cudaMemcpyHostToDevice, c->stream));
  CK_HG(encode_head_map(&g.amap, g.A.ptr, H, n16));
  if (!g.gemm_attr) {
    CK(cudaFuncSetAttribute(k_head_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, HG_SMEM));
    CK(cudaFuncSetAttribute(k_head_gemm2, cudaFuncAttributeMaxDynamicSharedMemorySize, HG2_SMEM));
    g.gemm_attr = true;
  }
  launch_head_gemm(c, g, (int)r0, (int)nb16, (int)n16, H);
  std::vector<HeadCount> h16((size_t)nb * n_rows);
  CK(cudaMemcpy2DAsync(h16.data(), sizeof(HeadCount) * n_rows, g.C.ptr, sizeof(HeadCount) * n16,
                       sizeof(HeadCount) * n_rows, nb, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (size_t k = 0; k < h16.size(); ++k) counts[k] = h16[k];
  return FSDA_OK;
  API_END
}

extern "C" int fsda_graph_fetch(fsda_ctx* c, int64_t* row_offsets, int64_t* col_indices) {
  API_BEGIN(c)
  GraphBufs& g = c->knn;
  if (!g.offs.ptr) return fail(FSDA_EINVAL, "no graph built on this context");
  if (row_offsets)
    CK(cudaMemcpyAsync(row_offsets, g.offs.ptr, sizeof(long long) * (g.n + 1), cudaMemcpyDeviceToHost,
                       c->stream));
  if (col_indices && g.nnz)
    CK(cudaMemcpyAsync(col_indices, g.cols.ptr, sizeof(long long) * g.nnz, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return FSDA_OK;
  API_END
}
