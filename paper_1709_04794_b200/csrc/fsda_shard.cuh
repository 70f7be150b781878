// fsda_shard.cuh — the FSDA sweep row-sharded over several GPUs,
// included by fsda_capi.cu after its helpers.
//
// Rank g holds the contiguous row block [bounds[g], bounds[g+1]) of X (CSR +
// its own CSC) and of L (rows, global columns remapped to the all-gather
// layout), and that block's labels.  The D-length Krylov vectors and the
// scalar recurrences are replicated: every rank runs the identical CG step
// (krylov.py:211-268) on identical data, so no scalar collective is needed.
// Per iteration, the operator w -> X_c^T M X w (sda.py:169-172) is
//
//   K1   y_g = X_g p                              local rows
//   AG   y   = all_gather(y_g)  (maxc per rank)   L reads neighbours' y
//   K2   z_g = M_g y                              local rows of the smoother
//   K3   [q_g | sum z_g] = [X_g^T z_g | sum z_g]  local CSC, D + 1 partials
//   RS   rank r receives slice r of every rank's partial and sums them in
//        rank order (acc = part_0; acc = acc + part_g) — a deterministic
//        reduce-scatter by send/recv
//   AG   q = all_gather(slices)                   replicated D + 1
//   K4   q - mu sum z, p.q, r, r.r, p, shift scalars (replicated)
//
// The summation order is fixed by the partition: a column sum is the
// rank-ordered sum of each rank's canonical column tree over its own rows,
// sum(z), the class sums and the orientation dots likewise; every row sum is
// unchanged.  At world 1 every value equals the single-GPU solve's bit for
// bit; at world > 1 oracle/fsda_oracle.c's partitioned mode reproduces it.
//
// Two exchange backends, one code path:
//   * NCCL (one process per GPU, fsda_shard_init with an ncclUniqueId): the
//     iteration is captured once into a CUDA graph with its NCCL calls and
//     launched max_iter times (guarded kernels idle after the solve
//     finishes, so every rank issues the same collectives);
//   * local ranks (several contexts in one process, the tests): the same
//     phases, exchanges as device-to-device copies ordered by events — no
//     kernel ever waits on another rank's kernel.
// NCCL is loaded at run time (dlopen of libnccl.so.2, the copy torch already
// mapped when present), so the library itself has no link dependency on it.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

namespace {

// ------------------------------------------------------------ NCCL by dlopen
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // torch's copy, if mapped
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
    api.Send = (decltype(api.Send))sym("ncclSend");
    api.Recv = (decltype(api.Recv))sym("ncclRecv");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.Send &&
             api.Recv && api.GroupStart && api.GroupEnd && api.GetErrorString;
    if (!api.ok) api.err = "libnccl.so.2 lacks a needed symbol";
  });
  return api;
}

struct NcclError {
  ncclResult_t r;
  const char* what;
};
#define NK(call)                                             \
  do {                                                       \
    ncclResult_t r_ = (call);                                \
    if (r_ != ncclSuccess) throw NcclError{r_, #call};       \
  } while (0)

// ------------------------------------------------------------------ kernels

// out[k] = part[0][k] + part[1][k] + ... (rank order, acc starts at part 0)
__global__ void k_rank_sum(const double* __restrict__ part, int world, long long m,
                           double* __restrict__ out) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < m;
       k += (long long)gridDim.x * blockDim.x) {
    double acc = part[k];
    for (int g = 1; g < world; ++g) acc = acc + part[(long long)g * m + k];
    out[k] = acc;
  }
}

// class means from the rank-summed class sums (sda.py:126-127)
__global__ void k_shard_class_means(const double* __restrict__ sums, CgScalars* sc, double n1,
                                    double n2) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    sc->class_mean1 = sums[0] / n1;
    sc->class_mean2 = sums[1] / n2;
  }
}

// flip flags from the rank-summed orientation dots (sda.py:280-281)
__global__ void k_shard_flip_flags(const double* __restrict__ dots, ShiftState ss, int ns) {
  for (int s = threadIdx.x; s < ns; s += blockDim.x) ss.flip[s] = dots[s] < 0.0 ? 1 : 0;
}

// ------------------------------------------------------------------ driver

struct ShardRun {
  std::vector<fsda_ctx*> r;  // the ranks this process drives (1 with NCCL)
  int world = 1;
  bool nccl = false;
  long long S = 0;           // slice of the D + 1 reduce-scatter
};

// all_gather: rank g's send(g)[0..count) lands at recv(r) + g * count on every rank r
template <typename FS, typename FR>
void x_allgather(ShardRun& R, FS send, FR recv, size_t count) {
  if (R.nccl) {
    fsda_ctx* c = R.r[0];
    NK(nccl_api().AllGather(send(0), recv(0), count, ncclDouble, (ncclComm_t)c->nccl, c->stream));
    return;
  }
  const int G = R.world;
  for (int g = 0; g < G; ++g) CK(cudaEventRecord(R.r[g]->ev_x, R.r[g]->stream));
  for (int r = 0; r < G; ++r) {
    for (int g = 0; g < G; ++g) {
      CK(cudaStreamWaitEvent(R.r[r]->stream, R.r[g]->ev_x, 0));
      if (count)
        CK(cudaMemcpyAsync(recv(r) + (size_t)g * count, send(g), count * sizeof(double),
                           cudaMemcpyDeviceToDevice, R.r[r]->stream));
    }
  }
  // a rank's send buffer is rewritten only after every rank copied it
  for (int r = 0; r < G; ++r) CK(cudaEventRecord(R.r[r]->ev_y, R.r[r]->stream));
  for (int g = 0; g < G; ++g)
    for (int r = 0; r < G; ++r) CK(cudaStreamWaitEvent(R.r[g]->stream, R.r[r]->ev_y, 0));
}

// all_to_all of S-sized slices: slice r of rank g's send lands at recv(r) + g * S
template <typename FS, typename FR>
void x_alltoall(ShardRun& R, FS send, FR recv, size_t S) {
  const int G = R.world;
  if (R.nccl) {
    fsda_ctx* c = R.r[0];
    const int me = c->rank;
    NcclApi& A = nccl_api();
    NK(A.GroupStart());
    for (int peer = 0; peer < G; ++peer) {
      if (peer == me) continue;
      NK(A.Send(send(0) + (size_t)peer * S, S, ncclDouble, peer, (ncclComm_t)c->nccl, c->stream));
      NK(A.Recv(recv(0) + (size_t)peer * S, S, ncclDouble, peer, (ncclComm_t)c->nccl, c->stream));
    }
    NK(A.GroupEnd());
    CK(cudaMemcpyAsync(recv(0) + (size_t)me * S, send(0) + (size_t)me * S, S * sizeof(double),
                       cudaMemcpyDeviceToDevice, c->stream));
    return;
  }
  for (int g = 0; g < G; ++g) CK(cudaEventRecord(R.r[g]->ev_x, R.r[g]->stream));
  for (int r = 0; r < G; ++r)
    for (int g = 0; g < G; ++g) {
      CK(cudaStreamWaitEvent(R.r[r]->stream, R.r[g]->ev_x, 0));
      CK(cudaMemcpyAsync(recv(r) + (size_t)g * S, send(g) + (size_t)r * S, S * sizeof(double),
                         cudaMemcpyDeviceToDevice, R.r[r]->stream));
    }
  for (int r = 0; r < G; ++r) CK(cudaEventRecord(R.r[r]->ev_y, R.r[r]->stream));
  for (int g = 0; g < G; ++g)
    for (int r = 0; r < G; ++r) CK(cudaStreamWaitEvent(R.r[g]->stream, R.r[r]->ev_y, 0));
}

// q (D + 1, replicated) = rank-ordered sum of every rank's qpart: RS + AG
void x_sum_d1(ShardRun& R) {
  const int G = R.world;
  const long long S = R.S;
  x_alltoall(R, [&](int g) { return (const double*)R.r[g]->qpart.ptr; },
             [&](int r) { return R.r[r]->qrecv.ptr; }, (size_t)S);
  for (fsda_ctx* c : R.r) {
    k_rank_sum<<<grid_for(S, 256), 256, 0, c->stream>>>(c->qrecv.ptr, G, S, c->qown.ptr);
    CKL();
  }
  x_allgather(R, [&](int g) { return (const double*)R.r[g]->qown.ptr; },
              [&](int r) { return R.r[r]->q.ptr; }, (size_t)S);
}

// m replicated scalars = rank-ordered sum of every rank's spart[0..m)
void x_sum_small(ShardRun& R, int m) {
  x_allgather(R, [&](int g) { return (const double*)R.r[g]->spart.ptr; },
              [&](int r) { return R.r[r]->sall.ptr; }, (size_t)m);
  for (fsda_ctx* c : R.r) {
    k_rank_sum<<<1, 256, 0, c->stream>>>(c->sall.ptr, R.world, m, c->spart.ptr + 256);
    CKL();
  }
}

// One iteration on every driven rank (K1 .. K4 + the shift update).
void shard_iteration(ShardRun& R, double alpha, int ns, bool v32) {
  const long long d = R.r[0]->d;
  for (fsda_ctx* c : R.r) {
    Enq e{c};
    enq_xrows(e, c->p.ptr, c->y.ptr, 1, v32);
  }
  const size_t vb = v32 ? sizeof(float) : sizeof(double);
  // y all-gather in units of doubles (fp32 storage: maxc floats, rounded up)
  const size_t cnt = (size_t)((R.r[0]->maxc * vb + 7) / 8);
  x_allgather(R, [&](int g) { return (const double*)R.r[g]->y.ptr; },
              [&](int r) { return R.r[r]->ypad.ptr; }, cnt);
  for (fsda_ctx* c : R.r) {
    Enq e{c};
    enq_smoother(e, alpha, c->ypad.ptr, c->z.ptr, 1, v32);
    // raw local X^T z into qpart[0..D), sum(z_g) into qpart[D] (K3's last CTA)
    enq_xt(e, c->z.ptr, c->qpart.ptr, 0, nullptr, 1, c->part_n.ptr, c->qpart.ptr + d, v32);
  }
  x_sum_d1(R);
  for (fsda_ctx* c : R.r) {
    launch_cg_step(c, ns, d, 0, 0, 1, c->q.ptr + d);
    launch_shift_update(c, ns, d, c->stream, 1);
  }
}

}  // namespace

void shard_release_comm(fsda_ctx* c) {
  if (c->nccl) nccl_api().CommDestroy((ncclComm_t)c->nccl);
  c->nccl = nullptr;
}

extern "C" {

int fsda_nccl_unique_id(uint8_t* out) {
  if (!out) return fail(FSDA_EINVAL, "null output");
  NcclApi& A = nccl_api();
  if (!A.ok) return fail(FSDA_ECUDA, "%s", A.err.c_str());
  ncclUniqueId id;
  ncclResult_t r = A.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(FSDA_ECUDA, "ncclGetUniqueId: %s", A.GetErrorString(r));
  memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return FSDA_OK;
}

int fsda_shard_init(fsda_ctx* c, int world, int rank, const int64_t* row_bounds,
                    const uint8_t* nccl_id) {
  API_BEGIN(c)
  if (world < 1 || rank < 0 || rank >= world) return fail(FSDA_EINVAL, "bad world / rank");
  if (!row_bounds) return fail(FSDA_EINVAL, "row_bounds is null");
  long long maxc = 0;
  for (int g = 0; g < world; ++g) {
    if (row_bounds[g + 1] < row_bounds[g]) return fail(FSDA_EINVAL, "row_bounds must be non-decreasing");
    maxc = std::max<long long>(maxc, row_bounds[g + 1] - row_bounds[g]);
  }
  if (!c->has_x || c->n != row_bounds[rank + 1] - row_bounds[rank])
    return fail(FSDA_EINVAL, "upload this rank's X rows before fsda_shard_init");
  if (c->nccl) {
    nccl_api().CommDestroy((ncclComm_t)c->nccl);
    c->nccl = nullptr;
  }
  c->world = world;
  c->rank = rank;
  c->maxc = (maxc + 1) & ~1LL;  // even: an fp32 slot is a whole number of doubles
  c->shard_n_global = row_bounds[world];
  if (nccl_id) {
    NcclApi& A = nccl_api();
    if (!A.ok) return fail(FSDA_ECUDA, "%s", A.err.c_str());
    ncclUniqueId id;
    memcpy(id.internal, nccl_id, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t comm;
    ncclResult_t r = A.CommInitRank(&comm, world, id, rank);
    if (r != ncclSuccess) return fail(FSDA_ECUDA, "ncclCommInitRank: %s", A.GetErrorString(r));
    c->nccl = comm;
  }
  if (!c->ev_x) CK(cudaEventCreateWithFlags(&c->ev_x, cudaEventDisableTiming));
  if (!c->ev_y) CK(cudaEventCreateWithFlags(&c->ev_y, cudaEventDisableTiming));
  c->invalidate_graph();
  return FSDA_OK;
  API_END
}

// One row-sharded FSDA sweep (sda.py:293-320).  ctxs: the ranks this process
// drives — one context with an NCCL communicator, or all `world` contexts of
// a local group (same process).  probe (D), betas replicated; n1, n2: global
// class counts.  Outputs: directions (n_shifts x D, replicated), scores of
// every driven rank's rows (n_shifts x rows, rank blocks side by side per
// shift: scores[s * rows_total + local offset]), residuals, iterations,
// converged, n_applies, fail_iter.
int fsda_solve_sharded(fsda_ctx** ctxs, int n_ctx, double alpha, const double* betas, int ns,
                       double tol, int64_t max_iter, const double* probe, int64_t n1, int64_t n2,
                       double* directions, double* scores, double* residuals, int64_t* iterations,
                       uint8_t* converged, int64_t* n_applies, int64_t* fail_iter) {
  if (!ctxs || n_ctx < 1) return fail(FSDA_EINVAL, "no contexts");
  ShardRun R;
  for (int k = 0; k < n_ctx; ++k) {
    if (!ctxs[k]) return fail(FSDA_EINVAL, "null context");
    R.r.push_back(ctxs[k]);
  }
  fsda_ctx* c0 = ctxs[0];
  R.world = c0->world;
  R.nccl = c0->nccl != nullptr;
  if (R.nccl ? n_ctx != 1 : n_ctx != R.world)
    return fail(FSDA_EINVAL, "pass the one NCCL rank of this process, or all %d local ranks", R.world);
  for (int k = 0; k < n_ctx; ++k) {
    fsda_ctx* c = ctxs[k];
    if (c->world != R.world || (!R.nccl && c->rank != k))
      return fail(FSDA_EINVAL, "contexts must be ranks 0..world-1 of one fsda_shard_init group");
    if (!c->has_x || !c->has_l || !c->has_labels) return fail(FSDA_EINVAL, "rank %d: upload X, L and labels", k);
    if (c->d != c0->d) return fail(FSDA_EINVAL, "ranks disagree on D");
    if (c->n_global != c->world * c->maxc || c->row_base != (long long)c->rank * c->maxc)
      return fail(FSDA_EINVAL, "rank %d: L must be uploaded in the all-gather layout (n_global = world * maxc, "
                               "row_base = rank * maxc, columns remapped)", k);
  }
  if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(FSDA_EINVAL, "alpha must lie in [0, 1], got %g", alpha);
  if (n1 <= 0 || n2 <= 0) return fail(FSDA_EINVAL, "both classes need at least one labeled sample");
  if (ns <= 0 || ns > FSDA_MAX_SHIFTS) return fail(FSDA_EINVAL, "bad shift count");
  if (ns > 256) return fail(FSDA_EINVAL, "the sharded solve takes at most 256 shifts");
  for (int s = 0; s < ns; ++s) {
    if (!std::isfinite(betas[s])) return fail(FSDA_EINVAL, "shifts must be finite");
    if (s == 0 && betas[s] < 0) return fail(FSDA_EINVAL, "shifts must be non-negative");
    if (s > 0 && !(betas[s] > betas[s - 1])) return fail(FSDA_EINVAL, "shifts must be strictly ascending");
  }
  if (!(tol > 0)) return fail(FSDA_EINVAL, "tol must be positive");
  const long long d = c0->d;
  const double ell = (double)(n1 + n2);
  std::vector<std::unique_lock<std::mutex>> locks;
  for (fsda_ctx* c : R.r) locks.emplace_back(c->mu);
  try {
    CK(cudaSetDevice(c0->device));
    R.S = cdiv(d + 1, R.world);
    for (fsda_ctx* c : R.r) {
      c->solve_kind = 0;
      c->solve_abs_tol = 0;
      upload_solve_params(c, betas, ns, probe, max_iter);
      c->ypad.ensure((size_t)R.world * std::max<long long>(c->maxc, 1));
      c->y.ensure((size_t)std::max<long long>(c->maxc, 1));  // the all-gather reads a whole slot
      c->qpart.ensure((size_t)R.world * R.S);
      c->qrecv.ensure((size_t)R.world * R.S);
      c->qown.ensure((size_t)R.S);
      c->q.ensure((size_t)R.world * R.S);
      c->spart.ensure(512);
      c->sall.ensure((size_t)R.world * 256);
      CK(cudaMemsetAsync(c->qpart.ptr, 0, sizeof(double) * R.world * R.S, c->stream));
    }
    const bool v32 = f32(c0);
    ShiftState ss0 = c0->shifts();
    (void)ss0;
    Trace tr;
    auto sync_mark = [&](const char* what) {
      if (!tr.on) return;
      for (fsda_ctx* c : R.r) CK(cudaStreamSynchronize(c->stream));
      tr.mark(what);
    };
    sync_mark("shard: params");
    // ---- setup: mu, rhs, CG init (sda.py:297-301, krylov.py:185-208)
    for (fsda_ctx* c : R.r) {
      ShiftState ss = c->shifts();
      k_solve_reset<<<1, 256, 0, c->stream>>>(c->sc, ss, ns, max_iter, tol, 0);
      CKL();
      k_indicator<<<grid_for(c->n, 256), 256, 0, c->stream>>>(c->labels.ptr, c->ind.ptr, (int)c->n);
      CKL();
      Enq e{c};
      enq_xt(e, c->ind.ptr, c->qpart.ptr, 0, nullptr, 0, nullptr);
      CK(cudaMemsetAsync(c->qpart.ptr + d, 0, sizeof(double), c->stream));
    }
    x_sum_d1(R);
    for (fsda_ctx* c : R.r) {  // mu = (sum_g X_g^T 1_l) / ell
      k_center<<<grid_for(d, 256), 256, 0, c->stream>>>(nullptr, c->q.ptr, d, ell);
      CKL();
      CK(cudaMemcpyAsync(c->mu_v.ptr, c->q.ptr, sizeof(double) * d, cudaMemcpyDeviceToDevice, c->stream));
      Enq e{c};
      enq_xrows(e, c->probe.ptr, c->t.ptr, 0);  // t = X_g r
      const long long nl = n_leaves(c->n);
      k_class_sums<<<grid_for(std::max(nl, 1LL), WARPS_PER_BLOCK), LEAF_THREADS, 0, c->stream>>>(
          c->t.ptr, c->labels.ptr, c->n, c->part_n.ptr, nl, c->sc, 1.0, 1.0);
      CKL();
      CK(cudaMemcpyAsync(c->spart.ptr, &c->sc->class_mean1, 2 * sizeof(double), cudaMemcpyDeviceToDevice,
                         c->stream));
    }
    x_sum_small(R, 2);
    for (fsda_ctx* c : R.r) {
      k_shard_class_means<<<1, 32, 0, c->stream>>>(c->spart.ptr + 256, c->sc, (double)n1, (double)n2);
      CKL();
      const long long nl = n_leaves(c->n);
      k_apply_w<<<grid_for(std::max(nl, 1LL), WARPS_PER_BLOCK), LEAF_THREADS, 0, c->stream>>>(
          c->labels.ptr, c->wv.ptr, c->n, c->part_n.ptr, nl, c->sc);
      CKL();
      Enq e{c};
      enq_xt(e, c->wv.ptr, c->qpart.ptr, 0, nullptr, 0, nullptr);
      CK(cudaMemcpyAsync(c->qpart.ptr + d, &c->sc->sum_z, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    }
    x_sum_d1(R);
    for (fsda_ctx* c : R.r) {  // b = X^T w - mu sum(w)
      k_center<<<grid_for(d, 256), 256, 0, c->stream>>>(c->mu_v.ptr, c->q.ptr, d, 1.0);
      CKL();
      CK(cudaMemcpyAsync(c->b.ptr, c->q.ptr, sizeof(double) * d, cudaMemcpyDeviceToDevice, c->stream));
      launch_cg_init(c, c->b.ptr, d, ns);
    }
    // ---- the iterations: every rank issues max_iter of them (identical
    // collectives on all ranks); the kernels idle once the solve finished
    sync_mark("shard: setup");
    if (R.nccl) {
      fsda_ctx* c = c0;
      char key[160];
      snprintf(key, sizeof(key), "shard|%a|%d|%lld|%a|%llu|%d|%d|%d", alpha, ns, (long long)max_iter, tol,
               g_alloc_gen.load(), c->su_mode, c->nslots, c->store_bits);
      if (!(c->exec && c->graph_key == key)) {
        c->invalidate_graph();
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        try {
          shard_iteration(R, alpha, ns, v32);
        } catch (...) {
          cudaGraph_t junk;
          cudaStreamEndCapture(c->stream, &junk);
          if (junk) cudaGraphDestroy(junk);
          throw;
        }
        CK(cudaStreamEndCapture(c->stream, &g));
        c->graph = g;
        CK(cudaGraphInstantiate(&c->exec, g, 0));
        c->graph_key = key;
      }
      for (long long it = 0; it < max_iter; ++it) CK(cudaGraphLaunch(c->exec, c->stream));
    } else {
      for (long long it = 0; it < max_iter; ++it) shard_iteration(R, alpha, ns, v32);
    }
    sync_mark("shard: iterations");
    // ---- tail: directions, residuals, local projections, orientation
    for (fsda_ctx* c : R.r) {
      ShiftState ss = c->shifts();
      launch_final_shift(c, ns, d);
      k_cg_finish<<<1, 32, 0, c->stream>>>(c->sc, ss, ns);
      CKL();
      k_transpose_sols<<<grid_for(d * ns, 256), 256, 0, c->stream>>>(c->sols.ptr, c->wT.ptr, d, ns);
      CKL();
      const long long n = c->n, nlN = n_leaves(n);
      if (n > 0) {
        k_spmm_scores<<<grid_for(n, 8), 256, 0, c->stream>>>(c->x_rowptr.ptr, c->x_cols.ptr, c->wT.ptr,
                                                             c->scores.ptr, (int)n, ns);
        CKL();
        dim3 g(grid_for(nlN, WARPS_PER_BLOCK), ns);
        k_orient<<<g, LEAF_THREADS, 0, c->stream>>>(c->labels.ptr, c->scores.ptr, n, c->part_o.ptr, nlN);
        CKL();
        k_orient_final<<<ns, 256, 0, c->stream>>>(c->part_o.ptr, nlN, ss, c->spart.ptr);
        CKL();
      } else {
        CK(cudaMemsetAsync(c->spart.ptr, 0, sizeof(double) * ns, c->stream));
      }
    }
    x_sum_small(R, ns);
    long long rows_total = 0;
    for (fsda_ctx* c : R.r) rows_total += c->n;
    long long off = 0;
    for (fsda_ctx* c : R.r) {
      ShiftState ss = c->shifts();
      k_shard_flip_flags<<<1, 256, 0, c->stream>>>(c->spart.ptr + 256, ss, ns);
      CKL();
      dim3 g((unsigned)std::min<long long>(grid_for(std::max(c->n, d), 256), 1024), ns);
      k_flip<<<g, 256, 0, c->stream>>>(c->scores.ptr, c->sols.ptr, c->n, d, ss);
      CKL();
      if (scores && c->n > 0)
        CK(cudaMemcpy2DAsync(scores + off, sizeof(double) * rows_total, c->scores.ptr, sizeof(double) * c->n,
                             sizeof(double) * c->n, ns, cudaMemcpyDeviceToHost, c->stream));
      off += c->n;
    }
    for (fsda_ctx* c : R.r) CK(cudaStreamSynchronize(c->stream));
    tr.mark("shard: tail");
    // results: replicated state, read from the first driven rank
    SolveOut o{directions, nullptr, residuals, iterations, converged, n_applies, fail_iter};
    locks.clear();
    return read_results(c0, ns, o, nullptr);
  } catch (CudaError& e) {
    return fail(FSDA_ECUDA, "CUDA error %s at %s (line %d)", cudaGetErrorString(e.err), e.what, e.line);
  } catch (NcclError& e) {
    return fail(FSDA_ECUDA, "NCCL error %s at %s", nccl_api().GetErrorString(e.r), e.what);
  }
}

}  // extern "C"
