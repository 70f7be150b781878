// graph_gemm.cuh — the k-NN / threshold graph's head-count GEMM on the
// 5th-generation tensor cores, hand-written for sm_100a (
// reference: sdakit/graph.py:79-111, where each row block's X_blk X^T is a
// scipy sparse product).
//
//   C[b][j] = sum_h A[r0 + b][h] * A[j][h]      b < nb, j < n16
//
// A is the N16 x H 0/1 int8 head matrix (row-major: K-major for both MMA
// operands), C the nb16 x n16 block of exact head counts, 16-bit (counts are
// at most H <= 16384), read by k_knn_scan / k_knn_refine / k_graph_threshold.
// Integer arithmetic: the counts are exact and equal to any other GEMM's.
//
// The product path is k_head_gemm2: clusters of two CTAs (the two SMs of a
// TPC) on 256 x 256 tiles, tcgen05.mma.cta_group::2 (see its comment below);
// 4.06 int8 POPS per cfg2 block, 87 % of the imma pipe (profiles/
// r02_graph_gemm.md).  k_head_gemm, the single-CTA form below, is kept as the
// FSDA_B200_HEAD_GEMM=1sm alternative; its structure is the same:
//
// One persistent CTA per SM, 192 threads, warp-specialised:
//   warp 0     TMA producer: per K step (128 bytes of H) one 128 x 128 tile of
//              A_blk and two 128 x 128 tiles of A (256 rows of j) land in a
//              4-stage shared-memory ring (128-byte swizzle, mbarrier
//              complete_tx);
//   warp 1     MMA issuer: one thread issues tcgen05.mma.kind::i8 (M 128,
//              N 256, K 32; four per K step) into a TMEM accumulator;
//              tcgen05.commit frees the ring slot and, after the last K step,
//              hands the accumulator to the epilogue;
//   warps 2-5  epilogue: tcgen05.ld of the 128 x 256 int32 accumulator (each
//              warp its 32-lane quarter), packed to 16-bit counts and stored
//              straight to C, 8 per 16-byte store.
// TMEM holds two accumulators (2 x 256 of its 512 columns), so the epilogue
// of tile t overlaps the MMAs of tile t+1.  Tiles run m-fastest over the
// grid: the A_blk tiles stay L2-resident and the CTAs in flight share the
// same few j tiles.
#pragma once

#include <cuda.h>

namespace fsda {

constexpr int HG_BM = 128;          // rows of A_blk per tile (TMEM lanes)
constexpr int HG_BN = 256;          // rows of A (j) per tile (TMEM columns)
constexpr int HG_BK = 128;          // bytes of H per pipeline stage (one 128-byte swizzle atom)
constexpr int HG_STAGES = 4;
constexpr int HG_THREADS = 192;
constexpr int HG_A_BYTES = HG_BM * HG_BK;                 // 16 KB
constexpr int HG_B_BYTES = HG_BN * HG_BK;                 // 32 KB
constexpr int HG_STAGE_BYTES = HG_A_BYTES + HG_B_BYTES;   // 48 KB
constexpr int HG_SMEM = HG_STAGES * HG_STAGE_BYTES + 1024 + 256;  // + alignment + barriers

__device__ __forceinline__ unsigned hg_smem(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void hg_bar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void hg_bar_wait(unsigned bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.b32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void hg_bar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void hg_bar_expect(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

// 2-D tiled TMA load (box {128 bytes of H, 128 rows}) completing on bar.
__device__ __forceinline__ void hg_tma_load(unsigned dst, const CUtensorMap* map, int x, int y, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}

// Shared-memory matrix descriptor (tcgen05 "version 1"): K-major operand in
// the 128-byte swizzle layout TMA writes — rows of 128 bytes, 8-row groups
// 1024 bytes apart (SBO), leading offset unused for swizzled K-major (1).
__device__ __forceinline__ unsigned long long hg_desc(unsigned saddr) {
  unsigned long long d = 0;
  d |= (unsigned long long)((saddr & 0x3FFFF) >> 4);       // start address
  d |= (unsigned long long)1 << 16;                        // LBO (unused)
  d |= (unsigned long long)(1024 >> 4) << 32;              // SBO
  d |= (unsigned long long)1 << 46;                        // descriptor version (sm_100)
  d |= (unsigned long long)2 << 61;                        // SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::i8: D s32, A and B unsigned 8-bit, both
// K-major, N = 256, M = 128.
constexpr unsigned HG_IDESC = (2u << 4) | (0u << 7) | (0u << 10) | ((unsigned)(HG_BN >> 3) << 17) |
                              ((unsigned)(HG_BM >> 4) << 24);

__device__ __forceinline__ void hg_mma(unsigned tmem_d, unsigned long long adesc, unsigned long long bdesc,
                                       int accumulate) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(HG_IDESC), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void hg_commit(unsigned bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

__device__ __forceinline__ void hg_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void hg_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// 32 consecutive accumulator columns of this thread's TMEM lane.
__device__ __forceinline__ void hg_tmem_ld32(unsigned taddr, int (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// C (nb16 x ldc, row-major int32) = A[r0 .. r0 + nb16) . A[0 .. n16)^T over
// H = kb * 128 columns.  m_tiles = ceil(nb16 / 128), n_tiles = ceil(n16 / 256).
__global__ void __launch_bounds__(HG_THREADS, 1) k_head_gemm(const __grid_constant__ CUtensorMap amap, int r0,
                                                           int nb16, int n16, int kb, HeadCount* __restrict__ C,
                                                           long long ldc, int m_tiles, int n_tiles) {
  extern __shared__ __align__(1024) unsigned char hg_raw[];
  // 1024-byte aligned ring (the swizzle pattern is anchored to 1024 B)
  unsigned char* ring = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<size_t>(hg_raw) + 1023) & ~(size_t)1023);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(ring + HG_STAGES * HG_STAGE_BYTES);
  // bars: full[4], empty[4], tmem_full[2], tmem_empty[2]; then the TMEM base
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(bars + 2 * HG_STAGES + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned full0 = hg_smem(bars), empty0 = hg_smem(bars + HG_STAGES);
  const unsigned tfull0 = hg_smem(bars + 2 * HG_STAGES), tempty0 = hg_smem(bars + 2 * HG_STAGES + 2);
  if (threadIdx.x == 0) {
    for (int s = 0; s < HG_STAGES; ++s) {
      hg_bar_init(full0 + 8 * s, 1);
      hg_bar_init(empty0 + 8 * s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      hg_bar_init(tfull0 + 8 * s, 1);
      hg_bar_init(tempty0 + 8 * s, 4);   // the four epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&amap)) : "memory");
  }
  if (warp == 1) {  // TMEM: two 256-column accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(hg_smem(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  hg_fence_before();
  __syncthreads();
  hg_fence_after();
  const unsigned tmem = *tmem_slot;
  const int tiles = m_tiles * n_tiles;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      int stage = 0;
      unsigned phase = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int m = t % m_tiles, n = t / m_tiles;
        for (int k = 0; k < kb; ++k) {
          hg_bar_wait(empty0 + 8 * stage, phase ^ 1u);
          const unsigned sa = hg_smem(ring + stage * HG_STAGE_BYTES), sb = sa + HG_A_BYTES;
          const unsigned fb = full0 + 8 * stage;
          hg_bar_expect(fb, HG_STAGE_BYTES);
          hg_tma_load(sa, &amap, k * HG_BK, r0 + m * HG_BM, fb);
          hg_tma_load(sb, &amap, k * HG_BK, n * HG_BN, fb);
          hg_tma_load(sb + HG_A_BYTES, &amap, k * HG_BK, n * HG_BN + HG_BM, fb);
          if (++stage == HG_STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      int stage = 0;
      unsigned phase = 0;
      int local = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++local) {
        const int acc = local & 1;
        hg_bar_wait(tempty0 + 8 * acc, ((local >> 1) & 1) ^ 1u);
        hg_fence_after();
        const unsigned d = tmem + (unsigned)(acc * HG_BN);
        for (int k = 0; k < kb; ++k) {
          hg_bar_wait(full0 + 8 * stage, phase);
          hg_fence_after();
          const unsigned sa = hg_smem(ring + stage * HG_STAGE_BYTES), sb = sa + HG_A_BYTES;
          const unsigned long long ad = hg_desc(sa), bd = hg_desc(sb);
#pragma unroll
          for (int kk = 0; kk < HG_BK / 32; ++kk)  // K = 32 bytes per MMA: +2 in the 16-byte address field
            hg_mma(d, ad + 2ull * kk, bd + 2ull * kk, (k | kk) != 0);
          hg_commit(empty0 + 8 * stage);      // the slot is free once these MMAs have read it
          if (k == kb - 1) hg_commit(tfull0 + 8 * acc);
          if (++stage == HG_STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else {
    // ---- epilogue: warp w owns TMEM lanes 32 (w % 4) .. + 31
    const int q = warp & 3;
    int local = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++local) {
      const int m = t % m_tiles, n = t / m_tiles;
      const int acc = local & 1;
      hg_bar_wait(tfull0 + 8 * acc, (local >> 1) & 1);
      hg_fence_after();
      const int b = m * HG_BM + q * 32 + lane;  // row of the C block
      HeadCount* crow = C + (long long)b * ldc;
#pragma unroll 1
      for (int c0 = 0; c0 < HG_BN; c0 += 32) {
        int v[32];
        hg_tmem_ld32(tmem + ((unsigned)(q * 32) << 16) + (unsigned)(acc * HG_BN + c0), v);
        const int j0 = n * HG_BN + c0;
        if (b < nb16) {
#pragma unroll
          for (int u = 0; u < 4; ++u)  // 8 counts (16 bits each) per 16-byte store
            if (j0 + 8 * u < n16) {
              const int* w = v + 8 * u;
              *reinterpret_cast<uint4*>(crow + j0 + 8 * u) =
                  make_uint4(__byte_perm(w[0], w[1], 0x5410), __byte_perm(w[2], w[3], 0x5410),
                             __byte_perm(w[4], w[5], 0x5410), __byte_perm(w[6], w[7], 0x5410));
            }
        }
      }
      hg_fence_before();
      __syncwarp();
      if (lane == 0) hg_bar_arrive(tempty0 + 8 * acc);
    }
  }
  hg_fence_before();
  __syncthreads();
  hg_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// ---------------------------------------------------------------------------
// The CTA-pair form (cta_group::2): a cluster of two CTAs on the two SMs of a
// TPC computes a 256 x 256 tile.  CTA r loads rows [128 r, 128 r + 128) of the
// tile's A_blk rows and of its A (j) rows — 32 KB per K step instead of the
// 48 KB a 1-SM 128 x 256 tile needs — and the leader's single thread issues
// tcgen05.mma.cta_group::2.kind::i8 (M 256, N 256): each SM's tensor core
// reads its own A half and both B halves, and writes its 128 x 256 quarter of
// the accumulator into its own TMEM.  Both CTAs' TMA loads complete on the
// leader's ring barrier (cta_group::2 TMA), the MMA commits multicast to both
// CTAs' slot and accumulator barriers, and the epilogue warps of both CTAs
// release an accumulator through the leader's barrier (8 arrivals).
constexpr int HG2_STAGES = 6;
constexpr int HG2_HALF = HG_BM * HG_BK;            // 16 KB: one 128-row half
constexpr int HG2_STAGE_BYTES = 2 * HG2_HALF;       // A half + B half per CTA
constexpr int HG2_SMEM = HG2_STAGES * HG2_STAGE_BYTES + 1024 + 256;
constexpr unsigned HG2_IDESC = (2u << 4) | ((unsigned)(HG_BN >> 3) << 17) | ((unsigned)(256 >> 4) << 24);
constexpr unsigned HG_PEER_MASK = 0xFEFFFFFFu;      // shared::cluster address of the pair's leader

__device__ __forceinline__ unsigned hg_cta_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void hg_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void hg_tma_load2(unsigned dst, const CUtensorMap* map, int x, int y, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(bar & HG_PEER_MASK)
      : "memory");
}

__device__ __forceinline__ void hg_mma2(unsigned tmem_d, unsigned long long adesc, unsigned long long bdesc,
                                        int accumulate) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p; }" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(HG2_IDESC), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void hg_commit2(unsigned bar) {
  asm volatile(
      "{ .reg .b16 m; mov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m; }" ::"r"(bar)
      : "memory");
}

// arrive on the barrier at the same offset in the pair's leader CTA
__device__ __forceinline__ void hg_arrive_leader(unsigned bar) {
  unsigned remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(bar));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

__global__ void __launch_bounds__(HG_THREADS, 1) k_head_gemm2(const __grid_constant__ CUtensorMap amap, int r0,
                                                            int nb16, int n16, int kb, HeadCount* __restrict__ C,
                                                            long long ldc, int m_tiles, int n_tiles) {
  extern __shared__ __align__(1024) unsigned char hg_raw[];
  unsigned char* ring = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<size_t>(hg_raw) + 1023) & ~(size_t)1023);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(ring + HG2_STAGES * HG2_STAGE_BYTES);
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(bars + 2 * HG2_STAGES + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned rank = hg_cta_rank();
  const unsigned full0 = hg_smem(bars), empty0 = hg_smem(bars + HG2_STAGES);
  const unsigned tfull0 = hg_smem(bars + 2 * HG2_STAGES), tempty0 = hg_smem(bars + 2 * HG2_STAGES + 2);
  if (threadIdx.x == 0) {
    for (int s = 0; s < HG2_STAGES; ++s) {
      hg_bar_init(full0 + 8 * s, 1);     // the leader's producer (+ both CTAs' bytes)
      hg_bar_init(empty0 + 8 * s, 1);    // the MMA's multicast commit
    }
    for (int s = 0; s < 2; ++s) {
      hg_bar_init(tfull0 + 8 * s, 1);
      hg_bar_init(tempty0 + 8 * s, 8);   // four epilogue warps in each CTA (leader's copy used)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&amap)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(hg_smem(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  hg_fence_before();
  hg_cluster_sync();
  hg_fence_after();
  const unsigned tmem = *tmem_slot;
  const int tiles = m_tiles * n_tiles;
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs: their halves)
      int stage = 0;
      unsigned phase = 0;
      for (int t = cluster; t < tiles; t += nclusters) {
        const int m = t % m_tiles, n = t / m_tiles;
        for (int k = 0; k < kb; ++k) {
          hg_bar_wait(empty0 + 8 * stage, phase ^ 1u);
          const unsigned sa = hg_smem(ring + stage * HG2_STAGE_BYTES), sb = sa + HG2_HALF;
          const unsigned fb = full0 + 8 * stage;
          if (rank == 0) hg_bar_expect(fb, 2 * HG2_STAGE_BYTES);
          hg_tma_load2(sa, &amap, k * HG_BK, r0 + m * 256 + (int)rank * HG_BM, fb);
          hg_tma_load2(sb, &amap, k * HG_BK, n * HG_BN + (int)rank * HG_BM, fb);
          if (++stage == HG2_STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ---- MMA issuer (the pair's leader)
      int stage = 0;
      unsigned phase = 0;
      int local = 0;
      for (int t = cluster; t < tiles; t += nclusters, ++local) {
        const int acc = local & 1;
        hg_bar_wait(tempty0 + 8 * acc, ((local >> 1) & 1) ^ 1u);
        hg_fence_after();
        const unsigned d = tmem + (unsigned)(acc * HG_BN);
        for (int k = 0; k < kb; ++k) {
          hg_bar_wait(full0 + 8 * stage, phase);
          hg_fence_after();
          const unsigned sa = hg_smem(ring + stage * HG2_STAGE_BYTES), sb = sa + HG2_HALF;
          const unsigned long long ad = hg_desc(sa), bd = hg_desc(sb);
#pragma unroll
          for (int kk = 0; kk < HG_BK / 32; ++kk) hg_mma2(d, ad + 2ull * kk, bd + 2ull * kk, (k | kk) != 0);
          hg_commit2(empty0 + 8 * stage);
          if (k == kb - 1) hg_commit2(tfull0 + 8 * acc);
          if (++stage == HG2_STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else {
    // ---- epilogue: this CTA's 128 rows of the tile, all 256 columns
    const int q = warp & 3;
    int local = 0;
    for (int t = cluster; t < tiles; t += nclusters, ++local) {
      const int m = t % m_tiles, n = t / m_tiles;
      const int acc = local & 1;
      hg_bar_wait(tfull0 + 8 * acc, (local >> 1) & 1);
      hg_fence_after();
      const int b = m * 256 + (int)rank * HG_BM + q * 32 + lane;
      HeadCount* crow = C + (long long)b * ldc;
#pragma unroll 1
      for (int c0 = 0; c0 < HG_BN; c0 += 32) {
        int v[32];
        hg_tmem_ld32(tmem + ((unsigned)(q * 32) << 16) + (unsigned)(acc * HG_BN + c0), v);
        const int j0 = n * HG_BN + c0;
        if (b < nb16) {
#pragma unroll
          for (int u = 0; u < 4; ++u)  // 8 counts (16 bits each) per 16-byte store
            if (j0 + 8 * u < n16) {
              const int* w = v + 8 * u;
              *reinterpret_cast<uint4*>(crow + j0 + 8 * u) =
                  make_uint4(__byte_perm(w[0], w[1], 0x5410), __byte_perm(w[2], w[3], 0x5410),
                             __byte_perm(w[4], w[5], 0x5410), __byte_perm(w[6], w[7], 0x5410));
            }
        }
      }
      hg_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) hg_bar_arrive(tempty0 + 8 * acc);
        else hg_arrive_leader(tempty0 + 8 * acc);
      }
    }
  }
  hg_fence_before();
  hg_cluster_sync();
  hg_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

}  // namespace fsda
