// Microbenchmark: random 8-byte gathers from a table spread over the shared
// memory of a thread-block cluster (distributed shared memory), against the
// same gathers from an L2-resident global table.  Decides whether a gather
// source of a few MB (y, z, the tail of p) is cheaper to serve from cluster
// DSMEM than from L2.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/dsmem_bench.bin tools/dsmem_bench.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

namespace cg = cooperative_groups;

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);                   \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

// Every CTA of a cluster holds `slice` doubles; index i lives in rank
// i / slice at offset i % slice.  Threads stream indices (coalesced) and sum
// the gathered values, U loads in flight.
template <int U>
__global__ void k_dsmem(const int* __restrict__ idx, long long n, const double* __restrict__ tab,
                        int slice, double* out) {
  extern __shared__ double st[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  for (int k = threadIdx.x; k < slice; k += blockDim.x) st[k] = tab[(long long)rank * slice + k];
  cl.sync();
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (long long i = tid; i + (U - 1) * stride < n; i += U * stride) {
    int ix[U];
#pragma unroll
    for (int u = 0; u < U; ++u) ix[u] = __ldg(idx + i + u * stride);
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = ix[u] / slice, o = ix[u] - r * slice;
      const double* p = cl.map_shared_rank(st, r);
      v[u] = p[o];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  cl.sync();  // keep every slice alive until all remote reads are done
  if (acc == 12345.0) out[0] = acc;
}

template <int U>
__global__ void k_l2(const int* __restrict__ idx, long long n, const double* __restrict__ tab,
                     double* out) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (long long i = tid; i + (U - 1) * stride < n; i += U * stride) {
    int ix[U];
#pragma unroll
    for (int u = 0; u < U; ++u) ix[u] = __ldg(idx + i + u * stride);
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(tab + ix[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 12345.0) out[0] = acc;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long long n = 1LL << 26;  // 67M gathers
  std::mt19937_64 rng(1);
  int* didx;
  double *dtab, *dout;
  const long long maxT = 1LL << 22;  // 32 MB
  CK(cudaMalloc(&didx, n * sizeof(int)));
  CK(cudaMalloc(&dtab, maxT * sizeof(double)));
  CK(cudaMalloc(&dout, 64));
  CK(cudaMemset(dtab, 0, maxT * sizeof(double)));
  std::vector<int> h(n);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto launch) {
    launch();
    CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    return best;
  };
  auto set_attrs = [&](auto kern) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  };
  set_attrs(k_dsmem<4>);
  set_attrs(k_dsmem<8>);
  set_attrs(k_dsmem<16>);
  for (int cs : {1, 2, 4, 8, 16}) {
    for (int slice_kb : {64, 128, 192, 224}) {
      const int slice = slice_kb * 1024 / 8;
      const long long T = (long long)cs * slice;
      for (long long i = 0; i < n; ++i) h[i] = (int)(rng() % T);
      CK(cudaMemcpy(didx, h.data(), n * sizeof(int), cudaMemcpyHostToDevice));
      for (int threads : {512, 1024}) {
        int max_clusters = 0;
        cudaLaunchConfig_t cfg = {};
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = (size_t)slice * 8;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(cs);
        if (cudaOccupancyMaxActiveClusters(&max_clusters, (void*)k_dsmem<8>, &cfg) != cudaSuccess ||
            max_clusters == 0) {
          cudaGetLastError();
          printf("cs=%2d slice=%3d KB threads=%4d: cannot launch\n", cs, slice_kb, threads);
          continue;
        }
        cfg.gridDim = dim3(cs * max_clusters);
        float best = 1e9;
        int bestU = 0;
        for (int U : {4, 8, 16}) {
          float ms = timeit([&] {
            if (U == 4) CK(cudaLaunchKernelEx(&cfg, k_dsmem<4>, (const int*)didx, n, (const double*)dtab, slice, dout));
            if (U == 8) CK(cudaLaunchKernelEx(&cfg, k_dsmem<8>, (const int*)didx, n, (const double*)dtab, slice, dout));
            if (U == 16) CK(cudaLaunchKernelEx(&cfg, k_dsmem<16>, (const int*)didx, n, (const double*)dtab, slice, dout));
          });
          if (ms < best) best = ms, bestU = U;
        }
        float l2 = timeit([&] { k_l2<8><<<sms * 8, 256>>>(didx, n, dtab, dout); });
        printf("cs=%2d slice=%3d KB table=%6.2f MB threads=%4d clusters=%3d: DSMEM %.1f G/s (U%d)   L2 same table %.1f G/s\n",
               cs, slice_kb, T * 8 / 1048576.0, threads, max_clusters, n / (best * 1e-3) / 1e9, bestU,
               n / (l2 * 1e-3) / 1e9);
      }
    }
  }
  // L2 reference at the FSDA vector sizes
  for (long long T : {500000LL, 1500000LL, 2000000LL, 8000000LL}) {
    if (T > maxT) break;
    for (long long i = 0; i < n; ++i) h[i] = (int)(rng() % T);
    CK(cudaMemcpy(didx, h.data(), n * sizeof(int), cudaMemcpyHostToDevice));
    float l2 = timeit([&] { k_l2<8><<<sms * 8, 256>>>(didx, n, dtab, dout); });
    printf("L2 table %.1f MB: %.1f G gathers/s\n", T * 8 / 1048576.0, n / (l2 * 1e-3) / 1e9);
  }
  return 0;
}
