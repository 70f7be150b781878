// Microbenchmark: throughput of random 8-byte gathers on one B200, to bound the
// gather kernels (K1/K2/K3).  Each thread streams int32 indices (coalesced) and
// sums table[idx]; variants differ in the table size (L1/L2 residency), the
// index distribution, and loads in flight per thread.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/gather_bench.bin tools/gather_bench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);                   \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

template <int U>
__global__ void __launch_bounds__(256) k_gather(const int* __restrict__ idx, long long n,
                                                const double* __restrict__ tab, double* out) {
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

// load modes: 0 ld.global.nc (L1-allocating), 1 ld.global.cg (L2 only), 2 ld.global.cs
template <int U, int MODE>
__global__ void __launch_bounds__(256) k_gather_mode(const int* __restrict__ idx, long long n,
                                                     const double* __restrict__ tab, double* out) {
  extern __shared__ double reserve[];
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (long long i = tid; i + (U - 1) * stride < n; i += U * stride) {
    int ix[U];
#pragma unroll
    for (int u = 0; u < U; ++u) ix[u] = __ldg(idx + i + u * stride);
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      v[u] = MODE == 0 ? __ldg(tab + ix[u]) : (MODE == 1 ? __ldcg(tab + ix[u]) : __ldcs(tab + ix[u]));
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 12345.0) reserve[0] = acc, out[0] = acc;
}

// indices only (stream bound)
__global__ void k_stream(const int* __restrict__ idx, long long n, double* out) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long acc = 0;
  for (long long i = tid; i < n; i += stride) acc += __ldg(idx + i);
  if (acc == 12345) out[0] = (double)acc;
}

// gathers from a shared-memory copy of the first T doubles
template <int U>
__global__ void __launch_bounds__(256) k_gather_smem(const int* __restrict__ idx, long long n,
                                                     const double* __restrict__ tab, int T,
                                                     double* out) {
  extern __shared__ double st[];
  for (int k = threadIdx.x; k < T; k += blockDim.x) st[k] = tab[k];
  __syncthreads();
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (long long i = tid; i + (U - 1) * stride < n; i += U * stride) {
    int ix[U];
#pragma unroll
    for (int u = 0; u < U; ++u) ix[u] = __ldg(idx + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += st[ix[u]];
  }
  if (acc == 12345.0) out[0] = acc;
}

int main(int argc, char** argv) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long long n = 1LL << 25;  // 33.5M gathers
  std::mt19937_64 rng(1);
  int* didx;
  double *dtab, *dout;
  const long long maxT = 1LL << 24;
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
  const int grid = sms * 8;
  if (argc > 2) {  // real index stream: raw int32 file, table size
    FILE* f = fopen(argv[1], "rb");
    std::vector<int> idx;
    int v;
    while (fread(&v, 4, 1, f) == 1) idx.push_back(v);
    fclose(f);
    const long long m = (long long)idx.size() & ~7LL;
    const long long T = atoll(argv[2]);
    CK(cudaMemcpy(didx, idx.data(), m * sizeof(int), cudaMemcpyHostToDevice));
    float ms8 = timeit([&] { k_gather<8><<<grid, 256>>>(didx, m, dtab, dout); });
    float ms4 = timeit([&] { k_gather<4><<<grid, 256>>>(didx, m, dtab, dout); });
    printf("file %s: %lld gathers, table %lld: U8 %.1f us (%.1f G/s), U4 %.1f us (%.1f G/s)\n", argv[1], m, T,
           ms8 * 1e3, m / (ms8 * 1e-3) / 1e9, ms4 * 1e3, m / (ms4 * 1e-3) / 1e9);
    return 0;
  }
  {
    const long long T = 200000;
    for (long long i = 0; i < n; ++i) h[i] = (int)(rng() % T);
    CK(cudaMemcpy(didx, h.data(), n * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(k_gather_mode<8, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_gather_mode<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_gather_mode<8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (int kb : {0, 32, 64, 100, 150, 200}) {
      // kb KB of shared memory per SM: 8 CTAs per SM share it
      const size_t per = (size_t)kb * 1024 / 8;
      float m0 = timeit([&] { k_gather_mode<8, 0><<<sms * 8, 256, per>>>(didx, n, dtab, dout); });
      float m1 = timeit([&] { k_gather_mode<8, 1><<<sms * 8, 256, per>>>(didx, n, dtab, dout); });
      float m2 = timeit([&] { k_gather_mode<8, 2><<<sms * 8, 256, per>>>(didx, n, dtab, dout); });
      printf("T=200000 smem/SM %3d KB: ldg %.1f  ldcg %.1f  ldcs %.1f G gathers/s\n", kb,
             n / (m0 * 1e-3) / 1e9, n / (m1 * 1e-3) / 1e9, n / (m2 * 1e-3) / 1e9);
    }
  }
  for (long long T : {4096LL, 32768LL, 100000LL, 200000LL, 1500000LL, 16000000LL}) {
    for (long long i = 0; i < n; ++i) h[i] = (int)(rng() % T);
    CK(cudaMemcpy(didx, h.data(), n * sizeof(int), cudaMemcpyHostToDevice));
    float ms_s = timeit([&] { k_stream<<<grid, 256>>>(didx, n, dout); });
    float ms1 = timeit([&] { k_gather<1><<<grid, 256>>>(didx, n, dtab, dout); });
    float ms4 = timeit([&] { k_gather<4><<<grid, 256>>>(didx, n, dtab, dout); });
    float ms8 = timeit([&] { k_gather<8><<<grid, 256>>>(didx, n, dtab, dout); });
    float ms16 = timeit([&] { k_gather<16><<<grid, 256>>>(didx, n, dtab, dout); });
    printf("T=%9lld (%7.1f KB)  idx-stream %.3f ms | gather U1 %.3f U4 %.3f U8 %.3f U16 %.3f ms "
           "=> best %.1f G gathers/s\n",
           T, T * 8 / 1024.0, ms_s, ms1, ms4, ms8, ms16,
           n / (std::min(std::min(ms1, ms4), std::min(ms8, ms16)) * 1e-3) / 1e9);
    if (T * 8 <= 200 * 1024) {
      CK(cudaFuncSetAttribute(k_gather_smem<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
      const int per = (int)std::max<long long>(1, (200 * 1024) / (T * 8));
      float mss = timeit([&] {
        k_gather_smem<8><<<sms * std::min(per, 8), 256, T * 8>>>(didx, n, dtab, (int)T, dout);
      });
      printf("    smem copy: %.3f ms => %.1f G gathers/s\n", mss, n / (mss * 1e-3) / 1e9);
    }
  }
  return 0;
}
