// Microbenchmark: cost of a cooperative grid barrier (cg::grid.sync and a
// hand-rolled one) vs a kernel boundary inside a CUDA graph, on 148 CTAs.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/bench_sync.cu -o /tmp/bs
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cgsync(int n, int* dummy) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < n; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) dummy[0] += n;
}

__device__ __forceinline__ void my_sync(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(ctr));
    } while (v < target);
  }
  __syncthreads();
}

__global__ void k_mysync(int n, unsigned* ctr) {
  for (int i = 0; i < n; ++i) my_sync(ctr, (unsigned)(i + 1) * gridDim.x);
}

__global__ void k_empty(int* d) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && d[0] == 12345) d[1] = 1;
}

int main() {
  int* dummy;
  unsigned* ctr;
  cudaMalloc(&dummy, 64);
  cudaMalloc(&ctr, 64);
  cudaMemset(dummy, 0, 64);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int threads : {256, 1024}) {
    for (int n : {0, 200}) {
      void* args[] = {&n, &dummy};
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a, st);
        cudaLaunchCooperativeKernel((void*)k_cgsync, 148, threads, args, 0, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("cg.sync   threads %4d n %3d : %8.2f us total\n", threads, n, best * 1e3);
      best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemsetAsync(ctr, 0, 4, st);
        void* args2[] = {&n, &ctr};
        cudaEventRecord(a, st);
        cudaLaunchCooperativeKernel((void*)k_mysync, 148, threads, args2, 0, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("my_sync   threads %4d n %3d : %8.2f us total\n", threads, n, best * 1e3);
    }
    // graph of 200 back-to-back empty kernels
    for (int n : {1, 200}) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
      for (int i = 0; i < n; ++i) k_empty<<<148, threads, 0, st>>>(dummy);
      cudaStreamEndCapture(st, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, st);
      cudaStreamSynchronize(st);
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a, st);
        cudaGraphLaunch(ge, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("graph     threads %4d n %3d : %8.2f us total\n", threads, n, best * 1e3);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
