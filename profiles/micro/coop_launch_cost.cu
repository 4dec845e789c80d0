// Device time per launch, back to back on one stream: a cooperative launch with one
// grid.sync() vs a plain launch with a hand-rolled grid barrier vs a plain launch without one.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/clc profiles/micro/coop_launch_cost.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(512) k_coop(int *out) {
  cg::this_grid().sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] += 1;
}
// sense-reversing barrier on a (count, generation) pair
__global__ void __launch_bounds__(512) k_plain_bar(unsigned *bar, int *out) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned *gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] += 1;
}
__global__ void __launch_bounds__(512) k_plain(int *out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] += 1;
}

int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  int *out;
  unsigned *bar;
  cudaMalloc(&out, 4);
  cudaMalloc(&bar, 8);
  cudaMemset(bar, 0, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int G : {1, 74, 148, 296}) {
    auto time = [&](auto launch) {
      for (int i = 0; i < 20; ++i) launch();
      cudaStreamSynchronize(s);
      cudaEventRecord(a, s);
      for (int i = 0; i < 200; ++i) launch();
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      return ms * 1e3f / 200;
    };
    const float tc = time([&] {
      void *args[] = {(void *)&out};
      cudaLaunchCooperativeKernel((void *)k_coop, dim3(G), dim3(512), args, 0, s);
    });
    const float tb = time([&] { k_plain_bar<<<G, 512, 0, s>>>(bar, out); });
    const float tp = time([&] { k_plain<<<G, 512, 0, s>>>(out); });
    printf("G=%3d  cooperative+grid.sync %.2f us  plain+own barrier %.2f us  plain %.2f us  (%s)\n", G, tc, tb,
           tp, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
