// Host cost of a kernel launch vs the size of its __grid_constant__ parameter (B200).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/lpc profiles/micro/launch_param_cost.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
template <int N> struct P { int n; int a[N]; };
template <int N> __global__ void k(const __grid_constant__ P<N> p, int *out) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && p.n < 0) out[0] = p.a[0];
}
template <int N> double run(cudaStream_t s, int *out) {
  P<N> p{};
  p.n = 1;
  for (int i = 0; i < 50; ++i) k<N><<<1, 32, 0, s>>>(p, out);
  cudaStreamSynchronize(s);
  double best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 200; ++i) k<N><<<1, 32, 0, s>>>(p, out);
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    best = std::min(best, std::chrono::duration<double, std::micro>(t1 - t0).count() / 200);
  }
  return best;
}
int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  int *out;
  cudaMalloc(&out, 4);
  printf("param bytes -> host us per launch\n");
  printf("%6zu %6.2f\n", sizeof(P<1>), run<1>(s, out));
  printf("%6zu %6.2f\n", sizeof(P<256>), run<256>(s, out));
  printf("%6zu %6.2f\n", sizeof(P<1024>), run<1024>(s, out));
  printf("%6zu %6.2f\n", sizeof(P<2048>), run<2048>(s, out));
  printf("%6zu %6.2f\n", sizeof(P<4096>), run<4096>(s, out));
  printf("%6zu %6.2f\n", sizeof(P<7000>), run<7000>(s, out));
  return 0;
}
