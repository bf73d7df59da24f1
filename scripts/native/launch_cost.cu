// Host cost of one kernel launch vs the size of its by-value parameters
// (cudaLaunchKernelEx with the programmatic-stream-serialization attribute,
// the way libmempool launches migrations).  Question: does the 4 KiB inline
// id list make a short migration's launch slower on the host?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o launch_cost launch_cost.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
struct Ids {
  int n;
  int ids[N];
};

template <int N>
__global__ void k(const __grid_constant__ Ids<N> p, int* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && p.n > 1000000) out[0] = p.ids[p.n % N];
}

template <int N>
double run(cudaStream_t s, int* out, int iters, bool pdl) {
  Ids<N> p{};
  p.n = 3;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(32);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  for (int i = 0; i < 100; ++i) cudaLaunchKernelEx(&cfg, k<N>, p, out);
  cudaStreamSynchronize(s);
  double best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < iters; ++i) cudaLaunchKernelEx(&cfg, k<N>, p, out);
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    double us = std::chrono::duration<double>(t1 - t0).count() * 1e6 / iters;
    if (us < best) best = us;
  }
  return best;
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int* out;
  cudaMalloc(&out, 4);
  const int iters = 2000;  // stays under the launch queue depth
  for (int pdl = 0; pdl < 2; ++pdl) {
    printf("{\"pdl\": %d, \"param_bytes_us\": {", pdl);
    printf("\"%zu\": %.3f, ", sizeof(Ids<8>), run<8>(s, out, iters, pdl));
    printf("\"%zu\": %.3f, ", sizeof(Ids<64>), run<64>(s, out, iters, pdl));
    printf("\"%zu\": %.3f, ", sizeof(Ids<256>), run<256>(s, out, iters, pdl));
    printf("\"%zu\": %.3f, ", sizeof(Ids<1000>), run<1000>(s, out, iters, pdl));
    printf("\"%zu\": %.3f}}\n", sizeof(Ids<4000>), run<4000>(s, out, iters, pdl));
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
