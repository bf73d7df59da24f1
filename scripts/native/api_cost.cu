// Host cost of the CUDA runtime calls on the migration path (one B200):
// each call timed back-to-back N times on an otherwise idle device.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void noop(int* p) { if (p && threadIdx.x == 1234567) *p = 1; }
struct Ids4K { int n; int ids[1000]; };
__global__ void noop_params(int* p, const Ids4K ids) { if (p && threadIdx.x == 1234567) *p = ids.ids[ids.n]; }

int main() {
  const int N = 20000;
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t ev, evt;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  cudaEventCreate(&evt);
  int *h, *d;
  cudaHostAlloc(&h, 1 << 20, cudaHostAllocMapped);
  cudaMalloc(&d, 1 << 20);
  noop<<<1, 32, 0, s1>>>(d);
  cudaDeviceSynchronize();
  auto T = [&](const char* name, auto f) {
    cudaDeviceSynchronize();
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < N; ++i) f(i);
    auto t1 = std::chrono::steady_clock::now();
    cudaDeviceSynchronize();
    printf("%-44s %7.2f us/call\n", name, std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
  };
  T("kernel launch <<<1,32>>>", [&](int) { noop<<<1, 32, 0, s1>>>(d); });
  T("kernel launch <<<148,32,192KiB smem>>> (noop)", [&](int) { noop<<<148, 32, 0, s1>>>(d); });
  Ids4K big{};
  big.n = 3;
  T("kernel launch with 4 KB of parameters", [&](int) { noop_params<<<1, 32, 0, s1>>>(d, big); });
  T("cudaEventRecord (no timing)", [&](int) { cudaEventRecord(ev, s1); });
  cudaEvent_t evi;
  cudaEventCreateWithFlags(&evi, cudaEventDisableTiming | cudaEventInterprocess);
  T("cudaEventRecord (interprocess event)", [&](int) { cudaEventRecord(evi, s1); });
  T("cudaStreamWaitEvent (interprocess event)", [&](int) { cudaStreamWaitEvent(s2, evi, 0); });
  T("record + wait (interprocess)", [&](int) { cudaEventRecord(evi, s1); cudaStreamWaitEvent(s2, evi, 0); });
  T("cudaEventRecord (timing)", [&](int) { cudaEventRecord(evt, s1); });
  T("cudaStreamWaitEvent", [&](int) { cudaStreamWaitEvent(s2, ev, 0); });
  T("record + wait (one link)", [&](int) { cudaEventRecord(ev, s1); cudaStreamWaitEvent(s2, ev, 0); });
  T("cudaMemcpyAsync H2D 64 B pinned", [&](int i) { cudaMemcpyAsync(d + (i & 1023) * 16, h, 64, cudaMemcpyHostToDevice, s1); });
  T("cudaMemcpyAsync D2D 64 B", [&](int i) { cudaMemcpyAsync(d + (i & 1023) * 16, d, 64, cudaMemcpyDeviceToDevice, s1); });
  T("cudaStreamQuery (idle)", [&](int) { cudaStreamQuery(s2); });
  T("cudaGetDevice", [&](int) { int x; cudaGetDevice(&x); });
  T("cudaSetDevice(0)", [&](int) { cudaSetDevice(0); });
  T("cudaGetLastError", [&](int) { cudaGetLastError(); });
  return 0;
}
