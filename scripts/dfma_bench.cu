// DFMA latency / throughput probe (sm_100a): one dependent chain per thread vs 8
// independent chains; also the same for FFMA.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH, typename T>
__global__ void chain(int iters, T a, T b, T* out, long long* cyc) {
  T s[CH];
  for (int c = 0; c < CH; ++c) s[c] = (T)(threadIdx.x + c);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) s[c] = fma(s[c], a, b);
  long long t1 = clock64();
  T acc = 0;
  for (int c = 0; c < CH; ++c) acc += s[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int CH, typename T>
void run(const char* nm, int blocks, int threads) {
  T* o; long long* c; cudaMalloc(&o, blocks * threads * sizeof(T)); cudaMalloc(&c, blocks * 8);
  int iters = 4096;
  chain<CH, T><<<blocks, threads>>>(iters, (T)0.999, (T)0.001, o, c);
  cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  double per = (double)h / (iters * CH);
  printf("%s chains=%d blocks=%d threads=%d: %.2f cycles per fma per thread (%.1f fma/clk/SM if %d blocks per SM)\n",
         nm, CH, blocks, threads, per, threads / per * (blocks / 148 > 0 ? blocks / 148 : 1), blocks / 148);
  cudaFree(o); cudaFree(c);
}
int main() {
  run<1, double>("DFMA", 148, 32);
  run<8, double>("DFMA", 148, 32);
  run<1, double>("DFMA", 148, 1024);
  run<8, double>("DFMA", 148, 1024);
  run<1, float>("FFMA", 148, 32);
  run<8, float>("FFMA", 148, 1024);
  return 0;
}
