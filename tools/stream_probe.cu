// Streaming-bandwidth probe for the access mixes of the hot path (tuning aid, not product):
// copy (1R1W), 3R2W (the two-step pass's HBM pattern), 4R2W (update), read-only.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/stream_probe.cu -o tools/bin/stream_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int R, int W>
__global__ void mix(const double2* __restrict__ a, const double2* __restrict__ b, const double2* __restrict__ c,
                    const double2* __restrict__ d, double2* __restrict__ x, double2* __restrict__ y, long n2) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) {
    double2 s = a[i];
    if (R > 1) { double2 t = b[i]; s.x += t.x; s.y += t.y; }
    if (R > 2) { double2 t = c[i]; s.x += t.x; s.y += t.y; }
    if (R > 3) { double2 t = d[i]; s.x += t.x; s.y += t.y; }
    if (W > 0) x[i] = s;
    if (W > 1) y[i] = make_double2(s.y, s.x);
    if (W == 0 && s.x == 12345.678) x[0] = s;
  }
}

template <int R, int W>
void run(const char* name, double2** v, long n2, int blocks, int threads) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) mix<R, W><<<blocks, threads>>>(v[0], v[1], v[2], v[3], v[4], v[5], n2);
  const int it = 20;
  cudaEventRecord(e0);
  for (int w = 0; w < it; ++w) mix<R, W><<<blocks, threads>>>(v[0], v[1], v[2], v[3], v[4], v[5], n2);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double bytes = (double)n2 * 16 * (R + W);
  printf("{\"mix\": \"%s\", \"blocks\": %d, \"threads\": %d, \"GBps\": %.1f}\n", name, blocks, threads,
         bytes * it / (ms * 1e-3) / 1e9);
}

int main() {
  const long n = 32768000;  // 320^3
  const long n2 = n / 2;
  double2* v[6];
  for (int k = 0; k < 6; ++k) {
    cudaMalloc(&v[k], n * 8);
    cudaMemset(v[k], 0, n * 8);
  }
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int bps : {4, 8, 16}) {
    run<1, 1>("1R1W", v, n2, sms * bps, 256);
    run<3, 2>("3R2W", v, n2, sms * bps, 256);
    run<4, 2>("4R2W", v, n2, sms * bps, 256);
    run<2, 1>("2R1W", v, n2, sms * bps, 256);
    run<1, 0>("1R0W", v, n2, sms * bps, 256);
  }
  return 0;
}
