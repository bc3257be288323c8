// FP64 roofline denominator probe for B200 (sm_100a).
// Measures DFMA throughput (independent chains) and DMMA m8n8k4 throughput,
// with CUDA events, after >= 1 s of warm-up at load (clocks ramp from idle),
// each timed launch tens of ms long.  Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

template <int CH>
__global__ void dfma_chain(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c0[2] = {0, 0}, c1[2] = {0, 0}, c2[2] = {0, 0}, c3[2] = {0, 0};
  for (int i = 0; i < iters; ++i) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0[0]), "+d"(c0[1]) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c1[0]), "+d"(c1[1]) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c2[0]), "+d"(c2[1]) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c3[0]), "+d"(c3[1]) : "d"(a), "d"(b));
  }
  double s = c0[0] + c0[1] + c1[0] + c1[1] + c2[0] + c2[1] + c3[0] + c3[1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void log_tput(double* out, int iters) {
  double x = 1.0 + threadIdx.x * 1e-7, acc = 0;
  for (int i = 0; i < iters; ++i) { acc += log(x); x += 1e-9; }
  if (acc == 12345.678) out[threadIdx.x] = acc;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* d; CK(cudaMalloc(&d, 4096 * sizeof(double)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 256, blocks = sms * 8;
  float ms = 0;
  // DFMA
  const int it = 2000000;
  for (int w = 0; w < 40; ++w) dfma_chain<8><<<blocks, threads>>>(d, it, 0.999999, 1e-7);
  CK(cudaDeviceSynchronize());
  double best_dfma = 0;
  for (int r = 0; r < 20; ++r) {
    cudaEventRecord(e0); dfma_chain<8><<<blocks, threads>>>(d, it, 0.999999, 1e-7); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * it * (double)blocks * threads / (ms * 1e-3);
    if (fl > best_dfma) best_dfma = fl;
  }
  // DMMA: 8x8x4 per warp per mma = 2*8*8*4 = 512 flop
  const int it2 = 500000;
  for (int w = 0; w < 10; ++w) dmma_loop<<<blocks, threads>>>(d, it2);
  CK(cudaDeviceSynchronize());
  double best_dmma = 0;
  for (int r = 0; r < 20; ++r) {
    cudaEventRecord(e0); dmma_loop<<<blocks, threads>>>(d, it2); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 512.0 * 4 * it2 * (double)blocks * (threads / 32) / (ms * 1e-3);
    if (fl > best_dmma) best_dmma = fl;
  }
  // libdevice log throughput
  const int it3 = 4000;
  for (int w = 0; w < 3; ++w) log_tput<<<blocks, threads>>>(d, it3);
  CK(cudaDeviceSynchronize());
  double best_log = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); log_tput<<<blocks, threads>>>(d, it3); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double lg = (double)it3 * blocks * threads / (ms * 1e-3);
    if (lg > best_log) best_log = lg;
  }
  printf("{\"sms\": %d, \"clock_khz_attr\": %d, \"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"log_per_s\": %.4e}\n",
         sms, clk, best_dfma * 1e-12, best_dmma * 1e-12, best_log);
  return 0;
}
