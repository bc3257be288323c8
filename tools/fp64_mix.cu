// Do DMMA (FP64 tensor, m8n8k4) and DFMA share the FP64 datapath on B200?
// Runs DMMA-only, DFMA-only and mixed loops with the same per-iteration work
// and prints their times: mixed ~= max(parts) means separate pipes, mixed ~=
// sum(parts) means one shared datapath.  One JSON line.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

template <int NMMA, int NFMA>
__global__ void mix(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-9 + c;
  double am = threadIdx.x * 1e-3, bm = 1.0 + threadIdx.x * 1e-4;
  double cm[4][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int m = 0; m < NMMA; ++m)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(cm[m & 3][0]), "+d"(cm[m & 3][1]) : "d"(am), "d"(bm));
#pragma unroll
    for (int f = 0; f < NFMA; ++f) x[f & 7] = fma(x[f & 7], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
#pragma unroll
  for (int m = 0; m < 4; ++m) s += cm[m][0] + cm[m][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int NMMA, int NFMA>
float run(double* d, int blocks, int threads, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) mix<NMMA, NFMA><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f, ms = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    mix<NMMA, NFMA><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0;
  CK(cudaSetDevice(0));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* d;
  CK(cudaMalloc(&d, 4096 * sizeof(double)));
  const int threads = 256, blocks = sms * 8, it = 20000;
  // per iteration and warp: 4 DMMA = 1024 FMA = 32 DFMA-warp-equivalents; 16 DFMA
  const float t_mma = run<4, 0>(d, blocks, threads, it);
  const float t_fma = run<0, 16>(d, blocks, threads, it);
  const float t_mix = run<4, 16>(d, blocks, threads, it);
  const float t_fma32 = run<0, 32>(d, blocks, threads, it);
  const float t_mix2 = run<2, 32>(d, blocks, threads, it);
  const double warps = (double)blocks * threads / 32;
  const double fl_mma = 4 * 512.0 * it * warps, fl_fma = 16 * 64.0 * it * warps;
  printf("{\"t_dmma4_ms\": %.3f, \"t_dfma16_ms\": %.3f, \"t_mix_ms\": %.3f, \"t_dfma32_ms\": %.3f, "
         "\"t_mix_dmma2_dfma32_ms\": %.3f, \"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f, \"mix_tflops\": %.2f}\n",
         t_mma, t_fma, t_mix, t_fma32, t_mix2, fl_mma / (t_mma * 1e-3) * 1e-12, fl_fma / (t_fma * 1e-3) * 1e-12,
         (fl_mma + fl_fma) / (t_mix * 1e-3) * 1e-12);
  return 0;
}
