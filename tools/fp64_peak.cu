// fp64 issue peak of the box ("measure the fp64 FMA peak").
// Each thread runs 8 independent chains of one fp64 op (DADD, DMUL or DFMA)
// for ITER iterations; 148 x 8 CTAs of 256 threads; best of 5 by CUDA events.
// Prints one JSON object: lane-ops/s for each op (a DFMA counts as one op).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_peak.cu -o fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITER = 4096, CH = 8;

template <int OP>
__global__ void __launch_bounds__(256) chains(double *out, double a, double b) {
  double v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < ITER; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) v[c] = __dadd_rn(v[c], a);
      else if (OP == 1) v[c] = __dmul_rn(v[c], b);
      else v[c] = __fma_rn(v[c], b, a);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += v[c];
  if (s == 12345.678) out[threadIdx.x] = s;   // keep the chains alive
}

template <int OP>
static double rate(double *out, int sms) {
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  chains<OP><<<blocks, threads>>>(out, 1e-9, 1.0000001);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    chains<OP><<<blocks, threads>>>(out, 1e-9, 1.0000001);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return (double)blocks * threads * ITER * CH / (best * 1e-3);
}

int main() {
  double *out;
  cudaMalloc(&out, 4096 * sizeof(double));
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const double add = rate<0>(out, sms), mul = rate<1>(out, sms), fma = rate<2>(out, sms);
  printf("{\"dadd_ops_per_s\": %.4e, \"dmul_ops_per_s\": %.4e, \"dfma_ops_per_s\": %.4e, "
         "\"sms\": %d, \"max_clock_khz\": %d, \"lanes_per_sm_per_clk_at_max\": %.2f, "
         "\"how\": \"8 independent chains/thread, 148x8 CTAs x 256 thr, 4096 iters, best of 5, CUDA events\"}\n",
         add, mul, fma, sms, clk, fma / sms / (clk * 1e3));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
