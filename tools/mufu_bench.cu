// MUFU (XU pipe) throughput on the B200: ex2.approx.ftz.f32 and rcp.approx.ftz.f32, 8 independent
// chains per thread, every SM busy.  Denominator of the MoL kernels' SFU roofline (bench.py).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mufu_bench tools/mufu_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void mufu_kernel(float* out, int iters) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = 0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float y;
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
      else asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
      x[i] = y * 0.5f;  // keep the chain (one FMUL per MUFU op)
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  float* out;
  cudaMalloc(&out, 4096);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  const char* names[2] = {"ex2.approx.ftz.f32", "rcp.approx.ftz.f32"};
  for (int op = 0; op < 2; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      if (op == 0) mufu_kernel<0><<<blocks, threads>>>(out, iters);
      else mufu_kernel<1><<<blocks, threads>>>(out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = double(blocks) * threads * iters * 8;
      if (rep == 1)
        printf("{\"op\": \"%s\", \"ops_per_s\": %.4e, \"per_sm_per_clk_at_max_clock\": %.2f, \"sms\": %d, \"max_clock_khz\": %d}\n",
               names[op], ops / (ms * 1e-3), ops / (ms * 1e-3) / sms / (clk * 1e3), sms, clk);
    }
  }
  return 0;
}
