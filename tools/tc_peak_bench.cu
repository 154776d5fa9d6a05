// tcgen05 dense MMA throughput on the B200, one CTA per SM, one thread issuing back-to-back
// M=128 x N=256 MMAs (smem operands, TMEM accumulator, the stage-1 filter's shapes):
// kind::i8 (s8 x s8 -> s32, K=32 per instruction) and kind::f16 (bf16 x bf16 -> f32, K=16).
// Denominators of the stage-1 roofline (bench.py uses 2 x the measured cuBLAS bf16 rate for int8).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_peak_bench tools/tc_peak_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_ilv(uint32_t addr) {  // interleave K-major: LBO 128 B, SBO 512 B
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(512 >> 4) << 32) | (1ull << 46);
}
constexpr uint32_t IDESC_I8 = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(256 >> 3) << 17) | (uint32_t(128 >> 4) << 24);
constexpr uint32_t IDESC_BF16 = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(256 >> 3) << 17) | (uint32_t(128 >> 4) << 24);

template <int KIND>
__global__ void __launch_bounds__(128, 1) tc_kernel(int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 32768 / 16; i += blockDim.x) reinterpret_cast<int4*>(sm)[i] = make_int4(0, 0, 0, 0);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 8192);
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = tm + (it & 1) * 256;
      if (KIND == 0) {  // two K=32 int8 MMAs = K 64
#pragma unroll
        for (int k = 0; k < 2; ++k)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                       "l"(desc_ilv(a + k * 256)), "l"(desc_ilv(b + k * 256)), "r"(IDESC_I8), "r"(k));
      } else {  // four K=16 bf16 MMAs = K 64
#pragma unroll
        for (int k = 0; k < 4; ++k)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                       "l"(desc_ilv(a + k * 256)), "l"(desc_ilv(b + k * 256)), "r"(IDESC_BF16), "r"(k));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
  if (threadIdx.x == 0 && iters < 0) *sink = tm;
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const int iters = 20000;
  const char* names[2] = {"kind::i8 s8xs8->s32 M128 N256", "kind::f16 bf16xbf16->f32 M128 N256"};
  for (int kind = 0; kind < 2; ++kind) {
    auto kern = kind == 0 ? tc_kernel<0> : tc_kernel<1>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      kern<<<sms, 128, 32768>>>(iters, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 2.0 * 128 * 256 * 64 * double(iters) * sms;
      if (rep == 1)
        printf("{\"mma\": \"%s\", \"tops_per_s\": %.1f, \"ms\": %.3f, \"err\": \"%s\"}\n", names[kind], ops / (ms * 1e-3) / 1e12, ms,
               cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
