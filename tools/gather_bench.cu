// Microbenchmark: random 1 KB block gather into shared memory (the MoL kernel's item fetch).
// Modes: 0 = one 1 KB cp.async.bulk per block (TMA), 1 = 16-byte cp.async, 2 = LDG.128 -> STS.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE, int DEPTH>
__global__ void gather(const uint4* __restrict__ src, const int* __restrict__ idx, int n_per_cta, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[DEPTH];
  const int t = threadIdx.x, nt = blockDim.x;
  if (t < DEPTH) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[t])), "r"(1));
  __syncthreads();
  const int* my = idx + (int64_t)blockIdx.x * n_per_cta;
  int acc = 0;
  if (MODE == 0) {
    // warp 0: lanes issue 16 copies per "stage", DEPTH stages in flight
    if (t < 32) {
      uint32_t ph[DEPTH] = {0};
      for (int base = 0, st = 0; base < n_per_cta; base += 16, st = (st + 1) % DEPTH) {
        if (base >= 16 * DEPTH) {
          asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @!P1 bra W;}" ::"r"(smem_u32(&bar[st])), "r"(ph[st]));
          ph[st] ^= 1;
        }
        if (t == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[st])), "r"(16 * 1024));
        __syncwarp();
        if (t < 16) {
          const uint4* s = src + (int64_t)my[base + t] * 64;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 1024, [%2];" ::"r"(smem_u32(sm + st * 16384 + t * 1024)), "l"(s), "r"(smem_u32(&bar[st])) : "memory");
        }
        __syncwarp();
      }
      for (int st = 0; st < DEPTH; ++st) {
        asm volatile("{.reg .pred P1; W2: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @!P1 bra W2;}" ::"r"(smem_u32(&bar[st])), "r"(ph[st]));
      }
    }
  } else if (MODE == 1) {
    // all threads: 16 B cp.async per thread per block chunk; commit groups, DEPTH in flight
    for (int base = 0, st = 0; base < n_per_cta; base += 16, st = (st + 1) % DEPTH) {
      for (int k = t; k < 16 * 64; k += nt) {
        const int b = k >> 6, c = k & 63;
        const uint4* s = src + (int64_t)my[base + b] * 64 + c;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm + st * 16384 + b * 1024 + c * 16)), "l"(s) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group %0;" ::"n"(DEPTH - 1) : "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else {
    for (int base = 0, st = 0; base < n_per_cta; base += 16 * DEPTH, st ^= 1) {
      uint4 v[DEPTH * 16 * 64 / 256 + 1];
      int nk = 0;
#pragma unroll
      for (int k0 = 0; k0 < 16 * 64 * DEPTH; k0 += 256) {
        const int k = k0 + t;
        const int b = k >> 6, c = k & 63;
        v[nk++] = __ldg(src + (int64_t)my[base + b] * 64 + c);
      }
      nk = 0;
#pragma unroll
      for (int k0 = 0; k0 < 16 * 64 * DEPTH; k0 += 256) {
        const int k = k0 + t;
        *reinterpret_cast<uint4*>(sm + (k % (16 * 64 * 4)) * 16) = v[nk++];
      }
    }
  }
  __syncthreads();
  acc += sm[t];
  if (acc == 12345) sink[0] = acc;
}

// gather4: one cp.async.bulk.tensor.2d ... tile::gather4 per 4 items (4 KB) — a quarter of the
// TMA requests of mode 0
template <int DEPTH>
__global__ void gather4_kernel(const __grid_constant__ CUtensorMap tmap, const int* __restrict__ idx, int n_per_cta, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[DEPTH];
  const int t = threadIdx.x;
  if (t < DEPTH) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[t])), "r"(1));
  __syncthreads();
  const int* my = idx + (int64_t)blockIdx.x * n_per_cta;
  if (t < 32) {
    uint32_t ph[DEPTH] = {0};
    for (int base = 0, st = 0; base < n_per_cta; base += 16, st = (st + 1) % DEPTH) {
      if (base >= 16 * DEPTH) {
        asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @!P1 bra W;}" ::"r"(smem_u32(&bar[st])), "r"(ph[st]));
        ph[st] ^= 1;
      }
      if (t == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[st])), "r"(16 * 1024));
      __syncwarp();
      if (t < 4) {
        const int* r = my + base + 4 * t;
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                     ::"r"(smem_u32(sm + st * 16384 + t * 4096)), "l"(&tmap), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]),
                       "r"(smem_u32(&bar[st])) : "memory");
      }
      __syncwarp();
    }
    for (int st = 0; st < DEPTH; ++st)
      asm volatile("{.reg .pred P1; W2: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @!P1 bra W2;}" ::"r"(smem_u32(&bar[st])), "r"(ph[st]));
  }
  __syncthreads();
  if (sm[t] == 123) sink[0] = 1;
}

// mixed: per 16-item stage, stages s with (s % 8) < TMA8 go through TMA gather4 (warp 0), the
// rest through 16-byte cp.async by warps 1..NW (LSU path) — do the two paths add up?
template <int TMA8, int NW>
__global__ void mixed_kernel(const __grid_constant__ CUtensorMap tmap, const uint4* __restrict__ src,
                             const int* __restrict__ idx, int n_per_cta, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[4];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (t < 4) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[t])), "r"(1));
  __syncthreads();
  const int* my = idx + (int64_t)blockIdx.x * n_per_cta;
  const int nst = n_per_cta / 16;
  if (warp == 0) {
    uint32_t ph[4] = {0, 0, 0, 0};
    int k = 0;
    for (int st = 0; st < nst; ++st) {
      if ((st & 7) >= TMA8) continue;
      const int b = k & 3;
      if (k >= 4) {
        asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @!P1 bra W;}" ::"r"(smem_u32(&bar[b])), "r"(ph[b]));
        ph[b] ^= 1;
      }
      if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[b])), "r"(16 * 1024));
      __syncwarp();
      if (lane < 4) {
        const int* r = my + st * 16 + 4 * lane;
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                     ::"r"(smem_u32(sm + b * 16384 + lane * 4096)), "l"(&tmap), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]),
                       "r"(smem_u32(&bar[b])) : "memory");
      }
      __syncwarp();
      ++k;
    }
    for (int b = 0; b < 4 && b < k; ++b)
      asm volatile("{.reg .pred P1; W2: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @!P1 bra W2;}" ::"r"(smem_u32(&bar[b])), "r"(ph[b]));
  } else if (warp <= NW) {
    const int tt = t - 32, nt = NW * 32;
    int k = 0;
    for (int st = 0; st < nst; ++st) {
      if ((st & 7) < TMA8) continue;
      uint8_t* dst = sm + 65536 + (k & 3) * 16384;
      for (int c = tt; c < 16 * 64; c += nt) {
        const int b = c >> 6, cc = c & 63;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + b * 1024 + cc * 16)), "l"(src + (int64_t)my[st * 16 + b] * 64 + cc) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 3;" ::: "memory");
      ++k;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  if (sm[t] == 123) sink[0] = 1;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int64_t X = 10'000'000;
  uint4* src;
  cudaMalloc(&src, X * 1024);
  cudaMemset(src, 1, X * 1024);
  const int ctas = 148, n_per = 16 * 2048;
  std::vector<int> h((size_t)ctas * n_per);
  std::mt19937 rng(1);
  for (auto& x : h) x = rng() % X;
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {  // "slice-major" locality: each CTA's blocks from a shared window of 64K items
      for (size_t i = 0; i < h.size(); ++i) {
        int w = (int)((i % n_per) / 512);
        h[i] = (w * 65536 + rng() % 65536) % X;
      }
    }
    int* idx;
    cudaMalloc(&idx, h.size() * 4);
    cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    int* sink;
    cudaMalloc(&sink, 4);
    auto run = [&](auto kern, int threads, int smem, const char* name) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      kern<<<ctas, threads, smem>>>(src, idx, n_per, sink);
      cudaEventRecord(a);
      for (int r = 0; r < 3; ++r) kern<<<ctas, threads, smem>>>(src, idx, n_per, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double bytes = 3.0 * ctas * n_per * 1024.0;
      printf("%s %-28s %7.1f GB/s  (%s)\n", pass ? "local " : "random", name, bytes / ms / 1e6,
             cudaGetErrorString(cudaGetLastError()));
    };
    run(gather<0, 4>, 32, 4 * 16384, "tma_bulk_1KB depth4");
    run(gather<0, 8>, 32, 8 * 16384, "tma_bulk_1KB depth8");
    run(gather<0, 12>, 32, 12 * 16384, "tma_bulk_1KB depth12");
    run(gather<1, 4>, 256, 4 * 16384, "cp.async16 256thr depth4");
    run(gather<1, 8>, 512, 8 * 16384, "cp.async16 512thr depth8");
    run(gather<2, 1>, 256, 4 * 16384, "ldg128 256thr 16/thr");
    run(gather<2, 2>, 256, 4 * 16384, "ldg128 256thr 32/thr");
    {
      EncodeFn enc = nullptr;
      cudaDriverEntryPointQueryResult q;
      cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
      CUtensorMap tm;
      cuuint64_t dims[2] = {256, (cuuint64_t)X};
      cuuint64_t strides[1] = {1024};
      cuuint32_t box[2] = {256, 1};
      cuuint32_t es[2] = {1, 1};
      for (int prom = 0; prom < 2; ++prom) {
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, prom ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
        auto k4 = gather4_kernel<4>;
        auto k8 = gather4_kernel<8>;
        auto runt = [&](auto kern, int smem, const char* name) {
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          cudaEvent_t a, b;
          cudaEventCreate(&a);
          cudaEventCreate(&b);
          kern<<<ctas, 32, smem>>>(tm, idx, n_per, sink);
          cudaEventRecord(a);
          for (int r2 = 0; r2 < 3; ++r2) kern<<<ctas, 32, smem>>>(tm, idx, n_per, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          double bytes = 3.0 * ctas * n_per * 1024.0;
          printf("%s %-28s %7.1f GB/s  (%s)\n", pass ? "local " : "random", name, bytes / ms / 1e6,
                 cudaGetErrorString(cudaGetLastError()));
        };
        runt(k4, 4 * 16384, prom ? "gather4 depth4 l2prom256" : "gather4 depth4");
        if (!prom) {
          auto runm = [&](auto kern, int nthreads, const char* name) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            kern<<<ctas, nthreads, 8 * 16384>>>(tm, src, idx, n_per, sink);
            cudaEventRecord(a);
            for (int r2 = 0; r2 < 3; ++r2) kern<<<ctas, nthreads, 8 * 16384>>>(tm, src, idx, n_per, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            double bytes = 3.0 * ctas * n_per * 1024.0;
            printf("%s %-28s %7.1f GB/s  (%s)\n", pass ? "local " : "random", name, bytes / ms / 1e6,
                   cudaGetErrorString(cudaGetLastError()));
          };
          runm(mixed_kernel<8, 8>, 32 * 9, "mixed tma 8/8");
          runm(mixed_kernel<6, 8>, 32 * 9, "mixed tma 6/8 + lsu 8w");
          runm(mixed_kernel<5, 8>, 32 * 9, "mixed tma 5/8 + lsu 8w");
          runm(mixed_kernel<4, 8>, 32 * 9, "mixed tma 4/8 + lsu 8w");
          runm(mixed_kernel<5, 16>, 32 * 17, "mixed tma 5/8 + lsu 16w");
          runm(mixed_kernel<0, 16>, 32 * 17, "mixed lsu only 16w");
        }
        runt(k8, 8 * 16384, prom ? "gather4 depth8 l2prom256" : "gather4 depth8");
      }
    }
    cudaFree(idx);
  }
  return 0;
}
