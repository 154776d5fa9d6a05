// Stage-1 corpus scan on the tensor cores: tcgen05 kind::i8 (s8 x s8 -> s32, exact) over
// [B queries x 64] x [items x 64]^T, with the h-indexer threshold filter fused into the TMEM
// epilogue (hindexer.py:94-112, 155-163; quant.py:83-90).  The B x X score matrix never exists:
// each (query, 256-item) tile of int32 accumulators is tested in registers and only passers are
// appended to the query's candidate list.  A second epilogue variant writes the scores (used for
// the lambda-row threshold sample, where the scores feed the n-th-largest selection).
//
// Layout: queries (B <= 1024, padded to blocks of 128) stay resident in shared memory for the
// whole launch (64 KB); item tiles of 256 rows (16 KB of codes in the cache's interleaved
// layout + 1 KB of scales + per-32-row scale min/max) stream through a 4-stage ring by bulk copy.
// Per (tile, query block) the single MMA thread issues one M=128 x N=256 x K=64 MMA pair into
// one of two 256-column TMEM buffers (double-buffered by job parity); epilogue warpgroup w tests
// columns [64w, 64w+64) (its 64-item quarter of the tile) of every job.
//
// Passers go to per-CTA private segments of each query's candidate list with shared-memory
// counters (no global atomics on the hot path); a compaction kernel concatenates the segments.
//
#include <algorithm>
#include <cmath>
#include <cstring>

#include "kernels.cuh"
#include "stage1.cuh"

namespace molr {
namespace s1tc {

constexpr int NT = 256;    // items per tile (MMA N)
constexpr int QB = 128;    // queries per block (MMA M)
constexpr int MAXQB = 8;   // queries per launch <= 1024
constexpr int NSTAGE = 4;
constexpr int SZ_CODES = NT * 64;                 // 16 KB
// stage: codes 16 KB | scales 1 KB | perm 1 KB | chunk min/max 64 B  (1 KB aligned: 19 KB)
constexpr int ST_SC = SZ_CODES, ST_PERM = SZ_CODES + NT * 4, ST_MM = SZ_CODES + NT * 8;
constexpr int SZ_STAGE = SZ_CODES + NT * 8 + 1024;
constexpr int OFF_A = 0;                          // MAXQB x 8 KB query codes (interleave)
constexpr int OFF_RING = OFF_A + MAXQB * 8192;
constexpr int OFF_T = OFF_RING + NSTAGE * SZ_STAGE;  // per-query threshold (f32 or s32), 4 KB
constexpr int OFF_CNT = OFF_T + MAXQB * QB * 4;      // per-query passer counters of this CTA, 4 KB
constexpr int NEPI = 4;    // epilogue warpgroups: warpgroup w owns tile columns [64w, 64w + 64)
constexpr int NBUF = 2;         // 256-column TMEM accumulators (parity of the job); WG w reads cols [64w, 64w+64)
constexpr int NTHREADS = 64 + NEPI * 128;
constexpr int OFF_BAR = OFF_CNT + MAXQB * QB * 4;
constexpr int NBAR = 2 * NSTAGE + 2 * NBUF;
constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
constexpr int SMEM_BYTES = OFF_TMEM + 16;

// FILTER_*: append passers' item ids (perm) per query; WRITE_*: write every score;
// KEYS_*: filter, but append the passers' ascending score keys (f32_key / i32_key) instead of ids
// (the threshold-estimation sample: only the order statistics of the passers are needed)
enum Mode { FILTER_SCALED = 0, FILTER_RAW = 1, WRITE_SCALED = 2, WRITE_RAW = 3, KEYS_SCALED = 4, KEYS_RAW = 5 };

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity), "r"(0x989680)
      : "memory");
}
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ uint64_t desc_ilv(uint32_t addr) {  // interleave K-major: LBO 128 B (K), SBO 512 B (rows)
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(512 >> 4) << 32) | (1ull << 46);
}
// kind::i8: A = B = signed 8-bit, D = s32, K-major, M = 128, N = 64
constexpr uint32_t IDESC_I8 = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(NT >> 3) << 17) | (uint32_t(QB >> 4) << 24);
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(IDESC_I8), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
#define TMEM_LD32(taddr, r)                                                                                         \
  asm volatile(                                                                                                     \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19," \
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                                   \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),  \
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),       \
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),      \
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                    \
      : "r"(taddr))

// wait for outstanding tcgen05.ld; the registers are in/out operands so no use of them can be
// scheduled above the wait
#define TMEM_WAIT32(r)                                                                                              \
  asm volatile("tcgen05.wait::ld.sync.aligned;"                                                                     \
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),    \
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]), \
                 "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]),            \
                 "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]),            \
                 "+r"(r[30]), "+r"(r[31])                                                                           \
               :                                                                                                    \
               : "memory")

struct Params {
  const int8_t* codes;    // interleaved rows, padded to NT
  const float* scales;    // padded
  const float2* chunk_mm; // per 32 rows (min, max) scale
  const int32_t* perm;    // stored row -> item id (filter modes)
  int64_t n;              // valid rows
  int B;                  // queries in this launch (<= 1024)
  const int8_t* qcodes;   // (B, 64) linear
  const uint32_t* tkeys;  // (B,) ascending-order threshold keys (filter modes)
  int strict;
  int64_t cap;            // per query: gridDim.x private segments of `seg` entries
  int64_t seg;
  int32_t* cand;          // (B, cap)
  int32_t* cta_counts;    // (B, gridDim.x) passers per (query, CTA) (may exceed seg: overflow)
  void* out;              // write modes: (B, ld) f32 / s32
  int64_t ld;
};

template <int MODE>
__global__ void __launch_bounds__(NTHREADS, 1) s1_tc_kernel(Params P) {
  constexpr bool WRITE = MODE == WRITE_SCALED || MODE == WRITE_RAW;
  constexpr bool KEYS = MODE == KEYS_SCALED || MODE == KEYS_RAW;
  constexpr bool RAW = (MODE == FILTER_RAW || MODE == WRITE_RAW || MODE == KEYS_RAW);
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t sbase = smem_u32(sm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = (P.B + QB - 1) / QB;
  const int64_t ntiles = (P.n + NT - 1) / NT;
  // each CTA scans one contiguous block of tiles, so its private candidate segments are in
  // ascending item order and the concatenated per-query lists are (nearly) id-sorted: stage 2
  // then walks every query's candidates through the same item window at the same time (L2 reuse)
  const int64_t tile_lo = (int64_t(blockIdx.x) * ntiles) / gridDim.x;
  const int64_t tile_hi = (int64_t(blockIdx.x + 1) * ntiles) / gridDim.x;
  auto bar = [&](int i) { return sbase + OFF_BAR + 8 * i; };
  auto full_bar = [&](int s) { return bar(s); };
  auto empty_bar = [&](int s) { return bar(NSTAGE + s); };
  auto tfull = [&](int e) { return bar(2 * NSTAGE + e); };
  auto tempty = [&](int e) { return bar(2 * NSTAGE + NBUF + e); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + OFF_TMEM);
  uint32_t* scnt = reinterpret_cast<uint32_t*>(sm + OFF_CNT);

  // ---- setup: query codes -> interleave operand blocks (zero padded), thresholds, barriers ----
  for (int i = threadIdx.x; i < nqb * QB * 4; i += blockDim.x) {
    const int q = i >> 2, c = i & 3;
    int4 v = make_int4(0, 0, 0, 0);
    if (q < P.B) v = __ldg(reinterpret_cast<const int4*>(P.qcodes + int64_t(q) * 64) + c);
    const int qb = q / QB, m = q % QB;
    *reinterpret_cast<int4*>(sm + OFF_A + qb * 8192 + (m >> 3) * 512 + c * 128 + (m & 7) * 16) = v;
  }
  if (!WRITE)
    for (int q = threadIdx.x; q < nqb * QB; q += blockDim.x) {
      uint32_t t = 0;
      if (q < P.B) t = RAW ? uint32_t(key_i32(__ldg(P.tkeys + q))) : __float_as_uint(key_f32(__ldg(P.tkeys + q)));
      reinterpret_cast<uint32_t*>(sm + OFF_T)[q] = t;
      scnt[q] = 0;
    }
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1 + NEPI * 128);
    }
    for (int e = 0; e < NBUF; ++e) {
      mbar_init(tfull(e), 1);
      mbar_init(tempty(e), NEPI * 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ================= producer =================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = tile_lo; tile < tile_hi; ++tile) {
        mbar_wait(empty_bar(stage), phase ^ 1);
        const uint32_t st = sbase + OFF_RING + stage * SZ_STAGE;
        mbar_arrive_expect_tx(full_bar(stage), SZ_CODES + NT * 4 + (WRITE ? 0 : 64) + ((WRITE || KEYS) ? 0 : NT * 4));
        bulk_g2s(st, P.codes + tile * SZ_CODES, SZ_CODES, full_bar(stage));
        bulk_g2s(st + ST_SC, P.scales + tile * NT, NT * 4, full_bar(stage));
        if (!WRITE) bulk_g2s(st + ST_MM, P.chunk_mm + tile * (NT / 32), 64, full_bar(stage));
        if (!WRITE && !KEYS) bulk_g2s(st + ST_PERM, P.perm + tile * NT, NT * 4, full_bar(stage));
        if (++stage == NSTAGE) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    // per (tile, query block): one M=128 x N=256 x K=64 MMA pair into the job's 256-column
    // buffer (parity jc & 1) once all four warpgroups have drained it; one wait per job
    // (blocking: the hardware sleeps the thread)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t jc = 0;  // (tile, query block) jobs issued: buffer = jc & 1, use = jc >> 1
      for (int64_t tile = tile_lo; tile < tile_hi; ++tile) {
        mbar_wait(full_bar(stage), phase);
        tc_fence_after();
        const uint32_t bt = sbase + OFF_RING + stage * SZ_STAGE;
        for (int qb = 0; qb < nqb; ++qb, ++jc) {
          const uint32_t at = sbase + OFF_A + qb * 8192;
          const int buf = int(jc & 1);
          mbar_wait(tempty(buf), ((jc >> 1) & 1) ^ 1);
          tc_fence_after();
          mma_i8(tmem_base + buf * 256, desc_ilv(at), desc_ilv(bt), 0);
          mma_i8(tmem_base + buf * 256, desc_ilv(at + 256), desc_ilv(bt + 256), 1);
          mma_commit(tfull(buf));
        }
        mma_commit(empty_bar(stage));
        if (++stage == NSTAGE) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else {
    // ================= epilogue warpgroups =================
    // WG w owns tile columns [64w, 64w+64) of every (tile, query block) job and TMEM buffers
    // 2w / 2w+1 (double-buffered: the MMA of job j+1 runs under job j's epilogue).
    const int w = (warp - 2) >> 2;
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int p = quarter * 32 + lane;
    const uint32_t tlane = (uint32_t)(quarter * 32) << 16;
    int stage = 0;
    uint32_t phase = 0;
    int64_t jc = 0;
    int32_t* cand_cta = P.cand ? P.cand + int64_t(blockIdx.x) * P.seg : nullptr;
    for (int64_t tile = tile_lo; tile < tile_hi; ++tile) {
      mbar_wait(full_bar(stage), phase);  // scales / perm / chunk bounds of this tile are in smem
      const uint8_t* st = sm + OFF_RING + stage * SZ_STAGE;
      const float* sc = reinterpret_cast<const float*>(st + ST_SC) + w * 64;
      const int32_t* pm = reinterpret_cast<const int32_t*>(st + ST_PERM) + w * 64;
      const float2* mm = reinterpret_cast<const float2*>(st + ST_MM) + w * 2;
      const int64_t row0 = tile * NT + w * 64;
      const int nvalid = (int)imax64(0, imin64(64, P.n - row0));
      for (int qb = 0; qb < nqb; ++qb, ++jc) {
        const int q = qb * QB + p;
        const int buf = int(jc & 1);
        const uint32_t tm = tmem_base + buf * 256 + w * 64 + tlane;
        mbar_wait(tfull(buf), uint32_t((jc >> 1) & 1));
        tc_fence_after();
        // warps whose 32 query rows are all padding (small batches) have nothing to test or write
        const bool live = qb * QB + quarter * 32 < P.B;
        if (!live) {
        } else if (WRITE) {
#pragma unroll 1
          for (int cc = 0; cc < 2; ++cc) {
            uint32_t a[32];
            TMEM_LD32(tm + cc * 32, a);
            TMEM_WAIT32(a);
            const int j0 = cc * 32;
            if (q < P.B && j0 < nvalid) {
              if (RAW) {
                int32_t* o = reinterpret_cast<int32_t*>(P.out) + int64_t(q) * P.ld + row0 + j0;
                if (nvalid - j0 >= 32 && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
#pragma unroll
                  for (int j = 0; j < 32; j += 4)
                    *reinterpret_cast<int4*>(o + j) = make_int4(int32_t(a[j]), int32_t(a[j + 1]), int32_t(a[j + 2]), int32_t(a[j + 3]));
                } else {
#pragma unroll
                  for (int j = 0; j < 32; ++j)
                    if (j0 + j < nvalid) o[j] = int32_t(a[j]);
                }
              } else {
                float* o = reinterpret_cast<float*>(P.out) + int64_t(q) * P.ld + row0 + j0;
                float v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __fmul_rn((float)int32_t(a[j]), sc[j0 + j]);
                if (nvalid - j0 >= 32 && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
#pragma unroll
                  for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                } else {
#pragma unroll
                  for (int j = 0; j < 32; ++j)
                    if (j0 + j < nvalid) o[j] = v[j];
                }
              }
            }
          }
        } else {
          // per thread: one query (TMEM lane), 64 item columns as 2 chunks of 32 rows
          const uint32_t traw = reinterpret_cast<const uint32_t*>(sm + OFF_T)[q];
          const float tf = __uint_as_float(traw);
          // strict (s > t) as s >= the next float above t (thresholds are finite scores);
          // raw: acc >= t (+1 when strict)
          const float tfe = P.strict ? __uint_as_float(tf >= 0.f ? (tf == 0.f ? 1u : traw + 1u) : traw - 1u) : tf;
          const int32_t ti = int32_t(traw) + (P.strict ? 1 : 0);
          const float4* sc4 = reinterpret_cast<const float4*>(sc);
          const float tlo = tf * (1.0f - 4e-6f), thi = tf * (1.0f + 4e-6f);
          uint32_t mask[2];
          uint32_t ra[32], rb[32];
          TMEM_LD32(tm, ra);
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            uint32_t* a = cc ? rb : ra;
            // integer bound L: acc >= L is necessary to pass anywhere in this 32-row chunk
            // (from the chunk's (1/min, 1/max) scale with a relative margin; computed while the
            // TMEM load is in flight).  Padding rows are masked below, so their bound is moot.
            int32_t L;
            if (RAW) {
              L = ti;  // exact
            } else {
              const float2 inv = mm[cc];
              // floor(x - 1) saturates (no wrap) for the hopeless chunks of very large |t|
              L = __float2int_rd(fmaf(tf >= 0.f ? tlo : thi, tf >= 0.f ? inv.y : inv.x, -1.0f));
            }
            TMEM_WAIT32(a);
            if (cc == 0) TMEM_LD32(tm + 32, rb);  // next chunk loads under this chunk's test
            const int j0 = cc * 32;
            // per 8-column group: max as a tree of four 3-input maxes; a warp vote per group makes
            // the group branches warp-uniform
            uint32_t m = 0;
#pragma unroll
            for (int g8 = 0; g8 < 4; ++g8) {
              const int32_t* v = reinterpret_cast<const int32_t*>(a) + g8 * 8;
              const int32_t gm = __vimax3_s32(__vimax3_s32(v[0], v[1], v[2]), __vimax3_s32(v[3], v[4], v[5]), max(v[6], v[7]));
              if (__any_sync(0xffffffffu, gm >= L)) {  // some lane may have a passer in this group: test all 8 exactly
                const int32_t* v = reinterpret_cast<const int32_t*>(a) + g8 * 8;
                uint32_t bits = 0;
                if (RAW) {
#pragma unroll
                  for (int jj = 0; jj < 8; ++jj) bits |= uint32_t(v[jj] >= L) << jj;
                } else {  // exact fp32 test: fl(acc * scale) >= t  (hindexer.py:111)
                  const float4 s0 = sc4[(j0 + g8 * 8) >> 2], s1 = sc4[((j0 + g8 * 8) >> 2) + 1];
                  const float sv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
                  for (int jj = 0; jj < 8; ++jj) bits |= uint32_t(__fmul_rn((float)v[jj], sv[jj]) >= tfe) << jj;
                }
                m |= bits << (g8 * 8);
              }
            }
            const int lim = nvalid - j0;  // valid columns in this chunk
            if (lim < 32) m &= lim <= 0 ? 0u : ((1u << lim) - 1u);
            mask[cc] = m;
            if (KEYS && m && q < P.B) {  // append the passers' ascending score keys now (a[] is live)
              uint32_t pos = atomicAdd(scnt + q, (uint32_t)__popc(m));
              while (m) {
                const int j = __ffs(m) - 1;
                m &= m - 1;
                uint32_t accv = 0;
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) accv = (jj == j) ? a[jj] : accv;  // static register select
                const int32_t acc = int32_t(accv);
                const uint32_t key = RAW ? i32_key(acc) : f32_key(__fmul_rn((float)acc, sc[j0 + j]));
                if ((int64_t)pos < P.seg) cand_cta[int64_t(q) * P.cap + pos] = int32_t(key);
                ++pos;
              }
            }
          }
          const int total = __popc(mask[0]) + __popc(mask[1]);
          if (!KEYS && total && q < P.B) {
            uint32_t pos = atomicAdd(scnt + q, (uint32_t)total);  // shared-memory counter
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
              uint32_t m = mask[cc];
              while (m) {
                const int j = __ffs(m) - 1;
                m &= m - 1;
                if ((int64_t)pos < P.seg) cand_cta[int64_t(q) * P.cap + pos] = pm[cc * 32 + j];
                ++pos;
              }
            }
          }
        }
        tc_fence_before();
        mbar_arrive(tempty(buf));
      }
      mbar_arrive(empty_bar(stage));
      if (++stage == NSTAGE) {
        stage = 0;
        phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (!WRITE)
    for (int q = threadIdx.x; q < P.B; q += blockDim.x) P.cta_counts[int64_t(q) * gridDim.x + blockIdx.x] = int32_t(scnt[q]);
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

// ---------------------------------------------------------------------------------------------
// Small batches (B <= 32): items in M, queries in N.  With a 128-query M block a batch of a few
// queries leaves most TMEM lanes (and so most epilogue warps) idle and one warp walks all 64
// columns of its quarter serially; swapping the operands puts 128 items in the TMEM lanes and the
// (<= 32) queries in the columns, so all 16 epilogue warps share every tile: warp (w, quarter)
// owns item rows (w & 1) * 128 + 32 * quarter + lane and queries [16 (w >> 1), +16).
// Per tile: two M=128 x N=32 x K=64 MMA pairs into one of two 64-column TMEM buffers.
constexpr int SB = 32;          // largest small launch (MMA N = 16 or 32 queries)
constexpr int S_NSTAGE = 8;
constexpr int S_OFF_A = 0;      // <= 64 x 64 B query codes (interleave), 4 KB
constexpr int S_OFF_RING = 4096;
constexpr int S_OFF_T = S_OFF_RING + S_NSTAGE * SZ_STAGE;
constexpr int S_OFF_CNT = S_OFF_T + SB * 4;
constexpr int S_OFF_BAR = S_OFF_CNT + SB * 4;
constexpr int S_OFF_TMEM = S_OFF_BAR + (2 * S_NSTAGE + 16) * 8;
constexpr int S_SMEM_BYTES = S_OFF_TMEM + 16;
template <int SBQ>
constexpr uint32_t idesc_i8_s() {
  return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(SBQ >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}

#define TMEM_LD16(taddr, r)                                                                                          \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),       \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])   \
               : "r"(taddr))
#define TMEM_WAIT16(r)                                                                                               \
  asm volatile("tcgen05.wait::ld.sync.aligned;"                                                                      \
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),     \
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])  \
               :                                                                                                     \
               : "memory")

template <int SBQ>
__device__ __forceinline__ void mma_i8_s(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc_i8_s<SBQ>()), "r"(accum)
      : "memory");
}

template <int MODE, int SBQ>
__global__ void __launch_bounds__(NTHREADS, 1) s1_small_kernel(Params P) {
  // SBQ = 16: every warp tests all (<= 16) queries and the two warp halves take alternate tiles
  // (two tiles in flight per warp slot); SBQ = 32: the halves split the queries 16 / 16
  constexpr bool SPLIT_T = SBQ == 16;
  constexpr int QW = SPLIT_T ? SBQ : SBQ / 2;  // query columns per epilogue warp
  constexpr int NB = 8;                // TMEM accumulator buffers: the MMA of later tiles never
                                       // waits for this tile's epilogue
  constexpr uint32_t TCOLS = NB * 2 * SBQ;
  constexpr int NARRIVE = SPLIT_T ? NEPI * 64 : NEPI * 128;  // epilogue threads per tile
  constexpr bool WRITE = MODE == WRITE_SCALED || MODE == WRITE_RAW;
  constexpr bool KEYS = MODE == KEYS_SCALED || MODE == KEYS_RAW;
  constexpr bool RAW = (MODE == FILTER_RAW || MODE == WRITE_RAW || MODE == KEYS_RAW);
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t sbase = smem_u32(sm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (P.n + NT - 1) / NT;
  const int64_t tile_lo = (int64_t(blockIdx.x) * ntiles) / gridDim.x;
  const int64_t tile_hi = (int64_t(blockIdx.x + 1) * ntiles) / gridDim.x;
  auto bar = [&](int i) { return sbase + S_OFF_BAR + 8 * i; };
  auto full_bar = [&](int s) { return bar(s); };
  auto empty_bar = [&](int s) { return bar(S_NSTAGE + s); };
  auto tfull = [&](int e) { return bar(2 * S_NSTAGE + e); };
  auto tempty = [&](int e) { return bar(2 * S_NSTAGE + 8 + e); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + S_OFF_TMEM);
  uint32_t* scnt = reinterpret_cast<uint32_t*>(sm + S_OFF_CNT);

  for (int i = threadIdx.x; i < SBQ * 4; i += blockDim.x) {
    const int q = i >> 2, c = i & 3;
    int4 v = make_int4(0, 0, 0, 0);
    if (q < P.B) v = __ldg(reinterpret_cast<const int4*>(P.qcodes + int64_t(q) * 64) + c);
    *reinterpret_cast<int4*>(sm + S_OFF_A + (q >> 3) * 512 + c * 128 + (q & 7) * 16) = v;
  }
  if (threadIdx.x < SBQ) {
    const int q = threadIdx.x;
    uint32_t t = 0;
    if (!WRITE && q < P.B) {
      // the exact per-query bound: scaled -> fl(acc * scale) >= tfe (strict as the next float
      // above t); raw -> acc >= t (+1 when strict)
      const uint32_t traw = RAW ? uint32_t(key_i32(__ldg(P.tkeys + q))) : __float_as_uint(key_f32(__ldg(P.tkeys + q)));
      if (RAW) {
        t = uint32_t(int32_t(traw) + (P.strict ? 1 : 0));
      } else {
        const float tf = __uint_as_float(traw);
        t = P.strict ? (tf >= 0.f ? (tf == 0.f ? 1u : traw + 1u) : traw - 1u) : traw;
      }
    }
    reinterpret_cast<uint32_t*>(sm + S_OFF_T)[q] = t;
    scnt[q] = 0;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < S_NSTAGE; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1 + NARRIVE);
    }
    for (int e = 0; e < NB; ++e) {
      mbar_init(tfull(e), 1);
      mbar_init(tempty(e), NARRIVE);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = tile_lo; tile < tile_hi; ++tile) {
        mbar_wait(empty_bar(stage), phase ^ 1);
        const uint32_t st = sbase + S_OFF_RING + stage * SZ_STAGE;
        mbar_arrive_expect_tx(full_bar(stage), SZ_CODES + NT * 4 + ((WRITE || KEYS) ? 0 : NT * 4));
        bulk_g2s(st, P.codes + tile * SZ_CODES, SZ_CODES, full_bar(stage));
        bulk_g2s(st + ST_SC, P.scales + tile * NT, NT * 4, full_bar(stage));
        if (!WRITE && !KEYS) bulk_g2s(st + ST_PERM, P.perm + tile * NT, NT * 4, full_bar(stage));
        if (++stage == S_NSTAGE) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t jc = 0;
      const uint32_t at = sbase + S_OFF_A;
      for (int64_t tile = tile_lo; tile < tile_hi; ++tile, ++jc) {
        mbar_wait(full_bar(stage), phase);
        const int buf = int(jc % NB);
        mbar_wait(tempty(buf), ((jc / NB) & 1) ^ 1);
        tc_fence_after();
        const uint32_t bt = sbase + S_OFF_RING + stage * SZ_STAGE;
#pragma unroll
        for (int mb = 0; mb < 2; ++mb) {  // item rows [128 mb, 128 mb + 128) -> columns [SBQ mb, +SBQ)
          mma_i8_s<SBQ>(tmem_base + buf * 2 * SBQ + mb * SBQ, desc_ilv(bt + mb * 8192), desc_ilv(at), 0);
          mma_i8_s<SBQ>(tmem_base + buf * 2 * SBQ + mb * SBQ, desc_ilv(bt + mb * 8192 + 256), desc_ilv(at + 256), 1);
        }
        mma_commit(tfull(buf));
        mma_commit(empty_bar(stage));
        if (++stage == S_NSTAGE) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else {
    const int w = (warp - 2) >> 2;
    const int quarter = warp & 3;
    const int mb = w & 1, qh = w >> 1;
    const int r = mb * 128 + quarter * 32 + lane;  // this thread's item row within the tile
    const int qo = SPLIT_T ? 0 : QW * qh;          // first query column of this warp
    const int nq = min(QW, P.B - qo);              // live query columns of this warp
    const uint32_t* tq = reinterpret_cast<const uint32_t*>(sm + S_OFF_T) + qo;
    uint32_t tv[QW];
#pragma unroll
    for (int j = 0; j < QW; ++j) tv[j] = tq[j];
    int stage = 0;
    uint32_t phase = 0;
    int64_t jc = 0;
    int32_t* cand_cta = P.cand ? P.cand + int64_t(blockIdx.x) * P.seg : nullptr;
    for (int64_t tile = tile_lo; tile < tile_hi; ++tile, ++jc) {
      const int buf = int(jc % NB);
      if (SPLIT_T && int(jc & 1) != qh) {  // the other half's tile (stage and buffer parity = jc's)
        if (++stage == S_NSTAGE) {
          stage = 0;
          phase ^= 1;
        }
        continue;
      }
      mbar_wait(full_bar(stage), phase);
      mbar_wait(tfull(buf), uint32_t((jc / NB) & 1));
      tc_fence_after();
      if (nq > 0) {
        const uint8_t* st = sm + S_OFF_RING + stage * SZ_STAGE;
        const float s = reinterpret_cast<const float*>(st + ST_SC)[r];
        const bool valid = tile * NT + r < P.n;
        uint32_t a[QW];
        const uint32_t ta = tmem_base + buf * 2 * SBQ + mb * SBQ + qo + ((uint32_t)(quarter * 32) << 16);
        static_assert(QW == 16, "one 16-column TMEM load per warp");
        TMEM_LD16(ta, a);
        TMEM_WAIT16(a);
        if (WRITE) {
          if (valid) {
#pragma unroll
            for (int j = 0; j < QW; ++j)
              if (j < nq) {
                const int64_t o = int64_t(qo + j) * P.ld + tile * NT + r;
                if (RAW) reinterpret_cast<int32_t*>(P.out)[o] = int32_t(a[j]);
                else reinterpret_cast<float*>(P.out)[o] = __fmul_rn((float)int32_t(a[j]), s);
              }
          }
        } else {
          uint32_t m = 0;
#pragma unroll
          for (int j = 0; j < QW; ++j) {
            const bool pass = RAW ? int32_t(a[j]) >= int32_t(tv[j]) : __fmul_rn((float)int32_t(a[j]), s) >= __uint_as_float(tv[j]);
            m |= uint32_t(pass && j < nq) << j;
          }
          if (!valid) m = 0;
          if (__any_sync(0xffffffffu, m != 0)) {
            const int32_t id = KEYS ? 0 : reinterpret_cast<const int32_t*>(st + ST_PERM)[r];
            while (m) {
              const int j = __ffs(m) - 1;
              m &= m - 1;
              uint32_t accv = 0;
#pragma unroll
              for (int jj = 0; jj < QW; ++jj) accv = (jj == j) ? a[jj] : accv;
              const int q = qo + j;
              const uint32_t pos = atomicAdd(scnt + q, 1u);
              if ((int64_t)pos < P.seg) {
                int32_t v = id;
                if (KEYS) v = int32_t(RAW ? i32_key(int32_t(accv)) : f32_key(__fmul_rn((float)int32_t(accv), s)));
                cand_cta[int64_t(q) * P.cap + pos] = v;
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(tempty(buf));
      mbar_arrive(empty_bar(stage));
      if (++stage == S_NSTAGE) {
        stage = 0;
        phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (!WRITE)
    for (int q = threadIdx.x; q < P.B; q += blockDim.x) P.cta_counts[int64_t(q) * gridDim.x + blockIdx.x] = int32_t(scnt[q]);
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TCOLS));
}

// Concatenate the per-CTA segments of each query's candidate list (row b: G segments of `seg`
// entries at src + b*cap_in + g*seg, counts cnt[b*G + g]) into dst + b*cap_out; counts[b] = the
// true total (may exceed cap_out); *max_cta = the largest per-CTA count (overflow if > seg).
__global__ void __launch_bounds__(256) compact_segments_kernel(int G, int64_t seg, int64_t cap_in, const int32_t* __restrict__ src,
                                                               const int32_t* __restrict__ cnt, int64_t cap_out,
                                                               int32_t* __restrict__ dst, int64_t* __restrict__ counts,
                                                               int* __restrict__ max_cta) {
  __shared__ int64_t pre[1025];
  const int b = blockIdx.x;
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    int mx = 0;
    // an overflowed segment (c > seg) kept only its first seg passers: the list stays consistent
    // (every position below counts[b] holds a passer) and max_cta reports the overflow
    for (int g = 0; g < G; ++g) {
      const int c = cnt[int64_t(b) * G + g];
      pre[g] = acc;
      acc += imin64(c, seg);
      mx = max(mx, c);
    }
    pre[G] = acc;
    if (blockIdx.y == 0) {
      counts[b] = acc;
      if (mx > 0) atomicMax(max_cta, mx);
    }
  }
  __syncthreads();
  for (int g = blockIdx.y; g < G; g += gridDim.y) {  // (query, group of segments) per block
    const int64_t n = pre[g + 1] - pre[g];
    const int32_t* s = src + int64_t(b) * cap_in + int64_t(g) * seg;
    int32_t* d = dst + int64_t(b) * cap_out + pre[g];
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
      if (pre[g] + i < cap_out) d[i] = s[i];
  }
}

// blocks per query for compact_segments_kernel: enough to cover the SMs for small batches
inline unsigned compact_split(const molr_ctx* ctx, int Bc, int G) {
  return (unsigned)std::max(1, std::min(G, (2 * ctx->num_sms + Bc - 1) / Bc));
}
}  // namespace s1tc

// ---------------------------------------------------------------------------------------------
// Float view (MOLR_S1_FLOAT, hindexer.py:112 `view @ q` in fp32) on the tensor cores.
//
// The reference's float score is an fp32 dot (NumPy/OpenBLAS); the product's fp32 definition is
// s1_dot_f32 (common.cuh: OpenBLAS's summation order), used by filter_scan_kernel /
// scan_scores_kernel and the exact re-check (the sample threshold comes from it).
// Operands are fp16 after an exact power-of-two scaling (view: one global sv putting max|v| in
// [2^14, 2^15); query: its own sq), so v = sv v' + dv with |dv| <= 2^-11 |v| + 2^-25 sv (the
// second term for fp16 subnormals) and likewise for q.  With fp32 accumulation of the exact
// fp16 products, D = sv sq sum v'q' differs from the fp32 score s by at most
//   (2^-10 + 2^-22 + 2*64*2^-24) sum|v_i q_i| + 2^-24 (sv ||q||_1 + sq ||v||_1) (1 + 2^-10)
//   <= EPS ||v||_2 ||q||_2 + 2^-21 (sv ||q||_2 + sq ||v||_2)      (||x||_1 <= 8 ||x||_2, d = 64)
// so per (query, row) with that margin m:  D >= t + m  -> passes for certain;  D < t - m -> fails
// for certain; otherwise the row is in the undecided band and is re-scored exactly in fp32 by
// recheck_band_kernel.  The candidate SET equals the fp32 scan's bit for bit; only the order of
// the list differs (certain passers in id order, then the re-checked band).  (A bf16 image would
// make the band 8x wider: 2^-7 instead of 2^-10.)
//
// Layout: the fp16 view in the interleaved K-major layout with 128 B rows (8-row groups of 1 KB),
// 256-row tiles of 32 KB + 1 KB of row norms + 32 B of chunk max norms per stage; all B <= 1024
// queries resident as fp16 (128 KB).  Per (tile, 128-query block): 4 x (M=128, N=256, K=16)
// kind::f16 MMAs into one of two 256-column TMEM buffers; the epilogue is the int8 kernel's with
// a float max tree and no scale (thresholds and margins pre-divided by sv sq, exactly).
namespace s1bf {
using s1tc::smem_u32; using s1tc::mbar_init; using s1tc::mbar_arrive; using s1tc::mbar_arrive_expect_tx; using s1tc::mbar_wait;
using s1tc::bulk_g2s; using s1tc::fence_async_smem; using s1tc::tc_fence_before; using s1tc::tc_fence_after; using s1tc::mma_commit;
constexpr float EPS = 0.000992f;  // > 2^-10 + 2^-22 + 2^-17 (+0.5%)
constexpr int NT = 256, QB = 128, MAXQB = 8, NSTAGE = 2, NBUF = 2, NEPI = 4;
constexpr int SZ_TILE = NT * 128;
constexpr int ST_NRM = SZ_TILE, ST_CMX = SZ_TILE + NT * 4;
constexpr int SZ_STAGE = SZ_TILE + NT * 4 + 1024;
constexpr int OFF_A = 0;
constexpr int OFF_RING = OFF_A + MAXQB * 16384;
constexpr int OFF_T = OFF_RING + NSTAGE * SZ_STAGE;
constexpr int OFF_E = OFF_T + MAXQB * QB * 4;
constexpr int OFF_CNT = OFF_E + MAXQB * QB * 4;
constexpr int OFF_BCNT = OFF_CNT + MAXQB * QB * 4;
constexpr int OFF_C = OFF_BCNT + MAXQB * QB * 4;
constexpr int OFF_SQ = OFF_C + MAXQB * QB * 4;
constexpr int OFF_BAR = OFF_SQ + MAXQB * QB * 4;
constexpr int NBAR = 2 * NSTAGE + 2 * NBUF;
constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
constexpr int SMEM_BYTES = OFF_TMEM + 16;
constexpr int NTHREADS = 64 + NEPI * 128;
static_assert(SMEM_BYTES <= 232448, "shared memory");
constexpr uint32_t IDESC = (1u << 4) | (uint32_t(NT >> 3) << 17) | (uint32_t(QB >> 4) << 24);  // f16 x f16 -> f32

__device__ __forceinline__ float fmax3(float a, float b, float c) {  // FMNMX3
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__host__ __device__ __forceinline__ int64_t bf_offset(int64_t r, int k) {  // element offset of v[r][k]
  return ((r >> 3) << 9) + int64_t(k >> 3) * 64 + ((r & 7) << 3) + (k & 7);
}
__device__ __forceinline__ uint64_t desc_bf(uint32_t addr) {  // interleave K-major: LBO 128 B, SBO 1 KB
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(1024 >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ void mma_bf(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(IDESC), "r"(accum)
      : "memory");
}
__device__ __forceinline__ float up_norm(float ss) { return sqrtf(ss) * (1.0f + 1e-6f) + 1e-30f; }

// power of two p with x / p in [2^14, 2^15) (1 for x == 0)
__host__ __device__ __forceinline__ float h_scale(float x) {
  if (!(x > 0.f)) return 1.f;
  int e;
  frexpf(x, &e);  // x = f 2^e, f in [0.5, 1)
  return ldexpf(1.f, e - 15);
}
__global__ void absmax_kernel(int64_t n, const float* __restrict__ v, unsigned* __restrict__ out) {
  float m = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(v[i]));
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));  // non-negative floats order as uints
}
// fp32 rows -> fp16(v / sv) interleaved image + row norms (padding rows zero)
__global__ void build_kernel(int64_t X, int64_t xr, const float* __restrict__ v, float inv_sv, __half* __restrict__ out,
                             float* __restrict__ nrm) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < xr; r += (int64_t)gridDim.x * blockDim.x) {
    float ss = 0.f;
    for (int c = 0; c < 8; ++c) {
      __align__(16) __half h[8];
      for (int j = 0; j < 8; ++j) {
        const float x = r < X ? v[r * 64 + c * 8 + j] : 0.f;
        ss = fmaf(x, x, ss);
        h[j] = __float2half_rn(x * inv_sv);  // exact power-of-two scaling, then one rounding
      }
      *reinterpret_cast<int4*>(out + bf_offset(r, c * 8)) = *reinterpret_cast<const int4*>(h);
    }
    nrm[r] = r < X ? up_norm(ss) : 0.f;
  }
}
__global__ void chunk_max_kernel(int64_t nch, const float* __restrict__ nrm, float* __restrict__ cmx) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nch; c += (int64_t)gridDim.x * blockDim.x) {
    float m = 0.f;
    for (int j = 0; j < 32; ++j) m = fmaxf(m, nrm[c * 32 + j]);
    cmx[c] = m;
  }
}

struct Params {
  const __half* view;
  float sv;               // the view's power-of-two scale
  const float* nrm;
  const float* cmx;
  int64_t n;
  int B;
  const float* q;         // (B, 64) fp32 queries
  const uint32_t* tkeys;  // (B,) threshold keys
  int64_t cap, seg;
  int32_t* cand;          // certain passers: (B, cap) as gridDim.x segments of seg
  int32_t* band;          // undecided rows, same shape
  int32_t* cta_counts;    // (B, gridDim.x)
  int32_t* cta_bcounts;
};

__global__ void __launch_bounds__(NTHREADS, 1) bf_kernel(Params P) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t sbase = smem_u32(sm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = (P.B + QB - 1) / QB;
  const int64_t ntiles = (P.n + NT - 1) / NT;
  const int64_t tile_lo = (int64_t(blockIdx.x) * ntiles) / gridDim.x;
  const int64_t tile_hi = (int64_t(blockIdx.x + 1) * ntiles) / gridDim.x;
  auto bar = [&](int i) { return sbase + OFF_BAR + 8 * i; };
  auto full_bar = [&](int s) { return bar(s); };
  auto empty_bar = [&](int s) { return bar(NSTAGE + s); };
  auto tfull = [&](int e) { return bar(2 * NSTAGE + e); };
  auto tempty = [&](int e) { return bar(2 * NSTAGE + NBUF + e); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + OFF_TMEM);
  uint32_t* scnt = reinterpret_cast<uint32_t*>(sm + OFF_CNT);
  uint32_t* sbcnt = reinterpret_cast<uint32_t*>(sm + OFF_BCNT);
  float* st_t = reinterpret_cast<float*>(sm + OFF_T);
  float* st_e = reinterpret_cast<float*>(sm + OFF_E);

  // per query: power-of-two scale sq, threshold t, margin factor e and constant margin c, all in
  // units of sv * sq (t' = t / (sv sq), e' = (EPS ||q|| + 2^-21 sq) / (sv sq),
  // c' = 2^-21 sv ||q|| / (sv sq)); then the queries -> fp16 operand blocks (zero padded)
  float* st_c = reinterpret_cast<float*>(sm + OFF_C);
  float* st_sq = reinterpret_cast<float*>(sm + OFF_SQ);
  for (int q = threadIdx.x; q < nqb * QB; q += blockDim.x) {
    float t = 0.f, e = 0.f, c = 0.f, sq = 1.f;
    if (q < P.B) {
      float ss = 0.f, mx = 0.f;
      for (int k = 0; k < 64; ++k) {
        const float x = __ldg(P.q + int64_t(q) * 64 + k);
        ss = fmaf(x, x, ss);
        mx = fmaxf(mx, fabsf(x));
      }
      sq = h_scale(mx);
      const float inv = 1.f / (P.sv * sq);  // exact (power of two)
      const float nq = up_norm(ss);
      t = key_f32(__ldg(P.tkeys + q)) * inv;
      e = (EPS * nq + 4.8e-7f * sq) * inv;  // 4.8e-7 = 2^-21 (1 + 0.7%)
      c = 4.8e-7f * P.sv * nq * inv;
    }
    st_t[q] = t;
    st_e[q] = e;
    st_c[q] = c;
    st_sq[q] = sq;
    scnt[q] = 0;
    sbcnt[q] = 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nqb * QB * 8; i += blockDim.x) {
    const int q = i >> 3, c = i & 7;
    const float inv_sq = 1.f / st_sq[q];
    __align__(16) __half h[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) h[j] = __float2half_rn(q < P.B ? __ldg(P.q + int64_t(q) * 64 + c * 8 + j) * inv_sq : 0.f);
    const int qb = q / QB, m = q % QB;
    *reinterpret_cast<int4*>(sm + OFF_A + qb * 16384 + (m >> 3) * 1024 + c * 128 + (m & 7) * 16) =
        *reinterpret_cast<const int4*>(h);
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1 + NEPI * 128);
    }
    for (int e = 0; e < NBUF; ++e) {
      mbar_init(tfull(e), 1);
      mbar_init(tempty(e), NEPI * 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = tile_lo; tile < tile_hi; ++tile) {
        mbar_wait(empty_bar(stage), phase ^ 1);
        const uint32_t st = sbase + OFF_RING + stage * SZ_STAGE;
        mbar_arrive_expect_tx(full_bar(stage), SZ_TILE + NT * 4 + 32);
        bulk_g2s(st, P.view + tile * (NT * 64), SZ_TILE, full_bar(stage));
        bulk_g2s(st + ST_NRM, P.nrm + tile * NT, NT * 4, full_bar(stage));
        bulk_g2s(st + ST_CMX, P.cmx + tile * (NT / 32), 32, full_bar(stage));
        if (++stage == NSTAGE) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t jc = 0;
      for (int64_t tile = tile_lo; tile < tile_hi; ++tile) {
        mbar_wait(full_bar(stage), phase);
        tc_fence_after();
        const uint32_t bt = sbase + OFF_RING + stage * SZ_STAGE;
        for (int qb = 0; qb < nqb; ++qb, ++jc) {
          const uint32_t at = sbase + OFF_A + qb * 16384;
          const int buf = int(jc & 1);
          mbar_wait(tempty(buf), ((jc >> 1) & 1) ^ 1);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < 4; ++k) mma_bf(tmem_base + buf * 256, desc_bf(at + k * 256), desc_bf(bt + k * 256), k > 0);
          mma_commit(tfull(buf));
        }
        mma_commit(empty_bar(stage));
        if (++stage == NSTAGE) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else {
    const int w = (warp - 2) >> 2;
    const int quarter = warp & 3;
    const int p = quarter * 32 + lane;
    const uint32_t tlane = (uint32_t)(quarter * 32) << 16;
    int stage = 0;
    uint32_t phase = 0;
    int64_t jc = 0;
    int32_t* cand_cta = P.cand + int64_t(blockIdx.x) * P.seg;
    int32_t* band_cta = P.band + int64_t(blockIdx.x) * P.seg;
    for (int64_t tile = tile_lo; tile < tile_hi; ++tile) {
      mbar_wait(full_bar(stage), phase);
      const uint8_t* st = sm + OFF_RING + stage * SZ_STAGE;
      const float* nrm = reinterpret_cast<const float*>(st + ST_NRM) + w * 64;
      const float* cmx = reinterpret_cast<const float*>(st + ST_CMX) + w * 2;
      const int64_t row0 = tile * NT + w * 64;
      const int nvalid = (int)imax64(0, imin64(64, P.n - row0));
      for (int qb = 0; qb < nqb; ++qb, ++jc) {
        const int q = qb * QB + p;
        const int buf = int(jc & 1);
        const uint32_t tm = tmem_base + buf * 256 + w * 64 + tlane;
        mbar_wait(tfull(buf), uint32_t((jc >> 1) & 1));
        tc_fence_after();
        bool released = false;
        if (qb * QB + quarter * 32 < P.B) {
          const float t = st_t[q], e = st_e[q];
          const float slack = st_c[q] + fabsf(t) * 1e-6f + 1e-30f;
          uint32_t cert[2], bnd[2];
          uint32_t ra[32], rb[32];
          TMEM_LD32(tm, ra);
          TMEM_LD32(tm + 32, rb);
          TMEM_WAIT32(ra);
          TMEM_WAIT32(rb);
          tc_fence_before();  // accumulators in registers: release the TMEM buffer early
          mbar_arrive(tempty(buf));
          released = true;
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            uint32_t* a = cc ? rb : ra;
            const float lo = t - (e * cmx[cc] + slack);  // below it the whole chunk fails for certain
            const float* v = reinterpret_cast<const float*>(a);
            // in a hit group: certain above the chunk's upper bound, band between the two bounds
            // (the chunk's max row norm for both: two compares per element)
            const float hi = t + (e * cmx[cc] + slack);
            uint32_t mc = 0, ml = 0;
#pragma unroll
            for (int g8 = 0; g8 < 4; ++g8) {
              const float* u = v + g8 * 8;
              const float gm = fmax3(fmax3(u[0], u[1], u[2]), fmax3(u[3], u[4], u[5]), fmaxf(u[6], u[7]));
              if (__any_sync(0xffffffffu, gm >= lo)) {
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                  mc |= uint32_t(u[jj] >= hi) << (g8 * 8 + jj);
                  ml |= uint32_t(u[jj] >= lo) << (g8 * 8 + jj);
                }
              }
            }
            const uint32_t mb = ml & ~mc;
            const int lim = nvalid - cc * 32;
            const uint32_t vm = lim >= 32 ? 0xffffffffu : (lim <= 0 ? 0u : ((1u << lim) - 1u));
            cert[cc] = mc & vm;
            bnd[cc] = mb & vm;
          }
          if (q < P.B) {
            const int nc = __popc(cert[0]) + __popc(cert[1]), nb = __popc(bnd[0]) + __popc(bnd[1]);
            if (nc) {
              uint32_t pos = atomicAdd(scnt + q, (uint32_t)nc);
#pragma unroll
              for (int cc = 0; cc < 2; ++cc)
                for (uint32_t m = cert[cc]; m; m &= m - 1, ++pos)
                  if ((int64_t)pos < P.seg) cand_cta[int64_t(q) * P.cap + pos] = int32_t(row0 + cc * 32 + __ffs(m) - 1);
            }
            if (nb) {
              uint32_t pos = atomicAdd(sbcnt + q, (uint32_t)nb);
#pragma unroll
              for (int cc = 0; cc < 2; ++cc)
                for (uint32_t m = bnd[cc]; m; m &= m - 1, ++pos)
                  if ((int64_t)pos < P.seg) band_cta[int64_t(q) * P.cap + pos] = int32_t(row0 + cc * 32 + __ffs(m) - 1);
            }
          }
        }
        if (!released) {
          tc_fence_before();
          mbar_arrive(tempty(buf));
        }
      }
      mbar_arrive(empty_bar(stage));
      if (++stage == NSTAGE) {
        stage = 0;
        phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  for (int q = threadIdx.x; q < P.B; q += blockDim.x) {
    P.cta_counts[int64_t(q) * gridDim.x + blockIdx.x] = int32_t(scnt[q]);
    P.cta_bcounts[int64_t(q) * gridDim.x + blockIdx.x] = int32_t(sbcnt[q]);
  }
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

// Small batches (B <= 32) of the float view: items in M, queries in N (as s1tc::s1_small_kernel).
// Per 256-row tile two M=128 x N=SBQ x K=64 fp16 MMA groups (4 x K=16 each) into one of 8 TMEM
// buffers; every epilogue thread owns one item row and classifies its 16 query columns as
// certain / band / fail with the row's own norm (no chunk pre-test needed: one row per thread).
constexpr int SS_NSTAGE = 4;
constexpr int SS_STAGE = SZ_TILE + NT * 4;  // fp16 tile + row norms (33 KB)
constexpr int SS_OFF_Q = 0;                 // <= 32 x 128 B queries
constexpr int SS_OFF_RING = 4096;
constexpr int SS_OFF_T = SS_OFF_RING + SS_NSTAGE * SS_STAGE;
constexpr int SS_OFF_E = SS_OFF_T + 128;
constexpr int SS_OFF_S = SS_OFF_E + 128;
constexpr int SS_OFF_SQ = SS_OFF_S + 128;
constexpr int SS_OFF_CNT = SS_OFF_SQ + 128;
constexpr int SS_OFF_BCNT = SS_OFF_CNT + 128;
constexpr int SS_OFF_BAR = SS_OFF_BCNT + 128;
constexpr int SS_OFF_TMEM = SS_OFF_BAR + (2 * SS_NSTAGE + 16) * 8;
constexpr int SS_SMEM = SS_OFF_TMEM + 16;
template <int SBQ>
constexpr uint32_t idesc_h_s() {
  return (1u << 4) | (uint32_t(SBQ >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}
template <int SBQ>
__device__ __forceinline__ void mma_h_s(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc_h_s<SBQ>()), "r"(accum)
      : "memory");
}
#define TMEM_LD16H(taddr, r)                                                                                         \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),       \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])   \
               : "r"(taddr))
#define TMEM_WAIT16H(r)                                                                                              \
  asm volatile("tcgen05.wait::ld.sync.aligned;"                                                                      \
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),     \
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])  \
               :                                                                                                     \
               : "memory")

template <int SBQ>
__global__ void __launch_bounds__(NTHREADS, 1) bf_small_kernel(Params P) {
  constexpr bool SPLIT_T = SBQ == 16;        // warp halves take alternate tiles (else split the queries)
  constexpr int QW = 16;
  constexpr int NB = 8;
  constexpr uint32_t TCOLS = NB * 2 * SBQ;
  constexpr int NARRIVE = SPLIT_T ? NEPI * 64 : NEPI * 128;
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t sbase = smem_u32(sm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (P.n + NT - 1) / NT;
  const int64_t tile_lo = (int64_t(blockIdx.x) * ntiles) / gridDim.x;
  const int64_t tile_hi = (int64_t(blockIdx.x + 1) * ntiles) / gridDim.x;
  auto bar = [&](int i) { return sbase + SS_OFF_BAR + 8 * i; };
  auto full_bar = [&](int s) { return bar(s); };
  auto empty_bar = [&](int s) { return bar(SS_NSTAGE + s); };
  auto tfull = [&](int e) { return bar(2 * SS_NSTAGE + e); };
  auto tempty = [&](int e) { return bar(2 * SS_NSTAGE + 8 + e); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + SS_OFF_TMEM);
  uint32_t* scnt = reinterpret_cast<uint32_t*>(sm + SS_OFF_CNT);
  uint32_t* sbcnt = reinterpret_cast<uint32_t*>(sm + SS_OFF_BCNT);
  float* st_t = reinterpret_cast<float*>(sm + SS_OFF_T);
  float* st_e = reinterpret_cast<float*>(sm + SS_OFF_E);
  float* st_s = reinterpret_cast<float*>(sm + SS_OFF_S);
  float* st_sq = reinterpret_cast<float*>(sm + SS_OFF_SQ);

  if (threadIdx.x < SBQ) {  // per query (as bf_kernel): scale, threshold, margin factor, constant slack
    const int q = threadIdx.x;
    float t = 0.f, e = 0.f, c = 0.f, sq = 1.f;
    if (q < P.B) {
      float ss = 0.f, mx = 0.f;
      for (int k = 0; k < 64; ++k) {
        const float x = __ldg(P.q + int64_t(q) * 64 + k);
        ss = fmaf(x, x, ss);
        mx = fmaxf(mx, fabsf(x));
      }
      sq = h_scale(mx);
      const float inv = 1.f / (P.sv * sq);
      const float nq = up_norm(ss);
      t = key_f32(__ldg(P.tkeys + q)) * inv;
      e = (EPS * nq + 4.8e-7f * sq) * inv;
      c = 4.8e-7f * P.sv * nq * inv;
    }
    st_t[q] = t;
    st_e[q] = e;
    st_s[q] = c + fabsf(t) * 1e-6f + 1e-30f;
    st_sq[q] = sq;
    scnt[q] = 0;
    sbcnt[q] = 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < SBQ * 8; i += blockDim.x) {
    const int q = i >> 3, c = i & 7;
    const float inv_sq = 1.f / st_sq[q];
    __align__(16) __half h[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) h[j] = __float2half_rn(q < P.B ? __ldg(P.q + int64_t(q) * 64 + c * 8 + j) * inv_sq : 0.f);
    *reinterpret_cast<int4*>(sm + SS_OFF_Q + (q >> 3) * 1024 + c * 128 + (q & 7) * 16) = *reinterpret_cast<const int4*>(h);
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < SS_NSTAGE; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1 + NARRIVE);
    }
    for (int e = 0; e < NB; ++e) {
      mbar_init(tfull(e), 1);
      mbar_init(tempty(e), NARRIVE);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = tile_lo; tile < tile_hi; ++tile) {
        mbar_wait(empty_bar(stage), phase ^ 1);
        const uint32_t st = sbase + SS_OFF_RING + stage * SS_STAGE;
        mbar_arrive_expect_tx(full_bar(stage), SZ_TILE + NT * 4);
        bulk_g2s(st, P.view + tile * (NT * 64), SZ_TILE, full_bar(stage));
        bulk_g2s(st + SZ_TILE, P.nrm + tile * NT, NT * 4, full_bar(stage));
        if (++stage == SS_NSTAGE) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t jc = 0;
      const uint32_t at = sbase + SS_OFF_Q;
      for (int64_t tile = tile_lo; tile < tile_hi; ++tile, ++jc) {
        mbar_wait(full_bar(stage), phase);
        const int buf = int(jc % NB);
        mbar_wait(tempty(buf), ((jc / NB) & 1) ^ 1);
        tc_fence_after();
        const uint32_t bt = sbase + SS_OFF_RING + stage * SS_STAGE;
#pragma unroll
        for (int mb = 0; mb < 2; ++mb)  // item rows [128 mb, +128) -> columns [SBQ mb, +SBQ)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_h_s<SBQ>(tmem_base + buf * 2 * SBQ + mb * SBQ, desc_bf(bt + mb * 16384 + k * 256), desc_bf(at + k * 256),
                         k > 0);
        mma_commit(tfull(buf));
        mma_commit(empty_bar(stage));
        if (++stage == SS_NSTAGE) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else {
    const int w = (warp - 2) >> 2;
    const int quarter = warp & 3;
    const int mb = w & 1, qh = w >> 1;
    const int r = mb * 128 + quarter * 32 + lane;
    const int qo = SPLIT_T ? 0 : QW * qh;
    const int nq = min(QW, P.B - qo);
    float tv[QW], ev[QW], sv[QW];
#pragma unroll
    for (int j = 0; j < QW; ++j) tv[j] = st_t[qo + j], ev[j] = st_e[qo + j], sv[j] = st_s[qo + j];
    int stage = 0;
    uint32_t phase = 0;
    int64_t jc = 0;
    int32_t* cand_cta = P.cand + int64_t(blockIdx.x) * P.seg;
    int32_t* band_cta = P.band + int64_t(blockIdx.x) * P.seg;
    for (int64_t tile = tile_lo; tile < tile_hi; ++tile, ++jc) {
      const int buf = int(jc % NB);
      if (SPLIT_T && int(jc & 1) != qh) {
        if (++stage == SS_NSTAGE) {
          stage = 0;
          phase ^= 1;
        }
        continue;
      }
      mbar_wait(full_bar(stage), phase);
      mbar_wait(tfull(buf), uint32_t((jc / NB) & 1));
      tc_fence_after();
      if (nq > 0) {
        const float nv = reinterpret_cast<const float*>(sm + SS_OFF_RING + stage * SS_STAGE + SZ_TILE)[r];
        const bool valid = tile * NT + r < P.n;
        uint32_t a[16];
        TMEM_LD16H(tmem_base + buf * 2 * SBQ + mb * SBQ + qo + ((uint32_t)(quarter * 32) << 16), a);
        TMEM_WAIT16H(a);
        uint32_t mc = 0, mbd = 0;
#pragma unroll
        for (int j = 0; j < QW; ++j) {
          const float d = __uint_as_float(a[j]);
          const float m = fmaf(ev[j], nv, sv[j]);
          const bool c = d >= tv[j] + m;
          const bool b = !c && d >= tv[j] - m;
          mc |= uint32_t(c && j < nq) << j;
          mbd |= uint32_t(b && j < nq) << j;
        }
        if (!valid) mc = mbd = 0;
        if (__any_sync(0xffffffffu, (mc | mbd) != 0)) {
          const int32_t id = int32_t(tile * NT + r);
          for (uint32_t m2 = mc; m2; m2 &= m2 - 1) {
            const int q = qo + __ffs(m2) - 1;
            const uint32_t pos = atomicAdd(scnt + q, 1u);
            if ((int64_t)pos < P.seg) cand_cta[int64_t(q) * P.cap + pos] = id;
          }
          for (uint32_t m2 = mbd; m2; m2 &= m2 - 1) {
            const int q = qo + __ffs(m2) - 1;
            const uint32_t pos = atomicAdd(sbcnt + q, 1u);
            if ((int64_t)pos < P.seg) band_cta[int64_t(q) * P.cap + pos] = id;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(tempty(buf));
      mbar_arrive(empty_bar(stage));
      if (++stage == SS_NSTAGE) {
        stage = 0;
        phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  for (int q = threadIdx.x; q < P.B; q += blockDim.x) {
    P.cta_counts[int64_t(q) * gridDim.x + blockIdx.x] = int32_t(scnt[q]);
    P.cta_bcounts[int64_t(q) * gridDim.x + blockIdx.x] = int32_t(sbcnt[q]);
  }
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TCOLS));
}

__global__ void seg_max_kernel(int64_t n, const int32_t* __restrict__ cnt, int* __restrict__ mx) {
  int m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, cnt[i]);
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0 && m > 0) atomicMax(mx, m);
}

// exact fp32 re-score of the undecided band (the s1_dot64 order of filter_scan_kernel);
// passers are appended after the query's certain passers (counts[b] = running total)
__global__ void __launch_bounds__(256) recheck_band_kernel(int G, int64_t seg, int64_t cap_in, const int32_t* __restrict__ band,
                                                           const int32_t* __restrict__ bcnt, const float* __restrict__ vf,
                                                           const float* __restrict__ qf, const uint32_t* __restrict__ tkeys,
                                                           int strict, int64_t cap_out, int32_t* __restrict__ cand,
                                                           int64_t* __restrict__ counts) {
  __shared__ __align__(16) float sq[64];
  const int b = blockIdx.x;
  if (threadIdx.x < 64) sq[threadIdx.x] = qf[int64_t(b) * 64 + threadIdx.x];
  __syncthreads();
  const uint32_t tk = tkeys[b];
  for (int g = blockIdx.y; g < G; g += gridDim.y) {  // (query, group of CTA segments) per block
    const int64_t n = imin64(bcnt[int64_t(b) * G + g], seg);
    const int32_t* src = band + int64_t(b) * cap_in + int64_t(g) * seg;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const int32_t r = src[i];
      const float4* v4 = reinterpret_cast<const float4*>(vf + int64_t(r) * 64);
      float v[64];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const float4 x = __ldg(v4 + k);
        v[4 * k] = x.x, v[4 * k + 1] = x.y, v[4 * k + 2] = x.z, v[4 * k + 3] = x.w;
      }
      const uint32_t key = f32_key(s1_dot64(v, sq));
      if (strict ? key > tk : key >= tk) {
        const int64_t pos = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(counts + b), 1ull);
        if (pos < cap_out) cand[int64_t(b) * cap_out + pos] = r;
      }
    }
  }
}
__global__ void gather_f32_rows_kernel(int64_t n, int64_t np, const float* __restrict__ vf, const int64_t* __restrict__ rows,
                                       float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np * 16; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i >> 4;
    const int c = int(i & 15);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < n) v = __ldg(reinterpret_cast<const float4*>(vf + rows[r] * 64) + c);
    reinterpret_cast<float4*>(out + r * 64)[c] = v;
  }
}
}  // namespace s1bf

bool s1_tc_supported(const molr_cache* c, int mode) {
  return c && mode != MOLR_S1_FLOAT && c->d1 == 64 && c->s1_codes && c->s1_chunk_mm && !dev_knob("MOLR_DISABLE_TC") &&
         !dev_knob("MOLR_S1_NO_TC");
}

// Scan rows [0, n) of an interleaved code matrix against B queries (chunks of 1024 per launch).
// filter: tkeys != nullptr -> append passers to cand / counts; else write scores to out (B, ld).
int s1_tc_scan(molr_ctx* ctx, int mode, const int8_t* codes, const float* scales, const float2* mm,
               const int32_t* perm, int64_t n, int B,
               const int8_t* qcodes, const uint32_t* tkeys, int strict, int64_t cap, int32_t* cand, int64_t* counts,
               void* out, int64_t ld, cudaStream_t s, bool emit_keys, const S1Deferred* defer) {
  using namespace s1tc;
  if (n <= 0 || B <= 0) return MOLR_OK;
  const bool raw = mode == MOLR_S1_INT8_RAW;
  const int m = tkeys ? (emit_keys ? (raw ? KEYS_RAW : KEYS_SCALED) : (raw ? FILTER_RAW : FILTER_SCALED))
                      : (raw ? WRITE_RAW : WRITE_SCALED);
  const int64_t ntiles = (n + NT - 1) / NT;
  const int grid = (int)std::min<int64_t>(ntiles, ctx->num_sms);
  const bool filter = tkeys != nullptr;
  // per-CTA private segments: expected cap/grid passers each, with headroom; one retry at the
  // exact maximum if a segment overflowed
  int64_t seg = filter ? (cap / grid) + (cap / grid) / 3 + 64 : 0;
  if (filter && defer) {
    seg = std::max<int64_t>(seg, defer->seg_min);
    if (defer->seg_used) *defer->seg_used = std::max<int64_t>(*defer->seg_used, seg);
  }
  for (int b0 = 0; b0 < B; b0 += MAXQB * QB) {
    const int Bc = std::min(B - b0, MAXQB * QB);
    for (int attempt = 0; attempt < 2; ++attempt) {
      Scratch priv, ccount, mx;
      Params P;
      P.codes = codes;
      P.scales = scales;
      P.chunk_mm = mm;
      P.perm = perm;
      P.n = n;
      P.B = Bc;
      P.qcodes = qcodes + int64_t(b0) * 64;
      P.tkeys = tkeys ? tkeys + b0 : nullptr;
      P.strict = strict;
      P.seg = seg;
      P.cap = int64_t(grid) * seg;
      P.cand = nullptr;
      P.cta_counts = nullptr;
      int* mxp = nullptr;
      if (filter) {
        MOLR_TRY(priv.alloc(size_t(Bc) * P.cap * 4, s));
        MOLR_TRY(ccount.alloc(size_t(Bc) * grid * 4, s));
        if (defer) {
          mxp = defer->seg_need;
        } else {
          MOLR_TRY(mx.alloc(4, s));
          MOLR_CUDA(cudaMemsetAsync(mx.p, 0, 4, s));
          mxp = mx.as<int>();
        }
        P.cand = priv.as<int32_t>();
        P.cta_counts = ccount.as<int32_t>();
      }
      P.out = out ? reinterpret_cast<char*>(out) + int64_t(b0) * ld * 4 : nullptr;
      P.ld = ld;
      const bool small = Bc <= SB && !dev_knob("MOLR_S1_NO_SMALL");
      auto launch = [&](auto kern) -> int {
        const int bytes = small ? S_SMEM_BYTES : SMEM_BYTES;
        MOLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        kern<<<grid, NTHREADS, bytes, s>>>(P);
        MOLR_LAUNCHED(ctx);
        return MOLR_OK;
      };
      if (small) {
        auto pick = [&](auto k16, auto k32) { return Bc <= 16 ? launch(k16) : launch(k32); };
        switch (m) {
          case FILTER_SCALED: MOLR_TRY(pick(s1_small_kernel<FILTER_SCALED, 16>, s1_small_kernel<FILTER_SCALED, 32>)); break;
          case FILTER_RAW: MOLR_TRY(pick(s1_small_kernel<FILTER_RAW, 16>, s1_small_kernel<FILTER_RAW, 32>)); break;
          case WRITE_SCALED: MOLR_TRY(pick(s1_small_kernel<WRITE_SCALED, 16>, s1_small_kernel<WRITE_SCALED, 32>)); break;
          case WRITE_RAW: MOLR_TRY(pick(s1_small_kernel<WRITE_RAW, 16>, s1_small_kernel<WRITE_RAW, 32>)); break;
          case KEYS_SCALED: MOLR_TRY(pick(s1_small_kernel<KEYS_SCALED, 16>, s1_small_kernel<KEYS_SCALED, 32>)); break;
          default: MOLR_TRY(pick(s1_small_kernel<KEYS_RAW, 16>, s1_small_kernel<KEYS_RAW, 32>)); break;
        }
      } else {
        switch (m) {
          case FILTER_SCALED: MOLR_TRY(launch(s1_tc_kernel<FILTER_SCALED>)); break;
          case FILTER_RAW: MOLR_TRY(launch(s1_tc_kernel<FILTER_RAW>)); break;
          case WRITE_SCALED: MOLR_TRY(launch(s1_tc_kernel<WRITE_SCALED>)); break;
          case WRITE_RAW: MOLR_TRY(launch(s1_tc_kernel<WRITE_RAW>)); break;
          case KEYS_SCALED: MOLR_TRY(launch(s1_tc_kernel<KEYS_SCALED>)); break;
          default: MOLR_TRY(launch(s1_tc_kernel<KEYS_RAW>)); break;
        }
      }
      if (!filter) break;
      compact_segments_kernel<<<dim3(Bc, compact_split(ctx, Bc, grid)), 256, 0, s>>>(
          grid, seg, P.cap, P.cand, P.cta_counts, cap, cand + int64_t(b0) * cap, counts + b0, mxp);
      MOLR_LAUNCHED(ctx);
      if (defer) break;  // checked by the caller after its end-of-call synchronisation
      int hmx = 0;
      MOLR_CUDA(cudaMemcpyAsync(&hmx, mx.p, 4, cudaMemcpyDeviceToHost, s));
      MOLR_CUDA(cudaStreamSynchronize(s));
      if (hmx <= seg) break;
      seg = hmx;  // a private segment overflowed: rerun with the exact maximum
    }
  }
  return MOLR_OK;
}

bool s1_bf_supported(const molr_cache* c, int mode) {
  return c && mode == MOLR_S1_FLOAT && c->d1 == 64 && c->s1_f32 && c->X > 0 && !dev_knob("MOLR_DISABLE_TC") && !dev_knob("MOLR_S1_NO_BF");
}

static int s1_bf_build(molr_cache* c, cudaStream_t s) {
  using namespace s1bf;
  if (c->s1_bf_ready.load(std::memory_order_acquire)) return MOLR_OK;
  std::lock_guard<std::mutex> g(c->seal_mu);
  if (c->s1_bf_ready.load()) return MOLR_OK;
  const int64_t xr = (c->X + NT - 1) / NT * NT;
  if (!c->s1_bf) {
    MOLR_CUDA(cudaMalloc(&c->s1_bf, size_t(xr) * 128));
    MOLR_CUDA(cudaMalloc(&c->s1_bnorm, size_t(xr) * 4));
    MOLR_CUDA(cudaMalloc(&c->s1_bnmax, size_t(xr / 32) * 4));
    c->bytes += xr * 128 + xr * 4 + xr / 8;
  }
  {
    Scratch mx;
    MOLR_TRY(mx.alloc(4, s));
    MOLR_CUDA(cudaMemsetAsync(mx.p, 0, 4, s));
    absmax_kernel<<<c->ctx->num_sms * 8, 256, 0, s>>>(c->X * 64, c->s1_f32, mx.as<unsigned>());
    MOLR_LAUNCHED(c->ctx);
    unsigned hm = 0;
    MOLR_CUDA(cudaMemcpyAsync(&hm, mx.p, 4, cudaMemcpyDeviceToHost, s));
    MOLR_CUDA(cudaStreamSynchronize(s));
    float m;
    memcpy(&m, &hm, 4);
    if (!std::isfinite(m)) MOLR_FAIL(MOLR_ERR_INVALID, "float stage-1 view holds a non-finite value");
    c->s1_hscale = h_scale(m);
  }
  build_kernel<<<c->ctx->num_sms * 8, 256, 0, s>>>(c->X, xr, c->s1_f32, 1.f / c->s1_hscale, c->s1_bf, c->s1_bnorm);
  MOLR_LAUNCHED(c->ctx);
  chunk_max_kernel<<<div_up(xr / 32, 256), 256, 0, s>>>(xr / 32, c->s1_bnorm, c->s1_bnmax);
  MOLR_LAUNCHED(c->ctx);
  MOLR_CUDA(cudaStreamSynchronize(s));
  c->s1_bf_ready.store(1, std::memory_order_release);
  return MOLR_OK;
}

// Filter every row of an fp16 view image against B queries: cand rows (B, cap) / counts (B,)
// exactly as the fp32 filter scan would produce them (as a set).
int s1_f16_filter(molr_ctx* ctx, const F16View& V, int B, const float* q, const uint32_t* tkeys, int strict,
                  int64_t cap, int32_t* cand, int64_t* counts, cudaStream_t s, const char* timer) {
  using namespace s1bf;
  const int64_t n = V.n;
  if (n <= 0 || B <= 0) return MOLR_OK;
  const int64_t ntiles = (n + NT - 1) / NT;
  const int grid = (int)std::min<int64_t>(ntiles, ctx->num_sms);
  int64_t seg = (cap / grid) + (cap / grid) / 3 + 64;
  MOLR_CUDA(cudaFuncSetAttribute(bf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
  for (int b0 = 0; b0 < B; b0 += MAXQB * QB) {
    const int Bc = std::min(B - b0, MAXQB * QB);
    for (int attempt = 0; attempt < 2; ++attempt) {
      Scratch priv, bpriv, ccount, bcount, mx;
      Params P;
      P.view = V.h;
      P.sv = V.sv;
      P.nrm = V.nrm;
      P.cmx = V.cmx;
      P.n = n;
      P.B = Bc;
      P.q = q + int64_t(b0) * 64;
      P.tkeys = tkeys + b0;
      P.seg = seg;
      P.cap = int64_t(grid) * seg;
      MOLR_TRY(priv.alloc(size_t(Bc) * P.cap * 4, s));
      MOLR_TRY(bpriv.alloc(size_t(Bc) * P.cap * 4, s));
      MOLR_TRY(ccount.alloc(size_t(Bc) * grid * 4, s));
      MOLR_TRY(bcount.alloc(size_t(Bc) * grid * 4, s));
      MOLR_TRY(mx.alloc(4, s));
      MOLR_CUDA(cudaMemsetAsync(mx.p, 0, 4, s));
      P.cand = priv.as<int32_t>();
      P.band = bpriv.as<int32_t>();
      P.cta_counts = ccount.as<int32_t>();
      P.cta_bcounts = bcount.as<int32_t>();
      {
        KTimer t(ctx, timer, s, double(Bc) * n);
        if (Bc <= 32 && !dev_knob("MOLR_S1_NO_SMALL")) {  // items-in-M variant for small batches
          auto kern = Bc <= 16 ? bf_small_kernel<16> : bf_small_kernel<32>;
          MOLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SS_SMEM));
          kern<<<grid, NTHREADS, SS_SMEM, s>>>(P);
        } else {
          bf_kernel<<<grid, NTHREADS, SMEM_BYTES, s>>>(P);
        }
        MOLR_LAUNCHED(ctx);
        s1tc::compact_segments_kernel<<<dim3(Bc, s1tc::compact_split(ctx, Bc, grid)), 256, 0, s>>>(
            grid, seg, P.cap, P.cand, P.cta_counts, cap, cand + int64_t(b0) * cap, counts + b0, mx.as<int>());
        MOLR_LAUNCHED(ctx);
        seg_max_kernel<<<div_up(int64_t(Bc) * grid, 256), 256, 0, s>>>(int64_t(Bc) * grid, P.cta_bcounts,
                                                                        mx.as<int>());
        MOLR_LAUNCHED(ctx);
      }
      int hmx = 0;
      MOLR_CUDA(cudaMemcpyAsync(&hmx, mx.p, 4, cudaMemcpyDeviceToHost, s));
      MOLR_CUDA(cudaStreamSynchronize(s));
      if (hmx > seg && attempt == 0) {
        seg = hmx;  // a private segment overflowed: rerun with the exact maximum
        continue;
      }
      const dim3 rg(Bc, std::max(1, std::min(grid, (4 * ctx->num_sms + Bc - 1) / Bc)));
      KTimer t(ctx, "stage1_band_recheck", s, double(Bc));
      recheck_band_kernel<<<rg, 256, 0, s>>>(grid, seg, P.cap, P.band, P.cta_bcounts, V.f32, P.q, P.tkeys, strict,
                                             cap, cand + int64_t(b0) * cap, counts + b0);
      MOLR_LAUNCHED(ctx);
      break;
    }
  }
  return MOLR_OK;
}

int s1_bf_scan(molr_ctx* ctx, const molr_cache* cc, int B, const float* q, const uint32_t* tkeys, int strict,
               int64_t cap, int32_t* cand, int64_t* counts, cudaStream_t s) {
  molr_cache* c = const_cast<molr_cache*>(cc);
  MOLR_TRY(s1_bf_build(c, s));
  F16View V{c->s1_bf, c->s1_bnorm, c->s1_bnmax, c->s1_hscale, c->s1_f32, c->X};
  return s1_f16_filter(ctx, V, B, q, tkeys, strict, cap, cand, counts, s, "stage1_filter_f16");
}

// fp16 image of `n` gathered fp32 rows (the sampled rows of the float view), at the view's scale
int s1_f16_image(molr_ctx* ctx, const molr_cache* cc, const int64_t* rows, int64_t n, Scratch& f32, Scratch& h,
                 Scratch& nrm, Scratch& cmx, F16View* out, cudaStream_t s) {
  using namespace s1bf;
  molr_cache* c = const_cast<molr_cache*>(cc);
  MOLR_TRY(s1_bf_build(c, s));  // (the view's scale)
  const int64_t np = (n + NT - 1) / NT * NT;
  MOLR_TRY(f32.alloc(size_t(np) * 256, s));
  MOLR_TRY(h.alloc(size_t(np) * 128, s));
  MOLR_TRY(nrm.alloc(size_t(np) * 4, s));
  MOLR_TRY(cmx.alloc(size_t(np / 32) * 4, s));
  gather_f32_rows_kernel<<<ctx->num_sms * 8, 256, 0, s>>>(n, np, c->s1_f32, rows, f32.as<float>());
  MOLR_LAUNCHED(ctx);
  build_kernel<<<ctx->num_sms * 8, 256, 0, s>>>(n, np, f32.as<float>(), 1.f / c->s1_hscale, h.as<__half>(),
                                                nrm.as<float>());
  MOLR_LAUNCHED(ctx);
  chunk_max_kernel<<<div_up(np / 32, 256), 256, 0, s>>>(np / 32, nrm.as<float>(), cmx.as<float>());
  MOLR_LAUNCHED(ctx);
  *out = F16View{h.as<__half>(), nrm.as<float>(), cmx.as<float>(), c->s1_hscale, f32.as<float>(), n};
  return MOLR_OK;
}

// keys[b, j] = f32_key(exact fp32 score of row rows_f32[ids[b, j]]) for the j < min(counts[b], cap)
__global__ void passer_keys_kernel(int B, int64_t cap, const int32_t* __restrict__ ids, const int64_t* __restrict__ counts,
                                   const float* __restrict__ vf, const float* __restrict__ qf, uint32_t* __restrict__ keys) {
  __shared__ __align__(16) float sq[64];
  const int b = blockIdx.x;
  if (threadIdx.x < 64) sq[threadIdx.x] = qf[int64_t(b) * 64 + threadIdx.x];
  __syncthreads();
  const int64_t n = imin64(counts[b], cap);
  for (int64_t i = blockIdx.y * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.y * blockDim.x) {
    const float4* v4 = reinterpret_cast<const float4*>(vf + int64_t(ids[int64_t(b) * cap + i]) * 64);
    float v[64];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float4 x = __ldg(v4 + k);
      v[4 * k] = x.x, v[4 * k + 1] = x.y, v[4 * k + 2] = x.z, v[4 * k + 3] = x.w;
    }
    keys[int64_t(b) * cap + i] = f32_key(s1_dot64(v, sq));
  }
}

int s1_passer_keys(molr_ctx* ctx, int B, int64_t cap, const int32_t* ids, const int64_t* counts, const float* vf,
                   const float* q, uint32_t* keys, cudaStream_t s) {
  if (B <= 0) return MOLR_OK;
  passer_keys_kernel<<<dim3(B, std::max(1, std::min(8, (2 * ctx->num_sms + B - 1) / B))), 256, 0, s>>>(
      B, cap, ids, counts, vf, q, keys);
  MOLR_LAUNCHED(ctx);
  return MOLR_OK;
}

}  // namespace molr
