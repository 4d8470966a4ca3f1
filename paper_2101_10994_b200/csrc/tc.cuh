// 5th-generation tensor cores (tcgen05) for the per-LOD decoder MLP.
//
// The hidden layer of a 128-point tile is one GEMM: H[128 x 128] =
// A[128 x 48] * B[48 x 128], A row m = (x, z_L, 1, 0...) of point m, B
// column j = (W1[j, :], b1[j], 0...) of hidden unit j. fp32 inputs are
// split into bf16 hi + lo parts and the product is taken as
// Ah*Bh + Ah*Bl + Al*Bh ("bf16x3"): ~2^-16 relative error per term, well
// inside the 1e-4 SDF tolerance, at the bf16 tensor rate. One thread issues
// the 9 tcgen05.mma (3 K-steps of 16 x 3 products) into a TMEM accumulator;
// each thread then reads its point's 128 hidden values back with
// tcgen05.ld and finishes relu . W2 + b2 in registers.
//
// Operands use the no-swizzle K-major canonical layout: 8-row x 16-byte core
// matrices, K-chunks 128 B apart (LBO), 8-row groups 768 B apart (SBO).
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"

namespace ng {
namespace tc {

constexpr int M = 128;          // points per tile (TMEM lanes)
constexpr int N = 128;          // hidden units (TMEM columns)
constexpr int K = 48;           // 3 x + 32 z + bias + 12 zero pad
constexpr int KSTEP = 16;       // bf16 MMA K
constexpr int CHUNKS = K / 8;   // 16-byte (8 x bf16) K-chunks per row
constexpr int LBO = 128;        // bytes between K-chunks of a core-matrix column
constexpr int SBO = CHUNKS * 128;   // bytes between 8-row groups
constexpr int TILE_BYTES = M * K * 2;   // one bf16 operand tile (A or B): 12 KiB

// Byte offset of element (row, k) in a tile.
__device__ __forceinline__ int tile_off(int row, int k) {
  return (row >> 3) * SBO + (k >> 3) * LBO + (row & 7) * 16 + (k & 7) * 2;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// Shared-memory matrix descriptor (SWIZZLE_NONE, K-major, sm_100 version 1).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((LBO >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((SBO >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version for tcgen05
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

// Instruction descriptor: kind::f16, A = B = bf16, D = f32, K-major both,
// N = 128, M = 128.
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                           ((uint32_t)(M >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(IDESC), "r"(accumulate));
}

__device__ __forceinline__ void commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(mbar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(mbar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// TMEM allocation (one warp; result written to shared memory).
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_free(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// 32 consecutive fp32 columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// bf16 hi / lo split of an fp32 value.
__device__ __forceinline__ void split_bf16(float a, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(a);
  lo = __float2bfloat16_rn(a - __bfloat162float(hi));
}

// Operand column layout (K = 48): x0 x1 x2 | bias input | 0 0 0 0 |
// z0..z31 | 0 x 8. z starts on a 16-byte chunk, so 4 consecutive channels
// are one 8-byte store of a row (the presummed gather writes z this way).
constexpr int KZ = 8;  // first z column
__device__ __forceinline__ int input_of_column(int k) {  // index into [x(3), z(32), 1] or -1 (zero)
  return k < 3 ? k : (k == 3 ? 35 : (k >= KZ && k < KZ + 32 ? 3 + (k - KZ) : -1));
}

// Write one operand row (48 values) as hi / lo tiles from v36 = [x, z, 1].
__device__ __forceinline__ void write_row(uint8_t* hi_tile, uint8_t* lo_tile, int row, const float* v36) {
#pragma unroll
  for (int c = 0; c < CHUNKS; ++c) {
    __align__(16) __nv_bfloat16 h[8], l[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int src = input_of_column(c * 8 + j);
      const float a = src >= 0 ? v36[src] : 0.f;
      split_bf16(a, h[j], l[j]);
    }
    const int off = tile_off(row, c * 8);
    *reinterpret_cast<uint4*>(hi_tile + off) = *reinterpret_cast<const uint4*>(h);
    *reinterpret_cast<uint4*>(lo_tile + off) = *reinterpret_cast<const uint4*>(l);
  }
}

// Issue H = A*B (bf16x3) into TMEM columns [tmem, tmem+128); one thread.
__device__ __forceinline__ void issue_gemm(uint32_t tmem, uint32_t a_hi, uint32_t a_lo, uint32_t b_hi,
                                           uint32_t b_lo, uint64_t* mbar) {
  fence_after_sync();
#pragma unroll
  for (int s = 0; s < K / KSTEP; ++s) {
    const uint32_t koff = s * 2 * LBO;  // 16 bf16 = two 16-byte chunks
    mma_bf16(tmem, smem_desc(a_hi + koff), smem_desc(b_hi + koff), s > 0);
    mma_bf16(tmem, smem_desc(a_hi + koff), smem_desc(b_lo + koff), 1);
    mma_bf16(tmem, smem_desc(a_lo + koff), smem_desc(b_hi + koff), 1);
  }
  commit(mbar);
}

}  // namespace tc
}  // namespace ng
