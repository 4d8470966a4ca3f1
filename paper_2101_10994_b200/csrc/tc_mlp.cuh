// Tensor-core decoder policy shared by the query, march and normals kernels.
#pragma once

#include "eval.cuh"
#include "tc.cuh"

namespace ng {

// NG_RESTAGE_ASYNC=0: the per-level decoder restage as a load-store loop (A/B builds)
#ifndef NG_RESTAGE_ASYNC
#define NG_RESTAGE_ASYNC 1
#endif

constexpr int DEC_TC_BYTES = 2 * tc::TILE_BYTES + 128 * 4 + 128;  // B_hi, B_lo, W2[128], b2 (+pad)

struct TcMlp {
  uint8_t* a_hi;
  uint8_t* a_lo;
  const uint8_t* dec_tiles;  // DEC_TC_BYTES per decoder, level dec_first first
  int dec_first;
  uint32_t tmem;
  uint64_t* mbar;
  uint32_t* phase;
  int wg;
  int bar_id;
  unsigned long long* prof = nullptr;  // NG_PROFILE: [6] += cycles at the group barrier, [7] += cycles GEMM + epilogue
  // one-level staging (k_query_tc): the CTA holds a single decoder's tiles
  // and re-stages level l from these fp32 decoders before its GEMMs
  const float* restage_src = nullptr;
  int restage_stride = 0;
  const uint8_t* restage_tiles = nullptr;  // or pre-converted tiles (DEC_TC_BYTES per level, dec_first first)

  __device__ __forceinline__ void prepare(int l) const;

  // The presummed gather writes z straight into the operand rows (lane =
  // channel quad), and the decoder then adds only x and the bias input.
  static constexpr bool kDirectZ = true;
  __device__ __forceinline__ void put_z4(int p, int sub, const float* acc) const {
    __align__(8) __nv_bfloat16 h[4], l4[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) tc::split_bf16(acc[e], h[e], l4[e]);
    const int off = tc::tile_off(32 * wg + p, tc::KZ + 4 * sub);
    *reinterpret_cast<uint2*>(a_hi + off) = *reinterpret_cast<const uint2*>(h);
    *reinterpret_cast<uint2*>(a_lo + off) = *reinterpret_cast<const uint2*>(l4);
  }
  __device__ __forceinline__ float decode_direct(int l, const float xf[3], bool& bad) const;

  __device__ __forceinline__ float operator()(int l, const float xf[3], const float* zrow, bool /*any*/,
                                              bool& bad) const {
#ifdef NG_PROFILE
    const long long t_in = clock64();
#endif
    const int lane = (int)lane_id();
    const int row = 32 * wg + lane;
    float v[36];
    v[0] = xf[0];
    v[1] = xf[1];
    v[2] = xf[2];
    load_zrow(zrow, v + 3);
    v[35] = 1.0f;  // bias input: B row 35 holds b1
    float chk = 0.f;
#pragma unroll
    for (int k = 0; k < 35; ++k) chk += v[k] - v[k];
    bad = !(chk == 0.f);
    tc::write_row(a_hi, a_lo, row, v);
    tc::fence_proxy_async();
    tc::fence_before_sync();
    tc::named_sync(bar_id, 128);
    const uint8_t* dt = dec_tiles + (restage_src ? (size_t)0 : (size_t)(l - dec_first) * DEC_TC_BYTES);
    if (wg == 0 && lane == 0)
      tc::issue_gemm(tmem, tc::smem_u32(a_hi), tc::smem_u32(a_lo), tc::smem_u32(dt), tc::smem_u32(dt + tc::TILE_BYTES),
                     mbar);
    tc::mbar_wait(mbar, *phase & 1u);
    *phase += 1;
    tc::fence_after_sync();
    const float* W2 = reinterpret_cast<const float*>(dt + 2 * tc::TILE_BYTES);
    float acc = W2[128];  // b2
    const uint32_t taddr = tmem + ((uint32_t)(32 * wg) << 16);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float h[32];
      tc::tmem_ld32(taddr + 32 * c, h);
#pragma unroll
      for (int i = 0; i < 32; ++i) acc = fmaf(W2[32 * c + i], fmaxf(h[i], 0.f), acc);
    }
    tc::fence_before_sync();
#ifdef NG_PROFILE
    if (prof && lane_id() == 0) prof[7] += (unsigned long long)(clock64() - t_in);
#endif
    return acc;
  }
};

__device__ __forceinline__ float TcMlp::decode_direct(int l, const float xf[3], bool& bad) const {
  const int lane = (int)lane_id();
  const int row = 32 * wg + lane;
  bad = !(isfinite(xf[0]) && isfinite(xf[1]) && isfinite(xf[2]));
  // chunk 0: x, the bias input, zeros; chunk 5: zeros (z is chunks 1-4)
  {
    const float c0[8] = {xf[0], xf[1], xf[2], 1.f, 0.f, 0.f, 0.f, 0.f};
    __align__(16) __nv_bfloat16 h[8], lo[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) tc::split_bf16(c0[j], h[j], lo[j]);
    const int off0 = tc::tile_off(row, 0), off5 = tc::tile_off(row, 40);
    *reinterpret_cast<uint4*>(a_hi + off0) = *reinterpret_cast<const uint4*>(h);
    *reinterpret_cast<uint4*>(a_lo + off0) = *reinterpret_cast<const uint4*>(lo);
    *reinterpret_cast<uint4*>(a_hi + off5) = make_uint4(0, 0, 0, 0);
    *reinterpret_cast<uint4*>(a_lo + off5) = make_uint4(0, 0, 0, 0);
  }
  tc::fence_proxy_async();
  tc::fence_before_sync();
#ifdef NG_PROFILE
  const long long t0 = clock64();
#endif
  tc::named_sync(bar_id, 128);
#ifdef NG_PROFILE
  const long long t1 = clock64();
#endif
  const uint8_t* dt = dec_tiles + (restage_src ? (size_t)0 : (size_t)(l - dec_first) * DEC_TC_BYTES);
  if (wg == 0 && lane == 0)
    tc::issue_gemm(tmem, tc::smem_u32(a_hi), tc::smem_u32(a_lo), tc::smem_u32(dt), tc::smem_u32(dt + tc::TILE_BYTES),
                   mbar);
  tc::mbar_wait(mbar, *phase & 1u);
  *phase += 1;
  tc::fence_after_sync();
  const float* W2 = reinterpret_cast<const float*>(dt + 2 * tc::TILE_BYTES);
  float acc = W2[128];  // b2
  const uint32_t taddr = tmem + ((uint32_t)(32 * wg) << 16);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    float hh[32];
    tc::tmem_ld32(taddr + 32 * c, hh);
#pragma unroll
    for (int i = 0; i < 32; ++i) acc = fmaf(W2[32 * c + i], fmaxf(hh[i], 0.f), acc);
  }
  tc::fence_before_sync();
#ifdef NG_PROFILE
  if (prof && lane == 0) {
    prof[6] += (unsigned long long)(t1 - t0);
    prof[7] += (unsigned long long)(clock64() - t1);
  }
#endif
  return acc;
}

// Convert packed fp32 decoders (ng_field layout) into bf16 hi/lo B tiles.
__device__ __forceinline__ void stage_decoder_tiles(uint8_t* dst, const float* __restrict__ src, int first, int last, int stride) {
  const int ndec = last - first + 1;
  for (int idx = threadIdx.x; idx < ndec * 128 * tc::CHUNKS; idx += blockDim.x) {
    const int d = idx / (128 * tc::CHUNKS);
    const int j = (idx / tc::CHUNKS) % 128;
    const int c = idx % tc::CHUNKS;
    const float* row = src + (size_t)(first - 1 + d) * stride + (size_t)j * NG_W1_STRIDE;
    __align__(16) __nv_bfloat16 h[8], lo[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int src = tc::input_of_column(c * 8 + q);  // W1b row = [x weights, z weights, b1]
      tc::split_bf16(src >= 0 ? __ldg(row + src) : 0.f, h[q], lo[q]);
    }
    uint8_t* t = dst + (size_t)d * DEC_TC_BYTES;
    const int off = tc::tile_off(j, c * 8);
    *reinterpret_cast<uint4*>(t + off) = *reinterpret_cast<const uint4*>(h);
    *reinterpret_cast<uint4*>(t + tc::TILE_BYTES + off) = *reinterpret_cast<const uint4*>(lo);
  }
  for (int idx = threadIdx.x; idx < ndec * 129; idx += blockDim.x) {
    const int d = idx / 129, j = idx % 129;
    const float* w2 = src + (size_t)(first - 1 + d) * stride + 128 * NG_W1_STRIDE;
    reinterpret_cast<float*>(dst + (size_t)d * DEC_TC_BYTES + 2 * tc::TILE_BYTES)[j] = __ldg(w2 + j);
  }
}


__device__ __forceinline__ void TcMlp::prepare(int l) const {
  if (!restage_src) return;
  // every group's previous GEMM has completed (each thread waited on its
  // mbarrier before leaving the decoder), so the tiles can be replaced
  tc::fence_before_sync();
  __syncthreads();
  if (restage_tiles) {  // a plain copy of the pre-converted tiles
    // as asynchronous 16-byte copies, all of a thread's in flight at once
    // (a load-store loop kept one load in flight per thread: ~4 dependent
    // L2 round trips per level with the whole CTA waiting), no registers held
    const uint4* src4 = reinterpret_cast<const uint4*>(restage_tiles + (size_t)(l - dec_first) * DEC_TC_BYTES);
    uint4* dst4 = reinterpret_cast<uint4*>(const_cast<uint8_t*>(dec_tiles));
#if NG_RESTAGE_ASYNC
    for (int i = threadIdx.x; i < DEC_TC_BYTES / 16; i += blockDim.x) cp_async16(dst4 + i, src4 + i);
    cp_async_commit();
    cp_async_wait_all();
#else
    for (int i = threadIdx.x; i < DEC_TC_BYTES / 16; i += blockDim.x) dst4[i] = __ldg(src4 + i);
#endif
  } else {
    stage_decoder_tiles(const_cast<uint8_t*>(dec_tiles), restage_src, l, l, restage_stride);
  }
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
}

// Shared-memory carve-up for a kernel with `groups` 4-warp tile groups.
struct TcSmem {
  uint8_t* dec_tiles;
  uint8_t* a_tiles;
  WarpScratch* ws;
  size_t ws_stride;  // bytes per warp's scratch
  uint64_t* mbar;
  uint32_t* tmem_slot;
  __device__ __forceinline__ WarpScratch& scratch(int w) const {
    return *reinterpret_cast<WarpScratch*>(reinterpret_cast<uint8_t*>(ws) + (size_t)w * ws_stride);
  }
};

// A kernel whose decoder takes z straight into the operand rows (the
// presummed path) never touches WarpScratch::zt: its warps get only the
// ids and weights, which frees shared memory for a fourth group with two
// decoders (the LOD blend) and for L1.
constexpr size_t WS_COMPACT_BYTES = offsetof(WarpScratch, zt);
static_assert(WS_COMPACT_BYTES % 16 == 0, "compact scratch keeps 16-byte alignment");

__host__ __device__ constexpr size_t tc_smem_bytes(int ndec, int groups, size_t ws_bytes = sizeof(WarpScratch)) {
  return (size_t)ndec * DEC_TC_BYTES + (size_t)groups * 2 * tc::TILE_BYTES + (size_t)groups * 4 * ws_bytes +
         (size_t)groups * 8 + 16;
}

__device__ __forceinline__ TcSmem tc_carve(uint8_t* smem, int ndec, int groups, size_t ws_bytes = sizeof(WarpScratch)) {
  TcSmem t;
  t.dec_tiles = smem;
  t.a_tiles = t.dec_tiles + (size_t)ndec * DEC_TC_BYTES;
  t.ws = reinterpret_cast<WarpScratch*>(t.a_tiles + (size_t)groups * 2 * tc::TILE_BYTES);
  t.ws_stride = ws_bytes;
  t.mbar = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(t.ws) + (size_t)groups * 4 * ws_bytes);
  t.tmem_slot = reinterpret_cast<uint32_t*>(t.mbar + groups);
  return t;
}

// TMEM allocations are powers of two >= 32 columns.
__host__ __device__ constexpr uint32_t tmem_cols(int groups) {
  return groups <= 1 ? 128u : (groups <= 2 ? 256u : 512u);
}

// CTA prologue: TMEM (128 columns per group), mbarriers, decoder B tiles.
__device__ __forceinline__ uint32_t tc_setup(const TcSmem& t, const float* decoders, int first, int last, int stride,
                                             int groups) {
  if ((threadIdx.x >> 5) == 0) tc::tmem_alloc(t.tmem_slot, tmem_cols(groups));
  if (threadIdx.x == 0)
    for (int i = 0; i < groups; ++i) tc::mbar_init(t.mbar + i, 1);
  stage_decoder_tiles(t.dec_tiles, decoders, first, last, stride);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  return *t.tmem_slot;
}

__device__ __forceinline__ void tc_teardown(uint32_t tmem_base, int groups) {
  tc::fence_before_sync();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) {
    tc::fence_after_sync();
    tc::tmem_free(tmem_base, tmem_cols(groups));
  }
}

__device__ __forceinline__ TcMlp tc_policy(const TcSmem& t, uint32_t tmem_base, int dec_first, uint32_t* phase) {
  const int w = threadIdx.x >> 5, g = w / 4;
  TcMlp m;
  m.a_hi = t.a_tiles + (size_t)g * 2 * tc::TILE_BYTES;
  m.a_lo = m.a_hi + tc::TILE_BYTES;
  m.dec_tiles = t.dec_tiles;
  m.dec_first = dec_first;
  m.tmem = tmem_base + 128 * g;
  m.mbar = t.mbar + g;
  m.phase = phase;
  m.wg = w % 4;
  m.bar_id = 1 + g;
  return m;
}

}  // namespace ng
