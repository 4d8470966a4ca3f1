// Batched SDF query with the decoder on the 5th-gen tensor cores (tc.cuh).
//
// CTA = 8 warps = 2 tile groups of 4 warps; a group owns a 128-point tile,
// a 128-column TMEM accumulator, an A operand tile pair and an mbarrier.
// Warps gather their 32 points' features channel-parallel exactly as the
// SIMT path (eval.cuh); at each output level the group writes its A rows,
// one thread issues the bf16x3 GEMM, and every thread reads its point's
// hidden row from TMEM for the relu . W2 epilogue. All requested decoders'
// B tiles stay resident in shared memory for the CTA's lifetime.
#include "eval.cuh"
#include "tc.cuh"

#include <algorithm>
#include <cstdlib>

namespace ng {

int grid_for(int64_t n, int nt);

constexpr int TQ_GROUPS = 2;
constexpr int TQ_NW = 4 * TQ_GROUPS;
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

  __device__ __forceinline__ float operator()(int l, const float xf[3], const float* zrow, bool /*any*/,
                                              bool& bad) const {
    const int lane = (int)lane_id();
    const int row = 32 * wg + lane;
    float v[36];
    v[0] = xf[0];
    v[1] = xf[1];
    v[2] = xf[2];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[3 + k] = zrow[k];
    v[35] = 1.0f;  // bias input: B row 35 holds b1
    float chk = 0.f;
#pragma unroll
    for (int k = 0; k < 35; ++k) chk += v[k] - v[k];
    bad = !(chk == 0.f);
    tc::write_row(a_hi, a_lo, row, v);
    tc::fence_proxy_async();
    tc::fence_before_sync();
    tc::named_sync(bar_id, 128);
    const uint8_t* dt = dec_tiles + (size_t)(l - dec_first) * DEC_TC_BYTES;
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
    return acc;
  }
};

// Convert packed fp32 decoders (ng_field layout) into bf16 hi/lo B tiles.
__device__ void stage_decoder_tiles(uint8_t* dst, const float* __restrict__ src, int first, int last, int stride) {
  const int ndec = last - first + 1;
  for (int idx = threadIdx.x; idx < ndec * 128 * tc::CHUNKS; idx += blockDim.x) {
    const int d = idx / (128 * tc::CHUNKS);
    const int j = (idx / tc::CHUNKS) % 128;
    const int c = idx % tc::CHUNKS;
    const float* row = src + (size_t)(first - 1 + d) * stride + (size_t)j * NG_W1_STRIDE;
    __align__(16) __nv_bfloat16 h[8], lo[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int k = c * 8 + q;
      tc::split_bf16(k < NG_W1_STRIDE ? __ldg(row + k) : 0.f, h[q], lo[q]);
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

__global__ void __launch_bounds__(TQ_NW * 32, 1) k_query_tc(const __grid_constant__ ng_octree tree, ng_field f,
                                                            ng_query_args a, int G, int out_mask, int dec_first,
                                                            int dec_last, const double* __restrict__ pts, int64_t n,
                                                            double* __restrict__ out, int ncols,
                                                            ng_counters* counters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int ndec = dec_last - dec_first + 1;
  uint8_t* dec_tiles = smem;
  uint8_t* a_tiles = dec_tiles + (size_t)ndec * DEC_TC_BYTES;            // per group: A_hi, A_lo
  WarpScratch* wsa = reinterpret_cast<WarpScratch*>(a_tiles + TQ_GROUPS * 2 * tc::TILE_BYTES);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(wsa + TQ_NW);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + TQ_GROUPS);

  const int w = threadIdx.x >> 5;
  const int g = w / 4, wg = w % 4;
  if (w == 0) tc::tmem_alloc(tmem_slot, 128 * TQ_GROUPS);
  if (threadIdx.x == 0) {
    for (int i = 0; i < TQ_GROUPS; ++i) tc::mbar_init(mbar + i, 1);
  }
  stage_decoder_tiles(dec_tiles, f.decoders, dec_first, dec_last, f.dec_stride);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem_base = *tmem_slot;

  uint32_t phase = 0;
  TcMlp mlp;
  mlp.a_hi = a_tiles + (size_t)g * 2 * tc::TILE_BYTES;
  mlp.a_lo = mlp.a_hi + tc::TILE_BYTES;
  mlp.dec_tiles = dec_tiles;
  mlp.dec_first = dec_first;
  mlp.tmem = tmem_base + 128 * g;
  mlp.mbar = mbar + g;
  mlp.phase = &phase;
  mlp.wg = wg;
  mlp.bar_id = 1 + g;

  EvalCtx c;
  c.Z = f.Z;
  c.dec = nullptr;
  c.dec_first = dec_first;
  c.dec_stride = f.dec_stride;
  c.h = f.h;
  c.gather_level = G;
  c.inside_level = a.inside_level;
  c.out_mask = out_mask;
  WarpScratch& ws = wsa[w];
  const bool blending = a.blend_base > 0;
  const double alpha = a.blend_alpha;
  LaneCounters lc;
  const int64_t n_tiles = (n + 127) / 128;
  for (int64_t tile = (int64_t)blockIdx.x * TQ_GROUPS + g; tile < n_tiles; tile += (int64_t)gridDim.x * TQ_GROUPS) {
    const int64_t i = tile * 128 + 32 * wg + lane_id();
    const bool act = i < n;
    double x[3] = {0.0, 0.0, 0.0};
    if (act) {
      x[0] = pts[3 * i];
      x[1] = pts[3 * i + 1];
      x[2] = pts[3 * i + 2];
    }
    int col = 0;
    double lo_v = 0.0, hi_v = 0.0;
    EvalLane r = warp_eval(tree, c, ws, act, x, mlp, [&](int L, float d, bool bad, const EvalLane& er) {
      if (act) {
        double v;
        if (!er.inside) {
          v = empty_value(tree, x);
        } else if (er.present & ((1u << L) - 1u)) {
          v = (double)d;
          lc.evals += 1;
          if (!((er.present >> (L - 1)) & 1u)) lc.missing += 1;
          if (bad) lc.nonfinite += 1;
        } else {
          v = empty_value(tree, x);
          lc.empty += 1;
        }
        if (blending) {
          if (L == a.blend_base) lo_v = v; else hi_v = v;
        } else {
          out[i * ncols + col] = v;
        }
      }
      ++col;
    });
    if (act) {
      if (!r.inside) lc.empty += 1;
      if (blending)
        out[i] = r.inside ? dadd(dmul(dsub(1.0, alpha), lo_v), dmul(alpha, hi_v)) : empty_value(tree, x);
    }
  }
  lc.flush(counters);
  tc::fence_before_sync();
  __syncthreads();
  if (w == 0) {
    tc::fence_after_sync();
    tc::tmem_free(tmem_base, 128 * TQ_GROUPS);
  }
}

size_t query_tc_smem_bytes(int ndec) {
  return (size_t)ndec * DEC_TC_BYTES + TQ_GROUPS * 2 * tc::TILE_BYTES + TQ_NW * sizeof(WarpScratch) +
         TQ_GROUPS * 8 + 16;
}

// Returns NG_ERR_CAPACITY when the tensor-core path cannot take the query
// (hidden width != 128 or too many decoders for shared memory).
int run_query_tc(const ng_octree& tree, const ng_field& f, const ng_query_args& a, int G, int out_mask,
                 int dec_first, int dec_last, int ncols, const double* pts, int64_t n, double* out,
                 ng_counters* counters, cudaStream_t s) {
  if (f.h != tc::N) return NG_ERR_CAPACITY;
  const size_t smem = query_tc_smem_bytes(dec_last - dec_first + 1);
  if (smem > 227 * 1024) return NG_ERR_CAPACITY;
  static size_t configured = 0;
  if (smem > configured) {
    int r = cuda_status(cudaFuncSetAttribute(k_query_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                        "k_query_tc smem attribute");
    if (r) return r;
    configured = smem;
  }
  const int64_t tiles = (n + 127) / 128;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((tiles + TQ_GROUPS - 1) / TQ_GROUPS, sm_count()));
  k_query_tc<<<(int)grid, TQ_NW * 32, smem, s>>>(tree, f, a, G, out_mask, dec_first, dec_last, pts, n, out, ncols,
                                                 counters);
  NG_CHECK_LAUNCH("k_query_tc");
  return NG_OK;
}

}  // namespace ng
