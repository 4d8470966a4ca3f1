// Batched SDF query with the decoder on the 5th-gen tensor cores (tc.cuh).
//
// CTA = 8 warps = 2 tile groups of 4 warps; a group owns a 128-point tile,
// a 128-column TMEM accumulator, an A operand tile pair and an mbarrier.
// Warps gather their 32 points' features channel-parallel exactly as the
// SIMT path (eval.cuh); at each output level the group writes its A rows,
// one thread issues the bf16x3 GEMM, and every thread reads its point's
// hidden row from TMEM for the relu . W2 epilogue. All requested decoders'
// B tiles stay resident in shared memory for the CTA's lifetime.
// Points per gather batch: 8 measured faster than 4 when the decoder
// restage and the corner sums cost more (1264 vs 1206 Mpoints/s); after
// those changes 4 is as fast or slightly faster (10.74 vs 10.77 ms,
// profiles/r02_final/gather_batch_ab.log) with fewer registers in flight.
#ifndef NG_GATHER_BATCH
#define NG_GATHER_BATCH 4
#endif
#include "tc_mlp.cuh"

#include <algorithm>
#include <cstdlib>

namespace ng {

int grid_for(int64_t n, int nt);

// 4 groups (16 warps) per CTA: the CTA holds one decoder level at a time and
// re-stages it per level (all groups step through the levels together), so
// the five decoders' tiles do not cap the CTA at 2 groups
#ifndef NG_TQ_GROUPS
#define NG_TQ_GROUPS 4
#endif
constexpr int TQ_GROUPS = NG_TQ_GROUPS;
// tiles claimed from a counter (1) or strided over the grid (0)
#ifndef NG_QUERY_DYNAMIC
#define NG_QUERY_DYNAMIC 1
#endif
constexpr int TQ_NW = 4 * TQ_GROUPS;

__global__ void __launch_bounds__(TQ_NW * 32, 1) k_query_tc(const __grid_constant__ ng_octree tree, ng_field f,
                                                            ng_query_args a, int G, int out_mask, int dec_first,
                                                            int dec_last, const double* __restrict__ pts, int64_t n,
                                                            double* __restrict__ out, int ncols,
                                                            ng_counters* counters, const uint8_t* tiles,
                                                            unsigned int* claim) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const TcSmem t = tc_carve(smem, 1, TQ_GROUPS);
  const int w = threadIdx.x >> 5;
  const int g = w / 4, wg = w % 4;
  const uint32_t tmem_base = tc_setup(t, f.decoders, dec_first, dec_first, f.dec_stride, TQ_GROUPS);
  uint32_t phase = 0;
  TcMlp mlp = tc_policy(t, tmem_base, dec_first, &phase);
  mlp.restage_src = f.decoders;
  mlp.restage_stride = f.dec_stride;
  mlp.restage_tiles = tiles;

  EvalCtx c;
  c.Z = f.Z;
  c.dec = nullptr;
  c.dec_first = dec_first;
  c.dec_stride = f.dec_stride;
  c.h = f.h;
  c.gather_level = G;
  c.inside_level = a.inside_level;
  c.out_mask = out_mask;
  WarpScratch& ws = t.ws[w];
  const bool blending = a.blend_base > 0;
  const double alpha = a.blend_alpha;
  LaneCounters lc;
  const int64_t n_tiles = (n + 127) / 128;
  // the CTA's groups take tiles together (the level restaging is CTA-wide),
  // claimed from a counter so a slow SM does not hold up the query's end
#if NG_QUERY_DYNAMIC
  __shared__ int64_t s_tb;
  while (true) {
    if (threadIdx.x == 0) s_tb = (int64_t)atomicAdd(claim, 1u) * TQ_GROUPS;
    __syncthreads();
    const int64_t tb = s_tb;
    __syncthreads();
    if (tb >= n_tiles) break;
#else
  for (int64_t tb = (int64_t)blockIdx.x * TQ_GROUPS; tb < n_tiles; tb += (int64_t)gridDim.x * TQ_GROUPS) {
#endif
    const int64_t tile = tb + g;
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
  tc_teardown(tmem_base, TQ_GROUPS);
}

size_t query_tc_smem_bytes(int) { return tc_smem_bytes(1, TQ_GROUPS); }

// The requested decoders as bf16 hi / lo B tiles (+ W2, b2), converted once
// per query so each CTA's per-level restage is a plain copy.
__global__ void k_query_tiles(ng_field f, int dec_first, int dec_last, uint8_t* tiles, unsigned int* claim) {
  if (threadIdx.x == 0) *claim = 0u;  // k_query_tc's tile counter
  stage_decoder_tiles(tiles, f.decoders, dec_first, dec_last, f.dec_stride);
}

// Returns NG_ERR_CAPACITY when the tensor-core path cannot take the query
// (hidden width != 128 or too many decoders for shared memory).
int run_query_tc(const ng_octree& tree, const ng_field& f, const ng_query_args& a, int G, int out_mask,
                 int dec_first, int dec_last, int ncols, const double* pts, int64_t n, double* out,
                 ng_counters* counters, cudaStream_t s) {
  if (f.h != tc::N) return NG_ERR_CAPACITY;
  const size_t smem = query_tc_smem_bytes(dec_last - dec_first + 1);
  if (smem > 227 * 1024) return NG_ERR_CAPACITY;
  if (int r = set_smem_limit((const void*)k_query_tc, smem)) return r;
  const int64_t tiles = (n + 127) / 128;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((tiles + TQ_GROUPS - 1) / TQ_GROUPS, sm_count()));
  const int ndec = dec_last - dec_first + 1;
  uint8_t* dtiles = nullptr;
  int r = malloc_async((void**)&dtiles, (size_t)ndec * DEC_TC_BYTES + 256, s, "query tiles alloc");
  if (r) return r;
  unsigned int* claim = reinterpret_cast<unsigned int*>(dtiles + (size_t)ndec * DEC_TC_BYTES);
  k_query_tiles<<<1, 512, 0, s>>>(f, dec_first, dec_last, dtiles, claim);
  NG_CHECK_LAUNCH("k_query_tiles");
  k_query_tc<<<(int)grid, TQ_NW * 32, smem, s>>>(tree, f, a, G, out_mask, dec_first, dec_last, pts, n, out, ncols,
                                                 counters, dtiles, claim);
  NG_CHECK_LAUNCH("k_query_tc");
  return cuda_status(cudaFreeAsync(dtiles, s), "query tiles free");
}

}  // namespace ng
