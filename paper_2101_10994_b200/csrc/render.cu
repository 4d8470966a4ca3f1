// Frame rendering: camera rays, sparse sphere tracing with persistent-lane
// ray compaction, central-difference normals and Lambert shading
// (render.py:43-448).
//
// The march is a persistent kernel: every lane owns one ray and, the moment
// that ray terminates, pulls the next one from a global work counter, so a
// warp keeps 32 live rays until the work runs out despite per-ray iteration
// counts ranging from 1 to ~100. Each iteration is one warp-cooperative
// evaluation (eval.cuh). All control-flow arithmetic (t, clamp, stop rules)
// is fp64 in the reference's operation order; only features and the MLP are
// fp32.
#include "tc_mlp.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <unordered_map>

namespace ng {

int grid_for(int64_t n, int nt);
size_t level_scratch_bytes(int64_t max_pairs);
int traverse_hits(const ng_octree& tree, const ng_ray* rays, int t, bool next_final, const ng_pair* in,
                  const int64_t* d_count_in, int64_t in_cap, ng_pair* out_pairs, ng_hit_pair* out_hits,
                  int64_t* d_count_out, int64_t out_cap, void* scratch, size_t scratch_bytes, cudaStream_t s,
                  int64_t* seg_start, int64_t* seg_end, const double* shared_origin);
int traverse_tiles(const ng_octree& tree, const ng_ray* rays, const int64_t* d_n, int64_t n_max, int target,
                   int4* items, unsigned long long* d_active, int64_t* counts,
                   ng_hit_pair* hits, int64_t hit_cap, void* ctl, int64_t* seg_start, int64_t* seg_end,
                   void* arena, size_t arena_bytes, unsigned long long* d_need, const double* shared_origin,
                   const CamSet* cam_rays, const ng_frame* defaults, uint32_t bg, int64_t n_host,
                   void* cont, cudaStream_t s);
size_t tile_cont_bytes();
size_t tile_cont_ready_bytes();
int64_t tile_traverse_limit(size_t arena_bytes, int64_t n_max);
int64_t tile_traverse_warps(int64_t n_max);
int tile_traverse_scap();
int tile_traverse_entry_bytes();

// NG_TILE_TRAVERSE=0 selects the level-by-level traversal launches
// (k_traverse_hits) instead of the warp-per-tile kernel.
static bool use_tile_traverse(int target) {
  static const bool on = env_int("NG_TILE_TRAVERSE", 1) != 0;
  return on && target >= 1 && target <= 9;  // list cells: <= 512 per axis
}

constexpr int R_NW = 8;  // warps per CTA for march / normals

// Pixel-centre rays, bit-exact with Camera.rays (render.py:74-88), fused with
// the per-pixel output defaults and the background colour.
__global__ void k_camera_rays(const __grid_constant__ CamSet cam, ng_ray* __restrict__ rays, ng_frame fr,
                              uint8_t bg0, uint8_t bg1, uint8_t bg2, int64_t* d_root_count,
                              int64_t* __restrict__ seg_start, int64_t* __restrict__ seg_end) {
  const int64_t n = (int64_t)cam.k * cam.n_per;
  if (blockIdx.x == 0 && threadIdx.x == 0 && d_root_count) *d_root_count = n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (seg_start) {  // rays without final-level pairs keep the empty segment
      seg_start[i] = 0;
      seg_end[i] = 0;
    }
    if (rays) {
      ng_ray r;
      camera_ray(cam, i, r);
      rays[i] = r;
    }
    if (fr.hit) {
      fr.hit[i] = 0;
      fr.t[i] = __longlong_as_double(0x7ff8000000000000ll);
      fr.normal[3 * i] = 0.0;
      fr.normal[3 * i + 1] = 0.0;
      fr.normal[3 * i + 2] = 0.0;
      fr.normal_ok[i] = 0;
      fr.iterations[i] = 0;
      fr.evals[i] = 0;
      fr.color[3 * i] = bg0;
      fr.color[3 * i + 1] = bg1;
      fr.color[3 * i + 2] = bg2;
    }
  }
}

__global__ void k_set_count(int64_t* p, int64_t v) { *p = v; }

// Zero a handful of small device regions in one launch (frame statistics,
// counters, traversal look-back states, histogram buckets) instead of one
// memset per region on the frame's critical path.
struct ZeroRegions {
  void* p[6];
  size_t bytes[6];
  int n;
};

__global__ void k_zero_regions(ZeroRegions z) {
  for (int k = 0; k < z.n; ++k) {
    uint8_t* b = (uint8_t*)z.p[k];
    const size_t n16 = z.bytes[k] / 16;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
      reinterpret_cast<uint4*>(b)[i] = make_uint4(0, 0, 0, 0);
    if (blockIdx.x == 0)
      for (size_t i = n16 * 16 + threadIdx.x; i < z.bytes[k]; i += blockDim.x) b[i] = 0;
  }
}

__global__ void k_frame_defaults(ng_frame fr, int64_t n, uint8_t bg0, uint8_t bg1, uint8_t bg2,
                                 int64_t* __restrict__ seg_start, int64_t* __restrict__ seg_end) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (seg_start) {
      seg_start[i] = 0;
      seg_end[i] = 0;
    }
    fr.hit[i] = 0;
    fr.t[i] = __longlong_as_double(0x7ff8000000000000ll);
    fr.normal[3 * i] = 0.0;
    fr.normal[3 * i + 1] = 0.0;
    fr.normal[3 * i + 2] = 0.0;
    fr.normal_ok[i] = 0;
    fr.iterations[i] = 0;
    fr.evals[i] = 0;
    fr.color[3 * i] = bg0;
    fr.color[3 * i + 1] = bg1;
    fr.color[3 * i + 2] = bg2;
  }
}

// ray_segments over the final list plus the list of rays that have one.
// Longest-first work order for the march: rays with more voxels in their
// list (grazing / silhouette rays) take more sphere-trace steps, so they are
// issued first and the persistent lanes do not end on a long serial tail.
constexpr int LEN_BUCKETS = 64;

__global__ void k_len_hist(const int32_t* __restrict__ active, const unsigned long long* __restrict__ d_n,
                           const int64_t* __restrict__ seg_start, const int64_t* __restrict__ seg_end,
                           unsigned int* __restrict__ hist) {
  __shared__ unsigned int h[LEN_BUCKETS];
  for (int i = threadIdx.x; i < LEN_BUCKETS; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int64_t n = (int64_t)*d_n;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = active[k];
    const int64_t len = seg_end[r] - seg_start[r];
    atomicAdd(&h[len < LEN_BUCKETS - 1 ? len : LEN_BUCKETS - 1], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < LEN_BUCKETS; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// Active rays (a non-empty segment) and their list-length histogram, one
// thread per ray: the active list for the march and the buckets of the
// longest-first order.
__global__ void k_active_hist(const int64_t* __restrict__ seg_start, const int64_t* __restrict__ seg_end, int64_t n,
                              int32_t* __restrict__ active, unsigned long long* d_active,
                              unsigned int* __restrict__ hist) {
  // per block: bucket counts in shared memory, the block's active rays
  // compacted with one global atomic (not one per warp)
  __shared__ unsigned int h[LEN_BUCKETS];
  __shared__ unsigned int wcount[32];
  __shared__ unsigned long long block_base;
  for (int i = threadIdx.x; i < LEN_BUCKETS; i += blockDim.x) h[i] = 0;
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += stride) {
    const int64_t r = base + threadIdx.x;
    const int64_t len = r < n ? seg_end[r] - seg_start[r] : 0;
    const bool has = len > 0;
    __syncthreads();
    if (has) atomicAdd(&h[len < LEN_BUCKETS - 1 ? len : LEN_BUCKETS - 1], 1u);
    const unsigned m = __ballot_sync(FULL, has);
    if (lane_id() == 0) wcount[w] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned int tot = 0;
      for (int q = 0; q < nw; ++q) {
        const unsigned int c = wcount[q];
        wcount[q] = tot;
        tot += c;
      }
      block_base = tot ? atomicAdd(d_active, (unsigned long long)tot) : 0ull;
    }
    __syncthreads();
    if (has) active[block_base + wcount[w] + __popc(m & lanemask_lt())] = (int32_t)r;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < LEN_BUCKETS; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

__global__ void k_len_scatter(const int32_t* __restrict__ active, const unsigned long long* __restrict__ d_n,
                              const int64_t* __restrict__ seg_start, const int64_t* __restrict__ seg_end,
                              const unsigned int* __restrict__ hist, unsigned int* __restrict__ cursor,
                              int32_t* __restrict__ sorted) {
  // bucket offsets (descending length), then per block: count the block's
  // rays per bucket in shared memory, reserve each bucket's range with one
  // global atomic, and scatter (order inside a bucket does not matter)
  __shared__ unsigned int off[LEN_BUCKETS];
  __shared__ unsigned int cnt[LEN_BUCKETS];
  __shared__ unsigned int base[LEN_BUCKETS];
  if (threadIdx.x == 0) {
    unsigned int run = 0;
    for (int b = LEN_BUCKETS - 1; b >= 0; --b) {
      off[b] = run;
      run += hist[b];
    }
  }
  const int64_t n = (int64_t)*d_n;
  for (int64_t k0 = blockIdx.x * (int64_t)blockDim.x; k0 < n; k0 += (int64_t)gridDim.x * blockDim.x) {
    for (int i = threadIdx.x; i < LEN_BUCKETS; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    const int64_t k = k0 + threadIdx.x;
    int32_t r = -1;
    int b = 0;
    unsigned int slot = 0;
    if (k < n) {
      r = active[k];
      const int64_t len = seg_end[r] - seg_start[r];
      b = len < LEN_BUCKETS - 1 ? (int)len : LEN_BUCKETS - 1;
      slot = atomicAdd(&cnt[b], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < LEN_BUCKETS; i += blockDim.x)
      base[i] = cnt[i] ? atomicAdd(&cursor[i], cnt[i]) : 0u;
    __syncthreads();
    if (r >= 0) sorted[off[b] + base[b] + slot] = r;
    __syncthreads();
  }
}

// Tile traversal: a tile list longer than the arena holds (`tile_need`
// against `lim`) asks for a rerun with the pair capacity whose arena share
// (`entry` bytes per pair per warp beyond the shared-memory lists, out of
// 16 bytes per unit of capacity) holds it, plus a quarter.
struct TileOverflow {
  const unsigned long long* need;  // null: level-by-level traversal
  int64_t lim, scap, warps, entry;
};

__device__ __forceinline__ int64_t tile_overflow(ng_frame_stats* st, const TileOverflow& T) {
  if (T.need == nullptr || (int64_t)*T.need <= T.lim) return 0;
  const int64_t spill = ((int64_t)*T.need - T.scap + 16) * 5 / 4;
  const int64_t want = spill * T.entry * T.warps / 16 + 4096;
  if (want > st->pair_need) st->pair_need = want;
  return 1;
}

__device__ __forceinline__ void finish_stats(ng_frame_stats* st, int n_levels, int64_t pair_cap, int64_t hit_cap,
                                             const unsigned long long* d_hits, const unsigned long long* d_active,
                                             const TileOverflow& T) {
  int64_t over = 0;
  if (T.need == nullptr)
    for (int t = 1; t < n_levels; ++t) over |= (st->pairs[t] > pair_cap);
  over |= (st->pairs[n_levels] > hit_cap);
  over |= tile_overflow(st, T);
  st->overflow = over;
  st->visible = (int64_t)*((volatile const unsigned long long*)d_hits);
  st->active_rays = (int64_t)*((volatile const unsigned long long*)d_active);
}

// The frame statistics, run by the last CTA of the primary march (no
// separate launch).
struct FinishArgs {
  ng_frame_stats* st;  // null: not this launch's job
  int n_levels;
  int64_t pair_cap, hit_cap;
  const unsigned long long* d_hits;
  const unsigned long long* d_active;
  unsigned int* done;  // CTAs finished (zeroed per frame)
  TileOverflow tov;
};

struct MarchArgs {
  ng_render_cfg cfg;
  int G, out_mask, dec_first, dec_last, passes;
  int blend_base;
  double blend_alpha;
  RaySrc rays;                   // ray records, or the camera's rays computed on the fly
  const int32_t* work;           // ray ids to trace, or null for 0..n_work-1
  const int4* items;             // or work items (ray, segment length, segment start lo / hi) from the tile traversal
  const unsigned long long* d_n_work;
  int64_t n_work;
  const ng_hit_pair* hits;
  int pair_cells;                // hits[].ray holds the voxel's packed cell (x | y << 10 | z << 20)
  const int64_t* seg_start;
  const int64_t* seg_end;
  uint8_t* hit;
  double* t;
  int32_t* iters;
  int32_t* evals;
  int32_t* hit_list;             // optional: ids of hit rays
  unsigned long long* d_hit_count;
  unsigned long long* work_counter;
  ng_counters* counters;
  unsigned long long* prof;      // optional: 4 counters per group (steps, busy lanes, t0, t1)
  int lane_cap;                  // max rays a warp marches at once (NG_MARCH_CAP, default 32)
  FinishArgs fin;
  // normals (render.py:277-300) in the march: every hit publishes 6 probe
  // items (slot * 6 + j); lanes without a ray evaluate them, and the lane
  // completing a slot's sixth probe forms the normal and shades the pixel
  int probes;
  unsigned long long* probe_next;  // next probe item to claim
  unsigned long long* rays_done;   // rays finished (hits published first)
  unsigned int* probe_cnt;         // per slot: bit 31 published, low bits probes done
  double* probe_val;               // per slot: the 6 probe values
  double* probe_pt;                // per slot: the hit point, written before the slot is published
  double* normal;
  uint8_t* normal_ok;
  uint8_t* color;                  // null: shading happens later (shadow pass)
};

constexpr unsigned PROBE_READY = 0x80000000u;
#ifdef NG_PROFILE
__device__ unsigned long long* g_timeline = nullptr;  // ng_march_timeline
#endif

// Release-ordered atomics for the probe slots: MEMBAR.ALL.GPU before the
// atomic, no L1 invalidation (a gpu-scope __threadfence or acquire emits
// CCTL.IVALL, which drops every warp's L1-cached table rows on the SM).
__device__ __forceinline__ unsigned atom_add_release(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_or_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
#ifndef NG_PROBE_GROUP_MAX_HEAVY
#define NG_PROBE_GROUP_MAX_HEAVY 64
#endif
#ifndef NG_PROBE_GROUP_MAX
#define NG_PROBE_GROUP_MAX 0  // a group takes probe items while it marches at most this many rays
#endif

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// One lane's query_field (render.py:155-171) result assembled from the
// decoder outputs emitted by warp_eval (blend of predict(base), predict(base+1)).
struct FieldValue {
  double lo = 0.0, hi = 0.0;
};

// The field's presummed tables serve this evaluation when they were built
// for its gather level and output levels and points are decoded only
// inside gather-level voxels (presum.cu).
__device__ __forceinline__ void use_presum(const ng_field& f, EvalCtx& c) {
  if (f.presum && f.presum_level == c.gather_level && f.presum_mask == c.out_mask &&
      c.inside_level == c.gather_level) {
    c.presum = f.presum;
    c.presum_offset = f.presum_offset;
    c.presum_corners = f.presum_corners;
  }
}

// query_field value (render.py:155-171) from one lane's evaluation.
__device__ __forceinline__ double field_value(const ng_octree& tree, const EvalLane& er, double lo, double hi,
                                              double alpha, const double x[3]) {
  if (!er.inside) return empty_value(tree, x);
  if (alpha != 0.0) return dadd(dmul(dsub(1.0, alpha), lo), dmul(alpha, hi));
  return lo;
}

// shade (render.py:303-314) of one hit pixel with its fp64 normal.
__device__ __forceinline__ void shade_rgb(const ng_render_cfg& cfg, const double nv[3], uint8_t* rgb_out) {
  double lam = dadd(dadd(dmul(nv[0], cfg.light[0]), dmul(nv[1], cfg.light[1])), dmul(nv[2], cfg.light[2]));
  lam = lam < 0.0 ? 0.0 : (lam > 1.0 ? 1.0 : lam);
  const double amb = cfg.ambient;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    double rgb = dmul(cfg.albedo[ch], dadd(amb, dmul(dsub(1.0, amb), lam)));
    rgb = rgb < 0.0 ? 0.0 : (rgb > 1.0 ? 1.0 : rgb);
    rgb_out[ch] = (uint8_t)dadd(dmul(rgb, 255.0), 0.5);
  }
}

// Decoder policy setup shared by the march and normals kernels: SIMT stages
// fp32 decoders; TC carves TMEM / A tiles / bf16 B tiles (tc_mlp.cuh).
template <bool TC>
struct DecoderSetup {
  float* dec = nullptr;
  WarpScratch* ws = nullptr;
  TcSmem t;
  uint32_t tmem_base = 0;
  __device__ __forceinline__ DecoderSetup(uint8_t* smem, const ng_field& f, int first, int last, int groups,
                                          size_t ws_bytes = sizeof(WarpScratch)) {
    if constexpr (TC) {
      t = tc_carve(smem, last - first + 1, groups, ws_bytes);
      tmem_base = tc_setup(t, f.decoders, first, last, f.dec_stride, groups);
      ws = t.ws;
    } else {
      dec = reinterpret_cast<float*>(smem);
      ws = reinterpret_cast<WarpScratch*>(dec + (last - first + 1) * f.dec_stride);
      stage_decoders(dec, f.decoders, first, last, f.dec_stride);
    }
  }
};

template <int NW, bool TC, bool PS>
__global__ void __launch_bounds__(NW * 32, TC ? 1 : 2) k_march(const __grid_constant__ ng_octree tree, ng_field f,
                                                              const __grid_constant__ MarchArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ int gflag[2][NW];  // step parity: a warp is never two steps ahead of its group
  constexpr int GROUPS = TC ? NW / 4 : 1;
  // (the presummed tensor-core march never touches WarpScratch::zt)
  constexpr size_t WSB = (TC && PS) ? WS_COMPACT_BYTES : sizeof(WarpScratch);
  DecoderSetup<TC> D(smem_raw, f, A.dec_first, A.dec_last, GROUPS, WSB);
  const int w = threadIdx.x >> 5;
  const int g = w / 4;
  WarpScratch& ws = TC ? D.t.scratch(w) : D.ws[w];
  uint32_t phase = 0;
  TcMlp tcm;
  if constexpr (TC) {
    tcm = tc_policy(D.t, D.tmem_base, A.dec_first, &phase);
#ifdef NG_PROFILE
    if (A.prof && (w & 3) == 0) tcm.prof = A.prof + NG_PROF_SLOTS * (blockIdx.x * GROUPS + g);
#endif
  }
  EvalCtx c;
#ifdef NG_PROFILE
  // the group leader's eval phases: slots 11 prologue, 12 staging, 13 gather, 14 decoder
  if (A.prof && (w & 3) == 0) c.dbg = A.prof + NG_PROF_SLOTS * (blockIdx.x * GROUPS + g) + 11;
  unsigned long long* const gprof = (A.prof && (w & 3) == 0 && lane_id() == 0)
                                        ? A.prof + NG_PROF_SLOTS * (blockIdx.x * GROUPS + g) : nullptr;
  long long ck = 0, ck_top = 0;
  bool light_step = false;
  auto mark = [&](int slot) {  // clock64 laps of the group leader (slots 8..)
    if (gprof) {
      const long long now = clock64();
      gprof[slot] += (unsigned long long)(now - ck);
      ck = now;
    }
  };
#else
  auto mark = [](int) {};
#endif
  c.Z = f.Z;
  c.dec = D.dec;
  c.dec_first = A.dec_first;
  c.dec_stride = f.dec_stride;
  c.h = f.h;
  c.gather_level = A.G;
  c.inside_level = A.cfg.trace_level;
  c.out_mask = A.out_mask;
  if constexpr (PS) use_presum(f, c);
  const int lane = (int)lane_id();
  const int64_t n_work = A.d_n_work ? (int64_t)*A.d_n_work : A.n_work;
  // Spread light loads over every warp: with fewer rays than lanes, each
  // warp marches at most `cap` rays at a time, so a step gathers fewer
  // points per warp (fewer dependent load rounds) and all SMs take part.
  const int64_t warps_total = (int64_t)gridDim.x * NW;
  const int64_t per_warp = (n_work + warps_total - 1) / warps_total;
  int cap = per_warp >= 32 ? 32 : (per_warp < 1 ? 1 : (int)per_warp);
  if (A.lane_cap > 0 && cap > A.lane_cap) cap = A.lane_cap;
  const int tl = A.cfg.trace_level + tree.n_virtual;
  const int res = tree.r0 << A.cfg.trace_level;
  const double edge = 2.0 / (double)res;
  const uint64_t* __restrict__ codes = tree.codes[tl];
  const double NaN = __longlong_as_double(0x7ff8000000000000ll);
  LaneCounters lc;

  int ray = -1;
  bool drained = false, ready = false;
  int64_t cur = 0, end = 0;
  double t = 0.0, prev = NaN;
  int it = 0, ev = 0;
  double o[3] = {0, 0, 0}, d[3] = {0, 0, 0};
  // the pair at `hidx`, kept in registers: a ray takes several steps per voxel
  int64_t hidx = -1;
  ng_hit_pair h{};
  // probe item held by a lane without a ray (-1: none), and its point
  int64_t pk = -1;
  bool pready = false, probes_done = !A.probes;
  int step_parity = 0;
  unsigned idle_ns = 256;  // back-off of a group waiting for probe items
  // rays the group marched last step: probes are taken only by groups with
  // none left, so they never lengthen the steps of a ray still marching
  int group_marching = 1;
  // with several rays queued per lane, groups rarely run dry before the end,
  // so lightly marching groups (<= 64 of 128 rays) also take probe items;
  // otherwise only groups with no rays left do (measured: 720p prefers 0,
  // 1080p LOD6 64)
  // (single-decoder frames only: with the LOD blend every probe costs two)
  const int probe_group_max = (n_work > 4 * (int64_t)gridDim.x * NW * 32 && A.passes == 1) ? NG_PROBE_GROUP_MAX_HEAVY
                                                                                          : NG_PROBE_GROUP_MAX;
  double px[3] = {0, 0, 0};
  const double eps = A.cfg.normal_eps;

  auto finish = [&](bool is_hit, double th) {
    A.hit[ray] = is_hit ? 1 : 0;
    A.t[ray] = is_hit ? th : NaN;
    A.iters[ray] = it;
    A.evals[ray] = ev;
    ray = -1;
  };

#ifdef NG_PROFILE
  unsigned long long t_top = 0;
#endif
  while (true) {
#ifdef NG_PROFILE
    if (A.prof && (w & 3) == 0 && lane == 0) t_top = globaltimer_ns();
    ck = clock64();
    ck_top = ck;
#endif
    // ---- acquire rays and advance each to its next query point (render.py:200-238)
    while (true) {
      const bool want = (ray < 0) && !drained && lane < cap;
      const unsigned wm = __ballot_sync(FULL, want);
      if (wm) {
        const int leader = __ffs(wm) - 1;
        unsigned long long b = 0;
        if (lane == leader) b = atomicAdd(A.work_counter, (unsigned long long)__popc(wm));
        b = __shfl_sync(FULL, b, leader);
        if (want) {
          const int64_t k = (int64_t)b + __popc(wm & lanemask_lt());
          if (k >= n_work) {
            drained = true;
          } else {
            if (A.items) {  // one load: ray and segment
              const int4 wi = A.items[k];
              ray = wi.x;
              cur = (int64_t)(uint32_t)wi.z | ((int64_t)wi.w << 32);
              end = cur + wi.y;
            } else {
              ray = A.work ? A.work[k] : (int)k;
              cur = A.seg_start[ray];
              end = A.seg_end[ray];
            }
            t = 0.0;
            prev = NaN;
            it = 0;
            ev = 0;
            ready = false;
            if (A.rays.cam_rays) {
              const int fc = A.rays.cam.frame_of(ray);  // the ray's frame in a batch
              const ng_camera& cm = A.rays.cam.cam[fc];
              camera_dir(cm, ray - (int64_t)fc * A.rays.cam.n_per, d);  // (the march needs no slab fields)
              o[0] = cm.position[0]; o[1] = cm.position[1]; o[2] = cm.position[2];
            } else {
              const ng_ray* rp = A.rays.rays + ray;
              o[0] = rp->o[0]; o[1] = rp->o[1]; o[2] = rp->o[2];
              d[0] = rp->d[0]; d[1] = rp->d[1]; d[2] = rp->d[2];
            }
          }
        }
      }
      if (ray >= 0 && !ready) {
        bool dead = false;
        while (true) {
          if (cur >= end || t > A.cfg.far_plane) {
            dead = true;
            break;
          }
          if (hidx != cur) {
            h = A.hits[cur];
            hidx = cur;
          }
          if (t >= h.t_exit) {
            ++cur;
            prev = NaN;
            continue;
          }
          if (t < h.t_enter) {
            const double t_in = dadd(h.t_enter, A.cfg.skip_eps);
            if (t_in >= h.t_exit) {  // grazing sliver thinner than the nudge
              ++cur;
              continue;
            }
            t = t_in;
          }
          break;
        }
        if (dead) {
          finish(false, 0.0);
          if (A.probes) atomicAdd(A.rays_done, 1ull);
        } else {
          ready = true;
        }
      }
      if (!__any_sync(FULL, ray < 0 && !drained && lane < cap)) break;
    }
    mark(8);  // ray claims + segment walk
    if (__any_sync(FULL, !probes_done)) {  // warp-uniform: the claim below is a warp collective
      // lanes out of rays claim probe items (warp-aggregated) ...
      const bool pw = !probes_done && ray < 0 && pk < 0 && (drained || lane >= cap) &&
                      (!TC || group_marching <= probe_group_max);
      const unsigned pm = __ballot_sync(FULL, pw);
      if (pm) {
        const int leader = __ffs(pm) - 1;
        unsigned long long b = 0;
        if (lane == leader) b = atomicAdd(A.probe_next, (unsigned long long)__popc(pm));
        b = __shfl_sync(FULL, b, leader);
        if (pw) {
          pk = (int64_t)(b + __popc(pm & lanemask_lt()));
          pready = false;
        }
      }
      // ... and start one once its hit is published; an item past the last
      // hit after every ray has finished ends the lane's probe work
      if (pk >= 0 && !pready && pk / 6 >= n_work) {  // no such hit can exist
        pk = -1;
        probes_done = true;
      }
      if (pk >= 0 && !pready) {
        const int64_t sl = pk / 6;
        unsigned st;
        // relaxed (no L1 invalidation, unlike ld.acquire / __threadfence): the
        // slot's data is read below with L2 (.cg) loads issued after the flag
        // is seen, and the publisher wrote it before its release
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(st) : "l"(A.probe_cnt + sl) : "memory");
        if (st & PROBE_READY) {
          // the hit point the publisher stored with the slot (one L2 round
          // trip, not hit_list -> t -> the camera ray)
          const int j = (int)(pk % 6), axis = j % 3;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            double v = __ldcg(A.probe_pt + 3 * sl + a);  // hit point o + t d (render.py:396)
            if (a == axis) v = (j < 3) ? dadd(v, eps) : dsub(v, eps);
            px[a] = np_min(np_max(v, -1.0), 1.0);  // render.py:289-293
          }
          pready = true;
        } else if (*((volatile unsigned long long*)A.rays_done) >= (unsigned long long)n_work &&
                   (unsigned long long)sl >= *((volatile unsigned long long*)A.d_hit_count)) {
          pk = -1;
          probes_done = true;
        }
      }
    }
    mark(9);  // probe claims
    const bool act = ray >= 0;
    const bool pact = pk >= 0 && pready;
    // a lane stays in the loop while it marches, holds a probe item or may
    // still claim one
    const bool alive = act || pk >= 0 || !probes_done || (!drained && lane < cap);
    int* gf = gflag[step_parity];
    if constexpr (TC) {
      // The group's 4 warps step together (one 128-row GEMM per output
      // level). Each warp posts its counts here; the decoder's group
      // barrier inside the evaluation orders them, and every warp reads the
      // group's totals after it (one barrier per step: a warp's acquire and
      // gather phases no longer wait for the slowest warp separately).
      const int wf = __popc(__ballot_sync(FULL, act || pact));
      const int wa = __popc(__ballot_sync(FULL, alive));
      const int wm = __popc(__ballot_sync(FULL, act));
      step_parity ^= 1;
      if (lane == 0) gf[w] = wf | (wa << 8) | (wm << 16);
      mark(10);  // (group flags posted)
    } else {
      if (!__any_sync(FULL, alive)) break;
      if (!__any_sync(FULL, act || pact)) {
        __nanosleep(256);
        continue;
      }
    }

    // ---- query point: x = o + t d clamped into the current voxel (render.py:244-245),
    // or the lane's normal probe
    double x[3] = {px[0], px[1], px[2]};
    if (act) {
      int cc[3];
      if (A.pair_cells) {
        const uint32_t pc = (uint32_t)h.ray;
        cc[0] = (int)(pc & 1023u);
        cc[1] = (int)((pc >> 10) & 1023u);
        cc[2] = (int)(pc >> 20);
      } else {
        const uint64_t code = __ldg(codes + h.voxel);
        cc[0] = (int)compact3(code);
        cc[1] = (int)compact3(code >> 1);
        cc[2] = (int)compact3(code >> 2);
      }
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double lo = cell_lo(cc[a], res);
        const double hi = dadd(lo, edge);
        const double top = dsub(hi, dmul(dsub(hi, lo), 1e-9));  // clamp_into, octree.py:293-300
        double v = dadd(o[a], dmul(t, d[a]));
        v = np_max(v, lo);
        v = np_min(v, top);
        x[a] = v;
      }
    }
    FieldValue fv;
    const bool eact = act || pact;
    auto emit = [&](int L, float dv, bool bad, const EvalLane& e) {
      if (!eact || !e.inside) return;
      double v;
      if (e.present & ((1u << L) - 1u)) {
        v = (double)dv;
        lc.evals += 1;
        if (!((e.present >> (L - 1)) & 1u)) lc.missing += 1;
        if (bad) lc.nonfinite += 1;
      } else {
        v = empty_value(tree, x);
        lc.empty += 1;
      }
      if (L == A.blend_base) fv.lo = v; else fv.hi = v;
    };
    EvalLane er;
    if constexpr (PS) {
      // x lies in the pair's voxel (clamped above), which is locate's answer
      // (a probe point is located as usual)
      // (four groups: 128 registers, so 4 points' rows per gather round)
      constexpr int GBM = NW >= 16 ? 4 : NG_GATHER_BATCH;
      if constexpr (TC) er = warp_eval_presum<GBM>(tree, c, ws, eact, x, tcm, emit, act ? (int64_t)h.voxel : -1);
      else er = warp_eval_presum<GBM>(tree, c, ws, eact, x, SimtMlp{c}, emit, act ? (int64_t)h.voxel : -1);
    } else {
      if constexpr (TC) er = warp_eval(tree, c, ws, eact, x, tcm, emit);
      else er = warp_eval(tree, c, ws, eact, x, SimtMlp{c}, emit);
    }
    auto dval_of = [&](const EvalLane& e, const FieldValue& v, const double* px) {
      return field_value(tree, e, v.lo, v.hi, A.blend_alpha, px);
    };

    mark(18);  // query point + evaluation
    if constexpr (TC) {
      const int gs = gf[4 * g] + gf[4 * g + 1] + gf[4 * g + 2] + gf[4 * g + 3];
      const int active = gs & 0xff, any_alive = (gs >> 8) & 0xff;
      group_marching = gs >> 16;
#ifdef NG_PROFILE
      if (gprof && active) {
        gprof[16] += 1;
        if (active <= 8) gprof[17] += 1;  // light steps: the tail's per-step latency
      }
      if (gprof && g_timeline && blockIdx.x < 16) {  // step timeline of 64 groups: (ns, busy lanes)
        const int gi = blockIdx.x * GROUPS + g;
        const unsigned k = (unsigned)gprof[20]++;
        if (gi < 64 && k < 512) {
          unsigned long long tnow;
          asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tnow));
          g_timeline[gi * 512 + k] = (tnow << 8) | (unsigned long long)(active & 0xff);
        }
      }
      light_step = active <= 8;
      if (A.prof && (w & 3) == 0 && lane == 0) {  // debug profile: per-group steps and busy lanes
        unsigned long long* pr = A.prof + NG_PROF_SLOTS * (blockIdx.x * GROUPS + g);
        const unsigned long long now = globaltimer_ns();
        if (pr[0] == 0) pr[2] = t_top;
        if (active) {
          pr[0] += 1;
          pr[1] += active;
        }
        pr[3] = now;
      }
#endif
      if (!any_alive) break;  // (no lane of the group was alive at this step's start)
      // waiting for hits to publish probe items: an empty step still runs
      // the group's GEMM, so back off (up to ~4 us) while nothing arrives
      if (!active) {
        __nanosleep(idle_ns);
        idle_ns = idle_ns < 4096 ? 2 * idle_ns : idle_ns;
      } else {
        idle_ns = 256;
      }
    }
    // ---- stop rules (render.py:247-272)
    if (eact && !er.inside) lc.empty += 1;  // query_field's own empty-space fallback
    if (pact) {
      // normals (render.py:294-299): g = (v+ - v-) / (2 eps) once all 6 are in
      const int64_t sl = pk / 6;
      __stcg(A.probe_val + pk, dval_of(er, fv, x));
      const unsigned old = atom_add_release(A.probe_cnt + sl, 1u);  // the value before the count
      if ((old & 0xffffu) == 5u) {  // the other five values are in L2: read them there
        double vals[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) vals[j] = __ldcg(A.probe_val + 6 * sl + j);
        const int32_t pix = __ldcg(A.hit_list + sl);
        const double two_eps = 2.0 * eps;
        double gr[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) gr[a] = dsub(vals[a], vals[3 + a]) / two_eps;
        const double nrm = __dsqrt_rn(dadd(dadd(dmul(gr[0], gr[0]), dmul(gr[1], gr[1])), dmul(gr[2], gr[2])));
        const bool ok = isfinite(nrm) && nrm > 1e-12;
        double nv[3] = {0.0, 0.0, 0.0};
        if (ok) {
#pragma unroll
          for (int a = 0; a < 3; ++a) nv[a] = gr[a] / nrm;
        }
#pragma unroll
        for (int a = 0; a < 3; ++a) A.normal[3 * (int64_t)pix + a] = nv[a];
        A.normal_ok[pix] = ok ? 1 : 0;
        if (A.color) shade_rgb(A.cfg, nv, A.color + 3 * (int64_t)pix);
      }
      pk = -1;
    }
    if (act) {
      double dval = dval_of(er, fv, x);
      ev += A.passes;
      it += 1;
      const bool is_hit = dval < A.cfg.delta;
      const bool stalled = !is_hit && (dval >= prev) && (fabs(dsub(dval, prev)) < A.cfg.osc_tol);
      if (is_hit) {
        const int r_id = ray;
        const double th = dadd(t, dval);
        finish(true, th);
        if (A.hit_list) {
          const unsigned long long slot = atomicAdd(A.d_hit_count, 1ull);
          A.hit_list[slot] = r_id;
          if (A.probes) {
#pragma unroll
            for (int a = 0; a < 3; ++a) __stcg(A.probe_pt + 3 * slot + a, dadd(o[a], dmul(th, d[a])));
            red_or_release(A.probe_cnt + slot, PROBE_READY);  // publish (t, hit_list, hit point written above)
          }
        }
        if (A.probes) atomicAdd(A.rays_done, 1ull);
      } else if (stalled || it >= A.cfg.max_iters) {
        finish(false, 0.0);
        if (A.probes) atomicAdd(A.rays_done, 1ull);
      } else {
        prev = dval;
        t = dadd(t, dval);
        ready = false;
      }
    }
    mark(15);  // stop rules, hit publication
#ifdef NG_PROFILE
    if (gprof && light_step) gprof[19] += (unsigned long long)(clock64() - ck_top);
#endif
  }
  lc.flush(A.counters);
  if (A.fin.st) {  // last CTA out writes the frame statistics
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(A.fin.done, 1u) == gridDim.x - 1) {
        __threadfence();
        finish_stats(A.fin.st, A.fin.n_levels, A.fin.pair_cap, A.fin.hit_cap, A.fin.d_hits, A.fin.d_active,
                     A.fin.tov);
      }
    }
  }
  if constexpr (TC) tc_teardown(D.tmem_base, GROUPS);
}

struct NormalArgs {
  ng_render_cfg cfg;
  int G, out_mask, dec_first, dec_last;
  int blend_base;
  double blend_alpha;
  const double* pts;                 // explicit points, or null: hit rays below
  int64_t n_pts;
  RaySrc rays;
  const int32_t* hit_list;
  const unsigned long long* d_hit_count;
  const double* t_hit;
  double* normal;                    // per point (explicit) or per ray
  uint8_t* ok;
  uint8_t* color;                    // per ray when shading in place, else null
  ng_counters* counters;
};

// Corner rows in flight per gather round in k_normals. The 6 probes of a
// unit are evaluated one after another, so their latency is on the frame's
// critical path; 8 points per round (64 loads per warp) halves the rounds.
#ifndef NORMALS_GATHER_BATCH
#define NORMALS_GATHER_BATCH 8
#endif

// normals (render.py:277-300) + shade (render.py:303-314) for hit pixels.
template <int NW, bool TC, bool PS>
__global__ void __launch_bounds__(NW * 32, TC ? 1 : 2) k_normals(const __grid_constant__ ng_octree tree, ng_field f,
                                                                const __grid_constant__ NormalArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  constexpr int GROUPS = TC ? NW / 4 : 1;
  DecoderSetup<TC> D(smem_raw, f, A.dec_first, A.dec_last, GROUPS);
  const int w = threadIdx.x >> 5;
  WarpScratch& ws = D.ws[w];
  uint32_t phase = 0;
  TcMlp tcm;
  if constexpr (TC) tcm = tc_policy(D.t, D.tmem_base, A.dec_first, &phase);
  EvalCtx c;
  c.Z = f.Z;
  c.dec = D.dec;
  c.dec_first = A.dec_first;
  c.dec_stride = f.dec_stride;
  c.h = f.h;
  c.gather_level = A.G;
  c.inside_level = A.cfg.trace_level;
  c.out_mask = A.out_mask;
  if constexpr (PS) use_presum(f, c);
  const int64_t n = A.pts ? A.n_pts : (int64_t)*A.d_hit_count;
  const double eps = A.cfg.normal_eps;
  LaneCounters lc;
  // work units: 32 points per warp (SIMT) or 128 per 4-warp group (TC)
  // work units: PPW points per warp, 4 warps per unit (TC) or one (SIMT).
  // PPW = 32 at full load; light loads are spread over every warp so each
  // evaluation gathers fewer points per warp (fewer dependent load rounds).
  constexpr int WPU = TC ? 4 : 1;
  constexpr int PER_CTA = TC ? NW / 4 : NW;
  const int my = TC ? w / 4 : w;
  const int64_t units_total = (int64_t)gridDim.x * PER_CTA;
  const int64_t per_warp = (n + units_total * WPU - 1) / (units_total * WPU);
  const int ppw = per_warp >= 32 ? 32 : (per_warp < 1 ? 1 : (int)per_warp);
  const int64_t unit = (int64_t)WPU * ppw;
  const int64_t n_units = (n + unit - 1) / unit;
  for (int64_t u = (int64_t)blockIdx.x * PER_CTA + my; u < n_units; u += units_total) {
    const int64_t i = u * unit + (TC ? (int64_t)ppw * (w % 4) : 0) + lane_id();
    const bool act = (int)lane_id() < ppw && i < n;
    int64_t dst = i;
    double p[3] = {0.0, 0.0, 0.0};
    if (act) {
      if (A.pts) {
        p[0] = A.pts[3 * i];
        p[1] = A.pts[3 * i + 1];
        p[2] = A.pts[3 * i + 2];
      } else {
        dst = A.hit_list[i];
        ng_ray rr;
        if (A.rays.cam_rays) camera_ray(A.rays.cam, dst, rr);
        else load_ray(A.rays.rays, dst, rr);
        const double th = A.t_hit[dst];
#pragma unroll
        for (int a = 0; a < 3; ++a) p[a] = dadd(rr.o[a], dmul(th, rr.d[a]));  // render.py:396
      }
    }
    double vals[6];
#pragma unroll 1
    for (int j = 0; j < 6; ++j) {
      const int axis = j % 3;
      double x[3] = {p[0], p[1], p[2]};
      x[axis] = (j < 3) ? dadd(x[axis], eps) : dsub(x[axis], eps);
#pragma unroll
      for (int a = 0; a < 3; ++a) x[a] = np_min(np_max(x[a], -1.0), 1.0);
      FieldValue fv;
      auto emit = [&](int L, float dv, bool bad, const EvalLane& e) {
        if (!act || !e.inside) return;
        double v;
        if (e.present & ((1u << L) - 1u)) {
          v = (double)dv;
          lc.evals += 1;
          if (!((e.present >> (L - 1)) & 1u)) lc.missing += 1;
          if (bad) lc.nonfinite += 1;
        } else {
          v = empty_value(tree, x);
          lc.empty += 1;
        }
        if (L == A.blend_base) fv.lo = v; else fv.hi = v;
      };
      EvalLane er;
      if constexpr (PS) {
        if constexpr (TC) er = warp_eval_presum<NORMALS_GATHER_BATCH>(tree, c, ws, act, x, tcm, emit);
        else er = warp_eval_presum<NORMALS_GATHER_BATCH>(tree, c, ws, act, x, SimtMlp{c}, emit);
      } else {
        if constexpr (TC) er = warp_eval<NORMALS_GATHER_BATCH>(tree, c, ws, act, x, tcm, emit);
        else er = warp_eval<NORMALS_GATHER_BATCH>(tree, c, ws, act, x, SimtMlp{c}, emit);
      }
      double v = 0.0;
      if (act) {
        if (!er.inside) {
          v = empty_value(tree, x);
          lc.empty += 1;
        } else if (A.blend_alpha != 0.0) {
          v = dadd(dmul(dsub(1.0, A.blend_alpha), fv.lo), dmul(A.blend_alpha, fv.hi));
        } else {
          v = fv.lo;
        }
      }
      vals[j] = v;
    }
    if (act) {
      const double two_eps = 2.0 * eps;
      double g[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) g[a] = dsub(vals[a], vals[3 + a]) / two_eps;
      const double nrm = __dsqrt_rn(dadd(dadd(dmul(g[0], g[0]), dmul(g[1], g[1])), dmul(g[2], g[2])));
      const bool ok = isfinite(nrm) && nrm > 1e-12;
      double nv[3] = {0.0, 0.0, 0.0};
      if (ok) {
#pragma unroll
        for (int a = 0; a < 3; ++a) nv[a] = g[a] / nrm;
      }
#pragma unroll
      for (int a = 0; a < 3; ++a) A.normal[3 * dst + a] = nv[a];
      A.ok[dst] = ok ? 1 : 0;
      if (A.color) shade_rgb(A.cfg, nv, A.color + 3 * dst);  // render.py:303-314, fp64 normal
    }
  }
  lc.flush(A.counters);
  if constexpr (TC) tc_teardown(D.tmem_base, GROUPS);
}

__global__ void k_shade(const uint8_t* __restrict__ hit, const double* __restrict__ normal, int64_t n,
                        ng_render_cfg cfg, uint8_t* __restrict__ color) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double rgb[3];
    if (hit[i]) {
      double lam = dadd(dadd(dmul(normal[3 * i], cfg.light[0]), dmul(normal[3 * i + 1], cfg.light[1])),
                        dmul(normal[3 * i + 2], cfg.light[2]));
      lam = lam < 0.0 ? 0.0 : (lam > 1.0 ? 1.0 : lam);
      for (int ch = 0; ch < 3; ++ch)
        rgb[ch] = dmul(cfg.albedo[ch], dadd(cfg.ambient, dmul(dsub(1.0, cfg.ambient), lam)));
    } else {
      for (int ch = 0; ch < 3; ++ch) rgb[ch] = cfg.background[ch];
    }
    for (int ch = 0; ch < 3; ++ch) {
      double v = rgb[ch] < 0.0 ? 0.0 : (rgb[ch] > 1.0 ? 1.0 : rgb[ch]);
      color[3 * i + ch] = (uint8_t)dadd(dmul(v, 255.0), 0.5);
    }
  }
}

__global__ void k_hit_points(const ng_ray* __restrict__ rays, const uint8_t* __restrict__ hit,
                             const double* __restrict__ t, int64_t n, double* __restrict__ pts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int a = 0; a < 3; ++a) pts[3 * i + a] = hit[i] ? dadd(rays[i].o[a], dmul(t[i], rays[i].d[a])) : 0.0;
  }
}

__global__ void k_finish_stats(ng_frame_stats* st, int n_levels, int64_t pair_cap, int64_t hit_cap,
                               const unsigned long long* d_hits, const unsigned long long* d_active,
                               TileOverflow T) {
  finish_stats(st, n_levels, pair_cap, hit_cap, d_hits, d_active, T);
}

// Shadow rays for the hit pixels: origin p + offset * n, direction = light.
__global__ void k_shadow_rays(const __grid_constant__ RaySrc rays, const int32_t* __restrict__ hit_list,
                              const unsigned long long* __restrict__ d_hits, const double* __restrict__ t_hit,
                              const double* __restrict__ normal, ng_render_cfg cfg, ng_ray* __restrict__ srays,
                              int64_t* d_root) {
  const int64_t n = (int64_t)*d_hits;
  if (blockIdx.x == 0 && threadIdx.x == 0) *d_root = n;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t px = hit_list[j];
    ng_ray r;
    ray_at(rays, px, r);
    const double th = t_hit[px];
    double o[3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
      o[a] = dadd(dadd(r.o[a], dmul(th, r.d[a])), dmul(cfg.shadow_offset, normal[3 * px + a]));
    ng_ray sr;
    make_ray(o[0], o[1], o[2], cfg.light[0], cfg.light[1], cfg.light[2], sr);
    srays[j] = sr;
  }
}

// Lambert shading of hit pixels with the shadow term (ambient only in shadow).
__global__ void k_shade_shadowed(const int32_t* __restrict__ hit_list, const unsigned long long* __restrict__ d_hits,
                                 const double* __restrict__ normal, const uint8_t* __restrict__ s_hit,
                                 ng_render_cfg cfg, uint8_t* __restrict__ color, int64_t* d_shadowed) {
  const int64_t n = (int64_t)*d_hits;
  int local = 0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t px = hit_list[j];
    double lam = 0.0;
    if (!s_hit[j]) {
      lam = dadd(dadd(dmul(normal[3 * px], cfg.light[0]), dmul(normal[3 * px + 1], cfg.light[1])),
                 dmul(normal[3 * px + 2], cfg.light[2]));
      lam = lam < 0.0 ? 0.0 : (lam > 1.0 ? 1.0 : lam);
    } else {
      ++local;
    }
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      double rgb = dmul(cfg.albedo[ch], dadd(cfg.ambient, dmul(dsub(1.0, cfg.ambient), lam)));
      rgb = rgb < 0.0 ? 0.0 : (rgb > 1.0 ? 1.0 : rgb);
      color[3 * px + ch] = (uint8_t)dadd(dmul(rgb, 255.0), 0.5);
    }
  }
  for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(FULL, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd((unsigned long long*)d_shadowed, (unsigned long long)local);
}

__global__ void k_shadow_overflow(ng_frame_stats* st, int n_levels, int64_t pair_cap, int64_t hit_cap,
                                  TileOverflow T) {
  int64_t over = 0;
  if (T.need == nullptr)
    for (int t = 1; t < n_levels; ++t) over |= (st->shadow_pairs[t] > pair_cap);
  over |= (st->shadow_pairs[n_levels] > hit_cap);
  over |= tile_overflow(st, T);
  if (over) st->overflow = 1;
}

// ------------------------------------------------------------------ host side

struct LodPlan {
  int G, out_mask, dec_first, dec_last, passes, blend_base;
  double alpha;
};

static LodPlan plan_lod(const ng_render_cfg& cfg) {
  // blend (field.py:226-239) / query_field (render.py:159) for the resolved lod
  LodPlan p;
  const double lod = cfg.lod < 1.0 ? 1.0 : cfg.lod;
  const int base = (int)floor(lod);
  const double alpha = lod - (double)base;
  p.blend_base = base;
  p.alpha = alpha;
  if (alpha == 0.0) {
    p.out_mask = 1 << (base - 1);
    p.G = std::max(base, cfg.trace_level);
    p.dec_first = p.dec_last = base;
    p.passes = 1;
  } else {
    p.out_mask = (1 << (base - 1)) | (1 << base);
    p.G = std::max(base + 1, cfg.trace_level);
    p.dec_first = base;
    p.dec_last = base + 1;
    p.passes = 2;
  }
  return p;
}

template <class K>
static int prep_kernel(K kernel, size_t smem, int nt, int& per_sm) {
  // dynamic shared memory limit per (device, kernel function)
  if (int r = set_smem_limit((const void*)kernel, smem)) return r;
  per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, nt, smem);
  if (per_sm < 1) per_sm = 1;
  return NG_OK;
}


static bool use_tc_decoder(const ng_field& f) {
  static const bool env = [] {
    const char* e = getenv("NG_DECODER");
    return !(e && strcmp(e, "simt") == 0);
  }();
  return env && f.h == tc::N;
}

// 4-warp tile groups per CTA: the march runs four (the whole TMEM, 128
// registers, 4-point gather rounds; 720p 0.651 -> 0.627 ms against three
// groups with 8-point rounds), the normals pass three; NG_TC_GROUPS
// overrides both (experiment knob)
static int tc_groups(int dflt) {
  static const int g = env_int("NG_TC_GROUPS", 0);
  return (g >= 1 && g <= 4) ? g : dflt;
}

template <class KT, class Args>
static int launch_tc(KT ktc, int groups, const ng_field& f, const ng_octree& tree, const Args& A, int64_t max_units,
                     bool cap_by_work, cudaStream_t s, size_t ws_bytes) {
  const int ndec = A.dec_last - A.dec_first + 1;
  const size_t smem = tc_smem_bytes(ndec, groups, ws_bytes);
  int per_sm, r;
  if ((r = prep_kernel(ktc, smem, groups * 128, per_sm))) return r;
  int64_t grid = (int64_t)sm_count() * per_sm;
  if (cap_by_work) grid = std::max<int64_t>(1, std::min<int64_t>(grid, (max_units + 127) / 128));
  ktc<<<(int)grid, groups * 128, smem, s>>>(tree, f, A);
  return NG_OK;
}

template <class KS, class K1, class K2, class K3, class K4, class Args>
static int launch_eval_kernel(KS ksimt, K1 k1, K2 k2, K3 k3, K4 k4, const ng_field& f, const ng_octree& tree,
                              const Args& A, int64_t max_units, bool cap_by_work, const char* name, cudaStream_t s,
                              int default_groups = 3, size_t ws_bytes = sizeof(WarpScratch)) {
  const int ndec = A.dec_last - A.dec_first + 1;
  int per_sm, r;
  int groups = tc_groups(default_groups);
  while (groups > 1 && tc_smem_bytes(ndec, groups, ws_bytes) > 227 * 1024) --groups;
  if (use_tc_decoder(f) && tc_smem_bytes(ndec, groups, ws_bytes) <= 227 * 1024) {
    if (groups == 1) r = launch_tc(k1, 1, f, tree, A, max_units, cap_by_work, s, ws_bytes);
    else if (groups == 2) r = launch_tc(k2, 2, f, tree, A, max_units, cap_by_work, s, ws_bytes);
    else if (groups == 3) r = launch_tc(k3, 3, f, tree, A, max_units, cap_by_work, s, ws_bytes);
    else r = launch_tc(k4, 4, f, tree, A, max_units, cap_by_work, s, ws_bytes);
    if (r) return r;
  } else {
    const size_t smem = (size_t)ndec * f.dec_stride * 4 + R_NW * sizeof(WarpScratch);
    if ((r = prep_kernel(ksimt, smem, R_NW * 32, per_sm))) return r;
    static const int cap = env_int("NG_MARCH_CTAS_PER_SM", 0);  // experiment knob for the persistent grid
    if (cap > 0 && cap < per_sm) per_sm = cap;
    int64_t grid = (int64_t)sm_count() * per_sm;
    if (cap_by_work) grid = std::max<int64_t>(1, std::min<int64_t>(grid, (max_units + 32 * R_NW - 1) / (32 * R_NW)));
    ksimt<<<(int)grid, R_NW * 32, smem, s>>>(tree, f, A);
  }
  NG_CHECK_LAUNCH(name);
  return NG_OK;
}

// Host mirror of use_presum: the presummed kernels are launched only when
// the field's tables match this evaluation.
static bool presum_applies(const ng_field& f, int G, int out_mask, int trace_level) {
  return f.presum && f.presum_level == G && f.presum_mask == out_mask && trace_level == G;
}

static int launch_march(const ng_octree& tree, const ng_field& f, MarchArgs& A, cudaStream_t s) {
  static const int cap_env = env_int("NG_MARCH_CAP", 32);
  A.lane_cap = cap_env;
  if (presum_applies(f, A.G, A.out_mask, A.cfg.trace_level))
    return launch_eval_kernel(k_march<R_NW, false, true>, k_march<4, true, true>, k_march<8, true, true>,
                              k_march<12, true, true>, k_march<16, true, true>, f, tree, A, 0, false, "k_march", s,
                              4, WS_COMPACT_BYTES);
  return launch_eval_kernel(k_march<R_NW, false, false>, k_march<4, true, false>, k_march<8, true, false>,
                            k_march<12, true, false>, k_march<16, true, false>, f, tree, A, 0, false, "k_march", s);
}

static int launch_normals(const ng_octree& tree, const ng_field& f, NormalArgs& A, int64_t max_n, cudaStream_t s) {
  if (presum_applies(f, A.G, A.out_mask, A.cfg.trace_level))
    return launch_eval_kernel(k_normals<R_NW, false, true>, k_normals<4, true, true>, k_normals<8, true, true>,
                              k_normals<12, true, true>, k_normals<16, true, true>, f, tree, A, max_n, true,
                              "k_normals", s);
  return launch_eval_kernel(k_normals<R_NW, false, false>, k_normals<4, true, false>, k_normals<8, true, false>,
                            k_normals<12, true, false>, k_normals<16, true, false>, f, tree, A, max_n, true,
                            "k_normals", s);
}

static void background_u8(const ng_render_cfg& cfg, uint8_t bg[3]) {
  for (int c = 0; c < 3; ++c) {
    double v = cfg.background[c] < 0.0 ? 0.0 : (cfg.background[c] > 1.0 ? 1.0 : cfg.background[c]);
    bg[c] = (uint8_t)(v * 255.0 + 0.5);
  }
}

// Workspace layout (all offsets 256-byte aligned).
struct WsLayout {
  size_t rays, pairs_a, pairs_b, hits, seg_start, seg_end, active, hit_list, scratch, ctr, total;
  size_t s_rays, s_hit, s_t, s_it, s_ev;  // shadow-ray pass
  size_t sorted, buckets;                 // longest-first march order
  size_t cont;                            // tile traversal continuations (split silhouette tiles)
  size_t probe_val, probe_cnt, probe_pt;  // normals evaluated in the march
  size_t scratch_bytes;
};

static size_t al(size_t x) { return (x + 255) & ~size_t(255); }

// list entries per warp the tile traversal's arena holds at least
// (NG_TILE_ARENA_MIN overrides: a test knob for the overflow / rerun path)
static int64_t tile_arena_min() {
  static const int64_t v = std::max(0, env_int("NG_TILE_ARENA_MIN", 2048));
  return v;
}

static WsLayout layout(int64_t n, int64_t pair_cap, int64_t hit_cap) {
  WsLayout L;
  size_t o = 0;
  L.rays = o; o = al(o + (size_t)n * sizeof(ng_ray));
  // the two pair buffers double as the tile traversal's spill arena: at
  // least TILE_ARENA_MIN list entries per warp whatever the frame size
  const size_t tile_arena = (size_t)tile_traverse_warps(n) * tile_arena_min() * tile_traverse_entry_bytes();
  const size_t pair_bytes = std::max((size_t)pair_cap * sizeof(ng_pair), tile_arena / 2);
  L.pairs_a = o; o = al(o + pair_bytes);
  L.pairs_b = o; o = al(o + pair_bytes);
  L.hits = o; o = al(o + (size_t)hit_cap * sizeof(ng_hit_pair));
  L.seg_start = o; o = al(o + (size_t)n * 8);
  L.seg_end = o; o = al(o + (size_t)n * 8);
  L.active = o; o = al(o + (size_t)n * 16);  // ray ids, or the tile traversal's 16-byte work items
  L.hit_list = o; o = al(o + (size_t)n * 4);
  // one look-back scratch region per traversal level, zeroed together once per pass
  L.scratch_bytes = al(level_scratch_bytes(std::max<int64_t>(std::max<int64_t>(pair_cap, n), 1)));
  L.scratch = o; o = al(o + L.scratch_bytes * NG_MAX_TLEVELS);
  L.ctr = o; o = al(o + 64);
  L.s_rays = o; o = al(o + (size_t)n * sizeof(ng_ray));
  L.s_hit = o; o = al(o + (size_t)n);
  L.s_t = o; o = al(o + (size_t)n * 8);
  L.s_it = o; o = al(o + (size_t)n * 4);
  L.s_ev = o; o = al(o + (size_t)n * 4);
  L.sorted = o; o = al(o + (size_t)n * 4);
  L.probe_val = o; o = al(o + (size_t)n * 6 * 8);
  L.probe_cnt = o; o = al(o + (size_t)n * 4);
  L.probe_pt = o; o = al(o + (size_t)n * 3 * 8);
  L.buckets = o; o = al(o + 2 * LEN_BUCKETS * 4);
  L.cont = o; o = al(o + tile_cont_bytes());
  L.total = o;
  return L;
}

// NG_MARCH_PROFILE=1: per-group march statistics (ng_march_profile).
#ifdef NG_PROFILE
extern "C" int ng_march_timeline(unsigned long long* host_out) {  // 64 groups x 512 steps, then reset
  unsigned long long* p = nullptr;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&p, g_timeline, sizeof(p));
  if (!p) {
    cudaMalloc((void**)&p, 64 * 512 * 8);
    cudaMemcpyToSymbol(g_timeline, &p, sizeof(p));
  } else if (host_out) {
    cudaMemcpy(host_out, p, 64 * 512 * 8, cudaMemcpyDeviceToHost);
  }
  cudaMemset(p, 0, 64 * 512 * 8);
  return 0;
}
#endif
static unsigned long long* g_prof = nullptr;
// (a debugging aid of one device: the buffer lives on the device current at
// the first frame)
static unsigned long long* march_profile_buffer() {
  static const bool on = [] {
    if (env_int("NG_MARCH_PROFILE", 0) != 1) return false;
    if (cudaMalloc((void**)&g_prof, 8 * NG_PROF_SLOTS * 4096) != cudaSuccess) return false;
    cudaMemset(g_prof, 0, 8 * NG_PROF_SLOTS * 4096);
    return true;
  }();
  return on ? g_prof : nullptr;
}

// Hit-filtered traversal of `rays` (root count already in counts[0]),
// per-ray segments and the list of rays with a segment, then the march
// arguments (outputs left to the caller).
static int trace_pass(const ng_octree& tree, const ng_render_cfg& cfg, const LodPlan& P, const ng_ray* rays,
                      int64_t n, int64_t* counts, const WsLayout& L, const ng_workspace& ws, char* b,
                      unsigned long long* d_active, unsigned long long* work_counter, cudaStream_t s,
                      MarchArgs& A, bool zeroed, const double* shared_origin, TileOverflow& tov,
                      const CamSet* cam_rays = nullptr, const ng_frame* defaults = nullptr, uint32_t bg = 0,
                      int64_t n_host = -1) {
  ng_pair* pa = (ng_pair*)(b + L.pairs_a);
  ng_pair* pb = (ng_pair*)(b + L.pairs_b);
  ng_hit_pair* hits = (ng_hit_pair*)(b + L.hits);
  int64_t* seg_start = (int64_t*)(b + L.seg_start);
  int64_t* seg_end = (int64_t*)(b + L.seg_end);
  int32_t* active = (int32_t*)(b + L.active);
  void* scratch = b + L.scratch;
  int r;
  // pass t expands the hits at level t into the hit children at level t+1;
  // the last pass writes the final (ray, voxel, t_enter, t_exit) list
  const int target = cfg.trace_level + tree.n_virtual;
  const ng_pair* in = nullptr;
  int64_t in_cap = n;
  unsigned int* buckets = (unsigned int*)(b + L.buckets);
  const bool tiles = use_tile_traverse(target);
  tov.need = nullptr;
  if (!zeroed && tiles) {  // the tile path reads only its control words (the march takes work items)
    int rz = cuda_status(cudaMemsetAsync(scratch, 0, 512, s), "tile traversal control words");
    if (!rz) rz = cuda_status(cudaMemsetAsync(b + L.cont, 0, tile_cont_ready_bytes(), s), "tile continuations");
    if (rz) return rz;
  } else if (!zeroed) {  // the primary pass has these zeroed by k_zero_regions and the ray kernel
    ZeroRegions z;
    z.n = 4;
    z.p[0] = scratch;
    z.bytes[0] = L.scratch_bytes * (size_t)target;
    z.p[1] = seg_start;
    z.bytes[1] = (size_t)n * 8;
    z.p[2] = seg_end;
    z.bytes[2] = (size_t)n * 8;
    z.p[3] = buckets;
    z.bytes[3] = 2 * LEN_BUCKETS * 4;
    k_zero_regions<<<grid_for(n / 2 + 1, 256), 256, 0, s>>>(z);
    NG_CHECK_LAUNCH("k_zero_regions");
  }
  if (tiles) {
    // one launch: level passes per 32-ray tile, the pair lists in shared
    // memory with the two pair buffers as the spill arena; the control words
    // (tile counter, hit cursor, longest tile list) live in the zeroed
    // look-back scratch
    const size_t arena_bytes = L.hits - L.pairs_a;
    unsigned long long* need = (unsigned long long*)((char*)scratch + 16);
    r = traverse_tiles(tree, rays, &counts[0], n, target, reinterpret_cast<int4*>(active), d_active, counts, hits, ws.hit_capacity, scratch, seg_start, seg_end,
                       b + L.pairs_a, arena_bytes, need, shared_origin, cam_rays, defaults, bg, n_host,
                       b + L.cont, s);
    if (r) return r;
    tov.need = need;
    tov.lim = tile_traverse_limit(arena_bytes, n);
    tov.scap = tile_traverse_scap();
    tov.warps = tile_traverse_warps(n);
    tov.entry = tile_traverse_entry_bytes();
  }
  for (int t = 0; t < (tiles ? 0 : target); ++t) {
    const bool last = (t + 1 == target);
    ng_pair* out = (t % 2 == 0) ? pa : pb;
    r = traverse_hits(tree, rays, t, last, in, &counts[t], in_cap, last ? nullptr : out, last ? hits : nullptr,
                      &counts[t + 1], last ? ws.hit_capacity : ws.pair_capacity,
                      (char*)scratch + (size_t)t * L.scratch_bytes, L.scratch_bytes, s,
                      last ? seg_start : nullptr, last ? seg_end : nullptr, shared_origin);
    if (r) return r;
    in = out;
    in_cap = ws.pair_capacity;
  }
  int32_t* sorted = (int32_t*)(b + L.sorted);
  if (!tiles) {  // the tile traversal appends the work list itself (tile order)
    k_active_hist<<<grid_for(n, 256), 256, 0, s>>>(seg_start, seg_end, n, active, d_active, buckets);
    NG_CHECK_LAUNCH("k_active_hist");
    k_len_scatter<<<grid_for(n, 256), 256, 0, s>>>(active, d_active, seg_start, seg_end, buckets,
                                                    buckets + LEN_BUCKETS, sorted);
    NG_CHECK_LAUNCH("k_len_scatter");
  }
  A.cfg = cfg;
  A.G = P.G;
  A.out_mask = P.out_mask;
  A.dec_first = P.dec_first;
  A.dec_last = P.dec_last;
  A.passes = P.passes;
  A.blend_base = P.blend_base;
  A.blend_alpha = P.alpha;
  A.rays.rays = rays;
  A.rays.cam_rays = cam_rays != nullptr;
  if (cam_rays) A.rays.cam = *cam_rays;
  // level-by-level path: longest segments first; the tile path marches in
  // tile order (measured the same on the 720p knot frame, and it saves the
  // histogram and scatter launches)
  A.work = tiles ? nullptr : sorted;
  A.items = tiles ? reinterpret_cast<const int4*>(active) : nullptr;
  A.d_n_work = d_active;
  A.n_work = 0;
  A.hits = hits;
  A.pair_cells = tiles ? 1 : 0;
  A.seg_start = seg_start;
  A.seg_end = seg_end;
  A.work_counter = work_counter;
  A.prof = march_profile_buffer();
  A.probes = 0;
  A.fin.st = nullptr;
  return NG_OK;
}

// A batch's cameras as the kernels take them (frame f = rays [f n, (f+1) n)).
static CamSet cam_set(const ng_camera* cams, int k) {
  CamSet cs{};
  for (int i = 0; i < k; ++i) cs.cam[i] = cams[i];
  cs.k = k;
  cs.n_per = (int64_t)cams[0].width * cams[0].local_rows;
  return cs;
}

static int render_common(const ng_octree& tree, const ng_field& f, const ng_render_cfg& cfg,
                         const CamSet* cam, const ng_ray* user_rays, int64_t n, const ng_frame& fr,
                         const ng_workspace& ws, ng_frame_stats* st, bool do_normals, cudaStream_t s) {
  if (cfg.trace_level < 0 || cfg.trace_level > tree.max_level) {
    set_error("trace level %d outside 0..%d", cfg.trace_level, tree.max_level);
    return NG_ERR_CONFIG;
  }
  if (cfg.lod > (double)f.n_decoders) {
    set_error("lod %g above max level %d", cfg.lod, f.n_decoders);
    return NG_ERR_CONFIG;
  }
  const WsLayout L = layout(n, ws.pair_capacity, ws.hit_capacity);
  if (ws.bytes < L.total) {
    set_error("render workspace %zu < %zu bytes", ws.bytes, L.total);
    return NG_ERR_CAPACITY;
  }
  char* b = (char*)ws.base;
  ng_ray* rays = user_rays ? (ng_ray*)user_rays : (ng_ray*)(b + L.rays);
  int32_t* hit_list = (int32_t*)(b + L.hit_list);
  // [0] active rays, [1] hits, [2] march work, [3] shadow active, [4] shadow work,
  // [5] probe items claimed, [6] rays finished, [7] march CTAs finished
  unsigned long long* ctr = (unsigned long long*)(b + L.ctr);
  int r;
  int64_t* seg_start = (int64_t*)(b + L.seg_start);
  int64_t* seg_end = (int64_t*)(b + L.seg_end);
  {
    // statistics, counters, the primary traversal's look-back states and the
    // length buckets, in one launch
    ZeroRegions z;
    z.n = 4;
    z.p[0] = st;
    z.bytes[0] = sizeof(ng_frame_stats);
    z.p[1] = ctr;
    z.bytes[1] = 64;
    z.p[2] = b + L.scratch;
    // (the tile traversal uses only its control words at the start)
    z.bytes[2] = use_tile_traverse(cfg.trace_level + tree.n_virtual)
                     ? 512
                     : L.scratch_bytes * (size_t)(cfg.trace_level + tree.n_virtual);
    z.p[3] = b + L.buckets;
    z.bytes[3] = 2 * LEN_BUCKETS * 4;
    z.p[4] = b + L.probe_cnt;
    z.bytes[4] = (size_t)n * 4;
    z.p[5] = b + L.cont;  // tile traversal continuations' ready counts
    z.bytes[5] = tile_cont_ready_bytes();
    z.n = 6;
    k_zero_regions<<<64, 256, 0, s>>>(z);
    NG_CHECK_LAUNCH("k_zero_regions");
  }
  uint8_t bg[3];
  background_u8(cfg, bg);
  const int target0 = cfg.trace_level + tree.n_virtual;
  // the tile traversal writes every ray's segment itself
  int64_t* zseg_s = use_tile_traverse(target0) ? nullptr : seg_start;
  int64_t* zseg_e = use_tile_traverse(target0) ? nullptr : seg_end;
  // with the tile traversal, camera rays are computed where they are used
  // (traversal, march, normals, shadow origins) instead of stored
  const bool cam_rays = cam != nullptr && use_tile_traverse(target0);
  // with camera rays computed on the fly the tile traversal also writes the
  // frame's per-pixel defaults and the root count: no separate ray kernel
  const uint32_t bg_packed = (uint32_t)bg[0] | ((uint32_t)bg[1] << 8) | ((uint32_t)bg[2] << 16);
  if (cam && cam_rays) {
    // (nothing: folded into k_traverse_tiles)
  } else if (cam) {
    k_camera_rays<<<grid_for(n, 256), 256, 0, s>>>(*cam, cam_rays ? nullptr : rays, fr, bg[0], bg[1], bg[2],
                                                   &st->pairs[0], zseg_s, zseg_e);
    NG_CHECK_LAUNCH("k_camera_rays");
  } else {
    k_frame_defaults<<<grid_for(n, 256), 256, 0, s>>>(fr, n, bg[0], bg[1], bg[2], zseg_s, zseg_e);
    NG_CHECK_LAUNCH("k_frame_defaults");
    k_set_count<<<1, 1, 0, s>>>(&st->pairs[0], n);  // root list (i, 0) of n rays
    NG_CHECK_LAUNCH("k_set_count");
  }
  // ---- traversal (traversal.py:207-247) + segments + march setup
  const int target = cfg.trace_level + tree.n_virtual;
  const LodPlan P = plan_lod(cfg);
  MarchArgs A;
  // camera rays share the eye position (a host value, captured into the
  // launches); the tile traversal takes each tile's from its frame's camera,
  // the level passes only when every camera of a batch has the same one
  const double* eye = nullptr;
  if (cam) {
    bool same = true;
    for (int i = 1; i < cam->k; ++i)
      for (int a = 0; a < 3; ++a) same = same && cam->cam[i].position[a] == cam->cam[0].position[a];
    if (same || cam_rays) eye = cam->cam[0].position;
  }
  TileOverflow tov;
  if ((r = trace_pass(tree, cfg, P, rays, n, st->pairs, L, ws, b, ctr + 0, ctr + 2, s, A, true,
                      eye, tov, cam_rays ? cam : nullptr, cam_rays ? &fr : nullptr,
                      bg_packed, cam_rays ? n : -1)))
    return r;
  A.hit = fr.hit;
  A.t = fr.t;
  A.iters = fr.iterations;
  A.evals = fr.evals;
  A.hit_list = hit_list;
  A.d_hit_count = ctr + 1;
  A.counters = &st->counters;
  // normals: probe items inside the march (default), or the k_normals pass
  // after it (NG_FUSED_PROBES=0)
  static const int fused_env = env_int("NG_FUSED_PROBES", 1) != 0;
  const bool fused = do_normals && fused_env;
  A.probes = fused ? 1 : 0;
  A.probe_next = ctr + 5;
  A.rays_done = ctr + 6;
  A.probe_cnt = (unsigned int*)(b + L.probe_cnt);
  A.probe_val = (double*)(b + L.probe_val);
  A.probe_pt = (double*)(b + L.probe_pt);
  A.normal = fr.normal;
  A.normal_ok = fr.normal_ok;
  A.color = cfg.shadows ? nullptr : fr.color;
  if (fused) {  // the statistics are final when the march ends: its last CTA writes them
    A.fin.st = st;
    A.fin.n_levels = target;
    A.fin.pair_cap = ws.pair_capacity;
    A.fin.hit_cap = ws.hit_capacity;
    A.fin.d_hits = ctr + 1;
    A.fin.d_active = ctr + 0;
    A.fin.done = reinterpret_cast<unsigned int*>(ctr + 7);
    A.fin.tov = tov;
  }
  if (ws.ev_march_begin && (r = cuda_status(cudaEventRecord((cudaEvent_t)ws.ev_march_begin, s), "event record")))
    return r;
  if ((r = launch_march(tree, f, A, s))) return r;
  if (ws.ev_trace_done && (r = cuda_status(cudaEventRecord((cudaEvent_t)ws.ev_trace_done, s), "event record")))
    return r;
  // ---- normals + shading (render.py:399-414, 440), when not in the march
  if (do_normals && !fused) {
    NormalArgs B;
    B.cfg = cfg;
    B.G = P.G;
    B.out_mask = P.out_mask;
    B.dec_first = P.dec_first;
    B.dec_last = P.dec_last;
    B.blend_base = P.blend_base;
    B.blend_alpha = P.alpha;
    B.pts = nullptr;
    B.n_pts = 0;
    B.rays = A.rays;
    B.hit_list = hit_list;
    B.d_hit_count = ctr + 1;
    B.t_hit = fr.t;
    B.normal = fr.normal;
    B.ok = fr.normal_ok;
    B.color = cfg.shadows ? nullptr : fr.color;
    B.counters = &st->counters;
    if ((r = launch_normals(tree, f, B, n, s))) return r;
  }
  if (!fused) {
    k_finish_stats<<<1, 1, 0, s>>>(st, target, ws.pair_capacity, ws.hit_capacity, ctr + 1, ctr + 0, tov);
    NG_CHECK_LAUNCH("k_finish_stats");
  }
  // ---- shadow rays toward the light (configs[4]) with the same traversal + march
  if (cfg.shadows && do_normals) {
    ng_ray* srays = (ng_ray*)(b + L.s_rays);
    k_shadow_rays<<<grid_for(n, 256), 256, 0, s>>>(A.rays, hit_list, ctr + 1, fr.t, fr.normal, cfg, srays,
                                                  &st->shadow_pairs[0]);
    NG_CHECK_LAUNCH("k_shadow_rays");
    MarchArgs S;
    TileOverflow stov;
    if ((r = trace_pass(tree, cfg, P, srays, n, st->shadow_pairs, L, ws, b, ctr + 3, ctr + 4, s, S, false,
                        nullptr, stov)))
      return r;
    S.hit = (uint8_t*)(b + L.s_hit);
    // the march writes only the rays that have a voxel segment: clear the rest
    // (a shadow ray that leaves the octree without a segment is unshadowed)
    if ((r = cuda_status(cudaMemsetAsync(S.hit, 0, (size_t)n, s), "shadow hit memset"))) return r;
    S.t = (double*)(b + L.s_t);
    S.iters = (int32_t*)(b + L.s_it);
    S.evals = (int32_t*)(b + L.s_ev);
    S.hit_list = nullptr;
    S.d_hit_count = nullptr;
    S.counters = &st->counters;
    if ((r = launch_march(tree, f, S, s))) return r;
    k_shade_shadowed<<<grid_for(n, 256), 256, 0, s>>>(hit_list, ctr + 1, fr.normal, S.hit, cfg, fr.color,
                                                     &st->shadowed);
    NG_CHECK_LAUNCH("k_shade_shadowed");
    k_shadow_overflow<<<1, 1, 0, s>>>(st, target, ws.pair_capacity, ws.hit_capacity, stov);
    NG_CHECK_LAUNCH("k_shadow_overflow");
  }
  return NG_OK;
}

}  // namespace ng

using namespace ng;

extern "C" {

int ng_camera_rays(const ng_camera* cam, ng_ray* rays, void* stream) {
  const CamSet cs = cam_set(cam, 1);
  const int64_t n = cs.n_per;
  k_camera_rays<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(cs, rays, ng_frame{}, 0, 0, 0, nullptr, nullptr,
                                                                            nullptr);
  NG_CHECK_LAUNCH("ng_camera_rays");
  return NG_OK;
}

// CUDA graphs of a frame's launches, captured on the caller's (non-default)
// stream in thread-local mode and replayed on any stream. Capturing here
// instead of through torch.cuda.graph keeps torch's caching allocators
// intact (its capture empties the device and pinned-host caches and
// synchronises the device), so a streaming loop that meets a new launch
// key does not fall back to cudaMalloc / cudaHostAlloc on every frame.
int ng_graph_capture_begin(void* stream) {
  return cuda_status(cudaStreamBeginCapture((cudaStream_t)stream, cudaStreamCaptureModeThreadLocal),
                     "cudaStreamBeginCapture");
}

int ng_graph_capture_end(void* stream, void** exec_out) {
  cudaGraph_t g = nullptr;
  if (int r = cuda_status(cudaStreamEndCapture((cudaStream_t)stream, &g), "cudaStreamEndCapture")) return r;
  cudaGraphExec_t e = nullptr;
  const int r = cuda_status(cudaGraphInstantiate(&e, g, 0), "cudaGraphInstantiate");
  cudaGraphDestroy(g);
  if (r) return r;
  *exec_out = (void*)e;
  return NG_OK;
}

int ng_graph_launch(void* exec, void* stream) {
  return cuda_status(cudaGraphLaunch((cudaGraphExec_t)exec, (cudaStream_t)stream), "cudaGraphLaunch");
}

int ng_graph_destroy(void* exec) {
  if (exec) cudaGraphExecDestroy((cudaGraphExec_t)exec);
  return NG_OK;
}

size_t ng_render_workspace_bytes(int64_t n_rays, int64_t pair_capacity, int64_t hit_capacity) {
  return layout(n_rays, pair_capacity, hit_capacity).total;
}

int ng_render_workspace_offsets(int64_t n_rays, int64_t pair_capacity, int64_t hit_capacity, int64_t* out,
                                int32_t n_out) {
  if (!out || n_out < 0 || n_rays < 0) {
    set_error("bad workspace-offset arguments");
    return NG_ERR_STRUCTURAL;
  }
  const WsLayout L = layout(n_rays, pair_capacity, hit_capacity);
  const int64_t v[5] = {(int64_t)L.hits, (int64_t)L.seg_start, (int64_t)L.seg_end, (int64_t)L.total,
                        (int64_t)L.scratch};
  for (int i = 0; i < n_out && i < 5; ++i) out[i] = v[i];
  return NG_OK;
}

int ng_render_frame(const ng_octree* tree, const ng_field* fld, const ng_render_cfg* cfg, const ng_camera* cam,
                    const ng_frame* frame, const ng_workspace* ws, ng_frame_stats* d_stats, void* stream) {
  return ng_render_batch(tree, fld, cfg, cam, 1, frame, ws, d_stats, stream);
}

int ng_render_batch(const ng_octree* tree, const ng_field* fld, const ng_render_cfg* cfg, const ng_camera* cams,
                    int32_t n_cams, const ng_frame* frame, const ng_workspace* ws, ng_frame_stats* d_stats,
                    void* stream) {
  if (!cams || n_cams < 1 || n_cams > NG_MAX_BATCH) {
    set_error("a batch holds 1..%d cameras, got %d", NG_MAX_BATCH, (int)n_cams);
    return NG_ERR_CONFIG;
  }
  const ng_camera& c0 = cams[0];
  if (c0.width < 1 || c0.local_rows < 0 || c0.band_rows < 1 || c0.band_stride < 1 || c0.band_offset < 0 ||
      c0.band_offset >= c0.band_stride) {
    set_error("bad camera band layout");
    return NG_ERR_CONFIG;
  }
  for (int i = 1; i < n_cams; ++i) {
    const ng_camera& c = cams[i];
    if (c.width != c0.width || c.height != c0.height || c.band_rows != c0.band_rows ||
        c.band_stride != c0.band_stride || c.band_offset != c0.band_offset || c.local_rows != c0.local_rows) {
      set_error("batch camera %d: size or band layout differs from camera 0", i);
      return NG_ERR_CONFIG;
    }
  }
  const CamSet cs = cam_set(cams, n_cams);
  return render_common(*tree, *fld, *cfg, &cs, nullptr, cs.n_per * n_cams, *frame, *ws, d_stats, true,
                       (cudaStream_t)stream);
}

int ng_render_rays(const ng_octree* tree, const ng_field* fld, const ng_render_cfg* cfg, const ng_ray* rays,
                   int64_t n_rays, const ng_frame* frame, const ng_workspace* ws, ng_frame_stats* d_stats,
                   int32_t do_normals, void* stream) {
  return render_common(*tree, *fld, *cfg, nullptr, rays, n_rays, *frame, *ws, d_stats, do_normals != 0,
                       (cudaStream_t)stream);
}

int ng_sphere_trace(const ng_octree* tree, const ng_field* fld, const ng_render_cfg* cfg, const ng_ray* rays,
                    int64_t n_rays, const ng_hit_pair* hits, const int64_t* d_hit_count,
                    const int64_t* seg_start, const int64_t* seg_end, uint8_t* hit, double* t_hit,
                    int32_t* iters, int32_t* evals, ng_counters* d_counters, void* stream) {
  if (n_rays <= 0) return NG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* work = nullptr;
  int r = malloc_async((void**)&work, 8, s, "ng_sphere_trace alloc");
  if (r) return r;
  if ((r = cuda_status(cudaMemsetAsync(work, 0, 8, s), "ng_sphere_trace memset"))) return r;
  const LodPlan P = plan_lod(*cfg);
  MarchArgs A;
  A.cfg = *cfg;
  A.G = P.G;
  A.out_mask = P.out_mask;
  A.dec_first = P.dec_first;
  A.dec_last = P.dec_last;
  A.passes = P.passes;
  A.blend_base = P.blend_base;
  A.blend_alpha = P.alpha;
  A.rays.rays = rays;
  A.rays.cam_rays = 0;
  A.work = nullptr;
  A.items = nullptr;
  A.d_n_work = nullptr;
  A.n_work = n_rays;
  A.hits = hits;
  A.pair_cells = 0;
  A.seg_start = seg_start;
  A.seg_end = seg_end;
  A.hit = hit;
  A.t = t_hit;
  A.iters = iters;
  A.evals = evals;
  A.hit_list = nullptr;
  A.d_hit_count = nullptr;
  A.work_counter = work;
  A.counters = d_counters;
  A.prof = nullptr;
  A.probes = 0;
  A.fin.st = nullptr;
  (void)d_hit_count;
  r = launch_march(*tree, *fld, A, s);
  cudaFreeAsync(work, s);
  return r;
}

int ng_normals(const ng_octree* tree, const ng_field* fld, const ng_render_cfg* cfg, const double* pts, int64_t k,
               double* normal, uint8_t* ok, ng_counters* d_counters, void* stream) {
  if (k <= 0) return NG_OK;
  const LodPlan P = plan_lod(*cfg);
  NormalArgs B;
  B.cfg = *cfg;
  B.G = P.G;
  B.out_mask = P.out_mask;
  B.dec_first = P.dec_first;
  B.dec_last = P.dec_last;
  B.blend_base = P.blend_base;
  B.blend_alpha = P.alpha;
  B.pts = pts;
  B.n_pts = k;
  B.rays.rays = nullptr;
  B.rays.cam_rays = 0;
  B.hit_list = nullptr;
  B.d_hit_count = nullptr;
  B.t_hit = nullptr;
  B.normal = normal;
  B.ok = ok;
  B.color = nullptr;
  B.counters = d_counters;
  return launch_normals(*tree, *fld, B, k, (cudaStream_t)stream);
}

int ng_shade(const uint8_t* hit, const double* normal, int64_t n, const ng_render_cfg* cfg, uint8_t* color,
             void* stream) {
  if (n <= 0) return NG_OK;
  k_shade<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(hit, normal, n, *cfg, color);
  NG_CHECK_LAUNCH("ng_shade");
  return NG_OK;
}

// Debug: copy the march profile (NG_PROF_SLOTS x uint64 per group: steps,
// busy lanes, first/last globaltimer ns, then the phase clocks listed in
// tools/march_profile.py) and reset it; 0 groups when profiling is off.
int ng_march_profile(unsigned long long* host_out, int max_groups) {
  if (!g_prof) return 0;
  cudaDeviceSynchronize();
  const int n = max_groups < 4096 ? max_groups : 4096;
  cudaMemcpy(host_out, g_prof, (size_t)n * 8 * NG_PROF_SLOTS, cudaMemcpyDeviceToHost);
  cudaMemset(g_prof, 0, 8 * NG_PROF_SLOTS * 4096);
  return n;
}

int ng_hit_points(const ng_ray* rays, const uint8_t* hit, const double* t, int64_t n, double* points,
                  void* stream) {
  if (n <= 0) return NG_OK;
  k_hit_points<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(rays, hit, t, n, points);
  NG_CHECK_LAUNCH("ng_hit_points");
  return NG_OK;
}

}  // extern "C"
