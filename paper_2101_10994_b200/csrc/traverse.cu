// Breadth-first ray-octree traversal (traversal.py:95-255, paper Alg. 1).
//
// One kernel per level fuses decide + exclusive scan + subdivide (or the
// final compactify): each persistent CTA takes tiles of (ray, voxel) pairs
// in order, runs the fp64 slab test, scans the per-pair child counts in
// shared memory, resolves its global offset with a decoupled look-back and
// writes the children front to back. List order is therefore identical to
// the reference's (grouped by ray, parents in order, children by octant ^
// direction mask), and every count stays on the device so a whole frame can
// be captured in one CUDA graph.
#include "common.cuh"

#include <algorithm>
#include <cstdlib>

namespace ng {

constexpr int TR_NT = 256;
constexpr int TR_ITEMS = 4;   // candidate passes (API path)
constexpr int TH_ITEMS = 4;   // hit-filtered passes (render path)

template <bool FINAL>
__global__ void __launch_bounds__(TR_NT) k_traverse_level(
    const __grid_constant__ ng_octree tree, const ng_ray* __restrict__ rays, int t,
    const ng_pair* __restrict__ in, const int64_t* __restrict__ d_count_in, int64_t in_cap,
    ng_pair* __restrict__ out_pairs, ng_hit_pair* __restrict__ out_hits,
    int64_t* __restrict__ d_count_out, int64_t out_cap, unsigned long long* states,
    unsigned int* tile_counter) {
  __shared__ int64_t sm_warp[TR_NT / 32 + 1];
  __shared__ int64_t sm_tile, sm_excl;
  int64_t n = *d_count_in;
  if (in != nullptr && n > in_cap) n = in_cap;
  const int level = t - tree.n_virtual;
  const int res = level_res(tree, level);
  const double edge = 2.0 / (double)res;
  const uint64_t* __restrict__ codes = tree.codes[t];
  const int32_t* __restrict__ cstart = FINAL ? nullptr : tree.child_start[t];
  const uint8_t* __restrict__ cmask = FINAL ? nullptr : tree.child_mask[t];
  const int64_t tile_elems = (int64_t)TR_NT * TR_ITEMS;
  const int64_t n_tiles = (n + tile_elems - 1) / tile_elems;
  if (n_tiles == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *d_count_out = 0;
    return;
  }
  while (true) {
    if (threadIdx.x == 0) sm_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const int64_t tile = sm_tile;
    if (tile >= n_tiles) break;
    const int64_t base = tile * tile_elems + (int64_t)threadIdx.x * TR_ITEMS;
    int32_t pr[TR_ITEMS], pv[TR_ITEMS], dmask[TR_ITEMS];
    int cnt[TR_ITEMS];
    double te[TR_ITEMS], tx[TR_ITEMS];
    int64_t sum = 0;
#pragma unroll
    for (int q = 0; q < TR_ITEMS; ++q) {
      const int64_t i = base + q;
      cnt[q] = 0;
      pr[q] = 0;
      pv[q] = 0;
      dmask[q] = 0;
      te[q] = 0.0;
      tx[q] = 0.0;
      if (i < n) {
        if (in != nullptr) {
          ng_pair p = in[i];
          pr[q] = p.ray;
          pv[q] = p.voxel;
        } else {
          pr[q] = (int32_t)i;
          pv[q] = 0;
        }
        ng_ray r;
        load_ray(rays, pr[q], r);
        dmask[q] = r.flags & 7;
        const uint64_t c = __ldg(codes + pv[q]);
        double lo[3], hi[3];
        lo[0] = cell_lo((int)compact3(c), res);
        lo[1] = cell_lo((int)compact3(c >> 1), res);
        lo[2] = cell_lo((int)compact3(c >> 2), res);
#pragma unroll
        for (int a = 0; a < 3; ++a) hi[a] = dadd(lo[a], edge);
        bool hit = slab_test(r, lo, hi, te[q], tx[q]);
        if (FINAL) {
          cnt[q] = hit ? 1 : 0;
        } else {
          cnt[q] = hit ? __popc((unsigned)__ldg(cmask + pv[q])) : 0;
        }
      }
      sum += cnt[q];
    }
    int64_t excl;
    const int64_t agg = block_excl_scan<TR_NT>(sum, excl, sm_warp);
    if (threadIdx.x < 32) {
      const int64_t e = tile_lookback_warp(states, tile, agg);
      if (threadIdx.x == 0) sm_excl = e;
    }
    __syncthreads();
    int64_t o = sm_excl + excl;
#pragma unroll
    for (int q = 0; q < TR_ITEMS; ++q) {
      if (cnt[q]) {
        if (FINAL) {
          if (o < out_cap) {
            ng_hit_pair h;
            h.ray = pr[q];
            h.voxel = pv[q];
            h.t_enter = te[q];
            h.t_exit = tx[q];
            out_hits[o] = h;
          }
          o += 1;
        } else {
          const unsigned m = __ldg(cmask + pv[q]);
          const int32_t first = __ldg(cstart + pv[q]);
          // front-to-back: octant k ^ dmask for k = 0..7 (traversal.py:32-37, 185-187)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int oct = k ^ dmask[q];
            if ((m >> oct) & 1u) {
              if (o < out_cap) {
                ng_pair p;
                p.ray = pr[q];
                p.voxel = first + __popc(m & ((1u << oct) - 1u));
                out_pairs[o] = p;
              }
              ++o;
            }
          }
        }
      }
    }
    if (tile == n_tiles - 1 && threadIdx.x == TR_NT - 1) *d_count_out = o;
    __syncthreads();
  }
}

// ray_segments (traversal.py:250-255): per-ray lower / upper bound of the ray
// id in the (ray-sorted) final list, so rays without pairs get the same
// insertion position numpy's searchsorted reports.
// Render-path variant of one BFS pass: the input pairs at level t are
// already known hits (or the implicit root list, tested here); each pair's
// occupied children are slab-tested in the parent's thread, front to back,
// and only hit children are written. The final hit list is therefore the
// same sequence the reference produces (its candidate lists filtered in
// order), with a fraction of the pair traffic: the ray record is read once
// per hit parent instead of once per candidate child.
template <bool NEXT_FINAL>
__global__ void __launch_bounds__(TR_NT) k_traverse_hits(
    const __grid_constant__ ng_octree tree, const ng_ray* __restrict__ rays, int t,
    const ng_pair* __restrict__ in, const int64_t* __restrict__ d_count_in, int64_t in_cap,
    ng_pair* __restrict__ out_pairs, ng_hit_pair* __restrict__ out_hits,
    int64_t* __restrict__ d_count_out, int64_t out_cap, unsigned long long* states,
    unsigned int* tile_counter, int64_t* __restrict__ seg_start, int64_t* __restrict__ seg_end,
    const SharedOrigin so) {
  __shared__ int64_t sm_warp[TR_NT / 32 + 1];
  __shared__ int64_t sm_tile, sm_excl;
  int64_t n = *d_count_in;
  if (in != nullptr && n > in_cap) n = in_cap;
  const int level = t - tree.n_virtual;
  const int cres = level_res(tree, level + 1);
  const uint64_t* __restrict__ codes = tree.codes[t];
  const int32_t* __restrict__ cstart = tree.child_start[t];
  const uint8_t* __restrict__ cmask = tree.child_mask[t];
  const int64_t tile_elems = (int64_t)TR_NT * TH_ITEMS;
  const int64_t n_tiles = (n + tile_elems - 1) / tile_elems;
  if (n_tiles == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *d_count_out = 0;
    return;
  }
  while (true) {
    if (threadIdx.x == 0) sm_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const int64_t tile = sm_tile;
    if (tile >= n_tiles) break;
    const int64_t base = tile * tile_elems + (int64_t)threadIdx.x * TH_ITEMS;
    int32_t pr[TH_ITEMS], pv[TH_ITEMS];
    unsigned hm[TH_ITEMS];  // bit k: k-th front-to-back child is hit
    int64_t sum = 0;
#pragma unroll
    for (int q = 0; q < TH_ITEMS; ++q) {
      const int64_t i = base + q;
      hm[q] = 0;
      pr[q] = 0;
      pv[q] = 0;
      if (i < n) {
        ng_ray r;
        bool parent_hit = true;
        if (in != nullptr) {
          const ng_pair p = in[i];
          pr[q] = p.ray;
          pv[q] = p.voxel;
          load_ray_slab(rays, pr[q], so, r);
        } else {  // implicit root list: the root box itself must be hit
          pr[q] = (int32_t)i;
          load_ray_slab(rays, pr[q], so, r);
          const double lo[3] = {-1.0, -1.0, -1.0}, hi[3] = {1.0, 1.0, 1.0};
          double a, b;
          parent_hit = slab_test(r, lo, hi, a, b);
        }
        if (parent_hit) {
          const unsigned m = __ldg(cmask + pv[q]);
          const uint64_t c = __ldg(codes + pv[q]);
          const int px = (int)compact3(c), py = (int)compact3(c >> 1), pz = (int)compact3(c >> 2);
          const int dm = r.flags & 7;
          ChildSlabs cs;
          child_slabs(r, px, py, pz, cres, cs);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int oct = k ^ dm;
            double a0, b0;
            if (((m >> oct) & 1u) && child_hit(cs, oct, a0, b0)) hm[q] |= 1u << k;
          }
          // the emit pass needs only the direction mask and the child mask
          // (and, for the final level, the slabs again): keep them packed
          if (hm[q]) hm[q] |= ((unsigned)dm << 8) | (m << 16);
        }
      }
      sum += __popc(hm[q] & 0xffu);
    }
    int64_t excl;
    const int64_t agg = block_excl_scan<TR_NT>(sum, excl, sm_warp);
    if (threadIdx.x < 32) {
      const int64_t e = tile_lookback_warp(states, tile, agg);
      if (threadIdx.x == 0) sm_excl = e;
    }
    __syncthreads();
    int64_t o = sm_excl + excl;
#pragma unroll
    for (int q = 0; q < TH_ITEMS; ++q) {
      // final level: each ray's [start, end) in the hit list (ray_segments,
      // traversal.py:250-255). A ray's pairs are contiguous in the input, so
      // its first pair knows the start and its last pair the end.
      if (NEXT_FINAL && seg_start != nullptr && base + q < n) {
        const int64_t i = base + q;
        const int32_t r = pr[q];
        const bool first = in == nullptr || i == 0 || in[i - 1].ray != r;
        const bool last = in == nullptr || i == n - 1 || in[i + 1].ray != r;
        if (first) seg_start[r] = o < out_cap ? o : out_cap;
        if (last) {
          const int64_t e = o + __popc(hm[q] & 0xffu);
          seg_end[r] = e < out_cap ? e : out_cap;
        }
      }
      if (!hm[q]) continue;
      const int dm = (int)((hm[q] >> 8) & 7u);
      const unsigned m = (hm[q] >> 16) & 0xffu;
      const int32_t first = __ldg(cstart + pv[q]);
      ChildSlabs cs;
      if (NEXT_FINAL) {
        ng_ray r;
        load_ray_slab(rays, pr[q], so, r);
        const uint64_t c = __ldg(codes + pv[q]);
        child_slabs(r, (int)compact3(c), (int)compact3(c >> 1), (int)compact3(c >> 2), cres, cs);
      }
      for (unsigned bits = hm[q] & 0xffu; bits; bits &= bits - 1) {
        const int k = __ffs(bits) - 1;
        const int oct = k ^ dm;
        const int32_t child = first + __popc(m & ((1u << oct) - 1u));
        if (o < out_cap) {
          if (NEXT_FINAL) {
            ng_hit_pair h;
            h.ray = pr[q];
            h.voxel = child;
            child_hit(cs, oct, h.t_enter, h.t_exit);
            out_hits[o] = h;
          } else {
            out_pairs[o] = ng_pair{pr[q], child};
          }
        }
        ++o;
      }
    }
    if (tile == n_tiles - 1 && threadIdx.x == TR_NT - 1) *d_count_out = o;
    __syncthreads();
  }
}

// Render-path traversal of a whole ray tile in one warp (all levels, one
// launch). A warp takes TT_RAYS consecutive rays and runs the same
// hit-filtered breadth-first passes as k_traverse_hits over its own pair
// lists, kept in shared memory (spilling to a per-warp global arena for
// silhouette tiles): decide + scan + subdivide become warp shuffles, with no
// grid-wide look-back and no launch per level. Each ray's final pairs come
// out in the reference's order (parents in list order, children front to
// back), so per-ray segments are the reference's sub-lists; only the
// placement of a tile's block in the final list depends on when the warp
// claims it (one atomic per tile), which the march does not see. The march
// knows each pair's ray from the segment it walks, so the `ray` field of
// these render lists carries the voxel's packed cell coordinates instead.
#ifndef NG_TT_RAYS
#define NG_TT_RAYS 32
#endif
#ifndef NG_TT_SCAP
#define NG_TT_SCAP 768  // 2 CTAs of 8 warps per SM at 14.2 KB per warp
#endif
#ifndef NG_TT_ITEMS
#define NG_TT_ITEMS 2
#endif
#ifndef NG_TT_WPB
#define NG_TT_WPB 8
#endif
#ifndef NG_TT_MINB
#define NG_TT_MINB 2  // CTAs per SM the register budget is sized for (1 lets ptxas take 150 registers: half the warps)
#endif
constexpr int TT_WPB = NG_TT_WPB;      // warps per CTA
constexpr int TT_RAYS = NG_TT_RAYS;    // rays per tile (<= 32: the ray slot is 5 bits of a list entry)
constexpr int TT_SCAP = NG_TT_SCAP;    // pairs per warp-local list held in shared memory
constexpr int TT_ITEMS = NG_TT_ITEMS;  // pairs per lane per round
constexpr int TT_ENTRY = 8;            // list entry: voxel i32 | cell x, y, z (9 bits each) + ray slot << 27
static_assert(TT_RAYS <= 32, "list entries keep a 5-bit ray slot");

struct TileWarp {
  double o[TT_RAYS][3];  // per-ray origins (unused when the rays share one)
  double inv[TT_RAYS][3];
  int flags[TT_RAYS];
  int seg_s[TT_RAYS], seg_e[TT_RAYS];
  int2 ent[2][TT_SCAP];
};

// A warp's pair list: entries in shared memory, the rest in its arena share.
// Cells are packed x | y << 9 | z << 18 (<= 512 per axis at the list's level).
struct TileList {
  int scap;  // entries held in shared memory (<= TT_SCAP)
  int2* s;
  int2* g;
};

__device__ __forceinline__ void tl_put(const TileList& b, int i, int32_t v, uint32_t c, int r, int64_t gcap) {
  const int2 e = make_int2(v, (int)(c | ((uint32_t)r << 27)));
  if (i < b.scap) b.s[i] = e;
  else if (i - b.scap < gcap) b.g[i - b.scap] = e;
}

__device__ __forceinline__ void tl_get(const TileList& b, int i, int32_t& v, uint32_t& c, int& r) {
  const int2 e = i < b.scap ? b.s[i] : b.g[i - b.scap];
  v = e.x;
  c = (uint32_t)e.y & 0x7ffffffu;
  r = (int)((uint32_t)e.y >> 27);
}

__device__ __forceinline__ int tl_ray(const TileList& b, int i) {
  const int y = i < b.scap ? b.s[i].y : b.g[i - b.scap].y;
  return (int)((uint32_t)y >> 27);
}

// arena per warp: [list 0 | list 1], gcap entries each
__device__ __forceinline__ TileList tile_list(TileWarp* W, uint8_t* ga, int64_t gcap, int k, int scap) {
  TileList b;
  b.scap = scap;
  b.s = W->ent[k];
  b.g = reinterpret_cast<int2*>(ga) + k * gcap;
  return b;
}

template <bool SO>
__device__ __forceinline__ void tw_ray(const TileWarp* W, const SharedOrigin& so, int rl, ng_ray& r) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    r.o[a] = SO ? so.o[a] : W->o[rl][a];
    r.inv[a] = W->inv[rl][a];
    r.d[a] = 0.0;
  }
  r.flags = W->flags[rl] & 0xff;
  r.pad = 0;
}

// ray flag: finite origin, finite nonzero direction on every axis (then no
// slab value is NaN and none of the zero-direction rules applies)
constexpr int TT_GENERAL = 1 << 8;

// Per-axis plane crossings of a cell's two child halves, in ray order:
// q0 <= q1 <= q2 are t at the near face, the mid plane and the far face.
// The planes are exact dyadic values and (p - o) * inv is monotone in p, so
// these are the reference's t1 / t2 of each child box, sorted.
__device__ __forceinline__ void axis_crossings(double o, double inv, bool neg, int pc, int cres, double& q0,
                                               double& q1, double& q2) {
  const double h = 2.0 / (double)cres;
  const double pf = dmul((double)(2 * pc + (neg ? 2 : 0) - cres / 2), h);  // -1 + e h, exact
  const double hs = neg ? -h : h;
  const double pm = dadd(pf, hs), pl = dadd(pm, hs);
  q0 = dmul(dsub(pf, o), inv);
  q1 = dmul(dsub(pm, o), inv);
  q2 = dmul(dsub(pl, o), inv);
}

// Hit bits of the 8 children of a hit parent cell, bit k = the k-th child
// front to back (octant k ^ dm), for a TT_GENERAL ray. Child k has per-axis
// interval [k_a ? q1 : q0, k_a ? q2 : q1]; ray_aabb_batch's test
// max(near) <= min(far) && min(far) >= 0 is the set of pairwise conditions
// near_a <= far_b and far_b >= 0. Those implied by the parent's own hit
// (max q0 <= min q2, min q2 >= 0: the same plane values) or by q0 <= q1 <= q2
// are dropped, leaving 21 comparisons.
__device__ __forceinline__ unsigned child_hits_ordered(const double q0[3], const double q1[3], const double q2[3]) {
  // children with local half v on axis a
  auto half = [](int a, int v) -> unsigned {
    const unsigned lo = a == 0 ? 0x55u : (a == 1 ? 0x33u : 0x0fu);
    return v ? (~lo & 0xffu) : lo;
  };
  unsigned mask = 0xffu;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      if (a == b) continue;
      if (!(q0[a] <= q1[b])) mask &= ~(half(a, 0) & half(b, 0));
      if (!(q1[a] <= q2[b])) mask &= ~(half(a, 1) & half(b, 1));
      if (!(q1[a] <= q1[b])) mask &= ~(half(a, 1) & half(b, 0));
    }
    if (!(q1[a] >= 0.0)) mask &= ~half(a, 0);
  }
  return mask;
}

// The literal child tests (child_slabs / child_hit, numpy's NaN rules) for
// the rare rays the ordered test excludes. Out of line, so the compiler
// cannot if-convert it into every item's instruction stream.
__device__ __noinline__ unsigned literal_child_hits(const ng_ray r, int px, int py, int pz, int cres) {
  ChildSlabs cs;
  child_slabs(r, px, py, pz, cres, cs);
  unsigned ho = 0;
#pragma unroll
  for (int oct = 0; oct < 8; ++oct) {
    double a0, b0;
    if (child_hit(cs, oct, a0, b0)) ho |= 1u << oct;
  }
  return ho;
}

// The literal slab values of one box (slab_test), out of line as above.
__device__ __noinline__ void literal_slab(const ng_ray r, const int cc[3], int res, double& t_enter, double& t_exit) {
  const double edge = 2.0 / (double)res;
  double lo[3], hi[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = cell_lo(cc[a], res);
    hi[a] = dadd(lo[a], edge);
  }
  slab_test(r, lo, hi, t_enter, t_exit);
}

// ray_aabb_batch's hit decision for a general ray (finite origin, finite
// nonzero 1/d): per axis the face crossings in ray order (monotone in the
// plane), then max(near) <= min(far) && min(far) >= 0; no NaN can occur.
__device__ __forceinline__ bool box_hit_ordered(const ng_ray& r, const double lo[3], const double hi[3]) {
  double ne = 0.0, fa = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const bool neg = (r.flags >> a) & 1;
    const double tn = dmul(dsub(neg ? hi[a] : lo[a], r.o[a]), r.inv[a]);
    const double tf = dmul(dsub(neg ? lo[a] : hi[a], r.o[a]), r.inv[a]);
    ne = a == 0 ? tn : (tn > ne ? tn : ne);
    fa = a == 0 ? tf : (tf < fa ? tf : fa);
  }
  return ne <= fa && fa >= 0.0;
}

// Octant-indexed bits -> front-to-back order: bit k <- bit k ^ dm.
__device__ __forceinline__ unsigned octants_front_to_back(unsigned x, int dm) {
  if (dm & 1) x = ((x & 0x55u) << 1) | ((x >> 1) & 0x55u);
  if (dm & 2) x = ((x & 0x33u) << 2) | ((x >> 2) & 0x33u);
  if (dm & 4) x = ((x & 0x0fu) << 4) | ((x >> 4) & 0x0fu);
  return x;
}


// Splitting silhouette tiles. A tile's time is proportional to its pairs
// (one warp runs every round), so a few grazing tiles (~3,000 final pairs,
// ~190 us) outlast all the others when a frame has few tiles per warp (a
// band of an N-GPU frame). After a level pass, a list longer than
// NG_TILE_SPLIT entries that covers several rays is cut at a ray boundary near
// its middle: the warp keeps the first rays and publishes the rest (their
// entries copied to a pool) as a continuation that any warp takes before a
// fresh tile. A ray's pairs stay in one part, and each part claims its own
// block of the hit list, so every ray's segment is still the reference's
// sub-list in order (traversal.py:207-247); only block placement changes.
// Run-time knobs (read once per process): NG_TILE_SPLIT, the list length
// above which a list is split (default 256; a huge value disables
// splitting), and NG_TILE_SPLIT_AHEAD, tiles per warp before the last tile
// is claimed at which splitting starts (default 0; the tests set both low
// to split every tile they can).
constexpr int TT_CONT_RECS = 16384;         // continuation records per pass
#ifndef NG_TT_HELPERS
#define NG_TT_HELPERS 2
#endif
constexpr int TT_HELPERS = NG_TT_HELPERS;   // warps per CTA that wait for continuations when idle
constexpr int64_t TT_CONT_POOL = 2 << 20;   // pooled list entries per pass
struct TileCont {
  int64_t r0;        // the tile's first ray
  int64_t pool_off;  // its entries in the pool
  int32_t nr, ja, jb;  // tile rays; the continuation's ray slots [ja, jb)
  int32_t pass;      // the next level pass
  int32_t count;     // entries
  int32_t pad;
};
// `cont` layout: per-record ready counts (u32, zeroed before every pass:
// each of the pushing warp's 32 lanes adds 1 with release after its pool
// stores), the records, the entry pool
size_t tile_cont_ready_bytes() { return (size_t)TT_CONT_RECS * 4; }
size_t tile_cont_bytes() {
  return tile_cont_ready_bytes() + (size_t)TT_CONT_RECS * sizeof(TileCont) + (size_t)TT_CONT_POOL * 8;
}

#ifdef NG_PROFILE
// NG_PROFILE builds: per tile (globaltimer start, end, final pairs, warp) for
// tools/tile_profile.py (ng_tile_profile_enable / ng_tile_profile_read)
__device__ unsigned long long* g_tile_prof = nullptr;
__device__ long long g_tile_prof_cap = 0;
__device__ unsigned long long* g_part_prof = nullptr;  // 8 words per part
__device__ unsigned int g_part_next = 0;
#endif

template <bool SO>
__global__ void __launch_bounds__(TT_WPB * 32, NG_TT_MINB) k_traverse_tiles(
    const __grid_constant__ ng_octree tree, const ng_ray* __restrict__ rays, const int64_t* __restrict__ d_n,
    int target, int64_t* counts, ng_hit_pair* __restrict__ hits, int64_t hit_cap, unsigned int* tile_counter,
    unsigned long long* hit_cursor, int64_t* __restrict__ seg_start, int64_t* __restrict__ seg_end,
    uint8_t* arena, int64_t gcap, int scap, unsigned long long* d_need, const SharedOrigin so0,
    const __grid_constant__ CamSet cams, int cam_rays, int4* __restrict__ items, unsigned long long* d_active,
    const ng_frame fr, uint32_t bg, int64_t n_host, int cull, uint8_t* __restrict__ cont, int split_at,
    int split_ahead) {
  extern __shared__ __align__(16) uint8_t tt_smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  TileWarp* W = reinterpret_cast<TileWarp*>(tt_smem) + warp;
  const int64_t gw = (int64_t)blockIdx.x * TT_WPB + warp;
  uint8_t* ga = arena + gw * gcap * (2 * TT_ENTRY);
  // the ray count: the caller's (then published as the root list length), or
  // the device count (shadow rays)
  const int64_t n = n_host >= 0 ? n_host : *d_n;
  if (n_host >= 0 && blockIdx.x == 0 && threadIdx.x == 0) *const_cast<int64_t*>(d_n) = n_host;
  // tiles never span two frames of a batch (each frame's camera is its
  // tiles' shared origin): frame f's tiles are [f tpf, (f + 1) tpf)
  const int64_t n_per = cam_rays ? cams.n_per : n;
  const int64_t tpf = (n_per + TT_RAYS - 1) / TT_RAYS;
  const int64_t n_tiles = (cam_rays ? cams.k : 1) * tpf;
  const int lim = scap + (int)gcap;
  int64_t level_cnt = 0;  // lane t: pairs emitted at traversal level t
  int need = 0;
  // continuation queue (control words after the tile counter, hit cursor
  // and longest list, zeroed with them, each group on its own 128-byte
  // line): `qstate` = records pushed << 32 | continuations finished (one
  // word, so one load is a consistent snapshot), the claim cursor, fresh
  // tiles finished, pool entries used
  unsigned long long* qstate = reinterpret_cast<unsigned long long*>(tile_counter + 32);
  unsigned int* q_head = tile_counter + 64;
  unsigned int* tiles_done = tile_counter + 96;
  unsigned int* pool_top = tile_counter + 16;
  unsigned int* ready = reinterpret_cast<unsigned int*>(cont);
  TileCont* recs = reinterpret_cast<TileCont*>(cont + (size_t)TT_CONT_RECS * 4);
  int2* pool = reinterpret_cast<int2*>(cont + (size_t)TT_CONT_RECS * (4 + sizeof(TileCont)));
  bool tiles_left = true;
  while (true) {
    // ---- work: a fresh tile while any is left (continuations only appear
    // once every tile is claimed), then published continuations; idle
    // helper warps wait while a part may still split
    int rec = -1;
    unsigned int tile = 0xffffffffu;
    if (lane == 0) {
      if (tiles_left) {
        tile = atomicAdd(tile_counter, 1u);
        if ((int64_t)tile >= n_tiles) {
          tiles_left = false;
          tile = 0xffffffffu;
        }
      }
      if (!tiles_left) {
        unsigned backoff = 256;
        int ticket = -1;  // a claimed queue position, served once published
        while (true) {
          const unsigned long long qs = *(volatile unsigned long long*)qstate;
          const unsigned tl = (unsigned)(qs >> 32), fin = (unsigned)qs;
          if (ticket < 0 && *(volatile unsigned*)q_head < tl) {
            ticket = (int)atomicAdd(q_head, 1u);  // (fetch-add: a CAS loop serialised the claims)
            if (ticket >= TT_CONT_RECS) ticket = INT_MAX;  // past the last record: never served
          }
          if (ticket >= 0 && (unsigned)ticket < tl) {
            rec = ticket;
            break;
          }
          // every part finished (fresh tiles, then every pushed continuation:
          // a push precedes its pusher's own finish) -> nothing can be pushed
          const bool all_done = *(volatile unsigned*)tiles_done >= (unsigned)n_tiles && fin == tl;
          if (ticket < 0 ? (warp >= TT_HELPERS || (all_done && *(volatile unsigned*)q_head >= tl)) : all_done)
            break;  // (non-helper warps leave when idle; a ticket is kept until served or moot)
          __nanosleep(backoff);
          backoff = backoff < 8192 ? 2 * backoff : backoff;
        }
      }
    }
    rec = __shfl_sync(FULL, rec, 0);
    tile = __shfl_sync(FULL, tile, 0);
    tiles_left = __shfl_sync(FULL, tiles_left, 0);
    if (rec < 0 && tile == 0xffffffffu) break;
#ifdef NG_PROFILE
    unsigned long long tp0 = 0;
    if (lane == 0) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tp0));
#endif
    int64_t r0;
    int nr, ja = 0, jb, t0 = 0;
    int nc = 0;
    int fcam = 0;        // the tile's frame (camera) in a batch
    SharedOrigin so = so0;
#ifdef NG_PROFILE
    int n_splits = 0;
    unsigned long long split_ns = 0;
#endif
    if (rec >= 0) {
      // ---- a continuation: its rays' slab data, its list at pass t0
      const TileCont* cr = recs + rec;
      if (lane == 0)
        while (ld_relaxed_u32(ready + rec) < 32u) __nanosleep(64);
      __syncwarp();
      r0 = __ldcg(&cr->r0);
      nr = __ldcg(&cr->nr);
      if (cam_rays) {
        fcam = cams.frame_of(r0);
#pragma unroll
        for (int a = 0; a < 3; ++a) so.o[a] = cams.cam[fcam].position[a];
      }
      ja = __ldcg(&cr->ja);
      jb = __ldcg(&cr->jb);
      t0 = __ldcg(&cr->pass);
      nc = __ldcg(&cr->count);
      const int64_t off = __ldcg(&cr->pool_off);
#pragma unroll
      for (int j0 = 0; j0 < TT_RAYS; j0 += 32) {
        const int j = j0 + lane;
        if (j >= ja && j < jb) {
          ng_ray r;
          if (SO && cam_rays) camera_ray(cams.cam[fcam], r0 - fcam * n_per + j, r);
          else load_ray_slab(rays, r0 + j, so, r);
          bool general = true;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            if (!SO) W->o[j][a] = r.o[a];
            W->inv[j][a] = r.inv[a];
            general = general && isfinite(r.o[a]) && isfinite(r.inv[a]) && !((r.flags >> (3 + a)) & 1);
          }
          W->flags[j] = r.flags | (general ? TT_GENERAL : 0);
        }
        W->seg_s[j] = 0;
        W->seg_e[j] = 0;
      }
      const TileList L0 = tile_list(W, ga, gcap, t0 & 1, scap);
      for (int i = lane; i < nc; i += 32) {
        const int2 e = __ldcg(pool + off + i);
        if (i < L0.scap) L0.s[i] = e;
        else if (i - L0.scap < gcap) L0.g[i - L0.scap] = e;
      }
      __syncwarp();
    } else {
    fcam = (int)((int64_t)tile / tpf);
    const int64_t tl0 = ((int64_t)tile - fcam * tpf) * TT_RAYS;  // first ray within the frame
    r0 = fcam * n_per + tl0;
    nr = (int)((n_per - tl0) < TT_RAYS ? (n_per - tl0) : TT_RAYS);
    jb = nr;
    if (cam_rays) {
#pragma unroll
      for (int a = 0; a < 3; ++a) so.o[a] = cams.cam[fcam].position[a];
    }
    // ---- the tile's rays, and the root list: rays whose box test hits B
    {
      const TileList L0 = tile_list(W, ga, gcap, 0, scap);
#pragma unroll
      for (int j0 = 0; j0 < TT_RAYS; j0 += 32) {
        const int j = j0 + lane;
        bool root = false;
        if (j < nr && fr.hit) {  // per-pixel output defaults (the march overwrites its rays')
          const int64_t i = r0 + j;
          fr.hit[i] = 0;
          fr.t[i] = __longlong_as_double(0x7ff8000000000000ll);
          fr.normal[3 * i] = 0.0;
          fr.normal[3 * i + 1] = 0.0;
          fr.normal[3 * i + 2] = 0.0;
          fr.normal_ok[i] = 0;
          fr.iterations[i] = 0;
          fr.evals[i] = 0;
          fr.color[3 * i] = (uint8_t)(bg & 0xffu);
          fr.color[3 * i + 1] = (uint8_t)((bg >> 8) & 0xffu);
          fr.color[3 * i + 2] = (uint8_t)((bg >> 16) & 0xffu);
        }
        if (j < nr) {
          ng_ray r;
          if (SO && cam_rays) camera_ray(cams.cam[fcam], tl0 + j, r);  // the camera's ray, not stored
          else load_ray_slab(rays, r0 + j, so, r);
          bool general = true;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            if (!SO) W->o[j][a] = r.o[a];
            W->inv[j][a] = r.inv[a];
            general = general && isfinite(r.o[a]) && isfinite(r.inv[a]) && !((r.flags >> (3 + a)) & 1);
          }
          W->flags[j] = r.flags | (general ? TT_GENERAL : 0);
          const double lo[3] = {-1.0, -1.0, -1.0}, hi[3] = {1.0, 1.0, 1.0};
          if (general) {
            root = box_hit_ordered(r, lo, hi);
            // a ray missing the box of the occupied finest voxels (the trace
            // level being the finest) hits none of them: each voxel box lies
            // inside it on the same dyadic planes, so the slab values nest
            // (the ordered-test argument); rays off the general path are not
            // culled
            if (root && cull) root = box_hit_ordered(r, tree.region_lo, tree.region_hi);
          } else {
            double a0, b0;
            root = slab_test(r, lo, hi, a0, b0);
          }
        }
        W->seg_s[j] = 0;
        W->seg_e[j] = 0;
        const unsigned rb = __ballot_sync(FULL, root);
        if (root) tl_put(L0, nc + __popc(rb & lanemask_lt()), 0, 0u, j, gcap);
        nc += __popc(rb);
      }
    }
    // (an arena too small for even the root list: truncate like any list,
    // and the overflow asks for a rerun)
    need = nc > need ? nc : need;
    nc = nc < lim ? nc : lim;
    }
    __syncwarp();
    // ---- level passes: hits at level t -> hit children at level t+1
    for (int t = t0; t < target; ++t) {
      const TileList src = tile_list(W, ga, gcap, t & 1, scap);
      const TileList dst = tile_list(W, ga, gcap, (t & 1) ^ 1, scap);
      const int cres = level_res(tree, t - tree.n_virtual + 1);
      const int32_t* __restrict__ cstart = tree.child_start[t];
      const uint8_t* __restrict__ cmask = tree.child_mask[t];
      int out = 0;
      const bool last_pass = t + 1 == target;
      int carry_prev = -1;  // ray of the previous round's last item
      for (int base = 0; base < nc; base += 32 * TT_ITEMS) {
        int32_t first[TT_ITEMS];
        uint32_t pcell[TT_ITEMS];
        int pr[TT_ITEMS];
        unsigned hm[TT_ITEMS];  // bits 0-7 hit children front to back, 8-10 dm, 16-23 child mask
        int sum = 0;
#pragma unroll
        for (int q = 0; q < TT_ITEMS; ++q) {
          const int i = base + lane * TT_ITEMS + q;
          hm[q] = 0;
          first[q] = 0;
          pcell[q] = 0;
          pr[q] = -1;
          if (i < nc) {
            int32_t pv;
            tl_get(src, i, pv, pcell[q], pr[q]);
            const unsigned m = __ldg(cmask + pv);
            first[q] = __ldg(cstart + pv);
            const int pc[3] = {(int)(pcell[q] & 511u), (int)((pcell[q] >> 9) & 511u), (int)(pcell[q] >> 18)};
            const int fl = W->flags[pr[q]];
            const int dm = fl & 7;
            unsigned hk;  // front-to-back hit bits
            if (fl & TT_GENERAL) {
              double q0[3], q1[3], q2[3];
#pragma unroll
              for (int a = 0; a < 3; ++a)
                axis_crossings(SO ? so.o[a] : W->o[pr[q]][a], W->inv[pr[q]][a], (dm >> a) & 1, pc[a], cres, q0[a],
                               q1[a], q2[a]);
              hk = child_hits_ordered(q0, q1, q2) & octants_front_to_back(m, dm);
            } else {
              ng_ray r;
              tw_ray<SO>(W, so, pr[q], r);
              hk = octants_front_to_back(literal_child_hits(r, pc[0], pc[1], pc[2], cres) & m, dm);
            }
            if (hk) hm[q] = hk | ((unsigned)dm << 8) | (m << 16);
          }
          sum += __popc(hm[q] & 0xffu);
        }
        const int incl = warp_incl_scan<int>(sum);
        int o = out + incl - sum;
        // last pass: each ray's final segment runs from its first parent's
        // first child to its last parent's last child (parents of a ray are
        // contiguous); neighbours' rays come from the adjacent lanes
        int nb_prev = 0, nb_next = 0;
        if (last_pass) {
          nb_prev = __shfl_up_sync(FULL, pr[TT_ITEMS - 1], 1);
          nb_next = __shfl_down_sync(FULL, pr[0], 1);
          if (lane == 0) nb_prev = carry_prev;
          if (lane == 31) nb_next = base + 32 * TT_ITEMS < nc ? tl_ray(src, base + 32 * TT_ITEMS) : -1;
          carry_prev = __shfl_sync(FULL, pr[TT_ITEMS - 1], 31);
        }
#pragma unroll
        for (int q = 0; q < TT_ITEMS; ++q) {
          if (last_pass && pr[q] >= 0) {
            const int prv = q > 0 ? pr[q - 1] : nb_prev;
            const int nxt = q + 1 < TT_ITEMS ? pr[q + 1] : nb_next;
            if (prv != pr[q]) W->seg_s[pr[q]] = o;
            if (nxt != pr[q]) W->seg_e[pr[q]] = o + __popc(hm[q] & 0xffu);
          }
          const int dm = (int)((hm[q] >> 8) & 7u);
          const unsigned m = (hm[q] >> 16) & 0xffu;
          const uint32_t c2 = pcell[q] << 1;  // 2 * (x, y, z), packed (parent cells < 256 per axis)
          for (unsigned bits = hm[q] & 0xffu; bits; bits &= bits - 1) {
            const int oct = (__ffs(bits) - 1) ^ dm;
            const uint32_t cc = c2 | (uint32_t)(oct & 1) | ((uint32_t)((oct >> 1) & 1) << 9) |
                                ((uint32_t)(oct >> 2) << 18);
            tl_put(dst, o, first[q] + __popc(m & ((1u << oct) - 1u)), cc, pr[q], gcap);
            ++o;
          }
        }
        out += __shfl_sync(FULL, incl, 31);
      }
      __syncwarp();
      if (lane == t + 1) level_cnt += out;
      need = out > need ? out : need;
      nc = out < lim ? out : lim;
      // ---- split a long list at a ray boundary near its middle (above)
      // (only once every tile is claimed: before that idle warps take fresh
      // tiles, and a split only adds work)
      if (t + 1 < target && out > split_at && out <= lim && jb - ja > 1 &&
          (int64_t)*(volatile unsigned int*)tile_counter + split_ahead * (int64_t)gridDim.x * TT_WPB >= n_tiles) {
#ifdef NG_PROFILE
        unsigned long long ts0 = 0;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(ts0));
        ++n_splits;
#endif
        // first entry of the ray holding the middle entry, else of the next ray
        const int rm = tl_ray(dst, nc / 2);
        int lo = 0, hi = nc / 2;  // lower bound of rm (entries are grouped by ray, ascending)
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (tl_ray(dst, mid) < rm) lo = mid + 1; else hi = mid;
        }
        int m = lo;
        if (m == 0) {
          lo = nc / 2;
          hi = nc;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (tl_ray(dst, mid) <= rm) lo = mid + 1; else hi = mid;
          }
          m = lo;
        }
        if (m > 0 && m < nc) {
          const int cnt = nc - m;
          int slot = -1;
          unsigned long long off = 0;
          if (lane == 0) {
            off = atomicAdd(pool_top, (unsigned)cnt);
            if ((int64_t)off + cnt <= TT_CONT_POOL) {
              const unsigned tl = (unsigned)(atomicAdd(qstate, 1ull << 32) >> 32);
              if (tl < (unsigned)TT_CONT_RECS) slot = (int)tl;
              else atomicAdd(qstate, 1ull);  // never published: counted finished (tickets past it are moot)
            }
          }
          slot = __shfl_sync(FULL, slot, 0);
          off = __shfl_sync(FULL, off, 0);
          if (slot >= 0) {
            for (int i = lane; i < cnt; i += 32) {
              const int k = m + i;
              __stcg(pool + off + i, k < dst.scap ? dst.s[k] : dst.g[k - dst.scap]);
            }
            const int jm = tl_ray(dst, m);
            if (lane == 0) {
              TileCont* cr = recs + slot;
              cr->r0 = r0;
              cr->pool_off = (int64_t)off;
              cr->nr = nr;
              cr->ja = jm;
              cr->jb = jb;
              cr->pass = t + 1;
              cr->count = cnt;
            }
            __syncwarp();
            red_add_release_u32(ready + slot, 1u);  // every lane: its pool stores (lane 0: the fields) first
            nc = m;
            jb = jm;
          }
        }
#ifdef NG_PROFILE
        unsigned long long ts1 = 0;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(ts1));
        split_ns += ts1 - ts0;
#endif
      }
    }
    // ---- final pairs: claim the tile's block of the hit list, write
    // (cell, voxel, t_enter, t_exit) and the per-ray segments (set above)
    const TileList fin = tile_list(W, ga, gcap, target & 1, scap);
    unsigned long long hb = 0;
    if (lane == 0 && nc > 0) hb = atomicAdd(hit_cursor, (unsigned long long)nc);
    const int64_t hbase = (int64_t)__shfl_sync(FULL, hb, 0);
    const int fres = level_res(tree, target - tree.n_virtual);
    for (int i = lane; i < nc; i += 32) {
      int32_t v;
      uint32_t c;
      int rl;
      tl_get(fin, i, v, c, rl);
      const int cc[3] = {(int)(c & 511u), (int)((c >> 9) & 511u), (int)(c >> 18)};
      ng_hit_pair h;
      // render lists: the voxel's cell x | y << 10 | z << 20 (the march knows its ray)
      h.ray = (int32_t)((uint32_t)cc[0] | ((uint32_t)cc[1] << 10) | ((uint32_t)cc[2] << 20));
      h.voxel = v;
      const int fl = W->flags[rl];
      if (fl & TT_GENERAL) {
        // the cell's slab interval per axis is [min, max] of its two plane
        // crossings, sorted by the direction sign (monotone, as above)
        double ne = 0.0, fa = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const bool neg = (fl >> a) & 1;
          const double h2 = 2.0 / (double)fres;
          const double pn = dmul((double)(cc[a] + (neg ? 1 : 0) - fres / 2), h2);
          const double pfar = dadd(pn, neg ? -h2 : h2);
          const double o = SO ? so.o[a] : W->o[rl][a];
          const double inv = W->inv[rl][a];
          const double tn = dmul(dsub(pn, o), inv), tf = dmul(dsub(pfar, o), inv);
          ne = a == 0 ? tn : (tn > ne ? tn : ne);
          fa = a == 0 ? tf : (tf < fa ? tf : fa);
        }
        h.t_enter = ne > 0.0 ? ne : 0.0;
        h.t_exit = fa;
      } else {
        ng_ray r;
        tw_ray<SO>(W, so, rl, r);
        literal_slab(r, cc, fres, h.t_enter, h.t_exit);
      }
      if (hbase + i < hit_cap) hits[hbase + i] = h;
    }
    __syncwarp();
#pragma unroll
    for (int j0 = 0; j0 < TT_RAYS; j0 += 32) {
      const int j = j0 + lane;
      bool has = false;
      int64_t s0 = 0, e0 = 0;
      if (j >= ja && j < jb) {
        s0 = hbase + W->seg_s[j];
        e0 = hbase + W->seg_e[j];
        s0 = s0 < hit_cap ? s0 : hit_cap;
        e0 = e0 < hit_cap ? e0 : hit_cap;
        seg_start[r0 + j] = s0;
        seg_end[r0 + j] = e0;
        has = e0 > s0;
      }
      // the march's work list: rays with a segment, appended per tile
      const unsigned am = __ballot_sync(FULL, has);
      unsigned long long ab = 0;
      if (lane == 0 && am) ab = atomicAdd(d_active, (unsigned long long)__popc(am));
      ab = __shfl_sync(FULL, ab, 0);
      if (has)  // (ray, segment length, segment start)
        items[ab + __popc(am & lanemask_lt())] =
            make_int4((int)(r0 + j), (int)(e0 - s0), (int)(uint32_t)s0, (int)(s0 >> 32));
    }
    __syncwarp();
    if (lane == 0) {  // (after this part's outputs)
      if (rec >= 0) atomicAdd(qstate, 1ull);
      else atomicAdd(tiles_done, 1u);
    }
#ifdef NG_PROFILE
    if (lane == 0 && g_part_prof) {
      unsigned long long tp1;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tp1));
      const unsigned k = atomicAdd(&g_part_next, 1u);
      if (k < (1u << 20)) {
        unsigned long long* pp = g_part_prof + 8 * (size_t)k;
        pp[0] = tp0; pp[1] = tp1; pp[2] = (unsigned long long)(long long)rec; pp[3] = tile;
        pp[4] = (unsigned long long)t0; pp[5] = (unsigned long long)gw; pp[6] = (unsigned long long)n_splits;
        pp[7] = split_ns;
      }
    }
#endif
#ifdef NG_PROFILE
    if (lane == 0 && rec < 0 && g_tile_prof && (long long)tile < g_tile_prof_cap) {
      unsigned long long tp1;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tp1));
      unsigned long long* pr = g_tile_prof + 4 * (int64_t)tile;
      pr[0] = tp0;
      pr[1] = tp1;
      pr[2] = (unsigned long long)nc;
      pr[3] = (unsigned long long)gw;
    }
#endif
  }
  if (lane >= 1 && lane <= target && level_cnt) atomicAdd((unsigned long long*)(counts + lane),
                                                          (unsigned long long)level_cnt);
  if (lane == 0 && need > scap) atomicMax(d_need, (unsigned long long)need);
}

__global__ void k_segments(const ng_hit_pair* __restrict__ hits, const int64_t* __restrict__ d_count,
                           int64_t cap, int64_t n_rays, int64_t* __restrict__ seg_start,
                           int64_t* __restrict__ seg_end) {
  int64_t n = *d_count;
  if (n > cap) n = cap;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rays;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (hits[mid].ray < r) lo = mid + 1; else hi = mid;
    }
    seg_start[r] = lo;
    hi = n;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (hits[mid].ray <= r) lo = mid + 1; else hi = mid;
    }
    seg_end[r] = lo;
  }
}

__global__ void k_rays_from_arrays(const double* __restrict__ o, const double* __restrict__ d, int64_t n,
                                   ng_ray* __restrict__ rays) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    ng_ray r;
    make_ray(o[3 * i], o[3 * i + 1], o[3 * i + 2], d[3 * i], d[3 * i + 1], d[3 * i + 2], r);
    rays[i] = r;
  }
}

__global__ void k_ray_aabb(const double* __restrict__ o, const double* __restrict__ d,
                           const double* __restrict__ lo, const double* __restrict__ hi, int64_t n,
                           double* __restrict__ te, double* __restrict__ tx, uint8_t* __restrict__ hit) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    ng_ray r;
    make_ray(o[3 * i], o[3 * i + 1], o[3 * i + 2], d[3 * i], d[3 * i + 1], d[3 * i + 2], r);
    double l[3] = {lo[3 * i], lo[3 * i + 1], lo[3 * i + 2]};
    double h[3] = {hi[3 * i], hi[3 * i + 1], hi[3 * i + 2]};
    double a, b;
    hit[i] = slab_test(r, l, h, a, b) ? 1 : 0;
    te[i] = a;
    tx[i] = b;
  }
}

// decide (traversal.py:95-110) on an explicit pair list.
__global__ void k_decide(const __grid_constant__ ng_octree tree, const ng_ray* __restrict__ rays, int t, int final,
                         const ng_pair* __restrict__ pairs, int64_t n, int64_t* __restrict__ D) {
  const int level = t - tree.n_virtual;
  const int res = level_res(tree, level);
  const double edge = 2.0 / (double)res;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    ng_pair p = pairs[i];
    ng_ray r;
    load_ray(rays, p.ray, r);
    const uint64_t c = tree.codes[t][p.voxel];
    double lo[3] = {cell_lo((int)compact3(c), res), cell_lo((int)compact3(c >> 1), res),
                    cell_lo((int)compact3(c >> 2), res)};
    double hi[3] = {dadd(lo[0], edge), dadd(lo[1], edge), dadd(lo[2], edge)};
    double a, b;
    const bool hit = slab_test(r, lo, hi, a, b);
    D[i] = final ? (hit ? 1 : 0) : (hit ? __popc((unsigned)tree.child_mask[t][p.voxel]) : 0);
  }
}

// subdivide (traversal.py:165-191) given D and S.
__global__ void k_subdivide(const __grid_constant__ ng_octree tree, const ng_ray* __restrict__ rays, int t,
                            const ng_pair* __restrict__ pairs, int64_t n, const int64_t* __restrict__ D,
                            const int64_t* __restrict__ S, ng_pair* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (D[i] <= 0) continue;
    ng_pair p = pairs[i];
    const int dm = rays[p.ray].flags & 7;
    const unsigned m = tree.child_mask[t][p.voxel];
    const int32_t first = tree.child_start[t][p.voxel];
    int64_t o = S[i];
    for (int k = 0; k < 8; ++k) {
      const int oct = k ^ dm;
      if ((m >> oct) & 1u) out[o++] = ng_pair{p.ray, first + __popc(m & ((1u << oct) - 1u))};
    }
  }
}

__global__ void k_compactify(const ng_pair* __restrict__ pairs, int64_t n, const int64_t* __restrict__ D,
                             const int64_t* __restrict__ S, ng_pair* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (D[i] == 1) out[S[i]] = pairs[i];
}

int grid_for(int64_t n, int nt = 256);

size_t level_scratch_bytes(int64_t max_pairs) {
  const int64_t tile = (int64_t)TR_NT * TR_ITEMS;
  int64_t tiles = (max_pairs + tile - 1) / tile;
  if (tiles < 1) tiles = 1;
  return 16 + (size_t)tiles * 8;
}

int traverse_level(const ng_octree& tree, const ng_ray* rays, int t, bool final, const ng_pair* in,
                   const int64_t* d_count_in, int64_t in_cap, ng_pair* out_pairs, ng_hit_pair* out_hits,
                   int64_t* d_count_out, int64_t out_cap, void* scratch, size_t scratch_bytes,
                   cudaStream_t s) {
  size_t need = level_scratch_bytes(in_cap);
  if (scratch_bytes < need) {
    set_error("ng_traverse_level: scratch %zu < %zu bytes", scratch_bytes, need);
    return NG_ERR_CAPACITY;
  }
  int r = cuda_status(cudaMemsetAsync(scratch, 0, need, s), "ng_traverse_level memset");
  if (r) return r;
  const int64_t tile = (int64_t)TR_NT * TR_ITEMS;
  int64_t tiles = (in_cap + tile - 1) / tile;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sm_count() * 6));
  unsigned int* counter = (unsigned int*)scratch;
  unsigned long long* states = (unsigned long long*)((char*)scratch + 16);
  if (final)
    k_traverse_level<true><<<grid, TR_NT, 0, s>>>(tree, rays, t, in, d_count_in, in_cap, out_pairs,
                                                  out_hits, d_count_out, out_cap, states, counter);
  else
    k_traverse_level<false><<<grid, TR_NT, 0, s>>>(tree, rays, t, in, d_count_in, in_cap, out_pairs,
                                                   out_hits, d_count_out, out_cap, states, counter);
  NG_CHECK_LAUNCH("ng_traverse_level");
  return NG_OK;
}

int traverse_hits(const ng_octree& tree, const ng_ray* rays, int t, bool next_final, const ng_pair* in,
                  const int64_t* d_count_in, int64_t in_cap, ng_pair* out_pairs, ng_hit_pair* out_hits,
                  int64_t* d_count_out, int64_t out_cap, void* scratch, size_t scratch_bytes, cudaStream_t s,
                  int64_t* seg_start, int64_t* seg_end, const double* shared_origin) {
  // the caller zeroes `scratch` (tile counter and look-back states) beforehand
  SharedOrigin so;
  so.shared = shared_origin != nullptr;
  for (int a = 0; a < 3; ++a) so.o[a] = shared_origin ? shared_origin[a] : 0.0;
  size_t need = level_scratch_bytes(in_cap);
  if (scratch_bytes < need) {
    set_error("traverse_hits: scratch %zu < %zu bytes", scratch_bytes, need);
    return NG_ERR_CAPACITY;
  }
  const int64_t tile = (int64_t)TR_NT * TR_ITEMS;
  int64_t tiles = (in_cap + tile - 1) / tile;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sm_count() * 6));
  unsigned int* counter = (unsigned int*)scratch;
  unsigned long long* states = (unsigned long long*)((char*)scratch + 16);
  if (next_final)
    k_traverse_hits<true><<<grid, TR_NT, 0, s>>>(tree, rays, t, in, d_count_in, in_cap, out_pairs, out_hits,
                                                 d_count_out, out_cap, states, counter, seg_start, seg_end, so);
  else
    k_traverse_hits<false><<<grid, TR_NT, 0, s>>>(tree, rays, t, in, d_count_in, in_cap, out_pairs, out_hits,
                                                  d_count_out, out_cap, states, counter, nullptr, nullptr, so);
  NG_CHECK_LAUNCH("k_traverse_hits");
  return NG_OK;
}

size_t tile_traverse_smem() { return sizeof(TileWarp) * TT_WPB; }
// NG_TILE_SCAP=k (test knob) holds only k entries of each list in shared
// memory, sending the rest through the arena.
int tile_traverse_scap() {
  static const int scap = std::max(0, std::min(TT_SCAP, env_int("NG_TILE_SCAP", TT_SCAP)));
  return scap;
}
static int tile_split_at() {
  static const int v = std::max(1, env_int("NG_TILE_SPLIT", 256));
  return v;
}
static int tile_split_ahead() {
  static const int v = std::max(0, env_int("NG_TILE_SPLIT_AHEAD", 0));
  return v;
}
int tile_traverse_entry_bytes() { return 2 * TT_ENTRY; }

// Warps the tile traversal runs with for up to `n_rays` rays (grid x
// TT_WPB: one resident wave, no more warps than tiles); the per-warp global
// arena is sized from this.
int64_t tile_traverse_warps(int64_t n_rays) {
  // resident CTAs per SM (an sm_100a property, the same on every B200)
  static const int per_sm = [] {
    int a = 0, b = 0;
    set_smem_limit((const void*)k_traverse_tiles<true>, tile_traverse_smem());
    set_smem_limit((const void*)k_traverse_tiles<false>, tile_traverse_smem());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_traverse_tiles<true>, TT_WPB * 32, tile_traverse_smem());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_traverse_tiles<false>, TT_WPB * 32, tile_traverse_smem());
    return std::max(1, std::min(a, b));
  }();
  const int64_t tiles = (n_rays + TT_RAYS - 1) / TT_RAYS;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((int64_t)sm_count() * per_sm,
                                                                  (tiles + TT_WPB - 1) / TT_WPB));
  return blocks * TT_WPB;
}

int traverse_tiles(const ng_octree& tree, const ng_ray* rays, const int64_t* d_n, int64_t n_max, int target,
                   int4* items, unsigned long long* d_active, int64_t* counts,
                   ng_hit_pair* hits, int64_t hit_cap, void* ctl, int64_t* seg_start, int64_t* seg_end,
                   void* arena, size_t arena_bytes, unsigned long long* d_need, const double* shared_origin,
                   const CamSet* cam_rays, const ng_frame* defaults, uint32_t bg, int64_t n_host,
                   void* cont, cudaStream_t s) {
  // `ctl` (512 bytes zeroed by the caller): u32 tile counter at 0, u64 hit
  // cursor at 8, longest list at 16, pool cursor at 64, continuation queue
  // words at 128, 256 and 384; `cont`:
  // tile_cont_bytes() of continuation records and pooled entries
  SharedOrigin so;
  so.shared = shared_origin != nullptr;
  for (int a = 0; a < 3; ++a) so.o[a] = shared_origin ? shared_origin[a] : 0.0;
  const int64_t warps = tile_traverse_warps(n_max);
  const int64_t gcap = (int64_t)(arena_bytes / (size_t)(warps * (2 * TT_ENTRY))) & ~int64_t(15);
  auto k = so.shared ? k_traverse_tiles<true> : k_traverse_tiles<false>;
  if (int r = set_smem_limit((const void*)k, tile_traverse_smem())) return r;  // per device
  k<<<(int)(warps / TT_WPB), TT_WPB * 32, tile_traverse_smem(), s>>>(
      tree, rays, d_n, target, counts, hits, hit_cap, (unsigned int*)ctl, (unsigned long long*)((char*)ctl + 8),
      seg_start, seg_end, (uint8_t*)arena, gcap, tile_traverse_scap(), d_need, so,
      cam_rays ? *cam_rays : CamSet{}, cam_rays != nullptr, items, d_active, defaults ? *defaults : ng_frame{},
      bg, n_host, target == tree.n_tlevels - 1, (uint8_t*)cont, tile_split_at(), tile_split_ahead());
  NG_CHECK_LAUNCH("k_traverse_tiles");
  return NG_OK;
}

// Longest tile list the arena (the two pair buffers) holds.
int64_t tile_traverse_limit(size_t arena_bytes, int64_t n_max) {
  const int64_t warps = tile_traverse_warps(n_max);
  return tile_traverse_scap() + ((int64_t)(arena_bytes / (size_t)(warps * (2 * TT_ENTRY))) & ~int64_t(15));
}

int segments(const ng_hit_pair* hits, const int64_t* d_count, int64_t cap, int64_t n_rays,
             int64_t* seg_start, int64_t* seg_end, cudaStream_t s) {
  k_segments<<<grid_for(n_rays), 256, 0, s>>>(hits, d_count, cap, n_rays, seg_start, seg_end);
  NG_CHECK_LAUNCH("ng_segments");
  return NG_OK;
}

}  // namespace ng

using namespace ng;

extern "C" {

size_t ng_level_scratch_bytes(int64_t max_pairs) { return level_scratch_bytes(max_pairs); }

int ng_traverse_level(const ng_octree* tree, const ng_ray* rays, int32_t t, int32_t final,
                      const ng_pair* in, const int64_t* d_count_in, int64_t in_capacity,
                      ng_pair* out_pairs, ng_hit_pair* out_hits, int64_t* d_count_out,
                      int64_t out_capacity, void* scratch, size_t scratch_bytes, void* stream) {
  if (t < 0 || t >= tree->n_tlevels || (!final && t + 1 >= tree->n_tlevels)) {
    set_error("no traversal level %d", t);
    return NG_ERR_STRUCTURAL;
  }
  return traverse_level(*tree, rays, t, final != 0, in, d_count_in, in_capacity, out_pairs, out_hits,
                        d_count_out, out_capacity, scratch, scratch_bytes, (cudaStream_t)stream);
}

int ng_segments(const ng_hit_pair* hits, const int64_t* d_count, int64_t capacity, int64_t n_rays,
                int64_t* seg_start, int64_t* seg_end, void* stream) {
  if (n_rays <= 0) return NG_OK;
  return segments(hits, d_count, capacity, n_rays, seg_start, seg_end, (cudaStream_t)stream);
}

int ng_decide(const ng_octree* tree, const ng_ray* rays, int32_t t, int32_t final, const ng_pair* pairs, int64_t n,
              int64_t* decisions, void* stream) {
  if (t < 0 || t >= tree->n_tlevels || (!final && t + 1 >= tree->n_tlevels)) {
    set_error("no traversal level %d", t);
    return NG_ERR_STRUCTURAL;
  }
  if (n <= 0) return NG_OK;
  k_decide<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(*tree, rays, t, final, pairs, n, decisions);
  NG_CHECK_LAUNCH("ng_decide");
  return NG_OK;
}

int ng_subdivide(const ng_octree* tree, const ng_ray* rays, int32_t t, const ng_pair* pairs, int64_t n,
                 const int64_t* D, const int64_t* S, ng_pair* out, void* stream) {
  if (t < 0 || t + 1 >= tree->n_tlevels) {
    set_error("no traversal level %d below which to subdivide", t);
    return NG_ERR_STRUCTURAL;
  }
  if (n <= 0) return NG_OK;
  k_subdivide<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(*tree, rays, t, pairs, n, D, S, out);
  NG_CHECK_LAUNCH("ng_subdivide");
  return NG_OK;
}

int ng_compactify(const ng_pair* pairs, int64_t n, const int64_t* D, const int64_t* S, ng_pair* out,
                  void* stream) {
  if (n <= 0) return NG_OK;
  k_compactify<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(pairs, n, D, S, out);
  NG_CHECK_LAUNCH("ng_compactify");
  return NG_OK;
}

int ng_rays_from_arrays(const double* o, const double* d, int64_t n, ng_ray* rays, void* stream) {
  if (n <= 0) return NG_OK;
  k_rays_from_arrays<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(o, d, n, rays);
  NG_CHECK_LAUNCH("ng_rays_from_arrays");
  return NG_OK;
}

int ng_ray_aabb(const double* o, const double* d, const double* lo, const double* hi, int64_t n,
                double* t_enter, double* t_exit, uint8_t* hit, void* stream) {
  if (n <= 0) return NG_OK;
  k_ray_aabb<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(o, d, lo, hi, n, t_enter, t_exit, hit);
  NG_CHECK_LAUNCH("ng_ray_aabb");
  return NG_OK;
}

}  // extern "C"

#ifdef NG_PROFILE
extern "C" int ng_part_profile(unsigned long long* host_out, int reset) {
  unsigned long long* p = nullptr;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&p, g_part_prof, sizeof(p));
  if (!p) {
    cudaMalloc((void**)&p, (size_t)8 * 8 << 20);
    cudaMemcpyToSymbol(g_part_prof, &p, sizeof(p));
  }
  unsigned n = 0;
  cudaMemcpyFromSymbol(&n, g_part_next, sizeof(n));
  if (n > (1u << 20)) n = 1u << 20;
  if (host_out && n) cudaMemcpy(host_out, p, (size_t)n * 64, cudaMemcpyDeviceToHost);
  if (reset) {
    unsigned z = 0;
    cudaMemcpyToSymbol(g_part_next, &z, sizeof(z));
  }
  return (int)n;
}
extern "C" int ng_tile_profile_enable(long long max_tiles) {
  unsigned long long* p = nullptr;
  if (cudaMalloc((void**)&p, (size_t)max_tiles * 32) != cudaSuccess) return NG_ERR_CUDA;
  cudaMemset(p, 0, (size_t)max_tiles * 32);
  cudaMemcpyToSymbol(g_tile_prof, &p, sizeof(p));
  cudaMemcpyToSymbol(g_tile_prof_cap, &max_tiles, sizeof(max_tiles));
  return NG_OK;
}
extern "C" int ng_tile_profile_read(unsigned long long* host_out, long long max_tiles) {
  unsigned long long* p = nullptr;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&p, g_tile_prof, sizeof(p));
  if (!p) return 0;
  cudaMemcpy(host_out, p, (size_t)max_tiles * 32, cudaMemcpyDeviceToHost);
  cudaMemset(p, 0, (size_t)max_tiles * 32);
  return 1;
}
#endif
