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
  const double cedge = 2.0 / (double)cres;
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
