// Shared device helpers for the nglod_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "../../include/nglod_b200.h"

namespace ng {

constexpr unsigned FULL = 0xffffffffu;

// ---------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);
int launch_status(const char* where);
int sm_count();                 // of the current device (cached per device)
int current_device();
// environment knob read once per process (call inside a function-local
// `static const` initialiser, which C++ makes thread-safe)
int env_int(const char* name, int def);
// raise a kernel's dynamic shared-memory limit on the CURRENT device
// (cudaFuncSetAttribute is per device); cached per (device, kernel),
// thread-safe
int set_smem_limit(const void* kernel, size_t bytes);
// cudaMallocAsync with the current device's stream-ordered pool told to keep
// its memory across synchronisations: with the default release threshold
// (0) every sync hands the pool's pages back and the next call maps them
// again, which made single configs[2] queries take 12 to 850 ms
int malloc_async(void** p, size_t bytes, cudaStream_t s, const char* where);

#define NG_CHECK_LAUNCH(name)                         \
  do {                                                \
    int _s = ::ng::launch_status(name);               \
    if (_s != NG_OK) return _s;                       \
  } while (0)

// ---------------------------------------------------------------- morton
// 21-bit coordinate spread, x in bit 0 of each triad (octree.py:35-60).
__host__ __device__ __forceinline__ uint64_t spread3(uint64_t v) {
  v &= 0x1FFFFFull;
  v = (v | (v << 32)) & 0x1F00000000FFFFull;
  v = (v | (v << 16)) & 0x1F0000FF0000FFull;
  v = (v | (v << 8)) & 0x100F00F00F00F00Full;
  v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

__host__ __device__ __forceinline__ uint32_t compact3(uint64_t v) {
  v &= 0x1249249249249249ull;
  v = (v ^ (v >> 2)) & 0x10C30C30C30C30C3ull;
  v = (v ^ (v >> 4)) & 0x100F00F00F00F00Full;
  v = (v ^ (v >> 8)) & 0x1F0000FF0000FFull;
  v = (v ^ (v >> 16)) & 0x1F00000000FFFFull;
  v = (v ^ (v >> 32)) & 0x1FFFFFull;
  return (uint32_t)v;
}

__host__ __device__ __forceinline__ uint64_t morton(uint32_t i, uint32_t j, uint32_t k) {
  return spread3(i) | (spread3(j) << 1) | (spread3(k) << 2);
}

// ---------------------------------------------------------------- exact fp64
// The reference computes in float64 with numpy's operation order; these
// helpers pin each rounding step so nvcc never contracts into an FMA.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// numpy minimum/maximum propagate NaN.
__device__ __forceinline__ double np_min(double a, double b) {
  return (a != a) ? a : ((b != b) ? b : (a < b ? a : b));
}
__device__ __forceinline__ double np_max(double a, double b) {
  return (a != a) ? a : ((b != b) ? b : (a > b ? a : b));
}

// Half-open binning: floor((x - (-1)) * (res / 2)) clipped to [0, res-1]
// (octree.py:134-139). res/2 is a power of two, so the product is exact.
__device__ __forceinline__ int bin_axis(double x, int res) {
  double f = dmul(dadd(x, 1.0), 0.5 * (double)res);
  double c = floor(f);
  int i = (c < 0.0) ? 0 : (c > (double)(res - 1) ? res - 1 : (int)c);
  return i;
}

// cell_origin (octree.py:142-143): -1 + ijk * (2/res); exact for our sizes.
__device__ __forceinline__ double cell_lo(int ijk, int res) {
  return dadd(-1.0, dmul((double)ijk, 2.0 / (double)res));
}

// ---------------------------------------------------------------- octree
__device__ __forceinline__ int level_res(const ng_octree& t, int level) {
  return level >= 0 ? (t.r0 << level) : (t.r0 >> (-level));
}

// Index of the voxel holding Morton code `code` at traversal level tl, or -1.
__device__ __forceinline__ int64_t rank_lookup(const uint64_t* __restrict__ bm,
                                               const uint32_t* __restrict__ rk, uint64_t code) {
  uint64_t w = __ldg(bm + (code >> 6));
  uint32_t b = (uint32_t)(code & 63);
  if (!((w >> b) & 1ull)) return -1;
  return (int64_t)__ldg(rk + (code >> 6)) + __popcll(w & ((1ull << b) - 1ull));
}

// ---------------------------------------------------------------- slab test
// ray_aabb_batch (octree.py:311-333) for one ray / one box, bit-exact.
__device__ __forceinline__ bool slab_test(const ng_ray& r, const double lo[3], const double hi[3],
                                          double& t_enter, double& t_exit) {
  double near = -INFINITY, far = INFINITY;
  bool nan_seen = false;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double an, af;
    if ((r.flags >> (3 + a)) & 1) {
      bool inside = (r.o[a] >= lo[a]) && (r.o[a] <= hi[a]);
      an = inside ? -INFINITY : INFINITY;
      af = inside ? INFINITY : -INFINITY;
    } else {
      double t1 = dmul(dsub(lo[a], r.o[a]), r.inv[a]);
      double t2 = dmul(dsub(hi[a], r.o[a]), r.inv[a]);
      an = np_min(t1, t2);
      af = np_max(t1, t2);
    }
    if (a == 0) {
      near = an;
      far = af;
    } else {
      near = np_max(near, an);
      far = np_min(far, af);
    }
  }
  nan_seen = (near != near) || (far != far);
  t_enter = np_max(near, 0.0);
  t_exit = far;
  return !nan_seen && (near <= far) && (far >= 0.0);
}

// Per-axis slab intervals of the two child halves of a parent cell. The
// child planes lo/mid/hi are exact dyadic values, so t = (plane - o) * inv
// per plane is bit-identical to ray_aabb_batch on each child box; a parent
// computes 9 plane distances once instead of 8 x 6.
struct ChildSlabs {
  double an[3][2];  // per axis, per half: min(t_lo, t_hi)
  double af[3][2];  // max(t_lo, t_hi)
};

__device__ __forceinline__ void child_slabs(const ng_ray& r, int px, int py, int pz, int cres, ChildSlabs& cs) {
  const int pc[3] = {px, py, pz};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double p0 = cell_lo(2 * pc[a], cres), p1 = cell_lo(2 * pc[a] + 1, cres),
                 p2 = cell_lo(2 * pc[a] + 2, cres);
    if ((r.flags >> (3 + a)) & 1) {
      const bool in0 = (r.o[a] >= p0) && (r.o[a] <= p1);
      const bool in1 = (r.o[a] >= p1) && (r.o[a] <= p2);
      cs.an[a][0] = in0 ? -INFINITY : INFINITY;
      cs.af[a][0] = in0 ? INFINITY : -INFINITY;
      cs.an[a][1] = in1 ? -INFINITY : INFINITY;
      cs.af[a][1] = in1 ? INFINITY : -INFINITY;
    } else {
      const double t0 = dmul(dsub(p0, r.o[a]), r.inv[a]);
      const double t1 = dmul(dsub(p1, r.o[a]), r.inv[a]);
      const double t2 = dmul(dsub(p2, r.o[a]), r.inv[a]);
      cs.an[a][0] = np_min(t0, t1);
      cs.af[a][0] = np_max(t0, t1);
      cs.an[a][1] = np_min(t1, t2);
      cs.af[a][1] = np_max(t1, t2);
    }
  }
}

// Slab test of child octant `oct` from precomputed halves (same reduction
// order as slab_test / ray_aabb_batch).
__device__ __forceinline__ bool child_hit(const ChildSlabs& cs, int oct, double& t_enter, double& t_exit) {
  // selects, not indexing: keeps ChildSlabs in registers
  const bool b0 = oct & 1, b1 = (oct >> 1) & 1, b2 = (oct >> 2) & 1;
  double near = b0 ? cs.an[0][1] : cs.an[0][0], far = b0 ? cs.af[0][1] : cs.af[0][0];
  near = np_max(near, b1 ? cs.an[1][1] : cs.an[1][0]);
  far = np_min(far, b1 ? cs.af[1][1] : cs.af[1][0]);
  near = np_max(near, b2 ? cs.an[2][1] : cs.an[2][0]);
  far = np_min(far, b2 ? cs.af[2][1] : cs.af[2][0]);
  t_enter = np_max(near, 0.0);
  t_exit = far;
  return (near <= far) && (far >= 0.0);
}

__device__ __forceinline__ void load_ray(const ng_ray* __restrict__ rays, int64_t i, ng_ray& r) {
  const double2* p = reinterpret_cast<const double2*>(rays + i);
  double2 a = __ldg(p + 0), b = __ldg(p + 1), c = __ldg(p + 2), d = __ldg(p + 3), e = __ldg(p + 4);
  r.o[0] = a.x; r.o[1] = a.y; r.o[2] = b.x;
  r.d[0] = b.y; r.d[1] = c.x; r.d[2] = c.y;
  r.inv[0] = d.x; r.inv[1] = d.y; r.inv[2] = e.x;
  r.flags = __double_as_longlong(e.y) & 0xffffffff;
  r.pad = 0;
}

// A pinhole camera's rays share one origin: the traversal then loads only
// the slab part of the record (1/d and the direction flags, bytes 48-79).
struct SharedOrigin {
  double o[3];
  int shared;
};

__device__ __forceinline__ void load_ray_slab(const ng_ray* __restrict__ rays, int64_t i, const SharedOrigin& so,
                                              ng_ray& r) {
  if (!so.shared) {
    load_ray(rays, i, r);
    return;
  }
  const double2* p = reinterpret_cast<const double2*>(rays + i);
  const double2 d = __ldg(p + 3), e = __ldg(p + 4);
  r.o[0] = so.o[0]; r.o[1] = so.o[1]; r.o[2] = so.o[2];
  r.d[0] = r.d[1] = r.d[2] = 0.0;  // not used by slab tests
  r.inv[0] = d.x; r.inv[1] = d.y; r.inv[2] = e.x;
  r.flags = __double_as_longlong(e.y) & 0xffffffff;
  r.pad = 0;
}

__device__ __forceinline__ void make_ray(double ox, double oy, double oz, double dx, double dy,
                                         double dz, ng_ray& r) {
  r.o[0] = ox; r.o[1] = oy; r.o[2] = oz;
  r.d[0] = dx; r.d[1] = dy; r.d[2] = dz;
  int flags = 0;
  double d3[3] = {dx, dy, dz};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    r.inv[a] = 1.0 / d3[a];
    if (d3[a] < 0.0) flags |= 1 << a;
    if (d3[a] == 0.0) flags |= 1 << (3 + a);
  }
  r.flags = flags;
  r.pad = 0;
}

// Pixel-centre ray i of a (band-tiled) pinhole camera, bit-exact with
// Camera.rays (render.py:74-88). Every kernel that needs a camera ray
// computes it with this one function, so a ray recomputed on the fly is
// the same ray everywhere.
// The unit direction of camera ray i (render.py:74-88); camera_ray below
// adds the origin and the slab fields (1/d, signs).
__device__ __forceinline__ void camera_dir(const ng_camera& cam, int64_t i, double dir[3]) {
  const int px_i = (int)(i % cam.width);
  const int lrow = (int)(i / cam.width);
  const int band = lrow / cam.band_rows;
  const int py_i = (band * cam.band_stride + cam.band_offset) * cam.band_rows + lrow % cam.band_rows;
  const double px = dmul(dmul(dsub(dmul(2.0, dadd((double)px_i, 0.5)) / (double)cam.width, 1.0), cam.tan_half),
                         cam.aspect);
  const double py = dmul(dsub(1.0, dmul(2.0, dadd((double)py_i, 0.5)) / (double)cam.height), cam.tan_half);
  double d[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) d[a] = dadd(dadd(cam.fwd[a], dmul(px, cam.right[a])), dmul(py, cam.up[a]));
  const double nrm = __dsqrt_rn(dadd(dadd(dmul(d[0], d[0]), dmul(d[1], d[1])), dmul(d[2], d[2])));
#pragma unroll
  for (int a = 0; a < 3; ++a) dir[a] = d[a] / nrm;
}

__device__ __forceinline__ void camera_ray(const ng_camera& cam, int64_t i, ng_ray& r) {
  double d[3];
  camera_dir(cam, i, d);
  make_ray(cam.position[0], cam.position[1], cam.position[2], d[0], d[1], d[2], r);
}

// The cameras of a frame batch (ng_render_batch): frame f's rays are rays
// [f n_per, (f + 1) n_per) of the launch, its pixels in its camera's order;
// a single frame is a batch of one. Kernels take it as a __grid_constant__
// parameter (a camera is picked with a run-time index).
struct CamSet {
  ng_camera cam[NG_MAX_BATCH];
  int64_t n_per;  // rays per frame
  int32_t k;      // frames
  int32_t pad;
  __host__ __device__ __forceinline__ int frame_of(int64_t i) const { return k > 1 ? (int)(i / n_per) : 0; }
};

// Ray i of a batch: its frame's camera ray (the same function as a single frame).
__device__ __forceinline__ void camera_ray(const CamSet& cs, int64_t i, ng_ray& r) {
  const int f = cs.frame_of(i);
  camera_ray(cs.cam[f], i - (int64_t)f * cs.n_per, r);
}

// Rays of a pass: explicit records, or (`cam_rays`) the cameras' rays
// computed where they are used instead of stored.
struct RaySrc {
  const ng_ray* rays;
  CamSet cam;
  int cam_rays;
};

__device__ __forceinline__ void ray_at(const RaySrc& S, int64_t i, ng_ray& r) {
  if (S.cam_rays) camera_ray(S.cam, i, r);
  else load_ray(S.rays, i, r);
}

// ---------------------------------------------------------------- warp utils
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(FULL, v, o);
    if ((int)lane_id() >= o) v += n;
  }
  return v;
}

// ---------------------------------------------------------------- look-back scan
// Single-pass decoupled look-back tile states: value in the low 62 bits,
// status in the top 2 (0 = not ready, 1 = aggregate, 2 = inclusive prefix).
constexpr uint64_t TS_AGG = 1ull << 62;
constexpr uint64_t TS_PREFIX = 2ull << 62;
constexpr uint64_t TS_VALUE = (1ull << 62) - 1;

// Called by one thread: publish this tile's aggregate and return the
// exclusive prefix of all earlier tiles.
__device__ __forceinline__ int64_t tile_lookback(unsigned long long* states, int64_t tile,
                                                 int64_t aggregate) {
  if (tile == 0) {
    __threadfence();
    atomicExch(states, (unsigned long long)(TS_PREFIX | (uint64_t)aggregate));
    return 0;
  }
  __threadfence();
  atomicExch(states + tile, (unsigned long long)(TS_AGG | (uint64_t)aggregate));
  int64_t excl = 0;
  int64_t p = tile - 1;
  while (true) {
    uint64_t s = *((volatile unsigned long long*)(states + p));
    uint64_t st = s & ~TS_VALUE;
    if (st == 0) continue;
    excl += (int64_t)(s & TS_VALUE);
    if (st == TS_PREFIX) break;
    --p;
  }
  __threadfence();
  atomicExch(states + tile, (unsigned long long)(TS_PREFIX | (uint64_t)(excl + aggregate)));
  return excl;
}

// Warp-parallel look-back (called by all 32 lanes of one warp): 32
// predecessors are inspected per round, so a tile resolves its prefix in
// about one L2 round trip instead of one per predecessor.
__device__ __forceinline__ int64_t tile_lookback_warp(unsigned long long* states, int64_t tile,
                                                      int64_t aggregate) {
  const int lane = (int)(threadIdx.x & 31);
  if (tile == 0) {
    if (lane == 0) {
      __threadfence();
      atomicExch(states, (unsigned long long)(TS_PREFIX | (uint64_t)aggregate));
    }
    return 0;
  }
  if (lane == 0) {
    __threadfence();
    atomicExch(states + tile, (unsigned long long)(TS_AGG | (uint64_t)aggregate));
  }
  int64_t excl = 0;
  int64_t base = tile - 1;
  while (true) {
    const int64_t p = base - lane;  // lane i looks at the i-th nearest predecessor
    uint64_t s = TS_PREFIX;         // before tile 0: an empty prefix
    if (p >= 0) {
      do {
        s = *((volatile unsigned long long*)(states + p));
      } while ((s & ~TS_VALUE) == 0);
    }
    const unsigned pm = __ballot_sync(FULL, (s & ~TS_VALUE) == TS_PREFIX);
    const int first = pm ? __ffs(pm) - 1 : 32;
    int64_t v = (lane <= first) ? (int64_t)(s & TS_VALUE) : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    excl += v;
    if (pm) break;
    base -= 32;
  }
  if (lane == 0) {
    __threadfence();
    atomicExch(states + tile, (unsigned long long)(TS_PREFIX | (uint64_t)(excl + aggregate)));
  }
  return excl;
}

// Block-wide exclusive scan of one int64 per thread; returns the block total.
template <int NT>
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t& excl, int64_t* sm_warp) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  int64_t inc = warp_incl_scan<int64_t>(v);
  if (l == 31) sm_warp[w] = inc;
  __syncthreads();
  if (w == 0) {
    int64_t x = (l < NT / 32) ? sm_warp[l] : 0;
    int64_t xi = warp_incl_scan<int64_t>(x);
    if (l < NT / 32) sm_warp[l] = xi - x;
    if (l == NT / 32 - 1) sm_warp[NT / 32] = xi;
  }
  __syncthreads();
  excl = sm_warp[w] + inc - v;
  int64_t total = sm_warp[NT / 32];
  return total;
}

// Flag words between warps of one grid: a relaxed load (no L1 invalidation)
// polled until set, and a release store after the data it publishes; the
// data is read with L2 (.cg) loads once the flag is seen.
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_add_release_u32(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace ng
