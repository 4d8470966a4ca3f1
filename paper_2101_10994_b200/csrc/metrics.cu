// Evaluation kernels that reuse the octree and the analytic SDFs
// (reference octfield/metrics.py).
//
//   k_trace_sdf      trace_oracle_rays (metrics.py:145-178): sphere tracing of
//                    a built-in ground-truth SDF from the domain-box entry,
//                    stop on d < delta, give up past the far plane
//   k_nearest_voxel  predict_signed_extension's outside branch
//                    (metrics.py:229-252): nearest occupied voxel of a level
//                    (first minimum, like numpy argmin), the clamped anchor
//                    and the separation, numpy's operation order
//   k_nn_dist        PointGrid.nearest_dist (metrics.py:64-112) as an exact
//                    brute-force minimum; the min over sqrt equals sqrt of the
//                    min squared distance (sqrt is monotone and correctly
//                    rounded)
#include "common.cuh"
#include "sdf.cuh"

namespace ng {

static inline int mgrid(int64_t n, int nt) { return (int)((n + nt - 1) / nt); }

__global__ void k_trace_sdf(int kind, const double* __restrict__ prm, int np_, const double* __restrict__ o,
                            const double* __restrict__ d, int64_t n, double delta, double far_plane, int max_iters,
                            uint8_t* hit, double* t_hit) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  ng_ray r;
  make_ray(o[3 * i], o[3 * i + 1], o[3 * i + 2], d[3 * i], d[3 * i + 1], d[3 * i + 2], r);
  const double lo[3] = {-1.0, -1.0, -1.0}, hi[3] = {1.0, 1.0, 1.0};
  double t, t_exit;
  bool alive = slab_test(r, lo, hi, t, t_exit);  // ray_aabb_batch against B (metrics.py:153-157)
  uint8_t h = 0;
  double th = NAN;
  for (int it = 0; it < max_iters && alive; ++it) {
    const double x = dadd(r.o[0], dmul(t, r.d[0]));
    const double y = dadd(r.o[1], dmul(t, r.d[1]));
    const double z = dadd(r.o[2], dmul(t, r.d[2]));
    const double dv = sdf_builtin(kind, prm, np_, x, y, z);
    if (dv < delta) {
      h = 1;
      th = dadd(t, dv);
      break;
    }
    t = dadd(t, dv);
    if (t > far_plane) alive = false;
  }
  hit[i] = h;
  t_hit[i] = th;
}

// Warp per query point; lanes stride over the level's voxels.
__global__ void k_nearest_voxel(const __grid_constant__ ng_octree tree, int level, const double* __restrict__ pts,
                                int64_t n, double* anchor, double* gap) {
  const int lane = threadIdx.x & 31;
  const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (q >= n) return;
  const int tl = level + tree.n_virtual;
  const int res = tree.r0 << level;
  const uint64_t* __restrict__ codes = tree.codes[tl];
  const int64_t V = tree.count[tl];
  const double qx[3] = {pts[3 * q], pts[3 * q + 1], pts[3 * q + 2]};
  const double edge = 2.0 / (double)res;
  double best = INFINITY;
  int64_t arg = -1;
  for (int64_t v = lane; v < V; v += 32) {
    const uint64_t c = __ldg(codes + v);
    const int ijk[3] = {(int)compact3(c), (int)compact3(c >> 1), (int)compact3(c >> 2)};
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double l = cell_lo(ijk[a], res), h = dadd(l, edge);  // voxel_bounds (octree.py:285-290)
      double g = np_max(np_max(dsub(l, qx[a]), dsub(qx[a], h)), 0.0);
      g = dmul(g, g);
      s = a == 0 ? g : dadd(s, g);
    }
    if (s < best) {  // strict: the first minimum per lane (lanes scan ascending v)
      best = s;
      arg = v;
    }
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const double ob = __shfl_xor_sync(FULL, best, off);
    const int64_t oa = __shfl_xor_sync(FULL, arg, off);
    if (ob < best || (ob == best && oa >= 0 && (arg < 0 || oa < arg))) {
      best = ob;
      arg = oa;
    }
  }
  if (lane < 3) {
    const uint64_t c = __ldg(codes + arg);
    const int ijk = (int)compact3(c >> lane);
    const double l = cell_lo(ijk, res), h = dadd(l, edge);
    // clamp_into (octree.py:293-300): clip(x, lo, hi - (hi - lo) * 1e-9)
    const double top = dsub(h, dmul(dsub(h, l), 1e-9));
    anchor[3 * q + lane] = np_min(np_max(qx[lane], l), top);
  }
  if (lane == 0) gap[q] = __dsqrt_rn(best);
}

constexpr int NN_NT = 128;
constexpr int NN_TILE = 1024;

__global__ void __launch_bounds__(NN_NT) k_nn_dist(const double* __restrict__ qp, int64_t nq,
                                                   const double* __restrict__ bp, int64_t nb, double* out) {
  __shared__ double sb[NN_TILE * 3];
  const int64_t i = (int64_t)blockIdx.x * NN_NT + threadIdx.x;
  const bool own = i < nq;
  const double x = own ? qp[3 * i] : 0.0, y = own ? qp[3 * i + 1] : 0.0, z = own ? qp[3 * i + 2] : 0.0;
  double best = INFINITY;
  for (int64_t t0 = 0; t0 < nb; t0 += NN_TILE) {
    const int cnt = (int)((nb - t0) < NN_TILE ? (nb - t0) : NN_TILE);
    __syncthreads();
    for (int k = threadIdx.x; k < cnt * 3; k += NN_NT) sb[k] = bp[3 * t0 + k];
    __syncthreads();
    for (int k = 0; k < cnt; ++k) {
      // norm(points - q): ((dx^2 + dy^2) + dz^2) (metrics.py:100-102)
      const double dx = dsub(sb[3 * k], x), dy = dsub(sb[3 * k + 1], y), dz = dsub(sb[3 * k + 2], z);
      const double s = dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz));
      best = s < best ? s : best;
    }
  }
  if (own) out[i] = __dsqrt_rn(best);
}

}  // namespace ng

using namespace ng;

extern "C" {

int ng_trace_sdf(int32_t kind, const double* params, int32_t n_params, const double* origins, const double* dirs,
                 int64_t n, double delta, double far_plane, int32_t max_iters, uint8_t* hit, double* t_hit,
                 void* stream) {
  if (kind < 1 || kind > 3) {
    set_error("unknown built-in sdf kind %d", kind);
    return NG_ERR_CONFIG;
  }
  if (n <= 0) return NG_OK;
  k_trace_sdf<<<mgrid(n, 128), 128, 0, (cudaStream_t)stream>>>(kind, params, n_params, origins, dirs, n, delta,
                                                                 far_plane, max_iters, hit, t_hit);
  NG_CHECK_LAUNCH("ng_trace_sdf");
  return NG_OK;
}

int ng_nearest_voxel(const ng_octree* tree, int32_t level, const double* pts, int64_t n, double* anchor, double* gap,
                     void* stream) {
  if (level < 0 || level > tree->max_level) {
    set_error("level %d outside 0..%d", level, tree->max_level);
    return NG_ERR_STRUCTURAL;
  }
  if (n <= 0) return NG_OK;
  k_nearest_voxel<<<mgrid(n * 32, 256), 256, 0, (cudaStream_t)stream>>>(*tree, level, pts, n, anchor, gap);
  NG_CHECK_LAUNCH("ng_nearest_voxel");
  return NG_OK;
}

int ng_nn_dist(const double* queries, int64_t nq, const double* points, int64_t np_, double* out, void* stream) {
  if (np_ <= 0) {
    set_error("empty point set");
    return NG_ERR_STRUCTURAL;
  }
  if (nq <= 0) return NG_OK;
  k_nn_dist<<<mgrid(nq, NN_NT), NN_NT, 0, (cudaStream_t)stream>>>(queries, nq, points, np_, out);
  NG_CHECK_LAUNCH("ng_nn_dist");
  return NG_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- epoch sampler
// _trace_to_surface (sampling.py:109-139) and _bisect_crossing (142-149) for
// a built-in SDF, one thread per ray, numpy's operation order: rays that
// start inside trace the negated field; a sign change between steps is
// refined by bisection. Writes the surface point (or NaN) per ray; the host
// keeps the hits in ray order.
namespace ng {
__global__ void k_surface_trace(int kind, const double* __restrict__ prm, int np_, const double* __restrict__ o,
                                const double* __restrict__ d, int64_t n, double tol, double t_max, int max_iters,
                                int bisect_iters, double* __restrict__ pts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double ox = o[3 * i], oy = o[3 * i + 1], oz = o[3 * i + 2];
  const double dx = d[3 * i], dy = d[3 * i + 1], dz = d[3 * i + 2];
  auto f_at = [&](double t) {
    return sdf_builtin(kind, prm, np_, dadd(ox, dmul(t, dx)), dadd(oy, dmul(t, dy)), dadd(oz, dmul(t, dz)));
  };
  const double f0 = sdf_builtin(kind, prm, np_, ox, oy, oz);
  const double side = f0 < 0.0 ? -1.0 : 1.0;
  double t = 0.0, f_prev = dmul(side, f0), t_prev = 0.0;
  double hit_t = NAN;
  if (!(fabs(f0) >= tol)) {
    hit_t = 0.0;
  } else {
    for (int it = 0; it < max_iters; ++it) {
      t = dadd(t, f_prev);
      const bool over = t > t_max;
      const double f = dmul(side, f_at(t));
      const bool done = (fabs(f) < tol) && !over;
      if (done) {
        hit_t = t;
        break;
      }
      if (f < 0.0 && !over) {  // crossed: bisect between the last two steps
        double lo = t_prev, hi = t;
        for (int b = 0; b < bisect_iters; ++b) {
          const double mid = dmul(0.5, dadd(lo, hi));
          const bool hs = dmul(side, f_at(mid)) < 0.0;
          hi = hs ? mid : hi;
          lo = hs ? lo : mid;
        }
        hit_t = dmul(0.5, dadd(lo, hi));
        break;
      }
      if (over) break;
      f_prev = f;
      t_prev = t;
    }
  }
  pts[3 * i] = dadd(ox, dmul(hit_t, dx));
  pts[3 * i + 1] = dadd(oy, dmul(hit_t, dy));
  pts[3 * i + 2] = dadd(oz, dmul(hit_t, dz));
}
}  // namespace ng

extern "C" int ng_surface_trace(int32_t kind, const double* params, int32_t n_params, const double* origins,
                                const double* dirs, int64_t n, double tol, double t_max, int32_t max_iters,
                                int32_t bisect_iters, double* points, void* stream) {
  if (kind < 1 || kind > 3) {
    ng::set_error("unknown built-in sdf kind %d", kind);
    return NG_ERR_CONFIG;
  }
  if (n <= 0) return NG_OK;
  ng::k_surface_trace<<<(int)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      kind, params, n_params, origins, dirs, n, tol, t_max, max_iters, bisect_iters, points);
  NG_CHECK_LAUNCH("ng_surface_trace");
  return NG_OK;
}
