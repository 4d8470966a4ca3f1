// The field API in float64 with the reference's semantics
// (field.py:104-239, 337-357; render.py:155-171): trilinear, sum_features,
// decode, predict, blend, forward's outputs and query_field, computed in
// fp64 from the caller's parameters as given (fp32 or fp64 arrays, upcast
// like `Z[ids].astype(np.float64)`). These serve the Python API, the
// training-forward semantics and the reference's own tests, whose
// tolerances (1e-10 .. 1e-15) sit below fp32. The hot paths -- the frame
// (render.cu), the batched configs[2] query (query_tc.cu) -- keep their
// fp32 tables and tensor-core decoder.
//
// Thread per point. Features: (C, m) fp64, row-major (the caller's array).
// Decoders: fp64 blocks in the training layout (trainer._pack64):
// W1b[h][36] (3 x weights, m feature weights, b1 in column 35), W2[h], b2.
#include "eval.cuh"

#include <algorithm>

namespace ng {

int grid_for(int64_t n, int nt);

struct Field64 {
  const double* Z;
  int m;
  const double* dec;
  int h;
  int n_dec;
  int stride;  // doubles per decoder block
};

// psi of one level added into z[0..m); returns false when no voxel holds x.
__device__ __forceinline__ bool add_level64(const ng_octree& tree, const double* __restrict__ Z, int m, int level,
                                            const double x[3], double* z) {
  const int64_t idx = locate_point(tree, x, level);
  if (idx < 0) return false;
  const int res = tree.r0 << level;
  const int tl = level + tree.n_virtual;
  const uint64_t code = tree.codes[tl][idx];
  const int cc[3] = {(int)compact3(code), (int)compact3(code >> 1), (int)compact3(code >> 2)};
  double u[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    // f = (x - DOMAIN_MIN) * (res / span); u = clip(f - cell, 0, 1)
    const double f = dsub(dmul(dadd(x[a], 1.0), 0.5 * (double)res), (double)cc[a]);
    u[a] = f < 0.0 ? 0.0 : (f > 1.0 ? 1.0 : f);
  }
  const int32_t* ids = tree.corners[tl] + 8 * idx;
  double psi[NG_FEAT_PAD];
  for (int c = 0; c < m; ++c) psi[c] = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double wx = (j & 1) ? u[0] : dsub(1.0, u[0]);
    const double wy = ((j >> 1) & 1) ? u[1] : dsub(1.0, u[1]);
    const double wz = ((j >> 2) & 1) ? u[2] : dsub(1.0, u[2]);
    const double w = dmul(dmul(wx, wy), wz);
    const double* row = Z + (int64_t)ids[j] * m;
    for (int c = 0; c < m; ++c) psi[c] = dadd(psi[c], dmul(w, __ldg(row + c)));
  }
  // z += psi (sum_features adds whole level records, field.py:164-168)
  for (int c = 0; c < m; ++c) z[c] = dadd(z[c], psi[c]);
  return true;
}

// d = W2 relu(W1 [x, z] + b1) + b2 in fp64 (field.py:172-182).
__device__ __forceinline__ double mlp64(const double* __restrict__ dec, int h, int m, const double x[3],
                                        const double* z) {
  const double* W2 = dec + (int64_t)h * NG_W1_STRIDE;
  double out = 0.0;
  for (int j = 0; j < h; ++j) {
    const double* row = dec + (int64_t)j * NG_W1_STRIDE;
    double pre = 0.0;
    pre = dadd(pre, dmul(__ldg(row + 0), x[0]));
    pre = dadd(pre, dmul(__ldg(row + 1), x[1]));
    pre = dadd(pre, dmul(__ldg(row + 2), x[2]));
    for (int c = 0; c < m; ++c) pre = dadd(pre, dmul(__ldg(row + 3 + c), z[c]));
    pre = dadd(pre, __ldg(row + NG_W1_STRIDE - 1));  // + b1
    out = dadd(out, dmul(__ldg(W2 + j), pre > 0.0 ? pre : 0.0));
  }
  return dadd(out, __ldg(W2 + h));  // + b2
}

__device__ __forceinline__ bool finite_inputs(const double x[3], const double* z, int m) {
  bool ok = isfinite(x[0]) && isfinite(x[1]) && isfinite(x[2]);
  for (int c = 0; c < m; ++c) ok = ok && isfinite(z[c]);
  return ok;
}

// trilinear (lo == hi: that level's psi) / sum_features (levels lo..hi summed).
__global__ void k_interp64(const __grid_constant__ ng_octree tree, const double* __restrict__ Z, int m,
                           const double* __restrict__ pts, int64_t n, int lo, int hi, double* __restrict__ z,
                           uint8_t* __restrict__ mask) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    double acc[NG_FEAT_PAD];
    for (int c = 0; c < m; ++c) acc[c] = 0.0;
    for (int l = lo; l <= hi; ++l) mask[i * (hi - lo + 1) + (l - lo)] = add_level64(tree, Z, m, l, x, acc);
    for (int c = 0; c < m; ++c) z[i * m + c] = acc[c];
  }
}

__global__ void k_decode64(const double* __restrict__ dec, int h, int m, const double* __restrict__ x,
                           const double* __restrict__ z, int64_t n, double* __restrict__ out,
                           unsigned long long* nonfinite) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double xi[3] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
    double zi[NG_FEAT_PAD];
    for (int c = 0; c < m; ++c) zi[c] = z[i * m + c];
    if (!finite_inputs(xi, zi, m) && nonfinite) atomicAdd(nonfinite, 1ull);
    out[i] = mlp64(dec, h, m, xi, zi);
  }
}

// predict at every level of out_mask (one column each, ascending), or the
// blend of blend_base / blend_base + 1; inside_level >= 0 is query_field:
// points outside that level's voxels take the empty-space value undecoded.
__global__ void k_query64(const __grid_constant__ ng_octree tree, Field64 f, ng_query_args a, int out_mask,
                          int G, const double* __restrict__ pts, int64_t n, double* __restrict__ out, int ncols,
                          ng_counters* counters) {
  LaneCounters lc;
  const bool blending = a.blend_base > 0;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    if (i < n) {
      const double x[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
      const bool inside = a.inside_level < 0 || locate_point(tree, x, a.inside_level) >= 0;
      if (!inside) {
        const double e = empty_value(tree, x);
        for (int c = 0; c < ncols; ++c) out[i * ncols + c] = e;
        lc.empty += 1;
      } else {
        double z[NG_FEAT_PAD];
        for (int c = 0; c < f.m; ++c) z[c] = 0.0;
        unsigned present = 0;
        int col = 0;
        double lo_v = 0.0, hi_v = 0.0;
        for (int L = 1; L <= G; ++L) {
          if (add_level64(tree, f.Z, f.m, L, x, z)) present |= 1u << (L - 1);
          if (!((out_mask >> (L - 1)) & 1)) continue;
          double v;
          if (present) {
            if (!finite_inputs(x, z, f.m)) lc.nonfinite += 1;
            v = mlp64(f.dec + (int64_t)(L - 1) * f.stride, f.h, f.m, x, z);
            lc.evals += 1;
            if (!((present >> (L - 1)) & 1u)) lc.missing += 1;
          } else {
            v = empty_value(tree, x);
            lc.empty += 1;
          }
          if (blending) {
            if (L == a.blend_base) lo_v = v; else hi_v = v;
          } else {
            out[i * ncols + col] = v;
          }
          ++col;
        }
        // (1 - alpha) * lo + alpha * hi (field.py:237-239)
        if (blending) out[i] = dadd(dmul(dsub(1.0, a.blend_alpha), lo_v), dmul(a.blend_alpha, hi_v));
      }
    }
  }
  lc.flush(counters);
}

}  // namespace ng

using namespace ng;

extern "C" {

int ng_interp64(const ng_octree* tree, const double* Z, int32_t m, const double* pts, int64_t n, int32_t level_lo,
                int32_t level_hi, double* z, uint8_t* mask, void* stream) {
  if (level_lo < 1 || level_hi > tree->max_level || level_lo > level_hi) {
    set_error("levels %d..%d outside 1..%d", level_lo, level_hi, tree->max_level);
    return NG_ERR_STRUCTURAL;
  }
  if (m < 1 || m > NG_FEAT_PAD) {
    set_error("feature dim %d outside 1..%d", m, NG_FEAT_PAD);
    return NG_ERR_STRUCTURAL;
  }
  if (n <= 0) return NG_OK;
  k_interp64<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(*tree, Z, m, pts, n, level_lo, level_hi, z, mask);
  NG_CHECK_LAUNCH("ng_interp64");
  return NG_OK;
}

int ng_decode64(const double* decoder, int32_t h, int32_t m, const double* x, const double* z, int64_t n,
                double* out, int64_t* d_nonfinite, void* stream) {
  if (m < 0 || m > NG_FEAT_PAD || h < 1) {
    set_error("decoder shape m=%d h=%d unsupported (m <= 32)", m, h);
    return NG_ERR_STRUCTURAL;
  }
  if (n <= 0) return NG_OK;
  k_decode64<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(decoder, h, m, x, z, n, out,
                                                                 (unsigned long long*)d_nonfinite);
  NG_CHECK_LAUNCH("ng_decode64");
  return NG_OK;
}

int ng_query64(const ng_octree* tree, const double* Z, int32_t m, const double* decoders, int32_t h,
               int32_t n_decoders, int32_t dec_stride, const ng_query_args* args, const double* pts, int64_t n,
               double* out, ng_counters* d_counters, void* stream) {
  const ng_query_args a = *args;
  int out_mask, G, ncols;
  if (m < 1 || m > NG_FEAT_PAD || h < 1 || n_decoders < 1 || dec_stride < h * NG_W1_STRIDE + h + 1) {
    set_error("field shape m=%d h=%d decoders=%d stride=%d unsupported", m, h, n_decoders, dec_stride);
    return NG_ERR_STRUCTURAL;
  }
  if (a.blend_base > 0) {
    if (a.blend_base + 1 > n_decoders || !(a.blend_alpha > 0.0 && a.blend_alpha < 1.0)) {
      set_error("blend level %d + %g outside 1..%d", a.blend_base, a.blend_alpha, n_decoders);
      return NG_ERR_STRUCTURAL;
    }
    out_mask = (1 << (a.blend_base - 1)) | (1 << a.blend_base);
    G = a.blend_base + 1;
    ncols = 1;
  } else {
    out_mask = a.out_levels;
    if (out_mask <= 0 || out_mask >= (1 << n_decoders)) {
      set_error("decoder levels mask 0x%x outside 1..%d", out_mask, n_decoders);
      return NG_ERR_STRUCTURAL;
    }
    G = 32 - __builtin_clz((unsigned)out_mask);
    ncols = __builtin_popcount((unsigned)out_mask);
  }
  if (a.inside_level > tree->max_level || G > tree->max_level) {
    set_error("query level above max %d", tree->max_level);
    return NG_ERR_STRUCTURAL;
  }
  if (n <= 0) return NG_OK;
  Field64 f{Z, m, decoders, h, n_decoders, dec_stride};
  k_query64<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(*tree, f, a, out_mask, G, pts, n, out, ncols,
                                                                d_counters);
  NG_CHECK_LAUNCH("ng_query64");
  return NG_OK;
}

}  // extern "C"
