// Batched SDF queries: predict / forward / blend / query_field
// (field.py:194-239, 337-357; render.py:155-171), locate (octree.py:259-282),
// sum_features / trilinear (field.py:138-169) and empty_space_value.
#include "eval.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace ng {

int grid_for(int64_t n, int nt);
int run_query_tc(const ng_octree& tree, const ng_field& f, const ng_query_args& a, int G, int out_mask,
                 int dec_first, int dec_last, int ncols, const double* pts, int64_t n, double* out,
                 ng_counters* counters, cudaStream_t s);

constexpr int Q_NW = 8;  // warps per CTA

size_t query_smem_bytes(int n_dec, int stride, int nw) {
  return (size_t)n_dec * stride * sizeof(float) + (size_t)nw * sizeof(WarpScratch);
}

template <int NW>
__global__ void __launch_bounds__(NW * 32) k_query(const __grid_constant__ ng_octree tree, ng_field f,
                                                  ng_query_args a, int G, int out_mask, int dec_first,
                                                  int dec_last, const double* __restrict__ pts, int64_t n,
                                                  double* __restrict__ out, int ncols,
                                                  ng_counters* counters) {
  extern __shared__ float4 smem4[];
  float* dec = reinterpret_cast<float*>(smem4);
  const int ndec = dec_last - dec_first + 1;
  WarpScratch* wsa = reinterpret_cast<WarpScratch*>(dec + ndec * f.dec_stride);
  stage_decoders(dec, f.decoders, dec_first, dec_last, f.dec_stride);
  const int w = threadIdx.x >> 5;
  WarpScratch& ws = wsa[w];
  EvalCtx c;
  c.Z = f.Z;
  c.dec = dec;
  c.dec_first = dec_first;
  c.dec_stride = f.dec_stride;
  c.h = f.h;
  c.gather_level = G;
  c.inside_level = a.inside_level;
  c.out_mask = out_mask;
  const bool blending = a.blend_base > 0;
  const double alpha = a.blend_alpha;
  LaneCounters lc;
  const int64_t n_chunks = (n + 31) / 32;
  for (int64_t chunk = (int64_t)blockIdx.x * NW + w; chunk < n_chunks; chunk += (int64_t)gridDim.x * NW) {
    const int64_t i = chunk * 32 + lane_id();
    const bool act = i < n;
    double x[3] = {0.0, 0.0, 0.0};
    if (act) {
      x[0] = pts[3 * i];
      x[1] = pts[3 * i + 1];
      x[2] = pts[3 * i + 2];
    }
    int col = 0;
    double lo_v = 0.0, hi_v = 0.0;
    EvalLane r = warp_eval(tree, c, ws, act, x, SimtMlp{c}, [&](int L, float d, bool bad, const EvalLane& er) {
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
      // blend (field.py:237-239): (1 - alpha) * lo + alpha * hi; points outside
      // the query_field level take the empty-space value directly (render.py:166-168)
      if (blending)
        out[i] = r.inside ? dadd(dmul(dsub(1.0, alpha), lo_v), dmul(alpha, hi_v)) : empty_value(tree, x);
    }
  }
  lc.flush(counters);
}

__global__ void k_locate(const __grid_constant__ ng_octree tree, const double* __restrict__ pts, int64_t n,
                         int level, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double x[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    out[i] = locate_point(tree, x, level);
  }
}

// sum_features / trilinear in float64 (thread per point; API path, not hot).
__global__ void k_interp(const __grid_constant__ ng_octree tree, const float* __restrict__ Z, int m,
                         const double* __restrict__ pts, int64_t n, int lo, int hi,
                         double* __restrict__ z, uint8_t* __restrict__ mask) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double x[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    for (int c = 0; c < m; ++c) z[i * m + c] = 0.0;
    for (int l = lo; l <= hi; ++l) {
      const int64_t idx = locate_point(tree, x, l);
      mask[i * (hi - lo + 1) + (l - lo)] = idx >= 0;
      if (idx < 0) continue;
      const int res = tree.r0 << l;
      const int tl = l + tree.n_virtual;
      const uint64_t code = tree.codes[tl][idx];
      const int cc[3] = {(int)compact3(code), (int)compact3(code >> 1), (int)compact3(code >> 2)};
      double u[3];
      for (int ax = 0; ax < 3; ++ax) {
        double fv = dsub(dmul(dadd(x[ax], 1.0), 0.5 * (double)res), (double)cc[ax]);
        u[ax] = fv < 0.0 ? 0.0 : (fv > 1.0 ? 1.0 : fv);
      }
      const int32_t* ids = tree.corners[tl] + 8 * idx;
      for (int j = 0; j < 8; ++j) {
        double wx = (j & 1) ? u[0] : dsub(1.0, u[0]);
        double wy = ((j >> 1) & 1) ? u[1] : dsub(1.0, u[1]);
        double wz = ((j >> 2) & 1) ? u[2] : dsub(1.0, u[2]);
        double wj = dmul(dmul(wx, wy), wz);
        const float* row = Z + (int64_t)ids[j] * NG_FEAT_PAD;
        for (int c = 0; c < m; ++c) z[i * m + c] = dadd(z[i * m + c], dmul(wj, (double)row[c]));
      }
    }
  }
}

__global__ void k_empty(const __grid_constant__ ng_octree tree, const double* __restrict__ pts, int64_t n,
                        double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double x[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    out[i] = empty_value(tree, x);
  }
}

// decode (field.py:172-182) on caller-supplied features; thread per point.
__global__ void k_decode(const float* __restrict__ dec, int h, int m, const double* __restrict__ x,
                         const double* __restrict__ z, int64_t n, double* __restrict__ out,
                         unsigned long long* nonfinite) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float xin[3] = {(float)x[3 * i], (float)x[3 * i + 1], (float)x[3 * i + 2]};
    __align__(16) float zr[32];
    for (int k = 0; k < 32; ++k) zr[k] = k < m ? (float)z[i * m + k] : 0.f;
    bool bad = false;
    float v = mlp_eval(dec, h, xin, zr, bad);
    bool xbad = !(isfinite(x[3 * i]) && isfinite(x[3 * i + 1]) && isfinite(x[3 * i + 2]));
    if ((bad || xbad) && nonfinite) atomicAdd(nonfinite, 1ull);
    out[i] = (double)v;
  }
}

int run_query(const ng_octree& tree, const ng_field& f, const ng_query_args& a, const double* pts, int64_t n,
              double* out, ng_counters* counters, cudaStream_t s) {
  int out_mask, G, ncols;
  if (a.blend_base > 0) {
    if (a.blend_base + 1 > f.n_decoders || !(a.blend_alpha > 0.0 && a.blend_alpha < 1.0)) {
      set_error("blend level %d + %g outside 1..%d", a.blend_base, a.blend_alpha, f.n_decoders);
      return NG_ERR_STRUCTURAL;
    }
    out_mask = (1 << (a.blend_base - 1)) | (1 << a.blend_base);
    G = a.blend_base + 1;
    ncols = 1;
  } else {
    out_mask = a.out_levels;
    if (out_mask <= 0 || out_mask >= (1 << f.n_decoders)) {
      set_error("decoder levels mask 0x%x outside 1..%d", out_mask, f.n_decoders);
      return NG_ERR_STRUCTURAL;
    }
    G = 32 - __builtin_clz((unsigned)out_mask);
    ncols = __builtin_popcount((unsigned)out_mask);
  }
  if (a.inside_level > tree.max_level) {
    set_error("query level %d above max %d", a.inside_level, tree.max_level);
    return NG_ERR_STRUCTURAL;
  }
  if (n <= 0) return NG_OK;
  const int dec_first = __builtin_ctz((unsigned)out_mask) + 1;
  const int dec_last = G;
  // tensor-core decoder (query_tc.cu) unless NG_DECODER=simt
  static const bool use_tc = [] {
    const char* e = getenv("NG_DECODER");
    return !(e && strcmp(e, "simt") == 0);
  }();
  if (use_tc) {
    int r = run_query_tc(tree, f, a, G, out_mask, dec_first, dec_last, ncols, pts, n, out, counters, s);
    if (r != NG_ERR_CAPACITY) return r;
  }
  const size_t smem = query_smem_bytes(dec_last - dec_first + 1, f.dec_stride, Q_NW);
  if (int r = set_smem_limit((const void*)k_query<Q_NW>, smem)) return r;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query<Q_NW>, Q_NW * 32, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t chunks = (n + 31) / 32;
  int64_t grid = std::min<int64_t>((chunks + Q_NW - 1) / Q_NW, (int64_t)sm_count() * per_sm);
  k_query<Q_NW><<<(int)grid, Q_NW * 32, smem, s>>>(tree, f, a, G, out_mask, dec_first, dec_last, pts, n, out,
                                                   ncols, counters);
  NG_CHECK_LAUNCH("ng_query");
  return NG_OK;
}

}  // namespace ng

using namespace ng;

extern "C" {

int ng_query(const ng_octree* tree, const ng_field* fld, const ng_query_args* args, const double* pts,
             int64_t n, double* out, ng_counters* d_counters, void* stream) {
  return run_query(*tree, *fld, *args, pts, n, out, d_counters, (cudaStream_t)stream);
}

int ng_decode(const float* decoder, int32_t h, int32_t m, const double* x, const double* z, int64_t n,
              double* out, int64_t* d_nonfinite, void* stream) {
  if (m > NG_FEAT_PAD || m < 0 || h < 1) {
    set_error("decoder shape m=%d h=%d unsupported (m <= 32)", m, h);
    return NG_ERR_STRUCTURAL;
  }
  if (n <= 0) return NG_OK;
  k_decode<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(decoder, h, m, x, z, n, out,
                                                               (unsigned long long*)d_nonfinite);
  NG_CHECK_LAUNCH("ng_decode");
  return NG_OK;
}

int ng_locate(const ng_octree* tree, const double* pts, int64_t n, int32_t level, int64_t* out_index,
              void* stream) {
  if (level < 0 || level > tree->max_level) {
    set_error("level %d outside 0..%d", level, tree->max_level);
    return NG_ERR_STRUCTURAL;
  }
  if (n <= 0) return NG_OK;
  k_locate<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(*tree, pts, n, level, out_index);
  NG_CHECK_LAUNCH("ng_locate");
  return NG_OK;
}

int ng_interp(const ng_octree* tree, const ng_field* fld, const double* pts, int64_t n, int32_t level_lo,
              int32_t level_hi, double* z, uint8_t* mask, void* stream) {
  if (level_lo < 1 || level_hi > tree->max_level || level_lo > level_hi) {
    set_error("levels %d..%d outside 1..%d", level_lo, level_hi, tree->max_level);
    return NG_ERR_STRUCTURAL;
  }
  if (n <= 0) return NG_OK;
  k_interp<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(*tree, fld->Z, fld->m, pts, n, level_lo,
                                                               level_hi, z, mask);
  NG_CHECK_LAUNCH("ng_interp");
  return NG_OK;
}

int ng_empty_value(const ng_octree* tree, const double* pts, int64_t n, double* out, void* stream) {
  if (n <= 0) return NG_OK;
  k_empty<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(*tree, pts, n, out);
  NG_CHECK_LAUNCH("ng_empty_value");
  return NG_OK;
}

}  // extern "C"
