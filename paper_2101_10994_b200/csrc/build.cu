// Octree construction on the device (octree.py:146-256).
//
// Occupancy lives in Morton-ordered bitmaps (one bit per cell, res^3 bits per
// level): marking is an atomicOr, np.unique's sorted order is the bit order,
// parent closure is a byte-OR, and every "searchsorted" of the reference
// becomes a rank query (word prefix popcount + popc within the word).
// All steps are deterministic; the result is bit-identical to build_octree.
#include "common.cuh"
#include "sdf.cuh"

#include <stdarg.h>
#include <stdlib.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <stdio.h>
#include <string.h>

namespace ng {

static thread_local char g_err[512];

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return NG_OK;
  set_error("%s: %s", where, cudaGetErrorString(e));
  return NG_ERR_CUDA;
}

int launch_status(const char* where) { return cuda_status(cudaGetLastError(), where); }

int malloc_async(void** p, size_t bytes, cudaStream_t s, const char* where) {
  static std::atomic<unsigned long long> kept{0};  // devices whose pool threshold is set (bit per device)
  const int d = current_device();
  const unsigned long long bit = 1ull << (d & 63);
  if (!(kept.load(std::memory_order_acquire) & bit)) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    kept.fetch_or(bit, std::memory_order_acq_rel);
  }
  return cuda_status(cudaMallocAsync(p, bytes, s), where);
}

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

int sm_count() {
  constexpr int kMaxDev = 64;
  static std::atomic<int> cached[kMaxDev];
  const int dev = current_device();
  const int slot = (dev >= 0 && dev < kMaxDev) ? dev : 0;
  int v = cached[slot].load(std::memory_order_relaxed);
  if (v <= 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    cached[slot].store(v, std::memory_order_relaxed);
  }
  return v;
}

int env_int(const char* name, int def) {
  const char* e = getenv(name);
  return e ? atoi(e) : def;
}

int set_smem_limit(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> have;
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(mu);
  size_t& h = have[{dev, kernel}];
  if (bytes > h) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(bytes, 48 * 1024));
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute");
    h = bytes;
  }
  return NG_OK;
}

// ------------------------------------------------------------------ kernels

__global__ void k_mark_samples(const double* __restrict__ pts, int64_t n, int res,
                               unsigned long long* bitmap) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int ci = bin_axis(pts[3 * i + 0], res);
    int cj = bin_axis(pts[3 * i + 1], res);
    int ck = bin_axis(pts[3 * i + 2], res);
    uint64_t c = morton(ci, cj, ck);
    atomicOr(bitmap + (c >> 6), 1ull << (c & 63));
  }
}

// _corner_test_codes (octree.py:238-243): cell (i,j,k) is occupied when the
// minimum of its 8 corner |d| (fp32) is <= tol, compared in fp64.
__global__ void k_mark_lattice(const float* __restrict__ absd, int res, double tol,
                               unsigned long long* bitmap) {
  const int64_t n1 = res + 1;
  const int64_t cells = (int64_t)res * res * res;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < cells;
       c += (int64_t)gridDim.x * blockDim.x) {
    int k = (int)(c % res);
    int j = (int)((c / res) % res);
    int i = (int)(c / ((int64_t)res * res));
    float m = INFINITY;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      int64_t ii = i + (q & 1), jj = j + ((q >> 1) & 1), kk = k + ((q >> 2) & 1);
      float v = __ldg(absd + (ii * n1 + jj) * n1 + kk);
      // np.minimum propagates NaN
      m = (m != m) ? m : ((v != v) ? v : fminf(m, v));
    }
    if ((double)m <= tol) {
      uint64_t code = morton(i, j, k);
      atomicOr(bitmap + (code >> 6), 1ull << (code & 63));
    }
  }
}

// built-in SDFs: sdf.cuh

__global__ void k_sdf_lattice(int kind, const double* __restrict__ prm, int np_, int res,
                              float* __restrict__ absd) {
  const int64_t n1 = res + 1;
  const int64_t tot = n1 * n1 * n1;
  const double step = 2.0 / (double)res;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < tot;
       c += (int64_t)gridDim.x * blockDim.x) {
    int64_t k = c % n1, j = (c / n1) % n1, i = c / (n1 * n1);
    // axis = DOMAIN_MIN + arange(n) * (span / res)  (octree.py:228)
    double x = dadd(-1.0, dmul((double)i, step));
    double y = dadd(-1.0, dmul((double)j, step));
    double z = dadd(-1.0, dmul((double)k, step));
    absd[c] = (float)fabs(sdf_builtin(kind, prm, np_, x, y, z));
  }
}

__global__ void k_sdf_eval(int kind, const double* __restrict__ prm, int np_,
                           const double* __restrict__ pts, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = sdf_builtin(kind, prm, np_, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
}

// Parent word w covers parent codes 64w..64w+63 = child bytes 64w..64w+63.
__global__ void k_bitmap_parent(const uint64_t* __restrict__ child, int64_t child_words,
                                uint64_t* __restrict__ parent, int64_t parent_words) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < parent_words;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint64_t out = 0;
    for (int q = 0; q < 8; ++q) {
      int64_t cw = 8 * w + q;
      uint64_t v = cw < child_words ? child[cw] : 0ull;
#pragma unroll
      for (int b = 0; b < 8; ++b)
        if ((v >> (8 * b)) & 0xffull) out |= 1ull << (8 * q + b);
    }
    parent[w] = out;
  }
}

// Exclusive popcount prefix per word (single pass, decoupled look-back).
constexpr int RANK_NT = 256;
constexpr int RANK_ITEMS = 8;
__global__ void __launch_bounds__(RANK_NT) k_bitmap_rank(const uint64_t* __restrict__ bm,
                                                         int64_t n_words, uint32_t* __restrict__ rank,
                                                         int64_t* d_total,
                                                         unsigned long long* states,
                                                         unsigned int* tile_counter) {
  __shared__ int64_t sm_warp[RANK_NT / 32 + 1];
  __shared__ int64_t sm_tile;
  __shared__ int64_t sm_excl;
  const int64_t tile_elems = (int64_t)RANK_NT * RANK_ITEMS;
  const int64_t n_tiles = (n_words + tile_elems - 1) / tile_elems;
  while (true) {
    if (threadIdx.x == 0) sm_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const int64_t tile = sm_tile;
    if (tile >= n_tiles) break;
    const int64_t base = tile * tile_elems + (int64_t)threadIdx.x * RANK_ITEMS;
    int cnt[RANK_ITEMS];
    int64_t sum = 0;
#pragma unroll
    for (int q = 0; q < RANK_ITEMS; ++q) {
      int64_t w = base + q;
      cnt[q] = (w < n_words) ? __popcll(bm[w]) : 0;
      sum += cnt[q];
    }
    int64_t excl;
    int64_t agg = block_excl_scan<RANK_NT>(sum, excl, sm_warp);
    if (threadIdx.x < 32) {
      const int64_t e = tile_lookback_warp(states, tile, agg);
      if (threadIdx.x == 0) sm_excl = e;
    }
    __syncthreads();
    int64_t run = sm_excl + excl;
#pragma unroll
    for (int q = 0; q < RANK_ITEMS; ++q) {
      int64_t w = base + q;
      if (w < n_words) rank[w] = (uint32_t)run;
      run += cnt[q];
    }
    if (tile == n_tiles - 1 && threadIdx.x == RANK_NT - 1) *d_total = run;
    __syncthreads();
  }
}

__global__ void k_bitmap_extract(const uint64_t* __restrict__ bm, const uint32_t* __restrict__ rank,
                                 int64_t n_words, uint64_t* __restrict__ codes) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_words;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint64_t v = bm[w];
    int64_t o = rank[w];
    while (v) {
      int b = __ffsll((long long)v) - 1;
      codes[o++] = (uint64_t)w * 64 + b;
      v &= v - 1;
    }
  }
}

__global__ void k_level_parents(const uint64_t* __restrict__ codes, int64_t n,
                                const uint64_t* __restrict__ pbm, const uint32_t* __restrict__ prk,
                                int32_t* __restrict__ parents) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    parents[i] = (int32_t)rank_lookup(pbm, prk, codes[i] >> 3);
}

__global__ void k_level_children(const uint64_t* __restrict__ codes, int64_t n,
                                 const uint64_t* __restrict__ cbm, const uint32_t* __restrict__ crk,
                                 int32_t* __restrict__ start, uint8_t* __restrict__ mask) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t first = codes[i] << 3;  // child codes first..first+7 share one byte
    uint64_t w = cbm[first >> 6];
    uint32_t b = (uint32_t)(first & 63);
    mask[i] = (uint8_t)((w >> b) & 0xffull);
    start[i] = (int32_t)(crk[first >> 6] + __popcll(w & ((1ull << b) - 1ull)));
  }
}

// _corner_table (octree.py:249-256): corner coords ijk + offset(j) encoded as
// Morton keys (coords <= res need one extra bit per axis).
__global__ void k_corner_mark(const uint64_t* __restrict__ codes, int64_t n,
                              unsigned long long* cbm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t c = codes[i];
    uint32_t x = compact3(c), y = compact3(c >> 1), z = compact3(c >> 2);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint64_t key = morton(x + (q & 1), y + ((q >> 1) & 1), z + ((q >> 2) & 1));
      atomicOr(cbm + (key >> 6), 1ull << (key & 63));
    }
  }
}

__global__ void k_corner_table(const uint64_t* __restrict__ codes, int64_t n,
                               const uint64_t* __restrict__ cbm, const uint32_t* __restrict__ crk,
                               int32_t offset, int32_t* __restrict__ corners) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t c = codes[i];
    uint32_t x = compact3(c), y = compact3(c >> 1), z = compact3(c >> 2);
    int32_t out[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint64_t key = morton(x + (q & 1), y + ((q >> 1) & 1), z + ((q >> 2) & 1));
      out[q] = offset + (int32_t)rank_lookup(cbm, crk, key);
    }
    int4* dst = reinterpret_cast<int4*>(corners + 8 * i);
    dst[0] = make_int4(out[0], out[1], out[2], out[3]);
    dst[1] = make_int4(out[4], out[5], out[6], out[7]);
  }
}

__global__ void k_cell_extent(const uint64_t* __restrict__ codes, int64_t n, int32_t* mm) {
  int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {-1, -1, -1};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t c = codes[i];
    int v[3] = {(int)compact3(c), (int)compact3(c >> 1), (int)compact3(c >> 2)};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = min(lo[a], v[a]);
      hi[a] = max(hi[a], v[a]);
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    for (int o = 16; o; o >>= 1) {
      lo[a] = min(lo[a], __shfl_xor_sync(FULL, lo[a], o));
      hi[a] = max(hi[a], __shfl_xor_sync(FULL, hi[a], o));
    }
  }
  if ((threadIdx.x & 31) == 0) {
    for (int a = 0; a < 3; ++a) {
      atomicMin(mm + a, lo[a]);
      atomicMax(mm + 3 + a, hi[a]);
    }
  }
}

__global__ void k_morton_encode(const int64_t* __restrict__ ijk, int64_t n, uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = morton((uint32_t)ijk[3 * i], (uint32_t)ijk[3 * i + 1], (uint32_t)ijk[3 * i + 2]);
}

__global__ void k_morton_decode(const uint64_t* __restrict__ codes, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t c = codes[i];
    out[3 * i] = compact3(c);
    out[3 * i + 1] = compact3(c >> 1);
    out[3 * i + 2] = compact3(c >> 2);
  }
}

int grid_for(int64_t n, int nt = 256) {
  int64_t b = (n + nt - 1) / nt;
  int64_t cap = (int64_t)sm_count() * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace ng

using namespace ng;

extern "C" {

int ng_abi_version(void) { return 1; }
const char* ng_last_error(void) { return ng::g_err; }
int ng_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return v;
}

int ng_morton_encode(const int64_t* ijk, int64_t n, uint64_t* codes, void* stream) {
  if (n <= 0) return NG_OK;
  k_morton_encode<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(ijk, n, codes);
  NG_CHECK_LAUNCH("ng_morton_encode");
  return NG_OK;
}

int ng_morton_decode(const uint64_t* codes, int64_t n, int64_t* ijk, void* stream) {
  if (n <= 0) return NG_OK;
  k_morton_decode<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(codes, n, ijk);
  NG_CHECK_LAUNCH("ng_morton_decode");
  return NG_OK;
}

int ng_build_mark_samples(const double* pts, int64_t n, int32_t res, uint64_t* bitmap, void* stream) {
  if (n <= 0) return NG_OK;
  k_mark_samples<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(pts, n, res,
                                                                 (unsigned long long*)bitmap);
  NG_CHECK_LAUNCH("ng_build_mark_samples");
  return NG_OK;
}

int ng_build_mark_lattice(const float* absd, int32_t res, double tol, uint64_t* bitmap, void* stream) {
  int64_t cells = (int64_t)res * res * res;
  k_mark_lattice<<<grid_for(cells), 256, 0, (cudaStream_t)stream>>>(absd, res, tol,
                                                                     (unsigned long long*)bitmap);
  NG_CHECK_LAUNCH("ng_build_mark_lattice");
  return NG_OK;
}

int ng_sdf_lattice(int32_t kind, const double* params, int32_t n_params, int32_t res, float* absd,
                   void* stream) {
  if (kind < 1 || kind > 3) {
    set_error("unknown built-in sdf kind %d", kind);
    return NG_ERR_STRUCTURAL;
  }
  int64_t n1 = res + 1;
  k_sdf_lattice<<<grid_for(n1 * n1 * n1), 256, 0, (cudaStream_t)stream>>>(kind, params, n_params,
                                                                           res, absd);
  NG_CHECK_LAUNCH("ng_sdf_lattice");
  return NG_OK;
}

int ng_sdf_eval(int32_t kind, const double* params, int32_t n_params, const double* pts, int64_t n,
                double* out, void* stream) {
  if (kind < 1 || kind > 3) {
    set_error("unknown built-in sdf kind %d", kind);
    return NG_ERR_STRUCTURAL;
  }
  if (n <= 0) return NG_OK;
  k_sdf_eval<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(kind, params, n_params, pts, n, out);
  NG_CHECK_LAUNCH("ng_sdf_eval");
  return NG_OK;
}

int ng_bitmap_parent(const uint64_t* child_bitmap, int64_t child_words, uint64_t* parent_bitmap,
                     int64_t parent_words, void* stream) {
  k_bitmap_parent<<<grid_for(parent_words), 256, 0, (cudaStream_t)stream>>>(
      child_bitmap, child_words, parent_bitmap, parent_words);
  NG_CHECK_LAUNCH("ng_bitmap_parent");
  return NG_OK;
}

int ng_bitmap_rank(const uint64_t* bitmap, int64_t n_words, uint32_t* rank, int64_t* d_total,
                   void* scratch, size_t scratch_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t tile = (int64_t)RANK_NT * RANK_ITEMS;
  int64_t tiles = (n_words + tile - 1) / tile;
  size_t need = 16 + (size_t)tiles * 8;
  if (scratch_bytes < need) {
    set_error("ng_bitmap_rank: scratch %zu < %zu bytes", scratch_bytes, need);
    return NG_ERR_CAPACITY;
  }
  if (n_words <= 0) {
    return cuda_status(cudaMemsetAsync(d_total, 0, 8, s), "ng_bitmap_rank");
  }
  int r = cuda_status(cudaMemsetAsync(scratch, 0, need, s), "ng_bitmap_rank memset");
  if (r) return r;
  unsigned int* counter = (unsigned int*)scratch;
  unsigned long long* states = (unsigned long long*)((char*)scratch + 16);
  int grid = (int)std::min<int64_t>(tiles, (int64_t)sm_count() * 4);
  k_bitmap_rank<<<grid, RANK_NT, 0, s>>>(bitmap, n_words, rank, d_total, states, counter);
  NG_CHECK_LAUNCH("ng_bitmap_rank");
  return NG_OK;
}

int ng_bitmap_extract(const uint64_t* bitmap, const uint32_t* rank, int64_t n_words, uint64_t* codes,
                      void* stream) {
  if (n_words <= 0) return NG_OK;
  k_bitmap_extract<<<grid_for(n_words), 256, 0, (cudaStream_t)stream>>>(bitmap, rank, n_words, codes);
  NG_CHECK_LAUNCH("ng_bitmap_extract");
  return NG_OK;
}

int ng_level_parents(const uint64_t* codes, int64_t n, const uint64_t* parent_bitmap,
                     const uint32_t* parent_rank, int32_t* parents, void* stream) {
  if (n <= 0) return NG_OK;
  k_level_parents<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(codes, n, parent_bitmap,
                                                                  parent_rank, parents);
  NG_CHECK_LAUNCH("ng_level_parents");
  return NG_OK;
}

int ng_level_children(const uint64_t* codes, int64_t n, const uint64_t* child_bitmap,
                      const uint32_t* child_rank, int32_t* child_start, uint8_t* child_mask,
                      void* stream) {
  if (n <= 0) return NG_OK;
  k_level_children<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(codes, n, child_bitmap, child_rank,
                                                                   child_start, child_mask);
  NG_CHECK_LAUNCH("ng_level_children");
  return NG_OK;
}

int ng_corner_mark(const uint64_t* codes, int64_t n, uint64_t* corner_bitmap, void* stream) {
  if (n <= 0) return NG_OK;
  k_corner_mark<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(codes, n,
                                                                (unsigned long long*)corner_bitmap);
  NG_CHECK_LAUNCH("ng_corner_mark");
  return NG_OK;
}

int ng_corner_table(const uint64_t* codes, int64_t n, const uint64_t* corner_bitmap,
                    const uint32_t* corner_rank, int32_t offset, int32_t* corners, void* stream) {
  if (n <= 0) return NG_OK;
  k_corner_table<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(codes, n, corner_bitmap, corner_rank,
                                                                 offset, corners);
  NG_CHECK_LAUNCH("ng_corner_table");
  return NG_OK;
}

int ng_cell_extent(const uint64_t* codes, int64_t n, int32_t* d_minmax6, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int32_t init[6] = {INT_MAX, INT_MAX, INT_MAX, -1, -1, -1};
  int r = cuda_status(cudaMemcpyAsync(d_minmax6, init, sizeof(init), cudaMemcpyHostToDevice, s),
                      "ng_cell_extent init");
  if (r) return r;
  // the host copy above is from a stack buffer: make it complete before returning
  r = cuda_status(cudaStreamSynchronize(s), "ng_cell_extent sync");
  if (r) return r;
  if (n <= 0) return NG_OK;
  k_cell_extent<<<grid_for(n), 256, 0, s>>>(codes, n, d_minmax6);
  NG_CHECK_LAUNCH("ng_cell_extent");
  return NG_OK;
}

}  // extern "C"
