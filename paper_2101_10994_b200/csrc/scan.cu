// exclusive_sum (traversal.py:113-144): single-pass int64 exclusive scan with
// decoupled look-back. Integer addition is associative, so the result is
// bit-equal to the serial reference for any tiling.
#include "common.cuh"

namespace ng {

constexpr int SCAN_NT = 256;
constexpr int SCAN_ITEMS = 8;

__global__ void __launch_bounds__(SCAN_NT) k_exclusive_sum(const int64_t* __restrict__ in, int64_t n,
                                                           int64_t* __restrict__ out,
                                                           unsigned long long* states,
                                                           unsigned int* tile_counter) {
  __shared__ int64_t sm_warp[SCAN_NT / 32 + 1];
  __shared__ int64_t sm_tile, sm_excl;
  const int64_t tile_elems = (int64_t)SCAN_NT * SCAN_ITEMS;
  const int64_t n_tiles = (n + tile_elems - 1) / tile_elems;
  while (true) {
    if (threadIdx.x == 0) sm_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const int64_t tile = sm_tile;
    if (tile >= n_tiles) break;
    // blocked arrangement: thread t owns items [base, base+ITEMS)
    const int64_t base = tile * tile_elems + (int64_t)threadIdx.x * SCAN_ITEMS;
    int64_t v[SCAN_ITEMS];
    int64_t sum = 0;
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS; ++q) {
      v[q] = (base + q < n) ? in[base + q] : 0;
      sum += v[q];
    }
    int64_t excl;
    int64_t agg = block_excl_scan<SCAN_NT>(sum, excl, sm_warp);
    if (threadIdx.x < 32) {
      const int64_t e = tile_lookback_warp(states, tile, agg);
      if (threadIdx.x == 0) sm_excl = e;
    }
    __syncthreads();
    int64_t run = sm_excl + excl;
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS; ++q) {
      if (base + q < n) out[base + q] = run;
      run += v[q];
    }
    __syncthreads();
  }
}

}  // namespace ng

using namespace ng;

extern "C" {

size_t ng_scan_scratch_bytes(int64_t n) {
  const int64_t tile = (int64_t)SCAN_NT * SCAN_ITEMS;
  int64_t tiles = (n + tile - 1) / tile;
  if (tiles < 1) tiles = 1;
  return 16 + (size_t)tiles * 8;
}

int ng_exclusive_sum_i64(const int64_t* in, int64_t n, int64_t* out, void* scratch,
                         size_t scratch_bytes, void* stream) {
  if (n <= 0) return NG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  size_t need = ng_scan_scratch_bytes(n);
  if (scratch_bytes < need) {
    set_error("ng_exclusive_sum_i64: scratch %zu < %zu bytes", scratch_bytes, need);
    return NG_ERR_CAPACITY;
  }
  int r = cuda_status(cudaMemsetAsync(scratch, 0, need, s), "ng_exclusive_sum_i64 memset");
  if (r) return r;
  const int64_t tile = (int64_t)SCAN_NT * SCAN_ITEMS;
  int64_t tiles = (n + tile - 1) / tile;
  int grid = (int)(tiles < (int64_t)sm_count() * 4 ? tiles : (int64_t)sm_count() * 4);
  k_exclusive_sum<<<grid, SCAN_NT, 0, s>>>(in, n, out, (unsigned long long*)((char*)scratch + 16),
                                           (unsigned int*)scratch);
  NG_CHECK_LAUNCH("ng_exclusive_sum_i64");
  return NG_OK;
}

}  // extern "C"
