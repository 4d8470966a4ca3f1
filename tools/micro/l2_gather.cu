// Microbenchmark: random 128-byte row gathers, the access pattern of the
// feature / presummed tables (one row = 32 fp32 channels). Eight lanes
// read one row with 16-byte loads (the gather layout of eval.cuh), rows are
// drawn by a hash (no index traffic), every warp keeps UNROLL x 4 rows in
// flight. Table sizes: 12 MB and 15 MB (the LOD5 presummed table and Z,
// L2-resident after the first pass), then 2 GB (HBM). Reports the best of
// 10 timed launches in GB/s of row bytes, and writes the L2 figure as JSON
// for bench.py (profiles/l2_gather_peak.json).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2_gather l2_gather.cu
//   ./l2_gather [json_out]
#include <cstdio>
#include <cstdint>
#include <vector>

#ifndef UNROLL
#define UNROLL 8
#endif

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__global__ void __launch_bounds__(256) k_gather(const int4* __restrict__ table, uint32_t rows, int iters,
                                                uint32_t seed, int4* __restrict__ sink) {
  const int lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int quad = lane & 7;   // 16-byte chunk of the row
  const int slot = lane >> 3;  // which of the 4 rows this instruction covers
  int4 acc = make_int4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
    int4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const uint32_t r = mix(seed ^ (warp * 0x9e3779b9U) ^ ((uint32_t)(it * UNROLL + u) * 4 + slot) * 0x85ebca6bU) % rows;
      v[u] = __ldg(table + (size_t)r * 8 + quad);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      acc.x ^= v[u].x;
      acc.y ^= v[u].y;
      acc.z ^= v[u].z;
      acc.w ^= v[u].w;
    }
  }
  if (acc.x == 0x7fffffff && acc.y == 1) sink[0] = acc;
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t big = (size_t)2 << 30;
  int4* table;
  int4* sink;
  cudaMalloc(&table, big);
  cudaMalloc(&sink, 64);
  cudaMemset(table, 1, big);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double l2_best = 0.0;
  const size_t sizes[] = {(size_t)12165504, (size_t)117197 * 128, big};
  for (size_t bytes : sizes) {
    const uint32_t rows = (uint32_t)(bytes / 128);
    for (int per_sm : {4, 8}) {
      const int grid = sms * per_sm, threads = 256, iters = 64;
      double best = 0.0;
      for (int rep = 0; rep < 12; ++rep) {
        cudaEventRecord(a);
        k_gather<<<grid, threads>>>(table, rows, iters, 1234u + rep, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        const double moved = (double)grid * threads / 32 * iters * UNROLL * 4 * 128;
        if (rep >= 2 && moved / (ms * 1e-3) / 1e9 > best) best = moved / (ms * 1e-3) / 1e9;
      }
      printf("table %8.1f MB, %d CTAs/SM x 256 threads: %8.1f GB/s of 128-B rows (%s)\n", bytes / 1e6, per_sm, best,
             cudaGetErrorString(cudaGetLastError()));
      if (bytes < ((size_t)64 << 20) && best > l2_best) l2_best = best;
    }
  }
  if (argc > 1) {
    FILE* f = fopen(argv[1], "w");
    if (f) {
      fprintf(f,
              "{\"gbs\": %.1f, \"what\": \"random 128-B row gathers (8 lanes x 16 B per row) from a 12-15 MB table "
              "resident in L2, best of 10 launches\", \"tool\": \"tools/micro/l2_gather.cu\", \"sms\": %d}\n",
              l2_best, sms);
      fclose(f);
    }
  }
  return 0;
}
