// Microbenchmark: cost of cooperative_groups grid.sync() on this GPU.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, unsigned long long* out) {
  cg::grid_group g = cg::this_grid();
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) g.sync();
  unsigned long long t1;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = t1 - t0;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d; cudaMalloc(&d, 8);
  for (int per : {1, 2}) for (int nt : {128, 256, 512}) {
    int grid = sms * per, iters = 2000;
    void* args[] = {&iters, &d};
    cudaLaunchCooperativeKernel((void*)k, grid, nt, args, 0, 0);
    cudaLaunchCooperativeKernel((void*)k, grid, nt, args, 0, 0);
    unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("grid %d x %d threads: %.3f us per grid.sync (%s)\n", grid, nt, h / 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
}
