// Microbenchmark: event-timed duration of an empty kernel and of a kernel
// whose threads do one dependent chain of global loads (latency calibration).
#include <cstdio>
__global__ void k_empty() {}
__global__ void k_chain(const int* __restrict__ p, int steps, int* out) {
  int i = threadIdx.x;
  for (int s = 0; s < steps; ++s) i = p[i];
  if (i == -1) *out = i;
}
int main() {
  int *d, *o;
  cudaMalloc(&d, 1 << 20);
  cudaMalloc(&o, 4);
  cudaMemset(d, 0, 1 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(a);
    for (int k = 0; k < 1000; ++k) k_empty<<<148, 256>>>();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("empty kernel back-to-back: %.2f us\n", ms);
    for (int steps : {1, 10, 100}) {
      cudaEventRecord(a);
      for (int k = 0; k < 100; ++k) k_chain<<<148, 256>>>(d, steps, o);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("chain %3d dependent L2 loads: %.2f us per kernel\n", steps, ms * 10.0);
    }
  }
}
