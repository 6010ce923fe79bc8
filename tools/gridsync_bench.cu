// microbenchmark: cost of cooperative_groups grid.sync() on this GPU
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, int* out) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; i++) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = iters;
}
int main() {
  int* out; cudaMalloc(&out, 4);
  for (int G : {16, 64, 128, 148}) for (int T : {256, 512}) {
    int iters = 2000;
    void* args[] = {&iters, &out};
    cudaLaunchCooperativeKernel((void*)k, G, T, args, 0, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k, G, T, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("G=%d T=%d: %.2f us per grid.sync (%s)\n", G, T, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
