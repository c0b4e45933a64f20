// Microbenchmark: cooperative grid.sync() cost vs grid size (B200).
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void k_sync(int iters, int* x) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) { if (threadIdx.x == 0 && blockIdx.x == i % gridDim.x) x[0] += 1; g.sync(); }
}
int main() {
  int* x; cudaMalloc(&x, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int grids[] = {1, 8, 37, 148, 296};
  for (int bs : {256, 512}) for (int G : grids) {
    int iters = 2000; void* args[] = {&iters, &x}; float ms;
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_sync, G, bs, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    printf("block %d grid %4d: %.2f us per grid.sync\n", bs, G, ms * 1e3 / iters);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
