// Microbenchmark: cooperative grid.sync() vs a release/acquire counter barrier
// (bar.sync; thread 0: atom.add.release.gpu + ld.acquire.gpu spin; bar.sync).
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ void ra_sync(unsigned* arrived) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned nb = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
    unsigned old, cur;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(arrived), "r"(nb) : "memory");
    do {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(arrived) : "memory");
    } while (((old ^ cur) & 0x80000000u) == 0);
  }
  __syncthreads();
}
__global__ void k_cg(int iters, int* x, unsigned*) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) { if (threadIdx.x == 0 && blockIdx.x == i % gridDim.x) x[0] += 1; g.sync(); }
}
__global__ void k_ra(int iters, int* x, unsigned* bar) {
  for (int i = 0; i < iters; ++i) { if (threadIdx.x == 0 && blockIdx.x == i % gridDim.x) x[0] += 1; ra_sync(bar); }
}
// correctness: every block adds its id to slot i, after the barrier every block checks the sum
__global__ void k_check(int iters, int* x, unsigned* bar, int* bad) {
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) atomicAdd(&x[i & 1], 1);
    ra_sync(bar);
    if (threadIdx.x == 0 && *(volatile int*)&x[i & 1] != gridDim.x * (i / 2 + 1)) atomicAdd(bad, 1);
    ra_sync(bar);
  }
}
int main() {
  int* x; unsigned* bar; int* bad;
  cudaMalloc(&x, 64); cudaMalloc(&bar, 4); cudaMalloc(&bad, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int grids[] = {2, 17, 148, 296};
  for (int v = 0; v < 2; ++v)
  for (int G : grids) {
    int iters = 4000; void* args[] = {&iters, &x, &bar}; float ms;
    cudaMemset(bar, 0, 4);
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel(v ? (void*)k_ra : (void*)k_cg, G, 512, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    printf("%s grid %4d: %.3f us per barrier\n", v ? "rel/acq" : "cg     ", G, ms * 1e3 / iters);
  }
  cudaMemset(x, 0, 64); cudaMemset(bar, 0, 4); cudaMemset(bad, 0, 4);
  int iters = 2000, G = 296; void* args2[] = {&iters, &x, &bar, &bad};
  cudaLaunchCooperativeKernel((void*)k_check, G, 512, args2, 0, 0);
  int hb = -1; cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  printf("check bad=%d err %s\n", hb, cudaGetErrorString(cudaGetLastError()));
}
