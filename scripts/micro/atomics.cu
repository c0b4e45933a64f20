// Microbenchmark: cost of warp-aggregated appends on one global counter vs
// block-aggregated appends (B200), n = 2M vertices, ~30% selected.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned lanemask_lt() { unsigned m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }
__global__ void k_warp(const int* parts, int n, int* list, unsigned long long* cnt) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < (n + 31) / 32 * 32; v += gridDim.x * blockDim.x) {
    bool take = v < n && parts[v] < 20;
    unsigned m = __ballot_sync(~0u, take);
    if (!m) continue;
    int leader = __ffs(m) - 1, lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(cnt, (unsigned long long)__popc(m));
    base = __shfl_sync(~0u, base, leader);
    if (take) list[base + __popc(m & lanemask_lt())] = v;
  }
}
__global__ void k_block(const int* parts, int n, int* list, unsigned long long* cnt) {
  __shared__ unsigned s_cnt; __shared__ unsigned long long s_base;
  for (int b0 = blockIdx.x * blockDim.x; b0 < n; b0 += gridDim.x * blockDim.x) {
    int v = b0 + threadIdx.x;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    bool take = v < n && parts[v] < 20;
    unsigned m = __ballot_sync(~0u, take);
    int leader = __ffs(m) - 1, lane = threadIdx.x & 31;
    unsigned off = 0;
    if (m && lane == leader) off = atomicAdd(&s_cnt, __popc(m));
    off = __shfl_sync(~0u, off, leader < 0 ? 0 : leader);
    __syncthreads();
    if (threadIdx.x == 0) s_base = atomicAdd(cnt, (unsigned long long)s_cnt);
    __syncthreads();
    if (take) list[s_base + off + __popc(m & lanemask_lt())] = v;
  }
}
__global__ void k_red_hot(const int* parts, int n, unsigned long long* H) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if (parts[v] < 20) atomicAdd(&H[parts[v] % 4], 1ull);
}
__global__ void k_red_agg(const int* parts, int n, unsigned long long* H) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < (n + 31) / 32 * 32; v += gridDim.x * blockDim.x) {
    int key = (v < n && parts[v] < 20) ? parts[v] % 4 : -1;
    unsigned peers = __match_any_sync(~0u, key);
    if (key >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&H[key], (unsigned long long)__popc(peers));
  }
}
int main() {
  const int n = 1 << 21;
  int *parts, *list; unsigned long long *cnt, *H;
  cudaMalloc(&parts, n * 4); cudaMalloc(&list, n * 4); cudaMalloc(&cnt, 8); cudaMalloc(&H, 64);
  int* h = new int[n];
  for (int i = 0; i < n; ++i) h[i] = (i / 32768) ;  // 64 parts of contiguous vertices
  cudaMemcpy(parts, h, n * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int grids[] = {148, 296, 592, 1184};
  for (int gi = 0; gi < 4; ++gi) {
    int G = grids[gi]; float ms;
    for (int r = 0; r < 3; ++r) {
      cudaMemset(cnt, 0, 8); cudaEventRecord(a); k_warp<<<G, 512>>>(parts, n, list, cnt); cudaEventRecord(b); cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b); printf("grid %4d warp-append  %8.1f us\n", G, ms * 1e3);
    for (int r = 0; r < 3; ++r) {
      cudaMemset(cnt, 0, 8); cudaEventRecord(a); k_block<<<G, 512>>>(parts, n, list, cnt); cudaEventRecord(b); cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b); printf("grid %4d block-append %8.1f us\n", G, ms * 1e3);
    for (int r = 0; r < 3; ++r) { cudaEventRecord(a); k_red_hot<<<G, 512>>>(parts, n, H); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&ms, a, b); printf("grid %4d red-hot      %8.1f us\n", G, ms * 1e3);
    for (int r = 0; r < 3; ++r) { cudaEventRecord(a); k_red_agg<<<G, 512>>>(parts, n, H); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&ms, a, b); printf("grid %4d red-agg      %8.1f us\n", G, ms * 1e3);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
