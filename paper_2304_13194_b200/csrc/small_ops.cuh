// small_ops.cuh — one-block forms of the scans, selects and key sorts that the
// coarsening runs once per level. On the small levels (the last ~12 of a
// mesh hierarchy) a library device-wide call is two to six launches of
// near-empty grids (8-46 us per call, measured); one block does the same
// work in a single short launch. Results are identical to the library calls
// (exclusive sums; selects keep ascending index order; sorts are full key
// sorts), so the callers fall back to CUB only above the size limits.
#pragma once
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>
#include "common.cuh"

namespace jet {

constexpr int SMALL_BT = 1024, SMALL_IPT = 16;
constexpr int64_t SMALL_SCAN_MAX = (int64_t)SMALL_BT * SMALL_IPT;  // items per one-block select
constexpr int SORT_BT = 512, SORT_IPT = 8;
constexpr int64_t SMALL_SORT_MAX = (int64_t)SORT_BT * SORT_IPT;    // keys per one-block sort

// 64-bit sums keep 8 items per thread in registers (16 spill at 1024 threads)
template <class T>
constexpr int scan_ipt() { return sizeof(T) > 4 ? SMALL_IPT / 2 : SMALL_IPT; }

template <class T>
__global__ void __launch_bounds__(SMALL_BT, 1) k_small_exclusive_sum(const T* __restrict__ in,
                                                                  T* __restrict__ out, int n) {
  constexpr int IPT = scan_ipt<T>();
  typedef cub::BlockScan<T, SMALL_BT, cub::BLOCK_SCAN_WARP_SCANS> BS;
  __shared__ typename BS::TempStorage ts;
  const int b = threadIdx.x * IPT;
  T v[IPT];
  T run = 0;
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    v[q] = b + q < n ? in[b + q] : T(0);
    run += v[q];
  }
  T pre;
  BS(ts).ExclusiveSum(run, pre);
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    if (b + q < n) out[b + q] = pre;
    pre += v[q];
  }
}

// out[i] = sum of in[0..i) for i < n; false when n is beyond one block.
template <class T>
bool small_exclusive_sum(Ctx& c, const char* name, const T* in, T* out, int64_t n) {
  if (n > (int64_t)SMALL_BT * scan_ipt<T>()) return false;
  if (n <= 0) return true;
  launch(c, name, 2.0 * sizeof(T) * n, [&] {
    k_small_exclusive_sum<T><<<1, SMALL_BT, 0, c.stream>>>(in, out, (int)n);
  });
  return true;
}

// Indices i in [0, n) with pred(i), ascending, and their count.
template <class Pred, class Cnt>
__global__ void __launch_bounds__(SMALL_BT, 1) k_small_select(Pred pred, int n, int32_t* __restrict__ out,
                                                           Cnt* count) {
  typedef cub::BlockScan<int, SMALL_BT> BS;
  __shared__ typename BS::TempStorage ts;
  const int b = threadIdx.x * SMALL_IPT;
  unsigned m = 0;
  int k = 0;
#pragma unroll
  for (int q = 0; q < SMALL_IPT; ++q)
    if (b + q < n && pred((int32_t)(b + q))) {
      m |= 1u << q;
      ++k;
    }
  int pre, tot;
  BS(ts).ExclusiveSum(k, pre, tot);
#pragma unroll
  for (int q = 0; q < SMALL_IPT; ++q)
    if (m >> q & 1u) out[pre++] = b + q;
  if (threadIdx.x == 0) *count = (Cnt)tot;
}

template <class Pred, class Cnt>
bool small_select(Ctx& c, const char* name, Pred pred, int64_t n, int32_t* out, Cnt* count) {
  if (n > SMALL_SCAN_MAX || n <= 0) return false;
  launch(c, name, 8.0 * n, [&] {
    k_small_select<Pred, Cnt><<<1, SMALL_BT, 0, c.stream>>>(pred, (int)n, out, count);
  });
  return true;
}

// Ascending sort of n 64-bit keys over bits [0, end_bit).
static __global__ void __launch_bounds__(SORT_BT, 1) k_small_sort_keys(const unsigned long long* __restrict__ in,
                                                             unsigned long long* __restrict__ out,
                                                             int n, int end_bit) {
  typedef cub::BlockRadixSort<unsigned long long, SORT_BT, SORT_IPT> BRS;
  __shared__ typename BRS::TempStorage ts;
  unsigned long long k[SORT_IPT];
#pragma unroll
  for (int q = 0; q < SORT_IPT; ++q) {
    const int i = threadIdx.x * SORT_IPT + q;  // blocked arrangement
    k[q] = i < n ? in[i] : ~0ull;
  }
  BRS(ts).Sort(k, 0, end_bit);
#pragma unroll
  for (int q = 0; q < SORT_IPT; ++q) {
    const int i = threadIdx.x * SORT_IPT + q;
    if (i < n) out[i] = k[q];
  }
}

inline bool small_sort_keys(Ctx& c, const char* name, const unsigned long long* in,
                            unsigned long long* out, int64_t n, int end_bit) {
  if (n > SMALL_SORT_MAX || n <= 0) return false;
  launch(c, name, 16.0 * n, [&] {
    k_small_sort_keys<<<1, SORT_BT, 0, c.stream>>>(in, out, (int)n, end_bit);
  });
  return true;
}

}  // namespace jet
