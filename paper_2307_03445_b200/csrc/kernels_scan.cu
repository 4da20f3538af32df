// kernels_scan.cu — exclusive prefix sum of int32 counts (bin offsets, contact-row offsets).
//
// Three passes: (1) each 1024-thread block scans a tile of 4096 counts with warp
// shuffles and writes the tile total, (2) one block scans the tile totals, (3) tiles add
// their offset.  out[n] receives the grand total.  Totals are < 2^31 by construction
// (capacities are checked against them on the device).
#include "dem_device.cuh"

namespace dem {

#ifndef DEM_SCAN_V4
#define DEM_SCAN_V4 1  // 16-byte loads and stores of whole 4-count groups (the arrays are 256-byte aligned)
#endif
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// block-wide exclusive scan of one value per thread; returns the block total in *total
__device__ __forceinline__ int block_excl_scan(int v, int* total) {
  __shared__ int warp_sums[32];
  __shared__ int block_total;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = warp_incl_scan(v);
  if (lane == 31) warp_sums[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int s = lane < (blockDim.x >> 5) ? warp_sums[lane] : 0;
    int si = warp_incl_scan(s);
    warp_sums[lane] = si - s;
    if (lane == 31) block_total = si;
  }
  __syncthreads();
  int res = incl - v + warp_sums[wid];
  if (total) *total = block_total;
  __syncthreads();
  return res;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(const int* __restrict__ in, int* __restrict__ out,
                                                             int* __restrict__ tile_sums, long long n,
                                                             const int* abort, const int* abort2, int packed) {
  pdl_wait_and_release();
  if ((abort && *abort) || (abort2 && *abort2)) return;
  const long long base = (long long)blockIdx.x * kScanTile + (long long)threadIdx.x * kScanItems;
  int v[kScanItems];
  int s = 0;
  const bool whole = DEM_SCAN_V4 && base + kScanItems <= n;  // one 16-byte load / store per thread
  if (whole) {
    const int4 q = *reinterpret_cast<const int4*>(in + base);
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  }
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (!whole) v[k] = (base + k < n) ? in[base + k] : 0;
    if (packed) v[k] = (v[k] & 0xffff) + ((unsigned)v[k] >> 16);  // bin counts: small + large inserts
    s += v[k];
  }
  int total;
  int off = block_excl_scan(s, &total);
  if (whole) {
    int4 q;
    q.x = off; q.y = off + v[0]; q.z = q.y + v[1]; q.w = q.z + v[2];
    *reinterpret_cast<int4*>(out + base) = q;
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      if (base + k < n) out[base + k] = off;
      off += v[k];
    }
  }
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_sums(int* tile_sums, int n_tiles, int* out_total,
                                                            const int* abort, const int* abort2) {
  pdl_wait_and_release();
  if ((abort && *abort) || (abort2 && *abort2)) return;
  int carry = 0;
  for (int b = 0; b < n_tiles; b += kScanThreads) {
    int i = b + threadIdx.x;
    int v = i < n_tiles ? tile_sums[i] : 0;
    int total;
    int ex = block_excl_scan(v, &total);
    if (i < n_tiles) tile_sums[i] = ex + carry;
    carry += total;
  }
  if (threadIdx.x == 0) *out_total = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_add(int* out, const int* tile_sums, long long n,
                                                           const int* abort, const int* abort2) {
  pdl_wait_and_release();
  if ((abort && *abort) || (abort2 && *abort2)) return;
  const int add = tile_sums[blockIdx.x];
  if (add == 0) return;
  const long long base = (long long)blockIdx.x * kScanTile;
  if (DEM_SCAN_V4 && base + kScanTile <= n) {
    int4* o = reinterpret_cast<int4*>(out + base);
    for (int k = threadIdx.x; k < kScanTile / 4; k += kScanThreads) {
      int4 q = o[k];
      q.x += add; q.y += add; q.z += add; q.w += add;
      o[k] = q;
    }
    return;
  }
  for (int k = threadIdx.x; k < kScanTile; k += kScanThreads)
    if (base + k < n) out[base + k] += add;
}

long long scan_tiles_needed(long long n) { return (n + kScanTile - 1) / kScanTile; }

// out must hold n + 1 ints; tmp must hold scan_tiles_needed(n) ints
void launch_excl_scan(const int* in, int* out, long long n, int* tmp, const int* abort, cudaStream_t s,
                      const int* abort2, int packed, bool pdl) {
  long long tiles = scan_tiles_needed(n);
  if (tiles == 0) {
    cudaMemsetAsync(out, 0, sizeof(int), s);
    return;
  }
  launch_k(k_scan_tiles, (unsigned)tiles, kScanThreads, s, pdl, in, out, tmp, n, abort, abort2, packed);
  launch_k(k_scan_sums, 1, kScanThreads, s, pdl, tmp, (int)tiles, out + n, abort, abort2);
  launch_k(k_scan_add, (unsigned)tiles, kScanThreads, s, pdl, out, tmp, n, abort, abort2);
}

}  // namespace dem
