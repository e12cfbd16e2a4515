// Device-wide exclusive scans with the total appended (out[n] = sum), for the
// one-time-per-window passes (option enumeration, candidate compaction, the
// multi-launch engine). Reduce-then-scan in three launches:
//   k_tile_sums   per tile of kScanTile elements: its sum (block reduction)
//   k_scan_sums   one CTA: exclusive scan of the tile sums, the total at out[n]
//   k_tile_scan   per tile: block-wide exclusive scan + the tile's offset
// Tiles are 8 elements per thread, loaded as contiguous runs per thread.
#include "ctx.cuh"

namespace mgs {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

// exclusive block scan of one value per thread; *total gets the block sum
template <class T>
__device__ T block_exclusive(T x, T* total) {
  __shared__ T warp_sums[kScanThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) warp_sums[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < kScanThreads / 32 ? warp_sums[lane] : T(0);
    T wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < kScanThreads / 32) warp_sums[lane] = wi - w;  // exclusive warp offsets
    if (lane == kScanThreads / 32 - 1) *total = wi;
  }
  __syncthreads();
  const T out = warp_sums[warp] + inc - x;
  __syncthreads();  // warp_sums is reused by the next call
  return out;
}

template <class T>
__global__ void __launch_bounds__(kScanThreads) k_tile_sums(const T* in, int n, T* sums) {
  __shared__ T total;
  const long long base = static_cast<long long>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
  T x = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (base + k < n) x += in[base + k];
  block_exclusive(x, &total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

template <class T>
__global__ void __launch_bounds__(kScanThreads) k_scan_sums(T* sums, int tiles, T* out_total) {
  __shared__ T total;
  T carry = 0;
  for (int t0 = 0; t0 < tiles; t0 += kScanThreads) {  // one CTA, kScanThreads tiles per round
    const int t = t0 + threadIdx.x;
    const T x = t < tiles ? sums[t] : T(0);
    const T ex = block_exclusive(x, &total);
    if (t < tiles) sums[t] = carry + ex;
    carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *out_total = carry;
}

template <class T>
__global__ void __launch_bounds__(kScanThreads) k_tile_scan(const T* in, int n, const T* offsets, T* out) {
  __shared__ T total;
  const long long base = static_cast<long long>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
  T v[kScanItems];
  T x = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = base + k < n ? in[base + k] : T(0);
    x += v[k];
  }
  T run = block_exclusive(x, &total) + offsets[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (base + k < n) {
      out[base + k] = run;
      run += v[k];
    }
}

template <class T>
void scan_impl(Ctx& c, const T* in, T* out, int n) {
  if (n <= 0) {
    MGS_CUDA_OK(cudaMemsetAsync(out, 0, sizeof(T), c.stream));
    return;
  }
  const int tiles = (n + kScanTile - 1) / kScanTile;
  T* sums = c.buf<T>(sizeof(T) == 4 ? "scan_tile_sums4" : "scan_tile_sums8", tiles);
  k_tile_sums<T><<<tiles, kScanThreads, 0, c.stream>>>(in, n, sums);
  k_scan_sums<T><<<1, kScanThreads, 0, c.stream>>>(sums, tiles, out + n);
  k_tile_scan<T><<<tiles, kScanThreads, 0, c.stream>>>(in, n, sums, out);
  c.kernel_launches += 3;
  MGS_CUDA_OK(cudaGetLastError());
}

}  // namespace

void exclusive_scan_i32(Ctx& c, const int32_t* in, int32_t* out, int n) { scan_impl(c, in, out, n); }
void exclusive_scan_u32(Ctx& c, const uint32_t* in, uint32_t* out, int n) { scan_impl(c, in, out, n); }

}  // namespace mgs
