// Device-wide exclusive scans with the total appended (out[n] = sum).
#include <cub/cub.cuh>

#include "ctx.cuh"

namespace mgs {

template <class T>
static void scan_impl(Ctx& c, const T* in, T* out, int n) {
  MGS_CUDA_OK(cudaMemsetAsync(out, 0, sizeof(T), c.stream));
  if (n <= 0) return;
  size_t tb = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb, in, out + 1, n, c.stream);
  void* tmp = c.buf<char>("cub_scan_tmp", tb);
  MGS_CUDA_OK(cub::DeviceScan::InclusiveSum(tmp, tb, in, out + 1, n, c.stream));
}

void exclusive_scan_i32(Ctx& c, const int32_t* in, int32_t* out, int n) { scan_impl(c, in, out, n); }
void exclusive_scan_u32(Ctx& c, const uint32_t* in, uint32_t* out, int n) { scan_impl(c, in, out, n); }

}  // namespace mgs
