// Pre-initialisation (plan_preinit + apply_preinit, preinit.hpp:41-114) for a
// batch of plans: an instance that step s+1 needs and step s does not have is
// created early during s when its slices are unused at s; a tenant whose every
// newly acquired inference instance at s+1 was pre-created that way pays no
// reconfiguration overhead there (its psi_eff override is 0).
//
// In option terms (identity of an instance = its (slice_start, size) range =
// its universe id, catalog.hpp:233-240):
//   A[o] = universe mask of every slot the option assigns (any task)
//   O[o] = slices held by those slots (occupied_slices, preinit.hpp:26-31)
//   pre-created during s = A[o_{s+1}] & ~A[o_s], keeping ranges whose slices
//                          do not meet O[o_s]
//   override(m, s+1)     = acquired = mask_m(o_{s+1}) & ~mask_m(o_s) is non-empty
//                          and inside pre-created(s)
// Everything at (plan, step, tenant) is independent: one thread each.
#include "ctx.cuh"

namespace mgs {
namespace {

// A[o] and O[o] from each option's configuration and labels
__global__ void k_opt_masks(DevSpace sp, const int32_t* slot_offset, const int32_t* slot_uid,
                            const uint32_t* slot_range, uint32_t* A, uint32_t* O) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < sp.n_opt; o += gridDim.x * blockDim.x) {
    const int cfg = sp.opt_config[o], b = slot_offset[cfg], n = slot_offset[cfg + 1] - b;
    uint32_t a = 0, occ = 0;
    for (int k = 0; k < n; ++k)
      if (sp.opt_labels[static_cast<size_t>(o) * MGS_MAX_SLOTS + k] != 0) {
        a |= 1u << slot_uid[b + k];
        occ |= slot_range[b + k];
      }
    A[o] = a;
    O[o] = occ;
  }
}

// pre-created universe mask fired during step s (0 for the last step)
__device__ __forceinline__ uint32_t precreated(const uint32_t* A, const uint32_t* O, const uint32_t* uni_range,
                                               int cur, int nxt) {
  uint32_t created = A[nxt] & ~A[cur], out = 0;
  while (created) {
    const int u = __ffs(created) - 1;
    created &= created - 1;
    if ((uni_range[u] & O[cur]) == 0) out |= 1u << u;  // only unused slices are touched
  }
  return out;
}

__global__ void k_preinit(DevSpace sp, int M, int S, const int32_t* plans, int n_plans, const uint32_t* A,
                          const uint32_t* O, const uint32_t* uni_range, uint8_t* overrides, uint32_t* fired) {
  const long long n = static_cast<long long>(n_plans) * S;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int s = static_cast<int>(i % S);
    const int32_t* plan = plans + (i / S) * S;
    if (fired) fired[i] = s + 1 < S ? precreated(A, O, uni_range, plan[s], plan[s + 1]) : 0u;
    const uint32_t pc = s > 0 ? precreated(A, O, uni_range, plan[s - 1], plan[s]) : 0u;
    for (int m = 0; m < M; ++m) {
      bool ov = false;
      if (pc) {
        const uint32_t before = s > 0 ? sp.opt_mask[plan[s - 1] * KM + m] : 0u;
        const uint32_t after = sp.opt_mask[plan[s] * KM + m];
        const uint32_t acquired = after & ~before;
        ov = acquired != 0 && (acquired & ~pc) == 0;
      }
      overrides[i * M + m] = ov ? 1 : 0;
    }
  }
}

}  // namespace

void preinit_overrides(Ctx& c, const Prepared& pr, const DevSpace& sp, const mgs_lattice& lat, const int32_t* d_plans,
                       int n_plans, uint8_t* d_overrides, uint32_t* d_fired) {
  const int M = pr.t.M, S = pr.t.S;
  const int nslots = lat.slot_offset[lat.n_configs];
  std::vector<uint32_t> slot_range(nslots), uni_range(32, 0);
  for (int i = 0; i < nslots; ++i) {
    uint32_t r = 0;
    for (int b = 0; b < lat.slot_size[i]; ++b) r |= 1u << (lat.slot_start[i] + b);  // range_mask (preinit.hpp:32-36)
    slot_range[i] = r;
    uni_range[pr.slot_uid[i]] = r;
  }
  int32_t* d_off = c.buf<int32_t>("pi_off", lat.n_configs + 1);
  int32_t* d_uid = c.buf<int32_t>("pi_uid", nslots);
  uint32_t* d_srange = c.buf<uint32_t>("pi_srange", nslots);
  uint32_t* d_urange = c.buf<uint32_t>("pi_urange", 32);
  uint32_t* A = c.buf<uint32_t>("pi_A", sp.n_opt);
  uint32_t* O = c.buf<uint32_t>("pi_O", sp.n_opt);
  MGS_CUDA_OK(cudaMemcpyAsync(d_off, lat.slot_offset, (lat.n_configs + 1) * 4, cudaMemcpyHostToDevice, c.stream));
  MGS_CUDA_OK(cudaMemcpyAsync(d_uid, pr.slot_uid.data(), nslots * 4, cudaMemcpyHostToDevice, c.stream));
  MGS_CUDA_OK(cudaMemcpyAsync(d_srange, slot_range.data(), nslots * 4, cudaMemcpyHostToDevice, c.stream));
  MGS_CUDA_OK(cudaMemcpyAsync(d_urange, uni_range.data(), 32 * 4, cudaMemcpyHostToDevice, c.stream));
  k_opt_masks<<<ceil_div(sp.n_opt, 256), 256, 0, c.stream>>>(sp, d_off, d_uid, d_srange, A, O);
  const long long n = static_cast<long long>(n_plans) * S;
  if (n > 0) k_preinit<<<ceil_div(n, 256), 256, 0, c.stream>>>(sp, M, S, d_plans, n_plans, A, O, d_urange, d_overrides, d_fired);
  c.kernel_launches += 2;
  MGS_CUDA_OK(cudaGetLastError());
  MGS_CUDA_OK(cudaStreamSynchronize(c.stream));  // host staging vectors above are freed on return
}

}  // namespace mgs
