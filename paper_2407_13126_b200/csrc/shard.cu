// Multi-GPU sharding through the C ABI, so C++ callers of
// the reference-facing API reach NCCL without Python: one process per GPU,
// one NCCL communicator per context, collectives on the context's stream.
//
//   mgs_nccl_unique_id / mgs_shard_init   ncclGetUniqueId / ncclCommInitRank
//   mgs_shard_attach                      use a caller's ncclComm_t
//   mgs_shard_allgather_i64               per-shard result rows -> every rank
//   mgs_shard_best                        per-shard best (objective, owner):
//                                         all-reduce(max) of the order-preserving
//                                         objective bits, then all-reduce(min)
//                                         of the owner among the maxima
//   mgs_solve_batch_sharded               windows [n*r/N, n*(r+1)/N) on rank r
//                                         (mgs_solve_batch), then an all-gather
//                                         of (status, objective, plan) rows
//
// NCCL is loaded with dlopen (libnccl.so.2, the same library the process may
// already hold through another framework), so the planner library itself has
// no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <functional>
#include <mutex>
#include <vector>

#include "ctx.cuh"


namespace mgs {
namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_gather && api.all_reduce &&
             api.error_string;
  });
  if (!api.ok) throw PlanFail{MGS_ERR_CUDA, "NCCL (libnccl.so.2) is not available"};
  return api;
}

void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw PlanFail{MGS_ERR_CUDA, std::string(what) + ": " + nccl().error_string(r)};
}

ncclComm_t comm_of(Ctx& c) {
  if (!c.nccl_comm) throw PlanFail{MGS_ERR_ARGUMENT, "no communicator: call mgs_shard_init or mgs_shard_attach"};
  return static_cast<ncclComm_t>(c.nccl_comm);
}

// all-gather of n int64 per rank (host in, host out), on the context's stream
void allgather_i64(Ctx& c, const int64_t* send, int64_t n, int64_t* recv) {
  int64_t* d_send = c.buf<int64_t>("sh_send", std::max<int64_t>(1, n));
  int64_t* d_recv = c.buf<int64_t>("sh_recv", std::max<int64_t>(1, n * c.world));
  MGS_CUDA_OK(cudaMemcpyAsync(d_send, send, n * 8, cudaMemcpyHostToDevice, c.stream));
  nccl_ok(nccl().all_gather(d_send, d_recv, static_cast<size_t>(n), ncclInt64, comm_of(c), c.stream), "ncclAllGather");
  MGS_CUDA_OK(cudaMemcpyAsync(recv, d_recv, n * c.world * 8, cudaMemcpyDeviceToHost, c.stream));
  MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
}

int64_t allreduce_i64(Ctx& c, int64_t v, ncclRedOp_t op) {
  int64_t* d = c.buf<int64_t>("sh_red", 1);
  MGS_CUDA_OK(cudaMemcpyAsync(d, &v, 8, cudaMemcpyHostToDevice, c.stream));
  nccl_ok(nccl().all_reduce(d, d, 1, ncclInt64, op, comm_of(c), c.stream), "ncclAllReduce");
  int64_t out = 0;
  MGS_CUDA_OK(cudaMemcpyAsync(&out, d, 8, cudaMemcpyDeviceToHost, c.stream));
  MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
  return out;
}

}  // namespace

void shard_release(Ctx& c) {
  if (c.nccl_comm && c.own_comm) nccl().comm_destroy(static_cast<ncclComm_t>(c.nccl_comm));
  c.nccl_comm = nullptr;
}

}  // namespace mgs

using mgs::Ctx;
using mgs::PlanFail;

int mgs_guarded_call(mgs_error* err, const std::function<void()>& f);

extern "C" {

int mgs_nccl_unique_id(uint8_t* id) {
  if (!id) return MGS_ERR_ARGUMENT;
  return mgs_guarded_call(nullptr, [&] {
    ncclUniqueId u;
    mgs::nccl_ok(mgs::nccl().get_unique_id(&u), "ncclGetUniqueId");
    static_assert(sizeof(u.internal) == MGS_NCCL_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id, u.internal, MGS_NCCL_ID_BYTES);
  });
}

int mgs_shard_init(mgs_ctx* ctx, int32_t world, int32_t rank, const uint8_t* id, mgs_error* err) {
  if (!ctx || world < 1 || rank < 0 || rank >= world || !id) return MGS_ERR_ARGUMENT;
  return mgs_guarded_call(err, [&] {
    Ctx& c = ctx->c;
    MGS_CUDA_OK(cudaSetDevice(c.device));
    mgs::shard_release(c);
    ncclUniqueId u;
    std::memcpy(u.internal, id, MGS_NCCL_ID_BYTES);
    ncclComm_t comm = nullptr;
    mgs::nccl_ok(mgs::nccl().comm_init_rank(&comm, world, u, rank), "ncclCommInitRank");
    c.nccl_comm = comm;
    c.own_comm = true;
    c.world = world;
    c.rank = rank;
  });
}

int mgs_shard_attach(mgs_ctx* ctx, void* nccl_comm, int32_t world, int32_t rank) {
  if (!ctx || !nccl_comm || world < 1 || rank < 0 || rank >= world) return MGS_ERR_ARGUMENT;
  return mgs_guarded_call(nullptr, [&] {
    Ctx& c = ctx->c;
    mgs::shard_release(c);
    c.nccl_comm = nccl_comm;
    c.own_comm = false;
    c.world = world;
    c.rank = rank;
  });
}

int mgs_shard_allgather_i64(mgs_ctx* ctx, const int64_t* send, int64_t n, int64_t* recv, mgs_error* err) {
  if (!ctx || n < 0 || (n > 0 && (!send || !recv))) return MGS_ERR_ARGUMENT;
  return mgs_guarded_call(err, [&] {
    Ctx& c = ctx->c;
    MGS_CUDA_OK(cudaSetDevice(c.device));
    mgs::allgather_i64(c, send, n, recv);
  });
}

int mgs_shard_best(mgs_ctx* ctx, double objective, double* best, int32_t* owner, mgs_error* err) {
  if (!ctx || !best || !owner || !(objective >= 0.0)) return MGS_ERR_ARGUMENT;
  return mgs_guarded_call(err, [&] {
    Ctx& c = ctx->c;
    MGS_CUDA_OK(cudaSetDevice(c.device));
    int64_t key = 0;  // non-negative doubles order like their bit patterns
    std::memcpy(&key, &objective, 8);
    const int64_t top = mgs::allreduce_i64(c, key, ncclMax);
    const int64_t who = mgs::allreduce_i64(c, key == top ? c.rank : c.world, ncclMin);
    std::memcpy(best, &top, 8);
    *owner = static_cast<int32_t>(who);
  });
}

int mgs_solve_batch_sharded(mgs_ctx* ctx, const mgs_problem* problems, int32_t n, int32_t s_max, int32_t* out_option,
                            double* out_objective, int32_t* status, mgs_error* err) {
  if (!ctx || n < 0 || s_max < 1 || (n > 0 && (!problems || !out_option || !out_objective || !status)))
    return MGS_ERR_ARGUMENT;
  return mgs_guarded_call(err, [&] {
    Ctx& c = ctx->c;
    MGS_CUDA_OK(cudaSetDevice(c.device));
    const int world = c.nccl_comm ? c.world : 1, rank = c.nccl_comm ? c.rank : 0;
    const int lo = static_cast<int>(static_cast<int64_t>(n) * rank / world);
    const int hi = static_cast<int>(static_cast<int64_t>(n) * (rank + 1) / world);
    const int per = (n + world - 1) / world;  // rows per rank in the gather (padded)
    const int width = 2 + s_max;              // status, objective bits, options
    std::vector<int32_t> opt(static_cast<size_t>(std::max(1, hi - lo)) * s_max, -1);
    std::vector<double> obj(std::max(1, hi - lo), 0.0);
    std::vector<int32_t> st(std::max(1, hi - lo), MGS_ERR_CUDA);
    if (hi > lo) {
      const int rc = mgs_solve_batch(ctx, problems + lo, hi - lo, s_max, opt.data(), obj.data(), st.data(), nullptr,
                                     nullptr);
      if (rc != MGS_OK) throw PlanFail{rc, "mgs_solve_batch failed on this shard"};
    }
    std::vector<int64_t> rows(static_cast<size_t>(per) * width, -1), all(static_cast<size_t>(per) * width * world);
    for (int i = 0; i < hi - lo; ++i) {
      int64_t* r = rows.data() + static_cast<size_t>(i) * width;
      r[0] = st[i];
      std::memcpy(&r[1], &obj[i], 8);
      for (int s = 0; s < s_max; ++s) r[2 + s] = opt[static_cast<size_t>(i) * s_max + s];
    }
    if (world > 1) {
      mgs::allgather_i64(c, rows.data(), static_cast<int64_t>(rows.size()), all.data());
    } else {
      all = rows;
    }
    for (int q = 0; q < world; ++q) {
      const int qlo = static_cast<int>(static_cast<int64_t>(n) * q / world);
      const int qhi = static_cast<int>(static_cast<int64_t>(n) * (q + 1) / world);
      for (int i = qlo; i < qhi; ++i) {
        const int64_t* r = all.data() + (static_cast<size_t>(q) * per + (i - qlo)) * width;
        status[i] = static_cast<int32_t>(r[0]);
        std::memcpy(&out_objective[i], &r[1], 8);
        for (int s = 0; s < s_max; ++s) out_option[static_cast<size_t>(i) * s_max + s] = static_cast<int32_t>(r[2 + s]);
      }
    }
  });
}

}  // extern "C"
