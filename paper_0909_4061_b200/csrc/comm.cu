// NCCL collectives of the C ABI (SURVEY.md §8b lr_comm_init, §8e): a caller
// without torch.distributed (the reference's own Python, a C program) runs
// the row-sharded path through these entries -- the passes over its rows of
// A are local (lr_gemm), A^H Y partials are all-reduced with
// lr_comm_allreduce, and lr_orth_sharded orthonormalizes a row-sharded panel
// with its Grams all-reduced.  NCCL is resolved at run time (dlopen of
// libnccl.so.2: the process's already-loaded copy when torch is present), so
// the library has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "common.cuh"

namespace lr {
namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(lib, "ncclGetUniqueId"));
    api.comm_init_rank =
        reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(lib, "ncclCommInitRank"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(lib, "ncclAllReduce"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(lib, "ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(lib, "ncclGetErrorString"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.all_reduce && api.comm_destroy;
  });
  return api;
}

void check_nccl(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const char* msg = nccl().error_string ? nccl().error_string(r) : "error";
  throw Error{LR_ECUDA, std::string(what) + ": " + msg};
}

}  // namespace

void comm_allreduce_wide(Handle* h, int dtype_wide, int64_t count, void* buf) {
  if (!h->nccl_comm || h->nranks <= 1 || count == 0) return;
  const size_t n = size_t(count) * (dtype_wide == LR_C128 ? 2 : 1);   // complex: two doubles
  check_nccl(nccl().all_reduce(buf, buf, n, ncclFloat64, ncclSum,
                               static_cast<ncclComm_t>(h->nccl_comm), h->stream),
             "ncclAllReduce");
}

void comm_destroy(Handle* h) {
  if (h->nccl_comm && nccl().ok) nccl().comm_destroy(static_cast<ncclComm_t>(h->nccl_comm));
  h->nccl_comm = nullptr;
  h->nranks = 1;
  h->rank = 0;
}

void comm_unique_id(void* out) {
  LR_REQUIRE(nccl().ok, LR_EUNSUPPORTED, "lr_comm: libnccl.so.2 not found");
  ncclUniqueId id;
  check_nccl(nccl().get_unique_id(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == LR_COMM_ID_BYTES, "ncclUniqueId size");
  std::memcpy(out, &id, sizeof(id));
}

void comm_init(Handle* h, const void* id, int nranks, int rank) {
  LR_REQUIRE(nccl().ok, LR_EUNSUPPORTED, "lr_comm: libnccl.so.2 not found");
  LR_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, LR_EINVAL, "lr_comm_init: bad rank");
  comm_destroy(h);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  check_nccl(nccl().comm_init_rank(&c, nranks, uid, rank), "ncclCommInitRank");
  h->nccl_comm = c;
  h->nranks = nranks;
  h->rank = rank;
}

}  // namespace lr
