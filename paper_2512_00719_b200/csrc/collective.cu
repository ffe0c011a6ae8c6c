// collective.cu — the token-id all-gather of the batch-sharded path
// (SURVEY §8(b) dp_allgather_tokens; reference: partition_batch + the
// DecisionLedger collection, transport.py:133-144, :400-433, service.py:743-748).
//
// The only cross-GPU exchange of the decision plane is one ncclAllGather of
// the int32 token ids per iteration (rows never cross GPUs, no vocab-axis
// collective).  NCCL is resolved at run time with dlopen: inside a PyTorch
// process the libnccl.so.2 torch already loaded is reused (RTLD_NOLOAD), so
// the library never drags a second NCCL into the process; elsewhere the
// system libnccl.so.2 is opened.  (A process that will import torch must do
// so before the first collective call — _native.load() imports torch first —
// or the system copy would shadow torch's.)  Nothing here links NCCL at
// build time.
#include <dlfcn.h>

#include <cstdio>
#include <cstring>
#include <mutex>

#include "decplane_b200.h"

namespace dp {
int set_last_error(int code, const char* msg);   // capi.cu
}

namespace {

// the subset of nccl.h this file needs (ABI-stable since NCCL 2.0)
typedef struct ncclComm* nccl_comm_t;
typedef struct { char internal[128]; } nccl_unique_id_t;
constexpr int kNcclInt32 = 2;   // ncclInt32
constexpr int kNcclSuccess = 0;

struct Nccl {
  void* so = nullptr;
  int (*get_unique_id)(nccl_unique_id_t*) = nullptr;
  int (*comm_init_rank)(nccl_comm_t*, int, nccl_unique_id_t, int) = nullptr;
  int (*comm_destroy)(nccl_comm_t) = nullptr;
  int (*all_gather)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(int) = nullptr;
};

Nccl g_nccl;
std::once_flag g_once;

const Nccl* nccl() {
  std::call_once(g_once, [] {
    void* so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // the copy the process already has
    if (!so) so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!so) so = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!so) return;
    Nccl n;
    n.so = so;
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(so, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(so, "ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(so, "ncclCommDestroy"));
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(dlsym(so, "ncclAllGather"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(so, "ncclGetErrorString"));
    if (n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.all_gather) g_nccl = n;
  });
  return g_nccl.so ? &g_nccl : nullptr;
}

int nccl_fail(const char* where, int r) {
  const Nccl* n = nccl();
  char msg[256];
  std::snprintf(msg, sizeof(msg), "%s: %s", where, n && n->error_string ? n->error_string(r) : "NCCL error");
  return dp::set_last_error(DP_ERR_CUDA, msg);
}
int no_nccl() { return dp::set_last_error(DP_ERR_UNSUPPORTED, "libnccl.so.2 not found (dlopen)"); }

}  // namespace

extern "C" {

DP_API int dp_nccl_available(void) { return nccl() ? 1 : 0; }

DP_API int dp_nccl_unique_id(uint8_t* id128) {
  const Nccl* n = nccl();
  if (!n) return no_nccl();
  if (!id128) return DP_ERR_ARG;
  nccl_unique_id_t id;
  const int r = n->get_unique_id(&id);
  if (r != kNcclSuccess) return nccl_fail("ncclGetUniqueId", r);
  std::memcpy(id128, id.internal, 128);
  return DP_OK;
}

DP_API int dp_nccl_comm_init(void** comm, int32_t nranks, const uint8_t* id128, int32_t rank) {
  const Nccl* n = nccl();
  if (!n) return no_nccl();
  if (!comm || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return DP_ERR_ARG;
  nccl_unique_id_t id;
  std::memcpy(id.internal, id128, 128);
  nccl_comm_t c = nullptr;
  const int r = n->comm_init_rank(&c, nranks, id, rank);   // on the caller's current device
  if (r != kNcclSuccess) return nccl_fail("ncclCommInitRank", r);
  *comm = c;
  return DP_OK;
}

DP_API int dp_nccl_comm_destroy(void* comm) {
  const Nccl* n = nccl();
  if (!n) return no_nccl();
  if (!comm) return DP_OK;
  const int r = n->comm_destroy(static_cast<nccl_comm_t>(comm));
  return r == kNcclSuccess ? DP_OK : nccl_fail("ncclCommDestroy", r);
}

DP_API int dp_allgather_tokens(const int32_t* local, int32_t* global, int64_t rows_per_rank, void* comm,
                               void* stream) {
  const Nccl* n = nccl();
  if (!n) return no_nccl();
  if (!comm || rows_per_rank < 0 || (rows_per_rank > 0 && (!local || !global))) return DP_ERR_ARG;
  if (rows_per_rank == 0) return DP_OK;
  const int r = n->all_gather(local, global, (size_t)rows_per_rank, kNcclInt32, static_cast<nccl_comm_t>(comm),
                              static_cast<cudaStream_t>(stream));
  return r == kNcclSuccess ? DP_OK : nccl_fail("ncclAllGather", r);
}

}  // extern "C"
