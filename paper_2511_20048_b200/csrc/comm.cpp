// Head-sharded multi-GPU plumbing: an NCCL communicator
// created inside the library from an ncclUniqueId that the caller distributes (rank 0
// creates it, torch.distributed broadcasts the 128 bytes), and an in-place all-gather
// of the head-sharded outputs.  NCCL is loaded with dlopen at spa_comm_create so the
// library loads (and its host logic is testable) on machines without NCCL or a GPU.
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <string>

#include "nccl.h"
#include "spa_internal.h"

namespace spa {
namespace {

struct NcclApi {
    void* handle = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

bool load_nccl(NcclApi* api, std::string* err) {
    static NcclApi cached;
    static bool tried = false, ok = false;
    if (!tried) {
        tried = true;
        const char* names[] = {std::getenv("SPA_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
        for (const char* n : names) {
            if (!n || !*n) continue;
            cached.handle = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (cached.handle) break;
        }
        if (cached.handle) {
            cached.get_unique_id = reinterpret_cast<decltype(cached.get_unique_id)>(dlsym(cached.handle, "ncclGetUniqueId"));
            cached.comm_init_rank = reinterpret_cast<decltype(cached.comm_init_rank)>(dlsym(cached.handle, "ncclCommInitRank"));
            cached.comm_destroy = reinterpret_cast<decltype(cached.comm_destroy)>(dlsym(cached.handle, "ncclCommDestroy"));
            cached.all_gather = reinterpret_cast<decltype(cached.all_gather)>(dlsym(cached.handle, "ncclAllGather"));
            cached.error_string = reinterpret_cast<decltype(cached.error_string)>(dlsym(cached.handle, "ncclGetErrorString"));
            ok = cached.get_unique_id && cached.comm_init_rank && cached.comm_destroy && cached.all_gather &&
                 cached.error_string;
        }
    }
    if (!ok) {
        *err = "cannot load NCCL (set SPA_NCCL_LIB to libnccl.so.2)";
        return false;
    }
    *api = cached;
    return true;
}

}  // namespace

int comm_all_gather(spa_comm* comm, const void* send, void* recv, size_t count, int is_bf16, void* stream,
                    std::string* err) {
    NcclApi api;
    if (!load_nccl(&api, err)) return 1;
    ncclResult_t r = api.all_gather(send, recv, count, is_bf16 ? ncclBfloat16 : ncclFloat32,
                                    static_cast<ncclComm_t>(comm->nccl_comm), static_cast<cudaStream_t>(stream));
    if (r != ncclSuccess) {
        *err = std::string("ncclAllGather: ") + api.error_string(r);
        return 1;
    }
    return 0;
}

}  // namespace spa

using namespace spa;

extern "C" {

spa_status spa_nccl_unique_id(void* out_id) {
    if (!out_id) return fail(SPA_ERR_INVALID_ARG, "null output");
    NcclApi api;
    std::string why;
    if (!load_nccl(&api, &why)) return fail(SPA_ERR_NCCL, why);
    ncclUniqueId id;
    ncclResult_t r = api.get_unique_id(&id);
    if (r != ncclSuccess) return fail(SPA_ERR_NCCL, std::string("ncclGetUniqueId: ") + api.error_string(r));
    std::memcpy(out_id, &id, sizeof(id));
    return SPA_OK;
}

spa_status spa_comm_create(const void* unique_id, int32_t rank, int32_t world, spa_comm** out) {
    if (!unique_id || !out || world <= 0 || rank < 0 || rank >= world)
        return fail(SPA_ERR_INVALID_ARG, "bad comm arguments");
    *out = nullptr;
    spa_comm* c = new spa_comm();
    c->rank = rank;
    c->world = world;
    if (world > 1) {
        NcclApi api;
        std::string why;
        if (!load_nccl(&api, &why)) {
            delete c;
            return fail(SPA_ERR_NCCL, why);
        }
        ncclUniqueId id;
        std::memcpy(&id, unique_id, sizeof(id));
        ncclComm_t nc = nullptr;
        ncclResult_t r = api.comm_init_rank(&nc, world, id, rank);
        if (r != ncclSuccess) {
            delete c;
            return fail(SPA_ERR_NCCL, std::string("ncclCommInitRank: ") + api.error_string(r));
        }
        c->nccl_comm = nc;
    }
    *out = c;
    return SPA_OK;
}

spa_status spa_comm_destroy(spa_comm* comm) {
    if (!comm) return SPA_OK;
    if (comm->nccl_comm) {
        NcclApi api;
        std::string why;
        if (load_nccl(&api, &why)) api.comm_destroy(static_cast<ncclComm_t>(comm->nccl_comm));
    }
    delete comm;
    return SPA_OK;
}

}  // extern "C"
