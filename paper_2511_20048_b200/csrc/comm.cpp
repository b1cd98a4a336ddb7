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

// ---------------------------------------------------------------------------------------------
// F1: the peer-memory region of the fused decode + all-gather.  One
// cudaMalloc per rank holds the gathered-output buffers and a signal pad; the other ranks
// map it with CUDA IPC (NVLink peer access), so the decode kernel can store its heads'
// outputs into every rank's buffer and release a flag into every rank's pad.

namespace {
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
constexpr size_t kSigBytes = 256;      // u32 flags [world] at 0, the status word at 128
constexpr size_t kStatusOff = 128;
}  // namespace

extern "C" {

spa_status spa_peer_create(int32_t rank, int32_t world, size_t buf_bytes, int32_t n_bufs, spa_peer** out) {
    if (!out) return fail(SPA_ERR_INVALID_ARG, "null output");
    *out = nullptr;
    if (world < 1 || world > 8 || rank < 0 || rank >= world || n_bufs < 1 || buf_bytes == 0)
        return fail(SPA_ERR_INVALID_ARG, "bad peer arguments (1 <= world <= 8, 0 <= rank < world, n_bufs >= 1)");
    spa_peer* p = new spa_peer();
    p->rank = rank;
    p->world = world;
    p->buf_bytes = buf_bytes;
    p->buf_stride = align256(buf_bytes);
    p->n_bufs = n_bufs;
    p->sig_off = p->buf_stride * size_t(n_bufs);
    cudaError_t e = cudaGetDevice(&p->device);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&p->base), p->sig_off + kSigBytes);
    if (e == cudaSuccess) e = cudaMemset(p->base + p->sig_off, 0, kSigBytes);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        if (p->base) cudaFree(p->base);
        delete p;
        return fail(SPA_ERR_CUDA, std::string("spa_peer_create: ") + cudaGetErrorString(e));
    }
    p->peer_base[rank] = p->base;
    p->connected = world == 1;
    *out = p;
    return SPA_OK;
}

spa_status spa_peer_ipc_handle(const spa_peer* peer, void* out_handle) {
    if (!peer || !out_handle) return fail(SPA_ERR_INVALID_ARG, "null argument");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, peer->base);
    if (e != cudaSuccess) return fail(SPA_ERR_CUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(out_handle, &h, sizeof(h));
    return SPA_OK;
}

spa_status spa_peer_connect(spa_peer* peer, const void* handles) {
    if (!peer || !handles) return fail(SPA_ERR_INVALID_ARG, "null argument");
    if (peer->connected) return fail(SPA_ERR_INVALID_ARG, "peer already connected");
    for (int k = 0; k < peer->world; ++k) {
        if (k == peer->rank) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const char*>(handles) + 64 * k, sizeof(h));
        void* ptr = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            for (int j = 0; j < k; ++j)
                if (peer->ipc_opened[j]) {
                    cudaIpcCloseMemHandle(peer->peer_base[j]);
                    peer->ipc_opened[j] = false;
                    peer->peer_base[j] = nullptr;
                }
            return fail(SPA_ERR_CUDA, "cudaIpcOpenMemHandle(rank " + std::to_string(k) + "): " + cudaGetErrorString(e));
        }
        peer->peer_base[k] = static_cast<char*>(ptr);
        peer->ipc_opened[k] = true;
    }
    peer->connected = true;
    return SPA_OK;
}

spa_status spa_peer_connect_local(spa_peer* const* peers, int32_t world) {
    if (!peers || world < 1 || world > 8) return fail(SPA_ERR_INVALID_ARG, "bad peer list");
    for (int i = 0; i < world; ++i) {
        if (!peers[i] || peers[i]->world != world || peers[i]->rank != i || peers[i]->device != peers[0]->device ||
            peers[i]->buf_stride != peers[0]->buf_stride || peers[i]->n_bufs != peers[0]->n_bufs)
            return fail(SPA_ERR_INVALID_ARG, "local peers must be ranks 0..world-1 of one world, device and size");
        if (peers[i]->connected && world > 1) return fail(SPA_ERR_INVALID_ARG, "peer already connected");
    }
    for (int i = 0; i < world; ++i) {
        for (int k = 0; k < world; ++k) peers[i]->peer_base[k] = peers[k]->base;
        peers[i]->connected = true;
    }
    return SPA_OK;
}

spa_status spa_peer_buffer(const spa_peer* peer, int32_t buf_idx, void** out_ptr) {
    if (!peer || !out_ptr) return fail(SPA_ERR_INVALID_ARG, "null argument");
    if (buf_idx < 0 || buf_idx >= peer->n_bufs) return fail(SPA_ERR_INVALID_ARG, "buffer index out of range");
    *out_ptr = peer->base + size_t(buf_idx) * peer->buf_stride;
    return SPA_OK;
}

spa_status spa_peer_status(const spa_peer* peer, int32_t* out_status) {
    if (!peer || !out_status) return fail(SPA_ERR_INVALID_ARG, "null argument");
    uint32_t st = 0;
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(&st, peer->base + peer->sig_off + kStatusOff, 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return fail(SPA_ERR_CUDA, std::string("spa_peer_status: ") + cudaGetErrorString(e));
    *out_status = int32_t(st);
    return SPA_OK;
}

spa_status spa_peer_destroy(spa_peer* peer) {
    if (!peer) return SPA_OK;
    for (int k = 0; k < peer->world; ++k)
        if (peer->ipc_opened[k]) cudaIpcCloseMemHandle(peer->peer_base[k]);
    if (peer->base) cudaFree(peer->base);
    delete peer;
    return SPA_OK;
}

}  // extern "C"

namespace spa {
// The launch description of one fused call (api.cpp); advances the epoch.
void peer_launch(spa_peer* peer, PeerLaunch* pl) {
    pl->rank = peer->rank;
    pl->world = peer->world;
    for (int k = 0; k < 8; ++k) {
        pl->delta[k] = k < peer->world ? (long long)(peer->peer_base[k] - peer->base) : 0;
        pl->sig_peer[k] = k < peer->world ? reinterpret_cast<unsigned*>(peer->peer_base[k] + peer->sig_off) : nullptr;
    }
    pl->sig_local = reinterpret_cast<unsigned*>(peer->base + peer->sig_off);
    pl->status = reinterpret_cast<unsigned*>(peer->base + peer->sig_off + kStatusOff);
    pl->epoch = ++peer->epoch;
}
}  // namespace spa
