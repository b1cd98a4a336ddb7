// C ABI entry points of the decode step (a5/a6), the head-sharded launcher (a7) and the
// fused decode + peer-memory all-gather (S8(f) F1).
#include <cmath>
#include <cstdint>
#include <string>

#include "spa_internal.h"

namespace spa {
// comm.cpp
int comm_all_gather(spa_comm* comm, const void* send, void* recv, size_t count, int is_bf16, void* stream,
                    std::string* err);
void peer_launch(spa_peer* peer, PeerLaunch* pl);
}  // namespace spa

using namespace spa;

static bool aligned4(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 3) == 0; }

static spa_status check_decode_args(const spa_plan* plan, int32_t layer, const void* q, int64_t q_sr, int64_t q_sh,
                                    const void* o, int64_t o_sr, int64_t o_sh, float scale) {
    if (!plan) return fail(SPA_ERR_INVALID_ARG, "null plan");
    const spa_pool* pool = plan->pool;
    if (pool->metadata_only) return fail(SPA_ERR_NO_DEVICE, "decode on a metadata-only pool");
    if (spa_status s = check_device(pool)) return s;
    if (plan->host.empty()) return fail(SPA_ERR_INVALID_ARG, "plan has not been built (spa_decode_plan)");
    if (!plan->uploaded)
        return fail(SPA_ERR_WORKSPACE, "the last spa_decode_plan did not reach the device (no or too small workspace)");
    if (layer < 0 || layer >= pool->cfg.num_layers) return fail(SPA_ERR_INVALID_ARG, "layer out of range");
    if (plan->n_req > 0 && (!q || !o)) return fail(SPA_ERR_INVALID_ARG, "null q or o");
    // 32-bit query loads and bf16x2 output stores need even element strides and 4-B alignment
    if (!aligned4(q) || !aligned4(o) || (q_sr | q_sh | o_sr | o_sh) & 1)
        return fail(SPA_ERR_INVALID_ARG, "q/o must be 4-byte aligned with even element strides");
    if (!std::isfinite(scale)) return fail(SPA_ERR_INVALID_ARG, "scale must be finite");
    return SPA_OK;
}

extern "C" {

spa_status spa_decode_attention(const spa_plan* plan, int32_t layer, const void* q, int64_t q_stride_req,
                                int64_t q_stride_head, void* o, int64_t o_stride_req, int64_t o_stride_head, float* lse,
                                int64_t lse_stride_req, int64_t lse_stride_head, float scale, void* stream) {
    if (spa_status s = check_decode_args(plan, layer, q, q_stride_req, q_stride_head, o, o_stride_req, o_stride_head,
                                         scale))
        return s;
    int err = launch_decode(plan, layer, q, q_stride_req, q_stride_head, o, o_stride_req, o_stride_head, lse,
                            lse_stride_req, lse_stride_head, scale, stream);
    if (err) return fail(SPA_ERR_CUDA, std::string("decode kernel: ") + cuda_error_string(err));
    return SPA_OK;
}

spa_status spa_merge_splits(int32_t n_req, int32_t num_heads, int32_t head_dim, const int32_t* rec_ptr,
                            const float* part_o, const float* part_lse, void* o, int64_t o_stride_req,
                            int64_t o_stride_head, float* lse, int64_t lse_stride_req, int64_t lse_stride_head,
                            void* stream) {
    if (n_req < 0 || num_heads <= 0 || head_dim <= 0 || head_dim % 4)
        return fail(SPA_ERR_INVALID_ARG, "bad merge sizes (head_dim must be a multiple of 4)");
    if (n_req == 0) return SPA_OK;
    if (!rec_ptr || !part_o || !part_lse || !o) return fail(SPA_ERR_INVALID_ARG, "null merge pointer");
    if (!aligned4(o) || (o_stride_req | o_stride_head) & 1 || (reinterpret_cast<uintptr_t>(part_o) & 15))
        return fail(SPA_ERR_INVALID_ARG, "o must be 4-B aligned with even strides; part_o 16-B aligned");
    int err = launch_merge(n_req, num_heads, head_dim, rec_ptr, part_o, part_lse, o, o_stride_req, o_stride_head, lse,
                           lse_stride_req, lse_stride_head, 0, stream);
    if (err) return fail(SPA_ERR_CUDA, std::string("merge kernel: ") + cuda_error_string(err));
    return SPA_OK;
}

spa_status spa_decode_attention_sharded(const spa_plan* plan, spa_comm* comm, int32_t layer, const void* q_local,
                                        int64_t q_stride_req, int64_t q_stride_head, void* o_gathered,
                                        float* lse_gathered, float scale, void* stream) {
    if (!comm) return fail(SPA_ERR_INVALID_ARG, "null comm");
    if (!plan) return fail(SPA_ERR_INVALID_ARG, "null plan");
    const auto& c = plan->pool->cfg;
    const int64_t N = plan->n_req, Hl = c.num_q_heads, D = c.head_dim;
    const size_t count = size_t(Hl * N * D);
    uint16_t* ob = static_cast<uint16_t*>(o_gathered);
    uint16_t* mine = ob ? ob + size_t(comm->rank) * count : nullptr;
    float* lmine = lse_gathered ? lse_gathered + size_t(comm->rank) * Hl * N : nullptr;
    // o[i][h] of this rank at mine[h * N * D + i * D]  (head-major slot of the gathered buffer)
    if (spa_status s = check_decode_args(plan, layer, q_local, q_stride_req, q_stride_head, mine, D, N * D, scale))
        return s;
    int err = launch_decode(plan, layer, q_local, q_stride_req, q_stride_head, mine, D, N * D, lmine, 1, N, scale,
                            stream);
    if (err) return fail(SPA_ERR_CUDA, std::string("decode kernel: ") + cuda_error_string(err));
    if (comm->world > 1 && N > 0) {
        std::string why;
        if (comm_all_gather(comm, mine, o_gathered, count, 1, stream, &why)) return fail(SPA_ERR_NCCL, why);
        if (lse_gathered && comm_all_gather(comm, lmine, lse_gathered, size_t(Hl * N), 0, stream, &why))
            return fail(SPA_ERR_NCCL, why);
    }
    return SPA_OK;
}

spa_status spa_decode_attention_fused_gather(const spa_plan* plan, spa_peer* peer, int32_t layer, const void* q_local,
                                             int64_t q_stride_req, int64_t q_stride_head, int32_t buf_idx,
                                             int32_t with_lse, float scale, void* stream) {
    if (!peer) return fail(SPA_ERR_INVALID_ARG, "null peer");
    if (!plan) return fail(SPA_ERR_INVALID_ARG, "null plan");
    if (!peer->connected) return fail(SPA_ERR_INVALID_ARG, "peer not connected (spa_peer_connect)");
    if (buf_idx < 0 || buf_idx >= peer->n_bufs) return fail(SPA_ERR_INVALID_ARG, "buffer index out of range");
    if (plan->mt == 8 || plan->cfg.merge_mode == 2)
        return fail(SPA_ERR_UNSUPPORTED, "fused gather needs a decode plan (max_rows <= 64) with merge_mode 0 or 1");
    const auto& c = plan->pool->cfg;
    const int64_t N = plan->n_req, Hl = c.num_q_heads, D = c.head_dim, W = peer->world;
    const size_t o_bytes = size_t(W * Hl * N * D) * 2;
    const size_t lse_off = (o_bytes + 255) & ~size_t(255);
    if ((with_lse ? lse_off + size_t(W * Hl * N) * 4 : o_bytes) > peer->buf_bytes)
        return fail(SPA_ERR_INVALID_ARG, "peer buffer too small for [world][Hq_local][N][d] (+ LSE)");
    char* buf = peer->base + size_t(buf_idx) * peer->buf_stride;
    uint16_t* mine = reinterpret_cast<uint16_t*>(buf) + size_t(peer->rank * Hl * N * D);
    float* lmine = with_lse ? reinterpret_cast<float*>(buf + lse_off) + size_t(peer->rank * Hl * N) : nullptr;
    if (spa_status s = check_decode_args(plan, layer, q_local, q_stride_req, q_stride_head, mine, D, N * D, scale))
        return s;
    PeerLaunch pl;
    peer_launch(peer, &pl);
    int err = launch_decode(plan, layer, q_local, q_stride_req, q_stride_head, mine, D, N * D, lmine, 1, N, scale,
                            stream, W > 1 ? &pl : nullptr);
    if (err) return fail(SPA_ERR_CUDA, std::string("decode kernel (fused gather): ") + cuda_error_string(err));
    return SPA_OK;
}

}  // extern "C"
