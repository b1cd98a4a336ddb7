// Paged KV pool: request table, lowest-free-id page allocator, refcounts, copy-free fork.
//
// Policy (DESIGN.md Sec. 3 readings #3, #4, #17; oracle/kvmodel.py P1-P6 is the
// independent model it is tested against bit-exactly):
//   - pages are taken lowest-free-id first; request ids are 1, 2, ... never reused;
//   - append is all-or-nothing; a page is taken exactly when length % page_size == 0;
//   - fork shares the parent's full pages of the prefix (refcount + 1) and copies the
//     partial page (copy-on-write at fork time), so a shared page is always full and
//     is never written again (append-only);
//   - free decrements refcounts; pages at 0 return to the free set.
// Speculative forks of the agent context c_i: PAPER.md:189, :198, :335.
#include <algorithm>
#include <cstring>
#include <unordered_set>

#include "spa_internal.h"

namespace spa {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

spa_status fail(spa_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

static spa_status check_pool(const spa_pool* p) {
    if (!p) return fail(SPA_ERR_INVALID_ARG, "null pool");
    return SPA_OK;
}

// Device work of a pool is launched on the calling thread's current device, which must be
// the device the pool was created on (its tensor maps and kernel attributes live there).
spa_status check_device(const spa_pool* p) {
    if (p->metadata_only) return SPA_OK;
    const int dev = current_device();
    if (dev != p->device)
        return fail(SPA_ERR_INVALID_ARG, "the current CUDA device (" + std::to_string(dev) +
                                             ") is not the pool's device (" + std::to_string(p->device) + ")");
    return SPA_OK;
}

}  // namespace spa

using namespace spa;

extern "C" {

int32_t spa_abi_version(void) { return SPA_ABI_VERSION; }

const char* spa_last_error(void) { return g_last_error.c_str(); }

static spa_status pool_create(const spa_pool_config* cfg, void* k_pool, void* v_pool, bool fp8, const float* kv_scale,
                              spa_pool** out) {
    if (!cfg || !out) return fail(SPA_ERR_INVALID_ARG, "null argument");
    *out = nullptr;
    const spa_pool_config& c = *cfg;
    if (c.num_layers <= 0 || c.num_q_heads <= 0 || c.num_kv_heads <= 0 || c.head_dim <= 0 || c.page_size <= 0 ||
        c.num_pages <= 0)
        return fail(SPA_ERR_INVALID_ARG, "pool sizes must be positive");
    if (c.num_q_heads % c.num_kv_heads) return fail(SPA_ERR_INVALID_ARG, "num_q_heads % num_kv_heads != 0");
    if ((k_pool == nullptr) != (v_pool == nullptr))
        return fail(SPA_ERR_INVALID_ARG, "k_pool and v_pool must both be device pointers or both NULL");
    const bool device = k_pool != nullptr;
    if (device) {
        if (c.head_dim != 64 && c.head_dim != 128) return fail(SPA_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
        if (c.page_size != kPageSize) return fail(SPA_ERR_UNSUPPORTED, "page_size must be 16");
        if ((reinterpret_cast<uintptr_t>(k_pool) | reinterpret_cast<uintptr_t>(v_pool)) & 127)
            return fail(SPA_ERR_INVALID_ARG, "k_pool / v_pool must be 128-byte aligned");
        const int64_t rows = int64_t(c.num_layers) * c.num_pages * c.num_kv_heads * c.page_size;
        if (rows >= (int64_t(1) << 31)) return fail(SPA_ERR_UNSUPPORTED, "pool exceeds 2^31 rows");
        if (fp8) {
            if (c.head_dim != 128) return fail(SPA_ERR_UNSUPPORTED, "fp8 KV pages need head_dim 128");
            if (!kv_scale) return fail(SPA_ERR_INVALID_ARG, "fp8 KV pages need kv_scale");
            if (rows * 2 >= (int64_t(1) << 31)) return fail(SPA_ERR_UNSUPPORTED, "fp8 pool exceeds 2^31 128-B rows");
        }
    }
    spa_pool* p = new spa_pool();
    p->cfg = c;
    p->k_pool = k_pool;
    p->v_pool = v_pool;
    p->metadata_only = !device;
    p->kv_fp8 = fp8;
    p->kv_scale = kv_scale;
    p->refcount.assign(c.num_pages, 0);
    for (int32_t i = 0; i < c.num_pages; ++i) p->free_set.insert(p->free_set.end(), i);
    if (device) {
        int dev = -1;
        int sms = device_sm_count(&dev);
        if (sms <= 0) {
            delete p;
            return fail(SPA_ERR_CUDA, std::string("cannot query the CUDA device: ") + cuda_error_string(-sms));
        }
        p->device = dev;
        p->sm_count = sms;
        int err = memset_pool(p);
        if (err) {
            delete p;
            return fail(SPA_ERR_CUDA, std::string("zero-filling the pool: ") + cuda_error_string(err));
        }
        std::string why;
        if (!make_tensor_maps(p, &why)) {
            delete p;
            return fail(SPA_ERR_CUDA, "cuTensorMapEncodeTiled: " + why);
        }
    }
    *out = p;
    return SPA_OK;
}

spa_status spa_pool_create(const spa_pool_config* cfg, void* k_pool, void* v_pool, spa_pool** out) {
    return pool_create(cfg, k_pool, v_pool, false, nullptr, out);
}

spa_status spa_pool_create_fp8(const spa_pool_config* cfg, void* kv_pool, const float* kv_scale, spa_pool** out) {
    // one interleaved buffer: page-head blocks of 4 KB = K (2 KB) then V^T (2 KB)
    return pool_create(cfg, kv_pool, kv_pool ? static_cast<char*>(kv_pool) + 2048 : nullptr, true, kv_scale, out);
}

spa_status spa_pool_destroy(spa_pool* pool) {
    delete pool;
    return SPA_OK;
}

spa_status spa_kv_alloc(spa_pool* pool, spa_req* out_req) {
    if (spa_status s = check_pool(pool)) return s;
    if (!out_req) return fail(SPA_ERR_INVALID_ARG, "null out_req");
    const int64_t id = pool->next_id++;
    pool->reqs.emplace(id, Request{});
    *out_req = id;
    return SPA_OK;
}

spa_status spa_kv_append(spa_pool* pool, int32_t n_req, const spa_req* reqs, const int32_t* n_new,
                         const void* k_new, const void* v_new, void* stream) {
    if (spa_status s = check_pool(pool)) return s;
    if (spa_status s = check_device(pool)) return s;
    if (n_req < 0 || (n_req > 0 && (!reqs || !n_new))) return fail(SPA_ERR_INVALID_ARG, "bad request list");
    const int ps = pool->cfg.page_size;
    std::unordered_set<int64_t> seen;
    for (int i = 0; i < n_req; ++i)
        if (!seen.insert(reqs[i]).second) return fail(SPA_ERR_INVALID_ARG, "append: request listed twice");
    int64_t need = 0, total = 0;
    for (int i = 0; i < n_req; ++i) {
        auto it = pool->reqs.find(reqs[i]);
        if (it == pool->reqs.end()) return fail(SPA_ERR_BAD_REQUEST, "append: unknown request " + std::to_string(reqs[i]));
        if (n_new[i] < 0) return fail(SPA_ERR_INVALID_ARG, "append: negative token count");
        const int64_t L = it->second.len;
        if (L + n_new[i] > int64_t(INT32_MAX)) return fail(SPA_ERR_INVALID_ARG, "append: length overflow");
        need += cdiv(L + n_new[i], ps) - cdiv(L, ps);
        total += n_new[i];
    }
    if (need > int64_t(pool->free_set.size()))
        return fail(SPA_ERR_NO_PAGES, "append needs " + std::to_string(need) + " pages, " +
                                          std::to_string(pool->free_set.size()) + " free");
    if (total > 0 && !pool->metadata_only && (!k_new || !v_new)) return fail(SPA_ERR_INVALID_ARG, "null k_new/v_new");
    std::vector<int32_t> slots;
    slots.reserve(total);
    for (int i = 0; i < n_req; ++i) {
        Request& r = pool->reqs[reqs[i]];
        for (int32_t t = 0; t < n_new[i]; ++t) {
            if (r.len % ps == 0) {
                const int32_t p = *pool->free_set.begin();
                pool->free_set.erase(pool->free_set.begin());
                pool->refcount[p] = 1;
                r.pages.push_back(p);
            }
            slots.push_back(r.pages.back() * ps + (r.len % ps));
            r.len += 1;
        }
    }
    if (!pool->metadata_only && total > 0) {
        int err = launch_append(pool, k_new, v_new, int32_t(total), slots, stream);
        if (err) return fail(SPA_ERR_CUDA, std::string("append kernel: ") + cuda_error_string(err));
    }
    return SPA_OK;
}

spa_status spa_fork_request(spa_pool* pool, spa_req parent, int32_t prefix_len, spa_req* out_child, void* stream) {
    if (spa_status s = check_pool(pool)) return s;
    if (spa_status s = check_device(pool)) return s;
    if (!out_child) return fail(SPA_ERR_INVALID_ARG, "null out_child");
    auto it = pool->reqs.find(parent);
    if (it == pool->reqs.end()) return fail(SPA_ERR_BAD_REQUEST, "fork: unknown parent " + std::to_string(parent));
    if (prefix_len < 0 || prefix_len > it->second.len)
        return fail(SPA_ERR_INVALID_ARG, "fork: prefix_len outside [0, parent length]");
    const int ps = pool->cfg.page_size;
    const int32_t full = prefix_len / ps, rem = prefix_len % ps;
    if (rem && pool->free_set.empty()) return fail(SPA_ERR_NO_PAGES, "fork: no free page for the partial page copy");
    if (rem && it->second.pages[full] < 0)
        return fail(SPA_ERR_INVALID_ARG, "fork: the partial page at the fork point was released (spa_kv_release_window)");
    Request child;
    child.len = prefix_len;
    child.pages.assign(it->second.pages.begin(), it->second.pages.begin() + full);
    for (int32_t p : child.pages)
        if (p >= 0) pool->refcount[p] += 1;   // released entries (-1) stay released in the child
    int32_t src = -1, dst = -1;
    if (rem) {
        dst = *pool->free_set.begin();
        pool->free_set.erase(pool->free_set.begin());
        pool->refcount[dst] = 1;
        src = it->second.pages[full];
        child.pages.push_back(dst);
    }
    const int64_t id = pool->next_id++;
    pool->reqs.emplace(id, std::move(child));
    *out_child = id;
    if (rem && !pool->metadata_only) {
        int err = launch_cow(pool, src, dst, rem, stream);
        if (err) return fail(SPA_ERR_CUDA, std::string("copy-on-write kernel: ") + cuda_error_string(err));
    }
    return SPA_OK;
}

spa_status spa_kv_free(spa_pool* pool, spa_req req) {
    if (spa_status s = check_pool(pool)) return s;
    auto it = pool->reqs.find(req);
    if (it == pool->reqs.end()) return fail(SPA_ERR_BAD_REQUEST, "free: unknown request " + std::to_string(req));
    for (int32_t p : it->second.pages) {
        if (p >= 0 && --pool->refcount[p] == 0) pool->free_set.insert(p);
    }
    pool->reqs.erase(it);
    return SPA_OK;
}

spa_status spa_kv_release_window(spa_pool* pool, int32_t n_req, const spa_req* reqs, int32_t window) {
    if (spa_status s = check_pool(pool)) return s;
    if (window <= 0) return fail(SPA_ERR_INVALID_ARG, "release_window: window must be > 0");
    if (n_req < 0 || (n_req > 0 && !reqs)) return fail(SPA_ERR_INVALID_ARG, "bad request list");
    for (int i = 0; i < n_req; ++i)
        if (pool->reqs.find(reqs[i]) == pool->reqs.end())
            return fail(SPA_ERR_BAD_REQUEST, "release_window: unknown request " + std::to_string(reqs[i]));
    const int64_t ps = pool->cfg.page_size;
    for (int i = 0; i < n_req; ++i) {
        Request& r = pool->reqs[reqs[i]];
        // append-then-attend (reading #8): the current step's query sits at len - 1 and reads
        // keys >= len - window, later queries only later keys, so page p (keys [p ps, p ps +
        // ps)) is dead once p ps + ps <= len - window
        const int64_t dead = std::max<int64_t>(0, (int64_t(r.len) - window) / ps);
        for (int64_t p = 0; p < std::min<int64_t>(dead, int64_t(r.pages.size())); ++p) {
            const int32_t id = r.pages[p];
            if (id < 0) continue;
            if (--pool->refcount[id] == 0) pool->free_set.insert(id);
            r.pages[p] = -1;
        }
    }
    return SPA_OK;
}

spa_status spa_kv_page_table(const spa_pool* pool, spa_req req, int32_t* out_pages, int32_t cap, int32_t* out_n_pages,
                             int32_t* out_len) {
    if (spa_status s = check_pool(pool)) return s;
    auto it = pool->reqs.find(req);
    if (it == pool->reqs.end()) return fail(SPA_ERR_BAD_REQUEST, "unknown request " + std::to_string(req));
    const auto& pg = it->second.pages;
    if (out_pages && cap > 0) std::memcpy(out_pages, pg.data(), sizeof(int32_t) * std::min<size_t>(cap, pg.size()));
    if (out_n_pages) *out_n_pages = int32_t(pg.size());
    if (out_len) *out_len = it->second.len;
    return SPA_OK;
}

spa_status spa_pool_refcounts(const spa_pool* pool, int32_t* out_refcount) {
    if (spa_status s = check_pool(pool)) return s;
    if (!out_refcount) return fail(SPA_ERR_INVALID_ARG, "null output");
    std::memcpy(out_refcount, pool->refcount.data(), sizeof(int32_t) * pool->refcount.size());
    return SPA_OK;
}

spa_status spa_pool_free_pages(const spa_pool* pool, int32_t* out_pages, int32_t cap, int32_t* out_n) {
    if (spa_status s = check_pool(pool)) return s;
    int32_t i = 0;
    if (out_pages)
        for (int32_t p : pool->free_set) {
            if (i >= cap) break;
            out_pages[i++] = p;
        }
    if (out_n) *out_n = int32_t(pool->free_set.size());
    return SPA_OK;
}

}  // extern "C"
