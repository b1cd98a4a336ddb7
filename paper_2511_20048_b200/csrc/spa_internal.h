// Internal declarations shared by the host core (pool.cpp, plan.cpp, api.cpp, comm.cpp)
// and the CUDA kernels (kernels.cu).  Nothing here is part of the public ABI.
#pragma once

#include <cstdint>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/spa.h"

namespace spa {

// ---------------------------------------------------------------------------- errors
void set_error(const std::string& msg);
spa_status fail(spa_status st, const std::string& msg);

// ---------------------------------------------------------------------------- plan metadata
// Device plan = one int32 array: a header, then the arrays below at the header offsets.
enum MetaHeader : int {
    H_N_REQ = 0,
    H_N_DESC = 1,
    H_N_ITEMS = 2,
    H_N_TEAMS = 3,
    H_N_RECORDS = 4,
    H_OFF_DESC = 5,
    H_OFF_MEMBER = 6,
    H_OFF_ITEM = 7,
    H_OFF_SCHED = 8,       // int32[kSchedSlots][kSchedStride], 128-B lines: line 0 = {queue head, finished
                           // CTAs, -, owner launch}; line 1 = {tail-merge queue head}
    H_OFF_QUEUE = 9,       // int32[n_items]: item indices, largest first
    H_OFF_PAGES = 10,
    H_OFF_REC_PTR = 11,
    H_TOTAL = 12,
    H_N_MEMBERS = 13,
    H_N_PAGES = 14,
    H_OFF_COUNTERS = 15,   // int32 [n_req][Hkv] record arrivals of the in-kernel merges (launch k of a plan
                           // completes a task at (k + 1) x its records; zeroed by the plan upload)
    H_OFF_MTASK = 16,      // int32 [n_mtask]: tail-merge subtasks (row * Hkv + kv_head) * 256 + (0: all G
                           // heads | 1 + head), earliest-ready first
    H_N_MTASK = 17,
    H_OFF_QITEM = 18,      // QItem[n_items]: the queue's items with their descriptors, in pop order
    H_WORDS = 20
};

// Work descriptor: keys [tok_start, tok_end) of one group-split or member-tail-split, read
// through pages[page_off .. page_off + n_main) (tok_start = first page * ps), then (folded
// member tails) pages [n_main, n_pages) of the same list: each member's own tail, read only
// by that member's rows (Member::tail_*).  kind: bit 0 some row also reads another
// descriptor; bit 2 the shared pages hold a member's newest token; bit 3 a folded tail does
// (the kernels do not prefetch such pages before their programmatic-dependency wait).
struct Desc {
    int32_t page_off, n_pages, tok_start, tok_end, member_off, n_members, kind, group;
    int32_t n_main, reserved0, reserved1, reserved2;
};
static_assert(sizeof(Desc) == 48, "Desc is 12 int32");

// One request (batch row) taking part in a descriptor.
struct Member {
    int32_t row;   // batch row (index into q / o / lse)
    int32_t lo;    // window lower bound: keys j < lo are masked for this member
    int32_t rec;   // partial record index, or -1: write final O / LSE directly
    int32_t hi;    // causal bound: keys j >= hi are masked for this row (decode: the length)
    // folded tail: descriptor pages [tail_k0, tail_k0 + tail_n) are this row's own, page
    // tail_k0 holding its tokens [tail_tok, tail_tok + ps); tail_n = 0: none
    int32_t tail_k0, tail_n, tail_tok, reserved;
};

struct Item {
    int32_t desc, kv_head;
};

// A queue entry as the kernels pop it: the item's descriptor copied next to its KV head, so
// a pop is one atomic and one 64-B load instead of four dependent loads (queue -> item ->
// descriptor)
struct QItem {
    Desc d;
    int32_t it, kv_head, desc, reserved;
};
static_assert(sizeof(QItem) == 64, "QItem is 16 int32");

constexpr int kPageSize = 16;          // tokens per page the kernels implement
constexpr int kPagesPerStage = 2;      // pages of one (KV head) streamed per pipeline stage
constexpr int kWarps = 4;              // warps per CTA of the decode kernel
constexpr int kSmemBudget = 196 * 1024;
constexpr int kSchedSlots = 4;         // work-queue counter slots per plan (launch i uses i % 4)
constexpr int kSchedStride = 64;       // int32 words per slot: two 128-B lines
constexpr int kMaxSplits = 64;         // automatic splits per range (shared region or member tail);
                                       // 2 kMaxSplits records per request keep the merge on its fast path

// ---------------------------------------------------------------------------- pool
struct Request {
    std::vector<int32_t> pages;
    int32_t len = 0;
};

}  // namespace spa

// CUtensorMap is 128 bytes, 64-B aligned; kept opaque here so host files need no cuda.h.
struct spa_tmap {
    alignas(64) unsigned char bytes[128];
};

struct spa_pool {
    spa_pool_config cfg;
    void* k_pool = nullptr;
    void* v_pool = nullptr;
    bool metadata_only = true;
    int device = -1;
    int sm_count = 0;
    std::unordered_map<int64_t, spa::Request> reqs;
    int64_t next_id = 1;
    std::vector<int32_t> refcount;
    std::set<int32_t> free_set;
    spa_tmap tmap_k, tmap_v;
    spa_tmap tmap_k1;   // K pool, one 64-column chunk per box (the extend kernel's key-contiguous stages)
    // F4 (spa_pool_create_fp8): e4m3 pages, K token-major, V transposed per page with the
    // slot permutation kF8VCol; static (k_scale, v_scale) per (layer, KV head), device fp32
    bool kv_fp8 = false;
    const float* kv_scale = nullptr;
};

struct spa_plan {
    spa_pool* pool = nullptr;
    spa_plan_config cfg{};
    int mt = 1;                 // m16 tiles (warps) per team: max_rows / 16
    int teams = 4;              // teams (work-item streams with private rings) per CTA
    bool teams_auto = true;     // teams chosen by the library (teams_per_cta 0, no SPA_TEAMS)
    int kw = 2;                 // key-split warps per row tile (1: a warp takes every page of a stage)
    bool auto_rows = false;     // max_rows 0: 16- or 32-row items chosen per batch (spa_decode_plan)
    int n_teams = 0;
    int num_ctas = 0;
    // host view of the last plan
    std::vector<int32_t> host;  // header + arrays (also the upload source, pinned copy below)
    std::vector<uint32_t> slot_mask;   // planner scratch: attended slots per page id (zero between plans)
    int32_t* pinned = nullptr;
    size_t pinned_words = 0;
    void* upload_event = nullptr;  // cudaEvent_t
    bool upload_pending = false;
    // caller-owned device workspace (spa_plan_set_workspace): plan metadata, then the split
    // partials (fp32 O, then LSE), each 256-B aligned; the library never allocates device memory
    void* ws = nullptr;
    size_t ws_bytes = 0;
    size_t ws_need = 0;         // bytes the last built plan needs (also after SPA_ERR_WORKSPACE)
    bool uploaded = false;      // the last built plan is on the device (decode launches allowed)
    int32_t* d_meta = nullptr;
    float* d_part_o = nullptr;
    float* d_part_lse = nullptr;
    int generation = 0;
    spa_plan_stats stats{};
    int32_t window = 0;
    int32_t n_req = 0;
    bool merge_all_s2 = false;  // every merge subtask is a whole (row, KV head) task of 2 records
    mutable int64_t launches = 0;  // decode launches since the last spa_decode_plan (queue slot owner ids)
    unsigned long long* trace = nullptr;   // spa_debug_set_trace: timeline buffer (device), or null
    int32_t trace_cap = 0;
};

namespace spa {
constexpr int kUploadNoWorkspace = -1;   // plan_upload: workspace missing or too small
size_t plan_workspace_need(const spa_plan* P);
}  // namespace spa

struct spa_comm {
    void* nccl_comm = nullptr;
    int rank = 0, world = 1;
};

// F1 fused decode + all-gather (comm.cpp): one device allocation per rank holding n_bufs
// gathered-output buffers and a signal pad, shared with the other ranks over CUDA IPC.
struct spa_peer {
    int rank = 0, world = 1, device = 0;
    size_t buf_bytes = 0, buf_stride = 0;
    int n_bufs = 0;
    char* base = nullptr;                 // this rank's allocation (cudaMalloc)
    size_t sig_off = 0;                   // signal pad: u32[world] at base + sig_off, then the status word
    char* peer_base[8] = {};              // each rank's allocation as mapped in this process
    bool ipc_opened[8] = {};
    bool connected = false;
    uint32_t epoch = 0;                   // fused launches so far (identical on every rank)
};

namespace spa {
// kernels.cu launchers (all return cudaError_t as int)
int launch_append(const spa_pool* pool, const void* k_new, const void* v_new, int32_t T_total,
                  const std::vector<int32_t>& dst_slots, void* stream);
int launch_cow(const spa_pool* pool, int32_t src_page, int32_t dst_page, int32_t rows, void* stream);
// F4: the V^T column of page slot s (0..15).  Slots (2t, 2t+1, 2t+8, 2t+9) sit in columns
// 4t..4t+3, so one 4-B shared-memory load gives a thread its mma.m16n8k16 B fragment of PV.
#ifdef __CUDACC__
#define SPA_HD __host__ __device__
#else
#define SPA_HD
#endif
SPA_HD inline int kF8VCol(int s) { return 4 * ((s & 7) >> 1) + (s & 1) + 2 * (s >> 3); }

struct PeerLaunch {   // F1: what the decode kernel needs to fan its outputs out and meet its peers
    int rank, world;
    long long delta[8];   // byte distance from this rank's output buffer to rank k's (mapped here)
    unsigned* sig_local;
    unsigned* sig_peer[8];
    unsigned epoch;
    unsigned* status;
};
int launch_decode(const spa_plan* plan, int32_t layer, const void* q, int64_t q_sr, int64_t q_sh, void* o,
                  int64_t o_sr, int64_t o_sh, float* lse, int64_t l_sr, int64_t l_sh, float scale, void* stream,
                  const PeerLaunch* peer = nullptr);
int launch_merge_tasks(const spa_plan* P, void* o, int64_t o_sr, int64_t o_sh, float* lse, int64_t l_sr, int64_t l_sh,
                       void* stream);
int launch_merge(int32_t n_req, int32_t num_heads, int32_t head_dim, const int32_t* rec_ptr, const float* part_o,
                 const float* part_lse, void* o, int64_t o_sr, int64_t o_sh, float* lse, int64_t l_sr, int64_t l_sh,
                 int grid_hint, void* stream);
bool merge_separately(const spa_plan* P, bool fan_out);   // decode.cu: merge_mode 0 -> merge_kernel
bool decode_teams_supported(int mt, int teams, int kw);   // decode.cu: compiled (row tiles, teams/CTA, key split)
// ext.cu: the tcgen05 kernel for 128-row (extend) plans
bool ext_supported(int head_dim);
int launch_ext(const spa_plan* plan, int32_t layer, const void* q, int64_t q_sr, int64_t q_sh, void* o, int64_t o_sr,
               int64_t o_sh, float* lse, int64_t l_sr, int64_t l_sh, float scale, void* stream);
int memset_pool(spa_pool* pool);
bool make_tensor_maps(spa_pool* pool, std::string* err);
int device_sm_count(int* device_out);
int current_device();   // cudaGetDevice, or -1
spa_status check_device(const spa_pool* pool);   // pool.cpp: the calling thread's device is the pool's
const char* cuda_error_string(int err);
}  // namespace spa
