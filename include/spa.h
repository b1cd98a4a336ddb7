/*
 * spa.h -- C ABI of the shared-prefix paged GQA decode-attention step under SPAgent's
 * action speculation (arXiv 2511.20048), B200 / sm_100a.
 *
 * What the calls compute, and where it is defined
 * ------------------------------------------------
 * SPAgent runs k short speculative requests beside each agent's main reasoning request
 * (Sec. III-B/C), so one engine decode iteration serves
 * N = N_m + N_s + N_a requests (Table I) and costs T_h(emptyset, N)
 * (Eq. 3).  Every speculative sample is drawn from the agent context
 * c_i ("all samples of one request share the same prefix"; c_i defined at
 * PAPER.md:135).  This library is the attention part of that decode iteration: paged
 * KV, copy-free forks of c_i, and per-layer decode attention that reads each shared
 * prefix page ONCE per (KV head, request group).  The paper itself never writes
 * attention down; the readings used for everything it leaves open are numbered in
 * DESIGN.md Sec. 3 ("reading #k").
 *
 * Conventions
 *  - All device memory named in these signatures is caller-owned (PyTorch allocates it)
 *    unless stated otherwise: the KV pools, q/o/lse, new K/V and the plan workspace
 *    (spa_plan_set_workspace) -- the plan path never calls cudaMalloc/cudaFree.  The library
 *    owns host metadata (request table, page tables, refcounts, free set, plans, a plan's
 *    pinned host staging buffer).  Exceptions, stated at their calls: the F1 peer regions
 *    (spa_peer_create, shared over CUDA IPC) and NCCL's own buffers.
 *  - bf16 means IEEE bfloat16 bit patterns (uint16).  Strides are in ELEMENTS.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Device work is
 *    stream-ordered; host metadata changes take effect when the call returns.
 *  - Threading: one host thread per pool (the caller serialises calls on a pool and on
 *    its plans).  spa_last_error() is thread-local.
 *  - Every call returns a spa_status; no exception ever crosses the ABI.  Host metadata
 *    mutations are all-or-nothing: on any error nothing observable changed.
 *  - Asynchronous kernel faults surface as SPA_ERR_CUDA on a later call.
 */
#ifndef SPA_H_
#define SPA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPA_ABI_VERSION 1

typedef enum spa_status {
    SPA_OK = 0,
    SPA_ERR_INVALID_ARG = 1,   /* bad shape/argument, duplicate request in a batch, prefix_len > length, empty request in a decode batch */
    SPA_ERR_NO_PAGES = 2,      /* the pool has too few free pages; nothing was changed */
    SPA_ERR_BAD_REQUEST = 3,   /* unknown or already-freed request id */
    SPA_ERR_CUDA = 4,          /* a CUDA runtime/driver call or kernel failed (see spa_last_error) */
    SPA_ERR_NCCL = 5,          /* NCCL could not be loaded or a collective failed */
    SPA_ERR_UNSUPPORTED = 6,   /* configuration the kernels do not implement (head_dim, page_size, ...) */
    SPA_ERR_NO_DEVICE = 7,     /* device work requested from a metadata-only pool */
    SPA_ERR_WORKSPACE = 8      /* the plan's caller-owned workspace is missing or too small
                                  (spa_plan_workspace_size gives the bytes needed) */
} spa_status;

typedef int64_t spa_req;                 /* request id: 1, 2, 3, ... never reused (reading #4) */
typedef struct spa_pool spa_pool;
typedef struct spa_plan spa_plan;
typedef struct spa_comm spa_comm;
typedef struct spa_peer spa_peer;

/* ---------------------------------------------------------------------------------
 * Paged KV pool
 * --------------------------------------------------------------------------------- */
typedef struct spa_pool_config {
    int32_t num_layers;     /* L                                                       */
    int32_t num_q_heads;    /* Hq held by this process (its shard when head-sharded)   */
    int32_t num_kv_heads;   /* Hkv held by this process; Hq % Hkv == 0, G = Hq / Hkv   */
    int32_t head_dim;       /* d: 64 or 128                                            */
    int32_t page_size;      /* tokens per page; the decode kernels require 16          */
    int32_t num_pages;      /* pages in the pool                                       */
} spa_pool_config;

/* Create a pool over caller-owned device memory.
 *   k_pool, v_pool: device, bf16 [L][num_pages][Hkv][page_size][d] each, 128-B aligned;
 *                   the SAME page id is used in every layer.  The library zero-fills
 *                   both at creation, so never-written slots of a page hold finite
 *                   values (masked keys are then multiplied by an exact 0).
 *   k_pool = v_pool = NULL creates a METADATA-ONLY pool: every host-side rule below
 *   applies, device work is skipped (used by CPU tests of the allocator and planner).
 * Errors: INVALID_ARG (non-positive sizes, Hq % Hkv), UNSUPPORTED (d not 64/128 or
 * page_size != 16 with device memory), CUDA. */
spa_status spa_pool_create(const spa_pool_config* cfg, void* k_pool, void* v_pool, spa_pool** out);
spa_status spa_pool_destroy(spa_pool* pool);

/* F4: a pool of FP8 (e4m3) KV pages -- half the bytes a decode
 * step reads.  Same paging rules and calls as spa_pool_create; head_dim must be 128.
 *   kv_scale: caller-owned device fp32 [L][Hkv][2] = (k_scale, v_scale) per layer and KV
 *     head, static (reading F4-a: a page of an append-only stream cannot fix its
 *     scale before it fills).  spa_kv_append still takes bf16 K/V and quantises on the way
 *     in:  code = e4m3 round-to-nearest-even, saturating at +-448, of fp32(x) / scale
 *     (IEEE fp32 division; oracle/fp8.py), and decode reads K = k_scale * code,
 *     V = v_scale * code.
 *   kv_pool: ONE caller-owned buffer, e4m3 [L][num_pages][Hkv][2][2048 B], 128-byte
 *     aligned: per (page, head) the K block [16 slots][128 ch] (token-major rows, as bf16
 *     pools) followed by the V block TRANSPOSED, [128 ch][16 slots], page slot s stored in
 *     column 4((s mod 8) div 2) + (s mod 2) + 2(s div 8) -- so a page-head's K and V are one
 *     4-KB TMA box and the decode kernel's f16 MMA fragments are single 4-byte loads.
 *     num_layers * num_pages * Hkv * 32 < 2^31.  (NULL: a metadata-only pool.)
 * Decode plans over it must use max_rows <= 64 (the tcgen05 extend kernel is bf16 only:
 * CUDA error "operation not supported" at launch otherwise). */
spa_status spa_pool_create_fp8(const spa_pool_config* cfg, void* kv_pool, const float* kv_scale, spa_pool** out);

/* a1: a new, empty request (length 0, no pages). */
spa_status spa_kv_alloc(spa_pool* pool, spa_req* out_req);

/* a2: append n_new[i] tokens to reqs[i], i < n_req, for ALL layers at once.
 *   reqs, n_new: host arrays.  A request may appear at most once (INVALID_ARG).
 *   k_new, v_new: device bf16 [L][T][Hkv][d], T = sum(n_new), tokens ordered request
 *   by request (in reqs order) then by position.  Paging policy (reading #4): request
 *   by request, token by token, a page is taken (lowest free id) exactly when
 *   length % page_size == 0.  If the pages needed exceed the free pages: NO_PAGES and
 *   nothing changes.  The query of a decode step attends to the key appended here
 *   (append-then-attend, reading #8). */
spa_status spa_kv_append(spa_pool* pool, int32_t n_req, const spa_req* reqs, const int32_t* n_new,
                         const void* k_new, const void* v_new, void* stream);

/* a3: copy-free fork of the first prefix_len tokens of `parent` (the k
 * speculative samples of PAPER.md:189/:198 reading context c_i).  The child shares
 * parent pages [0, prefix_len / page_size) (refcount + 1); if prefix_len % page_size
 * != 0 one fresh page receives a device copy of the parent's partial page, slots
 * [0, prefix_len % page_size), all layers (copy-on-write at fork time, reading #3).
 * 0 <= prefix_len <= length(parent), else INVALID_ARG. */
spa_status spa_fork_request(spa_pool* pool, spa_req parent, int32_t prefix_len, spa_req* out_child,
                            void* stream);

/* a8: release a request: refcount - 1 on each of its pages; pages reaching 0 return to
 * the free set.  The id is retired (later use: BAD_REQUEST). */
spa_status spa_kv_free(spa_pool* pool, spa_req req);

/* F4 (ring-buffer storage for sliding-window layers): release the
 * pages neither the current query nor any later query of reqs[i] can read under a sliding
 * window of `window` tokens (reading #9: a query at position q reads keys (q - window, q]).
 * Under append-then-attend (reading #8) the current step's query is the last appended
 * token, at position n - 1 for the current length n, so page p (keys [16p, 16p + 16)) is
 * released when 16p + 16 <= n - window: its refcount drops, at 0 it returns to the free
 * set, and the request's page-table entry becomes -1 (lengths and later entries are
 * unchanged).  Intended order per step: spa_kv_append, spa_kv_release_window(window),
 * spa_decode_plan(window).  For a pool that holds only windowed (local) layers this bounds
 * each request to about window/16 + 2 pages.  Host only.  Errors: window <= 0,
 * unknown request; later, a plan whose window reaches a released page (INVALID_ARG) and
 * a fork whose partial page was released (INVALID_ARG).  Forks copy released entries as -1. */
spa_status spa_kv_release_window(spa_pool* pool, int32_t n_req, const spa_req* reqs, int32_t window);

/* Inspection (bit-exact tests).  out_pages receives min(cap, n_pages) page ids. */
spa_status spa_kv_page_table(const spa_pool* pool, spa_req req, int32_t* out_pages, int32_t cap,
                             int32_t* out_n_pages, int32_t* out_len);
/* out_refcount: host int32[num_pages]. */
spa_status spa_pool_refcounts(const spa_pool* pool, int32_t* out_refcount);
/* Free page ids in increasing order; out_pages receives min(cap, n) of them. */
spa_status spa_pool_free_pages(const spa_pool* pool, int32_t* out_pages, int32_t cap, int32_t* out_n);

/* ---------------------------------------------------------------------------------
 * Step plan (a4): built once per decode step on the host, uploaded once, reused by
 * every layer.  Groups are requests that hold a resident page in common (forks of one
 * context, and forks of those).  Within a group, each maximal run of page indices over
 * which the same set of requests holds the same pages is one range (a prefix tree:
 * c_i shared by the main request and every speculative fork, a speculative prompt shared
 * by the k samples forked from it, then private tails; reading #18).  Work items are
 * (KV head, range split); each shared page is read once per (KV head, range) by one
 * CTA-team holding all R = members x G query rows (ranges with more than max_rows rows
 * are cut into chunks of max_rows rows that each read the pages).
 * --------------------------------------------------------------------------------- */
typedef struct spa_plan_config {
    int32_t sharing;        /* 1: group by shared prefix (default); 0: every request alone (control) */
    int32_t max_rows;       /* 16, 32, 64 or 128: query rows (requests x G) per work item; a range
                               with more rows is cut into chunks that each read its pages.
                               0 (default) = auto: per batch, 32 when ranges of more than 16
                               rows (k = 3 forks of a G = 5 context: 20 rows) hold > 30 % of the
                               pages, else 16 (G > 16: 32).  64: extend batches, one team;
                               128: the tcgen05 extend kernel (bf16, head_dim 128)              */
    int32_t split_pages;    /* max pages per split; 0 = auto (balance over the persistent grid)  */
    int32_t num_ctas;       /* persistent grid size; 0 = number of SMs                            */
    int32_t merge_mode;     /* where split partials are merged (spa_merge_splits semantics always):
                               0 (default): the library's choice -- inside the decode kernel, by
                                 teams that found the work queue empty (tail phase); fp8 pools
                                 decoded by one-warp teams (16-row items) without a peer
                                 fan-out: by the merge_kernel launch of mode 2 (measured faster);
                               1: inside the decode kernel, by the last item of each (request, KV
                                 head) to finish;
                               2: by a separate merge_kernel launch (programmatic dependent launch) */
    int32_t teams_per_cta;  /* work-item streams per CTA, each with a private shared-memory ring:
                               4 (default for max_rows 16): 4 x 3-stage rings; 2: 2 x 6; 1: 1 x 12
                               (deeper rings stream faster per item: small batches).  32-row
                               items use 4 teams of 2 warps (one per 16-row tile, each taking
                               every page of a stage).  fp8 pools, 16-row items: 0 selects 8
                               one-warp teams (each warp its own 3-stage ring of 2 pages), 12
                               (2-stage rings) for windowed plans; 1, 2 or 4 keep the
                               key-split pairs.  Must be 0 with max_rows 0.                      */
} spa_plan_config;

/* cfg may be NULL (defaults).  The plan keeps a pointer to `pool`. */
spa_status spa_plan_create(spa_pool* pool, const spa_plan_config* cfg, spa_plan** out);
spa_status spa_plan_destroy(spa_plan* plan);

/* Caller-owned plan workspace (all device memory is caller-owned).
 * Device memory, 256-B aligned, that holds the uploaded plan (queue, descriptors, page list,
 * merge counters) followed by the split partials (fp32 O [records][Hq][d], fp32 LSE).  Set
 * it before planning; spa_decode_plan / spa_extend_plan never allocate device memory.  A
 * plan that needs more than `bytes` fails with SPA_ERR_WORKSPACE (nothing is enqueued and
 * decode launches are refused until a plan succeeds); spa_plan_workspace_size then returns
 * the bytes that plan needs (after any plan call: the last plan's need), so the caller can
 * grow the buffer and plan again.  Changing the pointer invalidates the uploaded plan (plan
 * again) and bumps spa_plan_stats.generation (CUDA graphs captured over the old pointer are
 * stale).  The workspace must stay allocated while launches that use it are in flight.
 * Graph capture: a plan call on a capturing stream records the upload as a memcpy node
 * (from the plan's pinned staging buffer, which must already be large enough: plan the
 * same batch once before capturing), so replaying plan + decode launches is consistent. */
spa_status spa_plan_set_workspace(spa_plan* plan, void* workspace, size_t bytes);
spa_status spa_plan_workspace_size(const spa_plan* plan, size_t* out_bytes);

/* (Re)plan a decode batch: reqs[0..n_req) (host), all of length >= 1, no duplicates.
 *   window > 0: sliding window, request r attends to keys [max(0, n_r - window), n_r)
 *   (reading #9); window <= 0: full attention.  Batch row i of q/o/lse below is reqs[i].
 *   The plan's metadata is uploaded into the caller's workspace on `stream` (above);
 *   SPA_ERR_WORKSPACE if it does not fit. */
spa_status spa_decode_plan(spa_plan* plan, int32_t n_req, const spa_req* reqs, int32_t window, void* stream);

/* (Re)plan an EXTEND batch (the prefill of a speculative prompt
 * over its shared context): request i contributes n_query[i] >= 1 query
 * rows, its LAST n_query[i] tokens (already appended), so row token t < n_query[i] sits at
 * position p = n_i - n_query[i] + t and attends causally to keys [max(0, p + 1 - window),
 * p + 1) (window <= 0: [0, p + 1)).  Rows are numbered request-major, token-minor (the
 * packing of spa_kv_append's k_new/v_new); q/o/lse of spa_decode_attention are indexed by
 * this row number.  n_query = NULL means 1 for every request: spa_decode_plan.  Rows of
 * the requests sharing a prefix are one group (the shared pages are read once per KV head
 * and sub-group of max_rows / G rows); a request's own rows share its tail range. */
spa_status spa_extend_plan(spa_plan* plan, int32_t n_req, const spa_req* reqs, const int32_t* n_query,
                           int32_t window, void* stream);

typedef struct spa_plan_stats {
    int32_t n_req /* query rows */, n_groups, n_desc, n_items, n_records, n_teams, rows_max, generation;
    int64_t unique_tokens;    /* key tokens the work descriptors read, per KV head (a class cut
                                 into max_rows chunks counts once per chunk)                     */
    int64_t unshared_tokens;  /* sum over query rows of attended keys, per KV head (no sharing)  */
    int64_t pages_read;       /* pages read per KV head (page-granular, incl. partial pages)     */
    int64_t alg_tokens;       /* distinct (page, slot) keys any row attends to, per KV head: the
                                 algorithmic lower bound of SURVEY.md Sec. 8(d) (B_alg / (Hkv d 4)) */
} spa_plan_stats;
spa_status spa_plan_get_stats(const spa_plan* plan, spa_plan_stats* out);

/* a5 (+a6): decode attention of one layer for the planned batch.
 *   q:   device bf16, row i head h at q[i*q_stride_req + h*q_stride_head + c], c < d
 *   o:   device bf16, same indexing with o strides (head-major or request-major allowed)
 *   lse: device fp32 natural-log LSE of the scaled logits (reading #7) at
 *        lse[i*lse_stride_req + h*lse_stride_head], or NULL
 *   scale: softmax scale (reading #6; 1/sqrt(d) for Qwen2.5, 168^-1/2 for Gemma-3).
 * O is rounded to bf16 (RNE) from fp32 (reading #10).  If the plan split any request,
 * its fp32 partials are merged on the same stream (spa_merge_splits semantics). */
spa_status spa_decode_attention(const spa_plan* plan, int32_t layer,
                                const void* q, int64_t q_stride_req, int64_t q_stride_head,
                                void* o, int64_t o_stride_req, int64_t o_stride_head,
                                float* lse, int64_t lse_stride_req, int64_t lse_stride_head,
                                float scale, void* stream);

/* a6: split-KV partial-LSE merge (north_star; oracle/attention.py merge_partials).
 * For request i < n_req and head h < num_heads, partial records
 * s in [rec_ptr[i], rec_ptr[i+1]) hold part_o[(s*num_heads + h)*head_dim + c] (fp32) and
 * part_lse[s*num_heads + h] (natural log; -inf = empty split):
 *     LSE = m + ln sum_{s live} exp(LSE_s - m),  O = sum_s exp(LSE_s - LSE) O_s
 * all partials -inf -> O = 0, LSE = -inf.  Requests with an EMPTY record range are not
 * written (their output was produced directly).  All pointers are device pointers;
 * rec_ptr is int32[n_req + 1].  o is bf16 (RNE), lse may be NULL. */
spa_status spa_merge_splits(int32_t n_req, int32_t num_heads, int32_t head_dim, const int32_t* rec_ptr,
                            const float* part_o, const float* part_lse,
                            void* o, int64_t o_stride_req, int64_t o_stride_head,
                            float* lse, int64_t lse_stride_req, int64_t lse_stride_head, void* stream);

/* ---------------------------------------------------------------------------------
 * Multi-GPU: KV-head sharding with an NCCL all-gather of head outputs (a7).
 * Rank r of n holds KV heads [r Hkv/n, (r+1) Hkv/n) and q heads [r Hq/n, (r+1) Hq/n) in
 * its own pool (num_kv_heads / num_q_heads of its spa_pool_config are the LOCAL counts).
 * Every rank replays the same allocator calls, so page tables and plans are identical
 * without communication.  NCCL (libnccl.so.2) is loaded at spa_comm_create.
 * --------------------------------------------------------------------------------- */
spa_status spa_nccl_unique_id(void* out_id /* 128 bytes (ncclUniqueId) */);
/* Collective over `world` ranks; the calling thread's current CUDA device is used. */
spa_status spa_comm_create(const void* unique_id, int32_t rank, int32_t world, spa_comm** out);
spa_status spa_comm_destroy(spa_comm* comm);
/* Decode this rank's heads straight into its slot of o_gathered, then all-gather in place.
 *   q_local:     bf16 [N][Hq_local][d] with the given strides
 *   o_gathered:  bf16 [world][Hq_local][N][d] contiguous (= [Hq][N][d], head-major)
 *   lse_gathered: fp32 [world][Hq_local][N] or NULL */
spa_status spa_decode_attention_sharded(const spa_plan* plan, spa_comm* comm, int32_t layer,
                                        const void* q_local, int64_t q_stride_req, int64_t q_stride_head,
                                        void* o_gathered, float* lse_gathered, float scale, void* stream);

/* ---------------------------------------------------------------------------------
 * F1: fused decode + all-gather over NVLink peer memory.
 * The decode kernel (a5, with its in-kernel split merge a6) stores every output element
 * of this rank's heads straight into the same offset of EVERY rank's gathered buffer
 * (peer stores through CUDA IPC mappings), and the last CTA to finish releases a flag
 * into each peer's signal pad and waits for theirs -- the all-gather (a7) without an
 * NCCL launch, its transfer overlapping the kernel's math item by item.  The paper's
 * engine shards attention by tensor parallelism over NVLink GPUs.
 *
 * Memory: spa_peer_create allocates ONE device region per rank (library-owned, freed by
 * spa_peer_destroy): n_bufs buffers of buf_bytes (256-B aligned) + a signal pad.  Buffer
 * b of every rank holds, for a decode over N requests with Hq_local = Hq / world heads:
 *     O   bf16 [world][Hq_local][N][d]   at offset 0          (= [Hq][N][d], head-major)
 *     LSE fp32 [world][Hq_local][N]      at offset align256(world Hq_local N d 2)
 * Wiring: spa_peer_ipc_handle exports the region (64 bytes); the caller all-gathers the
 * handles (rank order) and passes them to spa_peer_connect, which opens the others.
 * spa_peer_connect_local wires `world` peers created in ONE process on ONE device
 * (virtual ranks: tests of the protocol on a single GPU; they must run on different
 * streams, since each rank's launch waits for the others').
 * Ordering contract: every rank makes the same sequence of fused calls (the epoch of a
 * call is its index in that sequence).  Any rank's call k+1 may start writing into every
 * rank's buffer as soon as ALL ranks have finished call k.  So a buffer that call k+1
 * writes must no longer be read on any rank once that rank's call k is done: e.g.
 * alternate two buffers and consume call k-1's output before issuing call k (stream
 * order), as a model's O projection between layers does.
 * Only decode plans (max_rows <= 64) with merge_mode 0 or 1 are supported
 * (SPA_ERR_UNSUPPORTED otherwise).  If a peer does not arrive within 20 s the kernel
 * gives up, and spa_peer_status reports 1 (0 = healthy). */
spa_status spa_peer_create(int32_t rank, int32_t world, size_t buf_bytes, int32_t n_bufs, spa_peer** out);
spa_status spa_peer_ipc_handle(const spa_peer* peer, void* out_handle /* 64 bytes */);
spa_status spa_peer_connect(spa_peer* peer, const void* handles /* world x 64 bytes, rank order */);
spa_status spa_peer_connect_local(spa_peer* const* peers, int32_t world);
spa_status spa_peer_buffer(const spa_peer* peer, int32_t buf_idx, void** out_ptr);
spa_status spa_peer_status(const spa_peer* peer, int32_t* out_status);   /* synchronises the device */
spa_status spa_peer_destroy(spa_peer* peer);
/* Decode this rank's heads into buffer buf_idx of every rank (O, and LSE if with_lse),
 * then meet the peers.  On return (stream-ordered) buffer buf_idx of this rank holds the
 * gathered O / LSE of all ranks.  q_local: bf16 [N][Hq_local][d] with the given strides. */
spa_status spa_decode_attention_fused_gather(const spa_plan* plan, spa_peer* peer, int32_t layer,
                                             const void* q_local, int64_t q_stride_req, int64_t q_stride_head,
                                             int32_t buf_idx, int32_t with_lse, float scale, void* stream);

/* Library info */
int32_t spa_abi_version(void);
const char* spa_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SPA_H_ */
