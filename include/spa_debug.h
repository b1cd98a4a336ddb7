/*
 * spa_debug.h -- read-only views of a plan's host-side arrays, for planner tests.
 *
 * The arrays are the exact int32 records uploaded to the device by spa_decode_plan.
 * Views stay valid until the next spa_decode_plan / spa_plan_destroy on the plan.
 *
 *   SPA_DBG_DESC      rows of 8: page_off, n_pages, tok_start, tok_end, member_off,
 *                     n_members, kind (bit 0: member tail, else shared; bit 2: holds a
 *                     member's newest token), group
 *                     -> keys [tok_start, tok_end) read through pages[page_off ..+n_pages)
 *   SPA_DBG_MEMBER    rows of 4: batch row, window lower bound lo, record (-1 = direct
 *                     output), reserved
 *   SPA_DBG_ITEM      rows of 2: descriptor, local KV head
 *   SPA_DBG_QUEUE     item indices in the order the persistent kernel's teams pop them
 *                     (dynamic longest-processing-time: largest first)
 *   SPA_DBG_PAGES     page ids referenced by descriptors
 *   SPA_DBG_REC_PTR   n_req + 1 offsets: partial records of batch row i
 */
#ifndef SPA_DEBUG_H_
#define SPA_DEBUG_H_

#include "spa.h"

#ifdef __cplusplus
extern "C" {
#endif

enum {
    SPA_DBG_DESC = 0,
    SPA_DBG_MEMBER = 1,
    SPA_DBG_ITEM = 2,
    SPA_DBG_QUEUE = 3,
    SPA_DBG_PAGES = 5,
    SPA_DBG_REC_PTR = 6
};

spa_status spa_plan_debug_array(const spa_plan* plan, int32_t which, const int32_t** out_data,
                                int64_t* out_len, int32_t* out_row_width);

/* Read-bandwidth probes (bench.py reports them as same-run ceilings next to the decode
 * kernel's achieved bandwidth).  Asynchronous on `stream`; time them with events.
 *   spa_debug_read_bw_ldg:   streaming 16-B loads over `bytes` of device memory at `buf`;
 *                            sink4 = 4 bytes of device scratch.
 *   spa_debug_pool_read_tma: the decode kernel's TMA/mbarrier pipeline without the math,
 *                            over every page and KV head of layers [0, layers) of both pools;
 *                            mode 0: 2-D 64x16 boxes (as the decode kernel), 1: 3-D
 *                            64x(d/64)x16 boxes, 2: 1-D cp.async.bulk of each 4 KB page-head.
 * Bytes read by the TMA probe: layers * (num_pages / 2 * 2) * Hkv * page_size * d * 2 * 2. */
spa_status spa_debug_read_bw_ldg(const void* buf, size_t bytes, void* sink4, void* stream);
spa_status spa_debug_pool_read_tma(const spa_pool* pool, int32_t layers, int32_t mode, void* stream);

/* Timeline trace of the decode kernel (performance analysis only).  While set, every
 * spa_decode_attention launch of `plan` writes, per warp (CTA-major), up to `cap` events of
 * 2 uint64 each into the caller-owned device buffer `buf`
 * (num_ctas * warps_per_cta * cap * 16 bytes, from spa_debug_plan_geometry):
 *   word 0: %globaltimer (ns, device-wide)
 *   word 1: (tag << 56) | (item or subtask & 0xffffff) << 32 | (clock64 & 0xffffffff)
 * tags: 1 kernel entry, 2 item start (first stage landed), 3 item end (output written),
 *       8 item's partial records counted in (in-kernel merge), 4 tail-merge subtask popped,
 *       7 its records complete, 5 subtask merged, 6 warp leaves the kernel.
 * Slots past a warp's last event are left untouched (zero the buffer first).  buf = NULL
 * turns tracing off.  Each launch overwrites the buffer. */
spa_status spa_debug_set_trace(spa_plan* plan, void* buf, int32_t cap);
spa_status spa_debug_plan_geometry(const spa_plan* plan, int32_t* out_num_ctas, int32_t* out_teams_per_cta,
                                   int32_t* out_warps_per_cta);

/* tcgen05 self-test (one CTA): q [128][128], k [32][128], v [32][128] bf16 row-major (device);
 * out_s [128][32] = q k^T (fp32), out_o [128][128] = bf16(out_s) v (fp32).  Exercises the
 * shared-memory / instruction descriptors and tensor-memory layouts of the extend kernel. */
spa_status spa_debug_umma_selftest(const void* q, const void* k, const void* v, float* out_s, float* out_o,
                                   void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPA_DEBUG_H_ */
