/*
 * spa_debug.h -- read-only views of a plan's host-side arrays, for planner tests.
 *
 * The arrays are the exact int32 records uploaded to the device by spa_decode_plan.
 * Views stay valid until the next spa_decode_plan / spa_plan_destroy on the plan.
 *
 *   SPA_DBG_DESC      rows of 8: page_off, n_pages, tok_start, tok_end, member_off,
 *                     n_members, kind (0 shared, 1 tail), group
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

#ifdef __cplusplus
}
#endif
#endif /* SPA_DEBUG_H_ */
