// a5: the shared-prefix paged GQA decode-attention kernel (sm_100a) and its launcher.
//
// Persistent grid: one CTA of 8 warps per SM.  A TEAM of MT x KW warps owns a private
// shared-memory ring of NS stages; each stage holds PPS pages of K and V for one KV head,
// brought in by ONE 3-D TMA box per (page, head) and tensor, completing on an mbarrier.
// Teams pop work items (descriptor, KV head) from a dynamic longest-first queue.  An item
// carries every query row of a request group (R = members x G <= 16 MT), so the pages of
// a shared agent context c_i are read from HBM once per (KV head, group) for the main
// request and all its speculative forks (north_star).
//   wt (0..MT-1)  which 16-row tile of the item's query rows a warp computes
//   wk (0..KW-1)  which pages of each stage a warp consumes (page j -> warp j % KW); the KW
//                 partial softmax states of a row tile are combined through shared memory
//                 at the end of the item (flash-decoding inside the team).
// QK^T and PV are mma.sync.m16n8k16 bf16 tiles (fp32 accumulate) fed by ldmatrix from the
// 128-B-swizzled tiles; the online softmax runs in the log2 domain with lazy rescaling.
// Each item writes either the final O (bf16) / LSE (fp32) of its rows or an fp32 partial
// record; partials are merged by the merge kernel (or in-kernel, fused_merge = 1 / 2).
// F8 = true (S8(f) F4, include/spa.h spa_pool_create_fp8): e4m3 pages, one 4-KB box per
// page-head (K rows then the transposed V block), f16 MMAs fed by 4-byte fragment loads
// and cvt.rn.f16x2.e4m3x2; the scales fold into the logit scale and 1/l.
// DecodeParams::fan (S8(f) F1, spa_decode_attention_fused_gather): every output store also
// goes to each peer rank's gathered buffer, and the last CTA meets the peers on flags.
#include <cstdlib>

#include "device_util.cuh"
#include "spa_internal.h"

namespace spa {

struct DecodeParams {
    const int32_t* meta;
    const __nv_bfloat16* q;
    long long q_sr, q_sh;
    __nv_bfloat16* o;
    long long o_sr, o_sh;
    float* lse;
    long long l_sr, l_sh;
    float* part_o;
    float* part_lse;
    float scale_log2;
    int layer_row_base;  // layer * num_pages * Hkv * 16
    int num_q_heads, group_size, num_kv_heads;
    int fused_merge;     // 0 merge kernel, 1 last arriver merges, 2 tail phase merges
    int launch;          // launch id since the plan was built: selects/owns a work-queue slot
    unsigned long long* trace;   // spa_debug_set_trace timeline (null: off)
    int trace_cap;
    unsigned poll_min, poll_max;   // tail-merge polling backoff (ns)
    // F1 fused all-gather (fan.n = world > 1): outputs also go to every peer's gathered
    // buffer; the last CTA to finish signals the peers and waits for theirs
    OutFan fan;
    int rank;
    unsigned epoch;
    unsigned* sig_local;               // this rank's signal pad: [world] u32, written by peers
    unsigned* sig_peer[kMaxPeers];     // peer k's signal pad as mapped here
    unsigned* status;                  // set to 1 if the peer wait timed out
    // F4 fp8 pages: (k_scale, v_scale) per (layer, KV head)
    const float* kv_scale;
    int layer;
};

// A popped work item as the producer hands it to its team (shared memory): the item and
// the descriptor fields the consumers need, so they do not re-read them from global memory.
struct TeamItem {
    int it, kv_head, n_pages, tok_start, tok_end, member_off, n_members, n_main;   // pages >= n_main: folded tails
};

#ifndef SPA_QK_CHAINS
#define SPA_QK_CHAINS 1
#endif
constexpr int kQkChains = SPA_QK_CHAINS;   // independent HMMA accumulation chains for QK^T

constexpr int kSmemMax = 232448;   // 227 KB: the sm_100 per-block dynamic shared memory limit

template <int D, int MT, int PPS, int TEAMS_, bool F8 = false, int KW_ = 2>
struct DecodeCfg {
    static constexpr int KW = KW_;                        // key-split warps per row tile (1 or 2)
    static constexpr int TEAM_WARPS = MT * KW;
    static constexpr int TEAMS = TEAMS_;                  // teams (independent rings) per CTA
    static constexpr int WARPS = TEAMS * TEAM_WARPS;
    static constexpr int PAGE_BYTES = kPageSize * D * (F8 ? 1 : 2);  // K (or V) of one page, one head
    static constexpr int STAGE_BYTES = PPS * 2 * PAGE_BYTES;
    // per (team, row tile): column-half exchange [2][16][D/2] fp32 + (m, l) [2][16][2]
    // (KW = 1: a warp holds a row tile's whole state, nothing to exchange)
    static constexpr int COMB_BYTES = KW == 2 ? TEAMS * MT * (2 * 16 * (D / 2) * 4 + 2 * 16 * 2 * 4) : 0;
    // barriers (full + empty), the team mailbox and the popped-item queue, for n stages
    static constexpr int misc(int n) { return TEAMS * n * 2 * 8 + TEAMS * 4 + TEAMS * (n + 2) * 32 + 16; }
    static constexpr int max_stages() {
        int n = 1;
        while (1024 + (n + 1) * TEAMS * STAGE_BYTES + misc(n + 1) + COMB_BYTES <= kSmemMax) ++n;
        return n;
    }
    static constexpr int NS = max_stages();
    static constexpr int MISC_BYTES = misc(NS);
    static constexpr int RING_BYTES = TEAMS * NS * STAGE_BYTES;
    static constexpr int QN = NS + 2;                     // popped-item queue entries per team
    static constexpr int OFF_BARS = RING_BYTES;
    static constexpr int OFF_SLOT = OFF_BARS + TEAMS * NS * 2 * 8;
    static constexpr int OFF_TQ = OFF_SLOT + TEAMS * 4;
    static constexpr int OFF_COMB = (OFF_TQ + TEAMS * QN * 32 + 15) & ~15;
    static constexpr int SMEM = 1024 + OFF_COMB + COMB_BYTES;
    static_assert(NS >= 2 && (TEAMS < 4 || NS >= 3 || (KW == 1 && TEAMS > 8)),
                  "pipeline needs >= 2 stages (3 with 4 key-split teams; 12 one-warp teams: 2)");
    static_assert(PPS % KW == 0, "each key-split warp takes whole pages");
    static_assert(KW == 1 || KW == 2, "one or two key-split warps per row tile");
    static_assert(OFF_COMB - OFF_BARS <= MISC_BYTES, "misc shared-memory region too small");
    static_assert(SMEM <= kSmemMax, "shared memory over the sm_100 limit");
};

template <int D, int MT, int PPS, int TEAMS, bool F8, int KW_>
__global__ void __launch_bounds__(DecodeCfg<D, MT, PPS, TEAMS, F8, KW_>::WARPS * 32, 1)
    decode_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                  const __grid_constant__ DecodeParams p) {
    using C = DecodeCfg<D, MT, PPS, TEAMS, F8, KW_>;
    static_assert(!F8 || D == 128, "fp8 pages: d = 128");
    constexpr int KW = C::KW;
    constexpr int JW = PPS / KW;   // pages per warp per stage
    constexpr int KS = D / 16;     // k16 steps over the head dimension
    constexpr int NT = D / 8;      // n8 tiles of the output
    constexpr int NTH = NT / 2;    // n8 tiles per column half
    extern __shared__ uint8_t smem_raw[];
    // 1024-B aligned by pointer arithmetic on the shared array (not through an integer cast),
    // so the compiler keeps the shared address space: LDS/STS instead of generic LD/ST
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);

    const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0);   // provably warp-uniform
    const int lane = threadIdx.x & 31;
    const int team = warp / C::TEAM_WARPS;
    const int tw = warp - team * C::TEAM_WARPS;
    const int wt = tw / KW, wk = tw - (tw / KW) * KW;
    const bool producer = tw == 0;
    const uint32_t ring = smem_u32(smem) + team * C::NS * C::STAGE_BYTES;
    const uint32_t bars = smem_u32(smem) + C::OFF_BARS;
    auto full_bar = [&](int s) { return bars + (team * C::NS + s) * 8; };
    auto empty_bar = [&](int s) { return bars + (C::TEAMS * C::NS + team * C::NS + s) * 8; };
    uint32_t* team_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_SLOT) + team;
    TeamItem* tq = reinterpret_cast<TeamItem*>(smem + C::OFF_TQ) + team * C::QN;
    float* comb = reinterpret_cast<float*>(smem + C::OFF_COMB) + (team * MT + wt) * (2 * 16 * (D / 2) + 2 * 16 * 2);
    float* ml = comb + 2 * 16 * (D / 2);
    auto team_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(C::TEAM_WARPS * 32) : "memory"); };
    auto pair_sync = [&]() {
        asm volatile("bar.sync %0, %1;" ::"r"(1 + C::TEAMS + team * MT + wt), "r"(KW * 32) : "memory");
    };

    if (threadIdx.x == 0) {
        for (int i = 0; i < C::TEAMS * C::NS; ++i) {
            mbar_init(bars + i * 8, 1);
            mbar_init(bars + (C::TEAMS * C::NS + i) * 8, C::TEAM_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // Programmatic dependent launch: this kernel may start while the previous kernel on the
    // stream (the previous layer's decode / merge) drains.  Until griddepcontrol.wait it
    // only reads what earlier stream work wrote (plan, KV pages other than the newest token
    // of each request) and its own layer's queue counters; queries, outputs, partials and
    // merge counters are touched after the wait.
    asm volatile("griddepcontrol.launch_dependents;");

    // timeline trace (spa_debug_set_trace): lane 0 of every warp records events
    unsigned long long* trace =
        p.trace ? p.trace + 2ull * (blockIdx.x * C::WARPS + warp) * p.trace_cap : nullptr;
    int tr_n = 0;
    auto tr = [&](unsigned long long tag, int id) {
        if (trace && lane == 0 && tr_n < p.trace_cap) {
            unsigned long long gt, ck;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(ck));
            trace[2 * tr_n] = gt;
            trace[2 * tr_n + 1] = (tag << 56) | ((unsigned long long)(id & 0xffffff) << 32) | (ck & 0xffffffffull);
            ++tr_n;
        }
    };
    tr(1, 0);

    const int32_t* meta = p.meta;
    const QItem* qitems = reinterpret_cast<const QItem*>(meta + meta[H_OFF_QITEM]);
    const Member* mems = reinterpret_cast<const Member*>(meta + meta[H_OFF_MEMBER]);

    const int32_t* pages = meta + meta[H_OFF_PAGES];
    const int32_t* rec_ptr = meta + meta[H_OFF_REC_PTR];
    int32_t* counters = const_cast<int32_t*>(meta) + meta[H_OFF_COUNTERS];
    int32_t* sched = const_cast<int32_t*>(meta) + meta[H_OFF_SCHED] + kSchedStride * (p.launch % kSchedSlots);
    const int n_items = meta[H_N_ITEMS];
    const int G = p.group_size, Hq = p.num_q_heads, Hkv = p.num_kv_heads;
    const OutFan* fan = p.fan.n > 1 ? &p.fan : nullptr;
    uint64_t policy = 0;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));

    // ---- producer (warp tw == 0 of the team, warp-collective; lane 0 issues): pops items
    //      from the dynamic queue and streams their stages NS ahead.  Page ids come from a
    //      two-block register cache (lane i holds page base+i and base+32+i) so the global
    //      page-list loads stay off the critical path.  TMA operands are broadcast from
    //      lane 0 (warp-uniform).  Queue empty: publish -1, complete the barrier without data.
    int p_item = -1, p_st = 0, p_n = 0;
    bool p_done = false, p_waited = false;
    int p_kv = 0, p_npages = 0, p_off = 0, p_nmain = 0, p_kind = 0;
    int pid_base = 0, pid_cur = 0, pid_next = 0;
    int q_ahead = -1;   // lane 0 of the producer: queue position reserved ~2 stages before it is needed
    auto issue_next = [&](int slot) {
        if (p_done) return;
        if (p_item < 0) {
            int qi = 0;
            if (lane == 0) {
                if (p_n == 0)   // the slot is ours once launch - kSchedSlots rewound it (rarely waits)
                    for (unsigned ns = 64; ld_acquire_gpu(sched + 3) != p.launch; ns = min(ns * 2, 1024u))
                        __nanosleep(ns);
                qi = q_ahead >= 0 ? q_ahead : atomicAdd(sched, 1);
                q_ahead = -1;
            }
            qi = __shfl_sync(0xffffffffu, qi, 0);
            const bool live_q = qi < n_items;
            const QItem qe = live_q ? qitems[qi] : QItem{};
            const int it = live_q ? qe.it : -1;
            TeamItem* e = &tq[p_n % C::QN];
            ++p_n;
            if (it < 0) {
                p_done = true;
                if (lane == 0) {
                    e->it = -1;
                    mbar_arrive(full_bar(slot));
                }
                return;
            }
            p_item = it;
            p_st = 0;
            const Desc& dsc = qe.d;
            const int kvh = qe.kv_head;
            if (lane == 0) *e = TeamItem{it, kvh, dsc.n_pages, dsc.tok_start, dsc.tok_end, dsc.member_off,
                                         dsc.n_members, dsc.n_main};
            if ((dsc.kind & 4) && !p_waited) {   // holds a newest token: wait for its producer
                asm volatile("griddepcontrol.wait;" ::: "memory");
                p_waited = true;
            }
            p_kv = kvh;
            p_npages = dsc.n_pages;
            p_nmain = dsc.n_main;
            p_kind = dsc.kind;
            p_off = dsc.page_off;
            pid_base = 0;
            pid_cur = lane < p_npages ? pages[p_off + lane] : 0;
            pid_next = 32 + lane < p_npages ? pages[p_off + 32 + lane] : 0;
        }
        const int p0 = p_st * PPS;
        const int npg = min(PPS, p_npages - p0);
        if ((p_kind & 8) && p0 + npg > p_nmain && !p_waited) {   // a folded tail holds a newest token
            asm volatile("griddepcontrol.wait;" ::: "memory");
            p_waited = true;
        }
        int row[PPS];
#pragma unroll
        for (int j = 0; j < PPS; ++j) {
            const int k = p0 + j;
            if (k >= pid_base + 32) {   // sequential: step to the next block, prefetch the one after
                pid_base += 32;
                pid_cur = pid_next;
                const int kk = pid_base + 32 + lane;
                pid_next = kk < p_npages ? pages[p_off + kk] : 0;
            }
            const int page = __shfl_sync(0xffffffffu, pid_cur, (k - pid_base) & 31);
            row[j] = __shfl_sync(0xffffffffu, p.layer_row_base + (page * Hkv + p_kv) * kPageSize, 0);
        }
        if (lane == 0) {
            const uint32_t fb = full_bar(slot);
            mbar_expect_tx(fb, npg * 2 * C::PAGE_BYTES);
            const uint32_t sb = ring + slot * C::STAGE_BYTES;
#pragma unroll
            for (int j = 0; j < PPS; ++j) {
                if (j < npg) {
                    if constexpr (F8) {   // one box: the page-head's K rows then its V^T rows (4 KB)
                        tma_load_3d(sb + j * 2 * C::PAGE_BYTES, &tmk, 0, 2 * row[j], 0, fb, policy);
                    } else {
                        tma_load_3d(sb + j * 2 * C::PAGE_BYTES, &tmk, 0, row[j], 0, fb, policy);
                        tma_load_3d(sb + j * 2 * C::PAGE_BYTES + C::PAGE_BYTES, &tmv, 0, row[j], 0, fb, policy);
                    }
                }
            }
        }
        __syncwarp();
        if (++p_st * PPS >= p_npages) p_item = -1;
        // reserve the next queue position two stages before this item runs out of stages to
        // issue: the atomic's round trip then overlaps this warp's compute instead of sitting
        // between items (a full item ahead would freeze the dynamic balance: measured 1.5x slower)
        if (lane == 0 && p_item >= 0 && q_ahead < 0 && (p_st + 2) * PPS >= p_npages) q_ahead = atomicAdd(sched, 1);
    };
    if (producer) {
        for (int s = 0; s < C::NS; ++s) issue_next(s);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");

    int slot = 0, c_n = 0;
    uint32_t phase = 0;
    // deferred record counting of the tail merge (fused_merge 2): the last item's members
    int pend_moff = 0, pend_nm = 0, pend_kv = 0;
    auto count_records = [&]() {   // producer warp; the other warp's stores are ordered before
        if (pend_nm > 0 && lane == 0) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            for (int mb = 0; mb < pend_nm; ++mb) {
                const Member mm = mems[pend_moff + mb];
                if (mm.rec >= 0)
                    asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;" ::"l"(counters + mm.row * Hkv + pend_kv)
                                 : "memory");
            }
        }
        pend_nm = 0;
    };
    // per-row state of the current item (row_setup fills it from global memory)
    int lo0 = 0, lo1 = 0, hi0 = INT_MAX, hi1 = INT_MAX;
    // folded tails (reading #21): item pages [tk, tk + tn) are the row's own, from token tt
    int tk0 = 0, tn0 = 0, tt0 = 0, tk1 = 0, tn1 = 0, tt1 = 0;
    uint32_t qa[KS][4];   // query A fragments (raw bf16 pairs until the F8 conversion)
    auto row_setup = [&](const TeamItem& d) {
        const int Rn = d.n_members * G;
        const int r0 = wt * 16 + (lane >> 2), r1 = r0 + 8;
        lo0 = lo1 = 0;
        hi0 = hi1 = INT_MAX;
        tk0 = tn0 = tt0 = tk1 = tn1 = tt1 = 0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) qa[ks][0] = qa[ks][1] = qa[ks][2] = qa[ks][3] = 0u;
        if (wt * 16 >= Rn) return;
        const __nv_bfloat16* q0 = nullptr;
        const __nv_bfloat16* q1 = nullptr;
        if (r0 < Rn) {
            const int mb = r0 / G;
            const Member m = mems[d.member_off + mb];
            lo0 = m.lo;
            hi0 = m.hi;
            tk0 = m.tail_k0;
            tn0 = m.tail_n;
            tt0 = m.tail_tok;
            q0 = p.q + m.row * p.q_sr + (d.kv_head * G + r0 - mb * G) * p.q_sh;
        }
        if (r1 < Rn) {
            const int mb = r1 / G;
            const Member m = mems[d.member_off + mb];
            lo1 = m.lo;
            hi1 = m.hi;
            tk1 = m.tail_k0;
            tn1 = m.tail_n;
            tt1 = m.tail_tok;
            q1 = p.q + m.row * p.q_sr + (d.kv_head * G + r1 - mb * G) * p.q_sh;
        }
        // fp8: the MMA's k index 2t+i (+8) reads channel 4t+i (+2) of each 16-channel block
        // -- the same permutation as the K fragment, so q.k is unchanged -- (f16 after the
        // conversion at item start)
        const int cq = F8 ? 4 * (lane & 3) : 2 * (lane & 3);
        const int c2 = F8 ? 2 : 8;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            if (q0) {
                qa[ks][0] = *reinterpret_cast<const uint32_t*>(q0 + ks * 16 + cq);
                qa[ks][2] = *reinterpret_cast<const uint32_t*>(q0 + ks * 16 + cq + c2);
            }
            if (q1) {
                qa[ks][1] = *reinterpret_cast<const uint32_t*>(q1 + ks * 16 + cq);
                qa[ks][3] = *reinterpret_cast<const uint32_t*>(q1 + ks * 16 + cq + c2);
            }
        }
    };
    while (true) {
        // the first stage of the next item (or the end-of-queue marker) has landed
        mbar_wait(full_bar(slot), phase);
        const TeamItem dsc = tq[c_n % C::QN];
        const int it = dsc.it;
        ++c_n;
        if (it < 0) {
            if (p.fused_merge == 2) {   // the last item's records: order both warps' stores first
                team_sync();
                if (producer) count_records();
            }
            break;
        }
        tr(2, it);
        const TeamItem& itm = dsc;
        const int R = dsc.n_members * G;
        const bool active = wt * 16 < R;   // identical for the KW warps of a row tile
        const int row0 = wt * 16 + (lane >> 2), row1 = row0 + 8;

        // ---- per-row setup: member, window bound lo and causal bound hi (keys [lo, hi) are
        //      live), query fragments (padding rows: q = 0, lo = 0, hi = INT_MAX).  (Loading
        //      them during the previous item's last stage instead measured 1-3 % slower.)
        row_setup(dsc);
        if (F8 && active)
#pragma unroll
            for (int ks = 0; ks < KS; ++ks)
#pragma unroll
                for (int e = 0; e < 4; ++e) qa[ks][e] = bf16x2_to_f16x2(qa[ks][e]);
        if (trace) {   // timeline: the row setup's loads have landed
            uint32_t d0 = qa[0][0] | qa[KS - 1][3] | uint32_t(lo0) | uint32_t(tk1);
            asm volatile("mov.b32 %0, %0;" : "+r"(d0));
            if (d0 == 0x9e3779b9u) tr(12, 0);
            tr(9, it);
        }
        // keys in [lo_warp, hi_warp) are live for every row of the warp: such pages need no mask
        int lo_warp = max(lo0, lo1), hi_warp = min(hi0, hi1);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo_warp = max(lo_warp, __shfl_xor_sync(0xffffffffu, lo_warp, o));
            hi_warp = min(hi_warp, __shfl_xor_sync(0xffffffffu, hi_warp, o));
        }
        hi_warp = min(hi_warp, dsc.tok_end);
        float scale_l2 = p.scale_log2, v_scale = 1.f;
        if (F8) {   // K = k_scale * code folds into the logit scale, V = v_scale * code into 1/l
            scale_l2 *= __ldg(p.kv_scale + (p.layer * Hkv + itm.kv_head) * 2) * kF8Unit;
            v_scale = __ldg(p.kv_scale + (p.layer * Hkv + itm.kv_head) * 2 + 1) * kF8Unit;
        }
        // running max per row, log2 units, raised lazily (only when a page's max exceeds it
        // by > kRescale, so P <= 2^kRescale); the same m is used for P, l and the LSE.
        constexpr float kRescale = 8.f;
        float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
        float acc[NT][4];
#pragma unroll
        for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;

        const int nst = (dsc.n_pages + PPS - 1) / PPS;
        for (int st = 0; st < nst; ++st) {
            if (st > 0) mbar_wait(full_bar(slot), phase);
            const int npg = min(PPS, dsc.n_pages - st * PPS);
#ifndef SPA_F8_EXP
#define SPA_F8_EXP 0
#endif
            // SPA_F8_EXP = 1 (timing experiments only, wrong results): fp8 consumers skip the math
            if (active && !(F8 && SPA_F8_EXP == 1)) {
                const uint32_t sb = ring + slot * C::STAGE_BYTES;
                float s[JW][2][4];
#pragma unroll
                for (int jj = 0; jj < JW; ++jj) {
                    const int j = wk + jj * KW;
#pragma unroll
                    for (int e = 0; e < 4; ++e) s[jj][0][e] = s[jj][1][e] = 0.f;
                    if (j < npg) {
                        const uint32_t kb = sb + j * 2 * C::PAGE_BYTES;
                        const int key = ((lane >> 4) << 3) + (lane & 7);
                        // QK^T over the head dimension as kQkChains independent accumulation
                        // chains per n8 tile (the HMMA dependency chain is the consumer's
                        // critical path), summed at the end
                        float sc[kQkChains][2][4];
#pragma unroll
                        for (int ch = 0; ch < kQkChains; ++ch)
#pragma unroll
                            for (int e = 0; e < 4; ++e) sc[ch][0][e] = sc[ch][1][e] = 0.f;
                        if constexpr (F8) {
                            // K rows of 128 e4m3 bytes, 128-B swizzled: key row nt*8 + g, channels
                            // 4t..4t+3 of 16-B chunk ks -> the f16 B fragment (k 2t, 2t+1, 2t+8, 2t+9)
#pragma unroll
                            for (int ks = 0; ks < KS; ++ks)
#pragma unroll
                                for (int nt = 0; nt < 2; ++nt) {
                                    const int kr = nt * 8 + (lane >> 2);
                                    const uint32_t w = lds32(kb + kr * 128 + (((ks ^ kr) & 7) << 4) + 4 * (lane & 3));
                                    uint32_t b0, b1;
                                    e4m3x4_to_f16x2x2(w, b0, b1);
                                    mma16816_f16(sc[ks % kQkChains][nt], qa[ks], b0, b1);
                                }
                        } else {
#pragma unroll
                            for (int ks = 0; ks < KS; ++ks) {
                                const int dcol = ks * 16 + ((lane >> 3) & 1) * 8;
                                const uint32_t addr =
                                    kb + (dcol >> 6) * 2048 + key * 128 + ((((dcol & 63) >> 3) ^ (key & 7)) << 4);
                                uint32_t b0, b1, b2, b3;
                                ldsm_x4(b0, b1, b2, b3, addr);
                                mma16816(sc[ks % kQkChains][0], qa[ks], b0, b1);
                                mma16816(sc[ks % kQkChains][1], qa[ks], b2, b3);
                            }
                        }
#pragma unroll
                        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                float acc_s = sc[0][nt][e];
#pragma unroll
                                for (int ch = 1; ch < kQkChains; ++ch) acc_s += sc[ch][nt][e];
                                s[jj][nt][e] = acc_s;
                            }
                    }
                }
                // mask + scale (log2 domain), row max over this warp's pages
                float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
                for (int jj = 0; jj < JW; ++jj) {
                    const int j = wk + jj * KW;
                    const int kpg = st * PPS + j;   // page index within the item
                    const bool tailp = kpg >= dsc.n_main;
                    const int tokp = dsc.tok_start + kpg * kPageSize;
                    const bool unmasked = !tailp && (j < npg) && (tokp >= lo_warp) && (tokp + kPageSize <= hi_warp);
                    if (unmasked) {
#pragma unroll
                        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float v = s[jj][nt][e] * scale_l2;
                                s[jj][nt][e] = v;
                                if (e < 2) mx0 = fmaxf(mx0, v);
                                else mx1 = fmaxf(mx1, v);
                            }
                    } else {
#pragma unroll
                        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const int off = nt * 8 + 2 * (lane & 3) + (e & 1);
                                const int lo = (e < 2) ? lo0 : lo1;
                                const int hi = (e < 2) ? hi0 : hi1;
                                int tok;
                                bool ok;
                                if (!tailp) {
                                    tok = tokp + off;
                                    ok = (j < npg) && (tok < dsc.tok_end) && (tok >= lo) && (tok < hi);
                                } else {   // a folded tail page: its owner's rows only
                                    const int rel = kpg - ((e < 2) ? tk0 : tk1);
                                    tok = ((e < 2) ? tt0 : tt1) + rel * kPageSize + off;
                                    ok = (j < npg) && rel >= 0 && rel < ((e < 2) ? tn0 : tn1) && (tok >= lo) && (tok < hi);
                                }
                                const float v = ok ? s[jj][nt][e] * scale_l2 : -INFINITY;
                                s[jj][nt][e] = v;
                                if (e < 2) mx0 = fmaxf(mx0, v);
                                else mx1 = fmaxf(mx1, v);
                            }
                    }
                }
                mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
                mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
                // -inf - -inf would be NaN: (m == -inf) means "no live key yet"
                const bool grow = (mx0 > m0 + kRescale) || (mx1 > m1 + kRescale) ||
                                  (m0 == -INFINITY && mx0 > -INFINITY) || (m1 == -INFINITY && mx1 > -INFINITY);
                if (__any_sync(0xffffffffu, grow)) {
                    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
                    const float al0 = (m0 == -INFINITY) ? 0.f : fast_exp2(m0 - mn0);
                    const float al1 = (m1 == -INFINITY) ? 0.f : fast_exp2(m1 - mn1);
                    m0 = mn0;
                    m1 = mn1;
                    l0 *= al0;
                    l1 *= al1;
#pragma unroll
                    for (int n = 0; n < NT; ++n) {
                        acc[n][0] *= al0;
                        acc[n][1] *= al0;
                        acc[n][2] *= al1;
                        acc[n][3] *= al1;
                    }
                }
                const float mu0 = (m0 == -INFINITY) ? 0.f : m0;
                const float mu1 = (m1 == -INFINITY) ? 0.f : m1;
                // P = exp2(s - m): l accumulates the fp32 P (the LSE carries no bf16 rounding);
                // the PV MMA takes P rounded to bf16 (A fragments).
#pragma unroll
                for (int jj = 0; jj < JW; ++jj) {
                    const int j = wk + jj * KW;
                    if (j < npg) {
                        float e[2][4];
#pragma unroll
                        for (int nt = 0; nt < 2; ++nt) {
                            e[nt][0] = fast_exp2(s[jj][nt][0] - mu0);
                            e[nt][1] = fast_exp2(s[jj][nt][1] - mu0);
                            e[nt][2] = fast_exp2(s[jj][nt][2] - mu1);
                            e[nt][3] = fast_exp2(s[jj][nt][3] - mu1);
                            l0 += e[nt][0] + e[nt][1];
                            l1 += e[nt][2] + e[nt][3];
                        }
                        uint32_t pa[4];
                        if constexpr (F8) {   // P <= 2^8 (lazy rescale): f16 holds it with 11 bits
                            pa[0] = pack_f16(e[0][0], e[0][1]);
                            pa[1] = pack_f16(e[0][2], e[0][3]);
                            pa[2] = pack_f16(e[1][0], e[1][1]);
                            pa[3] = pack_f16(e[1][2], e[1][3]);
                        } else {
                            pa[0] = pack_bf16(e[0][0], e[0][1]);
                            pa[1] = pack_bf16(e[0][2], e[0][3]);
                            pa[2] = pack_bf16(e[1][0], e[1][1]);
                            pa[3] = pack_bf16(e[1][2], e[1][3]);
                        }
                        const uint32_t vb = sb + j * 2 * C::PAGE_BYTES + C::PAGE_BYTES;
                        if constexpr (F8) {
                            // V^T: channel n*8 + g is 16-B chunk g of 128-B row n (swizzled: g ^ n),
                            // slots (2t, 2t+1, 2t+8, 2t+9) at bytes 4t..4t+3 of it (kF8VCol) -> the
                            // f16 B fragment of PV in one 4-B load
#pragma unroll
                            for (int n = 0; n < NT; ++n) {
                                const uint32_t w =
                                    lds32(vb + n * 128 + ((((lane >> 2) ^ n) & 7) << 4) + 4 * (lane & 3));
                                uint32_t b0, b1;
                                e4m3x4_to_f16x2x2(w, b0, b1);
                                mma16816_f16(acc[n], pa, b0, b1);
                            }
                        } else {
                            const int key = (((lane >> 3) & 1) << 3) + (lane & 7);
#pragma unroll
                            for (int dn = 0; dn < KS; ++dn) {
                                const int dchunk = 2 * dn + (lane >> 4);
                                const uint32_t addr =
                                    vb + (dchunk >> 3) * 2048 + key * 128 + (((dchunk & 7) ^ (key & 7)) << 4);
                                uint32_t b0, b1, b2, b3;
                                ldsm_x4_t(b0, b1, b2, b3, addr);
                                mma16816(acc[2 * dn], pa, b0, b1);
                                mma16816(acc[2 * dn + 1], pa, b2, b3);
                            }
                        }
                    }
                }
            }
            // ---- release the stage; the producer refills it NS stages ahead
            __syncwarp();
            if (lane == 0) mbar_arrive(empty_bar(slot));
            if (producer) {
                mbar_wait(empty_bar(slot), phase);   // acquire: both warps are past the stage
                if (pend_nm) {
                    tr(11, 0);
                    count_records();
                    tr(8, 0);
                }
                issue_next(slot);
            }
            if (++slot == C::NS) {
                slot = 0;
                phase ^= 1u;
            }
        }

        tr(10, it);
        // ---- epilogue (KW = 1): the warp holds its row tile's whole state; normalise and
        //      write every column
        if constexpr (KW == 1) {
            if (active) {
                l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
                l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
                l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
                l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
                const int c0 = 2 * (lane & 3);
#pragma unroll
                for (int rr = 0; rr < 2; ++rr) {
                    const int row = rr ? row1 : row0;
                    if (row < R) {
                        const int mb = row / G;
                        const Member m = mems[dsc.member_off + mb];
                        const int head = itm.kv_head * G + (row - mb * G);
                        const float l = rr ? l1 : l0;
                        const float mm = rr ? m1 : m0;
                        const float inv = l > 0.f ? v_scale / l : 0.f;
                        const float lse = l > 0.f ? (mm + log2f(l)) * 0.69314718055994531f : -INFINITY;
                        if (m.rec < 0) {
                            __nv_bfloat16* orow = p.o + m.row * p.o_sr + head * p.o_sh;
#pragma unroll
                            for (int n = 0; n < NT; ++n)
                                st_out2(fan, orow + n * 8 + c0, acc[n][2 * rr] * inv, acc[n][2 * rr + 1] * inv);
                            if ((lane & 3) == 0 && p.lse) st_out1(fan, p.lse + m.row * p.l_sr + head * p.l_sh, lse);
                        } else {
                            float* prow = p.part_o + ((long long)m.rec * Hq + head) * D;
#pragma unroll
                            for (int n = 0; n < NT; ++n)
                                *reinterpret_cast<float2*>(prow + n * 8 + c0) =
                                    make_float2(acc[n][2 * rr] * inv, acc[n][2 * rr + 1] * inv);
                            if ((lane & 3) == 0) p.part_lse[(long long)m.rec * Hq + head] = lse;
                        }
                    }
                }
            }
        }
        // ---- epilogue (KW = 2): combine the two key-split states of each row tile,
        //      normalise, and write each column half (warp wk owns columns [wk D/2, (wk+1) D/2)).
        if (KW == 2 && active) {
            l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
            l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
            l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
            l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
            const int r0 = lane >> 2, c0 = 2 * (lane & 3);
            // publish (m, l) and the OTHER warp's column half of the unscaled accumulator
            if ((lane & 3) == 0) {
                ml[(wk * 16 + r0) * 2 + 0] = m0;
                ml[(wk * 16 + r0) * 2 + 1] = l0;
                ml[(wk * 16 + r0 + 8) * 2 + 0] = m1;
                ml[(wk * 16 + r0 + 8) * 2 + 1] = l1;
            }
            // (register arrays need compile-time indices: one branch per key-split warp)
            auto publish = [&](float* dst, const float (*a)[4]) {
#pragma unroll
                for (int n = 0; n < NTH; ++n) {
                    const int col = n * 8 + c0;
                    *reinterpret_cast<float2*>(dst + r0 * (D / 2) + col) = make_float2(a[n][0], a[n][1]);
                    *reinterpret_cast<float2*>(dst + (r0 + 8) * (D / 2) + col) = make_float2(a[n][2], a[n][3]);
                }
            };
            if (wk == 0) publish(comb + 16 * (D / 2), acc + NTH);
            else publish(comb, acc);
            tr(13, 0);
            pair_sync();
            tr(14, 0);
            const int ow = 1 - wk;
            const float om0 = ml[(ow * 16 + r0) * 2 + 0], ol0 = ml[(ow * 16 + r0) * 2 + 1];
            const float om1 = ml[(ow * 16 + r0 + 8) * 2 + 0], ol1 = ml[(ow * 16 + r0 + 8) * 2 + 1];
            const float mt0 = fmaxf(m0, om0), mt1 = fmaxf(m1, om1);
            const float sa0 = m0 == -INFINITY ? 0.f : fast_exp2(m0 - mt0);
            const float sb0 = om0 == -INFINITY ? 0.f : fast_exp2(om0 - mt0);
            const float sa1 = m1 == -INFINITY ? 0.f : fast_exp2(m1 - mt1);
            const float sb1 = om1 == -INFINITY ? 0.f : fast_exp2(om1 - mt1);
            const float lt0 = l0 * sa0 + ol0 * sb0, lt1 = l1 * sa1 + ol1 * sb1;
            float half[NTH][4];
            auto gather = [&](const float* src, const float (*a)[4]) {
#pragma unroll
                for (int n = 0; n < NTH; ++n) {
                    const int col = n * 8 + c0;
                    const float2 x = *reinterpret_cast<const float2*>(src + r0 * (D / 2) + col);
                    const float2 y = *reinterpret_cast<const float2*>(src + (r0 + 8) * (D / 2) + col);
                    half[n][0] = a[n][0] * sa0 + x.x * sb0;
                    half[n][1] = a[n][1] * sa0 + x.y * sb0;
                    half[n][2] = a[n][2] * sa1 + y.x * sb1;
                    half[n][3] = a[n][3] * sa1 + y.y * sb1;
                }
            };
            if (wk == 0) gather(comb, acc);
            else gather(comb + 16 * (D / 2), acc + NTH);
            pair_sync();   // the exchange buffers may be rewritten by the next item
            tr(15, 0);
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const int row = rr ? row1 : row0;
                if (row < R) {
                    const int mb = row / G;
                    const Member m = mems[dsc.member_off + mb];
                    const int head = itm.kv_head * G + (row - mb * G);
                    const float l = rr ? lt1 : lt0;
                    const float mm = rr ? mt1 : mt0;
                    const float inv = l > 0.f ? v_scale / l : 0.f;
                    const float lse = l > 0.f ? (mm + log2f(l)) * 0.69314718055994531f : -INFINITY;
                    if (m.rec < 0) {
                        __nv_bfloat16* orow = p.o + m.row * p.o_sr + head * p.o_sh + wk * (D / 2);
#pragma unroll
                        for (int n = 0; n < NTH; ++n)
                            st_out2(fan, orow + n * 8 + c0, half[n][2 * rr] * inv, half[n][2 * rr + 1] * inv);
                        if ((lane & 3) == 0 && wk == 0 && p.lse) st_out1(fan, p.lse + m.row * p.l_sr + head * p.l_sh, lse);
                    } else {
                        float* prow = p.part_o + ((long long)m.rec * Hq + head) * D + wk * (D / 2);
#pragma unroll
                        for (int n = 0; n < NTH; ++n)
                            *reinterpret_cast<float2*>(prow + n * 8 + c0) =
                                make_float2(half[n][2 * rr] * inv, half[n][2 * rr + 1] * inv);
                        if ((lane & 3) == 0 && wk == 0) p.part_lse[(long long)m.rec * Hq + head] = lse;
                    }
                }
            }
        }

        tr(3, it);
        // ---- in-kernel split merge (fused_merge 1 / 2)
        bool any_partial = false;
        for (int mb = 0; mb < dsc.n_members; ++mb) any_partial |= mems[dsc.member_off + mb].rec >= 0;
        if (any_partial && p.fused_merge == 2) {
            // tail merge: this item's records are counted in (release) by the producer once
            // both warps have released the next stage -- off the item-to-item critical path
            pend_moff = dsc.member_off;
            pend_nm = dsc.n_members;
            pend_kv = itm.kv_head;
        } else if (any_partial && p.fused_merge == 1) {
            // the team barrier orders every lane's partial stores before the producer lane's
            // acq_rel arrival (release is cumulative); the last arriver acquires all of them.
            // Counters are never reset: launch k of the plan completes a (row, head) at
            // (k + 1) x its record count (the plan upload zeroes them).
            team_sync();
            uint32_t mask = 0;
            if (producer && lane == 0) {
                for (int mb = 0; mb < dsc.n_members; ++mb) {
                    const Member mm = mems[dsc.member_off + mb];
                    if (mm.rec < 0) continue;
                    const int nrec = rec_ptr[mm.row + 1] - rec_ptr[mm.row];
                    int* c = counters + mm.row * Hkv + itm.kv_head;
                    if (atom_add_acq_rel_gpu(c, 1) == (p.launch + 1) * nrec - 1) mask |= 1u << mb;
                }
                *team_slot = mask;
            }
            team_sync();
            mask = *team_slot;
            team_sync();
            while (mask) {
                const int mb = __ffs(mask) - 1;
                mask &= mask - 1;
                const Member mm = mems[dsc.member_off + mb];
                const int s0 = rec_ptr[mm.row], s1 = rec_ptr[mm.row + 1];
                __nv_bfloat16* orow = p.o + mm.row * p.o_sr;
                float* lrow = p.lse ? p.lse + mm.row * p.l_sr : nullptr;
                for (int hh = tw; hh < G; hh += C::TEAM_WARPS)
                    warp_merge_head<D>(p.part_o, p.part_lse, Hq, s0, s1, itm.kv_head * G + hh, orow, p.o_sh, lrow,
                                       p.l_sh, lane, D, fan);
            }
        }
    }

    // ---- tail merge (fused_merge == 2): every item has been popped; each WARP now pops
    //      merge subtasks -- a whole (request, KV head) task when G x S <= 32 (one warp,
    //      warp_merge_group), else one head of it -- waits until all of the task's records of
    //      this launch are counted in (every lane acquires; the items still running are owned
    //      by teams not in this loop), and merges.  Counters are never reset: launch k of the
    //      plan completes a task at (k + 1) x its record count.  One queue, popped in the
    //      plan's earliest-ready order.
    if (p.fused_merge == 2) {
        const int32_t* msub = meta + meta[H_OFF_MTASK];
        const int n_sub = meta[H_N_MTASK];
        int* qhead = sched + 32;   // own 128-B line
        while (true) {
            int t = 0;
            if (lane == 0) t = atomicAdd(qhead, 1);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= n_sub) break;
            const int code = msub[t];
            const int task = code >> 8, sub = code & 255;
            tr(4, t);
            const int row = task / Hkv, g = task - row * Hkv;
            const int s0 = rec_ptr[row], s1 = rec_ptr[row + 1];
            const int target = (p.launch + 1) * (s1 - s0);
            const int* c = counters + task;
            for (unsigned ns = p.poll_min; ld_acquire_gpu(c) < target; ns = min(ns * 2, p.poll_max)) __nanosleep(ns);
            tr(7, t);
            __nv_bfloat16* orow = p.o + row * p.o_sr;
            float* lrow = p.lse ? p.lse + row * p.l_sr : nullptr;
            if (sub == 0)
                warp_merge_group<D>(p.part_o, p.part_lse, Hq, s0, s1, g * G, G, orow, p.o_sh, lrow, p.l_sh, lane, D,
                                    fan);
            else
                warp_merge_head<D>(p.part_o, p.part_lse, Hq, s0, s1, g * G + sub - 1, orow, p.o_sh, lrow, p.l_sh, lane,
                                   D, fan);
            tr(5, t);
        }
    }
    tr(6, 0);
    // the last CTA to finish rewinds the queues for the next launch (stream-ordered)
    __syncthreads();
    if (threadIdx.x == 0) {
        // fused all-gather: this CTA's peer stores (ordered before by bar.sync) are made
        // visible system-wide before its arrival on the CTA counter (release pattern)
        if (fan) __threadfence_system();
        if (atomicAdd(sched + 1, 1) == int(gridDim.x) - 1) {
            sched[0] = 0;
            sched[1] = 0;
            sched[32] = 0;
            st_release_gpu(sched + 3, p.launch + kSchedSlots);   // hand the slot on
            if (fan) {
                // every CTA of this rank has arrived (acquire pattern), so all of this rank's
                // output stores precede the flags; then wait for every peer's flag of this epoch
                __threadfence_system();
                for (int k = 0; k < p.fan.n; ++k)
                    if (k != p.rank) st_release_sys(p.sig_peer[k] + p.rank, p.epoch);
                unsigned long long t0, t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
                for (int k = 0; k < p.fan.n; ++k) {
                    if (k == p.rank) continue;
                    while (int(ld_acquire_sys(p.sig_local + k) - p.epoch) < 0) {
                        __nanosleep(256);
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                        if (t - t0 > 20000000000ull) {   // 20 s: a peer never arrived; report, do not hang
                            *p.status = 1u;
                            break;
                        }
                    }
                }
            }
        }
    }
}

template <int D, int MT, int PPS, int TEAMS, bool F8 = false, int KW = 2>
static int launch_decode_t(const spa_plan* P, const DecodeParams& dp, void* stream) {
    using C = DecodeCfg<D, MT, PPS, TEAMS, F8, KW>;
    static std::atomic<unsigned long long> attr_done{0};
    if (int e = set_smem_attr_once(decode_kernel<D, MT, PPS, TEAMS, F8, KW>, C::SMEM, &attr_done)) return e;
    const CUtensorMap* tk = reinterpret_cast<const CUtensorMap*>(P->pool->tmap_k.bytes);
    const CUtensorMap* tv = reinterpret_cast<const CUtensorMap*>(P->pool->tmap_v.bytes);
    return launch_pdl(decode_kernel<D, MT, PPS, TEAMS, F8, KW>, dim3(P->num_ctas), dim3(C::WARPS * 32), C::SMEM,
                      stream, *tk, *tv, dp);
}

// F4 fp8 pages (d = 128): the same team shapes as bf16; SPA_F8_PPS pages per stage (4: the
// same 16-KB stages as bf16, two pages per warp per stage for ILP; 2 measured 12 % slower)
#ifndef SPA_F8_PPS
#define SPA_F8_PPS 4
#endif
static int launch_decode_f8(const spa_plan* P, const DecodeParams& dp, void* stream) {
    constexpr int S = SPA_F8_PPS;
    if (P->kw == 1) {   // one warp per 16-row tile: 8 or 12 one-warp teams (16 rows), 4 teams of 2 (32 rows)
        if (P->mt == 1 && P->teams == 12) return launch_decode_t<128, 1, 2, 12, true, 1>(P, dp, stream);
        if (P->mt == 1) return launch_decode_t<128, 1, 2, 8, true, 1>(P, dp, stream);
        return launch_decode_t<128, 2, S, 4, true, 1>(P, dp, stream);
    }
    if (P->mt == 1) {
        if (P->teams == 1) return launch_decode_t<128, 1, S, 1, true>(P, dp, stream);
        if (P->teams == 2) return launch_decode_t<128, 1, S, 2, true>(P, dp, stream);
        return launch_decode_t<128, 1, S, 4, true>(P, dp, stream);
    }
    if (P->mt == 4) return launch_decode_t<128, 4, S, 1, true>(P, dp, stream);
    if (P->teams == 1) return launch_decode_t<128, 2, S, 1, true>(P, dp, stream);
    return launch_decode_t<128, 2, S, 2, true>(P, dp, stream);
}

#ifndef SPA_KW1_PPS
#define SPA_KW1_PPS 1
#endif
template <int D>
static int launch_decode_d(const spa_plan* P, const DecodeParams& dp, void* stream) {
    // 32-row items, one warp per row tile over every page of a stage (no key split): 4 teams
    if (P->mt == 2 && P->kw == 1) return launch_decode_t<D, 2, 2, 4, false, 1>(P, dp, stream);
    // 16-row items, one-warp teams (8 per CTA, one page per stage)
    if (P->mt == 1 && P->kw == 1)
        return P->teams == 8 ? launch_decode_t<D, 1, SPA_KW1_PPS, 8, false, 1>(P, dp, stream)
                             : int(cudaErrorNotSupported);
    if (P->mt == 1) {
        if (P->teams == 1) return launch_decode_t<D, 1, 2, 1>(P, dp, stream);
        if (P->teams == 2) return launch_decode_t<D, 1, 2, 2>(P, dp, stream);
        return launch_decode_t<D, 1, 2, 4>(P, dp, stream);
    }
    if (P->mt == 4) return launch_decode_t<D, 4, 2, 1>(P, dp, stream);
    if (P->teams == 1) return launch_decode_t<D, 2, 2, 1>(P, dp, stream);
    return launch_decode_t<D, 2, 2, 2>(P, dp, stream);
}

bool decode_teams_supported(int mt, int teams, int kw) {
    if (kw == 1) return (mt == 2 && teams == 4) || (mt == 1 && (teams == 8 || teams == 12));
    if (mt == 4 || mt == 8) return teams == 1;
    return teams == 1 || teams == 2 || (teams == 4 && mt == 1);
}

// merge_mode 0 leaves the place of the split merge to the library: the kernel's tail phase,
// except for fp8 pools decoded by one-warp teams without a peer fan-out, whose split records
// are merged by the PDL-chained merge_kernel (BJ config 1 fp8: 75.9 vs 79.0 us per layer;
// bf16 key-split teams keep the tail phase: 109.3 vs 112.3; profiles/r02_merge_modes.txt)
bool merge_separately(const spa_plan* P, bool fan_out) {
    return P->cfg.merge_mode == 0 && P->pool->kv_fp8 && P->kw == 1 && P->mt == 1 && !fan_out;
}

int launch_decode(const spa_plan* P, int32_t layer, const void* q, int64_t q_sr, int64_t q_sh, void* o, int64_t o_sr,
                  int64_t o_sh, float* lse, int64_t l_sr, int64_t l_sh, float scale, void* stream,
                  const PeerLaunch* peer) {
    if (peer && (P->mt == 8 || P->cfg.merge_mode == 2)) return int(cudaErrorNotSupported);
    if (P->pool->kv_fp8 && P->mt == 8) return int(cudaErrorNotSupported);   // the tcgen05 extend kernel is bf16
    if (P->mt == 8)   // 128-row items: the tcgen05 extend kernel (ext.cu)
        return launch_ext(P, layer, q, q_sr, q_sh, o, o_sr, o_sh, lse, l_sr, l_sh, scale, stream);
    const auto& c = P->pool->cfg;
    const int32_t* H = P->host.data();
    if (H[H_N_ITEMS] == 0) return 0;
    DecodeParams dp{};
    dp.meta = P->d_meta;
    dp.q = static_cast<const __nv_bfloat16*>(q);
    dp.q_sr = q_sr;
    dp.q_sh = q_sh;
    dp.o = static_cast<__nv_bfloat16*>(o);
    dp.o_sr = o_sr;
    dp.o_sh = o_sh;
    dp.lse = lse;
    dp.l_sr = l_sr;
    dp.l_sh = l_sh;
    dp.part_o = P->d_part_o;
    dp.part_lse = P->d_part_lse;
    dp.scale_log2 = float(double(scale) * 1.4426950408889634);
    dp.layer_row_base = layer * c.num_pages * c.num_kv_heads * kPageSize;
    dp.num_q_heads = c.num_q_heads;
    dp.num_kv_heads = c.num_kv_heads;
    dp.group_size = c.num_q_heads / c.num_kv_heads;
    dp.fused_merge = P->cfg.merge_mode == 0 ? 2 : P->cfg.merge_mode == 1 ? 1 : 0;
    if (merge_separately(P, peer && peer->world > 1)) dp.fused_merge = 0;
    dp.launch = int(P->launches++);
    dp.trace = P->trace;
    dp.trace_cap = P->trace_cap;
    static const unsigned poll_min = std::getenv("SPA_POLL_MIN") ? unsigned(std::atoi(std::getenv("SPA_POLL_MIN"))) : 32u;
    static const unsigned poll_max = std::getenv("SPA_POLL_MAX") ? unsigned(std::atoi(std::getenv("SPA_POLL_MAX"))) : 256u;
    dp.poll_min = poll_min;
    dp.poll_max = poll_max;
    if (peer && peer->world > 1) {
        dp.fan.n = peer->world;
        for (int k = 0; k < peer->world; ++k) {
            dp.fan.delta[k] = peer->delta[k];
            dp.sig_peer[k] = peer->sig_peer[k];
        }
        dp.rank = peer->rank;
        dp.epoch = peer->epoch;
        dp.sig_local = peer->sig_local;
        dp.status = peer->status;
    }
    dp.kv_scale = P->pool->kv_scale;
    dp.layer = layer;
    int err = 0;
    if (P->pool->kv_fp8)
        err = launch_decode_f8(P, dp, stream);
    else
        err = c.head_dim == 64 ? launch_decode_d<64>(P, dp, stream) : launch_decode_d<128>(P, dp, stream);
    if (err) return err;
    if (H[H_N_RECORDS] > 0 && !dp.fused_merge)
        err = launch_merge(H[H_N_REQ], c.num_q_heads, c.head_dim, P->d_meta + H[H_OFF_REC_PTR], P->d_part_o,
                           P->d_part_lse, o, o_sr, o_sh, lse, l_sr, l_sh, P->num_ctas, stream);
    return err;
}

}  // namespace spa
