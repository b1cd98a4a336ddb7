// F2: shared-prefix EXTEND attention on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// Work items and queue are the planner's (plan.cpp, max_rows 128): an item is (descriptor,
// KV head) with up to 128 query rows -- the rows of every request sharing the range (a
// parent's decode token and its speculative fork's prompt tokens), G query
// heads per token.  At this many rows per KV byte (~80 flop/B for Qwen2.5's 16-token
// prompts) the step is a dense contraction: S = Q K^T and O = P V run as tcgen05.mma with
// M = 128 rows, fp32 accumulators in tensor memory.
//
// One CTA per SM, warp-specialised:
//   warp 0      K producer: pops items from the plan's dynamic queue and streams each stage's
//               keys (4 pages = 64 keys of one KV head, 16 KB, chunk by chunk so a stage's keys
//               are contiguous) into the K ring, one TMA box per lane;
//   warp 10     V producer: follows the K producer's items, streams the stage's V pages (one
//               box per page and lane) into the V ring.  The rings are separate because K is
//               consumed by S_j and freed as soon as that MMA completes, while V waits for P_j
//               (PV lags S by two stages); the two producers and the per-lane boxes exist
//               because one issuing thread cannot keep enough TMA traffic in flight
//               (scripts/micro/tma_rate.cu);
//   warp 1      S issuer (one elected lane): S_j = Q K_j^T (8 x M128 N64 K16, A = the item's Q
//               tile in tensor memory; B = the stage's keys, K-major SW128);
//   warp 12     PV issuer: O += P_j V_j (per page: M128 N128 K16, A = P in tensor memory,
//               B = the V page as an MN-major SW128 operand).  Two issuers because a thread's
//               tcgen05.mma issue blocks while the tensor pipe works: one issuer serialised S
//               and PV (measured: ~0.6 us of issue per 64-key stage);
//   warps 2-9   two softmax warpgroups, one thread per query row (tensor-memory lane) each;
//               WG k takes the stages of parity k: loads S, masks (window lo, causal hi,
//               range end), runs the online softmax in the log2 domain with lazy rescaling
//               (threshold 2^8) of its own accumulator O_k in tensor memory, writes P (bf16)
//               over S's columns; at item end the two (m, l, O_k) merge per row and bf16 O +
//               LSE (or an fp32 partial record for split ranges) are written.
// Tensor memory: S buffers 0-2 (64 columns each; PV lags S by 2 stages), the Q tile (64 columns:
// the A operand of S = Q K^T, so S reads only K from shared memory), O_0, O_1 (128 each).
#include "device_util.cuh"
#include "spa_internal.h"
#include "umma.cuh"

namespace spa {

#ifdef SPA_EXT_DEBUG_HANG   // (debug builds: a wait that spins ~forever traps with its identity)
__device__ int* g_ext_dbg;   // unused placeholder
__device__ __forceinline__ void ext_wait(uint32_t bar, uint32_t parity, int id, const volatile int* dbg = nullptr) {
    for (long long i = 0;; ++i) {
        uint32_t ok;
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
        if (ok) return;
        if (i == (1ll << 24)) {
            printf("ext_kernel hang: block %d thread %d wait id %d parity %u bar %u | prod n %d slot %d st %d nst %d | mma n %d g %d st %d nst %d | wg g %d n %d\n",
                   blockIdx.x, threadIdx.x, id, parity, (bar & 0xfff) >> 3, dbg ? dbg[0] : -1, dbg ? dbg[1] : -1,
                   dbg ? dbg[2] : -1, dbg ? dbg[3] : -1, dbg ? dbg[4] : -1, dbg ? dbg[5] : -1, dbg ? dbg[6] : -1,
                   dbg ? dbg[7] : -1, dbg ? dbg[8] : -1, dbg ? dbg[9] : -1);
            __trap();
        }
    }
}
#define EXT_WAIT(b, ph, id) do { ext_wait(b, ph, id, dbgw); __syncwarp(); } while (0)
#define EXT_DBG(i, v) (dbgw[i] = (v))
#else
// every wait reconverges its warp: the MMA issuer elects a lane right after waiting
#define EXT_WAIT(b, ph, id) do { mbar_wait(b, ph); __syncwarp(); } while (0)
#define EXT_DBG(i, v) ((void)0)
#endif

struct ExtParams {
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
    int layer_row_base;
    int num_q_heads, group_size, num_kv_heads;
    int launch;
    unsigned long long* trace;   // spa_debug_set_trace: per-warp events of CTA 0 (stage timeline)
    int trace_cap;
};

struct ExtItem {
    int it, kv_head, n_pages, tok_start, tok_end, member_off, n_members, kind, page_off, n_main;
};

namespace ext {
#ifndef SPA_EXT_EXP
#define SPA_EXT_EXP 0   // timing experiments (wrong results by design): 1 no MMAs, 2 no softmax math
#endif
constexpr int EXP = SPA_EXT_EXP;
constexpr int D = 128;
constexpr int PAGE_BYTES = kPageSize * D * 2;     // 4 KB: K (or V) of one page, one head
#ifndef SPA_EXT_PPS
#define SPA_EXT_PPS 4
#endif
constexpr int PPS = SPA_EXT_PPS;                  // pages per stage
constexpr int KPS = PPS * kPageSize;              // keys per stage (S columns)
static_assert(32 % PPS == 0, "producers refresh page ids per 32-page window");
constexpr int HALF_BYTES = PPS * PAGE_BYTES;      // K (or V) of one stage
// K stage: key-contiguous [2 chunks][KPS rows][128 B] (one MMA covers every key of the stage:
// N = KPS); V stage: page by page [page][2 chunks][16 rows][128 B] (one K=16 MMA each)
constexpr int K_CHUNK = KPS * 128;                // bytes per 64-column chunk of the stage's keys
constexpr int N_SLOTS = (232448 - 1024 - 4096) / HALF_BYTES;   // 16-KB ring slots (Q lives in tensor memory)
#ifndef SPA_EXT_NK
#define SPA_EXT_NK 4
#endif
constexpr int NK = SPA_EXT_NK;                    // K ring stages (held from TMA issue to S_j done)
constexpr int NV = N_SLOTS - NK;                  // V ring stages (held until PV_j, after P_j)
static_assert(NK >= 2 && NV >= 3, "ring depths");
constexpr int QN = NV + 12;  // popped-item queue entries: the leader runs at most NK + 3 stages
                             // (items, when items are one stage long) ahead of the PV issuer
constexpr int OFF_V = NK * HALF_BYTES;
constexpr int OFF_BAR = (NK + NV) * HALF_BYTES;
// barriers: kfull[NK], kempty[NK], vfull[NV], vempty[NV], s_full[4], p_full[4] (one per S
// buffer: a buffer's next S / P needs this round's P / S, so each barrier is at most one phase
// ahead of its waiter; 3 of the 4 are used), q_ready, o_full, pv_done[4] (PV of the stages
// using S buffer b)
constexpr int BAR_KFULL = 0, BAR_KEMPTY = NK, BAR_VFULL = 2 * NK, BAR_VEMPTY = 2 * NK + NV,
              BAR_SFULL = 2 * (NK + NV), BAR_PFULL = BAR_SFULL + 4, BAR_QREADY = BAR_SFULL + 8,
              BAR_OFULL = BAR_SFULL + 9, BAR_PVDONE = BAR_SFULL + 10, BAR_OFREE = BAR_SFULL + 14,
              N_BARS = BAR_SFULL + 15;
constexpr int OFF_TQ = OFF_BAR + N_BARS * 8;
constexpr int OFF_TSEQ = OFF_TQ + QN * int(sizeof(ExtItem));   // int[QN]: entry n published as n + 1
constexpr int OFF_ML = (OFF_TSEQ + QN * 4 + 15) & ~15;           // [2][2][128] fp32 + 8 flags
constexpr int OFF_TSLOT = OFF_ML + 4 * 128 * 4 + 8 * 4;
constexpr int SMEM = 1024 + OFF_TSLOT + 16 + 128;   // + debug words (hang-trap builds)
#ifndef SPA_EXT_KW
#define SPA_EXT_KW 1
#endif
constexpr int KW = SPA_EXT_KW;   // K producer warps: 1, or 2 (one 64-channel chunk each; warp 12)
static_assert(KW == 1 || KW == 2, "K producer warps");
// warps: 0 K producer (pops items), 1 S issuer, 2-9 softmax warpgroups, 10 V producer, 11 PV issuer,
// 12 (KW = 2) K producer of chunk 1
constexpr int THREADS = (11 + KW) * 32;
constexpr int WARP_V = 10, WARP_PV = 11, WARP_K1 = 12;
// tensor memory: S buffers 0..3 (KPS columns each; stage g uses g % 4), O_0, O_1 (128 each)
// tensor memory: S buffers 0..2 (KPS columns each; stage g uses g % 3 -- S_{g+3} waits for
// PV_g, the buffer's reader), the Q tile (bf16 pairs: D / 2 columns, the A operand of
// S = Q K^T, so the S MMAs read only K from shared memory), O_0, O_1
constexpr int NSB = 3;
constexpr uint32_t TMEM_COLS = 512, S_COL = 0, Q_COL = NSB * KPS, O_COL = 256;
static_assert(Q_COL + D / 2 <= O_COL, "S buffers + Q overlap O");
static_assert(SMEM <= 232448, "extend kernel shared memory");
}  // namespace ext

__global__ void __launch_bounds__(ext::THREADS, 1)
    ext_kernel(const __grid_constant__ CUtensorMap tmk1, const __grid_constant__ CUtensorMap tmv, const ExtParams p) {
    using namespace ext;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    auto bar = [&](int i) { return sbase + OFF_BAR + i * 8; };
    ExtItem* tq = reinterpret_cast<ExtItem*>(smem + OFF_TQ);
#ifdef SPA_EXT_DEBUG_HANG
    volatile int* dbgw = reinterpret_cast<volatile int*>(smem + OFF_TSLOT + 64);   // past the TMEM slot
#endif

    if (threadIdx.x == 0) {
        for (int i = 0; i < NK; ++i) {
            mbar_init(bar(BAR_KFULL + i), KW);   // one expect-tx arrival per K producer warp
            mbar_init(bar(BAR_KEMPTY + i), 1);
        }
        for (int i = 0; i < NV; ++i) {
            mbar_init(bar(BAR_VFULL + i), 1);
            mbar_init(bar(BAR_VEMPTY + i), 1);
        }
        for (int b = 0; b < 4; ++b) {
            mbar_init(bar(BAR_SFULL + b), 1);
            mbar_init(bar(BAR_PFULL + b), 128);
            mbar_init(bar(BAR_PVDONE + b), 1);
        }
        mbar_init(bar(BAR_QREADY), 256);
        mbar_init(bar(BAR_OFULL), 1);
        mbar_init(bar(BAR_OFREE), 256);
        for (int i = 0; i < QN; ++i) reinterpret_cast<int*>(smem + OFF_TSEQ)[i] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) umma::tmem_alloc(sbase + OFF_TSLOT, TMEM_COLS);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + OFF_TSLOT);
    asm volatile("griddepcontrol.launch_dependents;");
    if (p.trace && threadIdx.x == 0 && int(blockIdx.x) < p.trace_cap) {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        p.trace[2ull * (7ull * p.trace_cap + blockIdx.x)] = gt;
    }
    // stage timeline of CTA 0 (spa_debug_set_trace): lane 0 of warps 0..2 records (tag, clock64)
    unsigned long long* trace = (p.trace && blockIdx.x == 0 && (warp <= 2 || warp == WARP_PV) && lane == 0)
                                    ? p.trace + 2ull * (warp == WARP_PV ? 3 : warp) * p.trace_cap : nullptr;
    int tr_n = 0;
    auto tr = [&](unsigned long long tag, int id) {
        if (trace && tr_n < p.trace_cap) {
            unsigned long long gt, ck;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(ck));
            trace[2 * tr_n] = gt;
            trace[2 * tr_n + 1] = (tag << 56) | ((unsigned long long)(id & 0xffffff) << 32) | (ck & 0xffffffffull);
            ++tr_n;
        }
    };

    const int32_t* meta = p.meta;
    const QItem* qitems = reinterpret_cast<const QItem*>(meta + meta[H_OFF_QITEM]);
    const Member* mems = reinterpret_cast<const Member*>(meta + meta[H_OFF_MEMBER]);

    const int32_t* pages = meta + meta[H_OFF_PAGES];
    int32_t* sched = const_cast<int32_t*>(meta) + meta[H_OFF_SCHED] + kSchedStride * (p.launch % kSchedSlots);
    const int n_items = meta[H_N_ITEMS];
    const int G = p.group_size, Hq = p.num_q_heads, Hkv = p.num_kv_heads;
    (void)Hq;

    // A producer thread's TMA issue is slow and bounded by what it has in flight (measured,
    // scripts/micro/tma_rate.cu: one issuing lane streams ~1-2 TB/s chip-wide, four lanes
    // ~2.7-3.4, two warps x 4-8 lanes 5.3-7 TB/s): K and V are issued by separate warps, one
    // box per lane.
    uint64_t policy = 0;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    volatile int* tseq = reinterpret_cast<volatile int*>(smem + OFF_TSEQ);
    if (warp == 0) {
        // ------------------------------------------------------------ K producer (leader): pops items
        bool waited = false;
        int n = 0, g = 0;   // g: global stage counter (K slot g % NK)
        for (int k = 0;; ++k) {
            int qi = 0;
            if (lane == 0) {
                if (k == 0)   // the queue slot is ours once launch - kSchedSlots rewound it
                    for (unsigned ns = 64; ld_acquire_gpu(sched + 3) != p.launch; ns = min(ns * 2, 1024u))
                        __nanosleep(ns);
                qi = atomicAdd(sched, 1);
            }
            qi = __shfl_sync(0xffffffffu, qi, 0);
            const QItem qe = qi < n_items ? qitems[qi] : QItem{};
            const int it = qi < n_items ? qe.it : -1;
            ExtItem* e = &tq[n % QN];
            // the K slot of this item's first stage (or the end marker): its fill publishes the
            // entry to the MMA warp and the softmax WGs; tseq publishes it to the followers
            EXT_WAIT(bar(BAR_KEMPTY + g % NK), uint32_t(((g / NK) & 1) ^ 1), 1);
            if (it < 0) {
                if (lane == 0) {
                    e->it = -1;
                    __threadfence_block();
                    tseq[n % QN] = n + 1;
                    mbar_arrive(bar(BAR_KFULL + g % NK));
                }
                break;
            }
            const Desc& dsc = qe.d;
            const Item itm{qe.desc, qe.kv_head};
            if (lane == 0) {
                *e = ExtItem{it, itm.kv_head, dsc.n_pages, dsc.tok_start, dsc.tok_end, dsc.member_off, dsc.n_members,
                             dsc.kind, dsc.page_off, dsc.n_main};
                __threadfence_block();
                tseq[n % QN] = n + 1;
            }
            ++n;
            if ((dsc.kind & 4) && !waited) {   // holds newest tokens: wait for their producer
                asm volatile("griddepcontrol.wait;" ::: "memory");
                waited = true;
            }
            int pid_cur = lane < dsc.n_pages ? pages[dsc.page_off + lane] : 0;
            int pid_base = 0;
            const int nst = (dsc.n_pages + PPS - 1) / PPS;
            for (int st = 0; st < nst; ++st, ++g) {
                const int ks = g % NK;
                if (st > 0) EXT_WAIT(bar(BAR_KEMPTY + ks), uint32_t(((g / NK) & 1) ^ 1), 2);
                tr(10, st);
                const int p0 = st * PPS, npg = min(PPS, dsc.n_pages - p0);
                if ((dsc.kind & 8) && p0 + npg > dsc.n_main && !waited) {   // a folded tail's newest token
                    asm volatile("griddepcontrol.wait;" ::: "memory");
                    waited = true;
                }
                if (p0 >= pid_base + 32) {   // PPS divides 32: a stage never straddles a window
                    pid_base += 32;
                    pid_cur = pid_base + lane < dsc.n_pages ? pages[dsc.page_off + pid_base + lane] : 0;
                }
                // KW = 2: lane j < npg loads chunk 0 of page p0 + j; KW = 1: lane x < 2 npg loads
                // chunk x % 2 of page p0 + x / 2
                const int pj = KW == 2 ? lane : lane >> 1, ch = KW == 2 ? 0 : lane & 1;
                const int page = __shfl_sync(0xffffffffu, pid_cur, (p0 - pid_base + pj) & 31);
                const int row = p.layer_row_base + (page * Hkv + itm.kv_head) * kPageSize;
                const uint32_t fb = bar(BAR_KFULL + ks);
                if (lane == 0) mbar_expect_tx(fb, npg * PAGE_BYTES / KW);
                __syncwarp();
                if (lane < npg * (3 - KW))
                    tma_load_3d(sbase + ks * HALF_BYTES + ch * K_CHUNK + pj * 2048, &tmk1, 0, row, ch, fb, policy);
                __syncwarp();
                tr(12, st);
                if (lane == 0) {
                    EXT_DBG(0, n);
                    EXT_DBG(1, g);
                    EXT_DBG(2, st);
                    EXT_DBG(3, nst);
                }
            }
        }
    } else if (warp == WARP_V || warp == WARP_K1) {
        // ------------------------------------------------------------ followers: the V producer and (KW = 2) the
        // chunk-1 K producer walk the leader's items (published through tseq) and issue one
        // box per lane and page into their ring
        const bool is_v = warp == WARP_V;
        const int nring = is_v ? NV : NK;
        const uint32_t full0 = bar(is_v ? BAR_VFULL : BAR_KFULL), empty0 = bar(is_v ? BAR_VEMPTY : BAR_KEMPTY);
        const uint32_t ring0 = sbase + (is_v ? OFF_V : K_CHUNK);   // K1: chunk 1 of each K stage
        const CUtensorMap* tm = is_v ? &tmv : &tmk1;
        const uint32_t box_bytes = is_v ? PAGE_BYTES : PAGE_BYTES / 2, box_stride = is_v ? PAGE_BYTES : 2048;
        bool waited = false;
        int n = 0, g = 0;   // g: global stage counter (slot g % nring)
        while (true) {
            if (lane == 0)
                while (tseq[n % QN] != n + 1) __nanosleep(32);
            __syncwarp();
            __threadfence_block();
            const ExtItem e = tq[n % QN];
            ++n;
            if (e.it < 0) {
                if (!is_v) {   // the end marker's K slot also counts this warp's arrival
                    EXT_WAIT(empty0 + (g % nring) * 8, uint32_t(((g / nring) & 1) ^ 1), 13);
                    if (lane == 0) mbar_arrive(full0 + (g % nring) * 8);
                }
                break;
            }
            if ((e.kind & 4) && !waited) {
                asm volatile("griddepcontrol.wait;" ::: "memory");
                waited = true;
            }
            int pid_cur = lane < e.n_pages ? pages[e.page_off + lane] : 0;
            int pid_base = 0;
            const int nst = (e.n_pages + PPS - 1) / PPS;
            for (int st = 0; st < nst; ++st, ++g) {
                const int sl = g % nring;
                EXT_WAIT(empty0 + sl * 8, uint32_t(((g / nring) & 1) ^ 1), 11);
                const int p0 = st * PPS, npg = min(PPS, e.n_pages - p0);
                if ((e.kind & 8) && p0 + npg > e.n_main && !waited) {
                    asm volatile("griddepcontrol.wait;" ::: "memory");
                    waited = true;
                }
                if (p0 >= pid_base + 32) {
                    pid_base += 32;
                    pid_cur = pid_base + lane < e.n_pages ? pages[e.page_off + pid_base + lane] : 0;
                }
                const int page = __shfl_sync(0xffffffffu, pid_cur, (p0 - pid_base + lane) & 31);
                const int row = p.layer_row_base + (page * Hkv + e.kv_head) * kPageSize;
                const uint32_t fb = full0 + sl * 8;
                if (lane == 0) mbar_expect_tx(fb, npg * box_bytes);
                __syncwarp();
                if (lane < npg)
                    tma_load_3d(ring0 + sl * HALF_BYTES + lane * box_stride, tm, 0, row, is_v ? 0 : 1, fb, policy);
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ S issuer
        // S_g = Q K_g^T into S buffer g % 3 once K_g landed and PV_{g-3} (the buffer's last
        // reader) completed.  S and PV are issued by different warps: one thread's tcgen05.mma
        // issue blocks while the tensor pipe works, so one issuer serialises S and PV.  The
        // whole warp walks the pipeline (descriptors stay warp-uniform); one lane issues.
        int n = 0, g = 0;   // g: global stage counter (K slot g % NK, S buffer g % 3)
        uint32_t qph = 0;
        while (true) {
            EXT_WAIT(bar(BAR_KFULL + g % NK), uint32_t((g / NK) & 1), 3);
            const ExtItem e = tq[n % QN];
            ++n;
            if (e.it < 0) break;
            tr(22, n);
            EXT_WAIT(bar(BAR_QREADY), qph, 4);   // Q tile written (and the last item's O read out)
            qph ^= 1u;
            tr(23, n);
            const int nst = (e.n_pages + PPS - 1) / PPS;
            for (int st = 0; st < nst; ++st, ++g) {
                const int ks = g % NK;
                if (lane == 0) {
                    EXT_DBG(4, n);
                    EXT_DBG(5, g);
                    EXT_DBG(6, st);
                    EXT_DBG(7, nst);
                }
                if (st > 0) EXT_WAIT(bar(BAR_KFULL + ks), uint32_t((g / NK) & 1), 5);
                // S buffer g % 3 is free once PV_{g-3} completed (its completion (g-3)/3; the next
                // one needs S_g, so the parity is exact)
                if (g >= NSB) EXT_WAIT(bar(BAR_PVDONE + g % NSB), uint32_t(((g - NSB) / NSB) & 1), 14);
                tr(20, st);
                umma::fence_after();
                const int npg = min(PPS, e.n_pages - st * PPS);
                const uint64_t k_desc = umma::desc_k_sw128(sbase + ks * HALF_BYTES, 1024);
                const uint32_t sbuf = tmem + S_COL + (g % NSB) * KPS;
                const uint32_t id_s = umma::idesc_bf16_f32(128, npg * 16, false, false);
                if (umma::elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < D / 16 && !(EXP & 1); ++kk)   // A: Q columns (8 per K step); B: 16-B units
                        umma::mma_ts(sbuf, tmem + Q_COL + kk * 8,
                                     k_desc + uint64_t((kk >> 2) * (K_CHUNK >> 4) + (kk & 3) * 2), id_s, kk > 0);
                    umma::commit(bar(BAR_KEMPTY + ks));   // K slot free once S_g has read it
                    umma::commit(bar(BAR_SFULL + g % NSB));
                }
                __syncwarp();
                tr(21, st);
            }
        }
    } else if (warp == WARP_PV) {
        // ------------------------------------------------------------ PV issuer
        // O_{g & 1} += P_g V_g once the softmax WG wrote P_g and V_g landed; after an item's
        // last PV, o_full.  Follows the K producer's items through tseq.
        const uint32_t id_o = umma::idesc_bf16_f32(128, 128, false, true);
        int n = 0, g = 0;
        while (true) {
            if (lane == 0)
                while (tseq[n % QN] != n + 1) __nanosleep(32);
            __syncwarp();
            __threadfence_block();
            const ExtItem e = tq[n % QN];
            ++n;
            if (e.it < 0) break;
            if (n > 1) {   // the previous item's epilogue has read O_0 / O_1 (completion n - 2)
                EXT_WAIT(bar(BAR_OFREE), uint32_t((n - 2) & 1), 15);
                umma::fence_after();
            }
            bool o_written[2] = {false, false};   // O_k has received a PV in this item
            const int nst = (e.n_pages + PPS - 1) / PPS;
            for (int st = 0; st < nst; ++st, ++g) {
                const int b = g & 1, vs = g % NV, pn = min(PPS, e.n_pages - st * PPS);
                EXT_WAIT(bar(BAR_PFULL + g % NSB), uint32_t((g / NSB) & 1), 7);
                tr(24, g);
                EXT_WAIT(bar(BAR_VFULL + vs), uint32_t((g / NV) & 1), 12);
                tr(25, g);
                umma::fence_after();
                const uint64_t v_desc = umma::desc_mn_sw128(sbase + OFF_V + vs * HALF_BYTES, 2048, 1024);
                if (umma::elect_one()) {
                    for (int pg = 0; pg < pn && !(EXP & 1); ++pg)
                        umma::mma_ts(tmem + O_COL + b * 128, tmem + S_COL + (g % NSB) * KPS + pg * 8,
                                     v_desc + uint64_t((pg * PAGE_BYTES) >> 4), id_o, o_written[b] || pg > 0);
                    umma::commit(bar(BAR_VEMPTY + vs));
                    umma::commit(bar(BAR_PVDONE + g % NSB));
                }
                __syncwarp();
                tr(26, g);
                o_written[b] = true;
            }
            if (umma::elect_one()) umma::commit(bar(BAR_OFULL));   // the item's O is complete
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------ softmax warpgroups
        // WG k (warps 2 + 4k .. 5 + 4k) takes the stages of parity k (global stage counter)
        // with its own running (m, l) and its own O accumulator O_k; PV of stage g adds into
        // O_{g & 1}.  Rescaling O_k waits for the WG's previous PV (pv_done); the next PV into
        // O_k needs this stage's P, so nothing else writes O_k meanwhile.  At item end the two
        // halves merge.
        const int wgk = (warp - 2) >> 2;
        const int row = 32 * (warp & 3) + lane;          // query row = tensor-memory lane
        const uint32_t lane_off = uint32_t(32 * (warp & 3)) << 16;
        const uint32_t o_mine = tmem + lane_off + O_COL + wgk * 128;
        float* ml = reinterpret_cast<float*>(smem + OFF_ML);   // [2 WGs][2][128]: m, l per row
        asm volatile("griddepcontrol.wait;" ::: "memory");   // q and the outputs belong to the stream
        int g = 0;   // g: global stage counter (S buffer g % 3)
        uint32_t oph = 0;
        constexpr float kRescale = 8.f;
        auto wg_sync = [&]() { asm volatile("bar.sync 1, 256;" ::: "memory"); };
        // Items are read ahead through tseq: at the end of item n the next item's member rows
        // and Q half-rows are loaded while the last PVs run, written into tensor memory right
        // after o_full (every S of item n has completed by then), and q_ready lets the S issuer
        // start item n + 1 while this WG's epilogue reads O; the PV issuer waits for o_free.
        struct Rows {
            int lo, hi, mrow, rec, head, tk, tn, tt;   // tk, tn, tt: folded tail (Member::tail_*)
            bool live;
        };
        auto read_entry = [&](int idx) {
            if (lane == 0)
                while (tseq[idx % QN] != idx + 1) __nanosleep(32);
            __syncwarp();
            __threadfence_block();
            return tq[idx % QN];
        };
        auto load_rows = [&](const ExtItem& e, Rows& r, uint4* qv) {
            // padding rows attend to everything (their S is 0: Q is zero) so that their warp
            // keeps the unmasked fast path; their results are never stored
            r = Rows{0, 0x7fffffff, 0, -1, 0, 0, 0, 0, e.it >= 0 && row < e.n_members * G};
            if (r.live) {
                const int mb = row / G;
                const Member m = mems[e.member_off + mb];
                r.lo = m.lo;
                r.hi = m.hi;
                r.mrow = m.row;
                r.rec = m.rec;
                r.tk = m.tail_k0;
                r.tn = m.tail_n;
                r.tt = m.tail_tok;
                r.head = e.kv_head * G + (row - mb * G);
                const uint4* src = reinterpret_cast<const uint4*>(p.q + m.row * p.q_sr + r.head * p.q_sh) + wgk * 8;
#pragma unroll
                for (int u = 0; u < 8; ++u) qv[u] = src[u];
            } else {
#pragma unroll
                for (int u = 0; u < 8; ++u) qv[u] = make_uint4(0u, 0u, 0u, 0u);
            }
        };
        // this WG's half of the Q rows (channels [64 k, 64 k + 64)) into tensor-memory columns
        // Q_COL + 32 k .. (bf16 pairs, lane = row: the A operand layout of S), then q_ready
        auto put_q = [&](const uint4* qv) {
            umma::st32(tmem + lane_off + Q_COL + wgk * 32, reinterpret_cast<const float*>(qv));
            umma::wait_st();
            umma::fence_before();
            mbar_arrive(bar(BAR_QREADY));
        };
        ExtItem e = read_entry(0);
        int n = 1;
        Rows rw;
        {
            uint4 qv[8];
            load_rows(e, rw, qv);
            if (e.it >= 0) put_q(qv);
        }
        while (e.it >= 0) {
            tr(32, n);
            const int lo = rw.lo, hi = rw.hi, tk = rw.tk, tn = rw.tn, tt = rw.tt;
            // a warp whose 32 rows are all padding (R <= 96 of the 128-row tile) skips its tensor-
            // memory traffic: its P / O lanes hold stale values that only feed padding rows
            const bool wdead = 32 * (warp & 3) >= e.n_members * G;
            float m_run = -INFINITY, l_run = 0.f;
            bool mine_any = false;   // did this WG take a stage of the item (O_k written)?
            const int nst = (e.n_pages + PPS - 1) / PPS;
            for (int st = 0; st < nst; ++st, ++g) {
                if (threadIdx.x == 64) {
                    EXT_DBG(8, g);
                    EXT_DBG(9, n);
                }
                if ((g & 1) == wgk) {
                    EXT_WAIT(bar(BAR_SFULL + g % NSB), uint32_t((g / NSB) & 1), 9);
                    tr(30, st);
                    if ((EXP & 2) || wdead) {
                        umma::fence_before();
                        mbar_arrive(bar(BAR_PFULL + g % NSB));
                        mine_any = true;
                        continue;
                    }
                    umma::fence_after();
                    float s[KPS];
#pragma unroll
                    for (int c = 0; c < KPS / 32; ++c)
                        umma::ld32(tmem + lane_off + S_COL + (g % NSB) * KPS + c * 32, s + c * 32);
                    umma::wait_ld();
                    if (trace) {   // make the S-loaded stamp wait for the load's registers
                        float d0, d1;
                        asm volatile("mov.b32 %0, %1;" : "=f"(d0) : "f"(s[0]));
                        asm volatile("mov.b32 %0, %1;" : "=f"(d1) : "f"(s[KPS - 1]));
                        if (d0 == 1.2345f && d1 == 5.4321f) tr(42, st);
                    }
                    tr(37, st);
                    const int npg = min(PPS, e.n_pages - st * PPS);
                    const int tok0 = e.tok_start + st * KPS;
                    const int kmax = min(min(hi, e.tok_end), tok0 + npg * 16);   // keys [max(lo,tok0), kmax) live
                    float mx = -INFINITY;   // max of the raw logits (scale > 0 is applied in the exponent)
                    if (st * PPS + npg <= e.n_main && tok0 >= lo && tok0 + KPS <= kmax) {
#pragma unroll
                        for (int i = 0; i < KPS; ++i) mx = fmaxf(mx, s[i]);
                    } else if (st * PPS + npg <= e.n_main) {
#pragma unroll
                        for (int i = 0; i < KPS; ++i) {
                            const int tok = tok0 + i;
                            s[i] = (tok < kmax && tok >= lo) ? s[i] : -INFINITY;
                            mx = fmaxf(mx, s[i]);
                        }
                    } else {   // the stage reaches folded tail pages: their owner's rows only
#pragma unroll
                        for (int i = 0; i < KPS; ++i) {
                            const int kpg = st * PPS + i / 16;
                            bool ok;
                            if (kpg < e.n_main) {
                                const int tok = tok0 + i;
                                ok = tok < kmax && tok >= lo;
                            } else {
                                const int rel = kpg - tk, tok = tt + rel * 16 + (i & 15);
                                ok = i < npg * 16 && rel >= 0 && rel < tn && tok >= lo && tok < hi;
                            }
                            s[i] = ok ? s[i] : -INFINITY;
                            mx = fmaxf(mx, s[i]);
                        }
                    }
                    mx *= p.scale_log2;
                    tr(41, st);
                    // lazy rescale (P <= 2^kRescale), decided per warp: tensor-memory loads and
                    // stores are warp-collective, so a warp rescales all its rows together
                    const bool grow = mx > m_run + kRescale || (m_run == -INFINITY && mx > -INFINITY);
                    if (__any_sync(0xffffffffu, grow)) {
                        const float mn = fmaxf(m_run, mx);
                        const float al = (m_run == -INFINITY) ? 0.f : fast_exp2(m_run - mn);
                        l_run *= al;
                        m_run = mn;
                        if (mine_any) {   // O_k holds this WG's earlier stages
                            // PV of this WG's previous stage g - 2 may still run: wait for it.  pv_done[(g-2) % 3] completes once per 3
                            // stages; PV g+1 (same buffer) needs P g, so it cannot have
                            // completed yet and the parity of completion (g-2) / 3 is exact.
                            EXT_WAIT(bar(BAR_PVDONE + (g - 2) % NSB), uint32_t(((g - 2) / NSB) & 1), 10);
                            umma::fence_after();
#pragma unroll 1
                            for (int c = 0; c < 4; ++c) {
                                float ov[32];
                                umma::ld32(o_mine + c * 32, ov);
                                umma::wait_ld();
#pragma unroll
                                for (int i = 0; i < 32; ++i) ov[i] *= al;
                                umma::st32(o_mine + c * 32, ov);
                            }
                            umma::wait_st();
                            tr(40, st);
                        }
                    }
                    tr(38, st);
                    const float mu = m_run == -INFINITY ? 0.f : m_run;
                    uint32_t pk[KPS / 2];
                    float lp[4] = {0.f, 0.f, 0.f, 0.f};   // independent partial sums (short add chains)
#pragma unroll
                    for (int i = 0; i < KPS / 2; ++i) {
                        const float e0 = fast_exp2(fmaf(s[2 * i], p.scale_log2, -mu));
                        const float e1 = fast_exp2(fmaf(s[2 * i + 1], p.scale_log2, -mu));
                        lp[i & 3] += e0 + e1;
                        pk[i] = pack_bf16(e0, e1);
                    }
                    l_run += (lp[0] + lp[1]) + (lp[2] + lp[3]);
                    tr(39, st);
#pragma unroll
                    for (int c = 0; c < KPS / 32; ++c)
                        umma::st16(tmem + lane_off + S_COL + (g % NSB) * KPS + c * 16, pk + c * 16);
                    umma::wait_st();
                    umma::fence_before();
                    mbar_arrive(bar(BAR_PFULL + g % NSB));
                    tr(31, st);
                    mine_any = true;
                }
            }
            // ---- the next item: rows + Q loads in flight while the last PVs run
            const ExtItem nx = read_entry(n);
            ++n;
            Rows rn;
            uint4 qn[8];
            load_rows(nx, rn, qn);
            // ---- epilogue: both O halves complete; merge the two WGs' softmax states per row
            tr(34, n);
            EXT_WAIT(bar(BAR_OFULL), oph, 6);
            oph ^= 1u;
            tr(35, n);
            umma::fence_after();
            if (nx.it >= 0) put_q(qn);   // every S of this item completed before o_full
            const bool live = rw.live;
            const int mrow = rw.mrow, rec = rw.rec, head = rw.head;
            ml[(wgk * 2 + 0) * 128 + row] = m_run;
            ml[(wgk * 2 + 1) * 128 + row] = l_run;
            const uint32_t used = __ballot_sync(0xffffffffu, mine_any);   // uniform per WG
            if (lane == 0) reinterpret_cast<volatile uint32_t*>(ml + 512)[warp - 2] = used != 0;
            wg_sync();
            const float m0 = ml[row], l0 = ml[128 + row], m1 = ml[256 + row], l1 = ml[384 + row];
            const bool have0 = reinterpret_cast<volatile uint32_t*>(ml + 512)[(warp & 3) ^ 2] != 0;   // WG0 warp, same lanes
            const bool have1 = reinterpret_cast<volatile uint32_t*>(ml + 512)[4 + ((warp & 3) ^ 2)] != 0;
            const float M = fmaxf(m0, m1);
            const float a0 = m0 == -INFINITY ? 0.f : fast_exp2(m0 - M), a1 = m1 == -INFINITY ? 0.f : fast_exp2(m1 - M);
            const float L = l0 * a0 + l1 * a1;
            const float inv = L > 0.f ? 1.f / L : 0.f;
            const float w0 = a0 * inv, w1 = a1 * inv;
            // WG k writes output columns [64 k, 64 k + 64)
#pragma unroll 1
            for (int c = 0; c < 2 && !wdead; ++c) {
                const int col = wgk * 64 + c * 32;
                float o0[32], o1[32];
                if (have0) {
                    umma::ld32(tmem + lane_off + O_COL + col, o0);
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) o0[i] = 0.f;
                }
                if (have1) {
                    umma::ld32(tmem + lane_off + O_COL + 128 + col, o1);
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) o1[i] = 0.f;
                }
                umma::wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) o0[i] = o0[i] * w0 + o1[i] * w1;
                if (live && rec < 0) {
                    uint4* dst = reinterpret_cast<uint4*>(p.o + mrow * p.o_sr + head * p.o_sh + col);
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        dst[u] = make_uint4(pack_bf16(o0[8 * u], o0[8 * u + 1]), pack_bf16(o0[8 * u + 2], o0[8 * u + 3]),
                                            pack_bf16(o0[8 * u + 4], o0[8 * u + 5]),
                                            pack_bf16(o0[8 * u + 6], o0[8 * u + 7]));
                } else if (live) {
                    float4* dst = reinterpret_cast<float4*>(p.part_o + ((long long)rec * Hq + head) * D + col);
#pragma unroll
                    for (int u = 0; u < 8; ++u) dst[u] = make_float4(o0[4 * u], o0[4 * u + 1], o0[4 * u + 2], o0[4 * u + 3]);
                }
            }
            if (wgk == 0 && live) {
                const float lse = L > 0.f ? (M + log2f(L)) * 0.69314718055994531f : -INFINITY;
                if (rec < 0) {
                    if (p.lse) p.lse[mrow * p.l_sr + head * p.l_sh] = lse;
                } else {
                    p.part_lse[(long long)rec * Hq + head] = lse;
                }
            }
            umma::fence_before();
            mbar_arrive(bar(BAR_OFREE));   // O_0 / O_1 may take the next item's PVs
            wg_sync();   // ml is rewritten at the next item's end
            tr(36, n);
            e = nx;
            rw = rn;
        }
    }

    // ---- teardown: free tensor memory; the last CTA rewinds the queue slot
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    if (p.trace && threadIdx.x == 0 && int(blockIdx.x) < p.trace_cap) {   // per-CTA (start, end) in row 7
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        p.trace[2ull * (7ull * p.trace_cap + blockIdx.x) + 1] = gt;
    }
    if (warp == 1) umma::tmem_dealloc(tmem, TMEM_COLS);
    if (threadIdx.x == 0) {
        if (atomicAdd(sched + 1, 1) == int(gridDim.x) - 1) {
            sched[0] = 0;
            sched[1] = 0;
            sched[32] = 0;
            st_release_gpu(sched + 3, p.launch + kSchedSlots);
        }
    }
}

bool ext_supported(int head_dim) { return head_dim == ext::D; }

int launch_ext(const spa_plan* P, int32_t layer, const void* q, int64_t q_sr, int64_t q_sh, void* o, int64_t o_sr,
               int64_t o_sh, float* lse, int64_t l_sr, int64_t l_sh, float scale, void* stream) {
    const auto& c = P->pool->cfg;
    const int32_t* H = P->host.data();
    if (H[H_N_ITEMS] == 0) return 0;
    static std::atomic<unsigned long long> attr_done{0};
    if (int e = set_smem_attr_once(ext_kernel, ext::SMEM, &attr_done)) return e;
    // 16-B vector loads of q rows and stores of o rows
    if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(o)) % 16 || q_sr % 8 || q_sh % 8 || o_sr % 8 ||
        o_sh % 8)
        return int(cudaErrorMisalignedAddress);
    ExtParams ep{};
    ep.meta = P->d_meta;
    ep.q = static_cast<const __nv_bfloat16*>(q);
    ep.q_sr = q_sr;
    ep.q_sh = q_sh;
    ep.o = static_cast<__nv_bfloat16*>(o);
    ep.o_sr = o_sr;
    ep.o_sh = o_sh;
    ep.lse = lse;
    ep.l_sr = l_sr;
    ep.l_sh = l_sh;
    ep.part_o = P->d_part_o;
    ep.part_lse = P->d_part_lse;
    ep.scale_log2 = float(double(scale) * 1.4426950408889634);
    ep.layer_row_base = layer * c.num_pages * c.num_kv_heads * kPageSize;
    ep.num_q_heads = c.num_q_heads;
    ep.num_kv_heads = c.num_kv_heads;
    ep.group_size = c.num_q_heads / c.num_kv_heads;
    ep.launch = int(P->launches++);
    ep.trace = P->trace;
    ep.trace_cap = P->trace_cap;
    const CUtensorMap* tk = reinterpret_cast<const CUtensorMap*>(P->pool->tmap_k1.bytes);
    const CUtensorMap* tv = reinterpret_cast<const CUtensorMap*>(P->pool->tmap_v.bytes);
    int err = launch_pdl(ext_kernel, dim3(P->num_ctas), dim3(ext::THREADS), ext::SMEM, stream, *tk, *tv, ep);
    if (err) return err;
    // split partials: one warp per merge subtask of the plan in its own launch (programmatic
    // dependent launch; an in-kernel tail merge measured slower: the merges wait for the last
    // items, and its registers spill in the streaming loops)
    if (H[H_N_RECORDS] > 0) err = launch_merge_tasks(P, o, o_sr, o_sh, lse, l_sr, l_sh, stream);
    return err;
}

}  // namespace spa
