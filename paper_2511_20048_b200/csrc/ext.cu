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
//   warp 0      producer: pops items from the plan's dynamic queue and streams each stage
//               (2 pages of K and V of one KV head, 16 KB) into a 12-stage shared-memory
//               ring with one 3-D TMA box per (page, tensor);
//   warp 1      MMA issuer (one thread): S_j = Q K_j^T (per page: 8 x M128 N16 K16, A = the
//               item's Q tile, K-major SW128; B = the K page as TMA wrote it), then
//               O += P_{j-1} V_{j-1} (per page: M128 N128 K16, A = P in tensor memory,
//               B = the V page as an MN-major SW128 operand);
//   warps 2-5   softmax warpgroup, one thread per query row (tensor-memory lane): loads S_j,
//               masks (window lo, causal hi, range end), runs the online softmax in the
//               log2 domain with lazy rescaling of O (threshold 2^8, O rescaled in tensor
//               memory), writes P_j (bf16) over S_j's columns, and at item end normalises
//               O and writes bf16 O + LSE (or an fp32 partial record for split ranges).
// S is double-buffered in tensor memory (2 x 32 columns), O takes 128 columns.
#include "device_util.cuh"
#include "spa_internal.h"
#include "umma.cuh"

namespace spa {

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
};

struct ExtItem {
    int it, kv_head, n_pages, tok_start, tok_end, member_off, n_members, kind;
};

namespace ext {
constexpr int D = 128;
constexpr int PAGE_BYTES = kPageSize * D * 2;     // 4 KB: K (or V) of one page, one head
constexpr int STAGE_BYTES = 2 * 2 * PAGE_BYTES;   // 2 pages x (K, V)
constexpr int NS = 12;                            // ring stages
constexpr int QN = NS + 2;                        // popped-item queue entries
constexpr int OFF_Q = NS * STAGE_BYTES;           // Q tile: 2 chunks x 128 rows x 128 B
constexpr int OFF_BAR = OFF_Q + 32768;
// barriers: full[NS], empty[NS], s_full[2], p_full[2], q_ready, o_full, pv_done
constexpr int BAR_FULL = 0, BAR_EMPTY = NS, BAR_SFULL = 2 * NS, BAR_PFULL = 2 * NS + 2, BAR_QREADY = 2 * NS + 4,
              BAR_OFULL = 2 * NS + 5, BAR_PVDONE = 2 * NS + 6, N_BARS = 2 * NS + 7;
constexpr int OFF_TQ = OFF_BAR + N_BARS * 8;
constexpr int OFF_TSLOT = OFF_TQ + QN * int(sizeof(ExtItem));
constexpr int SMEM = 1024 + OFF_TSLOT + 16;
constexpr int THREADS = 192;
constexpr uint32_t TMEM_COLS = 256, S_COL = 0, O_COL = 128;
static_assert(SMEM <= 232448, "extend kernel shared memory");
}  // namespace ext

__global__ void __launch_bounds__(ext::THREADS, 1)
    ext_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv, const ExtParams p) {
    using namespace ext;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    auto bar = [&](int i) { return sbase + OFF_BAR + i * 8; };
    ExtItem* tq = reinterpret_cast<ExtItem*>(smem + OFF_TQ);

    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(bar(BAR_FULL + i), 1);
            mbar_init(bar(BAR_EMPTY + i), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(bar(BAR_SFULL + b), 1);
            mbar_init(bar(BAR_PFULL + b), 128);
        }
        mbar_init(bar(BAR_QREADY), 128);
        mbar_init(bar(BAR_OFULL), 1);
        mbar_init(bar(BAR_PVDONE), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) umma::tmem_alloc(sbase + OFF_TSLOT, TMEM_COLS);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + OFF_TSLOT);
    asm volatile("griddepcontrol.launch_dependents;");

    const int32_t* meta = p.meta;
    const Desc* descs = reinterpret_cast<const Desc*>(meta + meta[H_OFF_DESC]);
    const Member* mems = reinterpret_cast<const Member*>(meta + meta[H_OFF_MEMBER]);
    const Item* items = reinterpret_cast<const Item*>(meta + meta[H_OFF_ITEM]);
    const int32_t* queue = meta + meta[H_OFF_QUEUE];
    const int32_t* pages = meta + meta[H_OFF_PAGES];
    int32_t* sched = const_cast<int32_t*>(meta) + meta[H_OFF_SCHED] + kSchedStride * (p.launch % kSchedSlots);
    const int n_items = meta[H_N_ITEMS];
    const int G = p.group_size, Hq = p.num_q_heads, Hkv = p.num_kv_heads;
    (void)Hq;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        uint64_t policy = 0;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
        bool waited = false;
        int slot = 0, n = 0;
        uint32_t ph = 0;
        for (int k = 0;; ++k) {
            int qi = 0;
            if (lane == 0) {
                if (k == 0)   // the queue slot is ours once launch - kSchedSlots rewound it
                    for (unsigned ns = 64; ld_acquire_gpu(sched + 3) != p.launch; ns = min(ns * 2, 1024u))
                        __nanosleep(ns);
                qi = atomicAdd(sched, 1);
            }
            qi = __shfl_sync(0xffffffffu, qi, 0);
            const int it = qi < n_items ? queue[qi] : -1;
            ExtItem* e = &tq[n % QN];
            ++n;
            // the ring slot for this item's first stage (or the end marker)
            mbar_wait(bar(BAR_EMPTY + slot), ph ^ 1u);
            if (it < 0) {
                if (lane == 0) {
                    e->it = -1;
                    mbar_arrive(bar(BAR_FULL + slot));
                }
                break;
            }
            const Item itm = items[it];
            const Desc dsc = descs[itm.desc];
            if (lane == 0)
                *e = ExtItem{it, itm.kv_head, dsc.n_pages, dsc.tok_start, dsc.tok_end, dsc.member_off, dsc.n_members,
                             dsc.kind};
            if ((dsc.kind & 4) && !waited) {   // holds newest tokens: wait for their producer
                asm volatile("griddepcontrol.wait;" ::: "memory");
                waited = true;
            }
            int pid_cur = lane < dsc.n_pages ? pages[dsc.page_off + lane] : 0;
            int pid_base = 0;
            const int nst = (dsc.n_pages + 1) / 2;
            for (int st = 0; st < nst; ++st) {
                if (st > 0) mbar_wait(bar(BAR_EMPTY + slot), ph ^ 1u);
                const int p0 = st * 2, npg = min(2, dsc.n_pages - p0);
                int row[2];
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int kk = p0 + j;
                    if (kk >= pid_base + 32) {
                        pid_base += 32;
                        pid_cur = pid_base + lane < dsc.n_pages ? pages[dsc.page_off + pid_base + lane] : 0;
                    }
                    const int page = __shfl_sync(0xffffffffu, pid_cur, (kk - pid_base) & 31);
                    row[j] = p.layer_row_base + (page * Hkv + itm.kv_head) * kPageSize;
                }
                if (lane == 0) {
                    const uint32_t fb = bar(BAR_FULL + slot);
                    mbar_expect_tx(fb, npg * 2 * PAGE_BYTES);
                    const uint32_t sb = sbase + slot * STAGE_BYTES;
                    for (int j = 0; j < npg; ++j) {
                        tma_load_3d(sb + j * 2 * PAGE_BYTES, &tmk, 0, row[j], 0, fb, policy);
                        tma_load_3d(sb + j * 2 * PAGE_BYTES + PAGE_BYTES, &tmv, 0, row[j], 0, fb, policy);
                    }
                }
                __syncwarp();
                if (++slot == NS) {
                    slot = 0;
                    ph ^= 1u;
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t id_s = umma::idesc_bf16_f32(128, 16, false, false);
            const uint32_t id_o = umma::idesc_bf16_f32(128, 128, false, true);
            const uint32_t QB = sbase + OFF_Q;
            int slot = 0, n = 0;
            uint32_t ph = 0, qph = 0;
            uint32_t pph[2] = {0, 0};
            int g = 0;   // running stage counter (S buffer = g & 1)
            while (true) {
                mbar_wait(bar(BAR_FULL + slot), ph);
                const ExtItem e = tq[n % QN];
                ++n;
                if (e.it < 0) break;
                mbar_wait(bar(BAR_QREADY), qph);   // Q tile written (and the last item's O read out)
                qph ^= 1u;
                umma::fence_after();
                const int nst = (e.n_pages + 1) / 2;
                int prev_slot = 0, prev_npg = 0;
                for (int st = 0; st < nst; ++st, ++g) {
                    if (st > 0) mbar_wait(bar(BAR_FULL + slot), ph);
                    umma::fence_after();
                    const int npg = min(2, e.n_pages - st * 2);
                    const uint32_t sb = sbase + slot * STAGE_BYTES;
                    const uint32_t sbuf = tmem + S_COL + (g & 1) * 32;
                    for (int pg = 0; pg < npg; ++pg)
#pragma unroll
                        for (int ks = 0; ks < D / 16; ++ks) {
                            const uint64_t a = umma::desc_k_sw128(QB + (ks >> 2) * 16384 + (ks & 3) * 32, 1024);
                            const uint64_t b =
                                umma::desc_k_sw128(sb + pg * 2 * PAGE_BYTES + (ks >> 2) * 2048 + (ks & 3) * 32, 1024);
                            umma::mma_ss(sbuf + pg * 16, a, b, id_s, ks > 0);
                        }
                    umma::commit(bar(BAR_SFULL + (g & 1)));
                    if (st > 0) {   // O += P_{g-1} V_{g-1}
                        const int b = (g - 1) & 1;
                        mbar_wait(bar(BAR_PFULL + b), pph[b]);
                        pph[b] ^= 1u;
                        umma::fence_after();
                        const uint32_t psb = sbase + prev_slot * STAGE_BYTES;
                        for (int pg = 0; pg < prev_npg; ++pg)
                            umma::mma_ts(tmem + O_COL, tmem + S_COL + b * 32 + pg * 8,
                                         umma::desc_mn_sw128(psb + pg * 2 * PAGE_BYTES + PAGE_BYTES, 2048, 1024), id_o,
                                         st > 1 || pg > 0);
                        umma::commit(bar(BAR_EMPTY + prev_slot));
                        umma::commit(bar(BAR_PVDONE));
                    }
                    prev_slot = slot;
                    prev_npg = npg;
                    if (++slot == NS) {
                        slot = 0;
                        ph ^= 1u;
                    }
                }
                {   // the item's last PV, then O is complete
                    const int b = (g - 1) & 1;
                    mbar_wait(bar(BAR_PFULL + b), pph[b]);
                    pph[b] ^= 1u;
                    umma::fence_after();
                    const uint32_t psb = sbase + prev_slot * STAGE_BYTES;
                    for (int pg = 0; pg < prev_npg; ++pg)
                        umma::mma_ts(tmem + O_COL, tmem + S_COL + b * 32 + pg * 8,
                                     umma::desc_mn_sw128(psb + pg * 2 * PAGE_BYTES + PAGE_BYTES, 2048, 1024), id_o,
                                     nst > 1 || pg > 0);
                    umma::commit(bar(BAR_EMPTY + prev_slot));
                    umma::commit(bar(BAR_OFULL));
                }
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ softmax warpgroup
        const int row = 32 * (warp & 3) + lane;          // query row = tensor-memory lane
        const uint32_t lane_off = uint32_t(32 * (warp & 3)) << 16;
        const uint32_t q_row = smem_u32(smem + OFF_Q);
        asm volatile("griddepcontrol.wait;" ::: "memory");   // q and the outputs belong to the stream
        int slot = 0, n = 0, g = 0;
        uint32_t ph = 0, oph = 0, pvph = 0;
        uint32_t sph[2] = {0, 0};
        constexpr float kRescale = 8.f;
        while (true) {
            mbar_wait(bar(BAR_FULL + slot), ph);   // the item's first stage landed: its entry is valid
            const ExtItem e = tq[n % QN];
            ++n;
            if (e.it < 0) break;
            const int R = e.n_members * G;
            // ---- row setup + Q tile (K-major SW128: chunk c of row r at c * 16 KB + sw128(r, u))
            int lo = 0, hi = 0, mrow = 0, rec = -1, head = 0;
            const bool live = row < R;
            uint4 qv[16];
            if (live) {
                const int mb = row / G;
                const Member m = mems[e.member_off + mb];
                lo = m.lo;
                hi = m.hi;
                mrow = m.row;
                rec = m.rec;
                head = e.kv_head * G + (row - mb * G);
                const uint4* src = reinterpret_cast<const uint4*>(p.q + m.row * p.q_sr + head * p.q_sh);
#pragma unroll
                for (int u = 0; u < 16; ++u) qv[u] = src[u];
            } else {
#pragma unroll
                for (int u = 0; u < 16; ++u) qv[u] = make_uint4(0u, 0u, 0u, 0u);
            }
#pragma unroll
            for (int u = 0; u < 16; ++u)
                *reinterpret_cast<uint4*>(smem + OFF_Q + (u >> 3) * 16384 + umma::sw128_offset(row, u & 7)) = qv[u];
            umma::fence_proxy_async_smem();
            mbar_arrive(bar(BAR_QREADY));
            (void)q_row;

            float m_run = -INFINITY, l_run = 0.f;
            const int nst = (e.n_pages + 1) / 2;
            for (int st = 0; st < nst; ++st, ++g) {
                const int b = g & 1;
                mbar_wait(bar(BAR_SFULL + b), sph[b]);
                sph[b] ^= 1u;
                umma::fence_after();
                float s[32];
                umma::ld32(tmem + lane_off + S_COL + b * 32, s);
                umma::wait_ld();
                const int npg = min(2, e.n_pages - st * 2);
                const int tok0 = e.tok_start + st * 32;
                const int kmax = min(min(hi, e.tok_end), tok0 + npg * 16);   // keys [max(lo,tok0), kmax) live
                float mx = -INFINITY;
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const int tok = tok0 + i;
                    const float v = (tok < kmax && tok >= lo) ? s[i] * p.scale_log2 : -INFINITY;
                    s[i] = v;
                    mx = fmaxf(mx, v);
                }
                if (st > 0) {   // O holds P_{<st} V: PV of the previous stage must be complete
                    mbar_wait(bar(BAR_PVDONE), pvph);
                    pvph ^= 1u;
                }
                // lazy rescale (P <= 2^kRescale), decided per warp: tensor-memory loads and
                // stores are warp-collective, so a warp rescales all its rows together
                const bool grow = mx > m_run + kRescale || (m_run == -INFINITY && mx > -INFINITY);
                if (__any_sync(0xffffffffu, grow)) {
                    const float mn = fmaxf(m_run, mx);
                    const float al = (m_run == -INFINITY) ? 0.f : fast_exp2(m_run - mn);
                    l_run *= al;
                    m_run = mn;
                    if (st > 0) {
                        umma::fence_after();
#pragma unroll 1
                        for (int c = 0; c < 4; ++c) {
                            float ov[32];
                            umma::ld32(tmem + lane_off + O_COL + c * 32, ov);
                            umma::wait_ld();
#pragma unroll
                            for (int i = 0; i < 32; ++i) ov[i] *= al;
                            umma::st32(tmem + lane_off + O_COL + c * 32, ov);
                        }
                        umma::wait_st();
                    }
                }
                const float mu = m_run == -INFINITY ? 0.f : m_run;
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const float e0 = fast_exp2(s[2 * i] - mu), e1 = fast_exp2(s[2 * i + 1] - mu);
                    l_run += e0 + e1;
                    pk[i] = pack_bf16(e0, e1);
                }
                umma::st16(tmem + lane_off + S_COL + b * 32, pk);
                umma::wait_st();
                umma::fence_before();
                mbar_arrive(bar(BAR_PFULL + b));
                if (++slot == NS) {
                    slot = 0;
                    ph ^= 1u;
                }
                if (st + 1 < nst) mbar_wait(bar(BAR_FULL + slot), ph);   // keep the item walk in step
            }
            // ---- epilogue: O complete in tensor memory
            mbar_wait(bar(BAR_OFULL), oph);
            oph ^= 1u;
            umma::fence_after();
            const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
            const float lse = l_run > 0.f ? (m_run + log2f(l_run)) * 0.69314718055994531f : -INFINITY;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {   // warp-collective loads; live rows store
                float ov[32];
                umma::ld32(tmem + lane_off + O_COL + c * 32, ov);
                umma::wait_ld();
                if (live && rec < 0) {
                    uint4* dst = reinterpret_cast<uint4*>(p.o + mrow * p.o_sr + head * p.o_sh + c * 32);
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        dst[u] = make_uint4(pack_bf16(ov[8 * u] * inv, ov[8 * u + 1] * inv),
                                            pack_bf16(ov[8 * u + 2] * inv, ov[8 * u + 3] * inv),
                                            pack_bf16(ov[8 * u + 4] * inv, ov[8 * u + 5] * inv),
                                            pack_bf16(ov[8 * u + 6] * inv, ov[8 * u + 7] * inv));
                } else if (live) {
                    float4* dst = reinterpret_cast<float4*>(p.part_o + ((long long)rec * Hq + head) * D + c * 32);
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        dst[u] =
                            make_float4(ov[4 * u] * inv, ov[4 * u + 1] * inv, ov[4 * u + 2] * inv, ov[4 * u + 3] * inv);
                }
            }
            if (live && rec < 0) {
                if (p.lse) p.lse[mrow * p.l_sr + head * p.l_sh] = lse;
            } else if (live) {
                p.part_lse[(long long)rec * Hq + head] = lse;
            }
            umma::fence_before();
        }
    }

    // ---- teardown: free tensor memory; the last CTA rewinds the queue slot
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
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
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(ext_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ext::SMEM);
        if (e) return int(e);
        attr_set = true;
    }
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
    const CUtensorMap* tk = reinterpret_cast<const CUtensorMap*>(P->pool->tmap_k.bytes);
    const CUtensorMap* tv = reinterpret_cast<const CUtensorMap*>(P->pool->tmap_v.bytes);
    int err = launch_pdl(ext_kernel, dim3(P->num_ctas), dim3(ext::THREADS), ext::SMEM, stream, *tk, *tv, ep);
    if (err) return err;
    if (H[H_N_RECORDS] > 0)
        err = launch_merge(H[H_N_REQ], c.num_q_heads, c.head_dim, P->d_meta + H[H_OFF_REC_PTR], P->d_part_o,
                           P->d_part_lse, o, o_sr, o_sh, lse, l_sr, l_sh, P->num_ctas, stream);
    return err;
}

}  // namespace spa
