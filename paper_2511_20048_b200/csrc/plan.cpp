// Step planner: groups, splits, work items, static schedule.
//
// A decode batch under SPAgent holds main requests and the k speculative samples forked
// from each one's context c_i (PAPER.md:189, :198, :292 Table I, :335).  Requests whose
// page tables start with the same page id form a group; the group's shared region is the
// longest common page-id prefix of its members (reading #18).  For every KV head:
//   - one work descriptor per split of the shared region carries ALL R = members x G
//     query rows, so each shared page is read once per (KV head, group);
//   - each member's private tail [S, n_m) is its own descriptor (its rows only).
// Sliding windows (reading #9) restrict every range to the union of the members'
// windows; per-member lower bounds are applied as masks inside the kernel.
// Splits are sized so the persistent grid (num_ctas CTAs x teams) is balanced by a
// longest-processing-time (LPT) static assignment; a request that ends up in more than
// one descriptor gets fp32 partial records that spa_merge_splits combines.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <queue>
#include <unordered_map>
#include <unordered_set>

#include "../../include/spa_debug.h"
#include "spa_internal.h"

namespace spa {

int plan_upload(spa_plan* P, void* stream);  // kernels.cu
void plan_release(spa_plan* P);               // kernels.cu

namespace {

struct Fold {                  // a member tail read by its host range's last descriptor
    std::vector<int> rows;
    int32_t a, b;
    const std::vector<int32_t>* table;
};

struct Range {
    int kind;                 // bit 0: a row of the range also reads another range (partial records)
    int group;
    std::vector<int> members; // batch rows
    int32_t a, b;             // tokens [a, b)
    const std::vector<int32_t>* table;
    std::vector<Fold> folds;  // member tails appended to the range's last descriptor
};

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace
}  // namespace spa

using namespace spa;

extern "C" {

// Kernel geometry of a plan with `mt` 16-row tiles per item: teams per CTA and key-split
// warps per row tile.  32-row items take one warp per row tile over every page of a stage
// (kw 1, 4 teams: measured 1.4x the key-split layout at k = 3, profiles/r02_*).  fp8 pools
// take kw 1 for 16-row items too: 8 one-warp teams (each warp its own ring and producer: no
// partner to wait for at every stage, no column-half exchange at item end) measured 93 ->
// 80 us per layer on BJ config 1 (profiles/r02_fp8_kw1.txt); bf16 16-row items keep the
// key-split pairs (one-warp teams fit only one bf16 page per stage: 113 vs 112 us, Gemma
// local 116 vs 103 us).  An explicit teams_per_cta the kw-1 layout does not support keeps kw 2.
static spa_status set_geometry(spa_plan* P, int mt, int teams_req) {
    P->mt = mt;
    const bool fp8 = P->pool->kv_fp8;
    int teams = teams_req;
    if (const char* e = std::getenv("SPA_TEAMS")) teams = std::atoi(e);
    P->teams_auto = teams == 0;
    int kw = mt == 2 || (fp8 && mt == 1) ? 1 : 2;
    if (const char* e = std::getenv("SPA_KW")) kw = std::atoi(e) == 1 && mt <= 2 ? 1 : 2;
    if (teams == 0) teams = kw == 1 ? (mt == 1 ? 8 : 4) : mt == 1 ? 4 : mt == 2 ? 2 : 1;
    else if (kw == 1 && !decode_teams_supported(mt, teams, 1)) kw = 2;
    if (!decode_teams_supported(mt, teams, kw))
        return fail(SPA_ERR_UNSUPPORTED,
                    "teams_per_cta must be 1, 2 or 4 (4 only with max_rows 16 or 32, 1 with 64; 8 with one-warp teams)");
    P->teams = teams;
    P->kw = kw;
    P->n_teams = P->num_ctas * teams;
    return SPA_OK;
}

spa_status spa_plan_create(spa_pool* pool, const spa_plan_config* cfg, spa_plan** out) {
    if (!pool || !out) return fail(SPA_ERR_INVALID_ARG, "null argument");
    *out = nullptr;
    spa_plan_config c{};
    c.sharing = 1;
    if (cfg) c = *cfg;
    if (c.max_rows != 0 && c.max_rows != 16 && c.max_rows != 32 && c.max_rows != 64 && c.max_rows != 128)
        return fail(SPA_ERR_UNSUPPORTED, "max_rows must be 0 (auto), 16, 32, 64 or 128");
    if (c.max_rows == 128 && !ext_supported(pool->cfg.head_dim))
        return fail(SPA_ERR_UNSUPPORTED, "max_rows 128 (tcgen05 extend kernel) needs head_dim 128");
    if (c.split_pages < 0 || c.num_ctas < 0) return fail(SPA_ERR_INVALID_ARG, "negative plan option");
    if (c.merge_mode < 0 || c.merge_mode > 2) return fail(SPA_ERR_INVALID_ARG, "merge_mode must be 0, 1 or 2");
    if (c.max_rows == 0 && c.teams_per_cta != 0)
        return fail(SPA_ERR_INVALID_ARG, "max_rows 0 (auto) chooses teams_per_cta itself: pass 0");
    const int G = pool->cfg.num_q_heads / pool->cfg.num_kv_heads;
    if (G > (c.max_rows ? c.max_rows : 32)) return fail(SPA_ERR_UNSUPPORTED, "GQA group size exceeds max_rows");
    if (c.max_rows == 128 && c.merge_mode != 2 && c.merge_mode != 0)
        return fail(SPA_ERR_UNSUPPORTED, "max_rows 128 merges split partials with the merge kernel");
    spa_plan* P = new spa_plan();
    P->pool = pool;
    P->cfg = c;
    P->auto_rows = c.max_rows == 0;
    int ctas = c.num_ctas;
    if (ctas == 0) ctas = pool->sm_count > 0 ? pool->sm_count : 148;
    P->num_ctas = ctas;
    const int mt = c.max_rows ? c.max_rows / 16 : (G > 16 ? 2 : 1);
    if (spa_status st = set_geometry(P, mt, c.teams_per_cta)) {
        delete P;
        return st;
    }
    *out = P;
    return SPA_OK;
}

spa_status spa_plan_destroy(spa_plan* plan) {
    if (!plan) return SPA_OK;
    plan_release(plan);
    delete plan;
    return SPA_OK;
}

}  // extern "C"

namespace {

// One query row of the batch: a token of a request that attends to keys [lo, hi) of the
// request's KV (hi = its causal length, position + 1); `first_new` = the request's first
// token appended in this step (descriptors holding keys >= first_new are produced right
// before attention: the kernel does not prefetch them ahead of its dependency wait).
struct VRow {
    const Request* req;
    int32_t hi, first_new;
};

spa_status plan_rows(spa_plan* P, const std::vector<VRow>& V, int32_t window, void* stream);

}  // namespace

extern "C" {

spa_status spa_decode_plan(spa_plan* P, int32_t n_req, const spa_req* reqs, int32_t window, void* stream) {
    return spa_extend_plan(P, n_req, reqs, nullptr, window, stream);
}

spa_status spa_extend_plan(spa_plan* P, int32_t n_req, const spa_req* reqs, const int32_t* n_query, int32_t window,
                           void* stream) {
    if (!P) return fail(SPA_ERR_INVALID_ARG, "null plan");
    spa_pool* pool = P->pool;
    if (spa_status s = check_device(pool)) return s;
    if (n_req < 0 || (n_req > 0 && !reqs)) return fail(SPA_ERR_INVALID_ARG, "bad request list");
    std::vector<VRow> V;
    V.reserve(size_t(n_req));
    std::unordered_set<int64_t> seen;
    for (int i = 0; i < n_req; ++i)
        if (!seen.insert(reqs[i]).second) return fail(SPA_ERR_INVALID_ARG, "plan: request listed twice");
    for (int i = 0; i < n_req; ++i) {
        auto it = pool->reqs.find(reqs[i]);
        if (it == pool->reqs.end()) return fail(SPA_ERR_BAD_REQUEST, "plan: unknown request " + std::to_string(reqs[i]));
        const Request* r = &it->second;
        if (r->len <= 0) return fail(SPA_ERR_INVALID_ARG, "plan: decode over an empty request (reading #11)");
        const int32_t nq = n_query ? n_query[i] : 1;
        if (nq < 1 || nq > r->len) return fail(SPA_ERR_INVALID_ARG, "plan: n_query must be in [1, request length]");
        for (int32_t t = 0; t < nq; ++t) V.push_back(VRow{r, r->len - nq + t + 1, r->len - nq});
    }
    if (V.size() > size_t(1) << 30) return fail(SPA_ERR_INVALID_ARG, "plan: too many query rows");
    return plan_rows(P, V, window, stream);
}

}  // extern "C"

namespace {

spa_status plan_rows(spa_plan* P, const std::vector<VRow>& V, int32_t window, void* stream) {
    spa_pool* pool = P->pool;
    const int ps = pool->cfg.page_size;
    const int Hkv = pool->cfg.num_kv_heads;
    const int G = pool->cfg.num_q_heads / Hkv;
    const int n_req = int(V.size());   // query rows
    if (ps > 32) return fail(SPA_ERR_UNSUPPORTED, "plan: page_size > 32 (the planner keeps a 32-bit slot mask per page)");
    // window (reading #9): a query at position p attends to keys [p + 1 - W, p]
    std::vector<int32_t> lo(n_req);
    for (int i = 0; i < n_req; ++i) lo[i] = window > 0 ? std::max<int32_t>(0, V[i].hi - window) : 0;

    // ---- 1. groups (requests that share page ids; sharing off: each request alone), then
    //      sub-groups of at most max_rows / G rows (the rows of a request stay consecutive).
    //      Page ids are positional (a shared page sits at the same index in every table
    //      holding it).  Without released pages this is "same first page"; after
    //      spa_kv_release_window the members of a family may have released different
    //      leading pages, so requests are joined when one of a request's first kLinkPages
    //      resident pages is held by another.
    std::vector<int32_t> d(n_req, 0);   // index of the first resident page
    for (int i = 0; i < n_req; ++i) {
        const auto& t = V[i].req->pages;
        while (d[i] < int32_t(t.size()) && t[d[i]] < 0) ++d[i];
    }
    std::vector<std::vector<int>> groups;
    {
        std::vector<int> parent(n_req);
        for (int i = 0; i < n_req; ++i) parent[i] = i;
        auto find = [&](int x) {
            while (parent[x] != x) x = parent[x] = parent[parent[x]];
            return x;
        };
        if (P->cfg.sharing) {
            // Sharing is positional and prefix-shaped (a fork shares its parent's first pages,
            // spa_kv_release_window drops a prefix), so two requests share a resident page iff
            // they hold the same page at index max(d_i, d_j).  Probing every request at every
            // distinct first-resident index D (one index, 0, without releases) finds exactly
            // those pairs: O(N |D|) hash probes instead of one per resident page.
            std::vector<int32_t> D(d.begin(), d.end());
            std::sort(D.begin(), D.end());
            D.erase(std::unique(D.begin(), D.end()), D.end());
            std::unordered_map<int32_t, int> holder;
            holder.reserve(size_t(n_req) * 2);
            for (int i = 0; i < n_req; ++i) {
                const auto& t = V[i].req->pages;
                for (auto k = std::lower_bound(D.begin(), D.end(), d[i]); k != D.end() && *k < int32_t(t.size()); ++k) {
                    auto ins = holder.emplace(t[*k], i);
                    if (!ins.second) {   // another request holds this page: same family
                        const int a = find(i), b = find(ins.first->second);
                        if (a != b) parent[std::max(a, b)] = std::min(a, b);
                    }
                }
            }
        } else {
            // rows of one request (extend) stay together
            std::unordered_map<const Request*, int> first;
            for (int i = 0; i < n_req; ++i) {
                auto ins = first.emplace(V[i].req, i);
                if (!ins.second) parent[i] = ins.first->second;
            }
        }
        std::unordered_map<int, int> gi;
        for (int i = 0; i < n_req; ++i) {
            auto ins = gi.emplace(find(i), int(groups.size()));
            if (ins.second) groups.emplace_back();
            groups[ins.first->second].push_back(i);
        }
    }

    // ---- 2. ranges: a prefix tree of page-id runs per group (reading #18).  Sharing is
    //      positional and prefix-shaped, so over page index k the requests of a group that
    //      hold the same page at k form a class, and classes only split as k grows (between
    //      the indices where some request's needed range starts or ends).  Each maximal run
    //      of indices with the same class is one range holding the rows of exactly those
    //      requests: c_i read once by the main request and all its speculative forks, the
    //      speculative prompt read once by the k samples forked from it (PAPER.md:189, :198,
    //      :335; nested forks, reading #17), each request's private tail by its own rows.
    //      A class with more than max_rows / G rows is cut into chunks that re-read it.
    std::vector<Range> ranges, classes;   // classes: one per prefix-tree run, before max_rows chunking
    int n_groups = 0;
    int64_t unique_tokens = 0, unshared_tokens = 0;
    for (int i = 0; i < n_req; ++i) unshared_tokens += V[i].hi - lo[i];
    // true algorithmic lower bound: distinct (page, slot) key positions any row attends to
    int64_t alg_tokens = 0;
    {
        // page id -> bitmask of attended slots (ps <= 32), in a per-plan scratch array
        auto& slots = P->slot_mask;
        slots.resize(size_t(pool->cfg.num_pages), 0u);
        std::vector<int32_t> touched;
        for (int i = 0; i < n_req; ++i) {
            const auto& t = V[i].req->pages;
            const int32_t k0 = lo[i] / ps, k1 = int32_t(cdiv(V[i].hi, ps));
            for (int32_t k = k0; k < k1; ++k) {
                const int32_t pg = t[k];
                if (pg < 0) continue;   // a released page: refused below
                const int32_t a0 = k == k0 ? lo[i] - k * ps : 0;
                const int32_t b0 = k == k1 - 1 ? V[i].hi - k * ps : ps;
                const uint32_t bits = (b0 >= 32 ? 0xffffffffu : ((1u << b0) - 1u)) & ~((1u << a0) - 1u);
                if (!slots[pg]) touched.push_back(pg);
                slots[pg] |= bits;
            }
        }
        for (int32_t pg : touched) {
            alg_tokens += __builtin_popcount(slots[pg]);
            slots[pg] = 0u;
        }
    }
    struct Run {
        std::vector<int> reqs;   // request indices (into U) of the class
        int32_t k0, k1;          // page indices [k0, k1)
    };
    for (const auto& grp : groups) {
        const int gid = n_groups++;
        // requests of the group (rows of one request are consecutive in V) and their needed
        // token range [A, B) = [min lo, max hi) over their rows
        std::vector<int> ufirst;            // first row of each request
        std::vector<int> urow_end;          // one past its last row
        for (size_t x = 0; x < grp.size();) {
            size_t e = x;
            while (e < grp.size() && V[grp[e]].req == V[grp[x]].req && grp[e] == grp[x] + int(e - x)) ++e;
            ufirst.push_back(grp[x]);
            urow_end.push_back(grp[e - 1] + 1);
            x = e;
        }
        const int nu = int(ufirst.size());
        std::vector<int32_t> A(nu), B(nu);
        for (int u = 0; u < nu; ++u) {
            A[u] = INT32_MAX;
            B[u] = 0;
            for (int r = ufirst[u]; r < urow_end[u]; ++r) {
                A[u] = std::min(A[u], lo[r]);
                B[u] = std::max(B[u], V[r].hi);
            }
        }
        auto table = [&](int u) -> const std::vector<int32_t>& { return V[ufirst[u]].req->pages; };
        // events: page indices where a request's needed range starts or ends
        std::vector<int32_t> ev;
        for (int u = 0; u < nu; ++u) {
            ev.push_back(A[u] / ps);
            ev.push_back(int32_t(cdiv(B[u], ps)));
        }
        std::sort(ev.begin(), ev.end());
        ev.erase(std::unique(ev.begin(), ev.end()), ev.end());
        std::vector<Run> runs;
        // split S (all sharing page index k0, all active on [k0, k1)) into maximal runs
        std::vector<std::pair<std::vector<int>, int32_t>> work;
        for (size_t ei = 0; ei + 1 < ev.size(); ++ei) {
            const int32_t k0 = ev[ei], k1 = ev[ei + 1];
            std::vector<int> active;
            for (int u = 0; u < nu; ++u)
                if (A[u] / ps <= k0 && k0 < int32_t(cdiv(B[u], ps))) active.push_back(u);
            if (active.empty()) continue;
            auto partition = [&](const std::vector<int>& S, int32_t k) {
                std::vector<std::pair<int32_t, std::vector<int>>> cls;   // (page id, members), first-seen order
                for (int u : S) {
                    const int32_t pg = table(u)[k];
                    auto it = std::find_if(cls.begin(), cls.end(), [&](const auto& c) { return c.first == pg; });
                    if (it == cls.end()) cls.push_back({pg, {u}});
                    else it->second.push_back(u);
                }
                for (auto& c : cls) work.push_back({std::move(c.second), k});
            };
            work.clear();
            partition(active, k0);
            while (!work.empty()) {
                auto [S, ks] = std::move(work.back());
                work.pop_back();
                int32_t k = ks + 1;
                if (S.size() > 1) {
                    const auto& t0 = table(S[0]);
                    for (; k < k1; ++k) {
                        bool same = true;
                        for (size_t x = 1; x < S.size() && same; ++x) same = table(S[x])[k] == t0[k];
                        if (!same) break;
                    }
                } else {
                    k = k1;
                }
                runs.push_back(Run{S, ks, k});
                if (k < k1) partition(S, k);
            }
        }
        // merge runs of the same class that meet at an event boundary, then order by start
        std::sort(runs.begin(), runs.end(), [](const Run& x, const Run& y) {
            return x.reqs != y.reqs ? x.reqs < y.reqs : x.k0 < y.k0;
        });
        std::vector<Run> merged;
        for (auto& r : runs) {
            if (!merged.empty() && merged.back().reqs == r.reqs && merged.back().k1 == r.k0) merged.back().k1 = r.k1;
            else merged.push_back(std::move(r));
        }
        std::stable_sort(merged.begin(), merged.end(), [](const Run& x, const Run& y) {
            return x.reqs.size() != y.reqs.size() ? x.reqs.size() > y.reqs.size() : x.k0 < y.k0;
        });
        for (const auto& r : merged) {
            int32_t a = INT32_MAX, b = 0;
            for (int u : r.reqs) {
                a = std::min(a, A[u]);
                b = std::max(b, B[u]);
            }
            a = std::max(a, r.k0 * ps);
            b = std::min(b, r.k1 * ps);
            if (a >= b) continue;
            // rows of the class whose own keys [lo, hi) meet [a, b), in batch order
            std::vector<int> rows;
            for (int u : r.reqs)
                for (int x = ufirst[u]; x < urow_end[u]; ++x)
                    if (lo[x] < b && V[x].hi > a) rows.push_back(x);
            std::sort(rows.begin(), rows.end());
            classes.push_back(Range{r.reqs.size() > 1 ? 0 : 1, gid, std::move(rows), a, b, &table(r.reqs[0]), {}});
        }
    }

    // max_rows 0 (auto): 32-row items when classes of more than 16 rows (k = 3 forks of a
    // Qwen context: 4 x G = 20 rows) hold a large share of the pages, so each
    // is read once by one item instead of twice by 16-row chunks; else 16-row items
    if (P->auto_rows) {
        int64_t pages_all = 0, pages_big = 0;
        for (const auto& c : classes) {
            const int64_t np = cdiv(c.b, ps) - c.a / ps;
            pages_all += np;
            if (int64_t(c.members.size()) * G > 16) pages_big += np;
        }
        // (fp8 pools too since the one-warp-per-tile 32-row fp8 kernel: sweep B = 256, f = 0.75
        //  253 vs 266 us with 16-row items; profiles/r02_fp8_rows.txt)
        const int mt = G > 16 || pages_big * 10 > pages_all * 3 ? 2 : 1;
        if (mt != P->mt)
            if (spa_status st = set_geometry(P, mt, 0)) return st;
    }
    // fp8 one-warp teams: 12 per CTA (2-stage rings) for windowed plans, whose items are at
    // most a window long -- more warps hide the per-item setup and drain (Gemma-3 local
    // layers 86 -> 78 us) -- and 8 (3-stage rings) otherwise (config 1: 79 vs 84 us with 12;
    // profiles/r02_fp8_teams.txt)
    if (P->pool->kv_fp8 && P->mt == 1 && P->kw == 1 && P->teams_auto) {
        P->teams = window > 0 ? 12 : 8;
        P->n_teams = P->num_ctas * P->teams;
    }
    const int max_members = std::max(1, P->mt * 16 / G);
    for (auto& c : classes) {
        for (size_t c0 = 0; c0 < c.members.size(); c0 += max_members) {
            std::vector<int> chunk(c.members.begin() + c0,
                                   c.members.begin() + std::min(c.members.size(), c0 + max_members));
            // chunk rows may span requests: the page list is the same for all of them
            ranges.push_back(Range{c.kind, c.group, std::move(chunk), c.a, c.b, c.table, {}});
        }
    }

    // kind bit 0: some row of the range also takes part in another range (its outputs are
    // partial records whatever the split) -- the split-size model below charges their cost
    {
        std::vector<int32_t> cnt(n_req, 0);
        for (const auto& r : ranges)
            for (int m : r.members) ++cnt[m];
        for (auto& r : ranges) {
            r.kind = 0;
            for (int m : r.members) r.kind |= cnt[m] > 1 ? 1 : 0;
        }
    }

    // every page a range reads must be resident (spa_kv_release_window leaves -1 entries; a
    // plan whose window reaches back into them is the caller's error)
    for (const auto& r : ranges) {
        for (int32_t p = r.a / ps; p < int32_t(cdiv(r.b, ps)); ++p)
            if ((*r.table)[p] < 0)
                return fail(SPA_ERR_INVALID_ARG, "plan: a request's window needs a page released by spa_kv_release_window");
        for (const auto& f : r.folds)
            for (int32_t p = f.a / ps; p < int32_t(cdiv(f.b, ps)); ++p)
                if ((*f.table)[p] < 0)
                    return fail(SPA_ERR_INVALID_ARG, "plan: a request's window needs a page released by spa_kv_release_window");
    }

    // ---- 3. split size
    int64_t total_pages = 0;
    for (const auto& r : ranges) {
        unique_tokens += r.b - r.a;
        total_pages += cdiv(r.b, ps) - r.a / ps;
        for (const auto& f : r.folds) {
            unique_tokens += f.b - f.a;
            total_pages += cdiv(f.b, ps) - f.a / ps;
        }
    }
    static const int max_splits =
        std::getenv("SPA_MAX_SPLITS") ? std::max(1, std::atoi(std::getenv("SPA_MAX_SPLITS"))) : kMaxSplits;
    static const double tail_frac = std::getenv("SPA_TAIL_FRAC") ? std::atof(std::getenv("SPA_TAIL_FRAC")) : 0.0;
    static const int tail_div = std::getenv("SPA_TAIL_DIV") ? std::max(1, std::atoi(std::getenv("SPA_TAIL_DIV"))) : 8;
    int32_t C = P->cfg.split_pages;
    if (C <= 0) {
        const double target = double(total_pages * Hkv) / double(std::max(1, P->n_teams));
        if (const char* e = std::getenv("SPA_SPLIT_DIV")) {
            C = int32_t(std::ceil(target / std::max(0.25, std::atof(e))));
        } else {
            // choose the split size whose work items the kernel's dynamic largest-first queue
            // packs best onto n_teams teams: simulate list scheduling in LPT order (all teams
            // equally fast) and add the cost of the fp32 partial records the splits create.
            // Costs are in page units; an item costs its pages + 1 (pipeline refill + epilogue),
            // a partial record of R rows R / 16 pages written + read, and any merge a fixed
            // latency (~5 pages of one team's streaming).
            const double fs[] = {1.0, 1.5, 2.0, 3.0, 4.0};
            double best = 0;
            std::vector<double> costs;
            for (double f : fs) {
                const int32_t Cf = std::max<int32_t>(4, int32_t(std::ceil(target / f)));
                costs.clear();
                double rec_pages = 0;
                for (const auto& r : ranges) {
                    const int32_t pa = r.a / ps, pb = int32_t(cdiv(r.b, ps));
                    const int32_t Cr = std::max<int32_t>(Cf, int32_t(cdiv(pb - pa, max_splits)));
                    const int32_t n = int32_t(cdiv(pb - pa, Cr));
                    const double rows = double(r.members.size() * G);
                    int32_t fold_pages = 0;
                    for (const auto& f : r.folds) fold_pages += int32_t(cdiv(f.b, ps) - f.a / ps);
                    for (int32_t s = 0; s < n; ++s) {
                        const int32_t np = std::min(Cr, pb - pa - s * Cr) + (s == n - 1 ? fold_pages : 0);
                        const double c = np + 1 + (n > 1 || r.kind ? rows / 16.0 : 0.0);
                        for (int h = 0; h < Hkv; ++h) costs.push_back(c);
                    }
                    if (n > 1) rec_pages += n * rows / 16.0 * Hkv;
                }
                if (costs.size() > 50000) continue;
                std::sort(costs.begin(), costs.end(), std::greater<double>());
                std::priority_queue<double, std::vector<double>, std::greater<double>> q;
                for (int t = 0; t < P->n_teams; ++t) q.push(0.0);
                double makespan = 0;
                for (double c : costs) {
                    const double t0 = q.top();
                    q.pop();
                    q.push(t0 + c);
                    makespan = std::max(makespan, t0 + c);
                }
                const double score = makespan + rec_pages / P->n_teams + (rec_pages > 0 ? 5.0 : 0.0);
                if (C <= 0 || score < best * 0.98) {   // prefer fewer splits unless clearly better
                    best = score;
                    C = Cf;
                }
            }
            if (C <= 0) C = int32_t(std::ceil(target));
        }
        C = std::max(4, std::min(C, 1 << 20));
    }

    // cut points of a range: pieces of Cr pages, at most kMaxSplits splits per range (a
    // request then has <= 2 kMaxSplits partial records, shared + tail, which the merge reads in
    // chunks of 16 per L2 round trip), except that (automatic splits) the last tail_frac of a
    // long range is cut into pieces of Cr / tail_div pages.  The largest-first queue hands
    // those out last, so teams that finish early fill the end of the launch instead of idling
    // while slower teams finish their big pieces.
    auto cuts_of = [&](const Range& r) {
        const int32_t pa = r.a / ps, pb = int32_t(cdiv(r.b, ps));
        const int32_t Cr = P->cfg.split_pages > 0 ? C : std::max<int32_t>(C, int32_t(cdiv(pb - pa, max_splits)));
        std::vector<int32_t> cuts{pa};
        int32_t main_end = pb;
        const int32_t small = std::max<int32_t>(4, int32_t(cdiv(Cr, tail_div)));
        if (P->cfg.split_pages <= 0 && tail_frac > 0 && pb - pa >= 2 * small) {
            const int32_t tail = std::max<int32_t>(small, int32_t(std::lround((pb - pa) * tail_frac)));
            main_end = pb - std::min(tail, pb - pa - small);
        }
        for (int32_t s = pa + Cr; s < main_end; s += Cr) cuts.push_back(s);
        if (main_end > cuts.back()) cuts.push_back(main_end);
        for (int32_t s = main_end + small; s < pb; s += small) cuts.push_back(s);
        if (cuts.back() != pb) cuts.push_back(pb);
        return cuts;
    };

    // ---- 3b. fold member tails (reading #21): a range read by the rows of ONE request (its
    //      private tail: a speculative prompt, a parent's newest tokens) whose first page
    //      directly follows an UNSPLIT shared range holding all of those rows is appended to
    //      that range's descriptor instead of being a work item of its own: its pages are read
    //      once as before, but by the item that already holds the rows' softmax state, so the
    //      rows need no partial record and no split merge, and no tiny tail item costs a
    //      pipeline refill and an epilogue.  (A split host would keep its rows' records anyway;
    //      folding there only lengthens its last piece -- measured slower.)  The kernels mask
    //      a folded page for every row but its owner's.
    static const bool fold_tails = !std::getenv("SPA_FOLD") || std::atoi(std::getenv("SPA_FOLD")) != 0;
    if (fold_tails && P->cfg.sharing) {
        std::vector<char> dead(ranges.size(), 0);
        for (size_t t = 0; t < ranges.size(); ++t) {
            const Range& T = ranges[t];
            const Request* owner = V[T.members[0]].req;
            bool one = true;
            for (int m : T.members) one = one && V[m].req == owner;
            if (!one || !T.folds.empty()) continue;
            for (size_t h = 0; h < ranges.size(); ++h) {
                Range& Hr = ranges[h];
                if (h == t || dead[h] || Hr.group != T.group || int32_t(cdiv(Hr.b, ps)) != T.a / ps) continue;
                if (cuts_of(Hr).size() != 2) continue;   // split host: keep the tail an item
                bool multi = false, holds = true;
                for (int m : Hr.members) multi = multi || V[m].req != owner;
                for (int m : T.members) holds = holds && std::find(Hr.members.begin(), Hr.members.end(), m) != Hr.members.end();
                if (!multi || !holds) continue;
                Hr.folds.push_back(Fold{T.members, T.a, T.b, T.table});
                dead[t] = 1;
                break;
            }
        }
        std::vector<Range> kept;
        for (size_t t = 0; t < ranges.size(); ++t)
            if (!dead[t]) kept.push_back(std::move(ranges[t]));
        ranges.swap(kept);
    }

    // ---- 4. descriptors, members, pages
    std::vector<Desc> descs;
    std::vector<Member> members;
    std::vector<int32_t> pages;
    std::vector<int32_t> occ(n_req, 0);
    int64_t pages_read = 0;
    for (const auto& r : ranges) {
        const int32_t pa = r.a / ps;
        const std::vector<int32_t> cuts = cuts_of(r);
        for (size_t ci = 0; ci + 1 < cuts.size(); ++ci) {
            const int32_t s = cuts[ci], e = cuts[ci + 1];
            Desc d{};
            d.page_off = int32_t(pages.size());
            d.n_pages = e - s;
            d.tok_start = s * ps;
            d.tok_end = std::min<int32_t>(r.b, e * ps);
            d.member_off = int32_t(members.size());
            d.n_members = int32_t(r.members.size());
            d.kind = r.kind;
            // bit 2: the descriptor holds some member's newest token -- in a model step that
            // key/value is produced right before attention, so the kernel does not prefetch
            // it ahead of its programmatic-dependency wait
            for (int m : r.members)
                if (d.tok_end > V[m].first_new) d.kind |= 4;
            d.group = r.group;
            d.n_main = d.n_pages;
            for (int32_t p = s; p < e; ++p) pages.push_back((*r.table)[p]);
            for (int m : r.members) {
                members.push_back(Member{m, lo[m], 0, V[m].hi, 0, 0, 0, 0});
                occ[m] += 1;
            }
            if (ci + 2 == cuts.size()) {   // the range's last descriptor takes its folded tails
                for (const auto& f : r.folds) {
                    const int32_t fa = f.a / ps, fb = int32_t(cdiv(f.b, ps));
                    for (int m : f.rows) {
                        for (int32_t mi = d.member_off; mi < d.member_off + d.n_members; ++mi)
                            if (members[mi].row == m) {
                                members[mi].tail_k0 = d.n_pages;
                                members[mi].tail_n = fb - fa;
                                members[mi].tail_tok = fa * ps;
                            }
                        if (f.b > V[m].first_new) d.kind |= 8;
                    }
                    for (int32_t p = fa; p < fb; ++p) pages.push_back((*f.table)[p]);
                    d.n_pages += fb - fa;
                }
            }
            descs.push_back(d);
            pages_read += d.n_pages;
        }
    }
    std::vector<int32_t> rec_ptr(n_req + 1, 0);
    for (int i = 0; i < n_req; ++i) rec_ptr[i + 1] = rec_ptr[i] + (occ[i] > 1 ? occ[i] : 0);
    {
        std::vector<int32_t> next(rec_ptr.begin(), rec_ptr.end() - 1);
        for (auto& m : members) m.rec = occ[m.row] > 1 ? next[m.row]++ : -1;
    }
    const int32_t n_records = rec_ptr[n_req];

    // ---- 5. work items and the static LPT schedule over n_teams
    const int32_t n_desc = int32_t(descs.size());
    std::vector<Item> items;
    items.reserve(size_t(n_desc) * Hkv);
    for (int32_t d = 0; d < n_desc; ++d)
        for (int h = 0; h < Hkv; ++h) items.push_back(Item{d, h});
    const int32_t n_items = int32_t(items.size());
    std::vector<int32_t> order(n_items);
    std::iota(order.begin(), order.end(), 0);
    auto cost = [&](int32_t it) { return int64_t(descs[items[it].desc].n_pages) + 1; };
    // dynamic LPT: the kernel's teams pop items from this queue (largest first) with one
    // atomic each, so faster SMs take more work and the tail is made of the smallest items
    std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return cost(x) > cost(y); });
    const int T = P->n_teams;
    // kSchedSlots slots of {queue head, teams finished, tail-merge head, owner}: launch i of
    // this plan uses slot i % kSchedSlots once `owner` == i, so a launch may pop its queue
    // while its predecessors (programmatic dependent launch) still drain; the last team of
    // a launch rewinds the slot and hands it to launch i + kSchedSlots.
    std::vector<int32_t> sched(size_t(kSchedSlots) * kSchedStride, 0);
    for (int s = 0; s < kSchedSlots; ++s) sched[size_t(s) * kSchedStride + 3] = s;
    P->launches = 0;

    // tail-merge tasks (merge_mode 0): every (request with > 1 record, KV head), ordered
    // by the queue position of its last item, so the earliest-complete merges come first
    std::vector<int32_t> mtask;
    {
        std::vector<int32_t> last(size_t(n_req) * Hkv, -1);
        for (int32_t qi = 0; qi < n_items; ++qi) {
            const Item& itm = items[order[qi]];
            const Desc& d = descs[itm.desc];
            for (int32_t mi = d.member_off; mi < d.member_off + d.n_members; ++mi)
                if (members[mi].rec >= 0) last[size_t(members[mi].row) * Hkv + itm.kv_head] = qi;
        }
        std::vector<int32_t> tasks;
        for (int32_t t = 0; t < int32_t(last.size()); ++t)
            if (last[t] >= 0) tasks.push_back(t);
        std::stable_sort(tasks.begin(), tasks.end(), [&](int32_t a, int32_t b) { return last[a] < last[b]; });
        // subtask codes: task * 256 + 1 + hh (head hh alone: the heads of a task merge in
        // parallel, ~one L2 round trip after its last record; G <= max_rows <= 128 < 255) or,
        // when there are many more head merges than warps, task * 256 + 0 (one warp merges all G heads of the task with
        // their loads in flight together: fewer, longer subtasks; needs G x S <= 32)
        const int64_t warps_total = int64_t(P->num_ctas) * P->teams * P->mt * P->kw;
        // (the tcgen05 extend path merges with one warp per subtask in its own launch: whole tasks)
        bool whole = P->mt == 8 || int64_t(tasks.size()) * G > 4 * warps_total;
        if (const char* e = std::getenv("SPA_MERGE_WHOLE")) whole = std::atoi(e) != 0;   // tests: force a path
        P->merge_all_s2 = true;
        for (int32_t t : tasks) {
            const int32_t S = rec_ptr[t / Hkv + 1] - rec_ptr[t / Hkv];
            P->merge_all_s2 = P->merge_all_s2 && whole && S == 2 && G <= 8;
            if (whole && G <= 8 && G * S <= 32 && S <= 16) {
                mtask.push_back(t * 256);
            } else {
                for (int hh = 0; hh < G; ++hh) mtask.push_back(t * 256 + 1 + hh);
            }
        }
    }

    // ---- 6. serialise: header + arrays (int32 words)
    std::vector<int32_t>& H = P->host;
    H.assign(H_WORDS, 0);
    auto put = [&](int slot, const void* src, size_t words) {
        H[slot] = int32_t(H.size());
        const int32_t* w = static_cast<const int32_t*>(src);
        H.insert(H.end(), w, w + words);
        while (H.size() % 4) H.push_back(0);   // 16-B alignment of every array
    };
    put(H_OFF_DESC, descs.data(), descs.size() * (sizeof(Desc) / 4));
    put(H_OFF_MEMBER, members.data(), members.size() * (sizeof(Member) / 4));
    put(H_OFF_ITEM, items.data(), items.size() * 2);
    while (H.size() % 32) H.push_back(0);   // 128-B lines: the queue heads are hot atomics
    put(H_OFF_SCHED, sched.data(), sched.size());
    put(H_OFF_QUEUE, order.data(), order.size());
    {
        std::vector<QItem> qitems(order.size());
        for (size_t qi = 0; qi < order.size(); ++qi) {
            const Item& itm = items[order[qi]];
            qitems[qi] = QItem{descs[itm.desc], order[qi], itm.kv_head, itm.desc, 0};
        }
        while (H.size() % 16) H.push_back(0);   // 64-B aligned entries
        put(H_OFF_QITEM, qitems.data(), qitems.size() * (sizeof(QItem) / 4));
    }
    put(H_OFF_PAGES, pages.data(), pages.size());
    put(H_OFF_REC_PTR, rec_ptr.data(), rec_ptr.size());
    {
        const std::vector<int32_t> zeros(size_t(n_req) * Hkv, 0);
        put(H_OFF_COUNTERS, zeros.data(), zeros.size());
    }
    put(H_OFF_MTASK, mtask.data(), mtask.size());
    H[H_N_MTASK] = int32_t(mtask.size());
    H[H_N_REQ] = n_req;
    H[H_N_DESC] = n_desc;
    H[H_N_ITEMS] = n_items;
    H[H_N_TEAMS] = T;
    H[H_N_RECORDS] = n_records;
    H[H_N_MEMBERS] = int32_t(members.size());
    H[H_N_PAGES] = int32_t(pages.size());
    H[H_TOTAL] = int32_t(H.size());

    int rows_max = 0;
    for (const auto& d : descs) rows_max = std::max(rows_max, d.n_members * G);
    spa_plan_stats& st = P->stats;
    st.n_req = n_req;
    st.n_groups = n_groups;
    st.n_desc = n_desc;
    st.n_items = n_items;
    st.n_records = n_records;
    st.n_teams = T;
    st.rows_max = rows_max;
    st.unique_tokens = unique_tokens;
    st.alg_tokens = alg_tokens;
    st.unshared_tokens = unshared_tokens;
    st.pages_read = pages_read;
    P->window = window;
    P->n_req = n_req;

    P->uploaded = false;
    P->ws_need = plan_workspace_need(P);
    if (!pool->metadata_only) {
        int err = plan_upload(P, stream);
        if (err == kUploadNoWorkspace)
            return fail(SPA_ERR_WORKSPACE, "plan workspace missing or too small: " + std::to_string(P->ws_need) +
                                               " bytes needed, " + std::to_string(P->ws_bytes) +
                                               " set (spa_plan_workspace_size / spa_plan_set_workspace)");
        if (err) return fail(SPA_ERR_CUDA, std::string("plan upload: ") + cuda_error_string(err));
        P->uploaded = true;
    }
    st.generation = P->generation;
    return SPA_OK;
}

}  // namespace

extern "C" {

spa_status spa_plan_set_workspace(spa_plan* plan, void* workspace, size_t bytes) {
    if (!plan) return fail(SPA_ERR_INVALID_ARG, "null plan");
    if (!workspace && bytes) return fail(SPA_ERR_INVALID_ARG, "null workspace with nonzero size");
    if (reinterpret_cast<uintptr_t>(workspace) & 255) return fail(SPA_ERR_INVALID_ARG, "workspace must be 256-B aligned");
    if (workspace != plan->ws || bytes < plan->ws_need) {   // the built plan's device copy moves or no longer fits
        if (workspace != plan->ws) plan->generation++;
        plan->uploaded = false;
    }
    plan->ws = workspace;
    plan->ws_bytes = workspace ? bytes : 0;
    return SPA_OK;
}

spa_status spa_plan_workspace_size(const spa_plan* plan, size_t* out_bytes) {
    if (!plan || !out_bytes) return fail(SPA_ERR_INVALID_ARG, "null argument");
    *out_bytes = plan->host.size() >= size_t(H_WORDS) ? plan->ws_need : 0;
    return SPA_OK;
}

spa_status spa_plan_get_stats(const spa_plan* plan, spa_plan_stats* out) {
    if (!plan || !out) return fail(SPA_ERR_INVALID_ARG, "null argument");
    *out = plan->stats;
    return SPA_OK;
}

spa_status spa_plan_debug_array(const spa_plan* plan, int32_t which, const int32_t** out_data, int64_t* out_len,
                                int32_t* out_row_width) {
    if (!plan || !out_data || !out_len) return fail(SPA_ERR_INVALID_ARG, "null argument");
    const auto& H = plan->host;
    if (H.size() < size_t(H_WORDS)) return fail(SPA_ERR_INVALID_ARG, "plan has not been built");
    int slot = 0, width = 1;
    int64_t n = 0;
    switch (which) {
        case SPA_DBG_DESC: slot = H_OFF_DESC; width = int(sizeof(Desc) / 4); n = H[H_N_DESC]; break;
        case SPA_DBG_MEMBER: slot = H_OFF_MEMBER; width = int(sizeof(Member) / 4); n = H[H_N_MEMBERS]; break;
        case SPA_DBG_ITEM: slot = H_OFF_ITEM; width = 2; n = H[H_N_ITEMS]; break;
        case SPA_DBG_QUEUE: slot = H_OFF_QUEUE; n = H[H_N_ITEMS]; break;
        case SPA_DBG_PAGES: slot = H_OFF_PAGES; n = H[H_N_PAGES]; break;
        case SPA_DBG_REC_PTR: slot = H_OFF_REC_PTR; n = H[H_N_REQ] + 1; break;
        default: return fail(SPA_ERR_INVALID_ARG, "unknown debug array");
    }
    *out_data = H.data() + H[slot];
    *out_len = n * width;
    if (out_row_width) *out_row_width = width;
    return SPA_OK;
}

spa_status spa_debug_set_trace(spa_plan* plan, void* buf, int32_t cap) {
    if (!plan) return fail(SPA_ERR_INVALID_ARG, "null plan");
    if (buf && cap <= 0) return fail(SPA_ERR_INVALID_ARG, "trace capacity must be > 0");
    plan->trace = static_cast<unsigned long long*>(buf);
    plan->trace_cap = buf ? cap : 0;
    return SPA_OK;
}

spa_status spa_debug_plan_geometry(const spa_plan* plan, int32_t* out_num_ctas, int32_t* out_teams_per_cta,
                                   int32_t* out_warps_per_cta) {
    if (!plan || !out_num_ctas || !out_teams_per_cta || !out_warps_per_cta)
        return fail(SPA_ERR_INVALID_ARG, "null argument");
    *out_num_ctas = plan->num_ctas;
    *out_teams_per_cta = plan->teams;
    *out_warps_per_cta = plan->teams * plan->mt * plan->kw;   // a team = mt row tiles x kw key-split warps
    return SPA_OK;
}

}  // extern "C"
