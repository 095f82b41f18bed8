// a8 + a9 — host stages ② residual refinement and ③ final traversal
// (SURVEY §8.a a8-a9).  Plain multithreaded C++ over the host-
// resident rotated vectors X̂ and the full graph, fp32, compiler-vectorised.
// These are the paper's CPU stages (by design on the CPU), not a
// fallback for the GPU stage.
#include "host_stages.h"

#include <algorithm>
#include <atomic>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

namespace pa {

namespace {

struct Cand {
    float d;
    int32_t id;
    bool checked;
};
inline bool key_less(const Cand& a, const Cand& b) { return a.d < b.d || (a.d == b.d && a.id < b.id); }

// Exact visited set: open addressing over (epoch << 32 | id) slots; a slot with
// another epoch is empty, so a new query costs no clearing.
struct VisitedSet {
    std::vector<uint64_t> slots;
    uint32_t epoch = 0;
    size_t count = 0;
    unsigned log2 = 12;
    void reset() {
        if (slots.empty()) slots.assign((size_t)1 << log2, 0);
        ++epoch;
        if (epoch == 0) { std::fill(slots.begin(), slots.end(), 0); epoch = 1; }
        count = 0;
    }
    static inline uint32_t h(int32_t v) { return (uint32_t)v * 0x9E3779B1u; }
    bool insert(int32_t v) {   // true if newly inserted
        if ((count + 1) * 2 > slots.size()) grow();
        const size_t mask = slots.size() - 1;
        size_t i = h(v) >> (32 - log2);
        const uint64_t tag = ((uint64_t)epoch << 32) | (uint32_t)v;
        for (;;) {
            uint64_t s = slots[i];
            if ((uint32_t)(s >> 32) != epoch) { slots[i] = tag; ++count; return true; }
            if (s == tag) return false;
            i = (i + 1) & mask;
        }
    }
    void grow() {
        std::vector<uint64_t> old;
        old.swap(slots);
        ++log2;
        slots.assign((size_t)1 << log2, 0);
        uint32_t e = epoch;
        count = 0;
        for (uint64_t s : old)
            if ((uint32_t)(s >> 32) == e) insert((int32_t)(uint32_t)s);
    }
};

// 16 independent partial sums so the compiler emits packed FMAs (AVX2/AVX-512)
// without -ffast-math; the tail runs scalar.
inline float dist_full(const float* __restrict__ q, const float* __restrict__ x, int d, int metric) {
    float acc[16] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int i = 0;
    if (metric == 0) {
        for (; i + 16 <= d; i += 16)
            for (int j = 0; j < 16; ++j) { const float t = q[i + j] - x[i + j]; acc[j] += t * t; }
        float s = 0.f;
        for (int j = 0; j < 16; ++j) s += acc[j];
        for (; i < d; ++i) { const float t = q[i] - x[i]; s += t * t; }
        return s;
    }
    for (; i + 16 <= d; i += 16)
        for (int j = 0; j < 16; ++j) acc[j] += q[i + j] * x[i + j];
    float s = 0.f;
    for (int j = 0; j < 16; ++j) s += acc[j];
    for (; i < d; ++i) s += q[i] * x[i];
    return -s;
}

// Alg 1 with a sorted array C; `max_iters` < 0 ⇒ until no unchecked.
// Width w: each iteration marks the w smallest unchecked entries
// checked and visits their rows in key order; inserting the new keys one at a
// time with truncation to ef leaves the same C as merging them all and then
// resizing (truncation only drops keys that cannot be among the ef smallest).
template <class DistFn, class PrefetchFn>
void greedy(const int64_t* off, const int32_t* nb, DistFn dist, PrefetchFn prefetch, int ef, int w, long max_iters,
            std::vector<Cand>& C, VisitedSet& vis, int64_t& n_dist) {
    long it = 0;
    int32_t us[64];
    while (max_iters < 0 || it < max_iters) {
        int nu = 0;
        for (size_t i = 0; i < C.size() && nu < w; ++i)
            if (!C[i].checked) { C[i].checked = true; us[nu++] = C[i].id; }
        if (nu == 0) break;
        ++it;
        for (int x = 0; x < nu; ++x) {
            const int32_t u = us[x];
            // unvisited neighbours first (stored order), their rows prefetched, then distances
            int32_t fresh[64];
            for (int64_t e0 = off[u]; e0 < off[u + 1];) {
                int nf = 0;
                for (; e0 < off[u + 1] && nf < 64; ++e0) {
                    const int32_t v = nb[e0];
                    if (!vis.insert(v)) continue;
                    fresh[nf++] = v;
                    prefetch(v);
                }
                for (int i = 0; i < nf; ++i) {
                    const int32_t v = fresh[i];
                    ++n_dist;
                    Cand c{dist(v), v, false};
                    if ((int)C.size() == ef && !key_less(c, C.back())) continue;
                    auto pos = std::lower_bound(C.begin(), C.end(), c, key_less);
                    C.insert(pos, c);
                    if ((int)C.size() > ef) C.pop_back();
                }
            }
        }
    }
}

}  // namespace

void run_host_stages(const HostStageArgs& a) {
    int T = a.threads > 0 ? a.threads : (int)std::max(1u, std::thread::hardware_concurrency());
    if (T > a.m) T = (int)std::max<int64_t>(1, a.m);
    std::atomic<int64_t> next{0};
    std::atomic<int64_t> nd2{0}, nd3{0};
    const int D = a.dim, dp = a.rdim, dr = a.dim - a.rdim;
    auto worker = [&]() {
        VisitedSet vis;
        std::vector<float> qh(D);
        std::vector<Cand> C;
        int64_t my2 = 0, my3 = 0;
        for (;;) {
            const int64_t q = next.fetch_add(1);
            if (q >= a.m) break;
            if (a.wait_ready) a.wait_ready(a.ready_ctx, q);
            std::memcpy(qh.data(), a.qp + q * a.qp_stride, sizeof(float) * dp);
            if (dr > 0) std::memcpy(qh.data() + dp, a.qres + q * dr, sizeof(float) * dr);
            auto dfull = [&](int32_t v) { return dist_full(qh.data(), a.rotated + (int64_t)v * D, D, a.metric); };
            const int lines = std::min(8, (D * 4 + 63) / 64);
            auto pref = [&](int32_t v) {
                const char* r = reinterpret_cast<const char*>(a.rotated + (int64_t)v * D);
                for (int l = 0; l < lines; ++l) __builtin_prefetch(r + 64 * l, 0, 0);
            };
            vis.reset();
            C.clear();
            // ---- stage ②: full δ = GPU primary δ' + residual δ (Q22)
            const int32_t* ci = a.cand_ids + q * a.ef1;
            const float* cd = a.cand_d + q * a.ef1;
            for (int j = 0; j < a.ef1; ++j) {
                const int32_t v = ci[j];
                if (v < 0) continue;
                float full;
                if (a.recompute_primary) {
                    full = dfull(v);
                } else {
                    const float res = dr > 0 ? dist_full(qh.data() + dp, a.rotated + (int64_t)v * D + dp, dr, a.metric) : 0.f;
                    full = cd[j] + res;
                }
                C.push_back(Cand{full, v, false});
                vis.insert(v);
                ++my2;
            }
            std::sort(C.begin(), C.end(), key_less);
            if (a.flags & 2u) {                                   // PA_NO_STAGE2
                if ((int)C.size() > a.ef3) C.resize(a.ef3);
            } else {
                if ((int)C.size() > a.ef2) C.resize(a.ef2);
                greedy(a.sub.off, a.sub.nb, dfull, pref, a.ef2, a.width, a.refine_iters, C, vis, my2);
            }
            // ---- stage ③: Alg 1 on the full graph, carry entries unchecked, visited kept (Q23)
            // ef2 > ef3: keep the ef3 smallest now — the same set Alg 1's resize (l.11)
            // leaves after the first expansion, whose node is C[0] either way.
            if ((int)C.size() > a.ef3) C.resize(a.ef3);
            for (Cand& c : C) c.checked = false;
            greedy(a.full.off, a.full.nb, dfull, pref, a.ef3, a.width, -1, C, vis, my3);
            for (int j = 0; j < a.k; ++j) {
                const bool ok = j < (int)C.size();
                a.out_ids[q * a.k + j] = ok ? C[j].id : -1;
                a.out_d[q * a.k + j] = ok ? C[j].d : std::numeric_limits<float>::infinity();
            }
        }
        nd2 += my2;
        nd3 += my3;
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    if (a.sum_n_dist2) *a.sum_n_dist2 += nd2.load();
    if (a.sum_n_dist3) *a.sum_n_dist3 += nd3.load();
}

}  // namespace pa
