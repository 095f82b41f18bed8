// Traversal kernel template (a5 + a6), included by the per-variant instantiation units.
#pragma once
// a5 + a6 — stage ① traversal: Alg 1 over the sampled subgraph
// with reduced vectors, one warp per query, persistent grid with a
// global work counter.
//
// Per query (warp):
//   C        : sorted list of ≤ ef 64-bit keys (ord(δ)<<32 | id<<1 | checked) in
//              smem; lane l owns positions l, l+32, ... during a merge.
//   visited  : EXACT set (Alg 1's "unvisited" test, I4) — level 1 = open-addressing
//              int32 hash in smem (2^hash_log2 slots, accepts inserts while ≤ half
//              full); level 2 = per-warp open-addressing slab in global memory
//              (one atomicCAS per probe, used slots logged and zeroed at the end of
//              the query) once level 1 closes.  The paper's bloom filter
//              is NEXT-f1.
//   loop     : u ← smallest unchecked key (ballot scan from a "all checked before"
//              hint, Alg 1 l.5); the runner-up's ELL row is prefetched into L2;
//              ELL[u][lane] (one coalesced 128-B row per 32 neighbours, l.6);
//              test-and-insert visited (l.7); each new neighbour's lane gathers its
//              reduced row (float4 loads) and computes δ' in fp32 (l.8); keys
//              below C's current worst are merged by rank (l.9, l.11): for every
//              passing key the warp counts, with one shuffle and ef/32 ballots,
//              its rank in C and its shift of C's entries; everything moves in
//              place (registers hold the old C across one __syncwarp).
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "internal.h"

namespace pa {
namespace trav {
constexpr int kTW = 4;                 // warps per block
#ifndef PA_TRAV_MINB
#define PA_TRAV_MINB 6                 // min resident blocks per SM (register budget 65536/(128·this))
#endif
#ifndef PA_TRAV_MINB_BLOOM
#define PA_TRAV_MINB_BLOOM 9           // same, bloom visited set: 36 warps/SM (C2 A/B: 8 → 3.20 ms, 9 → 2.72, 10 → 3.00)
#endif
constexpr int kIterCap = 1000000;      // Q16 safety cap (status 2)
constexpr int kMaxWidth = 8;           // search width w ≤ 8 on the GPU
#ifndef PA_GROUP_L32
#define PA_GROUP_L32 4                 // lanes per row in the distance gathers, fp32 rows
#endif
#ifndef PA_GROUP_L16
#define PA_GROUP_L16 2                 // lanes per row, binary16 rows
#endif

// Bloom segment hash multipliers (odd; oracle O13 uses the same definition).
__device__ __forceinline__ constexpr uint32_t bloom_mult(int j) {
    return j == 0 ? 0x9E3779B1u : (j == 1 ? 0x85EBCA77u : 0xC2B2AE3Du);
}

__device__ __forceinline__ uint32_t hash1(int32_t v) { return (uint32_t)v * 0x9E3779B1u; }
__device__ __forceinline__ uint32_t hash2(int32_t v) { return ((uint32_t)v ^ 0x5bd1e995u) * 0x85EBCA77u; }

struct Visited {
    volatile int32_t* H;   // smem level 1
    int log2S;
    int count1;            // entries in level 1 (warp-uniform)
    uint32_t* G;           // global level 2 slab: 2^L slots (0 = empty, else id+1) ...
    uint32_t* log;         // ... followed by the log of slots used by the current query
    uint32_t gmask;
    int count2;            // entries in level 2 (warp-uniform)
};

// Compact level 1 (ids < 2^24, ≥ 2^11 slots): 16-bit slots.  The id is mapped by
// a bijection P on 24 bits; the top log2S bits of P(v) are its home slot and the
// slot stores the remaining 24−log2S bits with the displacement d ≤ 6 from home
// (quotienting), so (slot, stored value) identifies v exactly.  0xFFFF = empty.
// A full 7-slot window sends v to level 2 (lookups follow the same rule, so an
// id is in level 2 only if its window was full when it was inserted).
__device__ __forceinline__ uint32_t perm24(int32_t v) { return ((uint32_t)v * 0x9E3779B1u) & 0xFFFFFFu; }

// Returns true iff v was not yet visited (and is now).  `open1` is warp-uniform.
template <int VIS>
__device__ __forceinline__ bool visit(Visited& vs, int32_t v, bool open1, bool& in_l2, uint32_t& slot) {
    in_l2 = false;
    const uint32_t S = 1u << vs.log2S;
    if constexpr (VIS == 1) {
        volatile uint16_t* H16 = reinterpret_cast<volatile uint16_t*>(vs.H);
        const uint32_t P = perm24(v);
        const uint32_t home = P >> (24 - vs.log2S);
        const uint32_t rem = P & ((1u << (24 - vs.log2S)) - 1u);
        for (uint32_t d = 0; d < 7; ++d) {
            const uint32_t h = (home + d) & (S - 1);
            const uint16_t want = (uint16_t)((rem << 3) | d);
            const uint16_t cur = H16[h];
            if (cur == want) return false;
            if (cur == 0xFFFFu) {
                if (!open1) break;                               // not in level 1
                const unsigned short old = atomicCAS((unsigned short*)&H16[h], (unsigned short)0xFFFFu, want);
                if (old == 0xFFFFu) return true;
                if (old == want) return false;
            }
        }
    } else {
        uint32_t h = hash1(v) >> (32 - vs.log2S);
        for (uint32_t p = 0; p < S; ++p) {
            int32_t cur = vs.H[h];
            if (cur == v) return false;
            if (cur == -1) {
                if (!open1) break;                               // not in level 1
                int32_t old = atomicCAS((int32_t*)&vs.H[h], -1, v);
                if (old == -1) return true;
                if (old == v) return false;
            }
            h = (h + 1) & (S - 1);
        }
    }
    // level 2: one atomicCAS per probe (empty slots are 0; the query's used slots
    // are logged and zeroed when it finishes, so no epoch tags are needed)
    const uint32_t tag = (uint32_t)v + 1u;
    uint32_t g = hash2(v) & vs.gmask;
    for (uint32_t p = 0; p <= vs.gmask; ++p) {
        const uint32_t old = atomicCAS(&vs.G[g], 0u, tag);
        if (old == 0u) { in_l2 = true; slot = g; return true; }
        if (old == tag) return false;
        g = (g + 1) & vs.gmask;
    }
    return false;   // unreachable while count2 ≤ gmask/2 (guarded by the caller)
}

// Bulk prefetch of one reduced-vector row into L2 (sm_90+ cp.async.bulk.prefetch).
__device__ __forceinline__ void prefetch_row_l2(const void* p, int bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}

// Lookup-only probe of the level-1 hash (speculation; false negatives only cost a prefetch).
template <int VIS>
__device__ __forceinline__ bool visited_l1(const Visited& vs, int32_t v) {
    const uint32_t S = 1u << vs.log2S;
    if constexpr (VIS == 1) {
        const volatile uint16_t* H16 = reinterpret_cast<const volatile uint16_t*>(vs.H);
        const uint32_t P = perm24(v);
        const uint32_t home = P >> (24 - vs.log2S);
        const uint32_t rem = P & ((1u << (24 - vs.log2S)) - 1u);
        for (uint32_t d = 0; d < 7; ++d) {
            const uint16_t cur = H16[(home + d) & (S - 1)];
            if (cur == (uint16_t)((rem << 3) | d)) return true;
            if (cur == 0xFFFFu) return false;
        }
        return false;
    }
    uint32_t h = hash1(v) >> (32 - vs.log2S);
    for (uint32_t p = 0; p < 8; ++p) {
        const int32_t cur = vs.H[h];
        if (cur == v) return true;
        if (cur == -1) return false;
        h = (h + 1) & (S - 1);
    }
    return false;
}

template <int METRIC, int VIS, int SMAX, int DPS4, bool TRACE, bool H16>
__global__ void __launch_bounds__(kTW * 32, PA_TRAV_MINB) k_traverse(DevIndex ix, SearchArgs a) {
    const int ELLW = ix.ell_w, NCH = ix.ell_w >> 5;         // ELL row width 32 or 64
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int ef = a.ef, dps = ix.rdim_pad, S = 1 << a.hash_log2;
    const int efp = (ef + 1) & ~1;                      // keep qs 16-B aligned
    const int qlen = ix.qlen;                           // ≥ dps (fp32 rows) / ≥ rdim_h (fp16 rows)
    const size_t per_warp = (size_t)efp * 8 + (size_t)qlen * 4 + (size_t)S * (VIS == 1 ? 2 : 4);
    unsigned char* base = smem_raw + per_warp * w;
    uint64_t* C = reinterpret_cast<uint64_t*>(base);
    float* qs = reinterpret_cast<float*>(C + efp);
    int32_t* H = reinterpret_cast<int32_t*>(qs + qlen);
    const unsigned lt_mask = (1u << lane) - 1u;
    const int64_t gw = (int64_t)blockIdx.x * kTW + w;

    Visited vs;
    vs.H = H;
    vs.log2S = a.hash_log2;
    vs.G = reinterpret_cast<uint32_t*>(a.spill + ((int64_t)gw << a.spill_log2));   // 8 B × 2^L per warp
    vs.log = vs.G + ((size_t)1 << a.spill_log2);                                    // slots: 4 B × 2^L, log after
    vs.gmask = (1u << a.spill_log2) - 1u;
    const int cap1 = S >> 1, cap2 = (int)(vs.gmask >> 1);

    for (;;) {
        int64_t q = 0;
        if (lane == 0) q = atomicAdd(a.work, 1);
        q = __shfl_sync(kFull, (int)q, 0);
        if (q >= a.m) break;
        vs.count1 = 0;
        vs.count2 = 0;
        for (int i = lane; i < qlen; i += 32) qs[i] = i < dps ? a.qp[q * dps + i] : 0.f;
        int4* H4 = reinterpret_cast<int4*>(H);
        for (int i = lane; i < (S >> (VIS == 1 ? 3 : 2)); i += 32) H4[i] = make_int4(-1, -1, -1, -1);
        __syncwarp();

        int csz = 0, hint = 0, n_exp = 0, n_dist = 0, n_spill = 0, status = 0;

        // Visited test-and-insert for one batch of ≤32 candidate ids (one per
        // lane, −1 = none); returns whether this lane's id is new (Alg 1 l.6-7).
        auto visit_batch = [&](int32_t v) -> bool {
            const bool open1 = vs.count1 + 32 <= cap1;
            if (!open1 && vs.count2 + 32 > cap2) { status = 1; return false; }
            bool l2 = false;
            uint32_t slot = 0;
            const bool isnew = v >= 0 && visit<VIS>(vs, v, open1, l2, slot);
            const unsigned bal = __ballot_sync(kFull, isnew);
            const unsigned bl2 = __ballot_sync(kFull, l2);
            const int nnew = __popc(bal);
            if (l2) vs.log[vs.count2 + __popc(bl2 & lt_mask)] = slot;
            vs.count1 += nnew - __popc(bl2);
            vs.count2 += __popc(bl2);
            n_spill += __popc(bl2);
            if (TRACE && isnew) {
                int pos = n_dist + __popc(bal & lt_mask);
                if (pos < a.trace_cap) a.trace_visit[q * a.trace_cap + pos] = v;
            }
            n_dist += nnew;
            return isnew;
        };
        // δ' for the new ids (l.8) and rank-merge of the keys that beat C's worst (l.9, l.11).
        uint64_t minnew = kKeyInf;     // smallest new key of the current expansion
        auto merge_batch = [&](int32_t v, bool isnew, auto&& before_merge) {
            if (__ballot_sync(kFull, isnew) == 0) { before_merge(); return; }
            uint64_t key = kKeyInf;
            if (isnew) {
                float dv;
                if constexpr (H16)
                    dv = row_dist_h<METRIC, DPS4>(qs, reinterpret_cast<const __half*>(ix.reduced_h) + (int64_t)v * ix.rstride_h,
                                                  ix.rdim_h);
                else
                    dv = row_dist_t<METRIC, DPS4>(qs, ix.reduced + (int64_t)v * ix.rstride, dps);
                key = make_key(dv, v);
            }
            {
                const uint32_t hi = __reduce_min_sync(kFull, (uint32_t)(key >> 32));
                const uint32_t lo = __reduce_min_sync(kFull, (uint32_t)(key >> 32) == hi ? (uint32_t)key : 0xffffffffu);
                const uint64_t mk = ((uint64_t)hi << 32) | lo;
                minnew = mk < minnew ? mk : minnew;
            }
            before_merge();
            const uint64_t thresh = csz == ef ? C[ef - 1] : kKeyInf;
            const bool pass = key < thresh;                   // unique keys: strict
            const unsigned pb = __ballot_sync(kFull, pass);
            if (pb == 0) return;
            int minr;
            csz = rank_merge<SMAX>(C, csz, ef, key, pass, pb, lane, minr);
            hint = min(hint, minr);
        };

        // ---- a5: C := entries (Alg 1 l.3), visited := entries (Q15)
        for (int j0 = 0; j0 < a.E && status == 0; j0 += 32) {
            const int j = j0 + lane;
            const int32_t v = j < a.E ? a.entries[q * a.E + j] : -1;
            const bool isnew = visit_batch(v);
            if (status == 0) merge_batch(v, isnew, [] {});
        }
        // ---- a6: Alg 1 l.4-12.  Speculation: the runner-up unchecked node u2 is
        // the likely next expansion; its ELL row is loaded into registers (sv)
        // alongside u's, and the reduced rows of its not-yet-visited neighbours
        // are prefetched into L2 while u's distances are computed.  A correct
        // guess makes the next iteration's two dependent loads L2 hits; a wrong
        // guess only costs bandwidth.  The algorithm's decisions are unchanged.
        int32_t spec_u = -1;
        int32_t sv[2] = {-1, -1};
        if (!(a.flags & 4u)) {
            for (int it = 0; status == 0; ++it) {
                if (a.width > 1) {
                    // Search width w: the w smallest unchecked keys are
                    // marked checked together and their rows visited in key order; merging
                    // row by row with truncation leaves the same C as one merge + resize.
                    int ps[kMaxWidth];
                    int nu = 0;
                    for (int t = hint >> 5; t * 32 < csz && nu < a.width; ++t) {
                        const int i = t * 32 + lane;
                        unsigned b = __ballot_sync(kFull, i < csz && !key_checked(C[i]));
#pragma unroll
                        for (int x = 0; x < kMaxWidth; ++x)
                            if (b && nu < a.width) { ps[nu++] = t * 32 + __ffs(b) - 1; b &= b - 1; }
                    }
                    if (nu == 0) break;                                 // l.12: no unchecked node
                    int32_t us[kMaxWidth];
#pragma unroll
                    for (int x = 0; x < kMaxWidth; ++x) us[x] = x < nu ? key_id(C[ps[x]]) : -1;
                    __syncwarp();
                    if (lane == 0)
                        for (int x = 0; x < nu; ++x) C[ps[x]] |= 1ull;
                    hint = ps[nu - 1] + 1;
                    __syncwarp();
#pragma unroll
                    for (int x = 0; x < kMaxWidth; ++x) {
                        if (x >= nu || status != 0) break;
                        if (TRACE && lane == 0 && n_exp < a.trace_cap) a.trace_expand[q * a.trace_cap + n_exp] = us[x];
                        ++n_exp;
                        for (int c = 0; c < NCH && status == 0; ++c) {
                            const int32_t v = __ldg(ix.ell + (int64_t)us[x] * ELLW + c * 32 + lane);
                            const bool isnew = visit_batch(v);
                            if (status == 0) merge_batch(v, isnew, [] {});
                        }
                    }
                    if (it >= kIterCap) status = 2;
                    continue;
                }
                int p = -1, p2 = -1;
                for (int t = hint >> 5; t * 32 < csz; ++t) {
                    const int i = t * 32 + lane;
                    const bool un = i < csz && !key_checked(C[i]);
                    const unsigned b = __ballot_sync(kFull, un);
                    if (b) {
                        p = t * 32 + __ffs(b) - 1;
                        const unsigned b2 = b & (b - 1);
                        if (b2) p2 = t * 32 + __ffs(b2) - 1;
                        break;
                    }
                }
                if (p < 0) break;                                   // l.12: no unchecked node
                const uint64_t ku = C[p];
                const int32_t u = key_id(ku);
                int32_t vv[2] = {-1, -1};
                if (u == spec_u) {
                    vv[0] = sv[0];
                    vv[1] = sv[1];
                } else {
                    const int32_t* row = ix.ell + (int64_t)u * ELLW;
                    vv[0] = __ldg(row + lane);
                    if (NCH > 1) vv[1] = __ldg(row + 32 + lane);
                }
                const uint64_t key_p2 = p2 >= 0 ? C[p2] : kKeyInf;
                const int32_t u2 = p2 >= 0 ? key_id(key_p2) : -1;
                if (u2 >= 0 && u2 != u) {
                    const int32_t* row2 = ix.ell + (int64_t)u2 * ELLW;
                    sv[0] = __ldg(row2 + lane);
                    sv[1] = NCH > 1 ? __ldg(row2 + 32 + lane) : -1;
                }
                spec_u = u2 != u ? u2 : -1;
                minnew = kKeyInf;
                __syncwarp();
                if (lane == 0) C[p] = ku | 1ull;                    // mark checked
                hint = p + 1;
                if (TRACE && lane == 0 && n_exp < a.trace_cap) a.trace_expand[q * a.trace_cap + n_exp] = u;
                ++n_exp;
                __syncwarp();
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    if (c >= NCH || status != 0) break;
                    const bool isnew = visit_batch(vv[c]);
                    if (c == 0 && u2 >= 0) {
#pragma unroll
                        for (int c2 = 0; c2 < 2; ++c2) {
                            const int32_t w2 = sv[c2];
                            if (w2 >= 0 && !visited_l1<VIS>(vs, w2))
                                prefetch_row_l2(H16 ? (const void*)(reinterpret_cast<const __half*>(ix.reduced_h) +
                                                                     (int64_t)w2 * ix.rstride_h)
                                                    : (const void*)(ix.reduced + (int64_t)w2 * ix.rstride),
                                                H16 ? ix.rdim_h * 2 : dps * 4);
                        }
                    }
                    if (status == 0)
                        merge_batch(vv[c], isnew, [&] {
                            // The next expansion is exactly min(runner-up, best new key): issue its
                            // ELL row now so the load overlaps this merge (Alg 1 l.5 of the next step).
                            if (c != NCH - 1) return;
                            const uint64_t nk = minnew < key_p2 ? minnew : key_p2;
                            if (nk == kKeyInf) return;
                            const int32_t nu = key_id(nk);
                            if (nu == spec_u) return;
                            const int32_t* rown = ix.ell + (int64_t)nu * ELLW;
                            sv[0] = __ldg(rown + lane);
                            sv[1] = NCH > 1 ? __ldg(rown + 32 + lane) : -1;
                            spec_u = nu;
                        });
                }
                if (it >= kIterCap) status = 2;
            }
        }
        // ---- outputs (a7 candidate list + top-k)
        const float inf = __int_as_float(0x7f800000);
        if (a.cand_ids) {
            for (int i = lane; i < ef; i += 32) {
                a.cand_ids[q * ef + i] = i < csz ? key_id(C[i]) : -1;
                a.cand_d[q * ef + i] = i < csz ? key_dist(C[i]) : inf;
            }
        }
        for (int i = lane; i < a.k; i += 32) {
            a.out_ids[q * a.k + i] = i < csz ? key_id(C[i]) : -1;
            a.out_d[q * a.k + i] = i < csz ? key_dist(C[i]) : inf;
        }
        for (int i = lane; i < vs.count2; i += 32) vs.G[vs.log[i]] = 0u;   // reset the level-2 slots used
        __syncwarp();
        if (lane == 0) {
            if (a.counters) {
                int4 c4 = make_int4(n_exp, n_dist, n_spill, status);
                reinterpret_cast<int4*>(a.counters)[q] = c4;
            }
            if (TRACE) { a.trace_nexp[q] = n_exp; a.trace_nvis[q] = n_dist; }
        }
        __syncwarp();
    }
}


// ---------------------------------------------------------------------------
// Software-pipelined variant (ELL width 32).  Same algorithm, reordered so the
// gather latency of expansion i overlaps the merge of expansion i−1's keys:
//   1. visit u_i's neighbours; L2 bulk-prefetch the rows of the new ones;
//   2. merge the passing keys of expansion i−1 into C; scan C for its best
//      unchecked key r (the runner-up) and load r's ELL row speculatively;
//   3. δ' of u_i's new neighbours (rows now in L2), filter against C's worst;
//   4. u_{i+1} = min(r, best passing new key) — exactly Alg 1's next "first
//      unchecked node": r is C's best unchecked, and a passing new key beats C's
//      worst, so both are in the ef-truncated list; it is marked checked (in C,
//      or on the pending key before it is merged) and its row is fetched.
// The expansion and visit sequences are identical to the sequential kernel.
template <int METRIC, int VIS, int SMAX, int DPS4, bool TRACE, bool H16>
__global__ void __launch_bounds__(kTW * 32, VIS == 2 ? PA_TRAV_MINB_BLOOM : PA_TRAV_MINB) k_traverse_pipe(DevIndex ix, SearchArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int ef = a.ef, dps = ix.rdim_pad, S = 1 << a.hash_log2;
    const int efp = (ef + 1) & ~1;
    const int qlen = ix.qlen;
    const int bl = a.bloom_log2;                         // VIS == 2: 3 segments × 2^bl bits
    const size_t per_warp = (size_t)efp * 8 + (size_t)qlen * 4 + 128 +
                            (VIS == 2 ? ((size_t)3 << (bl - 3)) : (size_t)S * (VIS == 1 ? 2 : 4));
    unsigned char* base = smem_raw + per_warp * w;
    uint64_t* C = reinterpret_cast<uint64_t*>(base);
    float* qs = reinterpret_cast<float*>(C + efp);
    int32_t* scr = reinterpret_cast<int32_t*>(qs + qlen);      // 32 compacted new ids
    int32_t* H = scr + 32;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int64_t gw = (int64_t)blockIdx.x * kTW + w;

    Visited vs;
    vs.H = H;
    vs.log2S = a.hash_log2;
    vs.G = reinterpret_cast<uint32_t*>(a.spill + ((int64_t)gw << a.spill_log2));
    vs.log = vs.G + ((size_t)1 << a.spill_log2);
    vs.gmask = (1u << a.spill_log2) - 1u;
    const int cap1 = S >> 1, cap2 = (int)(vs.gmask >> 1);

    const unsigned char* rows = H16 ? reinterpret_cast<const unsigned char*>(ix.reduced_h)
                                    : reinterpret_cast<const unsigned char*>(ix.reduced);
    const int64_t stride = H16 ? (int64_t)ix.rstride_h * 2 : (int64_t)ix.rstride * 4;
    auto row_ptr = [&](int32_t v) -> const void* { return rows + (int64_t)v * stride; };
    const int row_bytes = H16 ? ix.rdim_h * 2 : dps * 4;
    const int nvr = row_bytes >> 4;                             // 16-B chunks per row
    // Keys of this batch's new ids (Alg 1 l.8): compacted, lane r holds the key of
    // the r-th new id (lane order), lanes ≥ #new hold kKeyInf.
    auto new_keys = [&](int32_t v, bool isnew) -> uint64_t {
        const unsigned bal = __ballot_sync(kFull, isnew);
        const int nnew = __popc(bal);
        if (nnew == 0) return kKeyInf;
        if (isnew) scr[__popc(bal & lt_mask)] = v;
        __syncwarp();
        const int32_t cid = lane < nnew ? scr[lane] : 0;
        __syncwarp();
#ifndef PA_WIDE_ROWS_MIN
#define PA_WIDE_ROWS_MIN 0             // fp32 rows of ≥ this many float4 gathered by 8 lanes (128-B lines); 0 = off
#endif
        constexpr int LF = (PA_WIDE_ROWS_MIN > 0 && DPS4 >= PA_WIDE_ROWS_MIN) ? 8 : PA_GROUP_L32;
        const float d = group_dists<METRIC, DPS4, H16, H16 ? PA_GROUP_L16 : LF, VIS != 2>(
            qs, rows, stride, nvr, cid, nnew, lane);
        return lane < nnew ? make_key(d, cid) : kKeyInf;
    };

    for (;;) {
        int64_t q = 0;
        if (lane == 0) q = atomicAdd(a.work, 1);
        q = __shfl_sync(kFull, (int)q, 0);
        if (q >= a.m) break;
        vs.count1 = 0;
        vs.count2 = 0;
        for (int i = lane; i < qlen; i += 32) qs[i] = i < dps ? a.qp[q * dps + i] : 0.f;
        int4* H4 = reinterpret_cast<int4*>(H);
        if constexpr (VIS == 2) {
            for (int i = lane; i < (3 << (bl - 7)); i += 32) H4[i] = make_int4(0, 0, 0, 0);
        } else {
            for (int i = lane; i < (S >> (VIS == 1 ? 3 : 2)); i += 32) H4[i] = make_int4(-1, -1, -1, -1);
        }
        __syncwarp();

        int csz = 0, hint = 0, n_exp = 0, n_dist = 0, n_spill = 0, status = 0;

        // Visited test-and-insert of one batch of ≤ 32 ids in stored order (lane
        // order; −1 = none); returns whether this lane's id is new (Alg 1 l.6-7).
        // `entries`: a5 inserts unconditionally (entries are distinct).
        auto visit_batch = [&](int32_t v, bool entries) -> bool {
            if constexpr (VIS == 2) {
                // Partitioned bloom filter (oracle O13): segment j holds
                // bit ((uint32)v·A_j) >> (32 − bl).  Sequential test-then-set in lane
                // order is reproduced exactly: lane b sees the filter plus the bits
                // of every valid lower lane (a lower lane that is itself judged
                // visited only adds bits already present), and per-segment hashing
                // means only equal positions within a segment can coincide, which
                // one match.any per segment detects.
                uint32_t* F = reinterpret_cast<uint32_t*>(H);
                const bool valid = v >= 0;
                const unsigned lower = __ballot_sync(kFull, valid) & lt_mask;
                bool covered = !entries;
                uint32_t wi[3], bm[3];
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    const uint32_t p = valid ? (((uint32_t)v * bloom_mult(j)) >> (32 - bl)) : 0xFFFFFFFFu;
                    wi[j] = ((uint32_t)j << (bl - 5)) + (p >> 5);
                    bm[j] = 1u << (p & 31);
                    if (!entries) {
                        const unsigned peers = __match_any_sync(kFull, p);
                        const bool c = (peers & lower) != 0 || (valid && (F[wi[j]] & bm[j]) != 0);
                        covered = covered && c;
                    }
                }
                const bool isnew = valid && !covered;
                __syncwarp();
                if (isnew) {
#pragma unroll
                    for (int j = 0; j < 3; ++j) atomicOr(&F[wi[j]], bm[j]);
                }
                __syncwarp();
                const unsigned bal = __ballot_sync(kFull, isnew);
                if (TRACE && isnew) {
                    const int pos = n_dist + __popc(bal & lt_mask);
                    if (pos < a.trace_cap) a.trace_visit[q * a.trace_cap + pos] = v;
                }
                n_dist += __popc(bal);
                return isnew;
            }
            const bool open1 = vs.count1 + 32 <= cap1;
            if (!open1 && vs.count2 + 32 > cap2) { status = 1; return false; }
            bool l2 = false;
            uint32_t slot = 0;
            const bool isnew = v >= 0 && visit<VIS>(vs, v, open1, l2, slot);
            const unsigned bal = __ballot_sync(kFull, isnew);
            const unsigned bl2 = __ballot_sync(kFull, l2);
            const int nnew = __popc(bal);
            if (l2) vs.log[vs.count2 + __popc(bl2 & lt_mask)] = slot;
            vs.count1 += nnew - __popc(bl2);
            vs.count2 += __popc(bl2);
            n_spill += __popc(bl2);
            if (TRACE && isnew) {
                const int pos = n_dist + __popc(bal & lt_mask);
                if (pos < a.trace_cap) a.trace_visit[q * a.trace_cap + pos] = v;
            }
            n_dist += nnew;
            return isnew;
        };
        auto merge_keys = [&](uint64_t key, bool pass, unsigned pb) {
            if (pb == 0) return;
            int minr;
            csz = rank_merge<SMAX>(C, csz, ef, key, pass, pb, lane, minr);
            hint = min(hint, minr);
        };
        // ---- a5: C := entries, visited := entries (sequential merges)
        for (int j0 = 0; j0 < a.E && status == 0; j0 += 32) {
            const int j = j0 + lane;
            const int32_t v = j < a.E ? a.entries[q * a.E + j] : -1;
            const bool isnew = visit_batch(v, true);
            if (status != 0) break;
            const uint64_t key = new_keys(v, isnew);
            const uint64_t thresh = csz == ef ? C[ef - 1] : kKeyInf;
            const bool pass = key < thresh;
            merge_keys(key, pass, __ballot_sync(kFull, pass));
        }
        // ---- a6: pipelined Alg 1 loop
        if (!(a.flags & 4u) && status == 0) {
            int p = -1;
            for (int t = hint >> 5; t * 32 < csz; ++t) {
                const int i = t * 32 + lane;
                const unsigned b = __ballot_sync(kFull, i < csz && !key_checked(C[i]));
                if (b) { p = t * 32 + __ffs(b) - 1; break; }
            }
            if (p >= 0) {
                int32_t u = key_id(C[p]);
                __syncwarp();
                if (lane == 0) C[p] |= 1ull;
                hint = p + 1;
                int32_t vv = __ldg(ix.ell + (int64_t)u * 32 + lane);
                uint64_t pkey = kKeyInf;          // pending keys of the previous expansion (unmerged)
                bool ppass = false;
                unsigned ppb = 0;
                int32_t spec_u = -1, sv = -1;
                for (int it = 0;; ++it) {
                    if (TRACE && lane == 0 && n_exp < a.trace_cap) a.trace_expand[q * a.trace_cap + n_exp] = u;
                    ++n_exp;
#ifndef PA_MERGE_FIRST
#define PA_MERGE_FIRST 1                // A/B on C1: 2% faster than merging after the visit
#endif
                    if (PA_MERGE_FIRST) {           // the merge overlaps the ELL-row load of u instead
                        merge_keys(pkey, ppass, ppb);
                        ppb = 0;
                    }
                    // 1. visit u's neighbours, prefetch the new rows into L2
                    const bool isnew = visit_batch(vv, false);
                    if (status != 0) break;
#ifndef PA_ROWPF
#define PA_ROWPF 0                      // L2 bulk prefetch of the new rows: A/B on C1 2.5% slower
#endif
                    if (PA_ROWPF && isnew) prefetch_row_l2(row_ptr(vv), row_bytes);
                    // 2. merge the previous expansion's keys; runner-up r; its row speculatively
                    if (!PA_MERGE_FIRST) {
                        merge_keys(pkey, ppass, ppb);
                        ppb = 0;
                    }
                    int pr = -1;
                    for (int t = hint >> 5; t * 32 < csz; ++t) {
                        const int i = t * 32 + lane;
                        const unsigned b = __ballot_sync(kFull, i < csz && !key_checked(C[i]));
                        if (b) { pr = t * 32 + __ffs(b) - 1; break; }
                    }
                    const uint64_t key_r = pr >= 0 ? C[pr] : kKeyInf;
#ifndef PA_SPEC
#define PA_SPEC 1                       // A/B on C1: 4% faster with the speculative runner-up row
#endif
                    if (PA_SPEC && pr >= 0 && key_id(key_r) != spec_u) {
                        spec_u = key_id(key_r);
                        sv = __ldg(ix.ell + (int64_t)spec_u * 32 + lane);
                    }
                    // 3. δ' of the new neighbours, filter against C's worst
                    const uint64_t key = new_keys(vv, isnew);
                    const uint64_t thresh = csz == ef ? C[ef - 1] : kKeyInf;
                    bool pass = key < thresh;
#ifndef PA_ELLPF
#define PA_ELLPF 0                      // L2 prefetch of passing keys' ELL rows: A/B on C1 3% slower
#endif
                    if (PA_ELLPF && pass) prefetch_row_l2(ix.ell + (int64_t)key_id(key) * 32, 128);
                    const unsigned pb = __ballot_sync(kFull, pass);
                    uint64_t nstar = kKeyInf;
                    if (pb) {
                        const uint64_t kk = pass ? key : kKeyInf;
                        const uint32_t hi = __reduce_min_sync(kFull, (uint32_t)(kk >> 32));
                        const uint32_t lo = __reduce_min_sync(kFull, (uint32_t)(kk >> 32) == hi ? (uint32_t)kk : 0xffffffffu);
                        nstar = ((uint64_t)hi << 32) | lo;
                    }
                    // 4. next expansion = min(r, best passing new key)
                    const uint64_t nxt = nstar < key_r ? nstar : key_r;
                    pkey = key;
                    ppb = pb;
                    if (nxt == kKeyInf) { ppass = pass; break; }   // no unchecked node left (pb == 0)
                    if (nxt == key_r) {
                        __syncwarp();
                        if (lane == 0) C[pr] = key_r | 1ull;
                        __syncwarp();                         // visible before the next merge reads C
                        hint = pr + 1;
                    } else {
                        hint = pr >= 0 ? pr : csz;
                        if (pass && key == nstar) pkey = key | 1ull;      // checked when it is merged
                    }
                    ppass = pass;
                    u = key_id(nxt);
                    vv = (u == spec_u) ? sv : __ldg(ix.ell + (int64_t)u * 32 + lane);
                    if (it >= kIterCap) { status = 2; break; }
                }
                merge_keys(pkey, ppass, ppb);        // pending keys (overflow / cap exits)
            }
        }
        // ---- outputs
        const float inf = __int_as_float(0x7f800000);
        if (a.cand_ids) {
            for (int i = lane; i < ef; i += 32) {
                a.cand_ids[q * ef + i] = i < csz ? key_id(C[i]) : -1;
                a.cand_d[q * ef + i] = i < csz ? key_dist(C[i]) : inf;
            }
        }
        for (int i = lane; i < a.k; i += 32) {
            a.out_ids[q * a.k + i] = i < csz ? key_id(C[i]) : -1;
            a.out_d[q * a.k + i] = i < csz ? key_dist(C[i]) : inf;
        }
        for (int i = lane; i < vs.count2; i += 32) vs.G[vs.log[i]] = 0u;
        __syncwarp();
        if (lane == 0) {
            if (a.counters) {
                int4 c4 = make_int4(n_exp, n_dist, n_spill, status);
                reinterpret_cast<int4*>(a.counters)[q] = c4;
            }
            if (TRACE) { a.trace_nexp[q] = n_exp; a.trace_nvis[q] = n_dist; }
        }
        __syncwarp();
    }
}

}  // namespace trav
}  // namespace pa

namespace pa {
namespace trav {

// ---------------------------------------------------------------------------
// NEXT-f3: stages ② and ③ on the GPU when the rotated full vectors X̂ fit in
// HBM (oracle O8-O9).  One warp per query, exact visited set (the
// compact/wide smem hash + global spill of the stage-① exact kernel):
//   ② C := the stage-① candidates with full δ (all visited, the ef2 best kept,
//      Q8 resize semantics), then `refine_iters` Alg 1 expansions on the
//      SUBGRAPH with full δ;
//   ③ every entry of C unchecked again, capacity ef3, Alg 1 on the FULL graph
//      with full δ until no unchecked node, the visited set carried over (Q23).
// PA_NO_STAGE2 skips ②'s expansions and keeps ef3 entries.  Rows of X̂ are
// gathered 8 lanes per row (128-B segments; D = 96 rows are 384 B).
#ifndef PA_REFINE_L
#define PA_REFINE_L 4                  // lanes per X̂ row in the stage ②③ gathers (A/B: 8 is 8% slower)
#endif
template <int METRIC, int VIS, int SMAX, int NVR>
#ifndef PA_REFINE_MINB
#define PA_REFINE_MINB 6
#endif
__global__ void __launch_bounds__(kTW * 32, PA_REFINE_MINB) k_refine(Refine23 a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int cap = max(a.ef2, a.ef3), S = 1 << a.hash_log2;
    const int efp = (cap + 1) & ~1;
    const int qlen = a.qlen;                                   // D rounded up to 4
    const size_t per_warp = (size_t)efp * 8 + (size_t)qlen * 4 + 128 + (size_t)S * (VIS == 1 ? 2 : 4);
    unsigned char* base = smem_raw + per_warp * w;
    uint64_t* C = reinterpret_cast<uint64_t*>(base);
    float* qs = reinterpret_cast<float*>(C + efp);
    int32_t* scr = reinterpret_cast<int32_t*>(qs + qlen);
    int32_t* H = scr + 32;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int64_t gw = (int64_t)blockIdx.x * kTW + w;
    Visited vs;
    vs.H = H;
    vs.log2S = a.hash_log2;
    vs.G = reinterpret_cast<uint32_t*>(a.spill + ((int64_t)gw << a.spill_log2));
    vs.log = vs.G + ((size_t)1 << a.spill_log2);
    vs.gmask = (1u << a.spill_log2) - 1u;
    const int cap1 = S >> 1, cap2 = (int)(vs.gmask >> 1);
    const unsigned char* rows = reinterpret_cast<const unsigned char*>(a.xhat);
    const int64_t stride = (int64_t)a.xstride * 4;
    const int nvr = qlen >> 2;

    for (;;) {
        int64_t q = 0;
        if (lane == 0) q = atomicAdd(a.work, 1);
        q = __shfl_sync(kFull, (int)q, 0);
        if (q >= a.m) break;
        vs.count1 = 0;
        vs.count2 = 0;
        for (int i = lane; i < qlen; i += 32)                   // q̂ = [q', q_res] (rotated query, fp32)
            qs[i] = i < a.dp ? a.qp[q * a.qp_stride + i] : (i < a.D ? a.qres[q * (a.D - a.dp) + (i - a.dp)] : 0.f);
        int4* H4 = reinterpret_cast<int4*>(H);
        for (int i = lane; i < (S >> (VIS == 1 ? 3 : 2)); i += 32) H4[i] = make_int4(-1, -1, -1, -1);
        __syncwarp();
        int csz = 0, hint = 0, status = 0, n2 = 0, n3 = 0;
        int ef = (a.flags & 2u) ? a.ef3 : a.ef2;                // current capacity of C
        int* nd = &n2;
        auto step = [&](int32_t v, bool unconditional) {
            const bool open1 = vs.count1 + 32 <= cap1;
            if (!open1 && vs.count2 + 32 > cap2) { status = 1; return; }
            bool l2 = false;
            uint32_t slot = 0;
            const bool isnew = v >= 0 && visit<VIS>(vs, v, open1, l2, slot);
            const unsigned bl2 = __ballot_sync(kFull, l2);
            if (l2) vs.log[vs.count2 + __popc(bl2 & lt_mask)] = slot;
            const unsigned bal = __ballot_sync(kFull, isnew);
            const int nnew = __popc(bal);
            vs.count1 += nnew - __popc(bl2);
            vs.count2 += __popc(bl2);
            *nd += nnew;
            (void)unconditional;
            if (nnew == 0) return;
            if (isnew) scr[__popc(bal & lt_mask)] = v;
            __syncwarp();
            const int32_t cid = lane < nnew ? scr[lane] : 0;
            __syncwarp();
            const float d = group_dists<METRIC, NVR, false, PA_REFINE_L, true>(qs, rows, stride, nvr, cid, nnew, lane);
            const uint64_t key = lane < nnew ? make_key(d, cid) : kKeyInf;
            const uint64_t thresh = csz == ef ? C[ef - 1] : kKeyInf;
            const bool pass = key < thresh;
            const unsigned pb = __ballot_sync(kFull, pass);
            if (pb == 0) return;
            int minr;
            csz = rank_merge<SMAX>(C, csz, ef, key, pass, pb, lane, minr);
            hint = min(hint, minr);
        };
        // Alg 1 loop; the runner-up unchecked node's ELL row is loaded speculatively
        // with the current one (it is the next expansion unless a new key beats it).
        auto expand = [&](const int32_t* ell, int ellw, int max_it) {
            int32_t spec_u = -1, sv0 = -1, sv1 = -1;
            for (int it = 0; status == 0 && (max_it < 0 || it < max_it); ++it) {
                if (a.width > 1) {                               // search width w (O6), as in k_traverse
                    int ps[kMaxWidth];
                    int nu = 0;
                    for (int t = hint >> 5; t * 32 < csz && nu < a.width; ++t) {
                        const int i = t * 32 + lane;
                        unsigned b = __ballot_sync(kFull, i < csz && !key_checked(C[i]));
#pragma unroll
                        for (int x = 0; x < kMaxWidth; ++x)
                            if (b && nu < a.width) { ps[nu++] = t * 32 + __ffs(b) - 1; b &= b - 1; }
                    }
                    if (nu == 0) break;
                    int32_t us[kMaxWidth];
#pragma unroll
                    for (int x = 0; x < kMaxWidth; ++x) us[x] = x < nu ? key_id(C[ps[x]]) : -1;
                    __syncwarp();
                    if (lane == 0)
                        for (int x = 0; x < nu; ++x) C[ps[x]] |= 1ull;
                    hint = ps[nu - 1] + 1;
                    __syncwarp();
#pragma unroll
                    for (int x = 0; x < kMaxWidth; ++x) {
                        if (x >= nu || status != 0) break;
                        step(__ldg(ell + (int64_t)us[x] * ellw + lane), false);
                        if (ellw > 32 && status == 0) step(__ldg(ell + (int64_t)us[x] * ellw + 32 + lane), false);
                    }
                    if (it >= kIterCap) status = 2;
                    continue;
                }
                int p = -1, p2 = -1;
                for (int t = hint >> 5; t * 32 < csz; ++t) {
                    const int i = t * 32 + lane;
                    const unsigned b = __ballot_sync(kFull, i < csz && !key_checked(C[i]));
                    if (b) {
                        p = t * 32 + __ffs(b) - 1;
                        const unsigned b2 = b & (b - 1);
                        if (b2) p2 = t * 32 + __ffs(b2) - 1;
                        break;
                    }
                }
                if (p < 0) break;                                // Alg 1 l.12
                const int32_t u = key_id(C[p]);
                int32_t v0, v1 = -1;
                if (u == spec_u) {
                    v0 = sv0; v1 = sv1;
                } else {
                    v0 = __ldg(ell + (int64_t)u * ellw + lane);
                    if (ellw > 32) v1 = __ldg(ell + (int64_t)u * ellw + 32 + lane);
                }
                spec_u = p2 >= 0 ? key_id(C[p2]) : -1;
                if (spec_u >= 0) {
                    sv0 = __ldg(ell + (int64_t)spec_u * ellw + lane);
                    sv1 = ellw > 32 ? __ldg(ell + (int64_t)spec_u * ellw + 32 + lane) : -1;
                }
                __syncwarp();
                if (lane == 0) C[p] |= 1ull;
                hint = p + 1;
                __syncwarp();
                step(v0, false);
                if (ellw > 32 && status == 0) step(v1, false);
                if (it >= kIterCap) status = 2;
            }
        };
        // ---- ② C := candidates with full δ, all visited (O8)
        for (int j0 = 0; j0 < a.ef1 && status == 0; j0 += 32) {
            const int j = j0 + lane;
            step(j < a.ef1 ? a.cand[q * a.ef1 + j] : -1, true);
        }
        if (!(a.flags & 2u) && a.refine_iters > 0) expand(a.sub_ell, a.sub_w, a.refine_iters);
        // ---- ③ carry unchecked, capacity ef3, Alg 1 on the full graph (O9)
        for (int i = lane; i < csz; i += 32) C[i] &= ~1ull;
        __syncwarp();
        ef = a.ef3;
        if (csz > ef) csz = ef;
        hint = 0;
        nd = &n3;
        expand(a.full_ell, a.full_w, -1);
        const float inf = __int_as_float(0x7f800000);
        for (int i = lane; i < a.k; i += 32) {
            a.out_ids[q * a.k + i] = i < csz ? key_id(C[i]) : -1;
            a.out_d[q * a.k + i] = i < csz ? key_dist(C[i]) : inf;
        }
        for (int i = lane; i < vs.count2; i += 32) vs.G[vs.log[i]] = 0u;
        __syncwarp();
        if (lane == 0 && a.counters) reinterpret_cast<int4*>(a.counters)[q] = make_int4(n2, n3, 0, status);
        __syncwarp();
    }
}

}  // namespace trav
}  // namespace pa
