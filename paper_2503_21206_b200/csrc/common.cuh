// Device helpers shared by the product kernels (NOT by the oracle).
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace pa {

constexpr uint64_t kKeyInf = ~0ull;
constexpr unsigned kFull = 0xffffffffu;

// Orderable 32-bit image of an fp32 distance: unsigned order == float order.
// −0.0 is canonicalised to +0.0 so that equal distances compare equal (Q13).
__device__ __forceinline__ uint32_t ord_of(float d) {
    uint32_t b = __float_as_uint(d == 0.0f ? 0.0f : d);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float dist_of_ord(uint32_t o) {
    uint32_t b = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
    return __uint_as_float(b);
}
// Candidate key: (ord(δ) << 32) | (id << 1) | checked.  Keys
// order by (δ, id) — the oracle's (δ, id) lexicographic order (Q13).
__device__ __forceinline__ uint64_t make_key(float d, int32_t id) {
    return ((uint64_t)ord_of(d) << 32) | ((uint64_t)(uint32_t)id << 1);
}
__device__ __forceinline__ int32_t key_id(uint64_t k) { return (int32_t)(((uint32_t)k) >> 1); }
__device__ __forceinline__ float key_dist(uint64_t k) { return dist_of_ord((uint32_t)(k >> 32)); }
__device__ __forceinline__ bool key_checked(uint64_t k) { return (k & 1ull) != 0; }

__device__ __forceinline__ uint64_t shfl_xor64(uint64_t v, int m) {
    uint32_t lo = __shfl_xor_sync(kFull, (uint32_t)v, m);
    uint32_t hi = __shfl_xor_sync(kFull, (uint32_t)(v >> 32), m);
    return ((uint64_t)hi << 32) | lo;
}

// Ascending bitonic sort of one 64-bit key per lane across the warp.
__device__ __forceinline__ uint64_t warp_sort32(uint64_t x, int lane) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            uint64_t y = shfl_xor64(x, j);
            bool up = (lane & k) == 0;
            bool lower = (lane & j) == 0;
            bool take_min = (lower == up);
            uint64_t mn = x < y ? x : y, mx = x < y ? y : x;
            x = take_min ? mn : mx;
        }
    }
    return x;
}

// Number of elements of sorted smem array a[0..n) strictly less than x.
__device__ __forceinline__ int lower_bound_smem(const uint64_t* a, int n, uint64_t x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Merge the warp-sorted keys `x` (nnew valid, ascending across lanes 0..nnew)
// into the sorted list A[0..csz) keeping the `cap` smallest; result in B.
// Rank-based: every key lands at (own index + rank in the other list).  Keys
// are unique (distinct ids), so the two rank counts partition positions.
// N is a 32-entry smem scratch.  Returns the new size.
__device__ __forceinline__ int warp_merge(const uint64_t* A, int csz, uint64_t x, int nnew,
                                          uint64_t* B, uint64_t* N, int cap, int lane) {
    N[lane] = x;
    __syncwarp();
    if (lane < nnew) {
        int pos = lane + lower_bound_smem(A, csz, x);
        if (pos < cap) B[pos] = x;
    }
    for (int i = lane; i < csz; i += 32) {
        uint64_t a = A[i];
        int pos = i + lower_bound_smem(N, nnew, a);
        if (pos < cap) B[pos] = a;
    }
    __syncwarp();
    int ns = csz + nnew;
    return ns < cap ? ns : cap;
}

#ifndef PA_MERGE_BS_MIN_SMAX
#define PA_MERGE_BS_MIN_SMAX 8         // binary-search merge from lists of > 128 keys (A/B: profiles/r2_ab_rank_merge.txt)
#endif
// Binary-search form of rank_merge (same positions, fewer instructions on long
// lists): every passing lane finds its key's rank rc in C by a binary search of
// the smem list (log2(32·SMAX) dependent loads).  Keys are unique, so entry i
// moves right by #{j : rc_j ≤ i}; for the entries lane l owns (i = l + 32t) that
// is #{j : t ≥ ⌈(rc_j − l)/32⌉⁺}: each broadcast (rc_j, key_j) adds one to byte
// ⌈(rc_j − l)/32⌉⁺ of a packed histogram and one multiply by 0x0101…01 turns the
// bytes into prefix sums (≤ 32 keys per byte: no carry).  A passing key lands at
// rc + #{passing keys below it}.
template <int SMAX>
__device__ __forceinline__ int rank_merge_bs(uint64_t* C, int csz, int cap, uint64_t key, bool pass, unsigned pb,
                                             int lane, int& minr) {
    static_assert(SMAX <= 16, "two histogram words");
    uint64_t c[SMAX];
#pragma unroll
    for (int t = 0; t < SMAX; ++t) {
        const int i = lane + 32 * t;
        c[t] = i < csz ? C[i] : kKeyInf;
    }
    constexpr int P = (32 * SMAX) >= 512 ? 512 : (32 * SMAX) >= 256 ? 256 : 128;   // ≤ 32·SMAX, 2P − 1 ≥ 32·SMAX
    int rc = 0;
    if (pass) {
#pragma unroll
        for (int step = P; step > 0; step >>= 1)
            if (rc + step <= csz && C[rc + step - 1] < key) rc += step;
    }
    minr = (int)__reduce_min_sync(kFull, pass ? (unsigned)rc : 0xFFFFFFFFu);
    const int np = __popc(pb);
    uint64_t h0 = 0, h1 = 0;
    int rn = 0;
    while (pb) {
        const int s = __ffs(pb) - 1;
        pb &= pb - 1;
        const int rj = __shfl_sync(kFull, rc, s);
        const uint32_t kh = __shfl_sync(kFull, (uint32_t)(key >> 32), s);
        const uint32_t kl = __shfl_sync(kFull, (uint32_t)key, s);
        rn += ((((uint64_t)kh << 32) | kl) < key) ? 1 : 0;
        const int d = rj - lane;
        const int tj = d <= 0 ? 0 : (d + 31) >> 5;
        if (tj < 8) h0 += 1ull << (8 * tj);
        else if (SMAX > 8 && tj < 16) h1 += 1ull << (8 * (tj - 8));
    }
    const uint64_t p0 = h0 * 0x0101010101010101ull;
    const uint64_t p1 = h1 * 0x0101010101010101ull + (p0 >> 56) * 0x0101010101010101ull;
    __syncwarp();
#pragma unroll
    for (int t = 0; t < SMAX; ++t) {
        const int i = lane + 32 * t;
        const int sh = (int)(((t < 8 ? p0 : p1) >> (8 * (t & 7))) & 0xFFu);
        const int pos = i + sh;
        if (i < csz && sh != 0 && pos < cap) C[pos] = c[t];
    }
    if (pass) {
        const int pos = rc + rn;
        if (pos < cap) C[pos] = key;
    }
    __syncwarp();
    minr = minr < cap ? minr : cap;
    return min(csz + np, cap);
}

// In-place rank merge of the passing lanes' keys (ballot `pb` ≠ 0) into the
// sorted smem list C[0..csz) with capacity cap ≤ 32·SMAX; returns the new size
// and (minr) the smallest position a new key landed at.  Every passing key is
// broadcast once; each lane counts how many of them precede each C entry it
// owns (the entry's right shift) and its own key's rank among them; the key's
// rank in C is a per-lane binary search.  Keys are unique, so the final
// positions rank_C(x) + #{passing < x} and i + shift(i) form a permutation and
// everything moves in place (the old C sits in registers across one __syncwarp).
template <int SMAX>
__device__ __forceinline__ int rank_merge(uint64_t* C, int csz, int cap, uint64_t key, bool pass, unsigned pb,
                                          int lane, int& minr) {
    if constexpr (SMAX >= PA_MERGE_BS_MIN_SMAX && SMAX <= 16) return rank_merge_bs<SMAX>(C, csz, cap, key, pass, pb, lane, minr);
    uint64_t c[SMAX];
    int sh[SMAX];
#pragma unroll
    for (int t = 0; t < SMAX; ++t) {
        const int i = lane + 32 * t;
        c[t] = i < csz ? C[i] : kKeyInf;
        sh[t] = 0;
    }
    const int np = __popc(pb);
    int rn = 0, rc = 0;
    minr = cap;
    // two passing keys per step: independent shuffles overlap, and each key's rank
    // in C is counted with SMAX ballots (no dependent binary search)
    while (pb) {
        const int s0 = __ffs(pb) - 1;
        pb &= pb - 1;
        const int s1 = pb ? __ffs(pb) - 1 : s0;
        const bool two = pb != 0;
        pb = two ? (pb & (pb - 1)) : pb;
        const uint32_t h0 = __shfl_sync(kFull, (uint32_t)(key >> 32), s0);
        const uint32_t l0 = __shfl_sync(kFull, (uint32_t)key, s0);
        const uint32_t h1 = __shfl_sync(kFull, (uint32_t)(key >> 32), s1);
        const uint32_t l1 = __shfl_sync(kFull, (uint32_t)key, s1);
        const uint64_t x0 = ((uint64_t)h0 << 32) | l0;
        const uint64_t x1 = ((uint64_t)h1 << 32) | l1;
        int r0 = 0, r1 = 0;
#pragma unroll
        for (int t = 0; t < SMAX; ++t) {
            const bool lt0 = c[t] < x0, lt1 = c[t] < x1;
            sh[t] += (lt0 ? 0 : 1) + ((two && !lt1) ? 1 : 0);
            r0 += __popc(__ballot_sync(kFull, lt0));
            r1 += __popc(__ballot_sync(kFull, lt1));
        }
        if (lane == s0) rc = r0;
        if (two && lane == s1) rc = r1;
        minr = min(minr, two ? min(r0, r1) : r0);
        rn += (x0 < key) ? 1 : 0;
        rn += (two && x1 < key) ? 1 : 0;
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < SMAX; ++t) {
        const int i = lane + 32 * t;
        const int pos = i + sh[t];
        if (i < csz && pos < cap) C[pos] = c[t];
    }
    if (pass) {
        const int pos = rc + rn;
        if (pos < cap) C[pos] = key;
    }
    __syncwarp();
    return min(csz + np, cap);
}

// Direct-form distance (Alg 1 l.8) between an smem query row and a global row
// of `dps` floats (multiple of 4, 16-B aligned): L2 = Σ(x−q)², IP = −Σ x·q.
// Four independent fp32 FMA chains over float4 slices (Q24: fp32, RNE, FMA).
template <int METRIC>
__device__ __forceinline__ float row_dist(const float* __restrict__ qs, const float* __restrict__ x, int dps) {
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const float4* q4 = reinterpret_cast<const float4*>(qs);
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    const int n4 = dps >> 2;
#pragma unroll 4
    for (int i = 0; i < n4; ++i) {
        float4 v = __ldg(x4 + i);
        float4 w = q4[i];
        if (METRIC == 0) {
            float d0 = v.x - w.x, d1 = v.y - w.y, d2 = v.z - w.z, d3 = v.w - w.w;
            a0 = fmaf(d0, d0, a0); a1 = fmaf(d1, d1, a1); a2 = fmaf(d2, d2, a2); a3 = fmaf(d3, d3, a3);
        } else {
            a0 = fmaf(v.x, w.x, a0); a1 = fmaf(v.y, w.y, a1); a2 = fmaf(v.z, w.z, a2); a3 = fmaf(v.w, w.w, a3);
        }
    }
    float s = (a0 + a1) + (a2 + a3);
    return METRIC == 0 ? s : -s;
}

// Packed fp32x2 arithmetic (sm_100 FADD2/FFMA2): each half is an IEEE fp32
// operation with round-to-nearest, bit-identical to the scalar FADD/FFMA, at
// half the issue slots.
__device__ __forceinline__ void sub2(float ax, float ay, float bx, float by, float& rx, float& ry) {
    asm("{.reg .b64 a, b, r;\n\t"
        "mov.b64 a, {%2, %3};\n\t"
        "mov.b64 b, {%4, %5};\n\t"
        "sub.rn.f32x2 r, a, b;\n\t"
        "mov.b64 {%0, %1}, r;}"
        : "=f"(rx), "=f"(ry) : "f"(ax), "f"(ay), "f"(bx), "f"(by));
}
__device__ __forceinline__ void fma2(float ax, float ay, float bx, float by, float& cx, float& cy) {
    asm("{.reg .b64 a, b, c;\n\t"
        "mov.b64 a, {%2, %3};\n\t"
        "mov.b64 b, {%4, %5};\n\t"
        "mov.b64 c, {%0, %1};\n\t"
        "fma.rn.f32x2 c, a, b, c;\n\t"
        "mov.b64 {%0, %1}, c;}"
        : "+f"(cx), "+f"(cy) : "f"(ax), "f"(ay), "f"(bx), "f"(by));
}
// acc[0..3] += (v − w)² (L2) or v·w (IP), component-wise: the same four fp32
// chains as the scalar code, issued as two packed pairs.
// PACKED selects the fp32x2 form: measured on C1 it is 9% slower in the fp32-row
// traversal (register pressure at the 80-register budget) and 1% faster with
// binary16 rows, so only the binary16 path uses it.
template <int METRIC, bool PACKED>
__device__ __forceinline__ void acc4(const float4 v, const float4 w, float& a0, float& a1, float& a2, float& a3) {
    if (!PACKED) {
        if (METRIC == 0) {
            const float d0 = v.x - w.x, d1 = v.y - w.y, d2 = v.z - w.z, d3 = v.w - w.w;
            a0 = fmaf(d0, d0, a0); a1 = fmaf(d1, d1, a1); a2 = fmaf(d2, d2, a2); a3 = fmaf(d3, d3, a3);
        } else {
            a0 = fmaf(v.x, w.x, a0); a1 = fmaf(v.y, w.y, a1); a2 = fmaf(v.z, w.z, a2); a3 = fmaf(v.w, w.w, a3);
        }
    } else if (METRIC == 0) {
        float d0, d1, d2, d3;
        sub2(v.x, v.y, w.x, w.y, d0, d1);
        sub2(v.z, v.w, w.z, w.w, d2, d3);
        fma2(d0, d1, d0, d1, a0, a1);
        fma2(d2, d3, d2, d3, a2, a3);
    } else {
        fma2(v.x, v.y, w.x, w.y, a0, a1);
        fma2(v.z, v.w, w.z, w.w, a2, a3);
    }
}

#ifndef PA_ROW_GROUP
#define PA_ROW_GROUP 16                // float4 loads of a row in flight before the first FMA
#endif
// Same, with the row length a compile-time number of float4s: every load of the
// row is issued before the first FMA (one DRAM round trip per row instead of
// one per unroll group); DPS4 == 0 falls back to the runtime loop.
template <int METRIC, int DPS4>
__device__ __forceinline__ float row_dist_t(const float* __restrict__ qs, const float* __restrict__ x, int dps) {
    if constexpr (DPS4 == 0) {
        return row_dist<METRIC>(qs, x, dps);
    } else {
        // rows longer than 16 float4 (d' > 64) go in 16-float4 groups to bound registers
        constexpr int G = (DPS4 % PA_ROW_GROUP == 0) ? PA_ROW_GROUP : (DPS4 > 16 ? 16 : DPS4);
        static_assert(DPS4 % G == 0, "row length must be a multiple of the group");
        const float4* x4 = reinterpret_cast<const float4*>(x);
        const float4* q4 = reinterpret_cast<const float4*>(qs);
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
        for (int g = 0; g < DPS4; g += G) {
            float4 v[G];
#pragma unroll
            for (int i = 0; i < G; ++i) v[i] = __ldg(x4 + g + i);
#pragma unroll
            for (int i = 0; i < G; ++i) acc4<METRIC, false>(v[i], q4[g + i], a0, a1, a2, a3);
        }
        const float s = (a0 + a1) + (a2 + a3);
        return METRIC == 0 ? s : -s;
    }
}

// Direct-form distance to a binary16-stored row (NEXT-f1: half the gather bytes).
// Values are widened exactly to fp32; arithmetic as in row_dist_t.  NV = number of
// 16-B vectors (8 halves each) per row, all loads in flight; NV == 0 → runtime loop.
__device__ __forceinline__ void acc8(const uint4 u, const float4 w0, const float4 w1, int metric, float& a0, float& a1,
                                     float& a2, float& a3) {
    const __half2* h = reinterpret_cast<const __half2*>(&u);
    const float2 f0 = __half22float2(h[0]), f1 = __half22float2(h[1]), f2 = __half22float2(h[2]), f3 = __half22float2(h[3]);
    if (metric == 0) {
        acc4<0, true>(make_float4(f0.x, f0.y, f1.x, f1.y), w0, a0, a1, a2, a3);
        acc4<0, true>(make_float4(f2.x, f2.y, f3.x, f3.y), w1, a0, a1, a2, a3);
    } else {
        acc4<1, true>(make_float4(f0.x, f0.y, f1.x, f1.y), w0, a0, a1, a2, a3);
        acc4<1, true>(make_float4(f2.x, f2.y, f3.x, f3.y), w1, a0, a1, a2, a3);
    }
}

template <int METRIC, int NV>
__device__ __forceinline__ float row_dist_h(const float* __restrict__ qs, const __half* __restrict__ x, int dph) {
    const uint4* x4 = reinterpret_cast<const uint4*>(x);
    const float4* q4 = reinterpret_cast<const float4*>(qs);
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    if constexpr (NV == 0) {
        for (int i = 0; i < (dph >> 3); ++i) acc8(__ldg(x4 + i), q4[2 * i], q4[2 * i + 1], METRIC, a0, a1, a2, a3);
    } else {
        uint4 v[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) v[i] = __ldg(x4 + i);
#pragma unroll
        for (int i = 0; i < NV; ++i) acc8(v[i], q4[2 * i], q4[2 * i + 1], METRIC, a0, a1, a2, a3);
    }
    const float s = (a0 + a1) + (a2 + a3);
    return METRIC == 0 ? s : -s;
}

// δ' of up to 32 new ids (compacted: lane r holds the r-th id in `cid`, r < nnew)
// with L lanes per row: lane j of group g reads 16-B chunks k·L + j of row
// RPP·p + g in pass p (RPP = 32/L rows per pass), so each load instruction
// fetches L·16 contiguous bytes of each of RPP rows (rows start on 128-B lines:
// `stride` bytes, a multiple of 128).  Measured on this GPU
// (scripts/micro/gather_bw.cu), random gathers with 16 B per lane per row cap at
// ~1.3 TB/s; 64-B (L = 4) and 128-B (L = 8) row segments reach 2.5–6 TB/s.  Partial
// sums are reduced over the L lanes (butterfly) and sent back to lane r.  NVR =
// 16-B chunks per row (fp32: d'/4, binary16: d'/8; 0 = runtime `nvr`).  Returns
// lane r's δ'.
// PACKED32: fp32 rows use the fp32x2 FADD2/FFMA2 form (bit-identical per element).
// Measured on C1: 6% faster in the exact-visited kernel, 4% slower in the bloom one.
#ifndef PA_DIST_PG_MUL
#define PA_DIST_PG_MUL 1               // × row passes whose loads are issued together (registers ↔ MLP)
#endif
template <int METRIC, int NVR, bool H16, int L, bool PACKED32>
__device__ __forceinline__ float group_dists(const float* __restrict__ qs, const unsigned char* __restrict__ base,
                                             int64_t stride, int nvr, int32_t cid, int nnew, int lane) {
    constexpr int RPP = 32 / L;
    const int g = lane / L, j = lane % L;
    const float4* q4 = reinterpret_cast<const float4*>(qs);
    constexpr int F = NVR > 0 ? (NVR + L - 1) / L : 1;      // chunks per lane (compile-time rows)
    // passes whose loads are in flight together (≈ 16 float4 registers); whole-line rows (L = 8) keep 2
#ifndef PA_WIDE_PG
#define PA_WIDE_PG 2
#endif
    constexpr int PG = (L == 8 && F == 4 ? PA_WIDE_PG : (F >= 4 ? 1 : (F >= 2 ? 2 : 4))) * PA_DIST_PG_MUL;
    float mine = 0.f;
#ifndef PA_DIST_PF
#define PA_DIST_PF 0                   // L2 bulk prefetch of the rows beyond the first PG passes
#endif
    // Rows of later load passes: one 1-D bulk L2 prefetch per row (lane r, row r), so
    // those passes' loads hit L2 instead of each paying a DRAM round trip.
    if (PA_DIST_PF && NVR > 0 && lane >= PG * RPP && lane < nnew)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                     :: "l"(base + (int64_t)cid * stride), "r"(NVR * 16) : "memory");
    // fp32 rows are loaded as float4 and binary16 rows as uint4 (no reinterpretation
    // copies); lanes of rows past nnew issue no load and their registers are left
    // unset: their sums stay inside their own L-lane group and are never returned
    // (a zero-fill select cost ~45 register moves per expansion, ncu r2 source counters).
#ifndef PA_DIST_NOZERO
#define PA_DIST_NOZERO 0
#endif
    using VT = typename std::conditional<H16, uint4, float4>::type;
    for (int p0 = 0; p0 * RPP < nnew; p0 += PG) {
        VT v[PG][F];
        int32_t rid[PG];
#pragma unroll
        for (int pp = 0; pp < PG; ++pp) {
            const int rr = (p0 + pp) * RPP + g;
            rid[pp] = __shfl_sync(kFull, PA_DIST_NOZERO == 2 && rr >= nnew ? 0 : cid, PA_DIST_NOZERO == 2 && rr >= nnew ? 0 : (rr & 31));
            if (NVR > 0) {
                const VT* row = reinterpret_cast<const VT*>(base + (int64_t)rid[pp] * stride);
                const bool ok = PA_DIST_NOZERO == 2 || rr < nnew;   // 2: rows past nnew re-read row 0 of the batch (L1 hit)
#pragma unroll
                for (int k = 0; k < F; ++k) {
#if PA_DIST_NOZERO == 1
                    if (k * L + j < NVR && ok) v[pp][k] = __ldg(row + k * L + j);
#elif PA_DIST_NOZERO == 2
                    if (k * L + j < NVR) v[pp][k] = __ldg(row + k * L + j);
#else
                    v[pp][k] = (k * L + j < NVR && ok) ? __ldg(row + k * L + j) : VT{};
#endif
                }
            }
        }
#pragma unroll
        for (int pp = 0; pp < PG; ++pp) {
            if ((p0 + pp) * RPP >= nnew) break;                    // warp-uniform
            const int rr = (p0 + pp) * RPP + g;
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
            if (NVR > 0) {
#pragma unroll
                for (int k = 0; k < F; ++k) {
                    const int c = k * L + j;
                    if (c >= NVR) continue;
                    if constexpr (H16) acc8(v[pp][k], q4[2 * c], q4[2 * c + 1], METRIC, a0, a1, a2, a3);
                    else acc4<METRIC, PACKED32>(v[pp][k], q4[c], a0, a1, a2, a3);
                }
            } else if (rr < nnew) {                                // runtime row length (trace builds)
                const uint4* row = reinterpret_cast<const uint4*>(base + (int64_t)rid[pp] * stride);
                for (int c = j; c < nvr; c += L) {
                    const uint4 u = __ldg(row + c);
                    if constexpr (H16) acc8(u, q4[2 * c], q4[2 * c + 1], METRIC, a0, a1, a2, a3);
                    else acc4<METRIC, false>(*reinterpret_cast<const float4*>(&u), q4[c], a0, a1, a2, a3);
                }
            }
            float sum = (a0 + a1) + (a2 + a3);
#pragma unroll
            for (int o = L / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(kFull, sum, o);
            const float t = __shfl_sync(kFull, sum, (lane % RPP) * L);
            if (lane / RPP == p0 + pp) mine = t;
        }
    }
    return METRIC == 0 ? mine : -mine;
}

__device__ __forceinline__ uint64_t warp_min64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t w = shfl_xor64(v, o);
        v = w < v ? w : v;
    }
    return v;
}

}  // namespace pa
