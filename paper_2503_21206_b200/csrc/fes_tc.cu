// a3 + a4 — FES bucketing and within-cell scoring on the tensor cores.
//
// Alg 2 assigns one GPU block per cluster and skips the queries
// routed elsewhere ("allocation-free").  Here:
//   k_bucket  : stable counting sort of the queries by routed cell → perm,
//               per-cell query offsets and per-cell 128-query tile offsets (a3).
//   k_fes_scores_tma : one CTA per (cell, 128 routed queries) tile — a grouped GEMM
//               S = Q'_tile · EV_cellᵀ on tcgen05 (kind::tf32, 3xTF32, M = 128,
//               N = 128 pool entries per pass, accumulator in TMEM); epilogue
//               score = ‖e‖² − 2 q'·e (L2) or −q'·e (IP) → global scratch.
//   k_fes_select : one warp per query keeps the E smallest (score, id) keys by a radix select
//               (Q10: the GEMM form is used for SELECTION only; stage ①
//               recomputes direct-form δ).  Splitting the selection out keeps
//               32+ warps per SM on it instead of the 4 epilogue warps of a tile.
// Every GEMM tile is dense (cell-centric tiling, Table 3 density mn/(r(m+n)),
// P:L417).
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "internal.h"
#include "umma.cuh"

namespace pa {

namespace {

constexpr int kM = 128;
constexpr int kN = 128;
constexpr int kThreads = 128;
constexpr int kMaxR = 64;

// ---------------------------------------------------------------- bucketing
__global__ void __launch_bounds__(1024, 1) k_bucket(const int32_t* __restrict__ cell, int64_t m, int r, int mq,
                                                    int32_t* __restrict__ perm, int32_t* __restrict__ qoff,
                                                    int32_t* __restrict__ toff) {
    __shared__ int cnt[kMaxR], base[kMaxR];
    __shared__ int wc[32][kMaxR];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    for (int c = tid; c < r; c += blockDim.x) cnt[c] = 0;
    __syncthreads();
    for (int64_t i = tid; i < m; i += blockDim.x) atomicAdd(&cnt[cell[i]], 1);
    __syncthreads();
    if (tid == 0) {
        int run = 0, trun = 0;
        for (int c = 0; c < r; ++c) {
            base[c] = run;
            qoff[c] = run;
            toff[c] = trun;
            run += cnt[c];
            trun += (cnt[c] + mq - 1) / mq;
        }
        qoff[r] = run;
        toff[r] = trun;
    }
    __syncthreads();
    for (int64_t t0 = 0; t0 < m; t0 += 1024) {
        for (int c = lane; c < r; c += 32) wc[w][c] = 0;
        __syncwarp();
        const int64_t i = t0 + tid;
        const bool ok = i < m;
        const int c = ok ? cell[i] : -1;
        const unsigned act = __ballot_sync(0xffffffffu, ok);
        unsigned peers = 0;
        int rk = 0;
        if (ok) {
            peers = __match_any_sync(act, c);
            rk = __popc(peers & ((1u << lane) - 1u));
            if (rk == 0) wc[w][c] = __popc(peers);
        }
        __syncthreads();
        for (int cc = tid; cc < r; cc += blockDim.x) {
            int run = base[cc];
            for (int ww = 0; ww < 32; ++ww) {
                const int x = wc[ww][cc];
                wc[ww][cc] = run;
                run += x;
            }
            base[cc] = run;
        }
        __syncthreads();
        if (ok) perm[wc[w][c] + rk] = (int32_t)i;
        __syncthreads();
    }
}

struct FesParams {
    const float* qp;
    int dps, kchunks;
    const int32_t* perm;
    const int32_t* qoff;
    const int32_t* toff;
    int r;
    const float* pool_vec;
    const float* pool_norm;
    const int32_t* pool_ids;
    const int32_t* cell_off;
    int metric;
    const float* pool_img;       // [chunks][kch][hi,lo][4096] pre-split, pre-swizzled B tiles (TMA source)
    const int32_t* chunk_off;    // [r+1] first 128-entry chunk of each cell
    float* scores;               // [m][sstride] GEMM-form scores, row = bucketed position
    int sstride;                 // ≥ max cell size, multiple of 4
    int E;
    int32_t* entries;
    bool fold_norm;              // pool_img carries ‖e‖² in K column dps (A has 1 there): acc = score
};


// Same GEMM, warp-specialised and pipelined: warp 4 (one elected thread) streams
// the cell's pre-split, pre-swizzled pool tiles with 1-D TMA bulk copies into a
// 2-stage smem ring (full/empty mbarriers) and issues the tcgen05.mma; the
// accumulator is double-buffered in TMEM (2 × 128 columns, ready/free
// mbarriers) so warps 0-3 drain chunk j (tcgen05.ld → scores) while the tensor
// core works on chunk j+1.
template <int METRIC>
__global__ void __launch_bounds__(160, 1) k_fes_scores_tma(FesParams p) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int t = blockIdx.x;
    if (t >= p.toff[p.r]) return;
    int c = 0;
    while (c + 1 < p.r && p.toff[c + 1] <= t) ++c;
    const int pos0 = p.qoff[c] + (t - p.toff[c]) * kM;
    const int nrows = min(kM, p.qoff[c + 1] - pos0);
    const int pb = p.cell_off[c], nc = p.cell_off[c + 1] - pb;
    const int kch = p.kchunks;
    const int nchunk = (nc + kN - 1) / kN;
    const int S = nchunk * kch;
    const float* img = p.pool_img + (size_t)p.chunk_off[c] * kch * 2 * 4096;

    unsigned char* a_hi = smem;                               // kch × 16 KB
    unsigned char* a_lo = a_hi + kch * 16384;
    unsigned char* bst = a_lo + kch * 16384;                  // 2 stages × (hi 16 KB | lo 16 KB)
    uint64_t* full = reinterpret_cast<uint64_t*>(bst + 2 * 32768);
    uint64_t* empty = full + 2;
    uint64_t* accf = empty + 2;
    uint64_t* acce = accf + 2;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(acce + 2);
    float* nrm = reinterpret_cast<float*>(tslot + 4);        // 4 warps × 32 pool norms (unfolded L2)
    float* stg = nrm + 128;                                   // 4 warps × 32 × 36 floats: store staging

    if (warp == 0) tmem_alloc(tslot, 2 * kN);
    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, 1);
            mbar_init(accf + i, 1);
            mbar_init(acce + i, kThreads);
        }
    }
    if (warp < 4) {                                           // A: routed [q', 1] rows, hi/lo, swizzled
        const int q = tid < nrows ? p.perm[pos0 + tid] : -1;
        for (int kc = 0; kc < kch; ++kc) {
#pragma unroll 8
            for (int k = 0; k < 32; ++k) {
                const int col = kc * 32 + k;
                const float a = q < 0 ? 0.f
                              : col < p.dps ? __ldg(p.qp + (int64_t)q * p.dps + col)
                              : (METRIC == 0 && p.fold_norm && col == p.dps ? 1.f : 0.f);
                float hi, lo;
                split_tf32(a, hi, lo);
                const uint32_t off = (uint32_t)kc * 16384 + sw128_off(tid, k);
                *reinterpret_cast<float*>(a_hi + off) = hi;
                *reinterpret_cast<float*>(a_lo + off) = lo;
            }
        }
        fence_proxy_async();
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == 4) {
        if (lane == 0) {
            const uint32_t idesc = make_idesc_tf32(kM, kN);
            auto issue = [&](int s) {
                const int st = s & 1;
                unsigned char* dst = bst + st * 32768;
                const float* src = img + (size_t)s * 2 * 4096;          // step s = (chunk s/kch, kc s%kch)
                mbar_expect_tx(full + st, 32768);
                tma_bulk_g2s(dst, src, 16384, full + st);
                tma_bulk_g2s(dst + 16384, src + 4096, 16384, full + st);
            };
            for (int s = 0; s < S && s < 2; ++s) issue(s);
            for (int s = 0; s < S; ++s) {
                const int st = s & 1, j = s / kch, kc = s % kch, acc = j & 1;
                if (kc == 0 && j >= 2) mbar_wait(acce + acc, ((j >> 1) - 1) & 1);
                mbar_wait(full + st, (s >> 1) & 1);
                tmem_fence_after();
                const uint32_t sah = smem_u32(a_hi) + kc * 16384, sal = smem_u32(a_lo) + kc * 16384;
                const uint32_t sbh = smem_u32(bst + st * 32768), sbl = sbh + 16384;
                const uint32_t td = tmem + (uint32_t)(acc * kN);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint32_t ko = kk * 32;
                    const uint32_t acc0 = (kc > 0 || kk > 0) ? 1u : 0u;
                    mma_tf32(td, make_desc_sw128(sah + ko), make_desc_sw128(sbh + ko), idesc, acc0);
                    mma_tf32(td, make_desc_sw128(sah + ko), make_desc_sw128(sbl + ko), idesc, 1u);
                    mma_tf32(td, make_desc_sw128(sal + ko), make_desc_sw128(sbh + ko), idesc, 1u);
                }
                mma_commit(empty + st);
                if (kc == kch - 1) mma_commit(accf + acc);
                if (s + 2 < S) {
                    mbar_wait(empty + st, (s >> 1) & 1);
                    issue(s + 2);
                }
            }
        }
        __syncwarp();
    } else {
        // Epilogue: thread t holds row t of each 32-column block (tcgen05.ld); the
        // block goes through smem so that every global store instruction writes
        // whole 128-B lines of 4 rows instead of 16 B of 32 rows.
        float* tile = stg + warp * (32 * 36);                 // 32 rows × 32 floats, row stride 36
        for (int j = 0; j < nchunk; ++j) {
            const int acc = j & 1;
            mbar_wait(accf + acc, (j >> 1) & 1);
            tmem_fence_after();
            for (int c0 = 0; c0 < kN; c0 += 32) {
                float v[32];
                tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(acc * kN + c0), v);
                const int jb = j * kN + c0;
                if (jb >= nc) continue;                        // warp-uniform
                float* nb = nrm + warp * 32;                   // unfolded L2: score = ‖e‖² + acc (acc = −2q'·e)
                __syncwarp();
                if (METRIC == 0 && !p.fold_norm) {
                    nb[lane] = jb + lane < nc ? __ldg(p.pool_norm + pb + jb + lane) : 0.f;
                    __syncwarp();
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj) v[jj] += nb[jj];
                }                                              // otherwise the accumulator IS the score
#pragma unroll
                for (int jj = 0; jj < 32; jj += 4)
                    *reinterpret_cast<float4*>(tile + lane * 36 + jj) = make_float4(v[jj], v[jj + 1], v[jj + 2], v[jj + 3]);
                __syncwarp();
                const int cc = (lane & 7) * 4;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int rl = i * 4 + (lane >> 3), rg = warp * 32 + rl;
                    if (rg < nrows && jb + cc < nc)
                        *reinterpret_cast<float4*>(p.scores + (int64_t)(pos0 + rg) * p.sstride + jb + cc) =
                            *reinterpret_cast<const float4*>(tile + rl * 36 + cc);
                }
            }
            tmem_fence_before();
            mbar_arrive(acce + acc);
        }
    }
    tmem_fence_before();
    __syncthreads();
    if (warp == 0) {
        tmem_fence_after();
        tmem_dealloc(tmem, 2 * kN);
    }
}

size_t fes_scores_tma_smem(int kch) {
    return (size_t)kch * 2 * 16384 + 2 * 32768 + 8 * 8 + 16 + 512 + 4 * 32 * 36 * 4;
}


// Selection (a4, the top-E of Alg 2's within-cell scores): one warp
// per routed query, a radix select on the orderable 32-bit images of the scores.
//   1. the row's words (ord of the GEMM-form score) are read once as float4 —
//      into a per-warp smem stage when the largest cell fits (STAGE), otherwise
//      re-read from L2 per pass — and the warp AND/OR give the common prefix;
//   2. radix passes of ≤ 8 bits below that prefix: a 256-bin smem histogram of
//      the in-range words, a warp scan finds the bin holding the E-th smallest;
//      stop as soon as every word up to the end of that bin is ≤ kSelMax = 256
//      words (≥ E by construction), i.e. T = the bin's last word;
//   3. the ≤ 256 words ≤ T become (score, pool id) keys and are bitonic-sorted in
//      registers; the first E are the entries.  All words of one value fall in
//      one bin, so ties are resolved by the key order (δ, id) exactly as the
//      oracle's O4.  A row whose E-th value is shared by more than ~256 words
//      (heavy ties; the integer fixtures) takes the threshold + rank-merge loop.
// Per query: 1 row read + ≤ 4 histogram passes over nc/32 words per lane + one
// ≤ 256-key sort, instead of the previous two-pass bound + smem sort of up to
// 512 keys (which dominated at E = 224, C2: 477 µs → see DESIGN §7).
constexpr int kSelMax = 256;          // keys sorted in registers (E ≤ 256)
constexpr int kSelWarps = 4;
#ifndef PA_SEL_STAGE_MAX
#define PA_SEL_STAGE_MAX 2048         // largest cell whose words are staged in smem (8 KB per warp)
#endif

// Ascending bitonic sort of n = 32·K 64-bit keys held in registers, element
// i = a·32 + lane in t[a]: partners at distance ≥ 32 are in the same lane.
template <int K>
__device__ __forceinline__ void warp_bitonic_regs(uint64_t (&t)[K], int lane) {
#pragma unroll
    for (int k = 2; k <= 32 * K; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
#pragma unroll
                for (int a = 0; a < K; ++a) {
                    const int b = a ^ (j >> 5);
                    if (b > a) {
                        const bool up = ((a * 32 + lane) & k) == 0;
                        const uint64_t x = t[a], y = t[b];
                        if ((x > y) == up) { t[a] = y; t[b] = x; }
                    }
                }
            } else {
#pragma unroll
                for (int a = 0; a < K; ++a) {
                    const uint64_t y = shfl_xor64(t[a], j);
                    const bool up = ((a * 32 + lane) & k) == 0;
                    const bool lower = (lane & j) == 0;
                    const uint64_t mn = t[a] < y ? t[a] : y, mx = t[a] < y ? y : t[a];
                    t[a] = (lower == up) ? mn : mx;
                }
            }
        }
    }
}

// per-warp smem: histogram [256] u32, key buffer [256] u64, compaction counter,
// then (STAGE) the row's words [wcap] u32.
__host__ __device__ constexpr size_t sel_warp_bytes(int wcap) {
    return 256 * 4 + kSelMax * 8 + 16 + (size_t)wcap * 4;
}

template <bool STAGE>
#ifndef PA_SEL_MINB
#define PA_SEL_MINB 8                  // min resident blocks per SM of k_fes_select: 64 registers, no spills (C2 A/B: select 0.28 -> 0.20 ms)
#endif
__global__ void __launch_bounds__(kSelWarps * 32, PA_SEL_MINB) k_fes_select(FesParams p, int64_t m, int wcap) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int E = p.E;
    unsigned char* base = smem_raw + (size_t)w * sel_warp_bytes(STAGE ? wcap : 0);
    uint32_t* hist = reinterpret_cast<uint32_t*>(base);
    uint64_t* keys = reinterpret_cast<uint64_t*>(base + 1024);
    int* cnt = reinterpret_cast<int*>(base + 1024 + kSelMax * 8);
    uint32_t* words = reinterpret_cast<uint32_t*>(base + 1024 + kSelMax * 8 + 16);
    const int64_t nwarps = (int64_t)gridDim.x * kSelWarps;
    for (int64_t pos = (int64_t)blockIdx.x * kSelWarps + w; pos < m; pos += nwarps) {
        int c = 0;
        for (int c0 = 1; c0 < p.r; c0 += 32) {
            const int cc = c0 + lane;
            c += __popc(__ballot_sync(kFull, cc < p.r && __ldg(p.qoff + cc) <= pos));
        }
        const int pb = __ldg(p.cell_off + c), nc = __ldg(p.cell_off + c + 1) - pb;
        const float4* srow4 = reinterpret_cast<const float4*>(p.scores + pos * p.sstride);
        const int32_t* prow = p.pool_ids + pb;
        const int32_t q = __ldg(p.perm + pos);
        const int n4 = (nc + 3) >> 2;
        // words of chunk i4 (4 consecutive entries); entries past the cell → all-ones,
        // never selected (every selected word is ≤ T < 0xffffffff or the index is checked)
        auto gload4 = [&](int i4) -> uint4 {
            const float4 v = srow4[i4];
            uint4 r;
            r.x = ord_of(v.x);
            r.y = i4 * 4 + 1 < nc ? ord_of(v.y) : 0xffffffffu;
            r.z = i4 * 4 + 2 < nc ? ord_of(v.z) : 0xffffffffu;
            r.w = i4 * 4 + 3 < nc ? ord_of(v.w) : 0xffffffffu;
            return r;
        };
        auto get4 = [&](int i4) -> uint4 {
            if constexpr (STAGE) return reinterpret_cast<const uint4*>(words)[i4];
            else return gload4(i4);
        };
        // ---- 1. read the row once (8 float4 loads in flight per lane), common prefix
        uint32_t wand = 0xffffffffu, wor = 0u;
        for (int t0 = 0; t0 * 32 < n4; t0 += 8) {
            uint4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i4 = (t0 + u) * 32 + lane;
                v[u] = i4 < n4 ? gload4(i4) : make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i4 = (t0 + u) * 32 + lane;
                if (i4 < n4) {
                    if constexpr (STAGE) reinterpret_cast<uint4*>(words)[i4] = v[u];
                    const uint32_t x[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (i4 * 4 + k < nc) { wand &= x[k]; wor |= x[k]; }
                }
            }
        }
        wand = __reduce_and_sync(kFull, wand);
        wor = __reduce_or_sync(kFull, wor);
        // ---- 2. threshold T: count(words ≤ T) in [min(nc, E), kSelMax]
        uint32_t T = 0xfffffffeu;                       // nc ≤ kSelMax: every entry
        bool ties = false;
        if (nc > kSelMax) {
            int nbits = 32 - __clz(wand ^ wor);         // bits below the common prefix
            uint32_t prefix = wand;                     // bits ≥ nbits are fixed
            int below = 0;                              // words < the current range
            if (nbits == 0) ties = true;                // every word equal (nc > 256 ties)
            while (!ties) {
                const int s = nbits > 8 ? nbits - 8 : 0;
                const uint32_t dmask = (1u << (nbits - s)) - 1u;
#pragma unroll
                for (int i = 0; i < 8; ++i) hist[lane * 8 + i] = 0;
                __syncwarp();
                for (int i4 = lane; i4 < n4; i4 += 32) {
                    const uint4 v = get4(i4);
                    const uint32_t x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (i4 * 4 + k < nc && (nbits == 32 || (x[k] >> nbits) == (prefix >> nbits)))
                            atomicAdd(&hist[(x[k] >> s) & dmask], 1u);
                }
                __syncwarp();
                uint32_t h[8], sum = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) { h[i] = hist[lane * 8 + i]; sum += h[i]; }
                uint32_t incl = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += y;
                }
                // the lane whose 8 bins hold the E-th smallest word
                const unsigned hit = __ballot_sync(kFull, below + (int)(incl - sum) < E && below + (int)incl >= E);
                const int src = __ffs(hit) - 1;
                int bin = 0, before = 0, inbin = 0;
                if (lane == src) {
                    int run = below + (int)(incl - sum);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        if (run < E && run + (int)h[i] >= E && inbin == 0) { bin = lane * 8 + i; before = run; inbin = (int)h[i]; }
                        run += (int)h[i];
                    }
                }
                bin = __shfl_sync(kFull, bin, src);
                before = __shfl_sync(kFull, before, src);
                inbin = __shfl_sync(kFull, inbin, src);
                const uint32_t pre = (nbits == 32 ? 0u : (prefix >> nbits) << nbits) | ((uint32_t)bin << s);
                if (before + inbin <= kSelMax) {       // every word ≤ the bin's last word
                    T = pre | ((1u << s) - 1u);
                    break;
                }
                if (s == 0) { ties = true; break; }     // > 256 words share the E-th value
                prefix = pre;
                below = before;
                nbits = s;
                __syncwarp();
            }
        }
        if (!ties) {
            // ---- 3. compact the ≤ 256 words ≤ T as (δ, id) keys, sort, emit the first E
            if (lane == 0) *cnt = 0;
            __syncwarp();
            for (int i4 = lane; i4 < n4; i4 += 32) {
                const uint4 v = get4(i4);
                const uint32_t x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int e = i4 * 4 + k;
                    if (e < nc && x[k] <= T) {
                        const int at = atomicAdd(cnt, 1);
                        keys[at] = ((uint64_t)x[k] << 32) | ((uint64_t)(uint32_t)__ldg(prow + e) << 1);
                    }
                }
            }
            __syncwarp();
            const int M = *cnt;
            auto sort_regs = [&](auto tag) {
                constexpr int K = decltype(tag)::value;
                uint64_t tk[K];
#pragma unroll
                for (int a = 0; a < K; ++a) tk[a] = a * 32 + lane < M ? keys[a * 32 + lane] : kKeyInf;
                warp_bitonic_regs<K>(tk, lane);
#pragma unroll
                for (int a = 0; a < K; ++a) {
                    const int j = a * 32 + lane;
                    if (j < E) p.entries[(int64_t)q * E + j] = j < M ? key_id(tk[a]) : -1;
                }
                for (int j = 32 * K + lane; j < E; j += 32) p.entries[(int64_t)q * E + j] = -1;
            };
            if (M <= 32) sort_regs(std::integral_constant<int, 1>{});
            else if (M <= 64) sort_regs(std::integral_constant<int, 2>{});
            else if (M <= 128) sort_regs(std::integral_constant<int, 4>{});
            else sort_regs(std::integral_constant<int, 8>{});
        } else {                                        // heavy ties: threshold + rank merge
            uint64_t* C = keys;
            int csz = 0;
            for (int j0 = 0; j0 < nc; j0 += 32) {
                const int j = j0 + lane;
                const uint64_t key = j < nc ? make_key(p.scores[pos * p.sstride + j], __ldg(prow + j)) : kKeyInf;
                const uint64_t thresh = csz == E ? C[E - 1] : kKeyInf;
                const bool pass = key < thresh;
                const unsigned pbal = __ballot_sync(kFull, pass);
                if (pbal == 0) continue;
                int minr;
                csz = rank_merge<8>(C, csz, E, key, pass, pbal, lane, minr);
            }
            for (int j = lane; j < E; j += 32) p.entries[(int64_t)q * E + j] = j < csz ? key_id(C[j]) : -1;
        }
        __syncwarp();
    }
}

size_t fes_scores_smem(int kch) { return fes_scores_tma_smem(kch); }

}  // namespace

bool fes_tc_supported(const DevIndex& ix, int E) {
    const int kch = (ix.rdim_pad + 31) / 32;
    return ix.pool_norm != nullptr && ix.fes_r <= kMaxR && E <= 256 && fes_scores_smem(kch) <= 227 * 1024;
}

size_t fes_tc_scratch_floats(const DevIndex& ix, int64_t m) {
    return (size_t)m * (size_t)ix.max_cell;
}

int launch_fes_tc(const DevIndex& ix, const SearchArgs& a, cudaStream_t s) {
    if (a.m == 0) return 0;
    k_bucket<<<1, 1024, 0, s>>>(a.cell, a.m, ix.fes_r, kM, a.perm, a.qoff, a.toff);
    FesParams p;
    p.qp = a.qp; p.dps = ix.rdim_pad; p.kchunks = (ix.rdim_pad + 31) / 32;
    p.perm = a.perm; p.qoff = a.qoff; p.toff = a.toff; p.r = ix.fes_r;
    p.pool_vec = ix.pool_vec; p.pool_norm = ix.pool_norm; p.pool_ids = ix.pool_ids; p.cell_off = ix.cell_off;
    p.metric = ix.metric; p.scores = a.fes_scores; p.sstride = ix.max_cell; p.E = a.E; p.entries = a.entries;
    p.pool_img = ix.pool_img; p.chunk_off = ix.chunk_off; p.fold_norm = ix.fes_fold_norm;
    const unsigned grid = (unsigned)((a.m + kM - 1) / kM + ix.fes_r);
    void* args[] = {&p};
    {
        const size_t smem = fes_scores_tma_smem(p.kchunks);
        void* fn = ix.metric == 0 ? (void*)k_fes_scores_tma<0> : (void*)k_fes_scores_tma<1>;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaLaunchKernel(fn, dim3(grid), dim3(160), args, smem, s);
    }
    // selection: the row's words staged in smem when the largest cell fits
    // PA_SEL_STAGE_MAX entries (occupancy vs re-reading the row from L2 per pass)
    const bool stage = ix.max_cell <= PA_SEL_STAGE_MAX;
    const int wcap = stage ? (ix.max_cell + 3) / 4 * 4 : 0;
    void* sel = stage ? (void*)k_fes_select<true> : (void*)k_fes_select<false>;
    const size_t ssm = (size_t)kSelWarps * sel_warp_bytes(wcap);
    cudaFuncSetAttribute(sel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
    int64_t m = a.m;
    int wc = wcap;
    void* args2[] = {&p, &m, &wc};
    cudaLaunchKernel(sel, dim3((unsigned)((a.m + kSelWarps - 1) / kSelWarps)), dim3(kSelWarps * 32), args2, ssm, s);
    return 3;
}

}  // namespace pa
