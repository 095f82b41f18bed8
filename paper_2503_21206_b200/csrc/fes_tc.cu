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
//   k_fes_select4 / k_fes_select3 (cells > 8192 entries) : one warp per query keeps the E smallest (score, id) keys
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


// Selection, two passes (far fewer instructions than merging every passing key):
//   1. every lane keeps the KP = ceil(E/32) smallest keys of its strided share in
//      registers; a bitwise search over the high (distance) words of those 32·KP
//      candidates gives T = the distance word of their E-th smallest — a bound ≥
//      the true E-th smallest distance of the row;
//   2. all keys with distance word ≤ T (the true top-E and typically a few more)
//      are compacted into a per-warp smem buffer and bitonic-sorted once; the
//      first E are the entries.  A row with more than kSelCap candidates (heavy
//      ties) falls back to the threshold + rank-merge loop.
constexpr int kSelCap = 512;

__device__ __forceinline__ void warp_bitonic_smem(uint64_t* a, int n, int lane) {
    for (int k = 2; k <= n; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < n; i += 32) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const uint64_t x = a[i], y = a[ixj];
                    const bool up = (i & k) == 0;
                    if ((x > y) == up) { a[i] = y; a[ixj] = x; }
                }
            }
            __syncwarp();
        }
}

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


// Same two-pass selection, latency-restructured (one warp per query):
//   * the routed cell is found lane-parallel (one ballot over qoff per 32 cells),
//   * pass 1 reads the row as float4 with NV loads in flight per lane and keeps
//     per-lane KP smallest 32-bit distance words only (ids are not needed to bound
//     the E-th smallest distance),
//   * pass 2 re-reads the row (L2), counts the words ≤ T per lane, places them by a
//     warp prefix sum and loads the pool ids of the selected entries only,
//   * ≤ 128 candidates are sorted in registers; larger sets take the smem sort,
//     more than kSelCap (heavy ties) the rank-merge fallback.
// Keys and hence entries are identical to k_fes_select4's.
#ifndef PA_SEL_MINB
#define PA_SEL_MINB 6
#endif
#ifndef PA_SEL_NV
#define PA_SEL_NV 8
#endif
template <int KPMAX, int SMAX, int NV>
__global__ void __launch_bounds__(128, PA_SEL_MINB) k_fes_select3(FesParams p, int64_t m) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // 2·ceil(E/32) words per lane: a lane rarely holds more of the row's E smallest
    // than that, so T is close to the true E-th smallest word and ≤ 128 keys pass
    const int E = p.E, KP = min(KPMAX, 2 * ((E + 31) / 32));
    uint64_t* buf = reinterpret_cast<uint64_t*>(smem_raw) + (size_t)w * kSelCap;
    const int64_t nwarps = (int64_t)gridDim.x * 4;
    for (int64_t pos = (int64_t)blockIdx.x * 4 + w; pos < m; pos += nwarps) {
        int c = 0;                                        // #cells cc in [1, r) starting at or before pos
        for (int c0 = 1; c0 < p.r; c0 += 32) {
            const int cc = c0 + lane;
            c += __popc(__ballot_sync(kFull, cc < p.r && __ldg(p.qoff + cc) <= pos));
        }
        const int pb = __ldg(p.cell_off + c), nc = __ldg(p.cell_off + c + 1) - pb;
        const float4* srow4 = reinterpret_cast<const float4*>(p.scores + pos * p.sstride);
        const int32_t* prow = p.pool_ids + pb;
        const int32_t q = __ldg(p.perm + pos);
        const int n4 = (nc + 3) >> 2;
        // ---- pass 1: per-lane KP smallest distance words
        uint32_t t[KPMAX];
#pragma unroll
        for (int i = 0; i < KPMAX; ++i) t[i] = 0xffffffffu;
        for (int i0 = 0; i0 < n4; i0 += 32 * NV) {
            float4 v[NV];
#pragma unroll
            for (int u = 0; u < NV; ++u) {
                const int i4 = i0 + u * 32 + lane;
                v[u] = i4 < n4 ? srow4[i4] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < NV; ++u) {
                const int e0 = (i0 + u * 32 + lane) * 4;
                const float f[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (e0 + k >= nc) continue;
                    uint32_t x = ord_of(f[k]);
                    if (x < t[KP - 1]) {
#pragma unroll
                        for (int i = 0; i < KPMAX; ++i)
                            if (i < KP && x < t[i]) { const uint32_t y = t[i]; t[i] = x; x = y; }
                    }
                }
            }
        }
        uint32_t T = 0xffffffffu;
        if (nc > E) {
            uint32_t lo = 0;                              // largest T with count(< T) < E
            for (int b = 31; b >= 0; --b) {
                const uint32_t trial = lo | (1u << b);
                int cnt = 0;
#pragma unroll
                for (int i = 0; i < KPMAX; ++i) cnt += (i < KP && t[i] < trial) ? 1 : 0;
                cnt = (int)__reduce_add_sync(kFull, (unsigned)cnt);
                if (cnt < E) lo = trial;
            }
            T = lo;
        }
        // ---- pass 2: compact every key with distance word ≤ T
        int M = 0;
        bool overflow = false;
        for (int i0 = 0; i0 < n4 && !overflow; i0 += 32 * NV) {
            float4 v[NV];
#pragma unroll
            for (int u = 0; u < NV; ++u) {
                const int i4 = i0 + u * 32 + lane;
                v[u] = i4 < n4 ? srow4[i4] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            uint32_t sel = 0;                             // bit u*4+k: element selected
            int cnt = 0;
#pragma unroll
            for (int u = 0; u < NV; ++u) {
                const int e0 = (i0 + u * 32 + lane) * 4;
                const float f[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const bool in = e0 + k < nc && ord_of(f[k]) <= T;
                    sel |= in ? (1u << (u * 4 + k)) : 0u;
                    cnt += in ? 1 : 0;
                }
            }
            int incl = cnt;                               // warp inclusive prefix sum of the counts
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += y;
            }
            const int total = __shfl_sync(kFull, incl, 31);
            if (M + total > kSelCap) { overflow = true; break; }
            int at = M + incl - cnt;
#pragma unroll
            for (int u = 0; u < NV; ++u) {
                const int e0 = (i0 + u * 32 + lane) * 4;
                const float f[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (sel & (1u << (u * 4 + k))) buf[at++] = make_key(f[k], __ldg(prow + e0 + k));
            }
            M += total;
        }
        __syncwarp();
        if (!overflow && M <= 128) {
            uint64_t t4[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) t4[a] = a * 32 + lane < M ? buf[a * 32 + lane] : kKeyInf;
            warp_bitonic_regs<4>(t4, lane);
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int j = a * 32 + lane;
                if (j < E) p.entries[(int64_t)q * E + j] = j < M ? key_id(t4[a]) : -1;
            }
            for (int j = 128 + lane; j < E; j += 32) p.entries[(int64_t)q * E + j] = -1;
        } else if (!overflow) {
            int n2 = 32;
            while (n2 < M) n2 <<= 1;
            for (int i = M + lane; i < n2; i += 32) buf[i] = kKeyInf;
            __syncwarp();
            warp_bitonic_smem(buf, n2, lane);
            for (int j = lane; j < E; j += 32) p.entries[(int64_t)q * E + j] = j < M ? key_id(buf[j]) : -1;
        } else {                                          // heavy ties: threshold + rank merge
            uint64_t* C = buf;
            int csz = 0;
            const float* srow = p.scores + pos * p.sstride;
            for (int j0 = 0; j0 < nc; j0 += 32) {
                const int j = j0 + lane;
                const uint64_t key = j < nc ? make_key(srow[j], __ldg(prow + j)) : kKeyInf;
                const uint64_t thresh = csz == E ? C[E - 1] : kKeyInf;
                const bool pass = key < thresh;
                const unsigned pbal = __ballot_sync(kFull, pass);
                if (pbal == 0) continue;
                int minr;
                csz = rank_merge<SMAX>(C, csz, E, key, pass, pbal, lane, minr);
            }
            for (int j = lane; j < E; j += 32) p.entries[(int64_t)q * E + j] = j < csz ? key_id(C[j]) : -1;
        }
        __syncwarp();
    }
}

// Selection with ~3× fewer instructions than k_fes_select3 (one warp per query):
//   pass 1: lane l reads float4 chunks t·32 + l of the row (t < 16·G, all of a
//           round's 8 loads in flight) and keeps the minimum distance word of each
//           group of G consecutive chunks of its own → ≤ 16 group minima per lane
//           (512 per warp, each an actual entry);
//   T     : a bitwise search over bits 31..8 of those minima for the smallest
//           24-bit prefix with ≥ E minima at or below it, low byte filled — at
//           least E entries have a word ≤ T, so the E smallest keys all do;
//   pass 2: every entry with word ≤ T is placed by a warp prefix sum as its index,
//           keys (score, pool id) are built for the ≤ kSelCap selected only, and
//           ≤ 128 are sorted in registers (smem sort / rank merge fallbacks).
// With 4-entry groups ~E·1.1 entries pass (vs > 128 for per-lane top-KP lists of
// words, which the previous selections sorted in smem).  Entries are identical.
template <int SMAX, int G>
__global__ void __launch_bounds__(128, 4) k_fes_select4(FesParams p, int64_t m) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int E = p.E;
    constexpr int NT = 16 * G;                            // float4 chunks per lane (nc ≤ 2048·G)
    uint64_t* buf = reinterpret_cast<uint64_t*>(smem_raw) + (size_t)w * kSelCap;
    const int64_t nwarps = (int64_t)gridDim.x * 4;
    for (int64_t pos = (int64_t)blockIdx.x * 4 + w; pos < m; pos += nwarps) {
        int c = 0;
        for (int c0 = 1; c0 < p.r; c0 += 32) {
            const int cc = c0 + lane;
            c += __popc(__ballot_sync(kFull, cc < p.r && __ldg(p.qoff + cc) <= pos));
        }
        const int pb = __ldg(p.cell_off + c), nc = __ldg(p.cell_off + c + 1) - pb;
        const float* srow = p.scores + pos * p.sstride;
        const float4* srow4 = reinterpret_cast<const float4*>(srow);
        const int32_t* prow = p.pool_ids + pb;
        const int32_t q = __ldg(p.perm + pos);
        const int n4 = (nc + 3) >> 2;
        auto word4 = [&](const float4 v, int i4, uint32_t (&wd)[4]) {
            const float f[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) wd[k] = (i4 * 4 + k < nc) ? ord_of(f[k]) : 0xffffffffu;
        };
        // ---- pass 1: group minima (fminf on the scores, ordered word of the minimum only)
        const float kInf = __int_as_float(0x7f800000);
        float fm[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) fm[i] = kInf;
#pragma unroll
        for (int t0 = 0; t0 < NT; t0 += 8) {
            if (t0 * 32 >= n4) break;                      // warp-uniform
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i4 = (t0 + u) * 32 + lane;
                v[u] = i4 < n4 ? srow4[i4] : make_float4(kInf, kInf, kInf, kInf);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i4 = (t0 + u) * 32 + lane;
                float4 x = v[u];
                if (i4 * 4 + 3 >= nc) {                    // ragged tail of the cell
                    if (i4 * 4 + 1 >= nc) x.y = kInf;
                    if (i4 * 4 + 2 >= nc) x.z = kInf;
                    if (i4 * 4 + 3 >= nc) x.w = kInf;
                }
                fm[(t0 + u) / G] = fminf(fm[(t0 + u) / G], fminf(fminf(x.x, x.y), fminf(x.z, x.w)));
            }
        }
        uint32_t mn[16];                                   // ord is monotone: ord(min) = min(ord)
#pragma unroll
        for (int i = 0; i < 16; ++i) mn[i] = ord_of(fm[i]);
        uint32_t T = 0xffffffffu;
        if (nc > E) {
            uint32_t lo = 0;                              // largest prefix with count(< prefix) < E
            for (int b = 31; b >= 12; --b) {
                const uint32_t trial = lo | (1u << b);
                int cnt = 0;
#pragma unroll
                for (int i = 0; i < 16; ++i) cnt += mn[i] < trial ? 1 : 0;
                cnt = (int)__reduce_add_sync(kFull, (unsigned)cnt);
                if (cnt < E) lo = trial;
            }
            T = lo | 0xfffu;                              // count(minima ≤ T) ≥ E
        }
        // ---- pass 2: indices of the entries with word ≤ T, by warp prefix sums
        int M = 0;
        bool overflow = false;
#pragma unroll
        for (int t0 = 0; t0 < NT; t0 += 8) {
            if (t0 * 32 >= n4 || overflow) break;          // warp-uniform
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i4 = (t0 + u) * 32 + lane;
                v[u] = i4 < n4 ? srow4[i4] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            uint32_t sel = 0;
            int cnt = 0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i4 = (t0 + u) * 32 + lane;
                uint32_t wd[4];
                word4(v[u], i4, wd);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const bool in = wd[k] <= T && i4 * 4 + k < nc;
                    sel |= in ? (1u << (u * 4 + k)) : 0u;
                    cnt += in ? 1 : 0;
                }
            }
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += y;
            }
            const int total = __shfl_sync(kFull, incl, 31);
            if (M + total > kSelCap) { overflow = true; break; }
            int at = M + incl - cnt;
            while (sel) {                                 // this lane's selected entries (~E/32 per round)
                const int b = __ffs(sel) - 1;
                sel &= sel - 1;
                buf[at++] = (uint64_t)(((t0 + (b >> 2)) * 32 + lane) * 4 + (b & 3));
            }
            M += total;
        }
        __syncwarp();
        if (!overflow) {
            for (int i = lane; i < M; i += 32) {          // keys of the selected entries only
                const int e = (int)buf[i];
                buf[i] = make_key(__ldg(srow + e), __ldg(prow + e));
            }
            __syncwarp();
        }
        auto sort_regs = [&](auto tag) {
            constexpr int K = decltype(tag)::value;
            uint64_t tk[K];
#pragma unroll
            for (int a = 0; a < K; ++a) tk[a] = a * 32 + lane < M ? buf[a * 32 + lane] : kKeyInf;
            warp_bitonic_regs<K>(tk, lane);
#pragma unroll
            for (int a = 0; a < K; ++a) {
                const int j = a * 32 + lane;
                if (j < E) p.entries[(int64_t)q * E + j] = j < M ? key_id(tk[a]) : -1;
            }
            for (int j = 32 * K + lane; j < E; j += 32) p.entries[(int64_t)q * E + j] = -1;
        };
        if (!overflow && M <= 128) {
            sort_regs(std::integral_constant<int, 4>{});
        } else if (!overflow && M <= 256) {
            sort_regs(std::integral_constant<int, 8>{});
        } else if (!overflow) {
            int n2 = 32;
            while (n2 < M) n2 <<= 1;
            for (int i = M + lane; i < n2; i += 32) buf[i] = kKeyInf;
            __syncwarp();
            warp_bitonic_smem(buf, n2, lane);
            for (int j = lane; j < E; j += 32) p.entries[(int64_t)q * E + j] = j < M ? key_id(buf[j]) : -1;
        } else {                                          // heavy ties: threshold + rank merge
            uint64_t* C = buf;
            int csz = 0;
            for (int j0 = 0; j0 < nc; j0 += 32) {
                const int j = j0 + lane;
                const uint64_t key = j < nc ? make_key(srow[j], __ldg(prow + j)) : kKeyInf;
                const uint64_t thresh = csz == E ? C[E - 1] : kKeyInf;
                const bool pass = key < thresh;
                const unsigned pbal = __ballot_sync(kFull, pass);
                if (pbal == 0) continue;
                int minr;
                csz = rank_merge<SMAX>(C, csz, E, key, pass, pbal, lane, minr);
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
    // selection: k_fes_select4 up to 8192-entry cells, k_fes_select3 above (same entries)
    void* sel;
    size_t ssm = (size_t)4 * kSelCap * 8;
    if (ix.max_cell <= 2048 * 4) {
        const int SM = a.E <= 64 ? 2 : a.E <= 128 ? 4 : 8;
        const int G = ix.max_cell <= 2048 ? 1 : ix.max_cell <= 4096 ? 2 : 4;
        void* t[3][3] = {{(void*)k_fes_select4<2, 1>, (void*)k_fes_select4<2, 2>, (void*)k_fes_select4<2, 4>},
                         {(void*)k_fes_select4<4, 1>, (void*)k_fes_select4<4, 2>, (void*)k_fes_select4<4, 4>},
                         {(void*)k_fes_select4<8, 1>, (void*)k_fes_select4<8, 2>, (void*)k_fes_select4<8, 4>}};
        sel = t[SM == 2 ? 0 : SM == 4 ? 1 : 2][G == 1 ? 0 : G == 2 ? 1 : 2];
    } else {
        constexpr int NV = PA_SEL_NV;
        sel = a.E <= 32 ? (void*)k_fes_select3<2, 2, NV> : a.E <= 64 ? (void*)k_fes_select3<4, 2, NV>
            : a.E <= 96 ? (void*)k_fes_select3<6, 4, NV> : a.E <= 128 ? (void*)k_fes_select3<8, 4, NV>
            : (void*)k_fes_select3<16, 8, NV>;
    }
    cudaFuncSetAttribute(sel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
    int64_t blocks = (a.m + 3) / 4;
    int64_t m = a.m;
    void* args2[] = {&p, &m};
    cudaLaunchKernel(sel, dim3((unsigned)blocks), dim3(128), args2, ssm, s);
    return 3;
}

}  // namespace pa
